"""tcgen05 fp16 GEMM (fq_gemm_tc.cu) against a float64 reference of the same
fp16-rounded operands. Tolerance: fp32 accumulation differences only, 1e-3
relative (the north_star's fp16 bar)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(gpu):
    import paper_2010_13887_b200 as pkg
    return pkg


def _ref(a16, b16, bias=None, act="none", res=None):
    import torch
    acc = a16.double() @ b16.double().T
    if bias is not None:
        acc = acc + bias.double()
    if act == "relu":
        acc = torch.relu(acc)
    elif act == "gelu":
        acc = torch.nn.functional.gelu(acc)
    if res is not None:
        acc = acc + res.double()
    return acc


def _rel(got, want):
    return float((got.double() - want).abs().max() / max(want.abs().max().item(), 1e-6))


@pytest.mark.parametrize("M,N,K", [
    (128, 64, 64), (1, 8, 16), (32, 512, 512), (100, 100, 72), (512, 1024, 1024),
    (512, 3072, 1024), (512, 1024, 4096), (300, 32000, 512), (8192, 3072, 1024),
    (2048, 4096, 1024), (512, 32000, 1024), (8192, 1024, 4096), (1000, 4000, 256)])
def test_tc_gemm_plain(P, M, N, K):
    import torch
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.float16)
    b = torch.randn(N, K, device="cuda", generator=g).to(torch.float16)
    out = torch.empty(M, N, device="cuda")
    P.gemm(a, b, out, transpose_b=True)
    torch.cuda.synchronize()
    assert _rel(out, _ref(a, b)) <= 1e-3, (M, N, K)


@pytest.mark.parametrize("act", ["none", "relu", "gelu"])
def test_tc_gemm_epilogue(P, act):
    import torch
    M, N, K = 384, 1536, 512
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.float16)
    b = torch.randn(N, K, device="cuda", generator=g).to(torch.float16)
    bias = torch.randn(N, device="cuda", generator=g)
    res = torch.randn(M, N, device="cuda", generator=g)
    out = torch.empty(M, N, device="cuda")
    P.gemm(a, b, out, transpose_b=True, bias=bias, activation=act, residual=res)
    assert _rel(out, _ref(a, b, bias, act, res)) <= 1e-3
    out16 = torch.empty(M, N, device="cuda", dtype=torch.float16)
    P.gemm(a, b, out16, transpose_b=True, bias=bias, activation=act)
    assert _rel(out16.float(), _ref(a, b, bias, act)) <= 8e-3  # fp16 output rounding


def test_tc_gemm_strided_output_and_accumulate(P):
    import torch
    M, N, K = 256, 256, 256
    a = torch.randn(M, K, device="cuda").to(torch.float16)
    b = torch.randn(N, K, device="cuda").to(torch.float16)
    big = torch.zeros(M, 2 * N, device="cuda")
    view = big[:, N:]
    view.fill_(1.0)
    P.gemm(a, b, view, transpose_b=True, accumulate=True)
    assert _rel(view, _ref(a, b) + 1.0) <= 1e-3
    assert float(big[:, :N].abs().max()) == 0.0


@pytest.mark.parametrize("M,N,K", [(512, 1024, 1024), (512, 1024, 4096), (300, 2048, 512),
                                   (128, 256, 1024), (512, 4096, 1024)])
def test_tc_gemm_all_plans(P, M, N, K):
    """Every schedule the dispatcher can pick — persistent tiles, multicast
    clusters (cm x cn) and split-K clusters reduced through DSMEM — computes
    the same GEMM (fused bias + ReLU + residual epilogue included)."""
    import ctypes
    import torch
    from paper_2010_13887_b200 import _abi
    lib = _abi.load()
    lib.fq_gemm_force_plan.argtypes = [ctypes.c_int] * 4
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.float16)
    b = torch.randn(N, K, device="cuda", generator=g).to(torch.float16)
    bias = torch.randn(N, device="cuda", generator=g)
    res = torch.randn(M, N, device="cuda", generator=g)
    want = _ref(a, b, bias, "relu", res)
    plans = [(64, 1, 1, 1), (128, 2, 1, 1), (128, 1, 2, 1), (32, 2, 4, 1), (256, 1, 1, 1)]
    plans += [(bn, 1, 1, s) for bn in (64, 128, 256) for s in (2, 3, 4, 8)]
    tried = 0
    try:
        for plan in plans:
            lib.fq_gemm_force_plan(*plan)
            out = torch.full((M, N), float("nan"), device="cuda")
            P.gemm(a, b, out, transpose_b=True, bias=bias, activation="relu", residual=res)
            torch.cuda.synchronize()
            assert _rel(out, want) <= 1e-3, plan
            tried += 1
    finally:
        lib.fq_gemm_force_plan(0, 0, 0, 1)
    assert tried == len(plans)


@pytest.mark.parametrize("M,N,K", [(8192, 3072, 1024), (512, 32000, 1024)])
def test_tc_gemm_wide_tile_epilogue(P, M, N, K):
    """Tile widths 192/224 (wave-quantisation plan) with the fused epilogue."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(N + K)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.float16)
    b = torch.randn(N, K, device="cuda", generator=g).to(torch.float16)
    bias = torch.randn(N, device="cuda", generator=g)
    res = torch.randn(M, N, device="cuda", generator=g)
    out = torch.empty(M, N, device="cuda")
    P.gemm(a, b, out, transpose_b=True, bias=bias, activation="relu", residual=res)
    torch.cuda.synchronize()
    assert _rel(out, _ref(a, b, bias, "relu", res)) <= 1e-3


@pytest.mark.parametrize("M,N,K", [(512, 1024, 1024), (512, 1024, 4096), (128, 1024, 1024),
                                   (300, 1024, 1024), (512, 768, 1024)])
def test_gemm_ln_equals_gemm_then_layer_norm(M, N, K):
    """fq_gemm_ln (the LayerNorm inside the split-K epilogue, row-block
    statistics exchanged between the CTAs) against fq_gemm (bias + residual)
    followed by fq_layer_norm: fp32 and fp16 outputs, repeated launches (the
    counters reset themselves). N = 768 takes the unfused fallback."""
    import torch
    from paper_2010_13887_b200 import _abi
    import paper_2010_13887_b200 as P
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randn(M, K, device="cuda", generator=g).half()
    w = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).half()
    bias = torch.randn(N, device="cuda", generator=g) * 0.1
    res = torch.randn(M, N, device="cuda", generator=g)
    gam = torch.randn(N, device="cuda", generator=g)
    bet = torch.randn(N, device="cuda", generator=g) * 0.1
    pre = torch.empty(M, N, device="cuda")
    P.gemm(a, w, pre, transpose_b=True, bias=bias, residual=res)
    want = torch.empty(M, N, device="cuda")
    want16 = torch.empty(M, N, device="cuda", dtype=torch.float16)
    hs = _abi.stream_handle
    _abi.call("fq_layer_norm", pre.data_ptr(), N, gam.data_ptr(), bet.data_ptr(), 1e-5, M, N,
              want.data_ptr(), N, want16.data_ptr(), N, hs())
    wsb = M * ((N + 127) // 128) * 16 + ((M + 127) // 128) * 8
    ws = torch.zeros((wsb + 15) // 16 * 4, dtype=torch.int32, device="cuda")
    for _ in range(3):
        out = torch.full((M, N), float("nan"), device="cuda")
        out16 = torch.empty(M, N, device="cuda", dtype=torch.float16)
        _abi.call("fq_gemm_ln", a.data_ptr(), K, w.data_ptr(), K, bias.data_ptr(), res.data_ptr(),
                  N, gam.data_ptr(), bet.data_ptr(), 1e-5, out.data_ptr(), N, out16.data_ptr(), N,
                  ws.data_ptr(), ws.numel() * 4, M, N, K, hs())
        torch.cuda.synchronize()
        assert float((out - want).abs().max()) <= 1e-5 * float(want.abs().max())
        assert int((out16.float() != want16.float()).sum()) <= M * N // 1000
    # counters back to zero
    nst = M * ((N + 127) // 128) * 4
    assert int(ws[nst:nst + ((M + 127) // 128) * 2].abs().sum()) == 0


@pytest.mark.parametrize("M,N,K", [(512, 1024, 1024), (512, 1024, 4096), (300, 1024, 1024),
                                   (128, 512, 2048), (512, 768, 1024)])
def test_gemm_ln_slab_path_bit_identical(M, N, K):
    """fq_gemm_ln with a workspace large enough for the split-K partial slabs:
    the GEMM writes one fp32 slab per K slice, fq_splitk_bias_residual_layer_norm
    sums them in split order — bit-identical to fq_gemm (in-kernel DSMEM
    reduction + bias + residual) followed by fq_layer_norm. N = 768 takes the
    unfused fallback."""
    import torch
    from paper_2010_13887_b200 import _abi
    import paper_2010_13887_b200 as P
    g = torch.Generator(device="cuda").manual_seed(7 * M + N + K)
    a = torch.randn(M, K, device="cuda", generator=g).half()
    w = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).half()
    bias = torch.randn(N, device="cuda", generator=g) * 0.1
    res = torch.randn(M, N, device="cuda", generator=g)
    gam = torch.randn(N, device="cuda", generator=g)
    bet = torch.randn(N, device="cuda", generator=g) * 0.1
    pre = torch.empty(M, N, device="cuda")
    P.gemm(a, w, pre, transpose_b=True, bias=bias, residual=res)
    want = torch.empty(M, N, device="cuda")
    want16 = torch.empty(M, N, device="cuda", dtype=torch.float16)
    hs = _abi.stream_handle
    _abi.call("fq_layer_norm", pre.data_ptr(), N, gam.data_ptr(), bet.data_ptr(), 1e-5, M, N,
              want.data_ptr(), N, want16.data_ptr(), N, hs())
    ws = torch.full((4 * M * N,), float("nan"), device="cuda")
    for _ in range(2):
        out = torch.full((M, N), float("nan"), device="cuda")
        out16 = torch.empty(M, N, device="cuda", dtype=torch.float16)
        _abi.call("fq_gemm_ln", a.data_ptr(), K, w.data_ptr(), K, bias.data_ptr(), res.data_ptr(),
                  N, gam.data_ptr(), bet.data_ptr(), 1e-5, out.data_ptr(), N, out16.data_ptr(), N,
                  ws.data_ptr(), ws.numel() * 4, M, N, K, hs())
        torch.cuda.synchronize()
        assert torch.equal(out, want)
        assert torch.equal(out16, want16)


@pytest.mark.parametrize("dt", ["f32", "fp16"])
@pytest.mark.parametrize("M,N,K,pad", [(200, 256, 256, 64), (512, 96, 512, 32), (77, 160, 128, 3)])
def test_tc_gemm_tma_store_strided_views(P, dt, M, N, K, pad):
    """The TMA-store epilogue writes through a tensor map with the output's
    leading dimension: a column slice of a wider buffer (ld = N + pad) gets
    exactly its M x N block, the padding columns stay untouched; pad = 3 makes
    the rows unaligned for TMA and takes the transposed-store path."""
    import torch
    dtype = torch.float32 if dt == "f32" else torch.float16
    g = torch.Generator(device="cuda").manual_seed(M + N + pad)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.float16)
    b = torch.randn(N, K, device="cuda", generator=g).to(torch.float16)
    bias = torch.randn(N, device="cuda", generator=g)
    big = torch.full((M, N + pad), 7.0, device="cuda", dtype=dtype)
    view = big[:, pad:]
    P.gemm(a, b, view, transpose_b=True, bias=bias, activation="relu")
    torch.cuda.synchronize()
    tol = 1e-3 if dt == "f32" else 8e-3
    assert _rel(view.float(), _ref(a, b, bias, "relu")) <= tol
    assert bool((big[:, :pad].float() == 7.0).all())


# ---------------------------------------------------------------------------
# exact fp32 mode on the tensor cores: 3xTF32 (fq_gemm_f32x3)

def _x3(P, a, b_nk, out, presplit=True, **kw):
    from paper_2010_13887_b200.model import X3Weight
    from paper_2010_13887_b200.tensor import gemm_x3
    if presplit:
        gemm_x3(a, X3Weight.from_kn(b_nk, transpose=False), out, **kw)
    else:  # raw fp32 K-major B through the reference's gemm API (split in smem)
        act = kw.pop("activation", "none")
        P.gemm(a, b_nk, out, transpose_b=True, activation=act, **kw)


@pytest.mark.parametrize("M,N,K", [
    (1, 8, 16), (100, 100, 72), (128, 64, 64), (512, 1024, 1024), (512, 3072, 1024),
    (512, 1024, 4096), (512, 4096, 1024), (300, 2000, 256), (512, 32000, 1024),
    (8192, 1024, 4096), (2048, 3072, 1024)])
def test_x3_gemm_matches_f64(P, M, N, K):
    """3xTF32 vs float64 on the same fp32 operands: fp32-GEMM accuracy, i.e.
    within 2x the error of an IEEE fp32 SGEMM (cuBLAS, TF32 off) of the same
    product, and <= 4e-6 of the output scale (the reference's own GEMM tests
    hold OpenBLAS to 1e-6 at K <= 64, test_tensor.py:51-58)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(M * 5 + N + K)
    a = torch.randn(M, K, device="cuda", generator=g)
    b = torch.randn(N, K, device="cuda", generator=g) * 0.03
    want = a.double() @ b.double().T
    scale = float(want.abs().max())
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    sgemm_err = float((a @ b.T).double().sub(want).abs().max()) / scale
    torch.backends.cuda.matmul.allow_tf32 = prev
    for presplit in (True, False):
        out = torch.empty(M, N, device="cuda")
        _x3(P, a, b, out, presplit=presplit)
        torch.cuda.synchronize()
        err = float((out.double() - want).abs().max()) / scale
        print(f"{M}x{N}x{K} presplit={presplit}: 3xTF32 {err:.2e}  fp32 SGEMM {sgemm_err:.2e}")
        assert err <= max(2 * sgemm_err, 5e-7) and err <= 1e-6, (M, N, K, presplit, err)
        if presplit:
            first = out.clone()
        else:  # in-kernel split == load-time split, bit for bit
            assert torch.equal(out, first)


@pytest.mark.parametrize("act", ["none", "relu", "gelu"])
def test_x3_gemm_epilogue_bits_vs_separate_ops(P, act):
    """The fused epilogue applies the reference's bias_residual_act semantics
    (kernels.py:39-53: fp32 bias add, act, fp32 residual add) to the 3xTF32
    accumulator: identical bits to the GEMM followed by fq_bias_residual_act."""
    import torch
    M, N, K = 384, 1536, 512
    g = torch.Generator(device="cuda").manual_seed(11)
    a = torch.randn(M, K, device="cuda", generator=g)
    b = torch.randn(N, K, device="cuda", generator=g) * 0.05
    bias = torch.randn(N, device="cuda", generator=g)
    res = torch.randn(M, N, device="cuda", generator=g)
    fused = torch.empty(M, N, device="cuda")
    _x3(P, a, b, fused, bias=bias, residual=res, activation=act)
    plain = torch.empty(M, N, device="cuda")
    _x3(P, a, b, plain)
    sep = P.fused_bias_residual_activation(plain, bias, res, act)
    assert torch.equal(fused, sep.data)


def test_x3_gemm_bits_independent_of_m(P):
    """Exact mode's plan depends on (N, K) only: a row block computed inside a
    512-row GEMM and alone (64 rows, as on 8 GPUs of a batch-sharded C2) has
    identical bits — the basis of the batch-sharding invariance."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(3)
    for N, K in ((1024, 1024), (3072, 1024), (1024, 4096), (32000, 1024)):
        a = torch.randn(512, K, device="cuda", generator=g)
        b = torch.randn(N, K, device="cuda", generator=g) * 0.03
        full = torch.empty(512, N, device="cuda")
        _x3(P, a, b, full)
        part = torch.empty(64, N, device="cuda")
        _x3(P, a[192:256].contiguous(), b, part)
        assert torch.equal(full[192:256], part), (N, K)


def test_x3_gemm_ln_slab_path_bit_identical(P):
    """fq_gemm_f32x3_ln: 4 K-slice slabs summed by the LN kernel == the split-K
    GEMM with its DSMEM reduction + fused bias/residual, then fq_layer_norm."""
    import torch
    from paper_2010_13887_b200 import _abi
    from paper_2010_13887_b200.model import X3Weight
    M, N, K = 512, 1024, 4096
    g = torch.Generator(device="cuda").manual_seed(9)
    a = torch.randn(M, K, device="cuda", generator=g)
    w = X3Weight.from_kn(torch.randn(N, K, device="cuda", generator=g) * 0.02, transpose=False)
    bias = torch.randn(N, device="cuda", generator=g)
    res = torch.randn(M, N, device="cuda", generator=g)
    gm = torch.rand(N, device="cuda", generator=g) + 0.5
    bt = torch.randn(N, device="cuda", generator=g)
    outs = []
    for ws_bytes in (4 * M * N * 4, 0):
        ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device="cuda")
        out = torch.empty(M, N, device="cuda")
        _abi.call("fq_gemm_f32x3_ln", a.data_ptr(), K, w.hi.data_ptr(), w.lo.data_ptr(), K,
                  bias.data_ptr(), res.data_ptr(), N, gm.data_ptr(), bt.data_ptr(), 1e-5,
                  out.data_ptr(), N, ws.data_ptr() if ws_bytes else None, ws_bytes, M, N, K,
                  _abi.stream_handle())
        outs.append(out)
    assert torch.equal(outs[0], outs[1])
    x = (a.double() @ (w.hi.double() + w.lo.double()).T + bias.double()) + res.double()
    mu, var = x.mean(1, keepdim=True), x.var(1, unbiased=False, keepdim=True)
    want = (x - mu) / torch.sqrt(var + 1e-5) * gm.double() + bt.double()
    assert float((outs[0].double() - want).abs().max()) <= 2e-5


# ---------------------------------------------------------------------------
# exact fp32 mode, 3xFP16 (fq_gemm_x3h): the engine's exact-mode GEMM

def _xh(a, b_nk, out, **kw):
    from paper_2010_13887_b200.model import XHWeight
    from paper_2010_13887_b200.tensor import gemm_xh, split_pair
    gemm_xh(split_pair(a), XHWeight.from_kn(b_nk, transpose=False), out, **kw)


def test_split_pair_exact_representation(P):
    """x = hi + lo * 2^-11 to 2^-22 relative (22 significant bits), hi the
    round-to-nearest fp16 of x (== the fp16 mode's operand)."""
    import torch
    from paper_2010_13887_b200.tensor import split_pair
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(300, 1000, device="cuda", generator=g) * torch.exp(
        torch.randn(300, 1000, device="cuda", generator=g) * 3).clamp(max=2e4)
    hi, lo = split_pair(x)
    torch.cuda.synchronize()
    assert torch.equal(hi, x.half())
    rec = hi.double() + lo.double() / 2048
    err = ((rec - x.double()).abs() / x.double().abs().clamp(min=6e-5)).max()
    assert float(err) <= 2.0 ** -21


@pytest.mark.parametrize("M,N,K", [
    (1, 8, 16), (100, 100, 72), (128, 64, 64), (512, 1024, 1024), (512, 3072, 1024),
    (512, 1024, 4096), (512, 4096, 1024), (300, 2000, 256), (512, 32000, 1024),
    (8192, 1024, 4096), (2048, 3072, 1024)])
def test_xh_gemm_matches_f64(P, M, N, K):
    """3xFP16 vs float64 on the same fp32 operands: fp32-GEMM accuracy — no
    worse than an IEEE fp32 SGEMM (cuBLAS, TF32 off) of the same product, the
    class of the reference's own OpenBLAS SGEMM, with a 5e-7 floor for short K
    (measured 1e-7 .. 1.5e-6 of the output scale; the 1024-element TMEM chunks
    of the K = 4096 slices give the largest)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(M * 5 + N + K)
    a = torch.randn(M, K, device="cuda", generator=g)
    b = torch.randn(N, K, device="cuda", generator=g) * 0.03
    want = a.double() @ b.double().T
    scale = float(want.abs().max())
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    sgemm_err = float((a @ b.T).double().sub(want).abs().max()) / scale
    torch.backends.cuda.matmul.allow_tf32 = prev
    out = torch.empty(M, N, device="cuda")
    _xh(a, b, out)
    torch.cuda.synchronize()
    err = float((out.double() - want).abs().max()) / scale
    print(f"{M}x{N}x{K}: 3xFP16 {err:.2e}  fp32 SGEMM {sgemm_err:.2e}")
    assert err <= max(sgemm_err, 5e-7), (M, N, K, err)


@pytest.mark.parametrize("act", ["none", "relu", "gelu"])
@pytest.mark.parametrize("M,N,K,with_res", [(384, 1536, 512, True), (512, 4096, 1024, False),
                                            (512, 3072, 1024, False), (4096, 3072, 1024, False)])
def test_xh_gemm_epilogue_bits_vs_separate_ops(P, act, M, N, K, with_res):
    """Fused bias / act / residual epilogue == the GEMM then fq_bias_residual_act
    (without a residual: the CTA-pair kernels of the decode FFN1 / QKV shapes,
    whose bias is staged in shared memory, one and several tiles per CTA)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(11 + M + N)
    a = torch.randn(M, K, device="cuda", generator=g)
    b = torch.randn(N, K, device="cuda", generator=g) * 0.05
    bias = torch.randn(N, device="cuda", generator=g)
    res = torch.randn(M, N, device="cuda", generator=g) if with_res else None
    fused = torch.empty(M, N, device="cuda")
    _xh(a, b, fused, bias=bias, residual=res, activation=act)
    plain = torch.empty(M, N, device="cuda")
    _xh(a, b, plain)
    sep = P.fused_bias_residual_activation(plain, bias, res, act)
    assert torch.equal(fused, sep.data)


@pytest.mark.parametrize("M", [512, 2048])
def test_xh_gemm_bits_independent_of_m(P, M):
    """The 3xFP16 numerics depend on (N, K) only: a row block computed inside
    an M-row GEMM and alone has identical bits (batch-sharding invariance),
    including where the kernel differs by M (4-slice shapes: split-K CTAs for
    M <= 1024, the persistent kernel with slice-long chunks above)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(3)
    for N, K in ((1024, 1024), (3072, 1024), (1024, 4096), (32000, 1024)):
        a = torch.randn(M, K, device="cuda", generator=g)
        b = torch.randn(N, K, device="cuda", generator=g) * 0.03
        full = torch.empty(M, N, device="cuda")
        _xh(a, b, full)
        part = torch.empty(64, N, device="cuda")
        _xh(a[192:256].contiguous(), b, part)
        assert torch.equal(full[192:256], part), (N, K)


def test_xh_gemm_ln_slab_path_bit_identical(P):
    """fq_gemm_x3h_ln: 4 K-slice slabs summed by the LN kernel == the split-K
    GEMM with its DSMEM reduction + fused bias/residual, then the LN; the fp16
    pair output == fq_split_f16 of the fp32 output."""
    import torch
    from paper_2010_13887_b200 import _abi
    from paper_2010_13887_b200.model import XHWeight
    from paper_2010_13887_b200.tensor import split_pair
    M, N, K = 512, 1024, 4096
    g = torch.Generator(device="cuda").manual_seed(9)
    a = torch.randn(M, K, device="cuda", generator=g)
    ap = split_pair(a)
    w = XHWeight.from_kn(torch.randn(N, K, device="cuda", generator=g) * 0.02, transpose=False)
    bias = torch.randn(N, device="cuda", generator=g)
    res = torch.randn(M, N, device="cuda", generator=g)
    gm = torch.rand(N, device="cuda", generator=g) + 0.5
    bt = torch.randn(N, device="cuda", generator=g)
    outs, pairs = [], []
    for ws_bytes in (4 * M * N * 4, 0):
        ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device="cuda")
        out = torch.empty(M, N, device="cuda")
        pr = torch.empty(2, M, N, dtype=torch.float16, device="cuda")
        _abi.call("fq_gemm_x3h_ln", ap[0].data_ptr(), ap[1].data_ptr(), K, w.hi.data_ptr(),
                  w.lo.data_ptr(), K, bias.data_ptr(), res.data_ptr(), N, gm.data_ptr(),
                  bt.data_ptr(), 1e-5, out.data_ptr(), N, pr[0].data_ptr(), pr[1].data_ptr(), N,
                  ws.data_ptr() if ws_bytes else None, ws_bytes, M, N, K, _abi.stream_handle())
        outs.append(out)
        pairs.append(pr)
    assert torch.equal(outs[0], outs[1])
    ref_pair = split_pair(outs[0])
    assert torch.equal(pairs[0][0], ref_pair[0]) and torch.equal(pairs[0][1], ref_pair[1])
    assert torch.equal(pairs[1][0], ref_pair[0]) and torch.equal(pairs[1][1], ref_pair[1])
    x = (a.double() @ (w.hi.double() + w.lo.double() / 2048).T + bias.double()) + res.double()
    mu, var = x.mean(1, keepdim=True), x.var(1, unbiased=False, keepdim=True)
    want = (x - mu) / torch.sqrt(var + 1e-5) * gm.double() + bt.double()
    assert float((outs[0].double() - want).abs().max()) <= 2e-5
