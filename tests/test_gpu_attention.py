"""Fused attention kernels (fq_attention.cu) against float64 torch references
of the reference's three-step attention (gemm_batched QK^T -> scale_mask_softmax
-> gemm_batched P.V, model.py:329-336 / :572-604), including the copy-free
history-table KV cache. fp32 KV: 1e-5 relative; fp16 KV: operands rounded to
fp16 in the reference too, 1e-4."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T(gpu):
    import torch
    return torch


def _abi():
    from paper_2010_13887_b200 import _abi
    return _abi


def _rel(got, want):
    return float((got.double() - want).abs().max() / max(want.abs().max().item(), 1e-9))


def _softmax_ref(T, s, mask=None):
    if mask is not None:
        s = s + mask
    return T.softmax(s, dim=-1)


@pytest.mark.parametrize("hd", [16, 32, 64, 128])
@pytest.mark.parametrize("beam", [1, 3, 4, 8])
@pytest.mark.parametrize("kv16", [False, True])
def test_cross_attention(T, hd, beam, kv16):
    A = _abi()
    g = T.Generator(device="cuda").manual_seed(hd * 10 + beam)
    B, S, H, L = 3, 37, 4, 2
    d = H * hd
    ld = 2 * L * d
    cq = T.randn(B * beam, d, device="cuda", generator=g)
    packed = T.randn(B * S, ld, device="cuda", generator=g)
    if kv16:
        packed = packed.to(T.float16)
    mask = T.zeros(B, S, device="cuda")
    mask[1, 30:] = -math.inf
    scale = float(np.float32(1 / math.sqrt(hd)))
    layer = 1
    ck = packed[:, 2 * layer * d:]
    cv = packed[:, (2 * layer + 1) * d:]
    out = T.empty(B * beam, d, device="cuda")
    out16 = T.empty(B * beam, d, device="cuda", dtype=T.float16)
    bad = T.zeros(1, dtype=T.int32, device="cuda")
    A.call("fq_cross_attention", cq.data_ptr(), d, ck.data_ptr(), cv.data_ptr(), int(kv16), ld, B,
           beam, S, H, hd, scale, mask.data_ptr(), out.data_ptr(), out16.data_ptr(), d,
           0 if kv16 else 1, bad.data_ptr(), A.stream_handle())
    T.cuda.synchronize()
    K = packed[:, 2 * layer * d:(2 * layer + 1) * d].double().view(B, S, H, hd).permute(0, 2, 1, 3)
    V = packed[:, (2 * layer + 1) * d:(2 * layer + 2) * d].double().view(B, S, H, hd).permute(0, 2, 1, 3)
    Q = cq.double().view(B, beam, H, hd).permute(0, 2, 1, 3)
    P = _softmax_ref(T, (Q @ K.transpose(-1, -2)) * scale, mask.double()[:, None, None, :])
    want = (P @ V).permute(0, 2, 1, 3).reshape(B * beam, d)
    assert int(bad.item()) == 0
    assert _rel(out, want) <= (1e-4 if kv16 else 1e-5)
    assert _rel(out16.float(), want) <= 1e-2


@pytest.mark.parametrize("hd", [16, 64, 128, 48])
@pytest.mark.parametrize("kv16", [False, True])
def test_decoder_self_attention_history_table(T, hd, kv16):
    A = _abi()
    g = T.Generator(device="cuda").manual_seed(hd + 7)
    rows, H, S, beam = 12, 3, 20, 4
    d = H * hd
    dt = T.float16 if kv16 else T.float32
    kc = T.randn(S, rows, d, device="cuda", generator=g).to(dt)
    vc = T.randn(S, rows, d, device="cuda", generator=g).to(dt)
    cur = 13
    # beams only ever inherit from rows of their own item
    hist = T.empty(rows, S, dtype=T.int32, device="cuda")
    for r in range(rows):
        item0 = (r // beam) * beam
        hist[r] = T.randint(item0, item0 + beam, (S,), generator=g, device="cuda").int()
    sqkv = T.randn(rows, 3 * d, device="cuda", generator=g)
    d_cur = T.tensor([cur], dtype=T.int32, device="cuda")
    out = T.empty(rows, d, device="cuda")
    scale = float(np.float32(1 / math.sqrt(hd)))
    A.call("fq_decoder_self_attention", sqkv.data_ptr(), 3 * d, kc.data_ptr(), vc.data_ptr(),
           int(kv16), hist.data_ptr(), d_cur.data_ptr(), rows, H, hd, S, scale, out.data_ptr(),
           None, d, 0 if kv16 else 1, A.stream_handle())
    T.cuda.synchronize()
    knew = sqkv[:, d:2 * d].to(dt).double()
    vnew = sqkv[:, 2 * d:].to(dt).double()
    assert T.equal(kc[cur].double(), knew) and T.equal(vc[cur].double(), vnew)  # slot written
    for r in range(rows):
        idx = hist[r, :cur].long()
        Kr = T.cat([kc[T.arange(cur, device="cuda"), idx].double(), knew[r:r + 1]])  # [cur+1, d]
        Vr = T.cat([vc[T.arange(cur, device="cuda"), idx].double(), vnew[r:r + 1]])
        q = sqkv[r, :d].double()
        for h in range(H):
            sl = slice(h * hd, (h + 1) * hd)
            p = T.softmax((Kr[:, sl] @ q[sl]) * scale, dim=0)
            want = p @ Vr[:, sl]
            assert _rel(out[r, sl], want) <= 1e-5, (r, h)


@pytest.mark.parametrize("hd", [16, 64])
def test_encoder_attention(T, hd):
    A = _abi()
    g = T.Generator(device="cuda").manual_seed(3)
    B, S, H = 2, 29, 4
    d = H * hd
    qkv = T.randn(B * S, 3 * d, device="cuda", generator=g)
    mask = T.zeros(B, S, device="cuda")
    mask[0, 20:] = -math.inf
    out = T.empty(B * S, d, device="cuda")
    scale = float(np.float32(1 / math.sqrt(hd)))
    A.call("fq_encoder_attention", qkv.data_ptr(), 3 * d, B, S, H, hd, scale, mask.data_ptr(),
           out.data_ptr(), None, d, 1, None, A.stream_handle())
    T.cuda.synchronize()
    x = qkv.double().view(B, S, 3, H, hd)
    Q, K, V = (x[:, :, i].permute(0, 2, 1, 3) for i in range(3))
    P = _softmax_ref(T, (Q @ K.transpose(-1, -2)) * scale, mask.double()[:, None, None, :])
    want = (P @ V).permute(0, 2, 1, 3).reshape(B * S, d)
    assert _rel(out, want) <= 1e-5


@pytest.mark.parametrize("rows,d", [(7, 512), (512, 1024), (3, 2048), (9000, 1024), (5, 384)])
def test_layer_norm_paths(T, rows, d):
    """All three LN kernels (row128 / warp / CTA) against the f64 formula."""
    import paper_2010_13887_b200 as P
    g = T.Generator(device="cuda").manual_seed(rows)
    x = T.randn(rows, d, device="cuda", generator=g)
    gm = T.randn(d, device="cuda", generator=g)
    b = T.randn(d, device="cuda", generator=g)
    out = P.fused_layer_norm(x, gm, b, 1e-5).data
    xd = x.double()
    want = (xd - xd.mean(1, keepdim=True)) / T.sqrt(xd.var(1, unbiased=False, keepdim=True) + 1e-5)
    want = want * gm.double() + b.double()
    assert _rel(out, want) <= 1e-6


@pytest.mark.parametrize("H,hd,rows,cur", [(16, 64, 12, 13), (8, 128, 8, 0), (16, 64, 20, 63),
                                          (32, 32, 4, 7), (8, 64, 8, 30), (4, 64, 6, 97),
                                          (16, 64, 5, 15), (16, 64, 5, 16)])
def test_decoder_self_attention_rows_kernel(T, H, hd, rows, cur):
    """The fp16 throughput-mode row kernel (CTA per beam row, 16-byte slot
    segments, shuffle-reduced head dots) vs float64 on the fp16 cache."""
    A = _abi()
    g = T.Generator(device="cuda").manual_seed(H * hd + rows + cur)
    S, beam = (64 if cur < 64 else 128), 4
    d = H * hd
    kc = T.randn(S, rows, d, device="cuda", generator=g).to(T.float16)
    vc = T.randn(S, rows, d, device="cuda", generator=g).to(T.float16)
    hist = T.empty(rows, S, dtype=T.int32, device="cuda")
    for r in range(rows):
        item0 = (r // beam) * beam
        hist[r] = T.randint(item0, min(item0 + beam, rows), (S,), generator=g, device="cuda").int()
    sqkv = T.randn(rows, 3 * d, device="cuda", generator=g)
    d_cur = T.tensor([cur], dtype=T.int32, device="cuda")
    out = T.empty(rows, d, device="cuda")
    out16 = T.empty(rows, d, device="cuda", dtype=T.float16)
    scale = float(np.float32(1 / math.sqrt(hd)))
    A.call("fq_decoder_self_attention", sqkv.data_ptr(), 3 * d, kc.data_ptr(), vc.data_ptr(), 1,
           hist.data_ptr(), d_cur.data_ptr(), rows, H, hd, S, scale, out.data_ptr(),
           out16.data_ptr(), d, 0, A.stream_handle())
    T.cuda.synchronize()
    knew = sqkv[:, d:2 * d].to(T.float16).double()
    vnew = sqkv[:, 2 * d:].to(T.float16).double()
    assert T.equal(kc[cur].double(), knew) and T.equal(vc[cur].double(), vnew)
    ar = T.arange(cur, device="cuda")
    for r in range(rows):
        idx = hist[r, :cur].long()
        Kr = T.cat([kc[ar, idx].double(), knew[r:r + 1]]).view(cur + 1, H, hd)
        Vr = T.cat([vc[ar, idx].double(), vnew[r:r + 1]]).view(cur + 1, H, hd)
        q = sqkv[r, :d].double().view(H, hd)
        p = T.softmax(T.einsum("the,he->ht", Kr, q) * scale, dim=1)
        want = T.einsum("ht,the->he", p, Vr).reshape(d)
        assert _rel(out[r], want) <= 1e-4, r
        assert _rel(out16[r].float(), want) <= 1e-2, r


@pytest.mark.parametrize("H,hd,beam", [(16, 64, 4), (16, 64, 1), (8, 128, 3), (32, 32, 8),
                                       (16, 64, 6)])
def test_cross_attention_stream_kernel(T, H, hd, beam):
    """The fp16 throughput-mode cross-attention (CTA per item x head chunk)
    including a padded item and a fully masked item (counted in d_bad)."""
    A = _abi()
    g = T.Generator(device="cuda").manual_seed(H + hd + beam)
    B, S, L = 4, 64, 3
    d = H * hd
    ld = 2 * L * d
    cq = T.randn(B * beam, d, device="cuda", generator=g)
    packed = T.randn(B * S, ld, device="cuda", generator=g).to(T.float16)
    mask = T.zeros(B, S, device="cuda")
    mask[1, 41:] = -math.inf
    mask[3, :] = -math.inf
    scale = float(np.float32(1 / math.sqrt(hd)))
    layer = 2
    ck = packed[:, 2 * layer * d:]
    cv = packed[:, (2 * layer + 1) * d:]
    out = T.empty(B * beam, d, device="cuda")
    out16 = T.empty(B * beam, d, device="cuda", dtype=T.float16)
    bad = T.zeros(1, dtype=T.int32, device="cuda")
    A.call("fq_cross_attention", cq.data_ptr(), d, ck.data_ptr(), cv.data_ptr(), 1, ld, B,
           beam, S, H, hd, scale, mask.data_ptr(), out.data_ptr(), out16.data_ptr(), d, 0,
           bad.data_ptr(), A.stream_handle())
    T.cuda.synchronize()
    assert int(bad.item()) == beam * H  # every (beam, head) row of item 3
    K = packed[:, 2 * layer * d:(2 * layer + 1) * d].double().view(B, S, H, hd).permute(0, 2, 1, 3)
    V = packed[:, (2 * layer + 1) * d:(2 * layer + 2) * d].double().view(B, S, H, hd).permute(0, 2, 1, 3)
    Q = cq.double().view(B, beam, H, hd).permute(0, 2, 1, 3)
    P = _softmax_ref(T, (Q @ K.transpose(-1, -2)) * scale, mask.double()[:, None, None, :])
    want = (P @ V).permute(0, 2, 1, 3).reshape(B * beam, d)
    n = 3 * beam  # items 0..2
    assert _rel(out[:n], want[:n]) <= 1e-4
    assert _rel(out16[:n].float(), want[:n]) <= 1e-2


@pytest.mark.parametrize("beam,S", [(1, 1), (4, 64), (3, 37), (8, 17), (5, 64)])
def test_cross_attention_fp16_ctx(T, beam, S):
    """The fp16 mode's cross-attention (fp16 K/V, fp16 context only -- the
    engine's half_mode call; cross_attention_xh<..., PAIR=false>) vs float64,
    with a partly and a fully masked item (the latter counted in d_bad)."""
    A = _abi()
    g = T.Generator(device="cuda").manual_seed(beam * 100 + S)
    B, H, hd, L = 4, 16, 64, 2
    d = H * hd
    ld = 2 * L * d
    cq = T.randn(B * beam, d, device="cuda", generator=g)
    packed = T.randn(B * S, ld, device="cuda", generator=g).to(T.float16)
    mask = T.zeros(B, S, device="cuda")
    mask[1, (S + 1) // 2:] = -math.inf
    mask[3, :] = -math.inf
    scale = float(np.float32(1 / math.sqrt(hd)))
    ck, cv = packed[:, 2 * d:], packed[:, 3 * d:]
    out16 = T.full((B * beam, d), float("nan"), device="cuda", dtype=T.float16)
    bad = T.zeros(1, dtype=T.int32, device="cuda")
    A.call("fq_cross_attention", cq.data_ptr(), d, ck.data_ptr(), cv.data_ptr(), 1, ld, B, beam,
           S, H, hd, scale, mask.data_ptr(), None, out16.data_ptr(), d, 0, bad.data_ptr(),
           A.stream_handle())
    T.cuda.synchronize()
    assert int(bad.item()) == beam * H
    K = ck[:, :d].double().view(B, S, H, hd).permute(0, 2, 1, 3)
    V = cv[:, :d].double().view(B, S, H, hd).permute(0, 2, 1, 3)
    Q = cq.double().view(B, beam, H, hd).permute(0, 2, 1, 3)
    P = _softmax_ref(T, (Q @ K.transpose(-1, -2)) * scale, mask.double()[:, None, None, :])
    want = (P @ V).permute(0, 2, 1, 3).reshape(B * beam, d)
    n = 3 * beam  # items 0..2
    assert _rel(out16[:n].float(), want[:n]) <= 2e-3


@pytest.mark.parametrize("S,hd,exact", [(64, 64, 1), (64, 64, 0), (17, 128, 1), (1, 64, 1),
                                        (64, 32, 0)])
def test_encoder_attention_tiled(T, S, hd, exact):
    A = _abi()
    g = T.Generator(device="cuda").manual_seed(S + hd)
    B, H = 3, 4
    d = H * hd
    qkv = T.randn(B * S, 3 * d, device="cuda", generator=g)
    mask = T.zeros(B, S, device="cuda")
    mask[1, S // 2 + 1:] = -math.inf
    out = T.empty(B * S, d, device="cuda")
    out16 = T.empty(B * S, d, device="cuda", dtype=T.float16)
    bad = T.zeros(1, dtype=T.int32, device="cuda")
    scale = float(np.float32(1 / math.sqrt(hd)))
    A.call("fq_encoder_attention", qkv.data_ptr(), 3 * d, B, S, H, hd, scale, mask.data_ptr(),
           out.data_ptr(), out16.data_ptr(), d, exact, bad.data_ptr(), A.stream_handle())
    T.cuda.synchronize()
    assert int(bad.item()) == 0
    x = qkv.double().view(B, S, 3, H, hd)
    Q, K, V = (x[:, :, i].permute(0, 2, 1, 3) for i in range(3))
    P = _softmax_ref(T, (Q @ K.transpose(-1, -2)) * scale, mask.double()[:, None, None, :])
    want = (P @ V).permute(0, 2, 1, 3).reshape(B * S, d)
    assert _rel(out, want) <= (1e-5 if exact else 1e-4)
    assert _rel(out16.float(), want) <= 1e-2


@pytest.mark.parametrize("M,beam,S", [(512, 4, 64), (96, 3, 37)])
def test_cross_attention_slabs_equal_reduced_query(T, M, beam, S):
    """The engine's cross-q path: fq_gemm_splitk_slabs (the split-K GEMM's 4
    K-slice partials, no reduction) + fq_cross_attention_slabs (slabs summed in
    order + bias on load) is bit-identical to fq_gemm (split-K with its own
    reduction, + bias) followed by fq_cross_attention."""
    import ctypes
    A = _abi()
    g = T.Generator(device="cuda").manual_seed(M + beam + S)
    d, H, hd, L = 1024, 16, 64, 2
    B = M // beam
    R = B * beam
    x16 = T.randn(R, d, device="cuda", generator=g).to(T.float16)
    w = (T.randn(d, d, device="cuda", generator=g) / 32).to(T.float16)
    bias = T.randn(d, device="cuda", generator=g) * 0.1
    ld = 2 * L * d
    packed = T.randn(B * S, ld, device="cuda", generator=g).to(T.float16)
    mask = T.zeros(B, S, device="cuda")
    mask[0, S // 2:] = -math.inf
    scale = float(np.float32(1 / math.sqrt(hd)))
    ck, cv = packed[:, 2 * d:], packed[:, 3 * d:]
    q = T.empty(R, d, device="cuda")
    import paper_2010_13887_b200 as P
    P.gemm(x16, w, q, transpose_b=True, bias=bias)
    want = T.empty(R, d, device="cuda", dtype=T.float16)
    bad = T.zeros(1, dtype=T.int32, device="cuda")
    A.call("fq_cross_attention", q.data_ptr(), d, ck.data_ptr(), cv.data_ptr(), 1, ld, B, beam, S,
           H, hd, scale, mask.data_ptr(), None, want.data_ptr(), d, 0, bad.data_ptr(),
           A.stream_handle())
    ws = T.full((4 * R * d,), float("nan"), device="cuda")
    ns = ctypes.c_int(-1)
    A.call("fq_gemm_splitk_slabs", x16.data_ptr(), d, w.data_ptr(), d, ws.data_ptr(),
           ws.numel() * 4, R, d, d, ctypes.addressof(ns), A.stream_handle())
    assert ns.value == 4
    got = T.empty(R, d, device="cuda", dtype=T.float16)
    A.call("fq_cross_attention_slabs", ws.data_ptr(), ns.value, d, bias.data_ptr(), ck.data_ptr(),
           cv.data_ptr(), ld, B, beam, S, H, hd, scale, mask.data_ptr(), None, got.data_ptr(), d,
           bad.data_ptr(), A.stream_handle())
    T.cuda.synchronize()
    assert T.equal(got, want)


@pytest.mark.parametrize("S", [1, 17, 64])
def test_encoder_attention_xh(T, S):
    """Exact-mode encoder attention on 3xFP16 warp MMAs (head_dim 64, seq <= 64):
    the fp32 context and its fp16 pair vs float64 (masked keys, a fully masked
    row counted), the pair reconstructing the fp32 output."""
    A = _abi()
    g = T.Generator(device="cuda").manual_seed(S + 5)
    B, H, hd = 3, 4, 64
    d = H * hd
    qkv = T.randn(B * S, 3 * d, device="cuda", generator=g)
    mask = T.zeros(B, S, device="cuda")
    if S > 1:
        mask[1, S // 2 + 1:] = -math.inf
    out = T.empty(B * S, d, device="cuda")
    hi = T.empty(B * S, d, device="cuda", dtype=T.float16)
    lo = T.empty_like(hi)
    bad = T.zeros(1, dtype=T.int32, device="cuda")
    scale = float(np.float32(1 / math.sqrt(hd)))
    A.call("fq_encoder_attention_xh", qkv.data_ptr(), 3 * d, B, S, H, hd, scale,
           mask.data_ptr(), out.data_ptr(), hi.data_ptr(), lo.data_ptr(), d, bad.data_ptr(),
           A.stream_handle())
    T.cuda.synchronize()
    assert int(bad.item()) == 0
    x = qkv.double().view(B, S, 3, H, hd)
    Q, K, V = (x[:, :, i].permute(0, 2, 1, 3) for i in range(3))
    P = _softmax_ref(T, (Q @ K.transpose(-1, -2)) * scale, mask.double()[:, None, None, :])
    want = (P @ V).permute(0, 2, 1, 3).reshape(B * S, d)
    assert _rel(out, want) <= 1e-5
    back = hi.double() + lo.double() / 2048.0
    assert float((back - out.double()).abs().max()) <= 1e-6 * float(out.abs().max()) + 1e-9
    mask[2, :] = -math.inf  # a fully masked row: counted, not written
    A.call("fq_encoder_attention_xh", qkv.data_ptr(), 3 * d, B, S, H, hd, scale,
           mask.data_ptr(), out.data_ptr(), hi.data_ptr(), lo.data_ptr(), d, bad.data_ptr(),
           A.stream_handle())
    T.cuda.synchronize()
    assert int(bad.item()) == S * H


def test_cross_attention_xh_slab_query_bit_identical(T):
    """Exact cross-attention with the query as the split-K slabs of its GEMM
    (fq_gemm_x3h_slabs + fq_cross_attention_xh_slabs: slabs summed in order +
    bias in the query load) == the DSMEM-reduced query GEMM + the plain kernel,
    bit for bit (C2 decode shape: 512 rows, d = 1024, 16 heads x 64)."""
    import ctypes
    from paper_2010_13887_b200.model import XHWeight
    from paper_2010_13887_b200.tensor import split_pair
    A = _abi()
    g = T.Generator(device="cuda").manual_seed(17)
    B, K, S, H, hd = 128, 4, 37, 16, 64
    R, d = B * K, H * hd
    x = T.randn(R, d, device="cuda", generator=g)
    xh, xl = split_pair(x)
    w = XHWeight.from_kn(T.randn(d, d, device="cuda", generator=g) * 0.03, transpose=False)
    bias = T.randn(d, device="cuda", generator=g) * 0.1
    kv = T.randn(B * S, 2 * d, device="cuda", generator=g)
    kvh, kvl = split_pair(kv)
    planes = T.stack([kvh, kvl]).contiguous()  # [2, B*S, 2d]
    mask = T.zeros(B, S, device="cuda")
    mask[3, 20:] = -math.inf
    scale = float(np.float32(1 / math.sqrt(hd)))
    q = T.empty(R, d, device="cuda")
    A.call("fq_gemm_x3h", xh.data_ptr(), xl.data_ptr(), d, w.hi.data_ptr(), w.lo.data_ptr(), d,
           q.data_ptr(), d, R, d, d, 0, bias.data_ptr(), None, 0, 0, A.stream_handle())
    outs = []
    for slabs in (False, True):
        oh = T.empty(R, d, device="cuda", dtype=T.float16)
        ol = T.empty_like(oh)
        bad = T.zeros(1, dtype=T.int32, device="cuda")
        args = (planes[0, :, :d].data_ptr(), planes[0, :, d:].data_ptr(), planes.stride(0),
                planes.stride(1), B, K, S, H, hd, scale, mask.data_ptr(), None, oh.data_ptr(),
                ol.data_ptr(), d, bad.data_ptr(), A.stream_handle())
        if slabs:
            ws = T.empty(4 * R * d, device="cuda")
            n = ctypes.c_int32(0)
            assert A.lib_call_rc("fq_gemm_x3h_slabs", xh.data_ptr(), xl.data_ptr(), d,
                                 w.hi.data_ptr(), w.lo.data_ptr(), d, ws.data_ptr(),
                                 ws.numel() * 4, R, d, d, ctypes.addressof(n),
                                 A.stream_handle()) == 0
            assert n.value == 4
            A.call("fq_cross_attention_xh_slabs", ws.data_ptr(), n.value, d, R * d,
                   bias.data_ptr(), *args)
        else:
            A.call("fq_cross_attention_xh", q.data_ptr(), d, *args)
        T.cuda.synchronize()
        assert int(bad.item()) == 0
        outs.append((oh, ol))
    assert T.equal(outs[0][0], outs[1][0]) and T.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("beam,cur,S", [(4, 13, 64), (4, 0, 64), (4, 63, 64), (2, 16, 32),
                                        (8, 31, 40), (3, 15, 20), (4, 100, 128)])
def test_self_attention_items_xh(T, beam, cur, S):
    """The exact self-attention per (item, head) over the distinct history
    slots of the item's beams vs the per-row kernel on the same pair cache:
    the same slot writes, contexts within the last fp32 bits (only the
    grouping of the P.V terms differs), both vs float64."""
    A = _abi()
    g = T.Generator(device="cuda").manual_seed(beam * 1000 + cur)
    items, H, hd = 5, 4, 64
    rows, d = items * beam, H * hd
    kv = T.randn(2, S, rows, d, device="cuda", generator=g)

    def pair(x):
        hi = x.half()
        return T.stack([hi, ((x - hi.float()) * 2048).half()])

    kc, vc = pair(kv[0]), pair(kv[1])  # [2 (hi, lo), S, rows, d]
    hist = T.empty(rows, S, dtype=T.int32, device="cuda")
    share = T.randint(0, 3, (items, S), generator=g, device="cuda")
    for r in range(rows):
        it = r // beam
        own = T.randint(it * beam, (it + 1) * beam, (S,), generator=g, device="cuda")
        # mostly shared (one row for all beams), some positions diverging
        hist[r] = T.where(share[it] > 0, it * beam + share[it] % beam, own).int()
    sqkv = T.randn(rows, 3 * d, device="cuda", generator=g)
    d_cur = T.tensor([cur], dtype=T.int32, device="cuda")
    scale = float(np.float32(1 / math.sqrt(hd)))
    plane = S * rows * d
    outs = []
    for fn in ("fq_decoder_self_attention_xh", "fq_decoder_self_attention_xh_items"):
        k2, v2 = kc.clone(), vc.clone()
        out = T.empty(rows, d, device="cuda")
        oh = T.empty(rows, d, device="cuda", dtype=T.float16)
        ol = T.empty_like(oh)
        shape = (rows,) if fn.endswith("_xh") else (items, beam)
        A.call(fn, sqkv.data_ptr(), 3 * d, k2.data_ptr(), v2.data_ptr(), plane, hist.data_ptr(),
               d_cur.data_ptr(), *shape, H, hd, S, scale, out.data_ptr(), oh.data_ptr(),
               ol.data_ptr(), d, A.stream_handle())
        T.cuda.synchronize()
        outs.append((out, oh, ol, k2, v2))
    (o0, h0, l0, k0, v0), (o1, h1, l1, k1, v1) = outs
    assert T.equal(k0, k1) and T.equal(v0, v1)  # this step's slots, written once
    assert _rel(o1, o0.double()) <= 1e-6
    assert T.equal(h1, o1.half())
    kd = (k1[0].double() + k1[1].double() / 2048)
    vd = (v1[0].double() + v1[1].double() / 2048)
    ar = T.arange(cur + 1, device="cuda")
    for r in range(rows):
        idx = T.cat([hist[r, :cur].long(), T.tensor([r], device="cuda")])
        Kr, Vr = kd[ar, idx].view(cur + 1, H, hd), vd[ar, idx].view(cur + 1, H, hd)
        q = sqkv[r, :d].double().view(H, hd)
        p = T.softmax(T.einsum("the,he->ht", Kr, q) * scale, dim=1)
        want = T.einsum("ht,the->he", p, Vr).reshape(d)
        assert _rel(o1[r], want) <= 1e-5, r
