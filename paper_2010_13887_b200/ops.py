"""Fused single-pass ops on the device (reference: pkg/src/fuseq/ops.py:81-218).

Each ``fused_*`` validates shapes with the reference's exceptions, makes
exactly one call into ``libfq_b200.so`` and increments ``fused_passes`` once
— the reference's counter contract. Inputs may be device torch tensors,
:class:`Tensor` views or host numpy arrays (copied in); outputs are device
tensors (``out=`` may alias ``x`` where the reference allows in-place).

The naive multi-pass family of the reference (ops.py:225-336) is the
eager-framework baseline and is not part of the B200 product.
"""

from __future__ import annotations

import math
from enum import Enum

import torch

from . import _abi
from .errors import DimensionError, FullMaskError
from .tensor import ACT_IDS, OpCounters, Tensor, as_device, global_counters, writeback


class FusedPassKind(str, Enum):
    """The six per-layer fused kernel kinds of an encoder layer (ops.py:45-58)."""

    QKV_BIAS_RESHAPE = "qkv_bias_reshape"
    ATTENTION_SCALE_MASK_SOFTMAX = "attention_scale_mask_softmax"
    ATTN_OUTPUT_BIAS_RESIDUAL = "attn_output_bias_residual"
    LAYER_NORM = "layer_norm"
    FFN_BIAS_ACTIVATION = "ffn_bias_activation"
    FFN_BIAS_RESIDUAL = "ffn_bias_residual"


def _ctr(counters) -> OpCounters:
    return counters if counters is not None else global_counters()


def _f32(x) -> torch.Tensor:
    return as_device(x, torch.float32)


def _out_like(out, shape) -> torch.Tensor:
    if out is None:
        return torch.empty(shape, dtype=torch.float32, device=torch.device("cuda"))
    o = as_device(out)
    if tuple(o.shape) != tuple(shape):
        raise DimensionError(f"output shape {tuple(o.shape)}, expected {tuple(shape)}")
    return o


def _rows(t: torch.Tensor, what: str) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise DimensionError(f"{what} must be 2D with unit column stride")
    return t.stride(0)


def fused_layer_norm(x, gamma, beta, eps: float = 1e-5, out=None, *, counters=None,
                     kind: str = FusedPassKind.LAYER_NORM.value) -> Tensor:
    """Row-wise (x - mean)/sqrt(var + eps)*gamma + beta in one kernel (ops.py:81)."""
    X, G, B = _f32(x), _f32(gamma), _f32(beta)
    if X.dim() != 2 or tuple(G.shape) != (X.shape[1],) or tuple(B.shape) != (X.shape[1],):
        raise DimensionError(f"layer_norm shapes: x {tuple(X.shape)}, gamma {tuple(G.shape)}, "
                             f"beta {tuple(B.shape)}")
    if eps < 0:
        raise DimensionError("eps must be non-negative")
    O = _out_like(out, X.shape)
    _abi.call("fq_layer_norm", X.data_ptr(), _rows(X, "x"), G.data_ptr(), B.data_ptr(), float(eps),
              X.shape[0], X.shape[1], O.data_ptr(), _rows(O, "out"), None, 0,
              _abi.stream_handle())
    _ctr(counters).count_fused(kind, X.numel() * 8)
    writeback(out, O)
    return Tensor(O)


def fused_attention_softmax(scores, scale: float, mask=None, out=None, *, counters=None,
                            kind: str = FusedPassKind.ATTENTION_SCALE_MASK_SOFTMAX.value) -> Tensor:
    """softmax(scores*scale + mask) over the last axis (ops.py:99-125). A fully
    masked row raises FullMaskError. ``scores`` may be a strided slice whose
    rows are contiguous (the decoder's sscores[..., :cur])."""
    S = _f32(scores)
    if S.dim() != 4:
        raise DimensionError(f"attention scores must be 4D, got {S.dim()}D")
    b, h, q, l = S.shape
    if S.stride(3) != 1 or S.stride(1) != q * S.stride(2) or S.stride(0) != h * S.stride(1):
        raise DimensionError("attention scores must have contiguous rows in a uniform grid")
    M = None
    if mask is not None:
        M = _f32(mask).reshape(-1, _f32(mask).shape[-1]).contiguous()
        if tuple(M.shape) != (b, l):
            raise DimensionError(f"mask shape {tuple(M.shape)} incompatible with scores "
                                 f"{tuple(S.shape)}")
    O = _out_like(out, S.shape)
    if O.stride(3) != 1 or O.stride(1) != q * O.stride(2) or O.stride(0) != h * O.stride(1):
        raise DimensionError("softmax output must have contiguous rows in a uniform grid")
    bad = torch.zeros(1, dtype=torch.int32, device=S.device)
    _abi.call("fq_scale_mask_softmax", S.data_ptr(), S.stride(2), O.data_ptr(), O.stride(2), b, h,
              q, l, float(scale), _abi.ptr(M), bad.data_ptr(), _abi.stream_handle())
    n_bad = int(bad.item())
    if n_bad:
        raise FullMaskError(f"{n_bad} attention row(s) fully masked")
    _ctr(counters).count_fused(kind, S.numel() * 8)
    writeback(out, O)
    return Tensor(O)


def fused_bias_residual_activation(x, bias, residual=None, activation: str = "none", out=None, *,
                                   counters=None, kind: str | None = None) -> Tensor:
    """activation(x + bias) (+ residual) in one kernel; GELU exact erf form (ops.py:128)."""
    X, B = _f32(x), _f32(bias)
    if X.dim() != 2 or tuple(B.shape) != (X.shape[1],):
        raise DimensionError(f"bias shapes: x {tuple(X.shape)}, bias {tuple(B.shape)}")
    if activation not in ACT_IDS:
        raise DimensionError(f"unknown activation {activation!r}")
    R, ldr = None, 0
    if residual is not None:
        R = _f32(residual)
        if tuple(R.shape) != tuple(X.shape):
            raise DimensionError(f"residual shape {tuple(R.shape)} != x shape {tuple(X.shape)}")
        ldr = _rows(R, "residual")
    O = _out_like(out, X.shape)
    _abi.call("fq_bias_residual_act", X.data_ptr(), _rows(X, "x"), B.data_ptr(), _abi.ptr(R), ldr,
              ACT_IDS[activation], X.shape[0], X.shape[1], O.data_ptr(), _rows(O, "out"),
              _abi.stream_handle())
    if kind is None:
        kind = (FusedPassKind.ATTN_OUTPUT_BIAS_RESIDUAL.value if R is not None
                else FusedPassKind.FFN_BIAS_ACTIVATION.value)
    _ctr(counters).count_fused(kind, X.numel() * (12 if R is not None else 8))
    writeback(out, O)
    return Tensor(O)


def fused_bias_residual_layer_norm(x, bias, residual, gamma, beta, eps: float = 1e-5, out=None,
                                   *, counters=None,
                                   kind: str = FusedPassKind.FFN_BIAS_RESIDUAL.value) -> Tensor:
    """layer_norm(x + bias + residual) in one kernel (ops.py:156)."""
    X, B, R = _f32(x), _f32(bias), _f32(residual)
    G, Be = _f32(gamma), _f32(beta)
    if X.dim() != 2 or tuple(B.shape) != (X.shape[1],) or tuple(R.shape) != tuple(X.shape):
        raise DimensionError(f"shapes: x {tuple(X.shape)}, bias {tuple(B.shape)}, "
                             f"residual {tuple(R.shape)}")
    if tuple(G.shape) != (X.shape[1],) or tuple(Be.shape) != (X.shape[1],):
        raise DimensionError(f"norm parameter shapes: gamma {tuple(G.shape)}, beta {tuple(Be.shape)}")
    O = _out_like(out, X.shape)
    _abi.call("fq_bias_residual_layer_norm", X.data_ptr(), _rows(X, "x"), B.data_ptr(),
              R.data_ptr(), _rows(R, "residual"), G.data_ptr(), Be.data_ptr(), float(eps),
              X.shape[0], X.shape[1], O.data_ptr(), _rows(O, "out"), None, 0,
              _abi.stream_handle())
    _ctr(counters).count_fused(kind, X.numel() * 12)
    writeback(out, O)
    return Tensor(O)


def fused_qkv_bias_reshape(qkv, bias, batch: int, seq: int, heads: int, q_out=None, k_out=None,
                           v_out=None, *, counters=None,
                           kind: str = FusedPassKind.QKV_BIAS_RESHAPE.value):
    """[batch*seq, 3d] + bias -> head-major [batch, heads, seq, hd] x3 (ops.py:173)."""
    X, B = _f32(qkv), _f32(bias)
    if X.dim() != 2 or X.shape[0] != batch * seq or X.shape[1] % 3:
        raise DimensionError(f"qkv shape {tuple(X.shape)} incompatible with batch {batch} seq {seq}")
    d = X.shape[1] // 3
    if tuple(B.shape) != (3 * d,) or d % heads:
        raise DimensionError(f"bias shape {tuple(B.shape)} or heads {heads} incompatible with d {d}")
    hd = d // heads
    shape4 = (batch, heads, seq, hd)
    Q, K, V = (_out_like(o, shape4) for o in (q_out, k_out, v_out))
    for t in (Q, K, V):
        if not t.is_contiguous():
            raise DimensionError("q/k/v outputs must be contiguous")
    _abi.call("fq_qkv_bias_reshape", X.data_ptr(), _rows(X, "qkv"), B.data_ptr(), batch, seq,
              heads, hd, Q.data_ptr(), K.data_ptr(), V.data_ptr(), _abi.stream_handle())
    _ctr(counters).count_fused(kind, X.numel() * 8)
    for o, t in ((q_out, Q), (k_out, K), (v_out, V)):
        writeback(o, t)
    return Tensor(Q), Tensor(K), Tensor(V)


def fused_bias_reshape_heads(x, bias, batch: int, seq: int, heads: int, out=None, *,
                             counters=None,
                             kind: str = FusedPassKind.QKV_BIAS_RESHAPE.value) -> Tensor:
    """Single-tensor variant of the QKV split (ops.py:194)."""
    X, B = _f32(x), _f32(bias)
    if X.dim() != 2 or X.shape[0] != batch * seq or tuple(B.shape) != (X.shape[1],):
        raise DimensionError(f"x shape {tuple(X.shape)} incompatible with batch {batch} seq {seq}")
    d = X.shape[1]
    if d % heads:
        raise DimensionError(f"d {d} not divisible by heads {heads}")
    O = _out_like(out, (batch, heads, seq, d // heads))
    if not O.is_contiguous():
        raise DimensionError("output must be contiguous")
    _abi.call("fq_bias_reshape_heads", X.data_ptr(), _rows(X, "x"), B.data_ptr(), batch, seq,
              heads, d // heads, O.data_ptr(), _abi.stream_handle())
    _ctr(counters).count_fused(kind, X.numel() * 8)
    writeback(out, O)
    return Tensor(O)


def fused_embed(tokens, embedding, scale: float, positions, pos_offset: int, seq: int, out=None,
                *, counters=None, kind: str = "embed_scale_pos") -> Tensor:
    """Embedding gather, sqrt(d) scaling and positional add in one pass (ops.py:211)."""
    T = as_device(tokens, torch.int64).contiguous()
    E, P = _f32(embedding), _f32(positions)
    O = _out_like(out, (T.shape[0], E.shape[1]))
    _abi.call("fq_embed_scale_pos", T.data_ptr(), T.shape[0], E.data_ptr(), E.shape[1],
              float(scale), P.data_ptr(), int(pos_offset), None, int(seq), O.data_ptr(), None,
              _abi.stream_handle())
    _ctr(counters).count_fused(kind, O.numel() * 8)
    writeback(out, O)
    return Tensor(O)


def _kv4(t, what: str) -> torch.Tensor:
    t = as_device(t, torch.float32)
    if t.dim() != 4 or not t.is_contiguous():
        raise DimensionError(f"{what} must be a contiguous [rows, heads, seq, head_dim] tensor")
    return t


def kv_append(new_k, new_v, cur: int, dst_k, dst_v):
    """Cache refresh without reorder (kernels.py:205-211, fq_kv_append):
    dst[r, :, cur, :] = new[r, :, 0, :] on the reference's [rows, heads, S, hd]
    layout. The engine's copy-free cache (``KVCache``) never needs it."""
    nk, nv = _kv4(new_k, "new_k"), _kv4(new_v, "new_v")
    dk, dv = _kv4(dst_k, "dst_k"), _kv4(dst_v, "dst_v")
    R, H, S, E = dk.shape
    if tuple(nk.shape) != (R, H, 1, E) or nv.shape != nk.shape or dv.shape != dk.shape:
        raise DimensionError("kv_append: new K/V must be [rows, heads, 1, head_dim]")
    _abi.call("fq_kv_append", nk.data_ptr(), nv.data_ptr(), int(cur), R, H, S, E, dk.data_ptr(),
              dv.data_ptr(), _abi.stream_handle())


def kv_gather_append(src_k, src_v, new_k, new_v, parents, cur: int, dst_k, dst_v):
    """Ping-pong beam reorder + append (kernels.py:189-201, fq_kv_gather_append):
    dst[r, :, :cur] = src[parents[r], :, :cur]; dst[r, :, cur] = new[r, :, 0]."""
    sk, sv = _kv4(src_k, "src_k"), _kv4(src_v, "src_v")
    nk, nv = _kv4(new_k, "new_k"), _kv4(new_v, "new_v")
    dk, dv = _kv4(dst_k, "dst_k"), _kv4(dst_v, "dst_v")
    R, H, S, E = dk.shape
    if sk.shape != dk.shape or tuple(nk.shape) != (R, H, 1, E):
        raise DimensionError("kv_gather_append: shapes differ")
    par = as_device(parents, torch.int64).contiguous()
    if tuple(par.shape) != (R,):
        raise DimensionError(f"parents must be [{R}]")
    _abi.call("fq_kv_gather_append", sk.data_ptr(), sv.data_ptr(), nk.data_ptr(), nv.data_ptr(),
              par.data_ptr(), int(cur), R, H, S, E, dk.data_ptr(), dv.data_ptr(),
              _abi.stream_handle())


def attention_scale(head_dim: int) -> float:
    """np.float32(1/sqrt(hd)) as the reference passes it (ops.py:121)."""
    return float(torch.tensor(1.0 / math.sqrt(head_dim), dtype=torch.float32))
