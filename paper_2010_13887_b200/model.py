"""Transformer encoder/decoder on the B200 (reference: pkg/src/fuseq/model.py).

Same configuration, weight layout and seeded initialisation as the reference
(model.py:44-260), so reference checkpoints (LSQW files, weights_io.py) and
``make_random_weights`` seeds load unchanged. The compute runs in HBM:

* weights are uploaded once per precision (``DeviceWeights``): ``fp32`` keeps
  the reference's input-major [in, out] matrices for the exact-mode FFMA GEMM;
  ``fp16`` casts and transposes them once to K-major [out, in] for the tcgen05
  GEMM (the paper's "fuse cast into weight loading"); the
  cross-attention K/V projections of all decoder layers are concatenated into
  one [d, 2*L*d] matrix so the per-request setup is a single large GEMM;
* an encoder layer is 7 launches: 4 GEMMs with fused epilogues (bias,
  activation, residual: the reference's bias_residual_act passes), one fused
  attention kernel (QK^T + masked softmax + P.V, merged heads), 2 layer norms;
* a decoder layer is 11 launches: 6 GEMMs, 2 attention kernels, 3 norms; the
  self-attention K/V cache is copy-free (``KVCache``): slot (t, r) is written
  once and a [rows, max_len] history table replaces the ping-pong gather of
  kernels.py:189-201.

Every intermediate is a view of the session arena (``plan_intermediates``).
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from .errors import CapacityError, ConsistencyError, DimensionError, FullMaskError, InputError
from .memory_plan import Arena, IntermediateSpec
from .ops import attention_scale
from .tensor import (ACT_IDS, OpCounters, Timers, as_device, gemm, gemm_x3, gemm_xh,
                     global_counters, split_pair)

# FQ_SELF_ITEMS=1: the exact-mode decoder self-attention per (item, head) over
# the history slots the beams share (read once). Opt-in: at C2 it reads 0.4x
# the bytes but runs 2.7% slower per request than the per-row kernel (fewer,
# longer dependent chunk chains; scripts/self_items_ab.sh)
_SELF_ITEMS = os.environ.get("FQ_SELF_ITEMS", "0") == "1"

F32 = np.float32
I64 = np.int64
PRECISIONS = ("fp32", "fp16")


# ---------------------------------------------------------------------------
# configuration and host weights  (model.py:44-278)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class ModelConfig:
    num_encoder_layers: int
    num_decoder_layers: int
    d_model: int
    d_ff: int
    num_heads: int
    vocab_size: int
    max_batch: int
    max_seq_len: int
    max_beam_size: int
    activation: str = "relu"
    tie_output: bool = True
    ln_eps: float = 1e-5

    def __post_init__(self):
        if self.d_model % self.num_heads:
            raise ConsistencyError(f"d_model {self.d_model} not divisible by heads {self.num_heads}")
        if self.vocab_size < 2:
            raise ConsistencyError("vocab_size must be at least 2")
        for name in ("max_batch", "max_seq_len", "max_beam_size", "num_heads", "d_model", "d_ff"):
            if getattr(self, name) < 1:
                raise ConsistencyError(f"{name} must be >= 1")
        if self.num_encoder_layers < 1 or self.num_decoder_layers < 0:
            raise ConsistencyError("need >= 1 encoder layer and >= 0 decoder layers")
        if self.activation not in ("none", "relu", "gelu"):
            raise ConsistencyError(f"unknown activation {self.activation!r}")

    @property
    def head_dim(self) -> int:
        return self.d_model // self.num_heads

    @property
    def max_rows(self) -> int:
        return self.max_batch * self.max_beam_size

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k in (
            "num_encoder_layers", "num_decoder_layers", "d_model", "d_ff", "num_heads",
            "vocab_size", "max_batch", "max_seq_len", "max_beam_size", "activation",
            "tie_output", "ln_eps")}


_ENC_FIELDS = ["w_qkv", "b_qkv", "w_out", "b_out", "ln1_gamma", "ln1_beta",
               "w_ff1", "b_ff1", "w_ff2", "b_ff2", "ln2_gamma", "ln2_beta"]
_DEC_FIELDS = ["w_qkv", "b_qkv", "w_self_out", "b_self_out", "ln1_gamma", "ln1_beta",
               "w_cross_q", "b_cross_q", "w_cross_k", "b_cross_k", "w_cross_v", "b_cross_v",
               "w_cross_out", "b_cross_out", "ln2_gamma", "ln2_beta",
               "w_ff1", "b_ff1", "w_ff2", "b_ff2", "ln3_gamma", "ln3_beta"]


@dataclass
class EncoderLayerWeights:
    w_qkv: np.ndarray
    b_qkv: np.ndarray
    w_out: np.ndarray
    b_out: np.ndarray
    ln1_gamma: np.ndarray
    ln1_beta: np.ndarray
    w_ff1: np.ndarray
    b_ff1: np.ndarray
    w_ff2: np.ndarray
    b_ff2: np.ndarray
    ln2_gamma: np.ndarray
    ln2_beta: np.ndarray


@dataclass
class DecoderLayerWeights:
    w_qkv: np.ndarray
    b_qkv: np.ndarray
    w_self_out: np.ndarray
    b_self_out: np.ndarray
    ln1_gamma: np.ndarray
    ln1_beta: np.ndarray
    w_cross_q: np.ndarray
    b_cross_q: np.ndarray
    w_cross_k: np.ndarray
    b_cross_k: np.ndarray
    w_cross_v: np.ndarray
    b_cross_v: np.ndarray
    w_cross_out: np.ndarray
    b_cross_out: np.ndarray
    ln2_gamma: np.ndarray
    ln2_beta: np.ndarray
    w_ff1: np.ndarray
    b_ff1: np.ndarray
    w_ff2: np.ndarray
    b_ff2: np.ndarray
    ln3_gamma: np.ndarray
    ln3_beta: np.ndarray


@dataclass(eq=False)
class ModelWeights:
    token_embedding: np.ndarray                    # [vocab, d]
    encoder: list
    decoder: list
    output_projection: np.ndarray | None = None    # [vocab, d] when untied

    def named_tensors(self, config: ModelConfig):
        """Canonical (name, array) order; the LSQW payload order (model.py:154)."""
        yield "token_embedding", self.token_embedding
        if not config.tie_output:
            yield "output_projection", self.output_projection
        for i, lw in enumerate(self.encoder):
            for f in _ENC_FIELDS:
                yield f"encoder.{i}.{f}", getattr(lw, f)
        for i, lw in enumerate(self.decoder):
            for f in _DEC_FIELDS:
                yield f"decoder.{i}.{f}", getattr(lw, f)

    def expected_shapes(self, config: ModelConfig) -> dict:
        d, ff, v = config.d_model, config.d_ff, config.vocab_size
        shapes = {"token_embedding": (v, d)}
        if not config.tie_output:
            shapes["output_projection"] = (v, d)
        enc = {"w_qkv": (d, 3 * d), "b_qkv": (3 * d,), "w_out": (d, d), "b_out": (d,),
               "ln1_gamma": (d,), "ln1_beta": (d,), "w_ff1": (d, ff), "b_ff1": (ff,),
               "w_ff2": (ff, d), "b_ff2": (d,), "ln2_gamma": (d,), "ln2_beta": (d,)}
        dec = {"w_qkv": (d, 3 * d), "b_qkv": (3 * d,), "w_self_out": (d, d), "b_self_out": (d,),
               "ln1_gamma": (d,), "ln1_beta": (d,)}
        for nm in ("cross_q", "cross_k", "cross_v", "cross_out"):
            dec[f"w_{nm}"], dec[f"b_{nm}"] = (d, d), (d,)
        dec.update({"ln2_gamma": (d,), "ln2_beta": (d,), "w_ff1": (d, ff), "b_ff1": (ff,),
                    "w_ff2": (ff, d), "b_ff2": (d,), "ln3_gamma": (d,), "ln3_beta": (d,)})
        for i in range(config.num_encoder_layers):
            shapes.update({f"encoder.{i}.{f}": s for f, s in enc.items()})
        for i in range(config.num_decoder_layers):
            shapes.update({f"decoder.{i}.{f}": s for f, s in dec.items()})
        return shapes

    def validate(self, config: ModelConfig):
        """model.py:189-208."""
        if len(self.encoder) != config.num_encoder_layers:
            raise ConsistencyError(f"{len(self.encoder)} encoder layers, config says "
                                   f"{config.num_encoder_layers}")
        if len(self.decoder) != config.num_decoder_layers:
            raise ConsistencyError(f"{len(self.decoder)} decoder layers, config says "
                                   f"{config.num_decoder_layers}")
        if config.tie_output and self.output_projection is not None:
            raise ConsistencyError("tie_output set but a separate output projection is present")
        if not config.tie_output and self.output_projection is None:
            raise ConsistencyError("untied config requires an output projection")
        expected = self.expected_shapes(config)
        for name, arr in self.named_tensors(config):
            if arr.shape != expected[name]:
                raise ConsistencyError(f"{name}: shape {arr.shape}, expected {expected[name]}")
            if arr.dtype != np.float32:
                raise ConsistencyError(f"{name}: dtype {arr.dtype}, engine computes in float32")
            if not np.isfinite(arr).all():
                raise ConsistencyError(f"{name}: contains non-finite values")

    def output_matrix(self, config: ModelConfig) -> np.ndarray:
        return self.token_embedding if config.tie_output else self.output_projection


def make_random_weights(config: ModelConfig, seed: int = 0) -> ModelWeights:
    """Seeded initialisation with the reference's draw order (model.py:214-260):
    embedding, untied projection, encoder layers, decoder layers; matrices
    N(0, sqrt(2/(m+n))), biases N(0, .02), gamma 1, beta 0, E ~ N(0, 1/sqrt d)."""
    rng = np.random.default_rng(seed)
    d, ff = config.d_model, config.d_ff

    def mat(m, n):
        return rng.normal(0.0, math.sqrt(2.0 / (m + n)), size=(m, n)).astype(F32)

    def vec(n):
        return rng.normal(0.0, 0.02, size=n).astype(F32)

    emb = rng.normal(0.0, 1.0 / math.sqrt(d), size=(config.vocab_size, d)).astype(F32)
    proj = None if config.tie_output else \
        rng.normal(0.0, 1.0 / math.sqrt(d), size=(config.vocab_size, d)).astype(F32)
    one, zero = (lambda: np.ones(d, F32)), (lambda: np.zeros(d, F32))
    enc = []
    for _ in range(config.num_encoder_layers):
        w_qkv, b_qkv, w_out, b_out = mat(d, 3 * d), vec(3 * d), mat(d, d), vec(d)
        w_ff1, b_ff1, w_ff2, b_ff2 = mat(d, ff), vec(ff), mat(ff, d), vec(d)
        enc.append(EncoderLayerWeights(w_qkv, b_qkv, w_out, b_out, one(), zero(),
                                       w_ff1, b_ff1, w_ff2, b_ff2, one(), zero()))
    dec = []
    for _ in range(config.num_decoder_layers):
        w_qkv, b_qkv, w_so, b_so = mat(d, 3 * d), vec(3 * d), mat(d, d), vec(d)
        cross = [(mat(d, d), vec(d)) for _ in range(4)]  # q, k, v, out
        w_ff1, b_ff1, w_ff2, b_ff2 = mat(d, ff), vec(ff), mat(ff, d), vec(d)
        dec.append(DecoderLayerWeights(
            w_qkv, b_qkv, w_so, b_so, one(), zero(),
            cross[0][0], cross[0][1], cross[1][0], cross[1][1],
            cross[2][0], cross[2][1], cross[3][0], cross[3][1], one(), zero(),
            w_ff1, b_ff1, w_ff2, b_ff2, one(), zero()))
    return ModelWeights(token_embedding=emb, encoder=enc, decoder=dec, output_projection=proj)


def sinusoidal_positions(max_len: int, d: int) -> np.ndarray:
    """model.py:263-270 (computed in f64 on the host once, uploaded as fp32)."""
    pos = np.arange(max_len, dtype=np.float64)[:, None]
    ang = pos / np.power(10000.0, np.arange(0, d, 2, dtype=np.float64)[None, :] / d)
    pe = np.zeros((max_len, d), np.float64)
    pe[:, 0::2] = np.sin(ang)
    pe[:, 1::2] = np.cos(ang[:, : d // 2])
    return pe.astype(F32)


def lengths_mask(lengths, seq: int) -> np.ndarray:
    """[batch, seq] additive mask: 0 valid, -inf padding (model.py:273-278)."""
    lengths = np.asarray(lengths, dtype=I64)
    m = np.zeros((lengths.shape[0], seq), dtype=F32)
    m[np.arange(seq)[None, :] >= lengths[:, None]] = -np.inf
    return m


# ---------------------------------------------------------------------------
# device-resident weights
# ---------------------------------------------------------------------------

class X3Weight:
    """An exact-mode GEMM weight: the tf32 hi and lo halves (hi + lo = w to
    2^-22 relative) of the reference's [in, out] matrix, stored K-major
    [out, in] for the 3xTF32 tcgen05 GEMM (fq_split_tf32, once at load)."""

    __slots__ = ("hi", "lo")

    def __init__(self, hi: torch.Tensor, lo: torch.Tensor):
        self.hi, self.lo = hi, lo

    @property
    def shape(self):
        return tuple(self.hi.shape)

    @classmethod
    def from_kn(cls, t: torch.Tensor, transpose: bool = True) -> "X3Weight":
        """Split a device fp32 [K, N] matrix (``transpose``) or [N, K] one."""
        rows, cols = t.shape
        shape = (cols, rows) if transpose else (rows, cols)
        hi = torch.empty(shape, dtype=torch.float32, device=t.device)
        lo = torch.empty_like(hi)
        _abi.call("fq_split_tf32", t.data_ptr(), rows, cols, int(transpose), hi.data_ptr(),
                  lo.data_ptr(), _abi.stream_handle())
        return cls(hi, lo)


class XHWeight:
    """An exact-mode GEMM weight for the 3xFP16 tcgen05 GEMM (fq_gemm_x3h): the
    fp16 pair hi + lo * 2^-11 (22 significant bits) of the reference's [in,
    out] matrix, stored K-major [out, in] (fq_split_f16, once at load)."""

    __slots__ = ("hi", "lo")

    def __init__(self, hi: torch.Tensor, lo: torch.Tensor):
        self.hi, self.lo = hi, lo

    @property
    def shape(self):
        return tuple(self.hi.shape)

    @classmethod
    def from_kn(cls, t: torch.Tensor, transpose: bool = True) -> "XHWeight":
        """Split a device fp32 [K, N] matrix (``transpose``) or [N, K] one."""
        rows, cols = t.shape
        shape = (cols, rows) if transpose else (rows, cols)
        hi = torch.empty(shape, dtype=torch.float16, device=t.device)
        lo = torch.empty_like(hi)
        _abi.call("fq_split_f16", t.data_ptr(), t.stride(0), rows, cols, int(transpose),
                  hi.data_ptr(), lo.data_ptr(), shape[1], _abi.stream_handle())
        return cls(hi, lo)


def xh_attention(config: ModelConfig) -> bool:
    """Exact mode runs attention on 3xFP16 warp MMAs over fp16-pair K/V for
    these head dims; others keep fp32 K/V and the FFMA exact attention."""
    return config.head_dim in (16, 32, 64, 128)


def half_operand(bufs, name: str, shape, half: bool):
    """The fp16 GEMM operand buffer of an fp32 activation: its fp16 copy in
    the fp16 mode, its exact-mode (hi, lo) pair in fp32 mode."""
    if half:
        return bufs.get(name, shape, torch.float16)
    t = bufs.get(name, (2,) + tuple(shape), torch.float16)
    return (t[0], t[1])


def fill_pair(a32, pair):
    """Exact mode: write the fp16 pair of ``a32`` (for producers that do not
    emit it themselves)."""
    if isinstance(pair, tuple):
        split_pair(a32, pair)


class DeviceWeights:
    """Weights uploaded once for one precision (cached per ModelWeights)."""

    _cache: dict = {}

    @classmethod
    def get(cls, config: ModelConfig, weights, precision: str) -> "DeviceWeights":
        if isinstance(weights, DeviceWeights):
            return weights
        # the positions table depends on max_seq_len and the output matrix on
        # tie_output: both belong to the key, not just the weight object
        key = (id(weights), precision, torch.cuda.current_device(), config.max_seq_len,
               config.tie_output, config.d_model)
        dw = cls._cache.get(key)
        if dw is None or dw.host is not weights:
            dw = DeviceWeights(config, weights, precision)
            cls._cache[key] = dw
        return dw

    def __init__(self, config: ModelConfig, weights: ModelWeights, precision: str = "fp32"):
        if precision not in PRECISIONS:
            raise InputError(f"unknown precision {precision!r}")
        self.config, self.host, self.precision = config, weights, precision
        self.half = precision == "fp16"
        dev = torch.device("cuda", torch.cuda.current_device())

        def f32(a):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=F32)).to(dev)

        def mat(a):  # GEMM B operand
            t = f32(a)
            if not self.half:
                return XHWeight.from_kn(t)                 # [N, K] fp16 hi + lo pair
            out = torch.empty((a.shape[1], a.shape[0]), dtype=torch.float16, device=dev)
            _abi.call("fq_cast_f16", t.data_ptr(), a.shape[0], a.shape[1], 1, out.data_ptr(),
                      _abi.stream_handle())
            return out                                     # [N, K] fp16, K-major

        self.embedding = f32(weights.token_embedding)
        out_m = weights.output_matrix(config)
        if self.half:
            self.out_proj = f32(out_m).to(torch.float16)   # [V, d] already K-major
        else:
            self.out_proj = self.embedding if config.tie_output else f32(out_m)
            self.out_xh = XHWeight.from_kn(self.out_proj, transpose=False)  # logits GEMM
        self.positions = f32(sinusoidal_positions(config.max_seq_len, config.d_model))
        self.enc = []
        for lw in weights.encoder:
            self.enc.append({
                "w_qkv": mat(lw.w_qkv), "b_qkv": f32(lw.b_qkv),
                "w_out": mat(lw.w_out), "b_out": f32(lw.b_out),
                "ln1_g": f32(lw.ln1_gamma), "ln1_b": f32(lw.ln1_beta),
                "w_ff1": mat(lw.w_ff1), "b_ff1": f32(lw.b_ff1),
                "w_ff2": mat(lw.w_ff2), "b_ff2": f32(lw.b_ff2),
                "ln2_g": f32(lw.ln2_gamma), "ln2_b": f32(lw.ln2_beta)})
        self.dec = []
        for lw in weights.decoder:
            self.dec.append({
                "w_qkv": mat(lw.w_qkv), "b_qkv": f32(lw.b_qkv),
                "w_so": mat(lw.w_self_out), "b_so": f32(lw.b_self_out),
                "ln1_g": f32(lw.ln1_gamma), "ln1_b": f32(lw.ln1_beta),
                "w_cq": mat(lw.w_cross_q), "b_cq": f32(lw.b_cross_q),
                "w_co": mat(lw.w_cross_out), "b_co": f32(lw.b_cross_out),
                "ln2_g": f32(lw.ln2_gamma), "ln2_b": f32(lw.ln2_beta),
                "w_ff1": mat(lw.w_ff1), "b_ff1": f32(lw.b_ff1),
                "w_ff2": mat(lw.w_ff2), "b_ff2": f32(lw.b_ff2),
                "ln3_g": f32(lw.ln3_gamma), "ln3_b": f32(lw.ln3_beta)})
        if weights.decoder:
            ckv = np.concatenate([np.concatenate([lw.w_cross_k, lw.w_cross_v], axis=1)
                                  for lw in weights.decoder], axis=1)  # [d, 2*L*d]
            bkv = np.concatenate([np.concatenate([lw.b_cross_k, lw.b_cross_v])
                                  for lw in weights.decoder])
            self.w_ckv, self.b_ckv = mat(ckv), f32(bkv)
        torch.cuda.synchronize()

    @property
    def act_dtype(self):
        return torch.float16 if self.half else torch.float32


# ---------------------------------------------------------------------------
# buffer providers
# ---------------------------------------------------------------------------

class HeapBuffers:
    """Fresh device allocations; for standalone op calls and tests."""

    def get(self, name: str, shape, dtype=torch.float32) -> torch.Tensor:
        return torch.empty(tuple(shape), dtype=dtype, device=torch.device("cuda"))


class ArenaBuffers:
    """Views into a planned HBM arena; the zero-allocation inference path."""

    def __init__(self, arena: Arena):
        self.arena = arena

    def get(self, name: str, shape, dtype=torch.float32) -> torch.Tensor:
        return self.arena.acquire(name, shape, dtype).data


def _lin(dw: DeviceWeights, a32, a16, w, out, *, bias=None, residual=None, act="none",
         counters=None, timers=None):
    """One GEMM with fused epilogue in the session precision."""
    if dw.half:
        gemm(a16, w, out, transpose_b=True, bias=bias, residual=residual, activation=act,
             counters=counters, timers=timers)
    elif isinstance(w, XHWeight):  # exact mode: a16 is the activation's fp16 pair
        gemm_xh(a16, w, out, bias=bias, residual=residual, activation=act, counters=counters,
                timers=timers)
    else:
        gemm_x3(a32, w, out, bias=bias, residual=residual, activation=act, counters=counters,
                timers=timers)


def _lin_pair(a16, w, pair, *, bias=None, act="none", counters=None):
    """Exact mode: a 3xFP16 GEMM whose output act(a . w^T + bias) is written
    only as the next GEMM's fp16 pair (fq_gemm_x3h_pair)."""
    hi, lo = a16
    ohi, olo = pair
    M, K = hi.shape
    N = w.shape[0]
    _abi.call("fq_gemm_x3h_pair", hi.data_ptr(), lo.data_ptr(), hi.stride(0), w.hi.data_ptr(),
              w.lo.data_ptr(), w.hi.stride(0), ohi.data_ptr(), olo.data_ptr(), ohi.stride(0), M,
              N, K, _abi.ptr(bias), ACT_IDS[act], _abi.stream_handle())
    (counters or global_counters()).count_gemm(hi.numel() * 4 + N * K * 4 + M * N * 4)


def _ln(x, g, b, eps, out, out16, residual=None, bias=None, counters=None, kind="layer_norm"):
    stream = _abi.stream_handle()
    rows, d = x.shape
    if isinstance(out16, tuple):  # exact mode: the output's fp16 pair for the next GEMM
        if residual is not None:
            raise InputError("bias+residual LN with an fp16 pair output is not fused")
        hi, lo = out16
        _abi.call("fq_layer_norm_xh", x.data_ptr(), x.stride(0), g.data_ptr(), b.data_ptr(), eps,
                  rows, d, _abi.ptr(out), out.stride(0) if out is not None else 0, hi.data_ptr(),
                  lo.data_ptr(), hi.stride(0), stream)
    elif residual is None:
        _abi.call("fq_layer_norm", x.data_ptr(), x.stride(0), g.data_ptr(), b.data_ptr(), eps, rows,
                  d, _abi.ptr(out), out.stride(0) if out is not None else 0, _abi.ptr(out16),
                  out16.stride(0) if out16 is not None else 0, stream)
    else:
        _abi.call("fq_bias_residual_layer_norm", x.data_ptr(), x.stride(0), bias.data_ptr(),
                  residual.data_ptr(), residual.stride(0), g.data_ptr(), b.data_ptr(), eps, rows,
                  d, _abi.ptr(out), out.stride(0) if out is not None else 0, _abi.ptr(out16),
                  out16.stride(0) if out16 is not None else 0, stream)
    (counters or global_counters()).count_fused(kind, x.numel() * 8)


def _lin_ln(dw: DeviceWeights, a32, a16, w, bias, residual, g, b, eps, out, out16, ws, *,
            counters=None, timers=None):
    """GEMM + bias + residual, then LayerNorm: one fq_gemm_ln launch in fp16 mode
    with a statistics workspace (the LN inside the split-K epilogue), else the
    GEMM and the LN kernel."""
    if dw.half and ws is not None:
        M, K = a16.shape
        N = w.shape[0]
        _abi.call("fq_gemm_ln", a16.data_ptr(), a16.stride(0), w.data_ptr(), w.stride(0),
                  bias.data_ptr(), residual.data_ptr(), residual.stride(0), g.data_ptr(),
                  b.data_ptr(), eps, out.data_ptr(), out.stride(0), _abi.ptr(out16),
                  out16.stride(0) if out16 is not None else 0, ws.data_ptr(),
                  ws.numel() * ws.element_size(), M, N, K, _abi.stream_handle())
        (counters or global_counters()).count_fused("layer_norm", M * N * 8)
        return
    if not dw.half and ws is not None and isinstance(w, XHWeight):
        # exact mode: 3xFP16 K-slice slabs + the LN kernel reducing them
        hi, lo = a16
        M, K = hi.shape
        N = w.shape[0]
        ohi, olo = out16 if out16 is not None else (None, None)
        _abi.call("fq_gemm_x3h_ln", hi.data_ptr(), lo.data_ptr(), hi.stride(0), w.hi.data_ptr(),
                  w.lo.data_ptr(), w.hi.stride(0), bias.data_ptr(), residual.data_ptr(),
                  residual.stride(0), g.data_ptr(), b.data_ptr(), eps, out.data_ptr(),
                  out.stride(0), _abi.ptr(ohi), _abi.ptr(olo),
                  ohi.stride(0) if ohi is not None else 0, ws.data_ptr(),
                  ws.numel() * ws.element_size(), M, N, K, _abi.stream_handle())
        (counters or global_counters()).count_gemm(hi.numel() * 4 + N * K * 4 + M * N * 4)
        (counters or global_counters()).count_fused("layer_norm", M * N * 8)
        return
    if not dw.half and ws is not None:  # exact mode: 3xTF32 K-slice slabs + the reducing LN
        M, K = a32.shape
        N = w.shape[0]
        _abi.call("fq_gemm_f32x3_ln", a32.data_ptr(), a32.stride(0), w.hi.data_ptr(),
                  w.lo.data_ptr(), w.hi.stride(0), bias.data_ptr(), residual.data_ptr(),
                  residual.stride(0), g.data_ptr(), b.data_ptr(), eps, out.data_ptr(),
                  out.stride(0), ws.data_ptr(), ws.numel() * ws.element_size(), M, N, K,
                  _abi.stream_handle())
        (counters or global_counters()).count_gemm(a32.numel() * 4 + 2 * N * K * 4 + M * N * 4)
        (counters or global_counters()).count_fused("layer_norm", M * N * 8)
        return
    tmp = out
    _lin(dw, a32, a16, w, tmp, bias=bias, residual=residual, counters=counters, timers=timers)
    _ln(tmp, g, b, eps, out, out16, counters=counters)


def ln_ws_bytes(rows: int, d: int, slabs: bool = True) -> int:
    """fq_gemm_ln workspace. ``slabs``: room for the split-K partial slabs (at
    most 4 K slices of [rows, d] fp32; the default path), else the co-resident
    variant's per-row, per-128-column-tile statistics + counters."""
    stats = rows * ((d + 127) // 128) * 16 + ((rows + 127) // 128) * 8
    return max(stats, 4 * rows * d * 4) if slabs else stats


def _check_tokens(tokens: np.ndarray, config: ModelConfig):
    if tokens.size and (tokens.min() < 0 or tokens.max() >= config.vocab_size):
        raise InputError(f"token id out of range [0, {config.vocab_size})")


# ---------------------------------------------------------------------------
# encoder  (model.py:306-445)
# ---------------------------------------------------------------------------

def encoder_layer_forward(x, layer, config: ModelConfig, mask=None, batch: int = 1, *,
                          prefix: str = "enc.l0", buffers=None, counters=None, timers=None,
                          precision: str = "fp32", x16=None, bad=None):
    """One encoder layer (post-LN): QKV GEMM(+bias) -> fused attention ->
    out GEMM(+bias+residual) -> LN -> FFN1 GEMM(+bias+act) -> FFN2
    GEMM(+bias+residual) -> LN. Returns (out fp32, out fp16 or None).

    ``layer`` is a device layer dict (DeviceWeights.enc[i]) or the reference's
    EncoderLayerWeights (uploaded on the fly)."""
    X = as_device(x, torch.float32)
    n, d = X.shape
    if n % batch:
        raise DimensionError(f"{n} rows not divisible by batch {batch}")
    seq = n // batch
    if batch > config.max_batch or seq > config.max_seq_len:
        raise CapacityError(f"batch {batch} x seq {seq} exceeds configured maxima")
    if isinstance(layer, EncoderLayerWeights):
        tmp = ModelWeights(np.zeros((config.vocab_size, d), F32), [layer], [])
        cfg1 = ModelConfig(**{**config.to_dict(), "num_encoder_layers": 1,
                              "num_decoder_layers": 0})
        layer = DeviceWeights(cfg1, tmp, precision).enc[0]
        dw_half = precision == "fp16"
    else:
        dw_half = not isinstance(layer["w_qkv"], (X3Weight, XHWeight))
    bufs = buffers if buffers is not None else HeapBuffers()
    ctr = counters or global_counters()
    h, hd, ff = config.num_heads, config.head_dim, config.d_ff
    act16 = torch.float16 if dw_half else torch.float32
    if dw_half and x16 is None:
        x16 = X.to(torch.float16)
    if not dw_half and x16 is None:  # exact mode: the input's fp16 pair
        x16 = split_pair(X)
    stream = _abi.stream_handle()

    class _P:  # precision shim for _lin
        half = dw_half

    # Counter contract (reference ops.py:45-58, test_acceptance.py:180-201): 6
    # GEMMs and one pass of each of the 6 FusedPassKinds per layer. Here the
    # passes run as 7 launches: QKV bias + head split in the QKV GEMM's
    # epilogue (heads are strided views), QK^T / softmax / P.V in ONE attention
    # kernel (its two tensor-core products count as the layer's batched GEMMs),
    # the out-projection's bias + residual and FFN1's bias + act in their GEMM
    # epilogues, the closing FFN2 bias + residual + LN in FFN2 + the LN kernel.
    qkv = bufs.get(f"{prefix}.qkv", (n, 3 * d))
    _lin(_P, X, x16, layer["w_qkv"], qkv, bias=layer["b_qkv"], counters=ctr, timers=timers)
    ctr.count_fused("qkv_bias_reshape", n * 3 * d * 8, launches=1)
    ctx = bufs.get(f"{prefix}.ctx", (n, d), act16)
    ctx16 = ctx
    if not dw_half and hd == 64 and seq <= 64:
        # exact mode on 3xFP16 warp MMAs, the ctx written as the GEMM's pair
        ctx16 = half_operand(bufs, f"{prefix}.ctx16", (n, d), False)
        _abi.call("fq_encoder_attention_xh", qkv.data_ptr(), qkv.stride(0), batch, seq, h, hd,
                  attention_scale(hd), _abi.ptr(mask),
                  ctx.data_ptr() if isinstance(layer["w_out"], X3Weight) else None,
                  ctx16[0].data_ptr(),
                  ctx16[1].data_ptr(), d, _abi.ptr(bad), stream)
    else:
        _abi.call("fq_encoder_attention", qkv.data_ptr(), qkv.stride(0), batch, seq, h, hd,
                  attention_scale(hd), _abi.ptr(mask), None if dw_half else ctx.data_ptr(),
                  ctx.data_ptr() if dw_half else None, d, 0 if dw_half else 1, _abi.ptr(bad),
                  stream)
        if not dw_half:
            ctx16 = half_operand(bufs, f"{prefix}.ctx16", (n, d), False)
            fill_pair(ctx, ctx16)
    ctr.count_fused("attention_scale_mask_softmax", n * d * 16)
    ctr.count_gemm(n * d * 8)  # QK^T, inside the fused attention kernel
    ctr.count_gemm(n * d * 8)  # P.V
    res1 = bufs.get(f"{prefix}.res1", (n, d))
    _lin(_P, ctx, ctx16, layer["w_out"], res1, bias=layer["b_out"], residual=X, counters=ctr,
         timers=timers)
    ctr.count_fused("attn_output_bias_residual", n * d * 12)
    norm1 = bufs.get(f"{prefix}.norm1", (n, d))
    norm1_16 = half_operand(bufs, f"{prefix}.norm1_16", (n, d), dw_half)
    _ln(res1, layer["ln1_g"], layer["ln1_b"], config.ln_eps, norm1, norm1_16, counters=ctr)
    if dw_half:
        ffn_h = bufs.get(f"{prefix}.ffn_h", (n, ff), act16)
        _lin(_P, norm1, norm1_16, layer["w_ff1"], ffn_h, bias=layer["b_ff1"],
             act=config.activation, counters=ctr, timers=timers)
        ffn_h16 = ffn_h
    else:  # exact mode: FFN1 writes the pair FFN2 reads, nothing else
        ffn_h = None
        ffn_h16 = half_operand(bufs, f"{prefix}.ffn_h16", (n, ff), False)
        _lin_pair(norm1_16, layer["w_ff1"], ffn_h16, bias=layer["b_ff1"], act=config.activation,
                  counters=ctr)
    ctr.count_fused("ffn_bias_activation", n * ff * 8)
    u = bufs.get(f"{prefix}.ffn_out", (n, d))
    _lin(_P, ffn_h, ffn_h16, layer["w_ff2"], u, bias=layer["b_ff2"], residual=norm1, counters=ctr,
         timers=timers)
    out = bufs.get(f"{prefix}.out", (n, d))
    out16 = half_operand(bufs, f"{prefix}.out16", (n, d), dw_half)
    _ln(u, layer["ln2_g"], layer["ln2_b"], config.ln_eps, out, out16, counters=ctr,
        kind="ffn_bias_residual")
    return out, out16


def encode(tokens, weights, config: ModelConfig, lengths=None, *, engine: str = "fused",
           buffers=None, positions=None, counters=None, timers=None, precision: str = "fp32",
           return_half: bool = False):
    """Stacked encoder over embedded + positional inputs (model.py:407-445).
    Returns the encoder memory [batch*seq, d_model] as a device fp32 tensor
    (plus its fp16 copy when ``return_half``)."""
    if engine != "fused":
        raise InputError("the B200 engine implements the fused path only")
    resident = isinstance(tokens, torch.Tensor) and tokens.is_cuda
    T = tokens if resident else np.asarray(tokens, dtype=I64)
    if T.ndim != 2:
        raise InputError(f"tokens must be [batch, seq], got {tuple(T.shape)}")
    batch, seq = T.shape
    if batch > config.max_batch or seq > config.max_seq_len:
        raise CapacityError(f"batch {batch} x seq {seq} exceeds configured maxima")
    if not resident:
        _check_tokens(T, config)
    dw = DeviceWeights.get(config, weights, precision)
    bufs = buffers if buffers is not None else HeapBuffers()
    ctr = counters or global_counters()
    n, d = batch * seq, config.d_model
    tok = bufs.get("enc.tokens", (n,), torch.int64)
    tok.copy_(T.reshape(-1) if resident else torch.from_numpy(T.reshape(-1)))
    mask = None
    if lengths is not None:
        mask = bufs.get("enc.mask", (batch, seq))
        mask.copy_(torch.from_numpy(lengths_mask(lengths, seq)))
    x = bufs.get("enc.x", (n, d))
    x16 = half_operand(bufs, "enc.x16", (n, d), dw.half)
    pos = as_device(positions, torch.float32) if positions is not None else dw.positions
    _abi.call("fq_embed_scale_pos", tok.data_ptr(), n, dw.embedding.data_ptr(), d,
              float(np.float32(math.sqrt(d))), pos.data_ptr(), 0, None, seq, x.data_ptr(),
              _abi.ptr(x16) if dw.half else None, _abi.stream_handle())
    fill_pair(x, x16)
    ctr.count_fused("embed_scale_pos", n * d * 8)
    bad = bufs.get("enc.bad", (1,), torch.int32)
    bad.zero_()
    for i, lw in enumerate(dw.enc):
        x, x16 = encoder_layer_forward(x, lw, config, mask, batch, prefix=f"enc.l{i}",
                                       buffers=bufs, counters=ctr, timers=timers,
                                       precision=precision, x16=x16, bad=bad)
    if int(bad.item()):
        raise FullMaskError(f"{int(bad.item())} attention row(s) fully masked")
    return (x, x16) if return_half else x


# ---------------------------------------------------------------------------
# decoder  (model.py:452-631)
# ---------------------------------------------------------------------------

class KVCache:
    """Copy-free self-attention cache (replaces model.py:452-512's ping-pong).

    Per decoder layer, K and V live in [max_seq_len, rows, d] (fp32 or fp16):
    slot (t, r) is written once, by row r at step t, inside the attention
    kernel. ``hist[r, t]`` names the physical row holding row r's position t;
    a beam reorder permutes ``hist`` rows (rows x max_len int32) instead of
    copying the K/V history. ``current_len`` grows by one per step; the device
    copy ``d_cur`` lets a captured step graph be replayed."""

    def __init__(self, config: ModelConfig, rows: int, buffers, prefix: str = "dec.cache",
                 precision: str = "fp32"):
        if rows > config.max_rows:
            raise CapacityError(f"{rows} rows exceed max batch*beam {config.max_rows}")
        S, d = config.max_seq_len, config.d_model
        self.config, self.rows, self.max_seq_len = config, rows, S
        # fp16 mode: fp16 [S, rows, d]; exact mode: the fp16 pair planes
        # [2, S, rows, d] (hi, lo) the 3xFP16 attention reads (fp32 [S, rows,
        # d] for head dims it does not cover)
        self.pairs = precision != "fp16" and xh_attention(config)
        self.kv_dtype = torch.float32 if precision != "fp16" and not self.pairs else torch.float16
        shape = (2, S, rows, d) if self.pairs else (S, rows, d)
        self._k = [buffers.get(f"{prefix}.l{i}.k", shape, self.kv_dtype)
                   for i in range(config.num_decoder_layers)]
        self._v = [buffers.get(f"{prefix}.l{i}.v", shape, self.kv_dtype)
                   for i in range(config.num_decoder_layers)]
        self.plane = S * rows * d
        self.hist = buffers.get(f"{prefix}.hist", (rows, S), torch.int32)
        self.d_cur = buffers.get(f"{prefix}.cur", (1,), torch.int32)
        self.reset()

    _IOTA: dict = {}

    def reset(self):
        # hist[r, t] = r: the identity history, from a per-device iota made once
        # (no allocation per request)
        key = (self.hist.device, self.rows)
        iota = KVCache._IOTA.get(key)
        if iota is None:
            iota = torch.arange(self.rows, dtype=torch.int32, device=self.hist.device)
            KVCache._IOTA[key] = iota
        self.hist.copy_(iota[:, None].expand_as(self.hist))
        self.d_cur.zero_()
        self.current_len = 0

    def begin_step(self, parents=None):
        """model.py:480-490: reorder only when parents != arange."""
        if self.current_len >= self.max_seq_len:
            raise CapacityError(f"KV cache full at {self.current_len} positions")
        if parents is not None:
            p = np.asarray(parents, dtype=I64)
            if not np.array_equal(p, np.arange(p.shape[0])):
                c = self.current_len
                idx = torch.from_numpy(p).to(self.hist.device)
                self.hist[:, :c] = self.hist[idx, :c].clone()

    def write(self, layer: int, new_k, new_v, timers=None):
        """Cache refresh (model.py:492-506): this step's K/V ([rows, heads, 1,
        hd] or [rows, d]) into slot (current_len, r) of every row; a pending
        reorder was already applied to ``hist`` by ``begin_step`` (no copy).
        The decode kernels write the slot themselves; this is the API path."""
        c, rows, d = self.current_len, self.rows, self.config.d_model
        for store, new in ((self._k, new_k), (self._v, new_v)):
            x = as_device(new, torch.float32).reshape(rows, d)
            if self.pairs:
                split_pair(x, (store[layer][0][c], store[layer][1][c]))
            else:
                store[layer][c].copy_(x.to(self.kv_dtype))

    def end_step(self):
        _abi.call("fq_step_advance", self.d_cur.data_ptr(), _abi.stream_handle())
        self.current_len += 1

    def _logical(self, store, layer: int) -> torch.Tensor:
        c, rows, h, hd = self.current_len, self.rows, self.config.num_heads, self.config.head_dim
        t = torch.arange(c, device=self.hist.device)
        phys = self.hist[:, :c].long()                       # [rows, c]
        st = store[layer]
        if self.pairs:  # x = hi + lo * 2^-11
            st = st[0].double() + st[1].double() / 2048.0
        g = st[t[None, :], phys]                             # [rows, c, d]
        return g.view(rows, c, h, hd).permute(0, 2, 1, 3).float()

    def k(self, layer: int) -> torch.Tensor:
        """Logical [rows, heads, current_len, hd] keys (gathered; for tests)."""
        return self._logical(self._k, layer)

    def v(self, layer: int) -> torch.Tensor:
        return self._logical(self._v, layer)


def build_cross_kv(memory, weights, config: ModelConfig, batch: int, seq: int, *,
                   buffers=None, counters=None, timers=None, precision: str = "fp32",
                   memory16=None):
    """Project the encoder memory into every decoder layer's cross K/V in ONE
    GEMM against the concatenated [d, 2*L*d] weight (model.py:515-534 runs
    2*L). Returns the packed [batch*seq, 2*L*d] tensor; layer i's K is columns
    [2*i*d, (2*i+1)*d) and V the next d columns — head h of item b at
    ``packed[b*seq:(b+1)*seq, off + h*hd : off + (h+1)*hd]``, the reference's
    [batch, heads, seq, hd] as a strided view (``cross_views``)."""
    dw = DeviceWeights.get(config, weights, precision)
    bufs = buffers if buffers is not None else HeapBuffers()
    M = as_device(memory, torch.float32)
    n, d, L = batch * seq, config.d_model, config.num_decoder_layers
    if not dw.half and xh_attention(config):  # exact: the fp16 pair planes [2, n, 2*L*d]
        if memory16 is None:
            memory16 = split_pair(M)
        pair = bufs.get("dec.cross_kv16", (2, n, 2 * L * d), torch.float16)
        _lin_pair(memory16, dw.w_ckv, (pair[0], pair[1]), bias=dw.b_ckv, counters=counters)
        return pair
    packed = bufs.get("dec.cross_kv", (n, 2 * L * d), dw.act_dtype)
    if memory16 is None:
        memory16 = M.to(torch.float16) if dw.half else split_pair(M)
    _lin(dw, M, memory16, dw.w_ckv, packed, bias=dw.b_ckv, counters=counters, timers=timers)
    return packed


def cross_views(packed: torch.Tensor, config: ModelConfig, batch: int, seq: int):
    """[(ck, cv)] per layer as [batch, heads, seq, hd] strided views (model.py:525-531)."""
    d, h, hd = config.d_model, config.num_heads, config.head_dim
    ld = packed.stride(0)
    out = []
    for i in range(config.num_decoder_layers):
        views = []
        for j in range(2):
            base = packed[:, (2 * i + j) * d:(2 * i + j + 1) * d]
            views.append(base.as_strided((batch, h, seq, hd), (seq * ld, hd, ld, 1)))
        out.append(tuple(views))
    return out


class DecoderStep:
    """The device decoder step over all rows (model.py:537-631). Holds the
    arena views it writes so a CUDA graph of :meth:`run` can be replayed."""

    def __init__(self, dw: DeviceWeights, config: ModelConfig, batch: int, beam: int,
                 enc_seq: int, cache: KVCache, cross_packed: torch.Tensor, enc_mask, buffers,
                 counters=None, timers=None, fuse_ln: bool = True):
        self.dw, self.config = dw, config
        self.batch, self.beam, self.rows, self.enc_seq = batch, beam, batch * beam, enc_seq
        self.cache, self.cross, self.mask = cache, cross_packed, enc_mask
        self.counters, self.timers = counters or global_counters(), timers
        R, d, ff, V = self.rows, config.d_model, config.d_ff, config.vocab_size
        b = buffers
        a16 = dw.act_dtype
        self.tokens = b.get("dec.tokens", (R,), torch.int64)
        self.x = b.get("dec.x", (R, d))
        hf = dw.half
        # fp16 GEMM operands: fp16 copies (fp16 mode) or exact-mode (hi, lo) pairs
        self.x16 = half_operand(b, "dec.x16", (R, d), hf)
        self.sqkv = b.get("dec.sqkv", (R, 3 * d))
        self.sctx = b.get("dec.sctx", (R, d), a16)
        self.sres = b.get("dec.sres", (R, d))
        self.snorm = b.get("dec.snorm", (R, d))
        self.snorm16 = half_operand(b, "dec.snorm16", (R, d), hf)
        self.cq = b.get("dec.cq", (R, d))
        self.cctx = b.get("dec.cctx", (R, d), a16)
        self.cres = b.get("dec.cres", (R, d))
        self.cnorm = b.get("dec.cnorm", (R, d))
        self.cnorm16 = half_operand(b, "dec.cnorm16", (R, d), hf)
        self.ffn_h = b.get("dec.ffn_h", (R, ff), a16)
        self.sctx16 = self.sctx if hf else half_operand(b, "dec.sctx16", (R, d), False)
        self.cctx16 = self.cctx if hf else half_operand(b, "dec.cctx16", (R, d), False)
        self.ffn_h16 = self.ffn_h if hf else half_operand(b, "dec.ffn_h16", (R, ff), False)
        self.u = b.get("dec.ffn_out", (R, d))
        self.logits = b.get("dec.logits", (R, V))
        self.bad = b.get("dec.bad", (1,), torch.int32)
        # GEMM + LN pairs as fq_gemm_ln. Default (fp16): the split-K GEMM writes
        # one partial slab per K slice and the LN kernel reduces them, so the
        # GEMM has no in-kernel (DSMEM) reduction. FQ_FUSE_LN=coresident: the LN
        # inside the split-K epilogue, measured slower at C2 (152k vs 165k
        # tok/s: the row block's statistics exchange waits for its slowest CTA).
        # FQ_FUSE_LN=0: GEMM with the reduction, then the LN kernel.
        self.ln_ws = None
        mode = os.environ.get("FQ_FUSE_LN", "slab")
        if fuse_ln and mode != "0" and (dw.half or mode == "slab"):
            # exact mode: the 3xTF32 split-K slabs summed by the LN kernel
            ws = b.get("dec.ln_ws", ((ln_ws_bytes(R, d) + 3) // 4,), torch.int32)
            if mode == "coresident":
                ws = ws[:(ln_ws_bytes(R, d, slabs=False) + 3) // 4]
                ws.zero_()
            self.ln_ws = ws
        # the cross-attention query GEMM as K-slice slabs summed by the
        # cross-attention kernel (no in-GEMM reduction), same bits
        self.q_slabs = (dw.half and self.ln_ws is not None and mode != "coresident" and
                        config.head_dim == 64 and beam <= 8 and enc_seq <= 64)
        self._nslab = ctypes.c_int(0)

    def _exact_layer(self, i, lw, x, x16, scale, stream):
        """One decoder layer after its QKV GEMM in exact mode: attention on the
        fp16 pair cache / cross K/V (fq_*_attention_xh, ctx emitted as pairs),
        the 3xFP16 GEMMs, and the split-K slab LNs emitting the next pairs."""
        c, dw, ctr, tm = self.config, self.dw, self.counters, self.timers
        R, d, h, hd = self.rows, c.d_model, c.num_heads, c.head_dim
        k, v = self.cache._k[i], self.cache._v[i]
        sh, sl = self.sctx16
        if self.beam > 1 and hd == 64 and _SELF_ITEMS:  # beams share history slots
            _abi.call("fq_decoder_self_attention_xh_items", self.sqkv.data_ptr(),
                      self.sqkv.stride(0), k.data_ptr(), v.data_ptr(), self.cache.plane,
                      self.cache.hist.data_ptr(), self.cache.d_cur.data_ptr(), self.batch,
                      self.beam, h, hd, c.max_seq_len, scale, None, sh.data_ptr(), sl.data_ptr(),
                      sh.stride(0), stream)
        else:
            _abi.call("fq_decoder_self_attention_xh", self.sqkv.data_ptr(), self.sqkv.stride(0),
                      k.data_ptr(), v.data_ptr(), self.cache.plane, self.cache.hist.data_ptr(),
                      self.cache.d_cur.data_ptr(), R, h, hd, c.max_seq_len, scale, None,
                      sh.data_ptr(), sl.data_ptr(), sh.stride(0), stream)
        ctr.count_fused("decoder_self_attention", R * d * 16)
        _lin_ln(dw, self.sctx, self.sctx16, lw["w_so"], lw["b_so"], x, lw["ln1_g"], lw["ln1_b"],
                c.ln_eps, self.snorm, self.snorm16, self.ln_ws, counters=ctr, timers=tm)
        cr = self.cross  # [2, n, 2*L*d] pair planes
        ld = cr.stride(1)
        ch, cl = self.cctx16
        # the cross query GEMM as its split-K slabs (in the LN workspace, free
        # between LN1 and the cross-out GEMM), summed + biased by the
        # cross-attention's query load: no DSMEM reduction, same bits
        nsl = ctypes.c_int32(0)
        qh, ql = self.snorm16
        w_cq = lw["w_cq"]
        rc = -1
        if self.ln_ws is not None:
            rc = _abi.lib_call_rc("fq_gemm_x3h_slabs", qh.data_ptr(), ql.data_ptr(), qh.stride(0),
                                  w_cq.hi.data_ptr(), w_cq.lo.data_ptr(), w_cq.hi.stride(0),
                                  self.ln_ws.data_ptr(), self.ln_ws.numel() * 4, R, d, d,
                                  ctypes.addressof(nsl), stream)
        if rc == 0:
            ctr.count_gemm(R * d * 4 + d * d * 4 + R * d * 4)
            _abi.call("fq_cross_attention_xh_slabs", self.ln_ws.data_ptr(), nsl.value, d, R * d,
                      lw["b_cq"].data_ptr(), cr[0, :, 2 * i * d:].data_ptr(),
                      cr[0, :, (2 * i + 1) * d:].data_ptr(), cr.stride(0), ld, self.batch,
                      self.beam, self.enc_seq, h, hd, scale, _abi.ptr(self.mask), None,
                      ch.data_ptr(), cl.data_ptr(), ch.stride(0), self.bad.data_ptr(), stream)
        else:
            _lin(dw, self.snorm, self.snorm16, w_cq, self.cq, bias=lw["b_cq"], counters=ctr,
                 timers=tm)
            _abi.call("fq_cross_attention_xh", self.cq.data_ptr(), self.cq.stride(0),
                      cr[0, :, 2 * i * d:].data_ptr(), cr[0, :, (2 * i + 1) * d:].data_ptr(),
                      cr.stride(0), ld, self.batch, self.beam, self.enc_seq, h, hd, scale,
                      _abi.ptr(self.mask), None, ch.data_ptr(), cl.data_ptr(), ch.stride(0),
                      self.bad.data_ptr(), stream)
        ctr.count_fused("cross_attention", R * d * 16)
        _lin_ln(dw, self.cctx, self.cctx16, lw["w_co"], lw["b_co"], self.snorm, lw["ln2_g"],
                lw["ln2_b"], c.ln_eps, self.cnorm, self.cnorm16, self.ln_ws, counters=ctr,
                timers=tm)
        _lin_pair(self.cnorm16, lw["w_ff1"], self.ffn_h16, bias=lw["b_ff1"], act=c.activation,
                  counters=ctr)
        _lin_ln(dw, self.ffn_h, self.ffn_h16, lw["w_ff2"], lw["b_ff2"], self.cnorm, lw["ln3_g"],
                lw["ln3_b"], c.ln_eps, self.x, self.x16, self.ln_ws, counters=ctr, timers=tm)

    def embed(self):
        """Decoder input of the current position (model.py:559)."""
        c, dw = self.config, self.dw
        R, d = self.rows, c.d_model
        _abi.call("fq_embed_scale_pos", self.tokens.data_ptr(), R, dw.embedding.data_ptr(), d,
                  float(np.float32(math.sqrt(d))), dw.positions.data_ptr(), 0,
                  self.cache.d_cur.data_ptr(), 1, self.x.data_ptr(),
                  _abi.ptr(self.x16) if dw.half else None, _abi.stream_handle())
        self.counters.count_fused("embed_scale_pos", R * d * 8)
        fill_pair(self.x, self.x16)  # exact mode: the step input's fp16 pair

    def run(self, embed: bool = True, logits: bool = True):
        """Embed -> L decoder layers -> logits. Position comes from cache.d_cur.
        ``embed=False``: the input rows (and in exact mode their fp16 pair) were
        already written by the previous step's fused HARS launch (fq_hars_step /
        fq_hars_merge_step) or by :meth:`embed`. ``logits=False``: stop after the
        layers (the output layer runs as fq_logits_hars on ``x16``)."""
        c, dw, ctr, tm = self.config, self.dw, self.counters, self.timers
        R, d, h, hd, L = self.rows, c.d_model, c.num_heads, c.head_dim, c.num_decoder_layers
        stream = _abi.stream_handle()
        scale = attention_scale(hd)
        kvdt = 0 if self.cache.kv_dtype == torch.float32 else 1
        exact = 0 if dw.half else 1
        if embed:
            self.embed()
        x, x16 = self.x, self.x16
        for i, lw in enumerate(dw.dec):
            _lin(dw, x, x16, lw["w_qkv"], self.sqkv, bias=lw["b_qkv"], counters=ctr, timers=tm)
            if self.cache.pairs:  # exact mode: 3xFP16 warp-MMA attention on the pair cache
                self._exact_layer(i, lw, x, x16, scale, stream)
                x, x16 = self.x, self.x16
                continue
            _abi.call("fq_decoder_self_attention", self.sqkv.data_ptr(), self.sqkv.stride(0),
                      self.cache._k[i].data_ptr(), self.cache._v[i].data_ptr(), kvdt,
                      self.cache.hist.data_ptr(), self.cache.d_cur.data_ptr(), R, h, hd,
                      c.max_seq_len, scale, None if dw.half else self.sctx.data_ptr(),
                      self.sctx.data_ptr() if dw.half else None, d, exact, stream)
            ctr.count_fused("decoder_self_attention", R * d * 16)
            fill_pair(self.sctx, self.sctx16)
            if self.ln_ws is not None:
                _lin_ln(dw, self.sctx, self.sctx16, lw["w_so"], lw["b_so"], x, lw["ln1_g"],
                        lw["ln1_b"], c.ln_eps, self.snorm, self.snorm16, self.ln_ws,
                        counters=ctr, timers=tm)
            else:
                _lin(dw, self.sctx, self.sctx16, lw["w_so"], self.sres, bias=lw["b_so"],
                     residual=x, counters=ctr, timers=tm)
                _ln(self.sres, lw["ln1_g"], lw["ln1_b"], c.ln_eps, self.snorm, self.snorm16,
                    counters=ctr)
            ld = self.cross.stride(0)
            ck = self.cross[:, 2 * i * d:]
            cv = self.cross[:, (2 * i + 1) * d:]
            nsl = 0
            if self.q_slabs:
                w = lw["w_cq"]
                _abi.call("fq_gemm_splitk_slabs", self.snorm16.data_ptr(), self.snorm16.stride(0),
                          w.data_ptr(), w.stride(0), self.ln_ws.data_ptr(),
                          self.ln_ws.numel() * self.ln_ws.element_size(), R, d, d,
                          ctypes.addressof(self._nslab), stream)
                nsl = self._nslab.value
            if nsl:
                ctr.count_gemm((R * d + d * d) * 2 + 4 * R * d * 4)
                _abi.call("fq_cross_attention_slabs", self.ln_ws.data_ptr(), nsl, d,
                          lw["b_cq"].data_ptr(), ck.data_ptr(), cv.data_ptr(), ld, self.batch,
                          self.beam, self.enc_seq, h, hd, scale, _abi.ptr(self.mask), None,
                          self.cctx.data_ptr(), d, self.bad.data_ptr(), stream)
            else:
                _lin(dw, self.snorm, self.snorm16, lw["w_cq"], self.cq, bias=lw["b_cq"],
                     counters=ctr, timers=tm)
                _abi.call("fq_cross_attention", self.cq.data_ptr(), self.cq.stride(0),
                          ck.data_ptr(), cv.data_ptr(), kvdt, ld, self.batch, self.beam,
                          self.enc_seq, h, hd, scale, _abi.ptr(self.mask),
                          None if dw.half else self.cctx.data_ptr(),
                          self.cctx.data_ptr() if dw.half else None, d, exact,
                          self.bad.data_ptr(), stream)
            ctr.count_fused("cross_attention", R * d * 16)
            fill_pair(self.cctx, self.cctx16)
            if self.ln_ws is not None:
                _lin_ln(dw, self.cctx, self.cctx16, lw["w_co"], lw["b_co"], self.snorm,
                        lw["ln2_g"], lw["ln2_b"], c.ln_eps, self.cnorm, self.cnorm16,
                        self.ln_ws, counters=ctr, timers=tm)
            else:
                _lin(dw, self.cctx, self.cctx16, lw["w_co"], self.cres, bias=lw["b_co"],
                     residual=self.snorm, counters=ctr, timers=tm)
                _ln(self.cres, lw["ln2_g"], lw["ln2_b"], c.ln_eps, self.cnorm, self.cnorm16,
                    counters=ctr)
            _lin(dw, self.cnorm, self.cnorm16, lw["w_ff1"], self.ffn_h, bias=lw["b_ff1"],
                 act=c.activation, counters=ctr, timers=tm)
            fill_pair(self.ffn_h, self.ffn_h16)
            if self.ln_ws is not None:
                _lin_ln(dw, self.ffn_h, self.ffn_h16, lw["w_ff2"], lw["b_ff2"], self.cnorm,
                        lw["ln3_g"], lw["ln3_b"], c.ln_eps, self.x, self.x16, self.ln_ws,
                        counters=ctr, timers=tm)
            else:
                _lin(dw, self.ffn_h, self.ffn_h16, lw["w_ff2"], self.u, bias=lw["b_ff2"],
                     residual=self.cnorm, counters=ctr, timers=tm)
                _ln(self.u, lw["ln3_g"], lw["ln3_b"], c.ln_eps, self.x, self.x16, counters=ctr)
            x, x16 = self.x, self.x16
        if not logits:
            return None
        _lin(dw, x, x16, dw.out_proj if dw.half else dw.out_xh, self.logits, counters=ctr,
             timers=tm)
        return self.logits


def decode_step(last_tokens, cache: KVCache, cross_kv, enc_mask, weights, config: ModelConfig,
                batch: int, beam: int, *, parents=None, buffers=None, positions=None,
                counters=None, timers=None, precision: str = "fp32", enc_seq: int | None = None):
    """One incremental decoder step over all batch*beam rows (model.py:537-631).
    ``cross_kv`` is the packed tensor from :func:`build_cross_kv`. Returns the
    device logits [batch*beam, vocab] (fp32)."""
    T = np.asarray(last_tokens, dtype=I64)
    rows = T.shape[0]
    if rows != batch * beam:
        raise DimensionError(f"{rows} rows != batch {batch} x beam {beam}")
    _check_tokens(T, config)
    dw = DeviceWeights.get(config, weights, precision)
    bufs = buffers if buffers is not None else HeapBuffers()
    if enc_seq is None:
        enc_seq = cross_kv.shape[-2] // batch
    cache.begin_step(parents)
    step = DecoderStep(dw, config, batch, beam, enc_seq, cache, cross_kv, enc_mask, bufs,
                       counters, timers)
    step.tokens.copy_(torch.from_numpy(T))
    step.bad.zero_()
    logits = step.run()
    if int(step.bad.item()):
        raise FullMaskError("fully masked cross-attention row")
    cache.end_step()
    return logits


# ---------------------------------------------------------------------------
# static intermediate enumeration for the arena  (model.py:772-860)
# ---------------------------------------------------------------------------

LH_SV_CAP = 128  # fq_logits_hars survivor slots per (row, column tile)


def logits_hars_tiles(config: ModelConfig, precision: str) -> int:
    """Column tiles per row of the fused logits + HARS stage-1 output layer
    (fq_logits_hars: 224-wide fp16 tiles; fq_logits_hars_x3h: 128-wide exact
    tiles), or 0 when the shape keeps the materialised logits."""
    V, d = config.vocab_size, config.d_model
    if precision == "fp16":
        ok = d % 64 == 0 and V >= 4096 and (V + 223) // 224 <= 256
        return (V + 223) // 224 if ok else 0
    ok = V % 128 == 0 and V >= 4096 and V // 128 <= 256 and d % 64 == 0
    return V // 128 if ok else 0


def plan_intermediates(config: ModelConfig, precision: str = "fp32",
                       batch: int | None = None) -> list[IntermediateSpec]:
    """Every intermediate of one max-shape request with its lifetime in the
    static op order: embed, encoder layers, cross-K/V setup, one decode step
    (steps reuse the same buffers), logits, HARS stage 1/2 and the beam state.
    Whole-request buffers (mask, cross K/V, KV cache, history table, beam
    state) live to the terminal op and are never shared."""
    B = config.max_batch if batch is None else int(batch)
    if not 0 < B <= config.max_batch:
        raise CapacityError(f"batch bucket {B} outside [1, {config.max_batch}]")
    S, K = config.max_seq_len, config.max_beam_size
    R = B * K
    d, ff, V = config.d_model, config.d_ff, config.vocab_size
    L, D = config.num_encoder_layers, config.num_decoder_layers
    bf = precision == "fp16"
    a = 2 if bf else 4  # activation bytes feeding GEMMs / attention
    h = 2 if bf else 4  # fp16 GEMM operand bytes: fp16 copy, or the exact mode's (hi, lo) pair
    n = B * S
    specs: list[IntermediateSpec] = []

    def add(name, nbytes, first, last):
        specs.append(IntermediateSpec(name, (int(nbytes) + 63) // 64 * 64, first, last))

    enc0 = 1
    setup = enc0 + 8 * L
    dec0 = setup + 2
    end = dec0 + 12 * max(D, 1) + 4
    add("enc.tokens", n * 8, 0, 0)
    add("enc.mask", n * 4, 0, end)
    add("enc.bad", 4, 0, setup)
    add("enc.x", n * d * 4, 0, enc0 + 2)
    add("enc.x16", n * d * h, 0, enc0)
    for i in range(L):
        b0 = enc0 + 8 * i
        add(f"enc.l{i}.qkv", n * 3 * d * 4, b0, b0 + 1)
        add(f"enc.l{i}.ctx", n * d * a, b0 + 1, b0 + 2)
        if not bf:
            add(f"enc.l{i}.ctx16", n * d * h, b0 + 1, b0 + 2)
        add(f"enc.l{i}.res1", n * d * 4, b0 + 2, b0 + 3)
        add(f"enc.l{i}.norm1", n * d * 4, b0 + 3, b0 + 5)
        add(f"enc.l{i}.norm1_16", n * d * h, b0 + 3, b0 + 4)
        if bf:
            add(f"enc.l{i}.ffn_h", n * ff * a, b0 + 4, b0 + 5)
        else:
            add(f"enc.l{i}.ffn_h16", n * ff * h, b0 + 4, b0 + 5)
        add(f"enc.l{i}.ffn_out", n * d * 4, b0 + 5, b0 + 6)
        last = setup if i == L - 1 else b0 + 8 + 2
        add(f"enc.l{i}.out", n * d * 4, b0 + 6, last)
        add(f"enc.l{i}.out16", n * d * h, b0 + 6, setup if i == L - 1 else b0 + 8)
    if D:
        if bf:
            add("dec.cross_kv", n * 2 * D * d * 2, setup, end)
        elif xh_attention(config):  # exact: the GEMM writes the pair planes the attention reads
            add("dec.cross_kv16", n * 2 * D * d * 4, setup, end)
        else:
            add("dec.cross_kv", n * 2 * D * d * 4, setup, end)
        kv = 2 if bf else 4
        for i in range(D):
            add(f"dec.cache.l{i}.k", S * R * d * kv, setup, end)
            add(f"dec.cache.l{i}.v", S * R * d * kv, setup, end)
        add("dec.cache.hist", R * S * 4, setup, end)
        add("dec.cache.cur", 4, setup, end)
        add("dec.tokens", R * 8, setup, end)
        add("dec.parents", R * 8, setup, end)
        add("dec.bad", 4, setup, end)
        add("dec.x", R * d * 4, dec0, end)
        add("dec.x16", R * d * h, dec0, end)
        for nm, sz in (("sqkv", R * 3 * d * 4), ("sctx", R * d * a), ("sres", R * d * 4),
                       ("snorm", R * d * 4), ("cq", R * d * 4), ("cctx", R * d * a),
                       ("cres", R * d * 4), ("cnorm", R * d * 4), ("ffn_h", R * ff * a),
                       ("ffn_out", R * d * 4)):
            add(f"dec.{nm}", sz, dec0, end - 3)
        add("dec.ln_ws", ln_ws_bytes(R, d), dec0, end - 3)  # split-K slabs (both modes)
        add("dec.snorm16", R * d * h, dec0, end - 3)
        add("dec.cnorm16", R * d * h, dec0, end - 3)
        if not bf:
            for nm, sz in (("sctx16", R * d * h), ("cctx16", R * d * h), ("ffn_h16", R * ff * h)):
                add(f"dec.{nm}", sz, dec0, end - 3)
        add("dec.logits", R * V * 4, end - 3, end)
        # HARS stage 1 / 2 and the device beam state (whole request)
        add("hars.k", R * 4, setup, end)  # persists across steps (fq_hars_merge_step)
        add("hars.len_pow", (S + 1) * 8, setup, end)
        add("hars.counters", (B + 1 + R) * 4, setup, end)
        add("hars.lse", R * 8, end - 2, end)
        add("hars.cand_idx", R * V * 4, end - 2, end)
        add("hars.cand_count", R * 8, end - 2, end)
        ldt = logits_hars_tiles(config, precision)
        if ldt:  # fq_logits_hars(_x3h) statistics (the fused logits + HARS stage-1 layer)
            add("hars.gmax", R * 32 * 4, setup, end)
            add("hars.tmax", R * ldt * 4, end - 3, end)
            add("hars.tsum", R * ldt * 8, end - 3, end)
            add("hars.svcnt", R * ldt * 4, end - 3, end)
            add("hars.sv", R * ldt * LH_SV_CAP * 8, end - 3, end)
            add("hars.ovf", 4, setup, end)
        for nm, sz in (("live", B * 4), ("step", B * 4), ("done", B * 4),
                       ("prefix", B * K * S * 4), ("cum", B * K * 8), ("fin_count", B * 4),
                       ("fin_tok", B * K * S * 4), ("fin_len", B * K * 4),
                       ("fin_score", B * K * 8), ("last_tok", B * K * 4), ("parent", B * K * 4),
                       ("n_done", 4)):
            add(f"beam.{nm}", sz, setup, end)
    return specs
