"""Device tensor views, GEMM, and instrumentation counters.

Mirrors pkg/src/fuseq/tensor.py: a :class:`Tensor` is a non-owning view (here
of device memory held by the session arena), ``gemm``/``gemm_batched`` keep
the reference's contract checks (shape, aliasing; tensor.py:173-227) and
count one call each, but the math runs in ``libfq_b200.so``: fp32 operands
take the exact-mode FFMA kernel, fp16 operands the tcgen05 tensor-core kernel.
``gemm`` additionally accepts a fused epilogue (bias, activation, residual):
the same fp32 operations the reference performs in the following
``bias_residual_act`` pass (kernels.py:39-53), fused into the GEMM store.
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from .errors import AliasingError, DimensionError

ACT_IDS = {"none": 0, "relu": 1, "gelu": 2}
_DT = {torch.float32: 0, torch.float16: 1}


@dataclass
class Tensor:
    """Shaped view over externally owned (arena) storage. Never owns memory."""

    data: torch.Tensor

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(self.data.shape)

    @property
    def strides(self) -> tuple[int, ...]:
        return tuple(self.data.stride())

    @property
    def nbytes(self) -> int:
        return self.data.numel() * self.data.element_size()

    def numpy(self) -> np.ndarray:
        return self.data.detach().float().cpu().numpy() if self.data.dtype == torch.float16 \
            else self.data.detach().cpu().numpy()


def device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def as_device(x, dtype=None) -> torch.Tensor:
    """Tensor / torch / numpy -> device torch tensor (numpy is copied in)."""
    if isinstance(x, Tensor):
        x = x.data
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(x))
    if not t.is_cuda:
        t = t.to(device(), non_blocking=False)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    if t.is_contiguous() and t.dim() > 1 and 1 in t.shape:
        # size-1 axes may carry any stride (numpy's x[None, :] gives 0); the
        # ABI reads leading dims from strides, so give them canonical values
        canon, acc = [], 1
        for s in reversed(t.shape):
            canon.append(acc)
            acc *= s
        t = t.as_strided(t.shape, tuple(reversed(canon)))
    return t


def writeback(out, dev: torch.Tensor):
    """The reference's ``out=`` contract for host arrays: a numpy ``out`` is
    written in place (the kernel ran on its device copy)."""
    if isinstance(out, np.ndarray):
        out[...] = dev.detach().cpu().numpy().reshape(out.shape)
    elif isinstance(out, Tensor) and not out.data.is_cuda:
        out.data.copy_(dev)
    elif isinstance(out, torch.Tensor) and not out.is_cuda:
        out.copy_(dev)


class OpCounters:
    """Monotonic instrumentation counters, guarded for concurrent use (tensor.py:58-110)."""

    def __init__(self):
        self._lock = threading.Lock()
        self.reset()

    def count_gemm(self, nbytes: int):
        with self._lock:
            self.gemm_calls += 1
            self.bytes_moved_estimate += nbytes

    def count_fused(self, kind: str, nbytes: int, launches: int = 1):
        with self._lock:
            self.fused_passes += launches
            self.bytes_moved_estimate += nbytes
            self.fused_kind_counts[kind] = self.fused_kind_counts.get(kind, 0) + launches

    def count_naive(self, kind: str, passes: int, nbytes: int, intermediates: int = 0):
        with self._lock:
            self.naive_passes += passes
            self.bytes_moved_estimate += nbytes
            self.naive_intermediates += intermediates
            self.naive_kind_counts[kind] = self.naive_kind_counts.get(kind, 0) + passes

    def reset(self):
        self.gemm_calls = 0
        self.fused_passes = 0
        self.naive_passes = 0
        self.bytes_moved_estimate = 0
        self.naive_intermediates = 0
        self.fused_kind_counts: dict[str, int] = {}
        self.naive_kind_counts: dict[str, int] = {}

    def snapshot(self) -> "CounterSnapshot":
        with self._lock:
            return CounterSnapshot(self.gemm_calls, self.fused_passes, self.naive_passes,
                                   self.bytes_moved_estimate, self.naive_intermediates,
                                   dict(self.fused_kind_counts), dict(self.naive_kind_counts))


@dataclass(frozen=True)
class CounterSnapshot:
    gemm_calls: int
    fused_passes: int
    naive_passes: int
    bytes_moved_estimate: int
    naive_intermediates: int
    fused_kind_counts: dict
    naive_kind_counts: dict

    def delta(self, earlier: "CounterSnapshot") -> "CounterSnapshot":
        def d(a, b):
            return {k: v - b.get(k, 0) for k, v in a.items() if v - b.get(k, 0)}
        return CounterSnapshot(self.gemm_calls - earlier.gemm_calls,
                               self.fused_passes - earlier.fused_passes,
                               self.naive_passes - earlier.naive_passes,
                               self.bytes_moved_estimate - earlier.bytes_moved_estimate,
                               self.naive_intermediates - earlier.naive_intermediates,
                               d(self.fused_kind_counts, earlier.fused_kind_counts),
                               d(self.naive_kind_counts, earlier.naive_kind_counts))


class Timers:
    """Profiling buckets (tensor.py:142-155). Device work is bracketed with CUDA
    events on the launching stream; ``get`` resolves them (one sync)."""

    def __init__(self):
        self.buckets: dict[str, float] = {}
        self._pending: list[tuple[str, torch.cuda.Event, torch.cuda.Event]] = []

    def add(self, bucket: str, seconds: float):
        self.buckets[bucket] = self.buckets.get(bucket, 0.0) + seconds

    def start(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def stop(self, bucket: str, start_event):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self._pending.append((bucket, start_event, e))

    def _resolve(self):
        if self._pending:
            torch.cuda.synchronize()
            for b, s, e in self._pending:
                self.add(b, s.elapsed_time(e) / 1e3)
            self._pending = []

    def get(self, bucket: str) -> float:
        self._resolve()
        return self.buckets.get(bucket, 0.0)

    def reset(self):
        self.buckets = {}
        self._pending = []


_global_counters = OpCounters()


def global_counters() -> OpCounters:
    return _global_counters


def reset_counters(counters: OpCounters | None = None):
    (counters or _global_counters).reset()


def read_counters(counters: OpCounters | None = None) -> CounterSnapshot:
    return (counters or _global_counters).snapshot()


def _span(t: torch.Tensor) -> tuple[int, int]:
    """[first byte, last byte + 1) touched by a strided view."""
    if t.numel() == 0:
        return (t.data_ptr(), t.data_ptr())
    hi = sum((s - 1) * st for s, st in zip(t.shape, t.stride()) if st > 0)
    return (t.data_ptr(), t.data_ptr() + (hi + 1) * t.element_size())


def _check_no_alias(out: torch.Tensor, *inputs: torch.Tensor):
    o0, o1 = _span(out)
    for a in inputs:
        a0, a1 = _span(a)
        if o0 < a1 and a0 < o1:
            raise AliasingError("gemm output overlaps an input buffer")


def _row_major(t: torch.Tensor, what: str) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise DimensionError(f"{what} must be a 2D view with unit column stride")
    return t.stride(0)


def gemm(a, b, out, *, transpose_b: bool = False, accumulate: bool = False,
         counters: OpCounters | None = None, timers: Timers | None = None,
         bias=None, residual=None, activation: str = "none"):
    """out = act(a @ op(b) (+ out) (+ bias)) (+ residual), one library call.

    fp32 a/b: exact-mode FFMA GEMM. fp16 a/b: tcgen05 GEMM (b must be the
    K-major [N, K] weight, i.e. ``transpose_b=True``). One call increments
    ``gemm_calls`` by one (tensor.py:204)."""
    A, B, O = as_device(a), as_device(b), as_device(out)
    if A.dim() != 2 or B.dim() != 2 or O.dim() != 2:
        raise DimensionError(f"gemm expects 2D operands, got {A.dim()}/{B.dim()}/{O.dim()}D")
    K = A.shape[1]
    N = B.shape[0] if transpose_b else B.shape[1]
    if (B.shape[1] if transpose_b else B.shape[0]) != K:
        raise DimensionError(f"gemm inner dims differ: {tuple(A.shape)} x {tuple(B.shape)}"
                             f"{'^T' if transpose_b else ''}")
    if tuple(O.shape) != (A.shape[0], N):
        raise DimensionError(f"gemm output shape {tuple(O.shape)}, expected {(A.shape[0], N)}")
    if A.dtype != B.dtype or A.dtype not in _DT or O.dtype not in _DT:
        raise DimensionError(f"gemm dtypes {A.dtype} x {B.dtype} -> {O.dtype} unsupported")
    _check_no_alias(O, A, B)
    lda, ldb, ldc = _row_major(A, "a"), _row_major(B, "b"), _row_major(O, "out")
    bias_t = as_device(bias, torch.float32) if bias is not None else None
    if bias_t is not None and tuple(bias_t.shape) != (N,):
        raise DimensionError(f"bias shape {tuple(bias_t.shape)} != ({N},)")
    res_t, ldr = None, 0
    if residual is not None:
        res_t = as_device(residual, torch.float32)
        if tuple(res_t.shape) != tuple(O.shape):
            raise DimensionError(f"residual shape {tuple(res_t.shape)} != {tuple(O.shape)}")
        ldr = _row_major(res_t, "residual")
    t0 = timers.start() if timers is not None else None
    _abi.call("fq_gemm", A.data_ptr(), _DT[A.dtype], lda, B.data_ptr(), _DT[B.dtype], ldb,
              int(transpose_b), O.data_ptr(), _DT[O.dtype], ldc, A.shape[0], N, K,
              int(accumulate), _abi.ptr(bias_t), _abi.ptr(res_t), ldr, ACT_IDS[activation],
              _abi.stream_handle())
    if timers is not None:
        timers.stop("gemm", t0)
    (counters or _global_counters).count_gemm(
        A.numel() * A.element_size() + B.numel() * B.element_size() + O.numel() * O.element_size())
    writeback(out, O)


def gemm_x3(a, w, out, *, accumulate: bool = False, counters: OpCounters | None = None,
            timers: Timers | None = None, bias=None, residual=None, activation: str = "none"):
    """Exact-mode engine GEMM on the tensor cores: out = act(a @ w^T (+ out)
    (+ bias)) (+ residual), ``a`` fp32 [M, K], ``w`` an ``X3Weight`` (the
    weight's tf32 hi / lo halves, K-major [N, K], split once at load) — the
    3xTF32 product of fq_gemm_f32x3. One call increments ``gemm_calls`` by one
    (tensor.py:204)."""
    A, O = as_device(a, torch.float32), as_device(out)
    if A.dim() != 2 or O.dim() != 2 or O.dtype != torch.float32:
        raise DimensionError("gemm_x3 expects 2D fp32 operands")
    N, K = w.shape
    if A.shape[1] != K or tuple(O.shape) != (A.shape[0], N):
        raise DimensionError(f"gemm_x3 shapes {tuple(A.shape)} x {(N, K)}^T -> {tuple(O.shape)}")
    _check_no_alias(O, A, w.hi, w.lo)
    lda, ldc = _row_major(A, "a"), _row_major(O, "out")
    res_t, ldr = None, 0
    if residual is not None:
        res_t = as_device(residual, torch.float32)
        ldr = _row_major(res_t, "residual")
    t0 = timers.start() if timers is not None else None
    _abi.call("fq_gemm_f32x3", A.data_ptr(), lda, w.hi.data_ptr(), w.lo.data_ptr(),
              w.hi.stride(0), O.data_ptr(), ldc, A.shape[0], N, K, int(accumulate),
              _abi.ptr(bias), _abi.ptr(res_t), ldr, ACT_IDS[activation], _abi.stream_handle())
    if timers is not None:
        timers.stop("gemm", t0)
    (counters or _global_counters).count_gemm(A.numel() * 4 + 2 * N * K * 4 + O.numel() * 4)


def split_pair(a, pair=None):
    """The exact mode's fp16 operand pair of an fp32 [M, K] matrix (x = hi +
    lo * 2^-11, fq_split_f16): into ``pair`` = (hi, lo) when given."""
    A = as_device(a, torch.float32)
    if pair is None:
        pair = tuple(torch.empty(A.shape, dtype=torch.float16, device=A.device) for _ in range(2))
    hi, lo = pair
    if tuple(hi.shape) != tuple(A.shape) or hi.stride(0) != lo.stride(0):
        raise DimensionError(f"pair shape {tuple(hi.shape)} != {tuple(A.shape)}")
    _abi.call("fq_split_f16", A.data_ptr(), _row_major(A, "a"), A.shape[0], A.shape[1], 0,
              hi.data_ptr(), lo.data_ptr(), hi.stride(0), _abi.stream_handle())
    return pair


def gemm_xh(a_pair, w, out, *, accumulate: bool = False, counters: OpCounters | None = None,
            timers: Timers | None = None, bias=None, residual=None, activation: str = "none"):
    """Exact-mode engine GEMM, 3xFP16 (fq_gemm_x3h): out = act(a @ w^T (+ out)
    (+ bias)) (+ residual) with ``a_pair`` the fp16 (hi, lo) pair of the fp32
    activation [M, K] (written by its producer, or ``split_pair``) and ``w`` an
    ``XHWeight`` (the weight's pair, K-major [N, K], split once at load). One
    call increments ``gemm_calls`` by one (tensor.py:204)."""
    hi, lo = a_pair
    O = as_device(out)
    if hi.dim() != 2 or O.dim() != 2 or O.dtype != torch.float32 or hi.dtype != torch.float16:
        raise DimensionError("gemm_xh expects an fp16 [M, K] pair and an fp32 output")
    N, K = w.shape
    if hi.shape[1] != K or tuple(O.shape) != (hi.shape[0], N) or lo.shape != hi.shape:
        raise DimensionError(f"gemm_xh shapes {tuple(hi.shape)} x {(N, K)}^T -> {tuple(O.shape)}")
    if hi.stride(0) != lo.stride(0):
        raise DimensionError("gemm_xh: hi and lo need the same leading dimension")
    _check_no_alias(O, hi, lo, w.hi, w.lo)
    lda, ldc = _row_major(hi, "a"), _row_major(O, "out")
    res_t, ldr = None, 0
    if residual is not None:
        res_t = as_device(residual, torch.float32)
        ldr = _row_major(res_t, "residual")
    t0 = timers.start() if timers is not None else None
    _abi.call("fq_gemm_x3h", hi.data_ptr(), lo.data_ptr(), lda, w.hi.data_ptr(), w.lo.data_ptr(),
              w.hi.stride(0), O.data_ptr(), ldc, hi.shape[0], N, K, int(accumulate),
              _abi.ptr(bias), _abi.ptr(res_t), ldr, ACT_IDS[activation], _abi.stream_handle())
    if timers is not None:
        timers.stop("gemm", t0)
    (counters or _global_counters).count_gemm(hi.numel() * 4 + N * K * 4 + O.numel() * 4)


def _batch_strides(t: torch.Tensor, lead: tuple[int, ...]) -> tuple[int, int, int, int]:
    """Express the leading dims of ``t`` (broadcast to ``lead``) as a two-level
    batch (n0, s0, n1, s1)."""
    shape = list(t.shape[:-2])
    strides = list(t.stride()[:-2])
    while len(shape) < len(lead):
        shape.insert(0, 1)
        strides.insert(0, 0)
    st = [0 if s == 1 and L != 1 else stv for s, stv, L in zip(shape, strides, lead)]
    if len(lead) == 1:
        return 1, 0, lead[0], st[0]
    if len(lead) == 2:
        return lead[0], st[0], lead[1], st[1]
    raise DimensionError("gemm_batched supports at most two leading dimensions")


def gemm_batched(a, b, out, *, transpose_b: bool = False,
                 counters: OpCounters | None = None, timers: Timers | None = None):
    """Batched out[..., :, :] = a[..., :, :] @ b[..., :, :] (tensor.py:207-227),
    fp32, one strided-batched launch; ``out`` may be a strided view (the
    merged-head ctx view, model.py:335)."""
    A, B, O = as_device(a), as_device(b), as_device(out)
    if A.dim() < 3 or B.dim() < 3:
        raise DimensionError("gemm_batched expects stacked operands (>=3D)")
    K = A.shape[-1]
    N = B.shape[-2] if transpose_b else B.shape[-1]
    if (B.shape[-1] if transpose_b else B.shape[-2]) != K:
        raise DimensionError(f"gemm_batched inner dims differ: {tuple(A.shape)} x {tuple(B.shape)}")
    lead = tuple(torch.broadcast_shapes(A.shape[:-2], B.shape[:-2]))
    if tuple(O.shape) != lead + (A.shape[-2], N):
        raise DimensionError(f"gemm_batched output shape {tuple(O.shape)}")
    for t, nm in ((A, "a"), (B, "b"), (O, "out")):
        if t.stride(-1) != 1 or t.dtype != torch.float32:
            raise DimensionError(f"gemm_batched {nm} must be fp32 with unit inner stride")
    _check_no_alias(O, A, B)
    n0, sa0, n1, sa1 = _batch_strides(A, lead)
    _, sb0, _, sb1 = _batch_strides(B, lead)
    _, sc0, _, sc1 = _batch_strides(O, lead)
    t0 = timers.start() if timers is not None else None
    _abi.call("fq_gemm_batched", A.data_ptr(), A.stride(-2), sa0, sa1, B.data_ptr(), B.stride(-2),
              sb0, sb1, int(transpose_b), O.data_ptr(), O.stride(-2), sc0, sc1, n0, n1,
              A.shape[-2], N, K, _abi.stream_handle())
    if timers is not None:
        timers.stop("gemm", t0)
    (counters or _global_counters).count_gemm(
        A.numel() * 4 + B.numel() * 4 + O.numel() * 4)
    writeback(out, O)


def wall() -> float:
    return time.perf_counter()
