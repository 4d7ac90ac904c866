"""ctypes binding of ``libfq_b200.so`` (include/fq_abi.h).

This is the layer where the reference calls ``kernels.*`` (numba) and
``np.matmul`` (OpenBLAS): every product op goes through ``call`` below into
the sm_100a library. There is no fallback — if the library is missing the
import of any op raises :class:`ExtensionError`.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (AliasingError, CapacityError, DimensionError, EngineError, ExtensionError,
                     ParameterError)

LIB_PATH = os.environ.get("FQ_LIB") or os.path.join(  # FQ_LIB: A/B builds (scripts/)
    os.path.dirname(os.path.abspath(__file__)), "_lib", "libfq_b200.so")

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int
F32 = ctypes.c_float
F64 = ctypes.c_double


class BeamStateC(ctypes.Structure):
    """fq_beam_state (fq_abi.h)."""
    _fields_ = [(n, P) for n in ("live", "step", "done", "prefix", "cum", "fin_count", "fin_tok",
                                 "fin_len", "fin_score", "last_tok", "parent", "n_done")]


SIGNATURES = {
    "fq_abi_version": ([], I32),
    "fq_last_error": ([], ctypes.c_char_p),
    "fq_num_sms": ([], I32),
    "fq_set_pdl": ([I32], I32),
    "fq_prepare": ([], I32),
    "fq_layer_norm": ([P, I64, P, P, F64, I64, I64, P, I64, P, I64, P], I32),
    "fq_bias_residual_layer_norm": ([P, I64, P, P, I64, P, P, F64, I64, I64, P, I64, P, I64, P],
                                    I32),
    "fq_splitk_bias_residual_layer_norm": ([P, I32, I64, P, P, I64, P, P, F64, I64, I64, P,
                                            I64, P, I64, P], I32),
    "fq_bias_residual_act": ([P, I64, P, P, I64, I32, I64, I64, P, I64, P], I32),
    "fq_qkv_bias_reshape": ([P, I64, P, I64, I64, I64, I64, P, P, P, P], I32),
    "fq_bias_reshape_heads": ([P, I64, P, I64, I64, I64, I64, P, P], I32),
    "fq_scale_mask_softmax": ([P, I64, P, I64, I64, I64, I64, I64, F32, P, P, P], I32),
    "fq_embed_scale_pos": ([P, I64, P, I64, F32, P, I64, P, I64, P, P, P], I32),
    "fq_kv_append": ([P, P, I64, I64, I64, I64, I64, P, P, P], I32),
    "fq_kv_gather_append": ([P, P, P, P, P, I64, I64, I64, I64, I64, P, P, P], I32),
    "fq_penalize_counts": ([P, I64, I64, I64, P, F32, P, I64, P], I32),
    "fq_gemm_ln": ([P, I64, P, I64, P, P, I64, P, P, F64, P, I64, P, I64, P, I64, I64, I64, I64,
                    P], I32),
    "fq_gemm": ([P, I32, I64, P, I32, I64, I32, P, I32, I64, I64, I64, I64, I32, P, P, I64, I32,
                 P], I32),
    "fq_gemm_plan": ([I64, I64, I64, P, P, P, P], I32),
    "fq_gemm_batched": ([P, I64, I64, I64, P, I64, I64, I64, I32, P, I64, I64, I64, I64, I64, I64,
                         I64, I64, P], I32),
    "fq_retrieve": ([P, I64, I64, I64, I64, P, P, I64, P, P, P, I64, P, P], I32),
    "fq_hars_select": ([P, I64, P, P, I64, P, BeamStateC, I64, I64, I64, I64, I64, P, P, I64,
                        P, P, P, P, I64, P], I32),
    "fq_hars_groups": ([BeamStateC, I64, I64, I64, I32, P, P], I32),
    "fq_hars_step": ([P, I64, BeamStateC, I64, I64, I64, I64, I64, P, P, I64, P, P, I64, P, P, P,
                      P, P, P, I64, F32, P, P, P, P, P], I32),
    "fq_logits_hars": ([P, I64, P, I64, I64, I64, I64, P, P, P, P, I64, P, P, I64, P], I32),
    "fq_hars_merge_step": ([BeamStateC, I64, I64, I64, I64, I64, P, P, I64, P, P, P, P, I64, I64,
                            P, P, I64, P, P, I64, P, P, P, P, P, P, P, I64, F32, P, P, P, P,
                            P], I32),
    "fq_beam_state_init": ([BeamStateC, I64, I64, I64, P], I32),
    "fq_step_advance": ([P, P], I32),
    "fq_finalize_beams": ([P, P, P, P, P, P, P, P, I64, I64, I64, F64, I64, P, P, P, P], I32),
    "fq_gemm_x3h_slabs": ([P, P, I64, P, P, I64, P, I64, I64, I64, I64, P, P], I32),
    "fq_cross_attention_xh_slabs": ([P, I64, I64, I64, P, P, P, I64, I64, I64, I64, I64, I64,
                                     I64, F32, P, P, P, P, I64, P, P], I32),
    "fq_encoder_attention_xh": ([P, I64, I64, I64, I64, I64, F32, P, P, P, P, I64, P, P], I32),
    "fq_sample_step": ([P, I64, P, P, I64, P, I64, I64, F64, I64, I64, I64, P, I64, P, P, P,
                        I64, I64, P, P, P, P, P, P, P, P], I32),
    "fq_encoder_attention": ([P, I64, I64, I64, I64, I64, F32, P, P, P, I64, I32, P, P], I32),
    "fq_decoder_self_attention": ([P, I64, P, P, I32, P, P, I64, I64, I64, I64, F32, P, P, I64,
                                   I32, P], I32),
    "fq_cross_attention": ([P, I64, P, P, I32, I64, I64, I64, I64, I64, I64, F32, P, P, P, I64,
                            I32, P, P], I32),
    "fq_cast_f16": ([P, I64, I64, I32, P, P], I32),
    "fq_cross_attention_slabs": ([P, I32, I64, P, P, P, I64, I64, I64, I64, I64, I64, F32, P, P,
                                  P, I64, P, P], I32),
    "fq_gemm_splitk_slabs": ([P, I64, P, I64, P, I64, I64, I64, I64, P, P], I32),
    "fq_gemm_f32x3": ([P, I64, P, P, I64, P, I64, I64, I64, I64, I32, P, P, I64, I32, P], I32),
    "fq_gemm_f32x3_ln": ([P, I64, P, P, I64, P, P, I64, P, P, F64, P, I64, P, I64, I64, I64, I64,
                          P], I32),
    "fq_split_tf32": ([P, I64, I64, I32, P, P, P], I32),
    "fq_gemm_x3h": ([P, P, I64, P, P, I64, P, I64, I64, I64, I64, I32, P, P, I64, I32, P], I32),
    "fq_logits_hars_x3h": ([P, P, I64, P, P, I64, I64, I64, I64, P, P, P, P, I64, P, P, I64, P],
                           I32),
    "fq_gemm_x3h_pair": ([P, P, I64, P, P, I64, P, P, I64, I64, I64, I64, P, I32, P], I32),
    "fq_gemm_x3h_ln": ([P, P, I64, P, P, I64, P, P, I64, P, P, F64, P, I64, P, P, I64, P, I64, I64,
                        I64, I64, P], I32),
    "fq_decoder_self_attention_xh": ([P, I64, P, P, I64, P, P, I64, I64, I64, I64, F32, P, P, P,
                                      I64, P], I32),
    "fq_decoder_self_attention_xh_items": ([P, I64, P, P, I64, P, P, I64, I64, I64, I64, I64, F32,
                                            P, P, P, I64, P], I32),
    "fq_cross_attention_xh": ([P, I64, P, P, I64, I64, I64, I64, I64, I64, I64, F32, P, P, P, P,
                               I64, P, P], I32),
    "fq_split_f16": ([P, I64, I64, I64, I32, P, P, I64, P], I32),
    "fq_layer_norm_xh": ([P, I64, P, P, F64, I64, I64, P, I64, P, P, I64, P], I32),
    "fq_splitk_bias_residual_layer_norm_xh": ([P, I32, I64, P, P, I64, P, P, F64, I64, I64, P, I64,
                                               P, P, I64, P], I32),
}

_ERRORS = {-1: DimensionError, -2: ParameterError, -3: AliasingError, -4: CapacityError,
           -5: ExtensionError, -6: EngineError}

_lib = None
_lock = threading.Lock()
_prepared = False
_NO_PREPARE = {"fq_abi_version", "fq_last_error", "fq_num_sms", "fq_prepare", "fq_gemm_plan",
               "fq_set_pdl", "fq_finalize_beams"}
_launches = [0]


def launch_count() -> int:
    """Kernels launched (or captured) through the ABI so far in this process."""
    return _launches[0]


def add_launches(n: int):
    """Account for kernels replayed from a captured CUDA graph."""
    _launches[0] += n


def load():
    """Load and type the library once. Raises ExtensionError when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ExtensionError(
                    f"{LIB_PATH} not built: run `python -m paper_2010_13887_b200.build` "
                    "(no CPU fallback exists)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


# Launch probe (bench.py): when PROBE is a list, every probed entry point is
# bracketed by timing events on the launching stream (external events, so they
# become event-record nodes inside a captured CUDA graph) and
# (name, args, start, end) is appended. Off (None) on the product path.
PROBE = None
PROBE_NAMES = ("fq_gemm", "fq_logits_hars", "fq_gemm_ln", "fq_gemm_splitk_slabs", "fq_gemm_f32x3",
               "fq_gemm_f32x3_ln", "fq_gemm_x3h", "fq_gemm_x3h_ln", "fq_gemm_x3h_pair", "fq_logits_hars_x3h")


def call(name: str, *args) -> int:
    """Invoke an fq_* entry point; map a negative status to the reference's
    exception class (errors.py) with the library's message."""
    global _prepared
    lib = load()
    if not _prepared and name not in _NO_PREPARE:
        rc = lib.fq_prepare()  # smem opt-ins, once, before any stream capture
        if rc < 0:
            raise ExtensionError(f"fq_prepare: {lib.fq_last_error().decode()}")
        _prepared = True
    if PROBE is not None and name in PROBE_NAMES:
        import torch
        e0 = torch.cuda.Event(enable_timing=True, external=True)
        e1 = torch.cuda.Event(enable_timing=True, external=True)
        e0.record()
        rc = getattr(lib, name)(*args)
        e1.record()
        PROBE.append((name, args, e0, e1, torch.cuda.is_current_stream_capturing()))
    else:
        rc = getattr(lib, name)(*args)
    if name not in _NO_PREPARE:
        # every other entry point launches one kernel; fq_gemm_ln two (the
        # split-K slab GEMM + the reducing LN, or the GEMM + LN fallback)
        _launches[0] += 2 if name in ("fq_gemm_ln", "fq_gemm_f32x3_ln", "fq_gemm_x3h_ln") else 1
    if rc < 0:
        msg = lib.fq_last_error().decode("utf-8", "replace")
        raise _ERRORS.get(rc, EngineError)(f"{name}: {msg}")
    return rc


def lib_call_rc(name: str, *args) -> int:
    """Like :func:`call` for an entry point whose "unsupported shape" status
    (FQ_ERR_UNSUPPORTED) is a routing answer (the caller falls back): returns
    that status instead of raising (any other error raises), counts a launch
    only on success."""
    global _prepared
    lib = load()
    if not _prepared:
        rc = lib.fq_prepare()
        if rc < 0:
            raise ExtensionError(f"fq_prepare: {lib.fq_last_error().decode()}")
        _prepared = True
    rc = getattr(lib, name)(*args)
    if rc >= 0:
        _launches[0] += 1
    elif rc != -6:  # only FQ_ERR_UNSUPPORTED is a routing answer
        msg = lib.fq_last_error().decode("utf-8", "replace")
        raise _ERRORS.get(rc, EngineError)(f"{name}: {msg}")
    return rc


def stream_handle() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()
