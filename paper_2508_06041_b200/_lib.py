"""ctypes binding of libdpq_b200.so (the C-ABI in include/dpq_b200.h).

There is no CPU fallback: every device entry point raises ``DeviceError``
when the library is missing or no CUDA device is usable.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdpq_b200.so")


class DeviceError(RuntimeError):
    """The B200 library failed (missing .so, no GPU, CUDA error)."""


class LayerDesc(C.Structure):
    _fields_ = [("rows", C.c_int32), ("cols", C.c_int32), ("n_bits", C.c_int32),
                ("b_min", C.c_int32), ("code_bytes", C.c_int32), ("codes_on_device", C.c_int32),
                ("codes", C.c_void_p), ("lo", C.c_void_p), ("hi", C.c_void_p)]


class SelDesc(C.Structure):
    _fields_ = [("l", C.c_int32), ("h", C.c_int32), ("prefill_bit", C.c_int32),
                ("est_kind", C.c_int32), ("prev_residual", C.c_int32), ("k", C.c_int32),
                ("g_dtype", C.c_int32), ("fx_bits_plus128", C.c_int32), ("T", C.c_double),
                ("slope", C.c_double), ("intercept", C.c_double), ("G", C.c_void_p)]


class ModelDesc(C.Structure):
    _fields_ = [("n_blocks", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("d_ff", C.c_int32), ("vocab", C.c_int32),
                ("seq_cap", C.c_int32), ("norm_eps", C.c_float), ("embed", C.c_void_p),
                ("lm_head", C.c_void_p), ("track_exact", C.c_int32),
                ("async_prev_block", C.c_int32), ("prime_from_prefill", C.c_int32),
                ("use_graph", C.c_int32), ("use_pdl", C.c_int32), ("use_persistent", C.c_int32)]


class TpDesc(C.Structure):
    _fields_ = [("tp_rank", C.c_int32), ("tp_size", C.c_int32), ("grid", C.c_int32), ("pad_", C.c_int32)]


P = C.c_void_p
I32 = C.c_int32
_SIGS = {
    "dpq_last_error": ([], C.c_char_p),
    "dpq_version": ([], C.c_int),
    "dpq_device_info": ([C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
    "dpq_store_create": ([C.c_int, C.c_int, C.POINTER(LayerDesc), C.POINTER(P)], C.c_int),
    "dpq_store_destroy": ([P], C.c_int),
    "dpq_store_append": ([P, C.c_int, C.POINTER(LayerDesc)], C.c_int),
    "dpq_store_layer_bytes": ([P, C.c_int, C.c_int, C.POINTER(C.c_int64)], C.c_int),
    "dpq_quantize_device": ([C.c_int, P, C.c_int, C.c_int, C.c_int, P, P, P, P], C.c_int),
    "dpq_gemv": ([P, C.c_int, C.c_int, P, P, P], C.c_int),
    "dpq_dequantize": ([P, C.c_int, C.c_int, P, P], C.c_int),
    "dpq_plan_create": ([P, C.c_int, C.POINTER(SelDesc), C.POINTER(P)], C.c_int),
    "dpq_plan_destroy": ([P], C.c_int),
    "dpq_select_gemv": ([P, C.c_int, P, P, P, P, P, P, P], C.c_int),
    "dpq_estimator_create": ([C.c_int, C.POINTER(SelDesc), C.c_int, C.POINTER(P)], C.c_int),
    "dpq_estimator_eval": ([P, P, C.POINTER(C.c_double), P], C.c_int),
    "dpq_estimator_destroy": ([P], C.c_int),
    "dpq_exact_error": ([P, C.c_int, C.c_int, C.c_int, P, C.POINTER(C.c_double), P], C.c_int),
    "dpq_session_create": ([P, P, C.POINTER(ModelDesc), C.POINTER(P)], C.c_int),
    "dpq_session_destroy": ([P], C.c_int),
    "dpq_session_reset": ([P], C.c_int),
    "dpq_session_step": ([P, C.c_int, C.c_int, P, P], C.c_int),
    "dpq_session_decode": ([P, C.c_int, P], C.c_int),
    "dpq_session_launch_steps": ([P, C.c_int, P], C.c_int),
    "dpq_session_trace": ([P, C.POINTER(C.c_int), P, P, P], C.c_int),
    "dpq_session_position": ([P, C.POINTER(C.c_int)], C.c_int),
    "dpq_session_is_persistent": ([P], C.c_int),
    "dpq_session_logits_dev": ([P, C.POINTER(P)], C.c_int),
    "dpq_session_engine_stages": ([P, C.POINTER(C.c_int), P, P], C.c_int),
    "dpq_session_profile_ops": ([P, C.c_int, C.c_int, P, C.c_int, C.POINTER(C.c_int)], C.c_int),
    "dpq_session_debug_times": ([P, P, C.c_int64, C.POINTER(C.c_int)], C.c_int),
    "dpq_session_sync": ([P], C.c_int),
    "dpq_session_logits": ([P, P], C.c_int),
    "dpq_session_create_tp": ([P, P, C.POINTER(ModelDesc), C.POINTER(TpDesc), C.POINTER(P)], C.c_int),
    "dpq_session_tp_arena": ([P, C.POINTER(P), C.POINTER(C.c_int64)], C.c_int),
    "dpq_session_tp_ipc_handle": ([P, P], C.c_int),
    "dpq_tp_ipc_open": ([C.c_int, P, C.POINTER(P)], C.c_int),
    "dpq_tp_ipc_close": ([C.c_int, P], C.c_int),
    "dpq_session_tp_connect": ([P, P], C.c_int),
    "dpq_repack_host": ([P, C.c_int, C.c_int, C.c_int, P, C.c_int64], C.c_int),
    "dpq_planes_bytes": ([C.c_int, C.c_int, C.c_int], C.c_int64),
}
EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def load():
    """Load libdpq_b200.so (raises DeviceError if it is missing)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(f"{LIB_PATH} not built (python -m paper_2508_06041_b200._build)")
            lib = C.CDLL(LIB_PATH)
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = load().dpq_last_error().decode(errors="replace")
        raise DeviceError(f"{what}: {msg}" if what else msg)


def call(name, *args):
    fn = getattr(load(), name)
    rc = fn(*args)
    if name not in ("dpq_planes_bytes", "dpq_version", "dpq_last_error", "dpq_session_is_persistent"):
        check(rc, name)
    return rc


def torch_device():
    """The current CUDA device as a torch.device; raises without a GPU."""
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device available: the dpq B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)
