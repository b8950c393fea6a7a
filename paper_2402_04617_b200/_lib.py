"""ctypes binding of libinfllm_b200.so (the C-ABI in include/infllm_b200.h).

The shared library is built in-tree (``make -C paper_2402_04617_b200`` or
``__graft_entry__.build()``). There is no fallback: if the library is missing
or a CUDA device is absent, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libinfllm_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "infllm_b200.h")

OK, ERR_CONFIG, ERR_STREAM, ERR_CUDA, ERR_NCCL, ERR_ARG = 0, 1, 2, 3, 4, 5
DTYPE_F32, DTYPE_BF16 = 0, 1
LOOKUP_MODES = {"encode_and_decode": 0, "decode_only": 1, "none": 2}
POSITION_MODES = {"clamped": 0, "absolute": 1}


class EngineConfig(C.Structure):
    """blockmem::EngineConfig (types.hpp:84-110)."""

    _fields_ = [
        ("chunk_size", C.c_int64),
        ("unit_size", C.c_int64),
        ("n_repr", C.c_int64),
        ("local_size", C.c_int64),
        ("init_size", C.c_int64),
        ("n_lookup", C.c_int64),
        ("hot_capacity", C.c_int64),
        ("decay", C.c_double),
        ("lookup_mode", C.c_int32),
        ("position_mode", C.c_int32),
    ]

    @classmethod
    def make(cls, **kw):
        c = cls()
        lib().infllm_config_default(C.byref(c))
        for k, v in kw.items():
            if k == "lookup_mode" and isinstance(v, str):
                v = LOOKUP_MODES[v]
            if k == "position_mode" and isinstance(v, str):
                v = POSITION_MODES[v]
            setattr(c, k, v)
        return c

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class ModelShape(C.Structure):
    """blockmem::ModelShape (types.hpp:29-49) + n_kv_heads (GQA)."""

    _fields_ = [
        ("n_layers", C.c_int32),
        ("n_heads", C.c_int32),
        ("n_kv_heads", C.c_int32),
        ("head_dim", C.c_int32),
        ("value_dim", C.c_int32),
    ]

    @classmethod
    def make(cls, n_heads=1, n_kv_heads=None, head_dim=64, value_dim=None, n_layers=1):
        return cls(n_layers, n_heads, n_kv_heads or n_heads, head_dim, value_dim or head_dim)


class LayerMetrics(C.Structure):
    _fields_ = [
        ("units", C.c_int64),
        ("hot_units", C.c_int64),
        ("peak_hot_units", C.c_int64),
        ("peak_hot_bytes", C.c_int64),
        ("hits", C.c_uint64),
        ("misses", C.c_uint64),
        ("loads", C.c_uint64),
        ("evictions", C.c_uint64),
        ("requested", C.c_uint64),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Segment(C.Structure):
    """infllm_segment: blockmem::SegmentView (attention.hpp:28-51)."""

    _fields_ = [("kind", C.c_int32), ("start_abs", C.c_int64), ("n_tokens", C.c_int64), ("keys", C.c_void_p),
                ("values", C.c_void_p)]


SEG_KINDS = {"initial": 0, "retrieved": 1, "local": 2}

ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                           C.c_void_p)

# name -> (restype, argtypes); must cover every function include/infllm_b200.h declares
P, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
i64p, f64p, i32p = C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_int32)
SIGNATURES = {
    "infllm_last_error": (C.c_char_p, []),
    "infllm_version": (C.c_char_p, []),
    "infllm_config_default": (C.c_int, [C.POINTER(EngineConfig)]),
    "infllm_config_validate": (C.c_int, [C.POINTER(EngineConfig), C.POINTER(ModelShape)]),
    "infllm_engine_create": (C.c_int, [C.POINTER(EngineConfig), C.POINTER(ModelShape), i32, i32, i32, i32,
                                       C.POINTER(P)]),
    "infllm_engine_destroy": (C.c_int, [P]),
    "infllm_engine_set_allgather": (C.c_int, [P, ALLGATHER_FN, P]),
    "infllm_engine_reserve": (C.c_int, [P, i64]),
    "infllm_nccl_unique_id": (C.c_int, [P]),
    "infllm_engine_set_comm": (C.c_int, [P, P, i32, i32]),
    "infllm_exchange_fold_host": (C.c_int, [f64p, i64, i32, i32, f64p]),
    "infllm_topk_host": (C.c_int, [f64p, i64, i64, i64p, i64p]),
    "infllm_engine_reset": (C.c_int, [P, P]),
    "infllm_engine_set_option": (C.c_int, [P, C.c_char_p, i64]),
    "infllm_encode_chunk": (C.c_int, [P, i32, P, P, P, i64, P, P]),
    "infllm_decode_step": (C.c_int, [P, i32, P, P, P, P, P]),
    "infllm_encode_stream": (C.c_int, [P, i32, P, P, P, i64, P, P]),
    "infllm_encode_stream_host": (C.c_int, [P, i32, P, P, P, i64, P, P]),
    "infllm_finish": (C.c_int, [P, P]),
    "infllm_retrieved_ids": (C.c_int, [P, i32, i64p, i64, i64p]),
    "infllm_get_layer_metrics": (C.c_int, [P, i32, C.POINTER(LayerMetrics)]),
    "infllm_unit_info": (C.c_int, [P, i32, i64, i64p, i64p, i64p, i64p]),
    "infllm_stream_state": (C.c_int, [P, i32, i64p, i64p, i64p, i64p, i64p]),
    "infllm_unit_freq": (C.c_int, [P, i32, f64p, i32p, i64]),
    "infllm_trace": (C.c_int, [P, i32, i64p, i64p, i32p, i64, i64p]),
    "infllm_kernel_launches": (C.c_int, [P, i64p]),
    "infllm_tier_stats": (C.c_int, [P, i32, i64p]),
    "infllm_decode_batch": (C.c_int, [C.POINTER(C.c_void_p), i32, i32, P, P, P, P, P]),
    "infllm_debug_host_times": (C.c_int, [P, i32]),
    "infllm_profile_begin": (C.c_int, [P, i32]),
    "infllm_profile_read": (C.c_int, [P, f64p, i64p, f64p, i64p]),
    "infllm_phase_timings": (C.c_int, [P, f64p, i64p]),
    "infllm_invariants": (C.c_int, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "infllm_select_representatives": (C.c_int, [P, P, i64, i64, i64, P, P]),
    "infllm_lookup": (C.c_int, [P, P, i32, i64, i64, i32, i32, i64, P, P, P]),
    "infllm_debug_tc_selftest": (C.c_int, [P, P, P, P, P, P]),
    "infllm_debug_kernel_bench": (C.c_int, [P, i32, i32, f64p]),
    "infllm_debug_timestamps": (C.c_int, [P]),
    "infllm_timeline_enable": (C.c_int, [i64]),
    "infllm_attend": (C.c_int, [C.POINTER(ModelShape), i32, i32, i64, C.POINTER(Segment), i32, P, P, P, i64, i64, P,
                                P, P, P]),
    "infllm_store_create": (C.c_int, [i64, f64, i32, i32, i32, i64, i32, i64, C.POINTER(P)]),
    "infllm_store_destroy": (C.c_int, [P]),
    "infllm_store_add_unit": (C.c_int, [P, P, i64, i64, i64p]),
    "infllm_store_begin_step": (C.c_int, [P, i64]),
    "infllm_store_lookup": (C.c_int, [P, P, i64, i64, i64p, i64p, P]),
    "infllm_store_update_frequency": (C.c_int, [P, i64p, f64p, i64]),
    "infllm_store_enforce_capacity": (C.c_int, [P]),
    "infllm_store_note_step_boundary": (C.c_int, [P]),
    "infllm_store_counters": (C.c_int, [P, C.POINTER(LayerMetrics)]),
    "infllm_store_trace": (C.c_int, [P, i64p, i64p, i32p, i64, i64p]),
    "infllm_store_unit_freq": (C.c_int, [P, f64p, i32p, i64]),
    "infllm_score_acc_create": (C.c_int, [i64, i32, i32, i32, i32, C.POINTER(P)]),
    "infllm_score_acc_destroy": (C.c_int, [P]),
    "infllm_score_acc_accumulate": (C.c_int, [P, P, i64, i64, P, i64, P]),
    "infllm_score_acc_finalize_front": (C.c_int, [P, i64, C.POINTER(C.c_float)]),
    "infllm_timeline_read": (C.c_int, [P, P, P, P, i64, i64p, i32]),
}


def build(force: bool = False) -> str:
    srcs = [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))] + [HEADER]
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= max(map(os.path.getmtime, srcs)):
        return LIB_PATH
    subprocess.check_call(["make", "-s", "-C", HERE, "libinfllm_b200.so"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built; run `make -C {HERE}` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class InfLLMError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class ConfigError(InfLLMError, ValueError):
    """blockmem::ConfigError (types.hpp:20-22)."""


class StreamError(InfLLMError):
    """blockmem::StreamError (types.hpp:24-26)."""


class CudaError(InfLLMError):
    pass


def check(rc):
    if rc != OK:
        msg = lib().infllm_last_error().decode()
        raise {ERR_CONFIG: ConfigError, ERR_STREAM: StreamError, ERR_CUDA: CudaError}.get(rc, InfLLMError)(rc, msg)
