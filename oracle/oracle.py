"""TEST INFRASTRUCTURE ONLY — ctypes binding of the CPU oracle.

`liboracle.so` is the plain-C++ restatement of the reference engine
(oracle/infllm_oracle.cpp, every function cites /root/reference file:line).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module; the product package never
does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

LOOKUP_MODES = {"encode_and_decode": 0, "decode_only": 1, "none": 2}
POSITION_MODES = {"clamped": 0, "absolute": 1}


class EngineConfig(C.Structure):
    """blockmem::EngineConfig (types.hpp:84-110); defaults per types.hpp:85-94."""

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
        d = dict(chunk_size=512, unit_size=128, n_repr=4, local_size=4096, init_size=128,
                 n_lookup=32, hot_capacity=32, decay=0.1, lookup_mode=0, position_mode=0)
        for k, v in kw.items():
            if k == "lookup_mode" and isinstance(v, str):
                v = LOOKUP_MODES[v]
            if k == "position_mode" and isinstance(v, str):
                v = POSITION_MODES[v]
            d[k] = v
        return cls(**d)

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class ModelShape(C.Structure):
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


def build(force: bool = False) -> str:
    """Compile liboracle.so (-O3, no -march: matches proj/CMakeLists.txt)."""
    src = os.path.join(HERE, "infllm_oracle.cpp")
    hdr = os.path.join(HERE, "infllm_oracle.h")
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return LIB_PATH
    subprocess.check_call(["make", "-s", "-C", HERE, "liboracle.so"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        i64p = C.POINTER(C.c_int64)
        f32p = C.POINTER(C.c_float)
        f64p = C.POINTER(C.c_double)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_engine_create.restype = P
        L.oracle_engine_create.argtypes = [C.POINTER(EngineConfig), C.POINTER(ModelShape), C.c_int32]
        L.oracle_engine_destroy.argtypes = [P]
        L.oracle_set_always_emit_weights.argtypes = [P, C.c_int32]
        L.oracle_step.argtypes = [P, C.c_int32, f32p, f32p, f32p, C.c_int64, C.c_int32, f32p, i64p,
                                  C.c_int64, i64p, f64p]
        L.oracle_finish.argtypes = [P]
        L.oracle_warm_start.argtypes = [P, C.c_int32, f32p, f32p, f32p, C.c_int64]
        L.oracle_layer_metrics.argtypes = [P, C.c_int32, C.POINTER(LayerMetrics)]
        L.oracle_stream_state.argtypes = [P, C.c_int32] + [i64p] * 5
        L.oracle_unit_info.argtypes = [P, C.c_int32, C.c_int64, i64p, i64p, i64p, i64p]
        L.oracle_unit_freq.argtypes = [P, C.c_int32, f64p, C.POINTER(C.c_int32), C.c_int64]
        L.oracle_trace.argtypes = [P, C.c_int32, i64p, i64p, C.POINTER(C.c_int32), C.c_int64, i64p]
        L.oracle_invariants.argtypes = [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.oracle_timings.argtypes = [P, f64p]
        L.oracle_evicted_scores.argtypes = [P, C.c_int32, f32p, C.c_int64, i64p]
        L.oracle_unit_repr_keys.argtypes = [P, C.c_int32, C.c_int64, f32p]
        L.oracle_select_representatives.argtypes = [f32p, C.c_int64, C.c_int64, i64p, i64p]
        L.oracle_argsort_topk.argtypes = [f64p, C.c_int64, C.c_int64, i64p, i64p]
        L.oracle_relevance_all.argtypes = [f32p, C.c_int64, C.c_int32, C.c_int32, C.c_int32, f32p,
                                           C.c_int64, C.c_int64, f64p]
        L.oracle_relevance_unit.restype = C.c_double
        L.oracle_relevance_unit.argtypes = [f32p, C.c_int64, C.c_int32, C.c_int32, C.c_int32, f32p,
                                            C.c_int64]
        L.oracle_mean_repr_relevance.restype = C.c_double
        L.oracle_mean_repr_relevance.argtypes = [f64p, C.c_int64, f64p, C.c_int64, C.c_int32,
                                                 C.c_int32, C.c_int32]
        L.oracle_dense_attention.argtypes = [f64p, f64p, f64p, C.c_int64, C.c_int32, C.c_int32,
                                             C.c_int32, C.c_int32, C.c_int32, C.c_int64, f64p]
        L.oracle_windowed_attention.argtypes = [f64p, f64p, f64p, C.c_int64, C.c_int32, C.c_int32,
                                                C.c_int32, C.c_int32, i64p, C.c_int64, C.c_int64,
                                                C.c_int64, C.c_int64, C.c_int32, f64p]
        L.oracle_batch_repr_scores.argtypes = [f64p, f64p, C.c_int64, C.c_int32, C.c_int32,
                                               C.c_int32, C.c_int64, f64p]
        L.oracle_noise_ids.argtypes = [C.c_uint64, C.c_int64, i64p]
        L.oracle_adapter_batch.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                           C.c_int32, i64p, C.c_int64, f32p, f32p, f32p]
        L.oracle_gaussian_fill.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, C.c_int32,
                                           C.c_int32, f32p]
        L.oracle_gen_planted.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.POINTER(EngineConfig),
                                         C.c_int64, C.c_int32, i64p, i64p, i64p, i64p, i64p]
        L.oracle_store_create.restype = P
        L.oracle_store_create.argtypes = [C.c_int64, C.c_double, C.c_int32, C.c_int32, C.c_int32, C.c_int64]
        L.oracle_store_destroy.argtypes = [P]
        L.oracle_store_add_unit.argtypes = [P, f32p, C.c_int64, C.c_int64, i64p]
        L.oracle_store_begin_step.argtypes = [P, C.c_int64]
        L.oracle_store_lookup.argtypes = [P, f32p, C.c_int64, C.c_int64, i64p, i64p]
        L.oracle_store_update_frequency.argtypes = [P, i64p, f64p, C.c_int64]
        L.oracle_store_enforce_capacity.argtypes = [P]
        L.oracle_store_note_step_boundary.argtypes = [P]
        L.oracle_store_counters.argtypes = [P, C.POINTER(LayerMetrics)]
        L.oracle_store_trace.argtypes = [P, i64p, i64p, C.POINTER(C.c_int32), C.c_int64, i64p]
        L.oracle_store_unit_freq.argtypes = [P, f64p, C.POINTER(C.c_int32), C.c_int64]
        L.oracle_score_acc_create.restype = P
        L.oracle_score_acc_create.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32]
        L.oracle_score_acc_destroy.argtypes = [P]
        L.oracle_score_acc_accumulate.argtypes = [P, f32p, C.c_int64, C.c_int64, f32p, C.c_int64]
        L.oracle_score_acc_finalize_front.argtypes = [P, C.c_int64, f32p]
        L.oracle_attend.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64,
                                    C.POINTER(C.c_int32), i64p, i64p, C.POINTER(f32p), C.POINTER(f32p), C.c_int32,
                                    f32p, f32p, f32p, C.c_int64, C.c_int64, f32p, f64p, f32p]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class ConfigError(OracleError):
    pass


class StreamError(OracleError):
    pass


def _check(rc):
    if rc != 0:
        msg = lib().oracle_last_error().decode()
        raise {1: ConfigError, 2: StreamError}.get(rc, OracleError)(rc, msg)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class StepResult:
    out: np.ndarray
    retrieved_ids: list
    masses: list


class OracleEngine:
    """StreamEngine<float> restatement with explicit per-step q/k/v."""

    def __init__(self, cfg: EngineConfig, shape: ModelShape, n_threads: int = 1):
        self.cfg, self.shape = cfg, shape
        h = lib().oracle_engine_create(C.byref(cfg), C.byref(shape), n_threads)
        if not h:
            msg = lib().oracle_last_error().decode()
            raise ConfigError(1, msg)
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().oracle_engine_destroy(self.h)
            except Exception:
                pass
            self.h = None

    def set_always_emit_weights(self, v=True):
        lib().oracle_set_always_emit_weights(self.h, int(v))

    def step(self, q, k, v, decode=False, layer=0) -> StepResult:
        q, k, v = f32(q), f32(k), f32(v)
        l_x = q.shape[0]
        H, dv = self.shape.n_heads, self.shape.value_dim
        out = np.zeros((l_x, H, dv), np.float32)
        cap = max(1, int(self.cfg.n_lookup))
        ids = np.zeros(cap, np.int64)
        masses = np.zeros(cap, np.float64)
        n = C.c_int64(0)
        _check(lib().oracle_step(self.h, layer, _p(q, C.c_float), _p(k, C.c_float), _p(v, C.c_float),
                                 l_x, int(decode), _p(out, C.c_float), _p(ids, C.c_int64), cap,
                                 C.byref(n), _p(masses, C.c_double)))
        return StepResult(out, ids[: n.value].tolist(), masses[: n.value].tolist())

    def finish(self):
        _check(lib().oracle_finish(self.h))

    def warm_start(self, q, k, v, layer=0):
        q, k, v = f32(q), f32(k), f32(v)
        _check(lib().oracle_warm_start(self.h, layer, _p(q, C.c_float), _p(k, C.c_float), _p(v, C.c_float),
                                       q.shape[0]))

    def metrics(self, layer=0):
        m = LayerMetrics()
        _check(lib().oracle_layer_metrics(self.h, layer, C.byref(m)))
        return m.as_dict()

    def stream_state(self, layer=0):
        vals = [C.c_int64() for _ in range(5)]
        _check(lib().oracle_stream_state(self.h, layer, *[C.byref(x) for x in vals]))
        return dict(zip(["tokens_fed", "steps", "initial_len", "local_len", "pending_partial"],
                        [x.value for x in vals]))

    def unit_info(self, uid, layer=0):
        s, z, n = C.c_int64(), C.c_int64(), C.c_int64()
        r = np.zeros(max(1, int(self.cfg.n_repr)), np.int64)
        _check(lib().oracle_unit_info(self.h, layer, uid, C.byref(s), C.byref(z), _p(r, C.c_int64),
                                      C.byref(n)))
        return dict(start_abs=s.value, size=z.value, repr_abs=r[: n.value].tolist())

    def unit_freq(self, n, layer=0):
        f = np.zeros(n, np.float64)
        hot = np.zeros(n, np.int32)
        _check(lib().oracle_unit_freq(self.h, layer, _p(f, C.c_double), _p(hot, C.c_int32), n))
        return f, hot

    def trace(self, layer=0, cap=1 << 20):
        st, un = np.zeros(cap, np.int64), np.zeros(cap, np.int64)
        hit = np.zeros(cap, np.int32)
        n = C.c_int64()
        _check(lib().oracle_trace(self.h, layer, _p(st, C.c_int64), _p(un, C.c_int64),
                                  _p(hit, C.c_int32), cap, C.byref(n)))
        k = min(n.value, cap)
        return list(zip(st[:k].tolist(), un[:k].tolist(), hit[:k].tolist()))

    def invariants(self):
        c, v = C.c_uint64(), C.c_uint64()
        lib().oracle_invariants(self.h, C.byref(c), C.byref(v))
        return c.value, v.value

    def timings(self):
        t = np.zeros(5, np.float64)
        lib().oracle_timings(self.h, _p(t, C.c_double))
        return dict(zip(["adapter", "lookup", "attend", "score", "evict"], t.tolist()))

    def evicted_scores(self, layer=0, cap=1 << 22):
        s = np.zeros(cap, np.float32)
        n = C.c_int64()
        _check(lib().oracle_evicted_scores(self.h, layer, _p(s, C.c_float), cap, C.byref(n)))
        return s[: min(cap, n.value)].copy()

    def unit_repr_keys(self, uid, layer=0):
        nr = len(self.unit_info(uid, layer)["repr_abs"])
        k = np.zeros((nr, self.shape.n_kv_heads, self.shape.head_dim), np.float32)
        _check(lib().oracle_unit_repr_keys(self.h, layer, uid, _p(k, C.c_float)))
        return k


# ---------------------------------------------------------------- standalone
class OracleStore:
    """TieredStore (memory.hpp:170-323) on an explicit representative index."""

    def __init__(self, hot_capacity, decay, H, Hkv, d, bytes_per_token):
        self.Hkv, self.d = Hkv, d
        self.h = lib().oracle_store_create(hot_capacity, decay, H, Hkv, d, bytes_per_token)

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_store_destroy(self.h)
            self.h = None

    def add_unit(self, repr_keys, unit_tokens):
        rk = f32(repr_keys)
        uid = C.c_int64()
        _check(lib().oracle_store_add_unit(self.h, _p(rk, C.c_float), rk.shape[0], unit_tokens, C.byref(uid)))
        return uid.value

    def begin_step(self, step):
        lib().oracle_store_begin_step(self.h, step)

    def lookup(self, q, k_m):
        q = f32(q)
        ids = np.zeros(max(1, k_m), np.int64)
        n = C.c_int64()
        _check(lib().oracle_store_lookup(self.h, _p(q, C.c_float), q.shape[0], k_m, _p(ids, C.c_int64), C.byref(n)))
        return ids[: n.value].tolist()

    def update_frequency(self, pairs):
        ids = np.array([p[0] for p in pairs] or [0], np.int64)
        ms = np.array([p[1] for p in pairs] or [0.0], np.float64)
        _check(lib().oracle_store_update_frequency(self.h, _p(ids, C.c_int64), _p(ms, C.c_double), len(pairs)))

    def enforce_capacity(self):
        _check(lib().oracle_store_enforce_capacity(self.h))

    def note_step_boundary(self):
        _check(lib().oracle_store_note_step_boundary(self.h))

    def counters(self):
        m = LayerMetrics()
        lib().oracle_store_counters(self.h, C.byref(m))
        return m.as_dict()

    def trace(self, cap=1 << 16):
        st, un = np.zeros(cap, np.int64), np.zeros(cap, np.int64)
        hit = np.zeros(cap, np.int32)
        n = C.c_int64()
        lib().oracle_store_trace(self.h, _p(st, C.c_int64), _p(un, C.c_int64), _p(hit, C.c_int32), cap, C.byref(n))
        k = min(n.value, cap)
        return list(zip(st[:k].tolist(), un[:k].tolist(), hit[:k].tolist()))

    def unit_freq(self, n):
        f = np.zeros(max(1, n), np.float64)
        hot = np.zeros(max(1, n), np.int32)
        lib().oracle_store_unit_freq(self.h, _p(f, C.c_double), _p(hot, C.c_int32), n)
        return f[:n], hot[:n]


class OracleScoreAccumulator:
    """ScoreAccumulator (repr_score.hpp:21-89)."""

    def __init__(self, local_size, H, Hkv, d):
        self.h = lib().oracle_score_acc_create(local_size, H, Hkv, d)

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_score_acc_destroy(self.h)
            self.h = None

    def accumulate(self, q, s, pending_keys):
        q, k = f32(q), f32(pending_keys)
        _check(lib().oracle_score_acc_accumulate(self.h, _p(q, C.c_float), q.shape[0], s, _p(k, C.c_float),
                                                 k.shape[0]))

    def finalize_front(self, n):
        out = np.zeros(max(1, n), np.float32)
        _check(lib().oracle_score_acc_finalize_front(self.h, n, _p(out, C.c_float)))
        return out[:n]


SEG_KINDS = {"initial": 0, "retrieved": 1, "local": 2}


def attend(segments, q, k, v, start_abs, local_size, position_mode="clamped", emit_weights=False):
    """attend (attention.hpp:116-230) over segments [(kind, start_abs, keys [n][Hkv][d], values [n][Hkv][dv])]
    plus the causal batch q [l_x][H][d], k/v [l_x][Hkv][*]; returns (out, seg_mass, weights|None)."""
    q, k, v = f32(q), f32(k), f32(v)
    l_x, H, d = q.shape
    Hkv, dv = v.shape[1], v.shape[2]
    ns = len(segments)
    kinds = (C.c_int32 * max(1, ns))(*[SEG_KINDS[s[0]] if isinstance(s[0], str) else s[0] for s in segments])
    starts = np.array([s[1] for s in segments] or [0], np.int64)
    keys = [f32(s[2]) for s in segments]
    vals = [f32(s[3]) for s in segments]
    ns_arr = np.array([x.shape[0] for x in keys] or [0], np.int64)
    f32p = C.POINTER(C.c_float)
    kp = (f32p * max(1, ns))(*[_p(x, C.c_float) for x in keys])
    vp = (f32p * max(1, ns))(*[_p(x, C.c_float) for x in vals])
    n_ctx = int(sum(x.shape[0] for x in keys))
    out = np.zeros((l_x, H, dv), np.float32)
    mass = np.zeros(max(1, ns), np.float64)
    w = np.zeros((H, l_x, n_ctx + l_x), np.float32) if emit_weights else None
    pm = POSITION_MODES[position_mode] if isinstance(position_mode, str) else position_mode
    _check(lib().oracle_attend(H, Hkv, d, dv, pm, local_size, kinds, _p(starts, C.c_int64), _p(ns_arr, C.c_int64), kp,
                               vp, ns, _p(q, C.c_float), _p(k, C.c_float), _p(v, C.c_float), l_x, start_abs,
                               _p(out, C.c_float), _p(mass, C.c_double), _p(w, C.c_float) if w is not None else None))
    return out, mass[:ns], w


def select_representatives(scores, r_k):
    s = f32(scores)
    idx = np.zeros(max(1, min(r_k, len(s))), np.int64)
    n = C.c_int64()
    _check(lib().oracle_select_representatives(_p(s, C.c_float), len(s), r_k, _p(idx, C.c_int64),
                                               C.byref(n)))
    return idx[: n.value].tolist()


def argsort_topk(values, k):
    v = f64(values)
    idx = np.zeros(max(1, len(v)), np.int64)
    n = C.c_int64()
    _check(lib().oracle_argsort_topk(_p(v, C.c_double), len(v), k, _p(idx, C.c_int64), C.byref(n)))
    return idx[: n.value].tolist()


def relevance_all(q, repr_keys):
    q, r = f32(q), f32(repr_keys)
    l_x, H, d = q.shape
    U, rk, Hkv, _ = r.shape
    rel = np.zeros(U, np.float64)
    _check(lib().oracle_relevance_all(_p(q, C.c_float), l_x, H, Hkv, d, _p(r, C.c_float), U, rk,
                                      _p(rel, C.c_double)))
    return rel


def relevance_unit(q, repr_keys):
    q, r = f32(q), f32(repr_keys)
    l_x, H, d = q.shape
    nr, Hkv, _ = r.shape
    return lib().oracle_relevance_unit(_p(q, C.c_float), l_x, H, Hkv, d, _p(r, C.c_float), nr)


def mean_repr_relevance(unit_keys, q):
    uk, q = f64(unit_keys), f64(q)
    n, Hkv, d = uk.shape
    l_x, H, _ = q.shape
    return lib().oracle_mean_repr_relevance(_p(uk, C.c_double), n, _p(q, C.c_double), l_x, H, Hkv, d)


def dense_attention(q, k, v, position_mode=1, local_size=1 << 40):
    q, k, v = f64(q), f64(k), f64(v)
    n, H, d = q.shape
    Hkv, dv = k.shape[1], v.shape[2]
    out = np.zeros((n, H, dv), np.float64)
    _check(lib().oracle_dense_attention(_p(q, C.c_double), _p(k, C.c_double), _p(v, C.c_double), n,
                                        H, Hkv, d, dv, position_mode, local_size,
                                        _p(out, C.c_double)))
    return out


def windowed_attention(q, k, v, schedule, init_size, local_size, unit_size, position_mode=0):
    q, k, v = f64(q), f64(k), f64(v)
    n, H, d = q.shape
    Hkv, dv = k.shape[1], v.shape[2]
    sch = np.ascontiguousarray(schedule, np.int64)
    out = np.zeros((n, H, dv), np.float64)
    _check(lib().oracle_windowed_attention(_p(q, C.c_double), _p(k, C.c_double), _p(v, C.c_double),
                                           n, H, Hkv, d, dv, _p(sch, C.c_int64), len(sch),
                                           init_size, local_size, unit_size, position_mode,
                                           _p(out, C.c_double)))
    return out


def batch_repr_scores(q, k, local_size):
    q, k = f64(q), f64(k)
    n, H, d = q.shape
    out = np.zeros(n, np.float64)
    _check(lib().oracle_batch_repr_scores(_p(q, C.c_double), _p(k, C.c_double), n, H, k.shape[1], d,
                                          local_size, _p(out, C.c_double)))
    return out


def noise_ids(seed, n):
    ids = np.zeros(n, np.int64)
    lib().oracle_noise_ids(seed, n, _p(ids, C.c_int64))
    return ids


def adapter_batch(seed, shape: ModelShape, ids, layer=0):
    ids = np.ascontiguousarray(ids, np.int64)
    n = len(ids)
    H, d, dv = shape.n_heads, shape.head_dim, shape.value_dim
    q = np.zeros((n, H, d), np.float32)
    k = np.zeros((n, H, d), np.float32)
    v = np.zeros((n, H, dv), np.float32)
    _check(lib().oracle_adapter_batch(seed, shape.n_layers, H, d, dv, layer, _p(ids, C.c_int64), n,
                                      _p(q, C.c_float), _p(k, C.c_float), _p(v, C.c_float)))
    return q, k, v


def gaussian(seed, tensor, n_tok, n_head, dim, tok0=0):
    x = np.zeros((n_tok, n_head, dim), np.float32)
    lib().oracle_gaussian_fill(seed, tensor, tok0, n_tok, n_head, dim, _p(x, C.c_float))
    return x


def gen_planted(seed, length, plant_len, cfg: EngineConfig, probe_len=4, align=False):
    ids = np.zeros(length, np.int64)
    a, pid, fu, lu = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    _check(lib().oracle_gen_planted(seed, length, plant_len, C.byref(cfg), probe_len, int(align),
                                    C.byref(a), C.byref(pid), C.byref(fu), C.byref(lu),
                                    _p(ids, C.c_int64)))
    return dict(plant_start=a.value, plant_id=pid.value,
                expected_units=list(range(fu.value, lu.value + 1)), token_ids=ids,
                probe_pos=length - probe_len, probe_len=probe_len)


def encode_schedule(length, chunk, decode_tail):
    """cli.cpp:133-142"""
    sched, left = [], length - decode_tail
    while left > 0:
        sched.append(min(chunk, left))
        left -= sched[-1]
    return sched + [1] * decode_tail


def run_engine(eng: OracleEngine, q, k, v, schedule, decode_tail=0):
    """run_engine_collect (cli.cpp:89-119) with explicit tensors: returns the
    stacked outputs [n][H][dv] and the per-step retrieved ids."""
    outs, ids = [], []
    fed = 0
    first_decode = len(schedule) - decode_tail
    for s, b in enumerate(schedule):
        r = eng.step(q[fed:fed + b], k[fed:fed + b], v[fed:fed + b], decode=s >= first_decode)
        outs.append(r.out)
        ids.append(r.retrieved_ids)
        fed += b
    return np.concatenate(outs, 0), ids
