"""TEST INFRASTRUCTURE ONLY — ctypes binding of oracle/_ref, the reference
engine compiled from /root/reference/proj/include where it lies (against the
Eigen-subset shim, see oracle/Makefile). Used to pin the oracle restatement
(tests/test_oracle_pin.py), to generate tests/golden fixtures
(tests/golden/make_golden.py) and, in bench.py's CPU legs only, to time the
reference beside the port on C0. /root/reference is absent on the GPU box:
there only the prebuilt oracle/_ref/*.so (shipped with the repo snapshot)
are loaded, never rebuilt.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from .oracle import EngineConfig, _p, f32, f64

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
REF_SRC = "/root/reference/proj/include/blockmem"


def available() -> bool:
    return os.path.isdir(REF_SRC) or os.path.exists(os.path.join(REF_DIR, "libblockmem_ref.so"))


def build():
    if os.path.isdir(REF_SRC):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])


_libs = {}


def lib(inject=True):
    key = bool(inject)
    if key not in _libs:
        name = "libblockmem_ref.so" if inject else "libblockmem_ref_adapter.so"
        path = os.path.join(REF_DIR, name)
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        P, i64p, f32p, f64p = C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_float), C.POINTER(C.c_double)
        L.ref_last_error.restype = C.c_char_p
        if inject:
            L.ref_set_inputs.argtypes = [C.c_int, f32p, f32p, f32p, C.c_int64, C.c_int, C.c_int, C.c_int]
        L.ref_engine_create.restype = P
        L.ref_engine_create.argtypes = [C.POINTER(EngineConfig), C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64]
        L.ref_engine_destroy.argtypes = [P]
        L.ref_set_always_emit_weights.argtypes = [P, C.c_int]
        L.ref_step.argtypes = [P, i64p, C.c_int64, C.c_int, f32p, i64p, C.c_int64, i64p]
        L.ref_finish.argtypes = [P]
        L.ref_metrics.argtypes = [P, C.c_int, i64p]
        L.ref_invariants.argtypes = [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.ref_stream_state.argtypes = [P, C.c_int, i64p]
        L.ref_unit_info.argtypes = [P, C.c_int, C.c_int64, i64p, i64p, i64p, i64p, f64p, C.POINTER(C.c_int)]
        L.ref_trace.argtypes = [P, C.c_int, i64p, i64p, C.POINTER(C.c_int), C.c_int64, i64p]
        L.ref_select_representatives.argtypes = [f32p, C.c_int64, C.c_int64, i64p, i64p]
        L.ref_argsort_topk.argtypes = [f64p, C.c_int64, C.c_int64, i64p, i64p]
        L.ref_dense_attention.argtypes = [f64p, f64p, f64p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_int64, f64p]
        L.ref_windowed_attention.argtypes = [f64p, f64p, f64p, C.c_int64, C.c_int, C.c_int, C.c_int, i64p,
                                             C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int, f64p]
        L.ref_batch_repr_scores.argtypes = [f64p, f64p, C.c_int64, C.c_int, C.c_int, C.c_int64, f64p]
        L.ref_accumulator_scores.argtypes = [f32p, f32p, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_int64, f32p]
        L.ref_store_lookup.argtypes = [f32p, C.c_int64, C.c_int, C.c_int, f32p, C.c_int64, C.c_int64, C.c_int64,
                                       f64p, i64p, i64p]
        _libs[key] = L
    return _libs[key]


def _check(L, rc):
    if rc != 0:
        raise RuntimeError(f"reference error [{rc}]: {L.ref_last_error().decode()}")


def expand_kv(x, n_heads):
    """GQA -> MHA by replicating each KV head over its query heads."""
    rep = n_heads // x.shape[1]
    return np.repeat(x, rep, axis=1)


class RefEngine:
    """blockmem::StreamEngine<float> (engine.hpp:63-395), the reference's own code."""

    def __init__(self, cfg: EngineConfig, n_heads, head_dim, value_dim=None, n_layers=1, seed=0, inject=True):
        self.L = lib(inject)
        self.inject = inject
        self.H, self.d, self.dv, self.n_layers = n_heads, head_dim, value_dim or head_dim, n_layers
        self.cfg = cfg
        self.h = self.L.ref_engine_create(C.byref(cfg), n_layers, n_heads, head_dim, self.dv, seed)
        if not self.h:
            raise RuntimeError(self.L.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_engine_destroy(self.h)
            self.h = None

    def set_inputs(self, q, k, v, layer=0):
        """q [n][H][d]; k/v [n][Hkv][d] (expanded to H heads here)."""
        q = f32(q)
        k = f32(expand_kv(k, self.H))
        v = f32(expand_kv(v, self.H))
        _check(self.L, self.L.ref_set_inputs(layer, _p(q, C.c_float), _p(k, C.c_float), _p(v, C.c_float),
                                             q.shape[0], self.H, self.d, self.dv))

    def set_always_emit_weights(self, v=True):
        self.L.ref_set_always_emit_weights(self.h, int(v))

    def step(self, l_x, decode=False, ids=None):
        cap = max(1, int(self.cfg.n_lookup))
        out = np.zeros((self.n_layers, l_x, self.H, self.dv), np.float32)
        ids_out = np.zeros((self.n_layers, cap), np.int64)
        n_ids = np.zeros(self.n_layers, np.int64)
        idp = None
        if ids is not None:
            ids = np.ascontiguousarray(ids, np.int64)
            idp = _p(ids, C.c_int64)
        _check(self.L, self.L.ref_step(self.h, idp, l_x, int(decode), _p(out, C.c_float), _p(ids_out, C.c_int64),
                                       cap, _p(n_ids, C.c_int64)))
        return out, [ids_out[l, : n_ids[l]].tolist() for l in range(self.n_layers)]

    def finish(self):
        _check(self.L, self.L.ref_finish(self.h))

    def metrics(self, layer=0):
        m = np.zeros(9, np.int64)
        _check(self.L, self.L.ref_metrics(self.h, layer, _p(m, C.c_int64)))
        keys = ["units", "hot_units", "peak_hot_units", "peak_hot_bytes", "hits", "misses", "loads",
                "evictions", "requested"]
        return dict(zip(keys, m.tolist()))

    def invariants(self):
        c, v = C.c_uint64(), C.c_uint64()
        self.L.ref_invariants(self.h, C.byref(c), C.byref(v))
        return c.value, v.value

    def stream_state(self, layer=0):
        s = np.zeros(5, np.int64)
        _check(self.L, self.L.ref_stream_state(self.h, layer, _p(s, C.c_int64)))
        return dict(zip(["tokens_fed", "steps", "initial_len", "local_len", "pending_partial"], s.tolist()))

    def unit_info(self, uid, layer=0):
        s, z, n = C.c_int64(), C.c_int64(), C.c_int64()
        r = np.zeros(max(1, int(self.cfg.n_repr)), np.int64)
        f = C.c_double()
        hot = C.c_int()
        _check(self.L, self.L.ref_unit_info(self.h, layer, uid, C.byref(s), C.byref(z), _p(r, C.c_int64),
                                            C.byref(n), C.byref(f), C.byref(hot)))
        return dict(start_abs=s.value, size=z.value, repr_abs=r[: n.value].tolist(), freq=f.value, hot=hot.value)

    def trace(self, layer=0, cap=1 << 20):
        st, un = np.zeros(cap, np.int64), np.zeros(cap, np.int64)
        hit = np.zeros(cap, np.int32)
        n = C.c_int64()
        _check(self.L, self.L.ref_trace(self.h, layer, _p(st, C.c_int64), _p(un, C.c_int64), _p(hit, C.c_int),
                                        cap, C.byref(n)))
        k = min(n.value, cap)
        return list(zip(st[:k].tolist(), un[:k].tolist(), hit[:k].tolist()))


def select_representatives(scores, r_k):
    L = lib(True)
    s = f32(scores)
    idx = np.zeros(max(1, len(s)), np.int64)
    n = C.c_int64()
    _check(L, L.ref_select_representatives(_p(s, C.c_float), len(s), r_k, _p(idx, C.c_int64), C.byref(n)))
    return idx[: n.value].tolist()


def argsort_topk(values, k):
    L = lib(True)
    v = f64(values)
    idx = np.zeros(max(1, len(v)), np.int64)
    n = C.c_int64()
    _check(L, L.ref_argsort_topk(_p(v, C.c_double), len(v), k, _p(idx, C.c_int64), C.byref(n)))
    return idx[: n.value].tolist()


def dense_attention(q, k, v, position_mode, local_size):
    L = lib(True)
    H = q.shape[1]
    q, k, v = f64(q), f64(expand_kv(k, H)), f64(expand_kv(v, H))
    n, _, d = q.shape
    dv = v.shape[2]
    out = np.zeros((n, H, dv), np.float64)
    _check(L, L.ref_dense_attention(_p(q, C.c_double), _p(k, C.c_double), _p(v, C.c_double), n, H, d, dv,
                                    position_mode, local_size, _p(out, C.c_double)))
    return out


def windowed_attention(q, k, v, schedule, init_size, local_size, unit_size, position_mode=0):
    L = lib(True)
    H = q.shape[1]
    q, k, v = f64(q), f64(expand_kv(k, H)), f64(expand_kv(v, H))
    n, _, d = q.shape
    dv = v.shape[2]
    sch = np.ascontiguousarray(schedule, np.int64)
    out = np.zeros((n, H, dv), np.float64)
    _check(L, L.ref_windowed_attention(_p(q, C.c_double), _p(k, C.c_double), _p(v, C.c_double), n, H, d, dv,
                                       _p(sch, C.c_int64), len(sch), init_size, local_size, unit_size,
                                       position_mode, _p(out, C.c_double)))
    return out


def batch_repr_scores(q, k, local_size):
    L = lib(True)
    H = q.shape[1]
    q, k = f64(q), f64(expand_kv(k, H))
    n, _, d = q.shape
    out = np.zeros(n, np.float64)
    _check(L, L.ref_batch_repr_scores(_p(q, C.c_double), _p(k, C.c_double), n, H, d, local_size,
                                      _p(out, C.c_double)))
    return out


def accumulator_scores(q, k, local_size, chunk):
    L = lib(True)
    H = q.shape[1]
    q, k = f32(q), f32(expand_kv(k, H))
    n, _, d = q.shape
    out = np.zeros(n, np.float32)
    _check(L, L.ref_accumulator_scores(_p(q, C.c_float), _p(k, C.c_float), n, H, d, local_size, chunk,
                                       _p(out, C.c_float)))
    return out


def store_lookup(q, repr_keys, k_m):
    """TieredStore::relevance_all + lookup (memory.hpp:217-269) on explicit
    representative keys repr_keys [U][r_k][Hkv][d]."""
    L = lib(True)
    H = q.shape[1]
    q = f32(q)
    r = f32(np.repeat(repr_keys, H // repr_keys.shape[2], axis=2))
    l_x, _, d = q.shape
    U, rk = r.shape[0], r.shape[1]
    rel = np.zeros(max(1, U), np.float64)
    ids = np.zeros(max(1, U), np.int64)
    n = C.c_int64()
    _check(L, L.ref_store_lookup(_p(q, C.c_float), l_x, H, d, _p(r, C.c_float), U, rk, k_m, _p(rel, C.c_double),
                                 _p(ids, C.c_int64), C.byref(n)))
    return rel[:U], ids[: n.value].tolist()
