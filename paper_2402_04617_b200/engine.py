"""Python mirror of the reference operator API for the InfLLM hot path.

``StreamEngine`` keeps the names and semantics of blockmem::StreamEngine
(engine.hpp:63-395): ``encode_chunk``, ``decode_step``, ``feed``, ``finish``,
``metrics``, plus store accessors mirroring TieredStore (memory.hpp:170-323).
The difference the reference itself documents as out of scope for its
adapter is that q/k/v are passed in explicitly as CUDA tensors:
q [l_x][n_heads][head_dim], k/v [l_x][n_kv_heads][dim].

Everything runs in libinfllm_b200.so (C-ABI, hand-written sm_100a kernels);
this module only marshals tensors and pointers.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import EngineConfig, LayerMetrics, ModelShape, check, lib

_DT = {torch.float32: _lib.DTYPE_F32, torch.bfloat16: _lib.DTYPE_BF16}


@dataclass
class LayerStepOutput:
    """LayerStepOutput (engine.hpp:25-30): attention output + retrieved ids."""

    out: torch.Tensor
    retrieved_ids: list


class StreamEngine:
    def __init__(self, config: EngineConfig, shape: ModelShape, dtype=torch.bfloat16, device=0,
                 kv_group_begin=0, kv_group_count=0):
        if not torch.cuda.is_available():
            raise RuntimeError("StreamEngine needs a CUDA device (B200); there is no CPU fallback")
        self.config, self.shape, self.dtype = config, shape, dtype
        self.device = torch.device("cuda", device)
        h = C.c_void_p()
        check(lib().infllm_engine_create(C.byref(config), C.byref(shape), _DT[dtype], device, kv_group_begin,
                                         kv_group_count, C.byref(h)))
        self.h = h
        g = kv_group_count if kv_group_count > 0 else shape.n_kv_heads
        self.n_kv_local = g
        self.n_heads_local = g * (shape.n_heads // shape.n_kv_heads)
        self._cb = None

    def close(self):
        if getattr(self, "h", None):
            try:
                lib().infllm_engine_destroy(self.h)
            except Exception:
                pass
            self.h = None

    __del__ = close

    # ---- configuration ----
    def reserve(self, max_tokens: int):
        check(lib().infllm_engine_reserve(self.h, int(max_tokens)))

    def reset(self, stream=None):
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        check(lib().infllm_engine_reset(self.h, st))

    def set_option(self, key: str, value: int):
        check(lib().infllm_engine_set_option(self.h, key.encode(), int(value)))

    def set_comm(self, rank: int, world: int, group=None):
        """KV-group sharding over the library's NCCL communicator (see shard.attach_nccl)."""
        from .shard import attach_nccl

        attach_nccl(self, rank, world, group)

    def set_allgather(self, fn):
        """fn(buf_ptr, rows, g0, g_count, g_total, stream_ptr) -> 0; see infllm_allgather_fn."""
        if fn is None:
            self._cb = None
            check(lib().infllm_engine_set_allgather(self.h, _lib.ALLGATHER_FN(), None))
            return
        self._cb = _lib.ALLGATHER_FN(lambda user, buf, rows, g0, gc, gt, st: fn(buf, rows, g0, gc, gt, st))
        check(lib().infllm_engine_set_allgather(self.h, self._cb, None))

    # ---- stream ----
    def _check_inputs(self, q, k, v):
        for t in (q, k, v):
            if t.device != self.device or t.dtype != self.dtype or not t.is_contiguous():
                raise ValueError("q/k/v must be contiguous tensors of the engine dtype on the engine device")

    def encode_chunk(self, q, k, v, layer=0, out=None, stream=None) -> torch.Tensor:
        """StreamEngine::encode_chunk (engine.hpp:92-97) for one layer."""
        self._check_inputs(q, k, v)
        lx = q.shape[0]
        if out is None:
            out = torch.empty((lx, self.n_heads_local, self.shape.value_dim), dtype=self.dtype, device=self.device)
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        check(lib().infllm_encode_chunk(self.h, layer, q.data_ptr(), k.data_ptr(), v.data_ptr(), lx, out.data_ptr(),
                                        st))
        return out

    def decode_step(self, q, k, v, layer=0, out=None, stream=None) -> torch.Tensor:
        """StreamEngine::decode_step (engine.hpp:100-103)."""
        self._check_inputs(q, k, v)
        if out is None:
            out = torch.empty((1, self.n_heads_local, self.shape.value_dim), dtype=self.dtype, device=self.device)
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        check(lib().infllm_decode_step(self.h, layer, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), st))
        return out

    def step(self, q, k, v, decode=False, layer=0) -> LayerStepOutput:
        out = self.decode_step(q, k, v, layer) if decode else self.encode_chunk(q, k, v, layer)
        return LayerStepOutput(out, self.retrieved_ids(layer))

    def feed(self, q, k, v, layer=0):
        """StreamEngine::feed (engine.hpp:106-112): whole sequence as chunks."""
        n, c = q.shape[0], int(self.config.chunk_size)
        outs = []
        for off in range(0, n, c):
            outs.append(self.encode_chunk(q[off:off + c], k[off:off + c], v[off:off + c], layer))
        return torch.cat(outs, 0)

    def encode_stream(self, q, k, v, out=None, layer=0, stream=None) -> torch.Tensor:
        """Whole-sequence feed through the C-ABI in one call (graph-replayed
        chunk schedule); q/k/v/out device tensors."""
        self._check_inputs(q, k, v)
        n = q.shape[0]
        if out is None:
            out = torch.empty((n, self.n_heads_local, self.shape.value_dim), dtype=self.dtype, device=self.device)
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        check(lib().infllm_encode_stream(self.h, layer, q.data_ptr(), k.data_ptr(), v.data_ptr(), n, out.data_ptr(),
                                         st))
        return out

    def encode_stream_host(self, q, k, v, out, layer=0, stream=None):
        """Host-buffer feed (pinned CPU tensors q/k/v/out) through the C-ABI."""
        for t in (q, k, v, out):
            if t.device.type != "cpu" or t.dtype != self.dtype or not t.is_contiguous():
                raise ValueError("host tensors must be contiguous CPU tensors of the engine dtype")
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        check(lib().infllm_encode_stream_host(self.h, layer, q.data_ptr(), k.data_ptr(), v.data_ptr(), q.shape[0],
                                              out.data_ptr(), st))
        return out

    def finish(self):
        """StreamEngine::finish (engine.hpp:115-119)."""
        check(lib().infllm_finish(self.h, torch.cuda.current_stream(self.device).cuda_stream))

    # ---- diagnostics ----
    def retrieved_ids(self, layer=0):
        cap = max(1, int(self.config.n_lookup))
        ids = np.zeros(cap, np.int64)
        n = C.c_int64()
        check(lib().infllm_retrieved_ids(self.h, layer, ids.ctypes.data_as(_lib.i64p), cap, C.byref(n)))
        return ids[: n.value].tolist()

    def metrics(self, layer=0):
        m = LayerMetrics()
        check(lib().infllm_get_layer_metrics(self.h, layer, C.byref(m)))
        return m.as_dict()

    def stream_state(self, layer=0):
        vals = [C.c_int64() for _ in range(5)]
        check(lib().infllm_stream_state(self.h, layer, *[C.byref(x) for x in vals]))
        return dict(zip(["tokens_fed", "steps", "initial_len", "local_len", "pending_partial"],
                        [x.value for x in vals]))

    def unit_info(self, uid, layer=0):
        s, z, n = C.c_int64(), C.c_int64(), C.c_int64()
        r = np.zeros(max(1, int(self.config.n_repr)), np.int64)
        check(lib().infllm_unit_info(self.h, layer, uid, C.byref(s), C.byref(z), r.ctypes.data_as(_lib.i64p),
                                     C.byref(n)))
        return dict(start_abs=s.value, size=z.value, repr_abs=r[: n.value].tolist())

    def unit_freq(self, n, layer=0):
        f = np.zeros(max(n, 1), np.float64)
        hot = np.zeros(max(n, 1), np.int32)
        check(lib().infllm_unit_freq(self.h, layer, f.ctypes.data_as(_lib.f64p), hot.ctypes.data_as(_lib.i32p), n))
        return f[:n], hot[:n]

    def trace(self, layer=0, cap=1 << 20):
        st, un = np.zeros(cap, np.int64), np.zeros(cap, np.int64)
        hit = np.zeros(cap, np.int32)
        n = C.c_int64()
        check(lib().infllm_trace(self.h, layer, st.ctypes.data_as(_lib.i64p), un.ctypes.data_as(_lib.i64p),
                                 hit.ctypes.data_as(_lib.i32p), cap, C.byref(n)))
        k = min(cap, n.value)
        return list(zip(st[:k].tolist(), un[:k].tolist(), hit[:k].tolist()))

    def tier_stats(self, layer=0):
        """Host tier counters: page loads, cache hits, H2D bytes, slots (infllm_tier_stats)."""
        out = (C.c_int64 * 4)()
        check(lib().infllm_tier_stats(self.h, int(layer), out))
        return dict(loads=out[0], cache_hits=out[1], h2d_bytes=out[2], slots=out[3])

    def kernel_launches(self):
        n = C.c_int64()
        check(lib().infllm_kernel_launches(self.h, C.byref(n)))
        return n.value

    def profile_begin(self, enable=True):
        check(lib().infllm_profile_begin(self.h, int(enable)))

    def phase_timings(self):
        """PhaseTimings (engine.hpp:43-49) of the profile window: device ms per phase."""
        ms = (C.c_double * 4)()
        n = (C.c_int64 * 4)()
        check(lib().infllm_phase_timings(self.h, ms, n))
        return {"lookup": ms[0], "attend": ms[1], "score": ms[2], "evict": ms[3]}

    def invariants(self):
        """(invariant_checks, invariant_violations) (engine.hpp:88-89)."""
        c, v = C.c_uint64(), C.c_uint64()
        check(lib().infllm_invariants(self.h, C.byref(c), C.byref(v)))
        return c.value, v.value

    def profile_read(self):
        a, b = C.c_double(), C.c_double()
        na, nb = C.c_int64(), C.c_int64()
        check(lib().infllm_profile_read(self.h, C.byref(a), C.byref(na), C.byref(b), C.byref(nb)))
        return dict(attn_ms=a.value, attn_launches=na.value, lookup_ms=b.value, lookup_launches=nb.value)


def decode_batch(engines, q, k, v, out=None, layer=0, stream=None):
    """One decode step of len(engines) independent sequences (infllm_decode_batch):
    q [B][H][d], k/v [B][H_kv][d] device tensors; returns out [B][H][d_v]."""
    e0 = engines[0]
    for t in (q, k, v):
        if t.device != e0.device or t.dtype != e0.dtype or not t.is_contiguous() or t.shape[0] != len(engines):
            raise ValueError("q/k/v must be contiguous [B][heads][dim] tensors of the engines' dtype/device")
    if out is None:
        out = torch.empty((len(engines), e0.n_heads_local, e0.shape.value_dim), dtype=e0.dtype, device=e0.device)
    hs = (C.c_void_p * len(engines))(*[e.h.value for e in engines])
    st = (stream or torch.cuda.current_stream(e0.device)).cuda_stream
    check(lib().infllm_decode_batch(hs, len(engines), layer, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                    st))
    return out


def select_representatives(scores: torch.Tensor, r_k: int, lens: torch.Tensor | None = None) -> torch.Tensor:
    """select_representatives (repr_score.hpp:94-112), batched over units on the GPU.
    scores [n_units][unit_len] fp32 CUDA -> idx [n_units][r_k] int64 (-1 = unused)."""
    if scores.dim() == 1:
        scores = scores[None]
    scores = scores.contiguous().float()
    n, ul = scores.shape
    idx = torch.empty((n, r_k), dtype=torch.int64, device=scores.device)
    lp = lens.contiguous().long().data_ptr() if lens is not None else None
    check(lib().infllm_select_representatives(scores.data_ptr(), lp, n, ul, r_k, idx.data_ptr(),
                                              torch.cuda.current_stream(scores.device).cuda_stream))
    return idx


def lookup(qsum: torch.Tensor, repr_keys: torch.Tensor, k_m: int):
    """TieredStore::relevance_all + lookup top-k (memory.hpp:217-253) on the GPU.
    qsum [n_kv][d] fp64 (chunk query sum per KV group), repr_keys
    [U][n_kv][r_k][d] (fp32/bf16) -> (rel [U] fp64, ids ascending)."""
    U, G, rk, d = repr_keys.shape
    rel = torch.empty(U, dtype=torch.float64, device=repr_keys.device)
    ids = torch.empty(max(1, min(k_m, U)), dtype=torch.int64, device=repr_keys.device)
    check(lib().infllm_lookup(qsum.contiguous().data_ptr(), repr_keys.contiguous().data_ptr(), _DT[repr_keys.dtype],
                              U, rk, G, d, k_m, rel.data_ptr(), ids.data_ptr(),
                              torch.cuda.current_stream(repr_keys.device).cuda_stream))
    return rel, ids[: min(k_m, U)]


def attend(segments, q, k, v, start_abs, local_size, position_mode="clamped", emit_weights=False, stream=None):
    """blockmem::attend (attention.hpp:116-230) on the GPU (infllm_attend).

    segments: [(kind, start_abs, keys [n][H_kv][d], values [n][H_kv][d_v])] device tensors, kind in
    "initial" / "retrieved" / "local" (attention.hpp:14-26), keys raw; q [l_x][H][d], k/v [l_x][H_kv][*]
    the causal batch at absolute positions start_abs... Returns (out [l_x][H][d_v], per-segment mass
    (engine.hpp:271-283), weights [H][l_x][n_ctx + l_x] fp32 or None)."""
    l_x, H, d = q.shape
    Hkv, dv = v.shape[1], v.shape[2]
    dt = _DT[q.dtype]
    for t in [q, k, v] + [x for s in segments for x in (s[2], s[3])]:
        if t.dtype != q.dtype or not t.is_contiguous() or t.device != q.device:
            raise ValueError("attend: contiguous tensors of one dtype on one device")
    ns = len(segments)
    segs = (_lib.Segment * max(1, ns))()
    for i, (kind, start, keys, vals) in enumerate(segments):
        segs[i] = _lib.Segment(_lib.SEG_KINDS[kind] if isinstance(kind, str) else kind, start, keys.shape[0],
                               keys.data_ptr(), vals.data_ptr())
    n_ctx = sum(s[2].shape[0] for s in segments)
    out = torch.empty((l_x, H, dv), dtype=q.dtype, device=q.device)
    mass = torch.zeros(max(1, ns), dtype=torch.float64, device=q.device)
    w = torch.empty((H, l_x, n_ctx + l_x), dtype=torch.float32, device=q.device) if emit_weights else None
    shape = ModelShape.make(n_heads=H, n_kv_heads=Hkv, head_dim=d, value_dim=dv)
    pm = _lib.POSITION_MODES[position_mode] if isinstance(position_mode, str) else position_mode
    st = (stream or torch.cuda.current_stream(q.device)).cuda_stream
    check(lib().infllm_attend(C.byref(shape), dt, pm, local_size, segs, ns, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                              l_x, start_abs, out.data_ptr(), mass.data_ptr(), w.data_ptr() if w is not None else None,
                              st))
    return out, mass[:ns], w


class TieredStore:
    """blockmem::TieredStore (memory.hpp:170-323) on the GPU (infllm_store_*)."""

    def __init__(self, hot_capacity, decay, n_heads, n_kv_heads, head_dim, n_repr=4, dtype=torch.bfloat16,
                 bytes_per_token=0):
        h = C.c_void_p()
        check(lib().infllm_store_create(hot_capacity, decay, n_heads, n_kv_heads, head_dim, n_repr, _DT[dtype],
                                        bytes_per_token, C.byref(h)))
        self.h, self.dtype, self.k_cap = h, dtype, 128

    def close(self):
        if getattr(self, "h", None):
            try:
                lib().infllm_store_destroy(self.h)
            except Exception:
                pass
            self.h = None

    __del__ = close

    def add_unit(self, repr_keys, unit_tokens):
        """add_unit (memory.hpp:196-212): repr_keys [n][H_kv][d] device -> unit id."""
        uid = C.c_int64()
        check(lib().infllm_store_add_unit(self.h, repr_keys.contiguous().data_ptr(), repr_keys.shape[0], unit_tokens,
                                          C.byref(uid)))
        return uid.value

    def begin_step(self, step):
        check(lib().infllm_store_begin_step(self.h, step))

    def lookup(self, q, k_m, rel=None):
        """lookup (memory.hpp:239-269): batch queries q [l_x][H][d] (device) -> ascending ids."""
        ids = np.zeros(max(1, k_m), np.int64)
        n = C.c_int64()
        check(lib().infllm_store_lookup(self.h, q.contiguous().data_ptr(), q.shape[0], k_m,
                                        ids.ctypes.data_as(_lib.i64p), C.byref(n),
                                        rel.data_ptr() if rel is not None else None))
        return ids[: n.value].tolist()

    def update_frequency(self, pairs):
        ids = np.array([p[0] for p in pairs] or [0], np.int64)
        ms = np.array([p[1] for p in pairs] or [0.0], np.float64)
        check(lib().infllm_store_update_frequency(self.h, ids.ctypes.data_as(_lib.i64p), ms.ctypes.data_as(_lib.f64p),
                                                  len(pairs)))

    def enforce_capacity(self):
        check(lib().infllm_store_enforce_capacity(self.h))

    def note_step_boundary(self):
        check(lib().infllm_store_note_step_boundary(self.h))

    def counters(self):
        m = LayerMetrics()
        check(lib().infllm_store_counters(self.h, C.byref(m)))
        return m.as_dict()

    def trace(self, cap=1 << 16):
        st, un = np.zeros(cap, np.int64), np.zeros(cap, np.int64)
        hit = np.zeros(cap, np.int32)
        n = C.c_int64()
        check(lib().infllm_store_trace(self.h, st.ctypes.data_as(_lib.i64p), un.ctypes.data_as(_lib.i64p),
                                       hit.ctypes.data_as(_lib.i32p), cap, C.byref(n)))
        k = min(cap, n.value)
        return list(zip(st[:k].tolist(), un[:k].tolist(), hit[:k].tolist()))

    def unit_freq(self, n):
        f = np.zeros(max(1, n), np.float64)
        hot = np.zeros(max(1, n), np.int32)
        check(lib().infllm_store_unit_freq(self.h, f.ctypes.data_as(_lib.f64p), hot.ctypes.data_as(_lib.i32p), n))
        return f[:n], hot[:n]


class ScoreAccumulator:
    """blockmem::ScoreAccumulator (repr_score.hpp:21-89) on the GPU (infllm_score_acc_*)."""

    def __init__(self, local_size, n_heads, n_kv_heads, head_dim, dtype=torch.float32):
        h = C.c_void_p()
        check(lib().infllm_score_acc_create(local_size, n_heads, n_kv_heads, head_dim, _DT[dtype], C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            try:
                lib().infllm_score_acc_destroy(self.h)
            except Exception:
                pass
            self.h = None

    __del__ = close

    def accumulate(self, q, s, pending_keys, stream=None):
        st = (stream or torch.cuda.current_stream(q.device)).cuda_stream
        check(lib().infllm_score_acc_accumulate(self.h, q.contiguous().data_ptr(), q.shape[0], s,
                                                pending_keys.contiguous().data_ptr(), pending_keys.shape[0], st))

    def finalize_front(self, n):
        torch.cuda.synchronize()
        out = np.zeros(max(1, n), np.float32)
        check(lib().infllm_score_acc_finalize_front(self.h, n, out.ctypes.data_as(C.POINTER(C.c_float))))
        return out[:n]
