"""KV-group sharding of one InfLLM stream across GPUs.

Attention, the local ring, the unit pages and the representative index are
partitioned by KV-head group: rank r owns groups [g0, g0 + g_count) and their
query heads. Everything a shard computes alone except three sums over ALL
heads — unit relevance (memory.hpp:221-228), representative scores
(repr_score.hpp:55-57) and attention masses (engine.hpp:278-281). For those
the engine writes fp64 per-group partials into a [rows][g_total] device
buffer (its own columns) and calls the exchange hook; after the hook every
shard holds every column and sums groups 0..g_total-1 in fixed order, so the
selected ids are bit-identical for any shard count (C-1 in SURVEY §8e).

Two transports:
  * ``attach_nccl`` — one process per GPU: the library's own NCCL
    communicator (ncclAllGather on the engine's streams, graph-capturable);
  * ``ThreadExchange`` — several shards driven by host threads in ONE process
    through the infllm_allgather_fn hook (a host-synchronised exchange: each
    shard syncs its stream, publishes its columns, waits for the others).
    Used to test sharding on a single GPU without kernels that wait on each
    other.
``fold_host`` / ``topk_host`` run the library's exchange arithmetic on the
host (the multi-process CPU tests drive it over gloo).
"""
from __future__ import annotations

import threading

import numpy as np
import torch


def shard_range(n_kv_heads: int, rank: int, world: int):
    """Contiguous, equal KV-group blocks: (g0, g_count) of `rank`."""
    if world < 1 or n_kv_heads % world != 0:
        raise ValueError(f"n_kv_heads ({n_kv_heads}) must be a multiple of the shard count ({world})")
    gc = n_kv_heads // world
    return rank * gc, gc


def attach_nccl(engine, rank: int, world: int, group=None) -> None:
    """Give `engine` (this rank's KV-group shard) the library's own NCCL
    communicator (infllm_engine_set_comm): rank 0 makes the 128-byte NCCL id,
    torch.distributed (any backend) broadcasts it, every rank joins. The
    engine then all-gathers its fp64 partials with ncclAllGather on its own
    streams, inside captured stream graphs (C-1), and with option
    gather_output the outputs of every head (C-2)."""
    import ctypes as C

    import torch.distributed as dist

    from ._lib import check, lib

    buf = (C.c_uint8 * 128)()
    if rank == 0:
        check(lib().infllm_nccl_unique_id(buf))
    box = [bytes(buf)]
    dist.broadcast_object_list(box, src=0, group=group)
    idb = (C.c_uint8 * 128).from_buffer_copy(box[0])
    check(lib().infllm_engine_set_comm(engine.h, idb, rank, world))


def fold_host(gathered: np.ndarray) -> np.ndarray:
    """The library's exchange arithmetic on the host (infllm_exchange_fold_host):
    gathered [world][rows][g_count] fp64 partial blocks, as an all-gather
    delivers them, -> per-row sums over all groups in group order 0..g_total-1
    (the order k_topk / k_finalize / the LRU use on the device)."""
    import ctypes as C

    from ._lib import check, lib

    g = np.ascontiguousarray(gathered, np.float64)
    world, rows, gc = g.shape
    out = np.zeros(max(rows, 1), np.float64)
    check(lib().infllm_exchange_fold_host(g.ctypes.data_as(C.POINTER(C.c_double)), rows, world, gc,
                                          out.ctypes.data_as(C.POINTER(C.c_double))))
    return out[:rows]


def topk_host(rel: np.ndarray, k: int) -> list:
    """TieredStore::lookup's selection (memory.hpp:240-253) on the host
    (infllm_topk_host): top k by (rel desc, id asc), returned ascending."""
    import ctypes as C

    from ._lib import check, lib

    r = np.ascontiguousarray(rel, np.float64)
    ids = np.zeros(max(1, k), np.int64)
    n = C.c_int64()
    check(lib().infllm_topk_host(r.ctypes.data_as(C.POINTER(C.c_double)), len(r), k,
                                 ids.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(n)))
    return ids[:n.value].tolist()


class _DevArray:
    """__cuda_array_interface__ view of an engine-owned fp64 device buffer."""

    def __init__(self, ptr, rows, cols):
        self.__cuda_array_interface__ = dict(shape=(rows, cols), typestr="<f8", data=(ptr, False), version=3,
                                             strides=None, stream=None)


def device_buffer(ptr: int, rows: int, cols: int, device) -> torch.Tensor:
    return torch.as_tensor(_DevArray(ptr, rows, cols), device=device)


class ThreadExchange:
    """Host-synchronised exchange among `n_shards` engines in one process,
    each driven by its own host thread."""

    def __init__(self, n_shards: int, device=0):
        self.n = n_shards
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.barrier = threading.Barrier(n_shards)
        self.host = None
        self.calls = 0
        self.errors = []

    def hook(self):
        def fn(buf_ptr, rows, g0, g_count, g_total, stream_ptr):
            try:
                torch.cuda.ExternalStream(stream_ptr, device=self.device).synchronize()
                buf = device_buffer(buf_ptr, rows, g_total, self.device)
                if self.barrier.wait() == 0:
                    self.host = np.zeros((rows, g_total), np.float64)
                    self.calls += 1
                self.barrier.wait()
                self.host[:, g0:g0 + g_count] = buf[:, g0:g0 + g_count].cpu().numpy()
                self.barrier.wait()
                buf.copy_(torch.from_numpy(self.host).to(self.device))
                torch.cuda.synchronize(self.device)
                self.barrier.wait()
                return 0
            except Exception as exc:  # kept for the caller; the C side reports INFLLM_ERR_NCCL
                self.errors.append(repr(exc))
                self.barrier.abort()
                return 1

        return fn
