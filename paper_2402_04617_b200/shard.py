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

Two hooks:
  * ``DistExchange`` — one process per GPU, ``torch.distributed`` all-gather
    (NCCL on GPUs; gloo works for the host-side logic tests);
  * ``ThreadExchange`` — several shards driven by host threads in ONE process
    (a host-synchronised exchange: each shard syncs its stream, publishes its
    columns, waits for the others). Used to test sharding on a single GPU
    without kernels that wait on each other.
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


def merge_columns(buf: torch.Tensor, gathered: torch.Tensor, g_count: int) -> None:
    """gathered [world][rows][g_count] (rank order == group order) -> buf [rows][g_total]."""
    world, rows, _ = gathered.shape
    buf.copy_(gathered.permute(1, 0, 2).reshape(rows, world * g_count))


def exchange(buf: torch.Tensor, g0: int, g_count: int, group=None) -> None:
    """All-gather the per-group partial columns of buf [rows][g_total] in place."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rows, g_total = buf.shape
    if world * g_count != g_total:
        raise ValueError("shards must own equal KV-group blocks")
    local = buf[:, g0:g0 + g_count].contiguous()
    gathered = torch.empty((world * rows, g_count), dtype=buf.dtype, device=buf.device)
    dist.all_gather_into_tensor(gathered, local, group=group)
    merge_columns(buf, gathered.view(world, rows, g_count), g_count)


class _DevArray:
    """__cuda_array_interface__ view of an engine-owned fp64 device buffer."""

    def __init__(self, ptr, rows, cols):
        self.__cuda_array_interface__ = dict(shape=(rows, cols), typestr="<f8", data=(ptr, False), version=3,
                                             strides=None, stream=None)


def device_buffer(ptr: int, rows: int, cols: int, device) -> torch.Tensor:
    return torch.as_tensor(_DevArray(ptr, rows, cols), device=device)


class DistExchange:
    """infllm_allgather_fn backed by torch.distributed (NCCL), issued on the
    engine's stream so it orders with the producing and consuming kernels."""

    def __init__(self, device, group=None):
        self.device = torch.device(device)
        self.group = group

    def __call__(self, buf_ptr, rows, g0, g_count, g_total, stream_ptr) -> int:
        try:
            if rows == 0:
                return 0
            buf = device_buffer(buf_ptr, rows, g_total, self.device)
            with torch.cuda.stream(torch.cuda.ExternalStream(stream_ptr, device=self.device)):
                exchange(buf, g0, g_count, self.group)
            return 0
        except Exception:  # the C side turns a non-zero return into INFLLM_ERR_NCCL
            return 1


class ThreadExchange:
    """Host-synchronised exchange among `n_shards` engines in one process,
    each driven by its own host thread."""

    def __init__(self, n_shards: int, device=0):
        self.n = n_shards
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.barrier = threading.Barrier(n_shards)
        self.host = None
        self.calls = 0

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
            except Exception:
                self.barrier.abort()
                return 1

        return fn
