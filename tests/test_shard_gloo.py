"""Host-side logic of KV-group sharding on CPU: world_size-2
torch.distributed (gloo) processes stand in for the NCCL ranks. Each rank
computes its KV groups' fp64 relevance partials, the all-gather delivers the
contiguous [rank][rows][groups] blocks NCCL would, and the library's own
exchange arithmetic (infllm_exchange_fold_host: the column fold in group
order the device runs after ncclAllGather) and its top-k (infllm_topk_host)
produce the ids, checked against the unsharded fold and the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2402_04617_b200.shard import fold_host, shard_range, topk_host


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def group_partials(q, reprk, groups):
    """Per-KV-group fp64 relevance partials (what the lookup kernel writes):
    col g = sum_r sum_d qsum_g[d] * repr[u, g, r, d]; q [l][H][d], reprk [U][G][r][d]."""
    l, H, d = q.shape
    G = reprk.shape[1]
    qs = q.astype(np.float64).reshape(l, G, H // G, d).sum(axis=(0, 2))  # [G][d]
    out = np.zeros((reprk.shape[0], G), np.float64)
    for g in groups:
        out[:, g] = np.einsum("d,urd->u", qs[g], reprk[:, g].astype(np.float64))
    return out


def topk_ids(rel, k):
    order = sorted(range(len(rel)), key=lambda i: (-rel[i], i))[:k]
    return sorted(order)


def _worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        G, U, k = 8, 500, 16
        rng = np.random.default_rng(0)  # same inputs on every rank
        q = rng.standard_normal((64, 32, 32)).astype(np.float32)
        reprk = rng.standard_normal((U, G, 4, 32)).astype(np.float32)
        g0, gc = shard_range(G, rank, world)
        mine = torch.from_numpy(np.ascontiguousarray(group_partials(q, reprk, range(g0, g0 + gc))[:, g0:g0 + gc]))
        gathered = torch.empty((world * U, gc), dtype=torch.float64)
        dist.all_gather_into_tensor(gathered, mine)  # [rank][rows][groups], as ncclAllGather delivers it
        rel = fold_host(gathered.numpy().reshape(world, U, gc))
        result_q.put((rank, rel.tobytes(), topk_host(rel, k)))
    finally:
        dist.destroy_process_group()


def test_shard_range():
    assert shard_range(8, 0, 2) == (0, 4) and shard_range(8, 1, 2) == (4, 4)
    assert [shard_range(8, r, 8) for r in range(8)] == [(r, 1) for r in range(8)]
    with pytest.raises(ValueError):
        shard_range(8, 0, 3)


def test_fold_host_group_order():
    """[rank][rows][groups] blocks fold as rank 0's groups, then rank 1's: group order 0..g_total-1."""
    g = np.arange(2 * 3 * 4, dtype=np.float64).reshape(2, 3, 4) + 0.25
    want = np.concatenate([g[0], g[1]], axis=1)
    ref = np.zeros(3)
    for c in range(8):  # sequential fold in group order, like k_topk
        ref = ref + want[:, c]
    assert fold_host(g).tobytes() == ref.tobytes()
    assert topk_host(np.array([1.0, 3.0, 3.0, -0.0, 0.0, 2.0]), 3) == [1, 2, 5]  # ties -> lower id


@pytest.mark.parametrize("world", [2])
def test_gloo_exchange_matches_unsharded(world):
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q_)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q_.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    # every rank ends with the same bits and the same ids ...
    assert all(r[1] == res[0][1] for r in res)
    assert all(r[2] == res[0][2] for r in res)
    # ... equal to the single-shard computation (sum of all groups in order)
    G, U, k = 8, 500, 16
    rng = np.random.default_rng(0)
    q = rng.standard_normal((64, 32, 32)).astype(np.float32)
    reprk = rng.standard_normal((U, G, 4, 32)).astype(np.float32)
    full = fold_host(group_partials(q, reprk, range(G))[None])  # one shard owning every group
    assert np.frombuffer(res[0][1], np.float64).tobytes() == full.tobytes()
    assert res[0][2] == topk_ids(full, k) == topk_host(full, k)
    # and the oracle's head-by-head relevance (memory.hpp:217-234) picks the same units
    from oracle import oracle as O

    orel = O.relevance_all(q, reprk.transpose(0, 2, 1, 3))
    assert np.allclose(orel, full, rtol=1e-12, atol=1e-9)
    assert sorted(O.argsort_topk(orel, k)) == res[0][2]
