"""Host-side logic of KV-group sharding on CPU: world_size-2
torch.distributed (gloo) processes run the same partial exchange the engine's
allgather hook performs on GPUs (paper_2402_04617_b200/shard.py), then the
fixed group-order sums and the (rel desc, id asc) top-k are checked against
the unsharded computation and the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2402_04617_b200.shard import merge_columns, shard_range


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
        from paper_2402_04617_b200.shard import exchange

        G, U, k = 8, 500, 16
        rng = np.random.default_rng(0)  # same inputs on every rank
        q = rng.standard_normal((64, 32, 32)).astype(np.float32)
        reprk = rng.standard_normal((U, G, 4, 32)).astype(np.float32)
        g0, gc = shard_range(G, rank, world)
        buf = torch.from_numpy(group_partials(q, reprk, range(g0, g0 + gc)))
        # the engine leaves the other shards' columns uninitialised: poison them
        mask = torch.ones(G, dtype=torch.bool)
        mask[g0:g0 + gc] = False
        buf[:, mask] = float("nan")
        exchange(buf, g0, gc)
        rel = buf.numpy().sum(axis=1)  # fixed group order 0..G-1, like k_topk
        result_q.put((rank, rel.tobytes(), topk_ids(rel, k)))
    finally:
        dist.destroy_process_group()


def test_shard_range():
    assert shard_range(8, 0, 2) == (0, 4) and shard_range(8, 1, 2) == (4, 4)
    assert [shard_range(8, r, 8) for r in range(8)] == [(r, 1) for r in range(8)]
    with pytest.raises(ValueError):
        shard_range(8, 0, 3)


def test_merge_columns_order():
    g = torch.arange(2 * 3 * 4, dtype=torch.float64).reshape(2, 3, 4)  # [world][rows][gc]
    buf = torch.zeros(3, 8, dtype=torch.float64)
    merge_columns(buf, g, 4)
    assert torch.equal(buf[:, :4], g[0]) and torch.equal(buf[:, 4:], g[1])


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
    full = group_partials(q, reprk, range(G)).sum(axis=1)
    assert np.frombuffer(res[0][1], np.float64).tobytes() == full.tobytes()
    assert res[0][2] == topk_ids(full, k)
    # and the oracle's head-by-head relevance (memory.hpp:217-234) picks the same units
    from oracle import oracle as O

    orel = O.relevance_all(q, reprk.transpose(0, 2, 1, 3))
    assert np.allclose(orel, full, rtol=1e-12, atol=1e-9)
    assert sorted(O.argsort_topk(orel, k)) == res[0][2]
