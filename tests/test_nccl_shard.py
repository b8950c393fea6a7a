"""KV-group sharding over the library's own NCCL communicator
(infllm_engine_set_comm): one process per GPU, the C-1 partial exchange and
the C-2 output all-gather issued by the library with ncclAllGather on the
engine's streams inside the graph-captured stream. Needs >= 2 GPUs (NCCL
does not put two ranks on one device); skipped otherwise. Checks: every
rank's retrieved units, representatives and trace equal the unsharded
engine's, the gathered outputs (all heads) match it within bf16 rounding."""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CFG = dict(chunk_size=512, unit_size=128, n_repr=4, local_size=2048, init_size=128, n_lookup=8, hot_capacity=16)


def _inputs(n):
    g = torch.Generator(device="cpu")
    g.manual_seed(5)
    q = torch.randn((n, 32, 128), generator=g).bfloat16()
    k = torch.randn((n, 8, 128), generator=g).bfloat16()
    v = torch.randn((n, 8, 128), generator=g).bfloat16()
    return q, k, v


def _worker(rank, world, port, n, q_):
    import torch.distributed as dist

    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine
    from paper_2402_04617_b200.shard import shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q, k, v = _inputs(n)
        g0, gc = shard_range(8, rank, world)
        rep = 4
        e = StreamEngine(EngineConfig.make(**CFG), ModelShape.make(n_heads=32, n_kv_heads=8, head_dim=128),
                         dtype=torch.bfloat16, device=rank, kv_group_begin=g0, kv_group_count=gc)
        e.set_comm(rank, world)
        e.set_option("gather_output", 1)
        dev = torch.device("cuda", rank)
        qs = q[:, g0 * rep:(g0 + gc) * rep].contiguous().to(dev)
        ks, vs = k[:, g0:g0 + gc].contiguous().to(dev), v[:, g0:g0 + gc].contiguous().to(dev)
        out = torch.empty((n, 32, 128), dtype=torch.bfloat16, device=dev)  # all heads (gather_output)
        e.reserve(n)
        e.encode_stream(qs, ks, vs, out=out)
        torch.cuda.synchronize(dev)
        q_.put((rank, out.float().cpu(), e.trace(), [e.unit_info(u)["repr_abs"] for u in range(e.metrics()["units"])]))
    finally:
        dist.destroy_process_group()


def test_nccl_sharded_stream_matches_unsharded():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (NCCL ranks on distinct devices)")
    import torch.multiprocessing as mp

    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine

    world, n = 2, 8192
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q_)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q_.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    q, k, v = _inputs(n)
    full = StreamEngine(EngineConfig.make(**CFG), ModelShape.make(n_heads=32, n_kv_heads=8, head_dim=128),
                        dtype=torch.bfloat16)
    fo = full.encode_stream(q.cuda(), k.cuda(), v.cuda()).float().cpu()
    reprs = [full.unit_info(u)["repr_abs"] for u in range(full.metrics()["units"])]
    for rank, out, trace, rabs in res:
        assert trace == full.trace(), f"rank {rank}: lookup trace differs"
        assert rabs == reprs
        err = (out - fo).abs().max().item() / fo.abs().max().item()
        assert err <= 1e-2, (rank, err)
