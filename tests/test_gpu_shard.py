"""KV-group sharding on the CUDA path, exercised on ONE GPU:
S shard engines (each owning n_kv/S KV groups and their query heads) are
driven by S host threads and exchange their fp64 partials through a
host-synchronised hook (ThreadExchange) — the same infllm_allgather_fn
contract the library's own NCCL exchange (infllm_engine_set_comm) fulfils
across GPUs (tests/test_nccl_shard.py). The sharded stream must select
bit-identical units and, without split-KV attention, reproduce the unsharded
outputs exactly (attention per head does not depend on the shard count); with
the automatic split-KV of a shard (few CTAs per GPU) the outputs agree within
the bf16 rounding of the split merge.
"""
import threading

import numpy as np
import pytest
import torch

from tests.parity_util import gaussian_inputs

pytestmark = pytest.mark.gpu


def _run_sharded(cfg_kw, H, Hkv, d, q, k, v, shards, dtype, chunk, options=None):
    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine
    from paper_2402_04617_b200.shard import ThreadExchange, shard_range

    shape = ModelShape.make(n_heads=H, n_kv_heads=Hkv, head_dim=d)
    rep = H // Hkv
    ex = ThreadExchange(shards)
    engines, outs, ids, errs = [], [None] * shards, [None] * shards, []
    for r in range(shards):
        g0, gc = shard_range(Hkv, r, shards)
        e = StreamEngine(EngineConfig.make(**cfg_kw), shape, dtype=dtype, kv_group_begin=g0, kv_group_count=gc)
        e.set_allgather(ex.hook())
        for key, val in (options or {}).items():
            e.set_option(key, val)
        engines.append(e)

    def drive(r):
        try:
            g0, gc = shard_range(Hkv, r, shards)
            e = engines[r]
            qs = q[:, g0 * rep:(g0 + gc) * rep].contiguous()
            ks, vs = k[:, g0:g0 + gc].contiguous(), v[:, g0:g0 + gc].contiguous()
            o, idl = [], []
            with torch.cuda.stream(torch.cuda.Stream()):
                for off in range(0, q.shape[0], chunk):
                    res = e.step(qs[off:off + chunk], ks[off:off + chunk], vs[off:off + chunk])
                    o.append(res.out.clone())
                    idl.append(res.retrieved_ids)
                torch.cuda.current_stream().synchronize()
            outs[r], ids[r] = torch.cat(o, 0), idl
        except Exception as exc:  # surfaced in the main thread
            errs.append(exc)
            ex.barrier.abort()

    th = [threading.Thread(target=drive, args=(r,)) for r in range(shards)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, (errs, ex.errors)
    return engines, torch.cat(outs, 1), ids, ex


@pytest.mark.parametrize("dtype,d,shards", [(torch.float32, 64, 2), (torch.bfloat16, 128, 2),
                                            (torch.bfloat16, 128, 4)])
def test_sharded_equals_unsharded(dtype, d, shards):
    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine

    cfg = dict(chunk_size=256, unit_size=128, n_repr=4, local_size=512, init_size=128, n_lookup=4, hot_capacity=6)
    H, Hkv, n, chunk = 16, 4, 3072, 256
    q, k, v = gaussian_inputs(17, n, H, Hkv, d, scale=0.3, bf16=dtype == torch.bfloat16)
    qt, kt, vt = (torch.from_numpy(x).cuda().to(dtype) for x in (q, k, v))

    full = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(n_heads=H, n_kv_heads=Hkv, head_dim=d),
                        dtype=dtype)
    full.set_option("attn_splits", 1)
    fo, fids = [], []
    for off in range(0, n, chunk):
        r = full.step(qt[off:off + chunk], kt[off:off + chunk], vt[off:off + chunk])
        fo.append(r.out)
        fids.append(r.retrieved_ids)
    fout = torch.cat(fo, 0)

    engines, sout, sids, ex = _run_sharded(cfg, H, Hkv, d, qt, kt, vt, shards, dtype, chunk, {"attn_splits": 1})
    assert ex.calls > 0, "no partial exchange happened"
    assert any(fids), "stream never looked up"
    for r in range(shards):
        assert sids[r] == fids, f"shard {r}: retrieved ids differ"
    assert torch.equal(sout, fout)
    fm = full.metrics()
    for e in engines:
        m = e.metrics()
        for key in ("units", "hot_units", "hits", "misses", "loads", "evictions", "requested"):
            assert m[key] == fm[key], key
        for u in range(fm["units"]):
            assert e.unit_info(u)["repr_abs"] == full.unit_info(u)["repr_abs"]
        assert e.trace() == full.trace()


@pytest.mark.parametrize("shards", [2, 4, 8])
def test_sharded_c2_config(shards):
    """BASELINE configs[2] settings (32 q / 8 kv heads, d 128, chunk 512, k_m 16,
    local 4096, init 128, hot 32), 24 steps (12K tokens, past the first
    evictions), N(0,1) bf16 inputs: every shard count selects the units of
    the unsharded engine at every step, with split-KV attention on the shards."""
    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine

    cfg = dict(chunk_size=512, unit_size=128, n_repr=4, local_size=4096, init_size=128, n_lookup=16,
               hot_capacity=32, decay=0.1)
    H, Hkv, d, n, chunk = 32, 8, 128, 12288, 512
    q, k, v = gaussian_inputs(29, n, H, Hkv, d, scale=1.0, bf16=True)
    qt, kt, vt = (torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (q, k, v))
    full = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(n_heads=H, n_kv_heads=Hkv, head_dim=d),
                        dtype=torch.bfloat16)
    fo, fids = [], []
    for off in range(0, n, chunk):
        r = full.step(qt[off:off + chunk], kt[off:off + chunk], vt[off:off + chunk])
        fo.append(r.out)
        fids.append(r.retrieved_ids)
    fout = torch.cat(fo, 0).float()
    engines, sout, sids, ex = _run_sharded(cfg, H, Hkv, d, qt, kt, vt, shards, torch.bfloat16, chunk)
    assert ex.calls > 0 and sum(bool(x) for x in fids) >= 12
    for r in range(shards):
        assert sids[r] == fids, f"shard {r}: retrieved ids differ"
    err = (sout.float() - fout).abs().max().item() / fout.abs().max().item()
    assert err <= 1e-2, err
    for e in engines:
        assert e.trace() == full.trace()
        assert e.metrics()["hits"] == full.metrics()["hits"]
