"""Planted-span recall (workload.hpp:35-127, SURVEY §8f / C3 semantics) and a
multi-layer stream, on the CUDA path against the oracle.

The planted stream repeats one token id over a 64-token span deep in the
evicted region and again on the final decode probes (q == k in the
reference adapter), so the lookup at the probes must retrieve the units that
hold the span. The GPU engine must pick the same units as the oracle at
every step, and the probe lookups must contain the expected units.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.parity_util import bf16_round, rel_err

pytestmark = pytest.mark.gpu


def test_planted_recall_bf16_d128():
    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine

    cfg_kw = dict(chunk_size=512, unit_size=128, n_repr=4, local_size=2048, init_size=128, n_lookup=8,
                  hot_capacity=16)
    n, H, d, probe = 12288, 4, 128, 4
    shape = O.ModelShape.make(n_heads=H, head_dim=d)
    plant = O.gen_planted(3, n, 64, O.EngineConfig.make(**cfg_kw), probe_len=probe, align=True)
    q, k, v = (bf16_round(x) for x in O.adapter_batch(3, shape, plant["token_ids"]))
    sched = O.encode_schedule(n, 512, probe)
    oeng = O.OracleEngine(O.EngineConfig.make(**cfg_kw), shape, n_threads=8)
    geng = StreamEngine(EngineConfig.make(**cfg_kw), ModelShape.make(n_heads=H, head_dim=d), dtype=torch.bfloat16)
    qt, kt, vt = (torch.from_numpy(x).cuda().bfloat16() for x in (q, k, v))
    fed, worst = 0, 0.0
    probe_ids = []
    for si, b in enumerate(sched):
        dec = si >= len(sched) - probe
        r = oeng.step(q[fed:fed + b], k[fed:fed + b], v[fed:fed + b], decode=dec)
        g = geng.step(qt[fed:fed + b], kt[fed:fed + b], vt[fed:fed + b], decode=dec)
        assert g.retrieved_ids == r.retrieved_ids, f"step {si}"
        worst = max(worst, rel_err(g.out.float().cpu().numpy(), r.out))
        if dec:
            probe_ids.append(g.retrieved_ids)
        fed += b
    assert worst <= 2e-2
    for ids in probe_ids:
        assert set(plant["expected_units"]) <= set(ids), (plant["expected_units"], ids)


def test_two_layers_fp32():
    """A reference step is one call per layer (engine.hpp:242): two layers with
    different inputs advance independently and each matches the oracle."""
    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine

    cfg_kw = dict(chunk_size=128, unit_size=128, n_repr=4, local_size=512, init_size=64, n_lookup=4,
                  hot_capacity=32)
    n, H, Hkv, d = 2048, 4, 2, 64
    rng = np.random.default_rng(9)
    data = [tuple((rng.standard_normal((n, h, d)) * s).astype(np.float32) for h, s in ((H, 0.3), (Hkv, 0.3), (Hkv, 1)))
            for _ in range(2)]
    oshape = O.ModelShape.make(n_heads=H, n_kv_heads=Hkv, head_dim=d, n_layers=2)
    oeng = O.OracleEngine(O.EngineConfig.make(**cfg_kw), oshape, n_threads=4)
    geng = StreamEngine(EngineConfig.make(**cfg_kw), ModelShape.make(n_heads=H, n_kv_heads=Hkv, head_dim=d,
                                                                     n_layers=2), dtype=torch.float32)
    dev = [tuple(torch.from_numpy(x).cuda() for x in layer) for layer in data]
    for off in range(0, n, 128):
        for layer in range(2):
            q, k, v = data[layer]
            r = oeng.step(q[off:off + 128], k[off:off + 128], v[off:off + 128], layer=layer)
            qt, kt, vt = dev[layer]
            g = geng.step(qt[off:off + 128].contiguous(), kt[off:off + 128].contiguous(),
                          vt[off:off + 128].contiguous(), layer=layer)
            assert g.retrieved_ids == r.retrieved_ids, (off, layer)
            assert rel_err(g.out.cpu().numpy(), r.out) <= 1e-5
    for layer in range(2):
        om, gm = oeng.metrics(layer), geng.metrics(layer)
        for key in ("units", "hits", "misses", "evictions", "requested"):
            assert om[key] == gm[key], (layer, key)
