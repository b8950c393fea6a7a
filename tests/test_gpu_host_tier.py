"""Host tier (north star: pinned-host unit store + GPU-resident unit cache
filled over PCIe on a side stream).

The reference's hot/cold tiers are bookkeeping only (memory.hpp:165-168,
SPEC.md:292): outputs never depend on where unit pages live. So the bar is
exact: with the host tier on, every output must be bitwise equal to the
HBM-resident engine's, ids / representatives / counters / trace identical,
and (through run_pair) equal to the oracle within the stated tolerances.
Small slot counts (2 k_m) force the cache to evict and re-load pages.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.parity_util import compare_state, gaussian_inputs, rel_err, run_pair

pytestmark = pytest.mark.gpu


def _engine(cfg, H, Hkv, d, dtype, slots, **opts):
    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine

    eng = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(n_heads=H, n_kv_heads=Hkv, head_dim=d), dtype=dtype)
    if slots:
        eng.set_option("host_tier_slots", slots)
    for key, val in opts.items():
        eng.set_option(key, val)
    return eng


@pytest.mark.parametrize("slots", [16, 64])
def test_tier_bitwise_equal_bf16_tc(slots):
    """tcgen05 attention reading cache slots == reading HBM unit pages, step by step."""
    cfg = dict(chunk_size=256, unit_size=128, n_repr=4, local_size=1024, init_size=128, n_lookup=8, hot_capacity=12)
    n = 8192
    q, k, v = gaussian_inputs(41, n, 8, 2, 128, scale=0.3, bf16=True)
    qt, kt, vt = [torch.from_numpy(x).cuda().bfloat16() for x in (q, k, v)]
    base = _engine(cfg, 8, 2, 128, torch.bfloat16, 0)
    tier = _engine(cfg, 8, 2, 128, torch.bfloat16, slots)
    retrieved = 0
    for off in range(0, n, 256):
        a = base.step(qt[off:off + 256], kt[off:off + 256], vt[off:off + 256])
        b = tier.step(qt[off:off + 256], kt[off:off + 256], vt[off:off + 256])
        assert a.retrieved_ids == b.retrieved_ids
        assert torch.equal(a.out, b.out), f"chunk at {off}"
        retrieved += len(a.retrieved_ids)
    assert base.metrics() == tier.metrics()
    assert base.trace() == tier.trace()
    st = tier.tier_stats()
    assert st["slots"] == slots
    assert st["loads"] + st["cache_hits"] == retrieved
    assert st["h2d_bytes"] == st["loads"] * 2 * 2 * 128 * 128 * 2  # K + V^T pages, 2 groups, bf16
    if slots == 16:
        assert st["loads"] > 16  # the cache had to evict and reload


def test_tier_oracle_fp32_ragged():
    """CUDA-core path (fp32, units not aligned to chunks, decode tail: units
    complete across steps and partial units are flushed) through the host
    tier against the oracle at 1e-5."""
    cfg = dict(chunk_size=100, unit_size=32, n_repr=3, local_size=256, init_size=40, n_lookup=5, hot_capacity=6)
    n = 3000
    q, k, v = gaussian_inputs(3, n, 8, 2, 32, scale=0.4)
    sched = O.encode_schedule(n, 100, 20)
    oeng, geng, recs = run_pair(cfg, 8, 2, 32, q, k, v, sched, decode_tail=20, finish=True,
                                options={"host_tier_slots": 10})
    worst = 0.0
    for r in recs:
        assert r["o_ids"] == r["g_ids"], f"step {r['step']}"
        worst = max(worst, rel_err(r["g_out"], r["o_out"]))
    assert worst <= 1e-5
    diffs, repr_bad = compare_state(oeng, geng)
    assert not diffs and not repr_bad
    assert oeng.trace() == geng.trace()
    assert geng.tier_stats()["loads"] > 0


def test_tier_absolute_positions():
    """Absolute position mode keeps rotated unit keys too (K_rot pages travel with K and V)."""
    cfg = dict(chunk_size=64, unit_size=32, n_repr=2, local_size=128, init_size=16, n_lookup=3, hot_capacity=4,
               position_mode=1)
    n = 1500
    q, k, v = gaussian_inputs(9, n, 4, 2, 32, scale=0.4)
    sched = O.encode_schedule(n, 64, 10)
    oeng, geng, recs = run_pair(cfg, 4, 2, 32, q, k, v, sched, decode_tail=10, options={"host_tier_slots": 6})
    for r in recs:
        assert r["o_ids"] == r["g_ids"]
        assert rel_err(r["g_out"], r["o_out"]) <= 1e-5
    assert geng.tier_stats()["loads"] > 0


def test_tier_graph_replay_and_host_stream():
    """Graph-captured streams through the host tier replay bit-exactly from a
    reset (the slot tables are part of the reset state), also with host q/k/v."""
    cfg = dict(chunk_size=256, unit_size=128, n_repr=4, local_size=1024, init_size=128, n_lookup=8, hot_capacity=12)
    n = 6000
    q, k, v = gaussian_inputs(32, n, 8, 2, 128, scale=0.3, bf16=True)
    qt, kt, vt = [torch.from_numpy(x).cuda().bfloat16() for x in (q, k, v)]
    ref = _engine(cfg, 8, 2, 128, torch.bfloat16, 0).feed(qt, kt, vt)
    eng = _engine(cfg, 8, 2, 128, torch.bfloat16, 16)
    eng.reserve(n)
    stats = None
    for rep in range(3):
        eng.reset()
        got = eng.encode_stream(qt, kt, vt)
        assert torch.equal(got, ref), f"replay {rep}"
        st = eng.tier_stats()
        assert stats is None or st == stats
        stats = st
    hq, hk, hv = [x.cpu().pin_memory() for x in (qt, kt, vt)]
    hout = torch.empty((n, 8, 128), dtype=torch.bfloat16).pin_memory()
    eng.reset()
    eng.encode_stream_host(hq, hk, hv, hout)
    torch.cuda.synchronize()
    assert torch.equal(hout, ref.cpu())


def test_tier_option_validation():
    from paper_2402_04617_b200 import InfLLMError

    cfg = dict(chunk_size=256, unit_size=128, n_repr=4, local_size=1024, init_size=128, n_lookup=8, hot_capacity=12)
    eng = _engine(cfg, 8, 2, 128, torch.bfloat16, 0)
    with pytest.raises(InfLLMError):
        eng.set_option("host_tier_slots", 15)  # < 2 k_m
    eng.reserve(4096)
    with pytest.raises(InfLLMError):
        eng.set_option("host_tier_slots", 32)  # pools already sized for HBM pages
