"""K4 decode attention (l_x = 1, split-KV on CUDA cores) and batched decode.

decode_step (engine.hpp:100-103) runs the full step with a single query row:
lookup of that token, attention over [initial | retrieved units | local |
itself], one evicted token per step once the window is full, a completed unit
every 128 steps, LRU. Bars: ids, representatives, counters and trace exact vs
the oracle; outputs within 2e-2 (bf16 inputs, oracle on the rounded values).
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.parity_util import compare_state, gaussian_inputs, rel_err, run_pair

pytestmark = pytest.mark.gpu

CFG = dict(chunk_size=256, unit_size=128, n_repr=4, local_size=1024, init_size=128, n_lookup=8, hot_capacity=12)


def _check(oeng, geng, recs, tol=2e-2):
    worst = 0.0
    for r in recs:
        assert r["o_ids"] == r["g_ids"], f"step {r['step']}: {r['o_ids']} vs {r['g_ids']}"
        worst = max(worst, rel_err(r["g_out"], r["o_out"]))
    assert worst <= tol, worst
    diffs, repr_bad = compare_state(oeng, geng)
    assert not diffs, diffs
    assert not repr_bad
    assert oeng.trace() == geng.trace()
    return worst


@pytest.mark.parametrize("slots", [0, 16])
def test_decode_kernel_vs_oracle(slots):
    """300 decode steps after a 4K prefill: units complete during decode (every
    128 evictions), retrieved units change every step; optionally through the
    host tier."""
    n_pre, n_dec = 4096, 300
    n = n_pre + n_dec
    q, k, v = gaussian_inputs(51, n, 8, 2, 128, scale=0.3, bf16=True)
    sched = O.encode_schedule(n_pre, 256, 0) + [1] * n_dec
    opts = {"host_tier_slots": slots} if slots else {}
    oeng, geng, recs = run_pair(CFG, 8, 2, 128, q, k, v, sched, decode_tail=n_dec, dtype=torch.bfloat16,
                                options=opts)
    _check(oeng, geng, recs)
    assert oeng.metrics()["units"] > (n_pre - 128 - 1024) // 128  # units were created during decode


def test_decode_kernel_matches_tc_path():
    """K4 vs the tcgen05 kernel on the same decode steps (C2 head shape)."""
    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine

    cfg = dict(chunk_size=512, unit_size=128, n_repr=4, local_size=2048, init_size=128, n_lookup=16, hot_capacity=32)
    n_pre, n_dec = 8192, 64
    q, k, v = gaussian_inputs(52, n_pre + n_dec, 32, 8, 128, scale=0.3, bf16=True)
    qt, kt, vt = [torch.from_numpy(x).cuda().bfloat16() for x in (q, k, v)]
    outs = []
    for dec in (1, 0):
        eng = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(n_heads=32, n_kv_heads=8, head_dim=128),
                           dtype=torch.bfloat16)
        eng.set_option("decode_kernel", dec)
        eng.encode_stream(qt[:n_pre], kt[:n_pre], vt[:n_pre])
        o = [eng.decode_step(qt[i:i + 1], kt[i:i + 1], vt[i:i + 1]).float().cpu() for i in range(n_pre, n_pre + n_dec)]
        outs.append((torch.cat(o).numpy(), eng.metrics(), eng.trace()))
    assert rel_err(outs[0][0], outs[1][0]) < 2e-2
    assert outs[0][1] == outs[1][1]
    assert outs[0][2] == outs[1][2]


@pytest.mark.parametrize("n_pre", [8192, 270336])
def test_decode_chain_matches_sequential_order(n_pre):
    """The decode chain (lookup first with the query sums formed from q, the
    front as its programmatic dependent, K4 behind both) against the
    front -> lookup -> K4 order: the arithmetic is the same, so outputs are
    bitwise equal; ids, counters and trace identical. C2 head shape, units
    completing during the decode (every 128 steps). n_pre = 270336: > 2048
    units, the streaming scan + merge-block lookup with the front between."""
    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine

    cfg = dict(chunk_size=512, unit_size=128, n_repr=4, local_size=2048, init_size=128, n_lookup=16, hot_capacity=32)
    n_dec = 200
    g = torch.Generator(device="cuda")
    g.manual_seed(54)
    qt = (torch.randn((n_pre + n_dec, 32, 128), generator=g, device="cuda") * 0.5).bfloat16()
    kt = (torch.randn((n_pre + n_dec, 8, 128), generator=g, device="cuda") * 0.5).bfloat16()
    vt = torch.randn((n_pre + n_dec, 8, 128), generator=g, device="cuda").bfloat16()
    runs = []
    for mode in (1, 0):
        eng = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(n_heads=32, n_kv_heads=8, head_dim=128),
                           dtype=torch.bfloat16)
        eng.set_option("decode_chain", mode)
        eng.reserve(n_pre + n_dec)
        eng.encode_stream(qt[:n_pre], kt[:n_pre], vt[:n_pre])
        o = [eng.decode_step(qt[i:i + 1], kt[i:i + 1], vt[i:i + 1]).clone() for i in range(n_pre, n_pre + n_dec)]
        runs.append((torch.cat(o), eng.metrics(), eng.trace()))
    assert torch.equal(runs[0][0], runs[1][0])
    assert runs[0][1] == runs[1][1]
    assert runs[0][2] == runs[1][2]


@pytest.mark.parametrize("batch", [1, 3])
def test_decode_merge_kernel_matches_last_split_merge(batch):
    """K4's split merge as its own launch (decode_merge_kernel = 1) against the
    merge in each group's last split: same arithmetic in the same order, so
    outputs are bitwise equal and masses (hence counters and trace) identical."""
    from paper_2402_04617_b200 import decode_batch

    cfg = dict(chunk_size=512, unit_size=128, n_repr=4, local_size=2048, init_size=128, n_lookup=16, hot_capacity=32)
    runs = []
    for mk in (1, 0):
        engs, data = _prefilled(cfg, 6144, list(range(60, 60 + batch)), H=32, Hkv=8)
        for e in engs:
            e.set_option("decode_merge_kernel", mk)
        outs = []
        for t in range(150):
            if batch == 1:
                qt, kt, vt = data[0]
                outs.append(engs[0].decode_step(qt[6144 + t:6145 + t], kt[6144 + t:6145 + t], vt[6144 + t:6145 + t]).clone())
            else:
                q = torch.stack([d[0][6144 + t] for d in data]).contiguous()
                k = torch.stack([d[1][6144 + t] for d in data]).contiguous()
                v = torch.stack([d[2][6144 + t] for d in data]).contiguous()
                outs.append(decode_batch(engs, q, k, v).clone())
        runs.append((torch.stack(outs), [e.metrics() for e in engs], [e.trace() for e in engs]))
    assert torch.equal(runs[0][0], runs[1][0])
    assert runs[0][1] == runs[1][1]
    assert runs[0][2] == runs[1][2]


def test_decode_from_empty_stream():
    """Decode-only stream from token 0 (no units for the first steps, init
    pinning while decoding): the window grows from one key."""
    cfg = dict(chunk_size=64, unit_size=128, n_repr=4, local_size=256, init_size=128, n_lookup=4, hot_capacity=8)
    n = 700
    q, k, v = gaussian_inputs(53, n, 8, 2, 128, scale=0.3, bf16=True)
    oeng, geng, recs = run_pair(cfg, 8, 2, 128, q, k, v, [1] * n, decode_tail=n, dtype=torch.bfloat16)
    _check(oeng, geng, recs)


def _prefilled(cfg, n_pre, seeds, H=8, Hkv=2):
    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine

    engs, data = [], []
    for sd in seeds:
        q, k, v = gaussian_inputs(sd, n_pre + 400, H, Hkv, 128, scale=0.3, bf16=True)
        e = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(n_heads=H, n_kv_heads=Hkv, head_dim=128),
                         dtype=torch.bfloat16)
        qt, kt, vt = [torch.from_numpy(x).cuda().bfloat16() for x in (q, k, v)]
        if n_pre:
            e.encode_stream(qt[:n_pre], kt[:n_pre], vt[:n_pre])
        engs.append(e)
        data.append((qt, kt, vt))
    return engs, data


@pytest.mark.parametrize("n_pre", [0, 3000])
def test_decode_batch_matches_per_sequence(n_pre):
    """decode_batch over 5 sequences (different contents, so different retrieved
    units; n_pre = 0: sequences start empty and pass through init pinning and
    their first units while batched) == decode_step per sequence: ids, counters,
    trace exact, outputs within bf16 rounding of the split-KV merge order."""
    from paper_2402_04617_b200 import decode_batch

    seeds = [61, 62, 63, 64, 65]
    steps = 300 if n_pre else 400
    a, da = _prefilled(CFG, n_pre, seeds)
    b, db = _prefilled(CFG, n_pre, seeds)
    worst = 0.0
    for t in range(n_pre, n_pre + steps):
        q = torch.stack([d[0][t] for d in db])
        k = torch.stack([d[1][t] for d in db])
        v = torch.stack([d[2][t] for d in db])
        got = decode_batch(b, q, k, v)
        for i, e in enumerate(a):
            ref = e.decode_step(da[i][0][t:t + 1], da[i][1][t:t + 1], da[i][2][t:t + 1])
            assert e.retrieved_ids() == b[i].retrieved_ids(), (t, i)
            worst = max(worst, rel_err(got[i].float().cpu().numpy(), ref[0].float().cpu().numpy()))
    assert worst < 2e-2, worst
    for ea, eb in zip(a, b):
        assert ea.metrics() == eb.metrics()
        assert ea.trace() == eb.trace()
        m = ea.metrics()
        for u in range(m["units"]):
            assert ea.unit_info(u) == eb.unit_info(u)


def test_decode_batch_of_one():
    """decode_batch over one sequence takes the single-sequence chain; calls of
    one and of two sequences alternate over the same engines (the LRU stream
    of a batched call carried into the next single call and back) and match
    decode_step per sequence: ids, counters, trace exact."""
    from paper_2402_04617_b200 import decode_batch

    seeds = [71, 72]
    a, da = _prefilled(CFG, 2500, seeds)
    b, db = _prefilled(CFG, 2500, seeds)
    worst = 0.0
    for t in range(2500, 2700):
        sub = [0] if t % 3 == 0 else [1] if t % 3 == 1 else [0, 1]
        q = torch.stack([db[i][0][t] for i in sub])
        k = torch.stack([db[i][1][t] for i in sub])
        v = torch.stack([db[i][2][t] for i in sub])
        got = decode_batch([b[i] for i in sub], q, k, v)
        for j, i in enumerate(sub):
            ref = a[i].decode_step(da[i][0][t:t + 1], da[i][1][t:t + 1], da[i][2][t:t + 1])
            assert a[i].retrieved_ids() == b[i].retrieved_ids(), (t, i)
            worst = max(worst, rel_err(got[j].float().cpu().numpy(), ref[0].float().cpu().numpy()))
    assert worst < 2e-2, worst
    for ea, eb in zip(a, b):
        assert ea.metrics() == eb.metrics()
        assert ea.trace() == eb.trace()


def test_decode_batch_vs_oracle():
    """One batched sequence set against the CPU oracle directly."""
    from paper_2402_04617_b200 import decode_batch

    n_pre, steps, seeds = 2048, 160, [71, 72]
    engs, data = _prefilled(CFG, n_pre, seeds)
    oengs = []
    for sd in seeds:
        q, k, v = gaussian_inputs(sd, n_pre + 400, 8, 2, 128, scale=0.3, bf16=True)
        oe = O.OracleEngine(O.EngineConfig.make(**CFG), O.ModelShape.make(n_heads=8, n_kv_heads=2, head_dim=128),
                            n_threads=8)
        for off in range(0, n_pre, 256):
            oe.step(q[off:off + 256], k[off:off + 256], v[off:off + 256])
        oengs.append((oe, q, k, v))
    worst = 0.0
    for t in range(n_pre, n_pre + steps):
        q = torch.stack([d[0][t] for d in data])
        k = torch.stack([d[1][t] for d in data])
        v = torch.stack([d[2][t] for d in data])
        got = decode_batch(engs, q, k, v).float().cpu().numpy()
        for i, (oe, oq, ok, ov) in enumerate(oengs):
            r = oe.step(oq[t:t + 1], ok[t:t + 1], ov[t:t + 1], decode=True)
            assert r.retrieved_ids == engs[i].retrieved_ids()
            worst = max(worst, rel_err(got[i:i + 1], r.out))
    assert worst < 2e-2, worst
    for i, (oe, *_) in enumerate(oengs):
        diffs, repr_bad = compare_state(oe, engs[i])
        assert not diffs and not repr_bad


@pytest.mark.parametrize("H,Hkv", [(8, 8), (4, 1), (16, 2), (24, 8)])
def test_decode_head_layouts(H, Hkv):
    """K4 + decode front over GQA ratios 1, 3, 4, 8 (MHA-like to 8 query heads
    per KV group): prefill, then decode steps that cross a unit boundary."""
    cfg = dict(chunk_size=256, unit_size=128, n_repr=4, local_size=512, init_size=128, n_lookup=4, hot_capacity=6)
    n_pre, n_dec = 1536, 140
    q, k, v = gaussian_inputs(80 + H, n_pre + n_dec, H, Hkv, 128, scale=0.3, bf16=True)
    sched = O.encode_schedule(n_pre, 256, 0) + [1] * n_dec
    oeng, geng, recs = run_pair(cfg, H, Hkv, 128, q, k, v, sched, decode_tail=n_dec, dtype=torch.bfloat16)
    _check(oeng, geng, recs)


def test_decode_batch_mixed_lengths():
    """decode_batch over sequences at different stream positions (empty, inside
    the first window, past several units) in the same batch."""
    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, decode_batch

    seeds, pres = [91, 92, 93], [0, 700, 3000]
    a, b, data = [], [], []
    for sd, n_pre in zip(seeds, pres):
        q, k, v = gaussian_inputs(sd, n_pre + 200, 8, 2, 128, scale=0.3, bf16=True)
        qt, kt, vt = [torch.from_numpy(x).cuda().bfloat16() for x in (q, k, v)]
        for lst in (a, b):
            e = StreamEngine(EngineConfig.make(**CFG), ModelShape.make(n_heads=8, n_kv_heads=2, head_dim=128),
                             dtype=torch.bfloat16)
            if n_pre:
                e.encode_stream(qt[:n_pre], kt[:n_pre], vt[:n_pre])
            lst.append(e)
        data.append((qt, kt, vt, n_pre))
    worst = 0.0
    for t in range(200):
        q = torch.stack([d[0][d[3] + t] for d in data])
        k = torch.stack([d[1][d[3] + t] for d in data])
        v = torch.stack([d[2][d[3] + t] for d in data])
        got = decode_batch(b, q, k, v)
        for i, (qt, kt, vt, n_pre) in enumerate(data):
            s = n_pre + t
            ref = a[i].decode_step(qt[s:s + 1], kt[s:s + 1], vt[s:s + 1])
            assert a[i].retrieved_ids() == b[i].retrieved_ids(), (t, i)
            worst = max(worst, rel_err(got[i].float().cpu().numpy(), ref[0].float().cpu().numpy()))
    assert worst < 2e-2
    for ea, eb in zip(a, b):
        assert ea.metrics() == eb.metrics() and ea.trace() == eb.trace()


def test_graph_recaptured_after_buffers_move():
    """encode_stream replays a captured graph when the stream state repeats
    (after reset). Decode steps past the reserved trace grow (move) buffers the
    graph baked in; the replay must not write into the freed memory: the
    second prefill matches the first bit for bit (outputs, trace), and a
    batched decode over engines that went through this runs clean."""
    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, decode_batch

    cfg = dict(chunk_size=512, unit_size=128, n_repr=4, local_size=2048, init_size=128, n_lookup=16, hot_capacity=32)
    n_pre, n_dec = 8192, 200
    q, k, v = gaussian_inputs(53, n_pre + n_dec, 32, 8, 128, scale=0.3, bf16=True)
    qt, kt, vt = [torch.from_numpy(x).cuda().bfloat16() for x in (q, k, v)]
    engs = [StreamEngine(EngineConfig.make(**cfg), ModelShape.make(n_heads=32, n_kv_heads=8, head_dim=128),
                         dtype=torch.bfloat16) for _ in range(3)]
    try:
        for e in engs:
            e.reserve(n_pre + 1)  # the decode tail grows the trace / unit pool past this
        e0 = engs[0]
        ob0 = torch.empty((n_pre, 32, 128), device="cuda", dtype=torch.bfloat16)  # same pointers: graph cache hit
        out1 = e0.encode_stream(qt[:n_pre], kt[:n_pre], vt[:n_pre], out=ob0).clone()
        tr1 = e0.trace()
        for t in range(n_pre, n_pre + n_dec):
            e0.decode_step(qt[t:t + 1], kt[t:t + 1], vt[t:t + 1])
        torch.cuda.synchronize()
        e0.reset()
        out2 = e0.encode_stream(qt[:n_pre], kt[:n_pre], vt[:n_pre], out=ob0).clone()
        torch.cuda.synchronize()
        assert torch.equal(out1, out2)
        assert e0.trace() == tr1
        for e in engs[1:]:
            e.encode_stream(qt[:n_pre], kt[:n_pre], vt[:n_pre])
        ob = torch.empty((3, 32, 128), device="cuda", dtype=torch.bfloat16)
        for t in range(n_pre, n_pre + 16):
            decode_batch(engs, qt[t].expand(3, 32, 128).contiguous(), kt[t].expand(3, 8, 128).contiguous(),
                         vt[t].expand(3, 8, 128).contiguous(), out=ob)
        torch.cuda.synchronize()
        assert torch.equal(ob[0], ob[1]) and torch.equal(ob[1], ob[2])
    finally:
        for e in engs:
            e.close()
