"""GPU engine (libinfllm_b200.so through the C-ABI) vs the CPU oracle.

Bars (BASELINE.json north_star): selected unit ids and representative
indices bit-exact; attention outputs within 1e-5 relative (||d||_inf /
||ref||_inf) in fp32 and 2e-2 in bf16 (oracle fed the bf16-rounded inputs).
LRU counters are compared exactly (they can legitimately flip only on
near-equal frequency scores; the cases below have none).
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.parity_util import compare_state, gaussian_inputs, rel_err, run_pair

pytestmark = pytest.mark.gpu

C0 = dict(chunk_size=128, unit_size=128, n_repr=4, local_size=512, init_size=64, n_lookup=4, hot_capacity=32,
          decay=0.1)


def _assert_pair(oeng, geng, recs, tol):
    worst = 0.0
    for r in recs:
        assert r["o_ids"] == r["g_ids"], f"step {r['step']}: ids {r['o_ids']} vs {r['g_ids']}"
        worst = max(worst, rel_err(r["g_out"], r["o_out"]))
    assert worst <= tol, f"max rel err {worst} > {tol}"
    diffs, repr_bad = compare_state(oeng, geng)
    assert not repr_bad, f"repr/unit mismatch in units {repr_bad[:10]}"
    assert not diffs, f"counter mismatch {diffs}"
    assert oeng.trace() == geng.trace()
    return worst


@pytest.mark.parametrize("seed", [0, 1])
def test_c0_adapter_fp32(seed):
    """C0 (configs[0]): 1 head, d 64, reference adapter inputs (q == k)."""
    n = 8192
    shape = O.ModelShape.make(n_heads=1, head_dim=64)
    q, k, v = O.adapter_batch(seed, shape, O.noise_ids(seed, n))
    sched = O.encode_schedule(n, 128, 32)
    oeng, geng, recs = run_pair(C0, 1, 1, 64, q, k, v, sched, decode_tail=32, finish=True)
    _assert_pair(oeng, geng, recs, 1e-5)


def test_c0_gaussian_q_fp32():
    n = 4096
    q, k, v = gaussian_inputs(7, n, 1, 1, 64, scale=0.3)
    sched = O.encode_schedule(n, 128, 16)
    oeng, geng, recs = run_pair(C0, 1, 1, 64, q, k, v, sched, decode_tail=16, finish=True)
    _assert_pair(oeng, geng, recs, 1e-5)


def test_gqa_fp32_ragged():
    """GQA 8/2, ragged chunks, units not aligned to chunks, small hot cache (evictions)."""
    cfg = dict(chunk_size=100, unit_size=32, n_repr=3, local_size=256, init_size=40, n_lookup=5, hot_capacity=6)
    n = 3000
    q, k, v = gaussian_inputs(3, n, 8, 2, 32, scale=0.4)
    sched = O.encode_schedule(n, 100, 20)
    oeng, geng, recs = run_pair(cfg, 8, 2, 32, q, k, v, sched, decode_tail=20, finish=True)
    _assert_pair(oeng, geng, recs, 1e-5)


@pytest.mark.parametrize("scale,bound", [(0.25, 1), (0.25, 0), (1.8, 1)])
def test_bf16_gqa_d128(scale, bound):
    """tcgen05 attention. scale 0.25: every row's score bound |q| |k|max is
    small (fixed-offset fast path); bound=0 forces the online-max path on the
    same data; scale 1.8 pushes the bound past 60 so CTAs fall back by
    themselves (larger scores also grow the bf16 rounding of the rotated
    operands, which is why the scale stops there)."""
    cfg = dict(chunk_size=256, unit_size=128, n_repr=4, local_size=1024, init_size=128, n_lookup=8, hot_capacity=12)
    n = 6144
    q, k, v = gaussian_inputs(11, n, 8, 2, 128, scale=scale, bf16=True)
    sched = O.encode_schedule(n, 256, 8)
    oeng, geng, recs = run_pair(cfg, 8, 2, 128, q, k, v, sched, decode_tail=8, dtype=torch.bfloat16,
                                options={"attn_score_bound": bound})
    _assert_pair(oeng, geng, recs, 2e-2)


@pytest.mark.parametrize("mode", ["decode_only", "none"])
def test_lookup_modes(mode):
    cfg = dict(C0, lookup_mode=mode)
    n = 2048
    q, k, v = gaussian_inputs(5, n, 2, 1, 64, scale=0.3)
    sched = O.encode_schedule(n, 128, 16)
    oeng, geng, recs = run_pair(cfg, 2, 1, 64, q, k, v, sched, decode_tail=16)
    _assert_pair(oeng, geng, recs, 1e-5)


def test_degenerate_vs_dense():
    """oracle-check #1 (cli.cpp:249-271): absolute positions, no eviction."""
    n = 1024
    shape = O.ModelShape.make(n_heads=2, head_dim=32)
    q, k, v = O.adapter_batch(0, shape, O.noise_ids(0, n))
    cfg = dict(C0, local_size=n, position_mode="absolute")
    sched = O.encode_schedule(n, 128, 32)
    oeng, geng, recs = run_pair(cfg, 2, 2, 32, q, k, v, sched, decode_tail=32)
    got = np.concatenate([r["g_out"] for r in recs], 0)
    want = O.dense_attention(q, k, v, 1, n)
    assert np.abs(got - want).max() <= 1e-5


def test_full_retrieval_vs_windowed():
    """oracle-check #2 (cli.cpp:274-299): k_m >= all units, clamped positions."""
    n = 2048
    shape = O.ModelShape.make(n_heads=2, head_dim=32)
    q, k, v = O.adapter_batch(1, shape, O.noise_ids(1, n))
    km = n // 128 + 2
    cfg = dict(C0, n_lookup=km, hot_capacity=km)
    sched = O.encode_schedule(n, 128, 32)
    oeng, geng, recs = run_pair(cfg, 2, 2, 32, q, k, v, sched, decode_tail=32)
    got = np.concatenate([r["g_out"] for r in recs], 0)
    want = O.windowed_attention(q, k, v, sched, 64, 512, 128, 0)
    assert np.abs(got - want).max() <= 1e-5


def test_select_and_lookup_standalone():
    from paper_2402_04617_b200 import lookup, select_representatives

    rng = np.random.default_rng(0)
    sc = rng.standard_normal((50, 128)).astype(np.float32)
    sc[3, :] = 1.0  # all ties -> lowest indices
    sc[4, [5, 9, 77, 100]] = 9.0
    idx = select_representatives(torch.from_numpy(sc).cuda(), 4).cpu().numpy()
    for u in range(50):
        assert idx[u].tolist() == O.select_representatives(sc[u], 4)
    # lookup over an explicit index
    U, G, rk, d, H = 300, 4, 4, 64, 8
    reprk = rng.standard_normal((U, G, rk, d)).astype(np.float32)
    qb = rng.standard_normal((16, H, d)).astype(np.float32)
    qsum = qb.astype(np.float64).reshape(16, G, H // G, d).sum(axis=(0, 2))
    rel, ids = lookup(torch.from_numpy(qsum).cuda(), torch.from_numpy(reprk).cuda(), 10)
    want = O.relevance_all(qb, reprk.transpose(0, 2, 1, 3))
    assert np.allclose(rel.cpu().numpy(), want, rtol=1e-12, atol=1e-9)
    top = sorted(O.argsort_topk(want, 10))
    assert ids.cpu().tolist() == top


def test_tc_vs_simt_c2_shape():
    """tcgen05 attention vs the CUDA-core kernel on the C2 head shape (32q/8kv,
    d128), several steady-state steps with staircase tiles and retrieved units."""
    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine

    cfg = dict(chunk_size=512, unit_size=128, n_repr=4, local_size=1024, init_size=128, n_lookup=8, hot_capacity=16)
    n = 4096
    q, k, v = gaussian_inputs(21, n, 32, 8, 128, scale=0.3, bf16=True)
    outs = []
    for tc in (1, 0):
        eng = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(n_heads=32, n_kv_heads=8, head_dim=128),
                           dtype=torch.bfloat16)
        eng.set_option("tc_attention", tc)
        qt, kt, vt = [torch.from_numpy(x).cuda().bfloat16() for x in (q, k, v)]
        outs.append((eng.feed(qt, kt, vt).float().cpu().numpy(), eng.metrics(), eng.kernel_launches()))
    assert rel_err(outs[0][0], outs[1][0]) < 2e-2
    assert outs[0][1] == outs[1][1]
    # and against the oracle on the last chunks
    ocfg = O.EngineConfig.make(**cfg)
    oeng = O.OracleEngine(ocfg, O.ModelShape.make(n_heads=32, n_kv_heads=8, head_dim=128), n_threads=8)
    got = []
    for off in range(0, n, 512):
        got.append(oeng.step(q[off:off + 512], k[off:off + 512], v[off:off + 512]).out)
    want = np.concatenate(got, 0)
    assert rel_err(outs[0][0], want) < 2e-2


def test_encode_stream_graph_matches_chunks():
    """infllm_encode_stream (graph-captured chunk schedule, replayed) and the
    host-buffer variant reproduce the per-chunk encode_chunk results exactly."""
    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine

    cfg = dict(chunk_size=256, unit_size=128, n_repr=4, local_size=1024, init_size=128, n_lookup=8, hot_capacity=12)
    n = 5000
    q, k, v = gaussian_inputs(31, n, 8, 2, 128, scale=0.3, bf16=True)
    qt, kt, vt = [torch.from_numpy(x).cuda().bfloat16() for x in (q, k, v)]
    shape = ModelShape.make(n_heads=8, n_kv_heads=2, head_dim=128)
    ref_eng = StreamEngine(EngineConfig.make(**cfg), shape, dtype=torch.bfloat16)
    ref = ref_eng.feed(qt, kt, vt)
    eng = StreamEngine(EngineConfig.make(**cfg), shape, dtype=torch.bfloat16)
    for rep in range(3):  # capture, then replays from a reset state
        eng.reset()
        got = eng.encode_stream(qt, kt, vt)
        assert torch.equal(got, ref), f"replay {rep}"
        assert eng.metrics() == ref_eng.metrics()
        assert eng.trace() == ref_eng.trace()
    hq, hk, hv = [x.cpu().pin_memory() for x in (qt, kt, vt)]
    hout = torch.empty((n, 8, 128), dtype=torch.bfloat16).pin_memory()
    eng.reset()
    eng.encode_stream_host(hq, hk, hv, hout)
    torch.cuda.synchronize()
    assert torch.equal(hout, ref.cpu())


@pytest.mark.parametrize("U,k", [(1, 1), (37, 16), (991, 16), (2048, 64), (5000, 32), (9000, 16)])
def test_topk_ties_and_sizes(U, k):
    """Exact top-k (rel desc, id asc) incl. heavy ties, via the standalone lookup
    (radix select path up to 8192 units, warp-selection path beyond)."""
    from paper_2402_04617_b200 import lookup

    rng = np.random.default_rng(U)
    G, rk, d, H = 2, 2, 32, 4
    reprk = rng.integers(-2, 3, size=(U, G, rk, d)).astype(np.float32)  # small ints: many exact ties
    qb = rng.integers(-1, 2, size=(3, H, d)).astype(np.float32)
    qsum = qb.astype(np.float64).reshape(3, G, H // G, d).sum(axis=(0, 2))
    rel, ids = lookup(torch.from_numpy(qsum).cuda(), torch.from_numpy(reprk).cuda(), k)
    want = O.relevance_all(qb, reprk.transpose(0, 2, 1, 3))
    assert np.array_equal(rel.cpu().numpy(), want)
    assert ids.cpu().tolist() == sorted(O.argsort_topk(want, k))


@pytest.mark.parametrize("U,k", [(991, 16), (2049, 16), (4063, 16), (3000, 128), (8159, 16), (20000, 32)])
def test_lookup_bf16_c2_shape(U, k):
    """The register-resident relevance scan (bf16, d 128, r_k 4, 8 KV groups) and
    the multi-block top-k at C2/C3 index sizes: small-integer data makes every
    fp64 sum exact, so rel must equal the oracle's bit for bit."""
    from paper_2402_04617_b200 import lookup

    rng = np.random.default_rng(U + k)
    G, rk, d, H = 8, 4, 128, 32
    reprk = rng.integers(-3, 4, size=(U, G, rk, d)).astype(np.float32)
    qb = rng.integers(-2, 3, size=(4, H, d)).astype(np.float32)
    qsum = qb.astype(np.float64).reshape(4, G, H // G, d).sum(axis=(0, 2))
    rel, ids = lookup(torch.from_numpy(qsum).cuda(), torch.from_numpy(reprk).cuda().bfloat16(), k)
    want = O.relevance_all(qb, reprk.transpose(0, 2, 1, 3))
    assert np.array_equal(rel.cpu().numpy(), want)
    assert ids.cpu().tolist() == sorted(O.argsort_topk(want, k))


@pytest.mark.parametrize("U,k", [(2049, 16), (4063, 16), (9000, 32), (40000, 16)])
def test_lookup_heavy_ties_twice(U, k):
    """The one-launch lookup (block lists + threshold-filtered final selection)
    on integer-valued representatives, so many units tie on relevance: ids
    bit-exact against the oracle's (rel desc, id asc) order, two calls in a row
    (the last-block counter is re-zeroed by the kernel)."""
    from paper_2402_04617_b200 import lookup

    rng = np.random.default_rng(U)
    reprk = rng.integers(-3, 4, size=(U, 8, 4, 128)).astype(np.float32)
    qb = rng.integers(-2, 3, size=(4, 32, 128)).astype(np.float32)
    qsum = qb.astype(np.float64).reshape(4, 8, 4, 128).sum(axis=(0, 2))
    want = O.relevance_all(qb, reprk.transpose(0, 2, 1, 3))
    for _ in range(2):
        rel, ids = lookup(torch.from_numpy(qsum).cuda(), torch.from_numpy(reprk).cuda().bfloat16(), k)
        assert np.array_equal(rel.cpu().numpy(), want)
        assert ids.cpu().tolist() == sorted(O.argsort_topk(want, k)), (U, k)


def test_encode_stream_replay_beyond_2048_units():
    """Graph replay of a stream whose lookups run the multi-block top-k
    (> 2048 units): scratch is sized before capture, so the captured graph
    replays (a graph holding an allocation cannot be relaunched) and repeats
    the first run exactly."""
    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine

    cfg = dict(chunk_size=512, unit_size=128, n_repr=4, local_size=512, init_size=128, n_lookup=8, hot_capacity=16)
    n = 2300 * 128
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    q = (torch.randn((n, 8, 128), generator=g, device="cuda") * 0.3).bfloat16()
    k = (torch.randn((n, 2, 128), generator=g, device="cuda") * 0.3).bfloat16()
    v = torch.randn((n, 2, 128), generator=g, device="cuda").bfloat16()
    eng = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(n_heads=8, n_kv_heads=2, head_dim=128),
                       dtype=torch.bfloat16)
    eng.reserve(n)
    first = eng.encode_stream(q, k, v).clone()
    m1, t1 = eng.metrics(), eng.trace()
    assert m1["units"] > 2048
    eng.reset()
    again = eng.encode_stream(q, k, v)
    torch.cuda.synchronize()
    assert torch.equal(first, again)
    assert eng.metrics() == m1 and eng.trace() == t1
