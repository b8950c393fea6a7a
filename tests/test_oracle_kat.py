"""Known-answer and property tests of the CPU oracle (test infrastructure).

The reference ships no test sources; its known answers are the
SPEC examples, ported here one by one (SPEC.md line cited per test), plus the
oracle-check acceptance criteria 1-4 (cli.cpp:249-342) at
small sizes. The oracle is the checker for every GPU parity test, so it is
pinned here before it is trusted (and bit-exactly against the compiled
reference in test_oracle_pin.py).
"""
import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import oracle as O

C0 = dict(chunk_size=128, unit_size=128, n_repr=4, local_size=512, init_size=64, n_lookup=4, hot_capacity=32,
          decay=0.1)


# ---------------------------------------------------------------- representatives
def test_select_representatives_kat():
    # scores [3,1,2,5], r_k 2 -> tokens {0, 3}
    assert O.select_representatives([3, 1, 2, 5], 2) == [0, 3]
    # a 1-token unit with r_k 4 returns that token
    assert O.select_representatives([0.7], 4) == [0]


def test_select_representatives_ties_prefer_lower_index():
    assert O.select_representatives([1, 1, 1, 1, 1], 3) == [0, 1, 2]
    assert O.select_representatives([0, 2, 2, 1, 2], 2) == [1, 2]


@settings(max_examples=200, deadline=None)
@given(st.lists(st.integers(-3, 3), min_size=1, max_size=64), st.integers(1, 8))
def test_select_representatives_property(scores, r_k):
    """repr_score.hpp:94-112: top min(r_k, n) by score desc, tie -> lower
    index, returned ascending."""
    s = np.asarray(scores, np.float32)
    order = sorted(range(len(s)), key=lambda i: (-s[i], i))[: min(r_k, len(s))]
    assert O.select_representatives(s, r_k) == sorted(order)


# ---------------------------------------------------------------- top-k
def test_argsort_topk_kat():
    # SPEC.md:396
    assert O.argsort_topk([3, 1, 2, 5], 2) == [3, 0]


@settings(max_examples=200, deadline=None)
@given(st.lists(st.integers(-4, 4), min_size=0, max_size=80), st.integers(0, 20))
def test_argsort_topk_property(vals, k):
    """memory.hpp:245-253 ordering: value desc, then id asc."""
    v = np.asarray(vals, np.float64)
    want = sorted(range(len(v)), key=lambda i: (-v[i], i))[: min(k, len(v))]
    assert O.argsort_topk(v, k) == want


# ---------------------------------------------------------------- repr scores
def test_repr_scores_zero_vectors():
    # SPEC.md:161
    z = np.zeros((16, 2, 8))
    assert np.all(O.batch_repr_scores(z, z, 4) == 0.0)


def test_repr_score_unit_vector_local_one():
    # l_L = 1 and q = k = e -> r_m = 1.0 (every token with a successor)
    n, d = 10, 8
    e = np.zeros((n, 1, d))
    e[:, :, 3] = 1.0
    r = O.batch_repr_scores(e, e, 1)
    assert np.all(r[: n - 1] == 1.0)


def test_incremental_scores_equal_batch():
    """incremental (ScoreAccumulator in the streaming engine)
    equals the batch computation within 1e-6 on 512 tokens with l_L = 64."""
    n, lL = 512, 64
    rng = np.random.default_rng(3)
    q = rng.standard_normal((n, 2, 16)).astype(np.float32)
    k = rng.standard_normal((n, 2, 16)).astype(np.float32)
    v = rng.standard_normal((n, 2, 16)).astype(np.float32)
    cfg = O.EngineConfig.make(chunk_size=32, unit_size=32, n_repr=2, local_size=lL, init_size=0, n_lookup=0,
                              hot_capacity=0)
    eng = O.OracleEngine(cfg, O.ModelShape.make(n_heads=2, head_dim=16))
    for off in range(0, n, 32):
        eng.step(q[off:off + 32], k[off:off + 32], v[off:off + 32])
    inc = eng.evicted_scores()
    batch = O.batch_repr_scores(q, k, lL)
    assert len(inc) == n - lL
    assert np.abs(inc.astype(np.float64) - batch[: len(inc)]).max() <= 1e-6


# ---------------------------------------------------------------- packing
def _packed_units(n_tokens, finish):
    cfg = O.EngineConfig.make(chunk_size=64, unit_size=128, n_repr=4, local_size=64, init_size=0, n_lookup=0,
                              hot_capacity=0)
    eng = O.OracleEngine(cfg, O.ModelShape.make(n_heads=1, head_dim=8))
    rng = np.random.default_rng(0)
    x = rng.standard_normal((n_tokens, 1, 8)).astype(np.float32)
    off = 0
    while off < n_tokens:
        b = min(64, n_tokens - off)
        eng.step(x[off:off + b], x[off:off + b], x[off:off + b])
        off += b
    if finish:
        eng.finish()
    return [eng.unit_info(u)["size"] for u in range(eng.metrics()["units"])], eng


def test_packing_256_evicted_two_units():
    # 256 evicted tokens -> 2 units
    sizes, _ = _packed_units(256 + 64, finish=False)
    assert sizes == [128, 128]


def test_packing_flush_at_stream_end():
    # 300 evicted at stream end -> 128, 128, 44
    sizes, eng = _packed_units(300 + 64, finish=True)
    assert sizes == [128, 128, 44]
    assert [eng.unit_info(u)["start_abs"] for u in range(3)] == [0, 128, 256]


# ---------------------------------------------------------------- relevance
def test_relevance_orthogonal_is_zero():
    # SPEC.md:229
    q = np.zeros((1, 1, 4), np.float32)
    q[0, 0, 0] = 1
    r = np.zeros((1, 1, 4), np.float32)
    r[0, 0, 1] = 1
    assert O.relevance_unit(q, r) == 0.0


def test_relevance_single_query_single_repr_is_dot():
    # SPEC.md:230
    rng = np.random.default_rng(1)
    q = rng.standard_normal((1, 1, 16)).astype(np.float32)
    r = rng.standard_normal((1, 1, 16)).astype(np.float32)
    want = float(np.dot(q[0, 0].astype(np.float64), r[0, 0].astype(np.float64)))
    assert abs(O.relevance_unit(q, r) - want) <= 1e-12 * max(1.0, abs(want))


def test_relevance_all_matches_unit_and_gqa_sum():
    rng = np.random.default_rng(2)
    q = rng.standard_normal((5, 4, 8)).astype(np.float32)
    reprk = rng.standard_normal((7, 3, 2, 8)).astype(np.float32)  # [U][r_k][Hkv][d]
    rel = O.relevance_all(q, reprk)
    for u in range(7):
        assert abs(rel[u] - O.relevance_unit(q, reprk[u])) <= 1e-12 * max(1.0, abs(rel[u]))
    qs = q.astype(np.float64).sum(0).reshape(2, 2, 8).sum(1)  # per KV group
    want = np.einsum("grd,urgd->u", qs[:, None, :].repeat(3, 1), reprk.astype(np.float64))
    assert np.allclose(rel, want, rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- lookup / LRU
def _stream(cfg_kw, n, H=1, d=16, seed=0):
    cfg = O.EngineConfig.make(**cfg_kw)
    eng = O.OracleEngine(cfg, O.ModelShape.make(n_heads=H, head_dim=d))
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((n, H, d)).astype(np.float32)
    k = rng.standard_normal((n, H, d)).astype(np.float32)
    v = rng.standard_normal((n, H, d)).astype(np.float32)
    recs = []
    for off in range(0, n, cfg_kw["chunk_size"]):
        b = min(cfg_kw["chunk_size"], n - off)
        recs.append(eng.step(q[off:off + b], k[off:off + b], v[off:off + b]))
    return eng, recs


def test_lookup_km_ge_units_returns_all_sorted():
    # SPEC.md:239
    cfg = dict(chunk_size=32, unit_size=32, n_repr=2, local_size=64, init_size=0, n_lookup=50, hot_capacity=50)
    eng, recs = _stream(cfg, 256)
    units_before_last = eng.metrics()["units"] - 1  # the last step's new unit is not yet visible
    assert recs[-1].retrieved_ids == list(range(units_before_last))


def test_lookup_km_zero_returns_none():
    # SPEC.md:240
    cfg = dict(chunk_size=32, unit_size=32, n_repr=2, local_size=64, init_size=0, n_lookup=0, hot_capacity=4)
    eng, recs = _stream(cfg, 256)
    assert all(r.retrieved_ids == [] for r in recs)
    assert eng.metrics()["requested"] == 0


def test_frequency_decay_zero_is_mass_and_two_steps_accumulate():
    """with d = 0 s_b equals the last mass; over two steps
    s_b = a*d + b for a unit attended in both."""
    for decay in (0.0, 0.5):
        cfg = dict(chunk_size=32, unit_size=32, n_repr=2, local_size=64, init_size=0, n_lookup=3, hot_capacity=8,
                   decay=decay)
        eng, recs = _stream(cfg, 320, seed=4)
        a, b = recs[-2], recs[-1]
        freq, hot = eng.unit_freq(eng.metrics()["units"])
        ma = dict(zip(a.retrieved_ids, a.masses))
        mb = dict(zip(b.retrieved_ids, b.masses))
        both = set(ma) & set(mb)
        assert both
        for u in both:
            assert hot[u]
            # every hot unit decays every step (memory.hpp:273-285); u was attended at both steps
            assert abs(freq[u] - (ma[u] * decay + mb[u])) <= 1e-12
        for u in set(mb) - set(ma):
            assert abs(freq[u] - mb[u]) <= 1e-12 or decay != 0.0


def test_capacity_evicts_smallest_scores():
    """the hot tier never exceeds capacity at a step boundary and
    evictions remove the minimum-score units (tie -> lower id)."""
    cfg = dict(chunk_size=32, unit_size=32, n_repr=2, local_size=64, init_size=0, n_lookup=4, hot_capacity=5,
               decay=0.3)
    eng, recs = _stream(cfg, 1024, seed=5)
    m = eng.metrics()
    assert m["hot_units"] <= 5 and m["peak_hot_units"] <= 5 + 4
    assert m["evictions"] == m["loads"] - m["hot_units"]
    assert m["hits"] + m["misses"] == m["requested"]


# ---------------------------------------------------------------- attention
def test_single_huge_key_returns_its_value():
    # SPEC.md:106
    rng = np.random.default_rng(6)
    n, d = 8, 16
    q = rng.standard_normal((n, 1, d)) * 0.01
    k = rng.standard_normal((n, 1, d)) * 0.01
    v = rng.standard_normal((n, 1, d))
    q[-1, 0] = 0
    q[-1, 0, 0] = 1.0
    k[2, 0] = 0
    k[2, 0, 0] = 1e4
    out = O.dense_attention(q, k, v, 1, 1 << 40)
    assert np.abs(out[-1, 0] - v[2, 0]).max() < 1e-9


def test_empty_window_returns_own_value():
    # the first token attends only to itself
    rng = np.random.default_rng(7)
    q, k, v = (rng.standard_normal((1, 2, 8)) for _ in range(3))
    out = O.dense_attention(q, k, v, 1, 1 << 40)
    assert np.abs(out[0] - v[0]).max() < 1e-12


def test_degenerate_engine_equals_dense():
    """oracle-check #1 (cli.cpp:249-271): absolute positions and a
    local window covering the stream make the engine plain causal attention."""
    n = 512
    shape = O.ModelShape.make(n_heads=2, head_dim=32)
    q, k, v = O.adapter_batch(0, shape, O.noise_ids(0, n))
    cfg = O.EngineConfig.make(**dict(C0, local_size=n, position_mode="absolute"))
    got, _ = O.run_engine(O.OracleEngine(cfg, shape), q, k, v, O.encode_schedule(n, 128, 16), 16)
    assert np.abs(got - O.dense_attention(q, k, v, 1, n)).max() <= 1e-5


def test_full_retrieval_equals_windowed():
    """oracle-check #2 (cli.cpp:274-299)."""
    n = 1536
    shape = O.ModelShape.make(n_heads=1, head_dim=32)
    q, k, v = O.adapter_batch(1, shape, O.noise_ids(1, n))
    km = n // 128 + 2
    cfg = O.EngineConfig.make(**dict(C0, n_lookup=km, hot_capacity=km))
    sched = O.encode_schedule(n, 128, 16)
    got, _ = O.run_engine(O.OracleEngine(cfg, shape), q, k, v, sched, 16)
    want = O.windowed_attention(q, k, v, sched, 64, 512, 128, 0)
    assert np.abs(got - want).max() <= 1e-5


def test_engine_token_conservation():
    """engine.hpp:370-380: init + local + pending + in_units == fed after every
    step of a C0 stream with decode tail (the softmax-row check of the same
    block is compared against the reference's own count in test_oracle_pin)."""
    n = 2048
    shape = O.ModelShape.make(n_heads=1, head_dim=64)
    q, k, v = O.adapter_batch(2, shape, O.noise_ids(2, n))
    eng = O.OracleEngine(O.EngineConfig.make(**C0), shape)
    fed = 0
    sched = O.encode_schedule(n, 128, 16)
    for si, b in enumerate(sched):
        eng.step(q[fed:fed + b], k[fed:fed + b], v[fed:fed + b], decode=si >= len(sched) - 16)
        fed += b
        s = eng.stream_state()
        in_units = sum(eng.unit_info(u)["size"] for u in range(eng.metrics()["units"]))
        assert s["tokens_fed"] == fed
        assert s["initial_len"] + s["local_len"] + s["pending_partial"] + in_units == fed
    checks, _ = eng.invariants()
    assert checks > 0


# ---------------------------------------------------------------- workload
def test_planted_expected_unit():
    # expected plant unit = (offset - l_I) / 128
    cfg = O.EngineConfig.make(**dict(C0, init_size=128, local_size=1024))
    p = O.gen_planted(5, 8192, 64, cfg, align=True)
    assert p["expected_units"][0] == (p["plant_start"] - 128) // 128


def test_max_window():
    # W = l_I + k_m * l_bs + l_L = 8320 for k_m 32 (defaults)
    c = O.EngineConfig.make()
    assert c.init_size + c.n_lookup * c.unit_size + c.local_size == 8320


def test_config_errors():
    with pytest.raises(O.ConfigError):
        O.OracleEngine(O.EngineConfig.make(hot_capacity=3, n_lookup=4), O.ModelShape.make())
    eng = O.OracleEngine(O.EngineConfig.make(**C0), O.ModelShape.make(head_dim=8))
    x = np.zeros((129, 1, 8), np.float32)
    with pytest.raises(O.StreamError):
        eng.step(x, x, x)  # chunk larger than chunk_size (engine.hpp:92-98)
    with pytest.raises(O.StreamError):
        eng.step(x[:2], x[:2], x[:2], decode=True)  # decode takes exactly one token
