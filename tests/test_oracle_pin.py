"""Pin the oracle restatement against the reference itself.

oracle/_ref/*.so is the reference engine compiled from its own headers where
they lie under /root/reference (oracle/Makefile `ref`, Eigen-subset shim in
oracle/eigen_shim). Every comparison here is BIT-EXACT: outputs, retrieved
ids, representative tokens, LRU counters, trace and invariant counts. Skipped
when neither the reference sources nor the prebuilt oracle/_ref exist.
"""
import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import oracle as O
from oracle import ref as R

pytestmark = pytest.mark.skipif(not R.available(), reason="reference not present (oracle/_ref unbuilt)")

C0 = dict(chunk_size=128, unit_size=128, n_repr=4, local_size=512, init_size=64, n_lookup=4, hot_capacity=32,
          decay=0.1)


def _run_both(cfg_kw, H, Hkv, d, q, k, v, schedule, decode_tail, ids=None, finish=True, seed=0):
    """Same stream through StreamEngine<float> (reference) and the oracle."""
    inject = ids is None
    cfg = O.EngineConfig.make(**cfg_kw)
    reng = R.RefEngine(cfg, H, d, v.shape[2], seed=seed, inject=inject)
    if inject:
        reng.set_inputs(q, k, v)
    oeng = O.OracleEngine(cfg, O.ModelShape.make(n_heads=H, n_kv_heads=Hkv, head_dim=d, value_dim=v.shape[2]),
                          n_threads=4)
    fed = 0
    first_decode = len(schedule) - decode_tail
    for si, b in enumerate(schedule):
        dec = si >= first_decode
        rout, rids = reng.step(b, decode=dec, ids=None if inject else ids[fed:fed + b])
        o = oeng.step(q[fed:fed + b], k[fed:fed + b], v[fed:fed + b], decode=dec)
        assert rids[0] == o.retrieved_ids, f"step {si}: ids"
        assert np.array_equal(rout[0], o.out), f"step {si}: attention output not bit-identical"
        fed += b
    if finish:
        reng.finish()
        oeng.finish()
    rm, om = reng.metrics(), oeng.metrics()
    assert rm == om
    for u in range(om["units"]):
        ru, ou = reng.unit_info(u), oeng.unit_info(u)
        assert (ru["start_abs"], ru["size"], ru["repr_abs"]) == (ou["start_abs"], ou["size"], ou["repr_abs"])
    assert reng.trace() == oeng.trace()
    assert reng.stream_state() == oeng.stream_state()
    assert reng.invariants() == oeng.invariants()
    return reng, oeng


@pytest.mark.parametrize("seed", [0, 1])
def test_c0_reference_adapter_bit_exact(seed):
    """C0 (BASELINE configs[0]) through the reference's own SyntheticAdapter
    (adapter.hpp:45-69, q == k) vs the oracle fed the restated adapter."""
    n = 4096
    shape = O.ModelShape.make(n_heads=1, head_dim=64)
    ids = O.noise_ids(seed, n)
    q, k, v = O.adapter_batch(seed, shape, ids)
    _run_both(C0, 1, 1, 64, q, k, v, O.encode_schedule(n, 128, 32), 32, ids=ids, seed=seed)


def test_gqa_ragged_injected_bit_exact():
    cfg = dict(chunk_size=100, unit_size=32, n_repr=3, local_size=256, init_size=40, n_lookup=5, hot_capacity=6)
    n = 2000
    rng = np.random.default_rng(3)
    q = (rng.standard_normal((n, 8, 32)) * 0.4).astype(np.float32)
    k = (rng.standard_normal((n, 2, 32)) * 0.4).astype(np.float32)
    v = rng.standard_normal((n, 2, 32)).astype(np.float32)
    _run_both(cfg, 8, 2, 32, q, k, v, O.encode_schedule(n, 100, 20), 20)


@pytest.mark.parametrize("mode", ["decode_only", "none"])
def test_lookup_modes_bit_exact(mode):
    n = 1536
    rng = np.random.default_rng(5)
    q = (rng.standard_normal((n, 2, 64)) * 0.3).astype(np.float32)
    k = (rng.standard_normal((n, 2, 64)) * 0.3).astype(np.float32)
    v = rng.standard_normal((n, 2, 64)).astype(np.float32)
    _run_both(dict(C0, lookup_mode=mode), 2, 2, 64, q, k, v, O.encode_schedule(n, 128, 16), 16)


def test_absolute_positions_bit_exact():
    n = 1536
    rng = np.random.default_rng(9)
    q = (rng.standard_normal((n, 2, 32)) * 0.3).astype(np.float32)
    k = (rng.standard_normal((n, 2, 32)) * 0.3).astype(np.float32)
    v = rng.standard_normal((n, 2, 32)).astype(np.float32)
    _run_both(dict(C0, position_mode="absolute"), 2, 2, 32, q, k, v, O.encode_schedule(n, 128, 8), 8)


def test_adapter_restatement_bit_exact():
    """oracle adapter_batch (adapter.hpp:45-69 + rng.hpp:11-64) reproduces the
    reference adapter's q/k/v: a one-step stream with dense-equivalent
    settings returns identical attention through both."""
    n = 128
    shape = O.ModelShape.make(n_heads=2, head_dim=16)
    ids = O.noise_ids(11, n)
    q, k, v = O.adapter_batch(0, shape, ids)
    cfg = dict(C0, local_size=n)
    _run_both(cfg, 2, 2, 16, q, k, v, [n], 0, ids=ids, finish=False)


# ---------------------------------------------------------------- standalone functions
@settings(max_examples=100, deadline=None)
@given(st.lists(st.integers(-3, 3), min_size=1, max_size=200), st.integers(1, 8))
def test_select_representatives_vs_reference(scores, r_k):
    assert O.select_representatives(scores, r_k) == R.select_representatives(scores, r_k)


@settings(max_examples=100, deadline=None)
@given(st.lists(st.integers(-4, 4), min_size=0, max_size=200), st.integers(0, 40))
def test_argsort_topk_vs_reference(vals, k):
    assert O.argsort_topk(vals, k) == R.argsort_topk(vals, k)


def test_store_lookup_vs_reference():
    """TieredStore::relevance_all + lookup (memory.hpp:217-269)."""
    rng = np.random.default_rng(4)
    for U, km in [(1, 4), (50, 8), (300, 16)]:
        q = rng.standard_normal((16, 4, 32)).astype(np.float32)
        reprk = rng.standard_normal((U, 4, 2, 32)).astype(np.float32)
        rrel, rids = R.store_lookup(q, reprk, km)
        orel = O.relevance_all(q, reprk)
        assert np.array_equal(rrel, orel)
        assert rids == sorted(O.argsort_topk(orel, km))


def test_dense_windowed_batch_vs_reference():
    """oracle.hpp:64-184 (the reference's own independent oracles)."""
    n = 700
    rng = np.random.default_rng(8)
    q = rng.standard_normal((n, 2, 16))
    k = rng.standard_normal((n, 2, 16))
    v = rng.standard_normal((n, 2, 16))
    for pm in (0, 1):
        assert np.array_equal(O.dense_attention(q, k, v, pm, 300), R.dense_attention(q, k, v, pm, 300))
    sched = O.encode_schedule(n, 128, 12)
    assert np.array_equal(O.windowed_attention(q, k, v, sched, 64, 256, 128, 0),
                          R.windowed_attention(q, k, v, sched, 64, 256, 128, 0))
    assert np.array_equal(O.batch_repr_scores(q, k, 64), R.batch_repr_scores(q, k, 64))
