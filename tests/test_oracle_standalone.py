"""CPU checks of the oracle's stand-alone operators (the checkers of the
C-ABI's infllm_attend / infllm_store_* / infllm_score_acc_*), against the
oracle's independent double-precision dense attention (oracle.hpp:64-97) and
against the oracle engine itself (the same TieredStore / ScoreAccumulator
arithmetic driven by StreamEngine::step)."""
import numpy as np

from oracle import oracle as O


def test_attend_absolute_one_local_segment_equals_dense():
    rng = np.random.default_rng(0)
    n, l_x, H, Hkv, d = 200, 24, 4, 2, 32
    q = rng.standard_normal((n, H, d)).astype(np.float32) * 0.5
    k = rng.standard_normal((n, Hkv, d)).astype(np.float32) * 0.5
    v = rng.standard_normal((n, Hkv, d)).astype(np.float32)
    c = n - l_x
    out, mass, w = O.attend([("local", 0, k[:c], v[:c])], q[c:], k[c:], v[c:], c, 1 << 20, "absolute",
                            emit_weights=True)
    want = O.dense_attention(q, k, v, 1)[c:]
    assert np.abs(out - want).max() <= 1e-5 * np.abs(want).max()
    assert np.allclose(w.sum(-1), 1.0, atol=1e-5)
    assert abs(mass[0] - w[:, :, :c].astype(np.float64).sum() / H) <= 1e-9 * max(1.0, mass[0])


def test_attend_clamped_matches_engine_step():
    """One engine step after a warm-up reproduces attend() over its own window:
    initial tokens, no units (lookup none), local window, batch."""
    cfg = dict(chunk_size=64, unit_size=32, n_repr=2, local_size=96, init_size=16, n_lookup=0, hot_capacity=4,
               lookup_mode="none")
    H, Hkv, d = 2, 1, 16
    rng = np.random.default_rng(1)
    n = 64 * 4
    q = rng.standard_normal((n, H, d)).astype(np.float32) * 0.5
    k = rng.standard_normal((n, Hkv, d)).astype(np.float32) * 0.5
    v = rng.standard_normal((n, Hkv, d)).astype(np.float32)
    e = O.OracleEngine(O.EngineConfig.make(**cfg), O.ModelShape.make(n_heads=H, n_kv_heads=Hkv, head_dim=d))
    for s in range(3):
        e.step(q[64 * s:64 * s + 64], k[64 * s:64 * s + 64], v[64 * s:64 * s + 64])
    st = e.stream_state()
    s0 = 192
    local0 = s0 - st["local_len"]
    init = st["initial_len"]
    r = e.step(q[s0:], k[s0:], v[s0:])
    segs = [("initial", 0, k[:init], v[:init]), ("local", local0, k[local0:s0], v[local0:s0])]
    out, _, _ = O.attend(segs, q[s0:], k[s0:], v[s0:], s0, 96, "clamped")
    assert np.abs(out - r.out).max() <= 1e-6 * np.abs(r.out).max()


def test_store_and_accumulator_smoke():
    rng = np.random.default_rng(2)
    st = O.OracleStore(3, 0.5, 4, 2, 8, 64)
    for _ in range(6):
        st.add_unit(rng.standard_normal((2, 2, 8)), 32)
    st.begin_step(0)
    ids = st.lookup(rng.standard_normal((5, 4, 8)), 4)
    assert ids == sorted(ids) and len(ids) == 4
    st.update_frequency([(i, 1.0 + i) for i in ids])
    st.enforce_capacity()
    st.note_step_boundary()
    c = st.counters()
    assert c["hot_units"] == 3 and c["evictions"] == 1 and c["misses"] == 4
    acc = O.OracleScoreAccumulator(8, 2, 1, 4)
    q = rng.standard_normal((12, 2, 4))
    keys = rng.standard_normal((12, 1, 4))
    acc.accumulate(q, 0, keys)
    sc = acc.finalize_front(4)
    # token m sees queries m+1 .. m+8 (all inside this batch for m < 4)
    want = [sum(float(q[i, h] @ keys[m, 0]) for i in range(m + 1, m + 9) for h in range(2)) / 8 for m in range(4)]
    assert np.allclose(sc, want, rtol=1e-6)
