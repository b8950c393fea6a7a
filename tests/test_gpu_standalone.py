"""Stand-alone operators of the drop-in boundary vs the CPU oracle:
infllm_attend (attention.hpp:116-230 + masses engine.hpp:271-283 + emitted
weights), infllm_store_* (TieredStore, memory.hpp:170-323) and
infllm_score_acc_* (ScoreAccumulator, repr_score.hpp:21-89).

Bars: attention outputs 1e-5 relative (||d||_inf / ||ref||_inf) in fp32 and
2e-2 in bf16 (oracle fed the bf16-rounded inputs); weights 1e-6 absolute and
masses 1e-5 relative in fp32; lookup ids, hit/miss counters and trace
bit-exact; frequency scores 1e-12 relative; finalized representative scores
1e-6 relative with identical representative selections.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.parity_util import bf16_round, rel_err

pytestmark = pytest.mark.gpu


def _window(rng, H, Hkv, d, bf16):
    def kv(n):
        k = rng.standard_normal((n, Hkv, d)).astype(np.float32) * 0.4
        v = rng.standard_normal((n, Hkv, d)).astype(np.float32)
        return (bf16_round(k), bf16_round(v)) if bf16 else (k, v)

    segs = [("initial", 0, *kv(64)), ("retrieved", 1000, *kv(128)), ("retrieved", 2304, *kv(100)),
            ("local", 4700, *kv(300))]
    q = rng.standard_normal((40, H, d)).astype(np.float32) * 0.4
    k, v = kv(40)
    if bf16:
        q = bf16_round(q)
    return segs, q, k, v


@pytest.mark.parametrize("dtype,mode,d", [(torch.float32, "clamped", 64), (torch.float32, "absolute", 64),
                                          (torch.bfloat16, "clamped", 128), (torch.float32, "clamped", 33)])
def test_attend_vs_oracle(dtype, mode, d):
    from paper_2402_04617_b200 import attend

    rng = np.random.default_rng(5)
    H, Hkv = 4, 2
    bf16 = dtype == torch.bfloat16
    segs, q, k, v = _window(rng, H, Hkv, d, bf16)
    start, L = 5000, 256  # local keys 4700..4999: the far ones are clamped at l_L
    o_out, o_mass, o_w = O.attend(segs, q, k, v, start, L, mode, emit_weights=True)
    dev = lambda x: torch.from_numpy(x).to("cuda", dtype)  # noqa: E731
    g_out, g_mass, g_w = attend([(s[0], s[1], dev(s[2]), dev(s[3])) for s in segs], dev(q), dev(k), dev(v), start, L,
                                mode, emit_weights=True)
    tol = 2e-2 if bf16 else 1e-5
    assert rel_err(g_out.float().cpu().numpy(), o_out) <= tol
    if not bf16:
        assert np.abs(g_w.cpu().numpy() - o_w).max() <= 1e-6
        assert np.allclose(g_mass.cpu().numpy(), o_mass, rtol=1e-5, atol=0)
        # softmax rows sum to one over the valid columns (engine.hpp check_softmax)
        assert np.allclose(g_w.sum(-1).cpu().numpy(), 1.0, atol=1e-5)


def test_attend_errors():
    from paper_2402_04617_b200 import StreamError, attend

    q = torch.zeros((0, 2, 64), device="cuda")
    with pytest.raises(StreamError):
        attend([], q, torch.zeros((0, 1, 64), device="cuda"), torch.zeros((0, 1, 64), device="cuda"), 0, 64)


@pytest.mark.parametrize("dtype,d", [(torch.float32, 64), (torch.bfloat16, 128)])
def test_store_vs_oracle(dtype, d):
    from paper_2402_04617_b200 import TieredStore

    rng = np.random.default_rng(9)
    H, Hkv, r_k, cap, k_m, decay = 8, 2, 4, 10, 6, 0.1
    bpt = Hkv * 2 * d * 2
    ost = O.OracleStore(cap, decay, H, Hkv, d, bpt)
    gst = TieredStore(cap, decay, H, Hkv, d, r_k, dtype, bpt)
    rnd = lambda *s: bf16_round(rng.standard_normal(s).astype(np.float32))  # noqa: E731
    dev = lambda x: torch.from_numpy(x).to("cuda", dtype)  # noqa: E731
    for u in range(40):
        n = r_k if u % 7 else 2  # a flushed partial unit keeps fewer representatives
        rk = rnd(n, Hkv, d)
        assert ost.add_unit(rk, 128) == gst.add_unit(dev(rk), 128) == u
    for step in range(30):
        if step % 10 == 9:  # the index grows between steps
            rk = rnd(r_k, Hkv, d)
            assert ost.add_unit(rk, 128) == gst.add_unit(dev(rk), 128)
        ost.begin_step(step)
        gst.begin_step(step)
        q = rnd(16, H, d)
        oid = ost.lookup(q, k_m)
        gid = gst.lookup(dev(q), k_m)
        assert gid == oid, f"step {step}: {gid} vs {oid}"
        pairs = [(i, float(rng.random())) for i in oid]
        ost.update_frequency(pairs)
        gst.update_frequency(pairs)
        ost.enforce_capacity()
        gst.enforce_capacity()
        ost.note_step_boundary()
        gst.note_step_boundary()
    assert gst.counters() == ost.counters()
    assert gst.trace() == ost.trace()
    n = ost.counters()["units"]
    of, oh = ost.unit_freq(n)
    gf, gh = gst.unit_freq(n)
    assert (oh == gh).all()
    assert np.allclose(gf, of, rtol=1e-12, atol=0)


def test_store_errors():
    from paper_2402_04617_b200 import StreamError, TieredStore

    gst = TieredStore(2, 0.1, 2, 1, 64, 4, torch.float32, 0)
    gst.add_unit(torch.randn((4, 1, 64), device="cuda"), 128)
    with pytest.raises(StreamError, match="not hot"):  # memory.hpp:277-279
        gst.update_frequency([(0, 1.0)])


def test_score_accumulator_vs_oracle():
    from paper_2402_04617_b200 import ScoreAccumulator, select_representatives

    rng = np.random.default_rng(3)
    H, Hkv, d, L = 4, 2, 64, 96
    oacc = O.OracleScoreAccumulator(L, H, Hkv, d)
    gacc = ScoreAccumulator(L, H, Hkv, d, torch.float32)
    keys = np.zeros((0, Hkv, d), np.float32)
    lo, s = 0, 0
    for b in [32, 40, 17, 64, 50, 33, 64, 29]:
        q = rng.standard_normal((b, H, d)).astype(np.float32)
        k = rng.standard_normal((b, Hkv, d)).astype(np.float32)
        keys = np.concatenate([keys, k], 0)
        oacc.accumulate(q, s, keys)
        gacc.accumulate(torch.from_numpy(q).cuda(), s, torch.from_numpy(keys).cuda())
        s += b
        # tokens that left the window (engine.hpp:306): their band is complete
        n_out = max(0, (s - lo) - L)
        if n_out:
            o = oacc.finalize_front(n_out)
            g = gacc.finalize_front(n_out)
            assert np.allclose(g, o, rtol=1e-6, atol=1e-7)
            so = O.select_representatives(o, 4)
            sg = select_representatives(torch.from_numpy(g).cuda(), 4)[0].tolist()
            assert [x for x in sg if x >= 0] == list(so)
            keys = keys[n_out:]
            lo += n_out
