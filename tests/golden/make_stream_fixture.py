"""Generate the C1 / C2 whole-stream parity fixtures from the CPU oracle.

TEST INFRASTRUCTURE. The oracle (oracle/liboracle.so) is the restatement of
the reference engine pinned bit-exact to the reference itself
(tests/test_oracle_pin.py); running the reference through the Eigen shim at
these sizes would take hours, the oracle (threads over heads) takes minutes.

    python tests/golden/make_stream_fixture.py c1   # 64 steps,  ~3 min on 8 cores
    python tests/golden/make_stream_fixture.py c2   # 256 steps, ~12 min on 8 cores
    python tests/golden/make_stream_fixture.py c4   # the c2 stream + 160 decode steps
    python tests/golden/make_stream_fixture.py c4_512k   # 512K tokens + 64 decode steps (~1 h)

BASELINE.json configs[1] (C1, Mistral-7B heads, 32K) and configs[2] (C2,
Llama-3-8B heads, 128K), exactly as bench.py runs them: 32 q / 8 kv heads,
d 128, chunk 512, unit 128, r_k 4, k_m 16, init 128, local 4096, hot 32,
decay 0.1, clamped positions, N(0,1) inputs rounded to bf16 (the oracle
consumes the bf16 values upcast to fp32). Inputs are regenerated from the
seed by `stream_inputs` (numpy PCG64, one draw per step), so the fixture holds
only what the GPU run is compared with:
  ids        per-step retrieved unit ids (-1 padded)           bit-exact
  unit_*     start/size/representative positions of every unit  bit-exact
  counters   units, hot, peak, hits, misses, loads, evictions, requested
  trace      (step, unit, hit) records                           bit-exact
  rows       oracle output rows {0, r_s, l_x-1} of every step, float16
  row_idx    r_s per step
  head_mean  mean |out| per step and head (all rows), float32
  out_inf    ||out||_inf per step (all rows)
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

HERE = os.path.dirname(os.path.abspath(__file__))

CFG = dict(chunk_size=512, unit_size=128, n_repr=4, local_size=4096, init_size=128, n_lookup=16, hot_capacity=32,
           decay=0.1)
SHAPE = dict(H=32, Hkv=8, d=128)
CASES = {"c1": dict(n=32768, seed=1), "c2": dict(n=131072, seed=2)}


def _bf16(x):
    import torch

    return torch.from_numpy(x).bfloat16().float().numpy()


def stream_inputs(seed, n, chunk=512):
    """Yields (q, k, v) per chunk step: N(0,1) float32 rounded to bf16."""
    rng = np.random.default_rng(seed)
    H, Hkv, d = SHAPE["H"], SHAPE["Hkv"], SHAPE["d"]
    for t0 in range(0, n, chunk):
        b = min(chunk, n - t0)
        q = _bf16(rng.standard_normal((b, H, d), dtype=np.float32))
        k = _bf16(rng.standard_normal((b, Hkv, d), dtype=np.float32))
        v = _bf16(rng.standard_normal((b, Hkv, d), dtype=np.float32))
        yield q, k, v


def row_pick(seed, steps, l_x=512):
    return np.random.default_rng(seed + 1000).integers(1, l_x - 1, size=steps)


def main(name):
    from oracle import oracle as O

    O.build()
    c = CASES[name]
    n, seed = c["n"], c["seed"]
    steps = n // CFG["chunk_size"]
    eng = O.OracleEngine(O.EngineConfig.make(**CFG),
                         O.ModelShape.make(n_heads=SHAPE["H"], n_kv_heads=SHAPE["Hkv"], head_dim=SHAPE["d"]),
                         n_threads=os.cpu_count() or 1)
    ridx = row_pick(seed, steps)
    ids = np.full((steps, CFG["n_lookup"]), -1, np.int64)
    rows = np.zeros((steps, 3, SHAPE["H"], SHAPE["d"]), np.float16)
    head_mean = np.zeros((steps, SHAPE["H"]), np.float32)
    out_inf = np.zeros(steps, np.float32)
    t0 = time.time()
    for s, (q, k, v) in enumerate(stream_inputs(seed, n)):
        r = eng.step(q, k, v)
        ids[s, :len(r.retrieved_ids)] = r.retrieved_ids
        rows[s] = r.out[[0, ridx[s], q.shape[0] - 1]].astype(np.float16)
        head_mean[s] = np.abs(r.out).mean(axis=(0, 2))
        out_inf[s] = np.abs(r.out).max()
        if s % 16 == 0:
            print(f"{name} step {s}/{steps} {time.time() - t0:.0f}s", flush=True)
    m = eng.metrics()
    U = m["units"]
    infos = [eng.unit_info(u) for u in range(U)]
    tr = np.array(eng.trace(), np.int64).reshape(-1, 3)
    np.savez_compressed(
        os.path.join(HERE, f"stream_{name}.npz"), n=n, seed=seed, ids=ids, rows=rows, row_idx=ridx,
        head_mean=head_mean, out_inf=out_inf,
        unit_start=np.array([i["start_abs"] for i in infos], np.int64),
        unit_size=np.array([i["size"] for i in infos], np.int64),
        unit_repr=np.array([i["repr_abs"] for i in infos], np.int64).reshape(U, -1),
        counters=np.array([m[k] for k in COUNTERS], np.int64), trace=tr)
    print(f"{name}: {steps} steps, {U} units, {len(tr)} trace records, {time.time() - t0:.0f}s; {m}")


COUNTERS = ["units", "hot_units", "peak_hot_units", "hits", "misses", "loads", "evictions", "requested"]


C4_DEC = 160  # decode steps after the C2 prefill (a unit completes every 128)


def decode_inputs(seed, steps):
    """One-token q/k/v per decode step, N(0,1) rounded to bf16."""
    rng = np.random.default_rng(seed)
    H, Hkv, d = SHAPE["H"], SHAPE["Hkv"], SHAPE["d"]
    for _ in range(steps):
        yield (_bf16(rng.standard_normal((1, H, d), dtype=np.float32)),
               _bf16(rng.standard_normal((1, Hkv, d), dtype=np.float32)),
               _bf16(rng.standard_normal((1, Hkv, d), dtype=np.float32)))


def main_c4(n=None, seed=None, out="stream_c4.npz", n_dec=None):
    """C4 at 128K: the C2 stream (seed 2) then C4_DEC decode steps (seed 4):
    per-step ids and output rows of the decode steps, final state. With n =
    524288 (`c4_512k`): the 512K context, whose lookup is the streaming scan."""
    from oracle import oracle as O

    O.build()
    n = n or CASES["c2"]["n"]
    seed = seed or CASES["c2"]["seed"]
    C4 = n_dec or C4_DEC
    eng = O.OracleEngine(O.EngineConfig.make(**CFG),
                         O.ModelShape.make(n_heads=SHAPE["H"], n_kv_heads=SHAPE["Hkv"], head_dim=SHAPE["d"]),
                         n_threads=os.cpu_count() or 1)
    t0 = time.time()
    for s, (q, k, v) in enumerate(stream_inputs(seed, n)):
        eng.step(q, k, v)
        if s % 32 == 0:
            print(f"c4 prefill step {s} {time.time() - t0:.0f}s", flush=True)
    ids = np.full((C4, CFG["n_lookup"]), -1, np.int64)
    rows = np.zeros((C4, SHAPE["H"], SHAPE["d"]), np.float32)
    for s, (q, k, v) in enumerate(decode_inputs(4, C4)):
        r = eng.step(q, k, v)
        ids[s, :len(r.retrieved_ids)] = r.retrieved_ids
        rows[s] = r.out[0]
    m = eng.metrics()
    U = m["units"]
    infos = [eng.unit_info(u) for u in range(U)]
    tr = np.array(eng.trace(), np.int64).reshape(-1, 3)
    np.savez_compressed(
        os.path.join(HERE, out), n=n, seed=seed, dec_seed=4, n_dec=C4, ids=ids, rows=rows.astype(np.float16),
        unit_start=np.array([i["start_abs"] for i in infos], np.int64),
        unit_size=np.array([i["size"] for i in infos], np.int64),
        unit_repr=np.array([i["repr_abs"] for i in infos], np.int64).reshape(U, -1),
        counters=np.array([m[k] for k in COUNTERS], np.int64), trace=tr)
    print(f"{out}: {C4} decode steps after {n} tokens, {U} units, {len(tr)} trace records, {time.time() - t0:.0f}s; {m}")

if __name__ == "__main__":
    for nm in sys.argv[1:] or ["c1", "c2", "c4"]:
        if nm == "c4":
            main_c4()
        elif nm == "c4_512k":
            main_c4(n=524288, seed=5, out="stream_c4_512k.npz", n_dec=64)
        else:
            main(nm)
