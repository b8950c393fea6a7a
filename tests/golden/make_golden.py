"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref, the
reference StreamEngine<float> compiled from /root/reference/proj/include).

Run here (the reference is not on the GPU box):  python tests/golden/make_golden.py

Each fixture holds the configuration, a checksum of the inputs (the inputs
are regenerated from seeds by the counter-based generators in the oracle),
the per-step retrieved unit ids, unit layout + representative tokens, LRU
counters, the lookup trace, a SHA-256 of the full attention output and the
output rows of the last tokens (float32, or float16 for the bf16 case whose
bar is 2e-2).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    # BASELINE configs[0] (C0) through the reference's own SyntheticAdapter, q == k
    "c0_adapter_seed0": dict(kind="adapter", seed=0, n=2048, tail=16, H=1, Hkv=1, d=64, keep=256, keep_dtype="f32",
                             cfg=dict(chunk_size=128, unit_size=128, n_repr=4, local_size=512, init_size=64,
                                      n_lookup=4, hot_capacity=32, decay=0.1)),
    # GQA 8/2, ragged chunks, units not aligned with chunks, hot-tier evictions
    "gqa_ragged": dict(kind="gaussian", seed=3, scale=0.4, n=1200, tail=20, H=8, Hkv=2, d=32, keep=120,
                       keep_dtype="f32", bf16=False,
                       cfg=dict(chunk_size=100, unit_size=32, n_repr=3, local_size=256, init_size=40, n_lookup=5,
                                hot_capacity=6, decay=0.1)),
    # the C1/C2 head geometry (d 128, GQA) at a small length, bf16-representable inputs
    "bf16_d128": dict(kind="gaussian", seed=11, scale=0.25, n=2048, tail=4, H=8, Hkv=2, d=128, keep=64,
                      keep_dtype="f16", bf16=True,
                      cfg=dict(chunk_size=256, unit_size=128, n_repr=4, local_size=512, init_size=128, n_lookup=4,
                               hot_capacity=6, decay=0.1)),
}


def bf16_round(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).bfloat16().float().numpy()


def make_inputs(c):
    """Deterministic inputs for case c (same function is used by the tests)."""
    if c["kind"] == "adapter":
        shape = O.ModelShape.make(n_heads=c["H"], head_dim=c["d"])
        ids = O.noise_ids(c["seed"], c["n"])
        q, k, v = O.adapter_batch(c["seed"], shape, ids)
        return q, k, v, ids
    n, s = c["n"], c["seed"]
    q = O.gaussian(s, 0, n, c["H"], c["d"]) * np.float32(c["scale"])
    k = O.gaussian(s, 1, n, c["Hkv"], c["d"]) * np.float32(c["scale"])
    v = O.gaussian(s, 2, n, c["Hkv"], c["d"])
    if c.get("bf16"):
        q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    return q, k, v, None


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def run_reference(c, q, k, v, ids):
    cfg = O.EngineConfig.make(**c["cfg"])
    inject = ids is None
    eng = R.RefEngine(cfg, c["H"], c["d"], c["d"], seed=c["seed"], inject=inject)
    if inject:
        eng.set_inputs(q, k, v)
    sched = O.encode_schedule(c["n"], c["cfg"]["chunk_size"], c["tail"])
    outs, step_ids = [], []
    fed = 0
    for si, b in enumerate(sched):
        out, rid = eng.step(b, decode=si >= len(sched) - c["tail"], ids=None if inject else ids[fed:fed + b])
        outs.append(out[0])
        step_ids.append(rid[0])
        fed += b
    out = np.concatenate(outs, 0)
    m = eng.metrics()
    units = [eng.unit_info(u) for u in range(m["units"])]
    return dict(out=out, step_ids=step_ids, metrics=m, trace=eng.trace(),
                units=[(u["start_abs"], u["size"], u["repr_abs"]) for u in units], sched=sched)


def main():
    assert R.available(), "needs the reference (oracle/_ref)"
    R.build()
    for name, c in CASES.items():
        q, k, v, ids = make_inputs(c)
        r = run_reference(c, q, k, v, ids)
        keep = r["out"][-c["keep"]:]
        keep = keep.astype(np.float16 if c["keep_dtype"] == "f16" else np.float32)
        flat_ids = np.array([i for s in r["step_ids"] for i in s], np.int64)
        offs = np.cumsum([0] + [len(s) for s in r["step_ids"]]).astype(np.int64)
        meta = dict(case=c, metrics=r["metrics"], units=r["units"], out_sha256=sha(r["out"]),
                    input_sha256=sha(q, k, v), n_steps=len(r["sched"]))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), meta=np.array(json.dumps(meta)), ids=flat_ids,
                            ids_offsets=offs, trace=np.array(r["trace"], np.int64).reshape(-1, 3),
                            out_tail=keep)
        print(f"{name}: {len(r['sched'])} steps, {r['metrics']['units']} units, "
              f"{sum(1 for s in r['step_ids'] if s)} lookups, out sha {meta['out_sha256'][:12]}")


if __name__ == "__main__":
    main()
