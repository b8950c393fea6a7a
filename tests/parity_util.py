"""Shared helpers for the GPU-vs-oracle parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np
import torch

from oracle import oracle as O


def bf16_round(x: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).bfloat16().float().numpy()


def gaussian_inputs(seed, n, H, Hkv, d, dv=None, scale=1.0, bf16=False):
    rng = np.random.default_rng(seed)
    dv = dv or d
    q = (rng.standard_normal((n, H, d)) * scale).astype(np.float32)
    k = (rng.standard_normal((n, Hkv, d)) * scale).astype(np.float32)
    v = rng.standard_normal((n, Hkv, dv)).astype(np.float32)
    if bf16:
        q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    return q, k, v


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def run_pair(cfg_kw, H, Hkv, d, q, k, v, schedule, decode_tail=0, dtype=torch.float32, oracle_threads=8,
             tc=True, finish=False, options=None):
    """Streams the same q/k/v through the GPU engine and the CPU oracle and
    returns per-step records for comparison."""
    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine

    dv = v.shape[2]
    ocfg = O.EngineConfig.make(**cfg_kw)
    oeng = O.OracleEngine(ocfg, O.ModelShape.make(n_heads=H, n_kv_heads=Hkv, head_dim=d, value_dim=dv),
                          n_threads=oracle_threads)
    geng = StreamEngine(EngineConfig.make(**cfg_kw), ModelShape.make(n_heads=H, n_kv_heads=Hkv, head_dim=d,
                                                                     value_dim=dv), dtype=dtype)
    if not tc:
        geng.set_option("tc_attention", 0)
    for key, val in (options or {}).items():
        geng.set_option(key, val)
    dev = torch.device("cuda")
    qt = torch.from_numpy(q).to(dev, dtype)
    kt = torch.from_numpy(k).to(dev, dtype)
    vt = torch.from_numpy(v).to(dev, dtype)
    recs = []
    fed = 0
    first_decode = len(schedule) - decode_tail
    for si, b in enumerate(schedule):
        dec = si >= first_decode
        r = oeng.step(q[fed:fed + b], k[fed:fed + b], v[fed:fed + b], decode=dec)
        g = geng.step(qt[fed:fed + b].contiguous(), kt[fed:fed + b].contiguous(), vt[fed:fed + b].contiguous(),
                      decode=dec)
        recs.append(dict(step=si, fed=fed, b=b, o_out=r.out, g_out=g.out.float().cpu().numpy(),
                         o_ids=r.retrieved_ids, g_ids=g.retrieved_ids))
        fed += b
    if finish:
        oeng.finish()
        geng.finish()
    return oeng, geng, recs


def compare_state(oeng, geng):
    om, gm = oeng.metrics(), geng.metrics()
    keys = ["units", "hot_units", "peak_hot_units", "hits", "misses", "loads", "evictions", "requested"]
    diffs = {k: (om[k], gm[k]) for k in keys if om[k] != gm[k]}
    n = om["units"]
    repr_bad = [u for u in range(n) if oeng.unit_info(u)["repr_abs"] != geng.unit_info(u)["repr_abs"]
                or oeng.unit_info(u)["start_abs"] != geng.unit_info(u)["start_abs"]
                or oeng.unit_info(u)["size"] != geng.unit_info(u)["size"]]
    return diffs, repr_bad
