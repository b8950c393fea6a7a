"""Command line for the B200 engine, mirroring the reference's `blockmem`
CLI (src/cli.cpp:396-540) for the subcommands on the hot path:

  bench  -- per-length streams, report rows as cmd_bench (cli.cpp:353-390):
            length, wall_ms, tokens_per_s, steps, units, peak_hot_units,
            peak_hot_bytes, hot_capacity, metrics{...} (metrics_to_json,
            cli.cpp:38-69)
  run    -- one stream with a decode tail (cmd_run, cli.cpp:169-199), optional
            engine trace export in the reference's text format
            (`step unit hit|miss`, cache_sim.hpp:181-184) and JSON report
  oracle-check -- the three self-checks of cmd_oracle_check (cli.cpp:239-351):
            the engine (on the GPU) against brute-force references restated
            from the reference's oracle.hpp (dense causal attention, windowed
            full-retrieval attention, batch representative scores), computed
            in float64 with torch on the same device; same JSON report
            (checks[{check, max_abs_err, mean_abs_err, compared, mismatches,
            tolerance, pass}], ok) and exit code (0 iff every check passes)

Engine flags mirror the EngineConfig field names; `--config file.json`
provides the base values (unknown keys rejected, config_io.hpp:16-40) and
explicit flags override it (cli.cpp:413-428). Inputs: the reference's
engine takes q/k/v from its synthetic adapter (q == k, adapter.hpp:63-65);
this engine takes explicit q/k/v, so the CLI feeds seeded Gaussian bf16
q/k/v of the model shape, generated on the device.

  python -m paper_2402_04617_b200.cli bench --lengths 32768,131072 --n_heads 32 --n_kv_heads 8 --head_dim 128
"""
from __future__ import annotations

import argparse
import json
import sys
import time

from ._lib import LOOKUP_MODES, POSITION_MODES, ConfigError

CONFIG_KEYS = ("chunk_size", "unit_size", "n_repr", "local_size", "init_size", "n_lookup", "hot_capacity", "decay",
               "lookup_mode", "position_mode")
LOOKUP_NAMES = {v: k for k, v in LOOKUP_MODES.items()}
POSITION_NAMES = {v: k for k, v in POSITION_MODES.items()}


def config_from_json(obj) -> dict:
    """engine_config_from_json (config_io.hpp:16-40): unknown keys rejected."""
    if not isinstance(obj, dict):
        raise ConfigError(-1, "engine config: expected a JSON object")
    for k in obj:
        if k not in CONFIG_KEYS:
            raise ConfigError(-1, f"engine config: unknown key '{k}'")
    out = dict(obj)
    for k, table in (("lookup_mode", LOOKUP_MODES), ("position_mode", POSITION_MODES)):
        if k in out and isinstance(out[k], str):
            if out[k] not in table:
                raise ConfigError(-1, f"engine config: unknown {k} '{out[k]}'")
            out[k] = table[out[k]]
    return out


def config_to_json(cfg) -> dict:
    """engine_config_to_json (config_io.hpp:42-55)."""
    d = cfg.as_dict()
    d["lookup_mode"] = LOOKUP_NAMES.get(d["lookup_mode"], d["lookup_mode"])
    d["position_mode"] = POSITION_NAMES.get(d["position_mode"], d["position_mode"])
    return d


def metrics_to_json(eng, n_layers: int, tokens: int, steps: int, wall_ms: float) -> dict:
    """metrics_to_json (cli.cpp:38-69). timings_ms: PhaseTimings
    (engine.hpp:43-49) as device time per phase (infllm_phase_timings; the
    phases overlap on the engine's streams) plus the stream's wall time; the
    adapter phase does not exist (q/k/v are inputs). invariant_checks /
    _violations: check_softmax on the device + check_conservation
    (engine.hpp:361-383)."""
    layers = []
    for li in range(n_layers):
        m = eng.metrics(li)
        req = m["requested"]
        layers.append({
            "units": m["units"], "hot_units": m["hot_units"], "peak_hot_units": m["peak_hot_units"],
            "peak_hot_bytes": m["peak_hot_bytes"], "hits": m["hits"], "misses": m["misses"], "loads": m["loads"],
            "evictions": m["evictions"], "requested": req, "hit_rate": m["hits"] / req if req else 0.0,
            "miss_rate": m["misses"] / req if req else 0.0,
        })
    ph = eng.phase_timings()
    checks, violations = eng.invariants()
    return {"tokens": tokens, "steps": steps, "invariant_checks": checks, "invariant_violations": violations,
            "timings_ms": {"adapter": 0.0, "lookup": ph["lookup"], "attend": ph["attend"], "score": ph["score"],
                           "evict": ph["evict"], "wall": wall_ms}, "layers": layers}


def _engine(args):
    import torch

    from . import EngineConfig, ModelShape, StreamEngine

    base = {}
    if args.config:
        with open(args.config) as f:
            base = config_from_json(json.load(f))
    for k in CONFIG_KEYS:
        v = getattr(args, k, None)
        if v is not None:
            base[k] = LOOKUP_MODES.get(v, v) if k == "lookup_mode" else POSITION_MODES.get(v, v) \
                if k == "position_mode" else v
    cfg = EngineConfig.make(**base)
    shape = ModelShape.make(n_heads=args.n_heads, n_kv_heads=args.n_kv_heads, head_dim=args.head_dim,
                            n_layers=args.n_layers)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    eng = StreamEngine(cfg, shape, dtype=dtype, device=args.device)
    if args.host_tier_slots:
        eng.set_option("host_tier_slots", args.host_tier_slots)
    return eng, cfg, shape, dtype


def _inputs(args, n, seed, dtype):
    import torch

    g = torch.Generator(device=f"cuda:{args.device}")
    g.manual_seed(seed)
    dev = f"cuda:{args.device}"
    kv = args.n_kv_heads or args.n_heads
    q = torch.randn((n, args.n_heads, args.head_dim), generator=g, device=dev).to(dtype)
    k = torch.randn((n, kv, args.head_dim), generator=g, device=dev).to(dtype)
    v = torch.randn((n, kv, args.head_dim), generator=g, device=dev).to(dtype)
    return q, k, v


def _stream(eng, args, q, k, v, decode_tail=0):
    """feed (engine.hpp:106-112) of every layer, then decode_tail decode steps; returns (wall_ms, steps)."""
    import torch

    n = q.shape[0]
    n_pre = n - decode_tail
    eng.profile_begin(True)  # per-phase device timings (timings_ms)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for li in range(args.n_layers):
        if n_pre > 0:
            eng.encode_stream(q[:n_pre], k[:n_pre], v[:n_pre], layer=li)
    for i in range(n_pre, n):
        for li in range(args.n_layers):
            eng.decode_step(q[i:i + 1], k[i:i + 1], v[i:i + 1], layer=li)
    eng.finish()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    c = int(eng.config.chunk_size)
    return wall, (n_pre + c - 1) // c + decode_tail


def cmd_bench(args) -> dict:
    rows = []
    cfg_json = None
    for i, length in enumerate(args.lengths):
        eng, cfg, shape, dtype = _engine(args)
        cfg_json = config_to_json(cfg)
        eng.reserve(length)
        q, k, v = _inputs(args, length, args.seed + i, dtype)
        if args.warmup:
            _stream(eng, args, q, k, v)
            eng.reset()
        wall, steps = _stream(eng, args, q, k, v)
        per = [eng.metrics(li) for li in range(args.n_layers)]
        rows.append({
            "length": length, "wall_ms": wall, "tokens_per_s": 1000.0 * length / wall if wall > 0 else 0.0,
            "steps": steps, "units": max(m["units"] for m in per),
            "peak_hot_units": max(m["peak_hot_units"] for m in per),
            "peak_hot_bytes": max(m["peak_hot_bytes"] for m in per), "hot_capacity": int(cfg.hot_capacity),
            "metrics": metrics_to_json(eng, args.n_layers, length, steps, wall),
        })
        eng.close()
    report = {"config": cfg_json, "seed": args.seed, "rows": rows}
    _write(args.out, report)
    return report


def cmd_run(args) -> dict:
    eng, cfg, shape, dtype = _engine(args)
    eng.reserve(args.length)
    q, k, v = _inputs(args, args.length, args.seed, dtype)
    wall, steps = _stream(eng, args, q, k, v, decode_tail=args.decode_tail)
    report = {"config": config_to_json(cfg), "seed": args.seed,
              "metrics": metrics_to_json(eng, args.n_layers, args.length, steps, wall)}
    if args.trace_out:  # export_engine_trace (cli.cpp:78-84), format cache_sim.hpp:181-184
        with open(args.trace_out, "w") as f:
            for li in range(args.n_layers):
                for step, unit, hit in eng.trace(li):
                    f.write(f"{step} {unit} {'hit' if hit else 'miss'}\n")
    _write(args.out, report)
    eng.close()
    return report


# ---------------------------------------------------------------- oracle-check
def _schedule(length, chunk, tail):
    """encode_schedule (cli.cpp:133-142)."""
    sched, left = [], length - tail
    while left > 0:
        sched.append(min(chunk, left))
        left -= sched[-1]
    return sched + [1] * tail


def _rope(x, pos):
    """detail::rotate (oracle.hpp:30-45 / rotary.hpp:15-51) in float64: pairs (2a, 2a+1),
    angle pos * 10000^(-2a/d); x [..., n, d], pos [n] (or a scalar)."""
    import torch

    d = x.shape[-1]
    a = torch.arange(d // 2, device=x.device, dtype=torch.float64)
    theta = torch.pow(torch.tensor(10000.0, dtype=torch.float64, device=x.device), -2.0 * a / d)
    pos = torch.as_tensor(pos, dtype=torch.float64, device=x.device)
    ang = pos.reshape(-1, 1) * theta if pos.dim() else pos * theta
    c, s = torch.cos(ang), torch.sin(ang)
    y = x.clone()
    x0, x1 = x[..., 0:2 * (d // 2):2], x[..., 1:2 * (d // 2):2]
    y[..., 0:2 * (d // 2):2] = x0 * c - x1 * s
    y[..., 1:2 * (d // 2):2] = x0 * s + x1 * c
    return y


def _report(name, got, want, tol):
    import torch

    err = (got.double() - want).abs()
    return {"check": name, "max_abs_err": float(err.max()), "mean_abs_err": float(err.mean()),
            "compared": int(err.numel()), "mismatches": int((err > tol).sum()), "tolerance": tol,
            "pass": bool((err > tol).sum() == 0)}


def _run_collect(eng, q, k, v, sched, tail):
    """run_engine_collect (cli.cpp:89-119) with explicit q/k/v: stacked outputs."""
    import torch

    outs, fed = [], 0
    first_decode = len(sched) - tail
    for i, b in enumerate(sched):
        sl = slice(fed, fed + b)
        if i >= first_decode:
            outs.append(eng.decode_step(q[sl].contiguous(), k[sl].contiguous(), v[sl].contiguous()))
        else:
            outs.append(eng.encode_chunk(q[sl].contiguous(), k[sl].contiguous(), v[sl].contiguous()))
        fed += b
    torch.cuda.synchronize()
    return torch.cat(outs, 0)


def cmd_oracle_check(args) -> dict:
    import torch

    from . import EngineConfig, ModelShape, ScoreAccumulator, StreamEngine

    base = {}
    if args.config:
        with open(args.config) as f:
            base = config_from_json(json.load(f))
    for kname in CONFIG_KEYS:
        val = getattr(args, kname, None)
        if val is not None:
            base[kname] = LOOKUP_MODES.get(val, val) if kname == "lookup_mode" else POSITION_MODES.get(val, val) \
                if kname == "position_mode" else val
    cfg0 = EngineConfig.make(**base)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    n, H, d = args.length, args.n_heads, args.head_dim
    Hkv = args.n_kv_heads or H
    rep_h = H // Hkv
    shape = ModelShape.make(n_heads=H, n_kv_heads=Hkv, head_dim=d)
    dev = torch.device("cuda", args.device)
    g = torch.Generator(device=dev)
    g.manual_seed(args.seed)
    q = torch.randn((n, H, d), generator=g, device=dev).to(dtype)
    k = torch.randn((n, Hkv, d), generator=g, device=dev).to(dtype)
    v = torch.randn((n, Hkv, d), generator=g, device=dev).to(dtype)
    q64, k64, v64 = q.double(), k.double(), v.double()
    tail = min(32, n // 8)
    tol_attn = 1e-5 if dtype == torch.float32 else 2e-2
    scale = 1.0 / d ** 0.5
    kh = k64.repeat_interleave(rep_h, dim=1)  # key / value of each query head's group
    vh = v64.repeat_interleave(rep_h, dim=1)
    pos = torch.arange(n, device=dev)
    checks = []

    def softmax_pv(logits, vals):  # detail::softmax_inplace (oracle.hpp:47-57), float64
        w = torch.softmax(logits, dim=-1)
        return torch.einsum("hij,hjd->hid", w, vals)

    # 1. degenerate configuration vs the dense causal oracle (cli.cpp:248-271, oracle.hpp:64-97)
    c = dict(cfg0.as_dict())
    c["local_size"] = max(c["local_size"], n)
    c["position_mode"] = POSITION_MODES["absolute"]
    sched = _schedule(n, c["chunk_size"], tail)
    eng = StreamEngine(EngineConfig.make(**c), shape, dtype=dtype, device=args.device)
    got = _run_collect(eng, q, k, v, sched, tail)
    eng.close()
    qa = _rope(q64.transpose(0, 1), pos)  # [H][n][d]
    ka = _rope(kh.transpose(0, 1), pos)
    logits = torch.einsum("hid,hjd->hij", qa, ka) * scale
    logits.masked_fill_(torch.triu(torch.ones(n, n, dtype=torch.bool, device=dev), 1), float("-inf"))
    want = softmax_pv(logits, vh.transpose(0, 1)).transpose(0, 1)
    checks.append(_report("degenerate_vs_dense", got, want, tol_attn))
    del logits, qa, ka

    # 2. full-retrieval configuration vs the windowed clamped oracle (cli.cpp:274-299, oracle.hpp:103-168)
    c = dict(cfg0.as_dict())
    c["position_mode"] = POSITION_MODES["clamped"]
    c["lookup_mode"] = LOOKUP_MODES["encode_and_decode"]
    c["n_lookup"] = n // c["unit_size"] + 2
    c["hot_capacity"] = max(c["hot_capacity"], c["n_lookup"])
    sched = _schedule(n, c["chunk_size"], tail)
    eng = StreamEngine(EngineConfig.make(**c), shape, dtype=dtype, device=args.device)
    got = _run_collect(eng, q, k, v, sched, tail)
    eng.close()
    L, I, U = c["local_size"], c["init_size"], c["unit_size"]
    q_abs = _rope(q64.transpose(0, 1), pos)
    q_cap = _rope(q64.transpose(0, 1), torch.tensor(float(L), device=dev))
    k_rot = _rope(kh.transpose(0, 1), pos)
    k_raw = kh.transpose(0, 1)
    want = torch.zeros((H, n, d), dtype=torch.float64, device=dev)
    fed = 0
    for b in sched:
        local_begin = max(0, fed - L)
        init_len = min(I, local_begin)
        evicted = max(0, local_begin - I)
        packed = evicted - evicted % U
        vis = torch.cat([torch.arange(0, init_len), torch.arange(I, I + packed), torch.arange(local_begin, fed + b)]).to(dev)
        rows = torch.arange(fed, fed + b, device=dev)
        dist = rows.view(-1, 1) - vis.view(1, -1)
        cap = (vis.view(1, -1) < local_begin) | (dist > L)
        s_cap = torch.einsum("hid,hjd->hij", q_cap[:, rows], k_raw[:, vis])
        s_abs = torch.einsum("hid,hjd->hij", q_abs[:, rows], k_rot[:, vis])
        logits = torch.where(cap, s_cap, s_abs) * scale
        logits.masked_fill_(dist < 0, float("-inf"))  # causal batch prefix
        want[:, fed:fed + b] = softmax_pv(logits, vh.transpose(0, 1)[:, vis])
        fed += b
    checks.append(_report("full_retrieval_vs_windowed", got, want.transpose(0, 1), tol_attn))

    # 3. incremental representative scores vs the batch definition (cli.cpp:301-342, oracle.hpp:173-184)
    L = int(cfg0.local_size)
    acc = ScoreAccumulator(L, H, Hkv, d, dtype)
    fed = 0
    while fed < n:
        b = min(int(cfg0.chunk_size), n - fed)
        acc.accumulate(q[fed:fed + b].contiguous(), fed, k[:fed + b].contiguous())
        fed += b
    got_r = torch.from_numpy(acc.finalize_front(n)).to(dev)
    acc.close()
    dots = torch.einsum("ihd,mhd->im", q64, kh)  # [query i][key m] summed over heads
    band = (pos.view(-1, 1) > pos.view(1, -1)) & (pos.view(-1, 1) <= pos.view(1, -1) + L)
    want_r = (dots * band).sum(0) / L
    checks.append(_report("repr_scores_incremental_vs_batch", got_r, want_r, 1e-6))

    report = {"seed": args.seed, "length": n, "config": config_to_json(cfg0), "dtype": args.dtype,
              "inputs": "seeded N(0,1) q/k/v on the device (the engine takes explicit q/k/v; SURVEY M7)",
              "checks": checks, "ok": all(ch["pass"] for ch in checks)}
    _write(args.out, report)
    return report


def _write(path, obj):
    if path:
        with open(path, "w") as f:
            f.write(json.dumps(obj, indent=2) + "\n")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="infllm-b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p):
        p.add_argument("--config", default="", help="engine config JSON file")
        for k in ("chunk_size", "unit_size", "n_repr", "local_size", "init_size", "n_lookup", "hot_capacity"):
            p.add_argument(f"--{k}", type=int)
        p.add_argument("--decay", type=float)
        p.add_argument("--lookup_mode", choices=sorted(LOOKUP_MODES))
        p.add_argument("--position_mode", choices=sorted(POSITION_MODES))
        p.add_argument("--n_layers", type=int, default=1)
        p.add_argument("--n_heads", type=int, default=32)
        p.add_argument("--n_kv_heads", type=int, default=8)
        p.add_argument("--head_dim", type=int, default=128)
        p.add_argument("--dtype", choices=("bf16", "f32"), default="bf16")
        p.add_argument("--device", type=int, default=0)
        p.add_argument("--host_tier_slots", type=int, default=0)
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--out", default="", help="JSON report path")

    b = sub.add_parser("bench", help="per-length streams (cmd_bench)")
    common(b)
    b.add_argument("--lengths", type=lambda s: [int(x) for x in s.split(",")], default=[8192, 32768])
    b.add_argument("--warmup", type=int, default=1, help="1: one untimed stream first (graph capture)")
    r = sub.add_parser("run", help="one stream with a decode tail (cmd_run)")
    common(r)
    r.add_argument("--length", type=int, default=8192)
    r.add_argument("--decode_tail", type=int, default=32)
    r.add_argument("--trace-out", dest="trace_out", default="")
    oc = sub.add_parser("oracle-check", help="compare the engine to brute-force references (cmd_oracle_check)")
    common(oc)
    oc.set_defaults(n_heads=4, n_kv_heads=2, head_dim=64, dtype="f32")
    oc.add_argument("--length", type=int, default=1024)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        if args.cmd == "oracle-check":
            rep = cmd_oracle_check(args)
            for ch in rep["checks"]:  # cli.cpp:511-516
                print(f"{ch['check']}: max_abs_err={ch['max_abs_err']:.3g} {'ok' if ch['pass'] else 'FAIL'}")
            return 0 if rep["ok"] else 1
        rep = cmd_bench(args) if args.cmd == "bench" else cmd_run(args)
    except Exception as ex:  # cli.cpp:533-538: one-line message, exit code 1
        print(f"error: {ex}", file=sys.stderr)
        return 1
    if args.cmd == "bench":
        for row in rep["rows"]:
            print(f"length={row['length']} tokens_per_s={row['tokens_per_s']:.1f} units={row['units']} "
                  f"peak_hot_units={row['peak_hot_units']}")
    else:
        m = rep["metrics"]
        print(f"tokens={m['tokens']} steps={m['steps']} units={m['layers'][0]['units']} "
              f"hit_rate={m['layers'][0]['hit_rate']:.3f}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
