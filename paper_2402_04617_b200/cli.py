"""Command line for the B200 engine, mirroring the reference's `blockmem`
CLI (src/cli.cpp:396-540) for the subcommands on the hot path:

  bench  -- per-length streams, report rows as cmd_bench (cli.cpp:353-390):
            length, wall_ms, tokens_per_s, steps, units, peak_hot_units,
            peak_hot_bytes, hot_capacity, metrics{...} (metrics_to_json,
            cli.cpp:38-69)
  run    -- one stream with a decode tail (cmd_run, cli.cpp:169-199), optional
            engine trace export in the reference's text format
            (`step unit hit|miss`, cache_sim.hpp:181-184) and JSON report

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
    """metrics_to_json (cli.cpp:38-69). The engine runs whole steps on the
    device without per-phase host timers, so timings_ms reports the stream's
    wall time; invariant counters are the reference's CPU self-checks and
    have no device counterpart (null)."""
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
    return {"tokens": tokens, "steps": steps, "invariant_checks": None, "invariant_violations": None,
            "timings_ms": {"stream": wall_ms}, "layers": layers}


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
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
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
