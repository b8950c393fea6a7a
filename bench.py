#!/usr/bin/env python
"""bench.py — InfLLM layer prefill tokens/s @128K context, Llama-3-8B heads.

Workload (BASELINE.json configs[2], the metric's config): one InfLLM layer,
32 query / 8 KV heads, d = 128, bf16, chunked prefill of a 131072-token
stream (chunk 512, unit 128, r_k 4, k_m 16, init 128, local window 4096,
hot capacity 32, decay 0.1). One bench "step" = the whole 128K-token stream
(256 chunk steps: lookup, attention, LRU, scoring, packing) through a freshly
reset engine. Inputs: synthetic N(0,1) q/k/v (seeded), resident in HBM
(1.5 GB > L2, so no flush is needed between steps).

--gpus N (torchrun): ONE 128K stream KV-group sharded over the N GPUs
(BASELINE configs[2]: rank r owns KV groups [r 8/N, (r+1) 8/N) and their
query heads; the library's NCCL communicator exchanges the fp64 score
partials every step (C-1) and all-gathers the outputs to every head (C-2);
strong scaling, value = that stream's tokens/s). The same ranks also time N
independent unsharded streams (one per GPU, no collective) and report it as
`replicas` (weak scaling) beside the headline.
--impl reference: the reference algorithm on the host CPU (the oracle port,
pinned bit-exact to the reference engine), rank 0 only.
"""
from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(chunk_size=512, unit_size=128, n_repr=4, local_size=4096, init_size=128, n_lookup=16, hot_capacity=32,
           decay=0.1, lookup_mode=0, position_mode=0)
SHAPE = dict(n_heads=32, n_kv_heads=8, head_dim=128)
N_TOKENS = 131072
METRIC = "InfLLM layer prefill tokens/s @128K ctx (Llama-3-8B heads), 1/2/4/8 B200"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return dict(hbm=j.get("hbm_gbs", 6650.0), bf16=j.get("bf16_tflops", 1590.0),
                    bf16_sust=j.get("bf16_tflops_sustained", 1400.0), src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sust=1400.0, src="fallback")


def stream_schedule(n, cfg):
    """Host replay of the stream arithmetic (engine.hpp:242-346): per chunk
    step (l_x, n_ctx keys before the chunk, units U at lookup, n_sel)."""
    steps = []
    fed = local_start = init_len = units = pend = 0
    C, L, I, bs, km = cfg["chunk_size"], cfg["local_size"], cfg["init_size"], cfg["unit_size"], cfg["n_lookup"]
    while fed < n:
        lx = min(C, n - fed)
        n_sel = min(km, units) if (km > 0 and units > 0) else 0
        local_len = fed - local_start
        steps.append(dict(lx=lx, n_ctx=init_len + n_sel * bs + local_len, units=units, n_sel=n_sel))
        overflow = max(0, local_len + lx - L)
        to_init = min(max(I - local_start, 0), overflow)
        pend += overflow - to_init
        units += pend // bs
        pend %= bs
        local_start += overflow
        init_len += to_init
        fed += lx
    return steps


def attention_flops(steps, H, d):
    """QK^T + PV over attended pairs only: 4 d H [l_x W + l_x(l_x+1)/2]."""
    return sum(4.0 * d * H * (s["lx"] * s["n_ctx"] + s["lx"] * (s["lx"] + 1) / 2) for s in steps)


def lookup_bytes(steps, cfg, Hkv, d, H, elem=2):
    """repr-index scan + chunk queries read."""
    return sum(s["units"] * cfg["n_repr"] * Hkv * d * elem + s["lx"] * H * d * elem for s in steps if s["n_sel"] > 0)


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs a moment to start: only rows taken after this point
            # (inside the timed region) are summarised
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0:
                time.sleep(0.01)
            self.first = len(self.rows)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        self.rows = self.rows[getattr(self, "first", 0):]
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        busy = [r for r in self.rows if (num(r[6]) or 0) > 0] or self.rows
        sm = [num(r[0]) for r in busy if num(r[0]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": num(self.rows[0][1]),
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------- reference arm
def cpu_sample(threads, steps=2, warm=8192, seed=0):
    """The reference algorithm (oracle port, bit-exact to the reference engine
    compiled here) on host cores: warm-start 8192 tokens of C2 through the
    window/packing bookkeeping, then time `steps` full steady-state chunk
    steps (lookup + attend + score + evict, PhaseTimings phases)."""
    from oracle import oracle as O

    O.build()
    H, Hkv, d = SHAPE["n_heads"], SHAPE["n_kv_heads"], SHAPE["head_dim"]
    C = CFG["chunk_size"]
    rng = np.random.default_rng(seed)
    n = warm + steps * C

    def bf(x):
        import torch
        return torch.from_numpy(x).bfloat16().float().numpy()

    q = bf(rng.standard_normal((n, H, d), dtype=np.float32))
    k = bf(rng.standard_normal((n, Hkv, d), dtype=np.float32))
    v = bf(rng.standard_normal((n, Hkv, d), dtype=np.float32))
    eng = O.OracleEngine(O.EngineConfig.make(**CFG), O.ModelShape.make(n_heads=H, n_kv_heads=Hkv, head_dim=d),
                         n_threads=threads)
    eng.warm_start(q[:warm], k[:warm], v[:warm])
    t0 = time.perf_counter()
    for s in range(steps):
        a = warm + s * C
        eng.step(q[a:a + C], k[a:a + C], v[a:a + C])
    dt = time.perf_counter() - t0
    return dict(value=steps * C / dt, unit="tokens/s", cores=threads, kind="port",
                sample=f"{steps} steady-state C2 chunk steps ({steps * C} tokens, window {CFG['init_size']}+"
                       f"{CFG['n_lookup']}x{CFG['unit_size']}+{CFG['local_size']}) after an {warm}-token warm start; "
                       f"oracle port of the reference engine (bit-exact pinned), {threads} threads over heads",
                seconds=dt)


C0_CFG = dict(chunk_size=128, unit_size=128, n_repr=4, local_size=512, init_size=64, n_lookup=4, hot_capacity=32,
              decay=0.1)


def cpu_reference_c0(n=8192, seed=0):
    """The reference itself (oracle/_ref: StreamEngine<float> compiled here from
    /root/reference's headers, prebuilt by build() and shipped with the repo)
    beside the oracle port on BASELINE configs[0] (C0: 1 head, d 64, 8K tokens,
    the reference's own synthetic adapter), both single-threaded: tokens/s of
    each and whether their outputs are bitwise equal. This calibrates the port
    that stands in for the reference at C2, where the reference has no
    warm-start path and a steady-state step would need minutes of ramp-up."""
    from oracle import oracle as O
    from oracle import ref as R

    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libblockmem_ref.so")):
        return {"available": False, "why": "oracle/_ref not built (needs /root/reference at build time)"}
    shape = O.ModelShape.make(n_heads=1, head_dim=64)
    ids = O.noise_ids(seed, n)
    q, k, v = O.adapter_batch(seed, shape, ids)
    sched = O.encode_schedule(n, C0_CFG["chunk_size"], 32)
    t0 = time.perf_counter()
    re = R.RefEngine(O.EngineConfig.make(**C0_CFG), 1, 64)
    re.set_inputs(q, k, v)
    ro = [re.step(b, decode=i >= len(sched) - 32)[0][0] for i, b in enumerate(sched)]
    t_ref = time.perf_counter() - t0
    t0 = time.perf_counter()
    oe = O.OracleEngine(O.EngineConfig.make(**C0_CFG), shape, n_threads=1)
    po, fed = [], 0
    for i, b in enumerate(sched):
        po.append(oe.step(q[fed:fed + b], k[fed:fed + b], v[fed:fed + b], decode=i >= len(sched) - 32).out)
        fed += b
    t_port = time.perf_counter() - t0
    return {"available": True, "workload": "C0 (configs[0]): 1 head, d 64, 8192-token adapter stream, chunk 128, "
                                           "window 512, k_m 4, 32 decode steps",
            "reference_tokens_per_s": n / t_ref, "port_tokens_per_s": n / t_port, "cores": 1,
            "outputs_bitwise_equal": bool(np.array_equal(np.concatenate(ro), np.concatenate(po)))}


def run_reference(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_sample(threads, steps=1, seed=i)
        if i >= args.warmup:
            vals.append(r)
    v = statistics.mean(x["value"] for x in vals)
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * CFG["chunk_size"] / v, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "C2: Llama-3-8B heads (32q/8kv, d128), 128K ctx chunked prefill, k_m 16, "
                                   "l_L 4096, l_I 128, chunk 512; CPU sample of steady-state chunk steps"},
            "cpu_baseline": {k: vals[-1][k] for k in ("unit", "cores", "kind", "sample")} | {"value": v},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    try:
        line["reference_c0"] = cpu_reference_c0()
    except Exception as ex:  # reported, not fatal
        line["reference_c0"] = {"available": False, "why": str(ex)}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- B200 arm
def run_b200(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    H, Hkv, d = SHAPE["n_heads"], SHAPE["n_kv_heads"], SHAPE["head_dim"]
    n, C = args.tokens, CFG["chunk_size"]
    g = torch.Generator(device=dev)
    g.manual_seed(1234)  # every rank draws the same full stream and keeps its shard
    Q = torch.randn((n, H, d), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    K = torch.randn((n, Hkv, d), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    V = torch.randn((n, Hkv, d), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    OUT = torch.empty((n, H, d), device=dev, dtype=torch.bfloat16)
    sharded = world > 1
    if sharded:
        from paper_2402_04617_b200.shard import shard_range

        g0, gc = shard_range(Hkv, rank, world)
        rep_h = H // Hkv
        QF, KF, VF = Q, K, V
        Q = QF[:, g0 * rep_h:(g0 + gc) * rep_h].contiguous()
        K, V = KF[:, g0:g0 + gc].contiguous(), VF[:, g0:g0 + gc].contiguous()
        eng = StreamEngine(EngineConfig.make(**CFG), ModelShape.make(**SHAPE), dtype=torch.bfloat16,
                           device=local_rank, kv_group_begin=g0, kv_group_count=gc)
        eng.set_comm(rank, world)
        eng.set_option("gather_output", 1)  # OUT holds every head on every rank (C-2)
    else:
        eng = StreamEngine(EngineConfig.make(**CFG), ModelShape.make(**SHAPE), dtype=torch.bfloat16,
                           device=local_rank)
    if args.no_tc:
        eng.set_option("tc_attention", 0)
    eng.reserve(n)
    stream = torch.cuda.current_stream(dev)

    def one_stream():
        eng.reset()
        eng.encode_stream(Q, K, V, out=OUT)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        one_stream()
    barrier()
    launches0 = eng.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            one_stream()
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    launches = eng.kernel_launches() - launches0
    # per-launch device times of the dominant kernel (attention) and of the
    # lookup: CUDA events recorded around every such launch, on the stream it
    # runs on, over a second pass of the same K streams. The event nodes
    # perturb the two-stream pipeline (~13% per stream), so the headline
    # region above carries none.
    eng.profile_begin(True)
    one_stream()  # captures the profiled graph variant
    barrier()
    eng.profile_begin(True)
    for _ in range(args.steps):
        one_stream()
    barrier()
    prof = eng.profile_read()
    eng.profile_begin(False)
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    value = n * args.steps / (ms / 1000.0)  # one stream (sharded over the ranks when world > 1)
    replicas = None
    if sharded:  # N independent unsharded streams, one per GPU (weak scaling, no collective)
        eng.set_option("gather_output", 0)
        rep_eng = StreamEngine(EngineConfig.make(**CFG), ModelShape.make(**SHAPE), dtype=torch.bfloat16,
                               device=local_rank)
        rep_eng.reserve(n)

        def rep_stream():
            rep_eng.reset()
            rep_eng.encode_stream(QF, KF, VF, out=OUT)

        for _ in range(args.warmup):
            rep_stream()
        barrier()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        for _ in range(args.steps):
            rep_stream()
        r1.record(stream)
        barrier()
        rms = torch.tensor([r0.elapsed_time(r1)], device=dev)
        dist.all_reduce(rms, op=dist.ReduceOp.MAX)
        replicas = {"value": world * n * args.steps / (float(rms.item()) / 1000.0), "unit": "tokens/s",
                    "scaling": "weak", "ms_per_step": float(rms.item()) / args.steps,
                    "what": f"{world} independent unsharded 128K streams, one per GPU, no collective"}
        rep_eng.close()

    # end-to-end through the C-ABI with HOST buffers: per chunk H2D of q/k/v
    # from pinned memory and D2H of the attention output, pipelined on copy
    # streams (inside the timed region)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(eng, Q, K, V, n, C, dev, args, world)

    steps = stream_schedule(n, CFG)
    flops = attention_flops(steps, H, d) * (Q.shape[1] / H)  # this rank's query heads
    peaks = load_peaks()
    attn_ms = prof["attn_ms"] / max(1, args.steps)
    achieved = flops / (attn_ms / 1000.0) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "attn_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                traffic = json.load(f).get("bytes_per_launch")
        except Exception:
            traffic = None
    lk_bytes = lookup_bytes(steps, CFG, Hkv, d, H)
    lk_ms = prof["lookup_ms"] / max(1, args.steps)
    iso = isolated_kernels(eng, steps, H, Hkv, d, dev) if (rank == 0 and not sharded) else {}
    extra = other_configs(Q, K, V, dev) if (rank == 0 and not args.no_extra and not sharded) else {}

    if rank == 0:
        cpu = cpu_all = cpu_c0 = None
        if world == 1 and not args.no_cpu:
            # the reference runs one stream per core (no intra-stream threads, proj/CMakeLists.txt;
            # parallel.hpp only spreads trials): the primary baseline is one core per stream
            try:
                cpu = cpu_sample(1, steps=1)
                cpu.pop("seconds", None)
            except Exception as ex:  # reported, not fatal
                cpu = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "port", "sample": f"failed: {ex}"}
            try:
                cpu_all = cpu_sample(os.cpu_count() or 1, steps=2)
                cpu_all.pop("seconds", None)
            except Exception as ex:
                cpu_all = {"value": None, "sample": f"failed: {ex}"}
            try:
                cpu_c0 = cpu_reference_c0()
            except Exception as ex:
                cpu_c0 = {"available": False, "why": str(ex)}
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "C2: Llama-3-8B heads (32q/8kv, d128), 131072-token chunked prefill of one "
                                   "InfLLM layer per GPU (chunk 512, unit 128, r_k 4, k_m 16, init 128, local 4096, "
                                   "hot 32); step = whole stream",
                       "tokens_per_step_per_gpu": n, "l2": "inputs 1.5 GB > L2 (no flush needed)",
                       "parallelism": (f"kv-group sharded over {world} GPUs (NCCL: per-step fp64 score partials "
                                       f"C-1, output all-gather C-2)") if sharded else "1 stream"},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peaks["bf16"], "unit": "TFLOP/s",
                         "frac": achieved / peaks["bf16"], "traffic": traffic,
                         # the kernel runs inside a 17 ms stream of back-to-back launches: the
                         # sustained matmul figure is the like-for-like denominator; frac keeps the
                         # burst one (the stricter of the two)
                         "frac_sustained": achieved / peaks["bf16_sust"],
                         "kernel": "attention (K3)", "flops_per_stream": flops,
                         "avg_launch_ms": attn_ms / len(steps), "launches_per_stream": len(steps),
                         "share_of_step": (attn_ms / (ms / args.steps)) if ms > 0 else None,
                         "timing": "CUDA events around every attention launch on its stream, over a second pass "
                                   "of the same K streams (event nodes perturb the pipeline, so the headline "
                                   "region has none); consecutive launches alternate between two streams and "
                                   "overlap at the handoff, so the event time is the union of the launches' "
                                   "[begin, end] intervals; achieved = algorithmic QK^T+PV flops / event time",
                         "peak_src": peaks["src"] + " burst bf16 (sustained %.1f)" % peaks["bf16_sust"],
                         "lookup": {"in_stream_gbs": lk_bytes / (lk_ms / 1000.0) / 1e9 if lk_ms > 0 else None,
                                    "peak_gbs": peaks["hbm"], "bytes_per_stream": lk_bytes,
                                    "in_stream_ms_per_stream": lk_ms,
                                    "note": "in-stream: the lookup shares the GPU with the attention of the previous "
                                            "step (20 free SMs); isolated: the last step's lookup launched alone as a "
                                            "one-token step launches it (whole GPU, graph-replayed); "
                                            "pipeline_grid_alone: the chunk step's grid launched alone"} | iso},
            "cpu_baseline": cpu,
            "cpu_baseline_all_cores": cpu_all,
            "cpu_reference_c0": cpu_c0,
            "e2e": e2e,
            "replicas": replicas,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "other_configs": extra,
        }
        print(json.dumps(line), flush=True)


def isolated_kernels(eng, steps, H, Hkv, d, dev):
    """Steady-state per-launch times of the lookup (relevance scan + exact top-k)
    and of the attention re-launched alone with the last chunk step's
    parameters (infllm_debug_kernel_bench; run after the timed work, it
    disturbs the engine state), plus the standalone lookup at the C3 index
    size (U = 8159 units, 1M-token stream) where the scan is HBM-sized."""
    import ctypes as C

    import torch

    from paper_2402_04617_b200 import _lib

    out = {}
    try:
        last = steps[-1]
        us = C.c_double()
        _lib.check(_lib.lib().infllm_debug_kernel_bench(eng.h, 1, 50, C.byref(us)))
        b = last["units"] * CFG["n_repr"] * Hkv * d * 2 + last["lx"] * H * d * 2
        out["isolated_us"] = us.value  # as a one-token step launches it (whole GPU)
        out["isolated_gbs"] = b / (us.value * 1e-6) / 1e9
        out["isolated_units"] = last["units"]
        _lib.check(_lib.lib().infllm_debug_kernel_bench(eng.h, 11, 50, C.byref(us)))
        out["pipeline_grid_alone_us"] = us.value  # the chunk step's few-fat-blocks grid, launched alone
        # standalone lookups on random bf16 indices, timed as CUDA-graph replays
        # (device time, no host gaps): the C3 index (8159 units, 1M-token stream)
        # and a 131072-unit index where the relevance scan is HBM-sized
        for tag, U, km in (("c3", 8159, CFG["n_lookup"]), ("scan131k", 131072, 0)):
            reprk = torch.randn(U, Hkv, CFG["n_repr"], d, device=dev).bfloat16()
            qsum = torch.randn(Hkv, d, device=dev, dtype=torch.float64)
            rel = torch.empty(U, device=dev, dtype=torch.float64)
            ids = torch.empty(max(1, km), device=dev, dtype=torch.int64)
            s_ = torch.cuda.Stream(dev)

            def call():
                _lib.check(_lib.lib().infllm_lookup(qsum.data_ptr(), reprk.data_ptr(), _lib.DTYPE_BF16, U,
                                                    CFG["n_repr"], Hkv, d, km, rel.data_ptr(), ids.data_ptr(),
                                                    s_.cuda_stream))
            with torch.cuda.stream(s_):
                call()
                torch.cuda.synchronize(dev)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s_):
                    for _ in range(10):
                        call()
                g.replay()
                torch.cuda.synchronize(dev)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s_)
                g.replay()
                e1.record(s_)
                torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1) / 10
            out[f"{tag}_units"] = U
            out[f"{tag}_us"] = ms * 1000.0
            out[f"{tag}_gbs"] = U * CFG["n_repr"] * Hkv * d * 2 / (ms * 1e-3) / 1e9
    except Exception as ex:  # diagnostic only
        out["isolated_error"] = str(ex)
    return out


def c1_stream(dev, steps=5):
    """BASELINE configs[1] (C1): Mistral-7B heads (32q/8kv, d 128), one 32K-token
    stream, same InfLLM settings; device-resident tokens/s (graph-replayed
    encode_stream, CUDA events) and the attention's roofline over its steps."""
    import torch

    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine

    n = 32768
    g = torch.Generator(device=dev)
    g.manual_seed(4321)
    H, Hkv, d = SHAPE["n_heads"], SHAPE["n_kv_heads"], SHAPE["head_dim"]
    q = torch.randn((n, H, d), generator=g, device=dev).bfloat16()
    k = torch.randn((n, Hkv, d), generator=g, device=dev).bfloat16()
    v = torch.randn((n, Hkv, d), generator=g, device=dev).bfloat16()
    eng = StreamEngine(EngineConfig.make(**CFG), ModelShape.make(**SHAPE), dtype=torch.bfloat16)
    eng.reserve(n)
    out = torch.empty_like(q)
    for _ in range(3):
        eng.reset()
        eng.encode_stream(q, k, v, out=out)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        eng.reset()
        eng.encode_stream(q, k, v, out=out)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / steps
    eng.profile_begin(True)
    eng.reset()
    eng.encode_stream(q, k, v, out=out)
    prof = eng.profile_read()
    eng.close()
    sch = stream_schedule(n, CFG)
    flops = attention_flops(sch, H, d)
    peak = load_peaks()["bf16"]
    return {"workload": "C1 (configs[1]): Mistral-7B-inst-v0.2 heads (32q/8kv, d128), one 32K-token stream, "
                        "unit 128, r_k 4, k_m 16, init 128, window 4K, chunk 512, bf16",
            "tokens_per_s": n / (ms / 1e3), "ms_per_stream": ms,
            "attention_tflops": flops / (prof["attn_ms"] / 1e3) / 1e12,
            "attention_frac_of_peak": flops / (prof["attn_ms"] / 1e3) / 1e12 / peak}


def decode_grid(dev, contexts=(131072, 524288), batches=(1, 2, 4, 8, 16, 32), dec_steps=48, dec_warm=8, rounds=3):
    """BASELINE configs[4] (C4): decode-step latency at 128K / 512K context for
    B = 1..32 independent sequences (infllm_decode_batch: every stage one
    launch for the batch; B = 1 is the single-sequence decode_step chain).
    The sequences are prefilled once per context through encode_stream; each
    B reuses the first B of them. Device time per step over dec_steps steps."""
    import torch

    import ctypes as C

    from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, _lib, decode_batch

    H, Hkv, d = SHAPE["n_heads"], SHAPE["n_kv_heads"], SHAPE["head_dim"]
    bmax = max(batches)
    rows = []
    for ctx in contexts:
        g = torch.Generator(device=dev)
        g.manual_seed(ctx)
        Q = torch.randn((ctx, H, d), generator=g, device=dev).bfloat16()
        K = torch.randn((ctx, Hkv, d), generator=g, device=dev).bfloat16()
        V = torch.randn((ctx, Hkv, d), generator=g, device=dev).bfloat16()
        tot = (rounds * dec_steps + dec_warm) * len(batches) + 4
        engs = []
        for _ in range(bmax):
            e = StreamEngine(EngineConfig.make(**CFG), ModelShape.make(**SHAPE), dtype=torch.bfloat16)
            e.reserve(ctx + tot + 1)
            e.encode_stream(Q, K, V)
            engs.append(e)
        del Q, K, V
        qd = torch.randn((tot, bmax, H, d), generator=g, device=dev).bfloat16()
        kd = torch.randn((tot, bmax, Hkv, d), generator=g, device=dev).bfloat16()
        vd = torch.randn((tot, bmax, Hkv, d), generator=g, device=dev).bfloat16()
        t = 0
        for B in batches:
            sub = engs[:B]
            res = torch.empty((B, H, d), device=dev, dtype=torch.bfloat16)
            for _ in range(dec_warm):
                decode_batch(sub, qd[t, :B].contiguous(), kd[t, :B].contiguous(), vd[t, :B].contiguous(), out=res)
                t += 1
            # the timed loop issues the C-ABI calls with their arguments prepared (what a
            # C++ host issues per step): Python-side argument checks stay outside
            lib_ = _lib.lib()
            st_ = torch.cuda.current_stream(dev).cuda_stream
            hs = (C.c_void_p * B)(*[e.h.value for e in sub])
            op = res.data_ptr()
            per_round = []
            gc.collect()
            gc.disable()  # no collector pause inside a timed round
            for _ in range(rounds):  # median of rounds: one-time driver / allocator stalls land in one
                qs = [qd[t + i, :B].contiguous() for i in range(dec_steps)]
                ks = [kd[t + i, :B].contiguous() for i in range(dec_steps)]
                vs = [vd[t + i, :B].contiguous() for i in range(dec_steps)]
                args = [(qs[i].data_ptr(), ks[i].data_ptr(), vs[i].data_ptr()) for i in range(dec_steps)]
                torch.cuda.synchronize(dev)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                if B == 1:
                    h0 = sub[0].h
                    for qp, kp, vp in args:
                        _lib.check(lib_.infllm_decode_step(h0, 0, qp, kp, vp, op, st_))
                else:
                    for qp, kp, vp in args:
                        _lib.check(lib_.infllm_decode_batch(hs, B, 0, qp, kp, vp, op, st_))
                e1.record()
                torch.cuda.synchronize(dev)
                t += dec_steps
                per_round.append(e0.elapsed_time(e1) / dec_steps)
            gc.enable()
            ms = sorted(per_round)[len(per_round) // 2]
            units = sub[0].metrics()["units"]
            kv_b = B * (CFG["init_size"] + CFG["n_lookup"] * CFG["unit_size"] + CFG["local_size"] + 1) * Hkv * d * 4
            ix_b = B * units * CFG["n_repr"] * Hkv * d * 2
            rows.append({"context": ctx, "batch": B, "step_us": ms * 1e3, "rounds_us": [x * 1e3 for x in per_round],
                         "tokens_per_s": B / (ms / 1e3),
                         "hbm_bytes_per_step": kv_b + ix_b, "hbm_gbs": (kv_b + ix_b) / (ms / 1e3) / 1e9})
        for e in engs:
            e.close()
        del engs, qd, kd, vd
        torch.cuda.empty_cache()
    return {"workload": "C4 (configs[4]): decode step latency, Llama-3-8B heads, 128K / 512K context, B "
                        "independent sequences per step (infllm_decode_batch; B = 1: decode_step chain)",
            "timing": f"CUDA events around {dec_steps} consecutive steps, median of {rounds} such rounds after "
                      f"{dec_warm} untimed steps (device time incl. host launch gaps); "
                      "the loop calls infllm_decode_step (B = 1) / infllm_decode_batch with prepared arguments",
            "hbm_bytes": "K/V^T of init + k_m units + local window + the new token, plus the repr index scan",
            "peak_gbs": load_peaks()["hbm"], "grid": rows}


def other_configs(Q, K, V, dev):
    """The other BASELINE.json configs, measured on the same box after the
    headline (not part of `value`): C1 (32K stream), C4 (decode grid) and C3
    (1M-token planted stream with the host-offloaded unit store and the
    32-slot GPU unit cache of SURVEY §8d: prefill tokens/s, probe recall,
    page loads / cache hit rate, H2D GB/s; tools/c3_planted.py)."""
    import torch

    out = {}
    for name, fn in (("c1_stream", lambda: c1_stream(dev)), ("c4_decode", lambda: decode_grid(dev))):
        try:
            out[name] = fn()
        except Exception as ex:  # reported, not fatal
            out[name] = {"error": str(ex)}
        torch.cuda.empty_cache()
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import c3_planted

        slots = 32
        ok, tps, ts = c3_planted.run(1 << 20, verbose=False, slots=slots)
        req = ts["loads"] + ts["cache_hits"]
        out["c3_host_tier"] = {
            "workload": f"C3 (configs[3]): 1M-token planted stream, unit pages in pinned host memory, {slots}-slot "
                        "GPU unit cache (host_tier_slots)", "tokens_per_s": tps, "probe_recall": 1.0 if ok else 0.0,
            "page_loads": ts["loads"], "cache_hit_rate": ts["cache_hits"] / max(req, 1),
            "miss_rate": ts["loads"] / max(req, 1),
            "h2d_gb": ts["h2d_bytes"] / 1e9, "h2d_gbs": ts["h2d_bytes"] / ((1 << 20) / tps) / 1e9}
    except Exception as ex:
        out["c3_host_tier"] = {"error": str(ex)}
    torch.cuda.empty_cache()
    return out


def bind_gpu_local_cpus(dev):
    """Run this thread on the CPUs local to the GPU's PCIe root (sysfs local_cpulist),
    so the pinned host buffers allocated next land on that NUMA node: on a
    two-socket host, buffers on the far node measured ~2/3 of the PCIe rate.
    Returns (previous affinity, cpulist text) or (None, None)."""
    import torch

    try:
        p = torch.cuda.get_device_properties(dev)
        bdf = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bdf}/local_cpulist") as f:
            txt = f.read().strip()
        cpus = set()
        for part in txt.split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        old = os.sched_getaffinity(0)
        cpus &= old
        if not cpus:
            return None, None
        os.sched_setaffinity(0, cpus)
        return old, txt
    except Exception:
        return None, None


def run_e2e(eng, Q, K, V, n, C, dev, args, world):
    """Same metric through the C-ABI with HOST buffers: infllm_encode_stream_host
    copies each chunk's q/k/v from pinned memory and each output chunk back
    (copy streams overlapped with compute), inside the timed region."""
    import torch

    old_aff, local_cpus = bind_gpu_local_cpus(dev)
    Hq = torch.empty(Q.shape, dtype=Q.dtype, pin_memory=True)
    Hk = torch.empty(K.shape, dtype=K.dtype, pin_memory=True)
    Hv = torch.empty(V.shape, dtype=V.dtype, pin_memory=True)
    Hq.copy_(Q)
    Hk.copy_(K)
    Hv.copy_(V)
    Hout = torch.empty(Q.shape, dtype=Q.dtype, pin_memory=True)
    eng.profile_begin(False)

    def stream_once():
        eng.reset()
        eng.encode_stream_host(Hq, Hk, Hv, Hout)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(max(1, args.warmup)):
        stream_once()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        stream_once()
    barrier()
    dt = time.perf_counter() - t0
    if world > 1:  # the slowest rank
        import torch.distributed as dist

        t = torch.tensor([dt], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    h2d_b = (Q.numel() + K.numel() + V.numel()) * Q.element_size()
    d2h_b = Q.numel() * Q.element_size()
    if old_aff is not None:
        os.sched_setaffinity(0, old_aff)
    # one stream (each rank holds its KV-group shard's q/k/v and outputs when world > 1)
    return {"value": n * args.steps / dt, "unit": "tokens/s", "h2d_bytes_per_step": h2d_b,
            "d2h_bytes_per_step": d2h_b, "host_buffers_numa_cpus": local_cpus,
            "note": "infllm_encode_stream_host: pinned-host q/k/v/out (allocated from the GPU's local "
                    "CPUs), per-chunk H2D/D2H on copy streams overlapped with compute, wall clock incl. copies"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--tokens", type=int, default=N_TOKENS)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-tc", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the C3 host-tier and C4 decode figures")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_b200(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
