# C3-style planted-span recall on the CUDA path (workload.hpp:35-127 semantics,
# GPU-generated data): random bf16 q/k/v for an n-token stream, one key vector
# (per KV head) repeated over a 64-token span at a random offset in the evicted
# region, and the last 4 tokens (decode steps) querying with that key. Reports
# prefill throughput and whether every probe lookup retrieved the span's units.
# slots > 0: host-offloaded unit store (pinned host pages) + an S-slot GPU unit
# cache (engine option host_tier_slots); reports page loads, cache hit rate
# and the achieved H2D GB/s of the page pulls.
#   python tools/c3_planted.py [n_tokens=1048576] [slots=0]
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine  # noqa: E402
import bench  # noqa: E402


def run(n, seed=0, verbose=True, slots=0):
    cfg, shape = bench.CFG, bench.SHAPE
    H, Hkv, d = shape["n_heads"], shape["n_kv_heads"], shape["head_dim"]
    L, I, bs, C = cfg["local_size"], cfg["init_size"], cfg["unit_size"], cfg["chunk_size"]
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    probe = 4
    npre = n - probe
    Q = torch.randn((n, H, d), generator=g, device="cuda").bfloat16()
    K = torch.randn((n, Hkv, d), generator=g, device="cuda").bfloat16()
    V = torch.randn((n, Hkv, d), generator=g, device="cuda").bfloat16()
    # plant: offset in [I, npre - L - bs - 64], unit-aligned like gen_planted(align=True)
    hi = npre - L - bs - 64
    a = I + int(torch.randint(0, (hi - I) // bs, (1,), generator=g, device="cuda").item()) * bs
    key = torch.randn((Hkv, d), generator=g, device="cuda") * 3.0
    # q == k for the planted token id (adapter.hpp:63-65): the span scores itself
    # into the unit's representatives; the probes query with the same vector
    K[a:a + 64] = key.bfloat16()
    Q[a:a + 64] = key.repeat_interleave(H // Hkv, 0).bfloat16()
    Q[npre:] = (key.repeat_interleave(H // Hkv, 0) * 3.0).bfloat16()
    expected = sorted({(t - I) // bs for t in (a, a + 63)})
    eng = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(**shape), dtype=torch.bfloat16)
    if slots:
        eng.set_option("host_tier_slots", slots)
    eng.reserve(n)
    out = torch.empty((npre, H, d), device="cuda", dtype=torch.bfloat16)
    eng.encode_stream(Q[:npre], K[:npre], V[:npre], out=out)  # graph capture + first replay
    eng.reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.encode_stream(Q[:npre], K[:npre], V[:npre], out=out)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ts = eng.tier_stats() if slots else None
    hits = []
    for i in range(npre, n):
        r = eng.step(Q[i:i + 1], K[i:i + 1], V[i:i + 1], decode=True)
        hits.append(set(expected) <= set(r.retrieved_ids))
    m = eng.metrics()
    if verbose:
        print(f"n={n}: prefill {npre} tokens in {dt * 1e3:.1f} ms = {npre / dt / 1e6:.2f} Mtok/s "
              f"(units {m['units']}, plant at {a}, expected units {expected}), probe recall "
              f"{sum(hits)}/{len(hits)}", flush=True)
        if ts:
            req = ts["loads"] + ts["cache_hits"]
            print(f"  host tier: {slots} GPU slots, {ts['loads']} page loads / {req} retrieved units "
                  f"(cache hit rate {ts['cache_hits'] / max(req, 1):.3f}; reference LRU misses {m['misses']}), "
                  f"{ts['h2d_bytes'] / 1e9:.2f} GB H2D = {ts['h2d_bytes'] / dt / 1e9:.1f} GB/s over the prefill",
                  flush=True)
    return all(hits), npre / dt, ts


if __name__ == "__main__":
    run(int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20, slots=int(sys.argv[2]) if len(sys.argv) > 2 else 0)
