# C4 decode (BASELINE.json configs[4]): B independent sequences of one InfLLM
# layer (Llama-3-8B heads, C2 settings), each first prefilled to `ctx` tokens
# through encode_stream, then decoded token by token (engine.hpp:100-103:
# lookup of the single token, attention over init | 16 units | local window,
# eviction of one token, LRU). Each sequence's decode_step is issued on its own
# CUDA stream so the B sequences' kernels overlap on the GPU ("streams"), or all
# B sequences go through one infllm_decode_batch call per step ("batched": each
# stage one launch for the whole batch). Reports the wall latency of one decode
# step of the batch (host launch included) and tokens/s.
#   python tools/decode_bench.py [ctx=131072,524288] [B=1,2,4,8,16,32] [steps=32] [mode=batched|streams]
import json
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, decode_batch  # noqa: E402
import bench  # noqa: E402


def run(ctx, batches, steps=32, warm=4, mode="batched"):
    cfg, shape = bench.CFG, bench.SHAPE
    H, Hkv, d = shape["n_heads"], shape["n_kv_heads"], shape["head_dim"]
    g = torch.Generator(device="cuda")
    g.manual_seed(ctx)
    Q = torch.randn((ctx, H, d), generator=g, device="cuda").bfloat16()
    K = torch.randn((ctx, Hkv, d), generator=g, device="cuda").bfloat16()
    V = torch.randn((ctx, Hkv, d), generator=g, device="cuda").bfloat16()
    bmax = max(batches)
    tot = steps + warm
    qd = torch.randn((bmax, tot, 1, H, d), generator=g, device="cuda").bfloat16()
    kd = torch.randn((bmax, tot, 1, Hkv, d), generator=g, device="cuda").bfloat16()
    vd = torch.randn((bmax, tot, 1, Hkv, d), generator=g, device="cuda").bfloat16()
    out = torch.empty((bmax, 1, H, d), device="cuda", dtype=torch.bfloat16)
    qd, kd, vd = qd.contiguous(), kd.contiguous(), vd.contiguous()
    rows = []
    engines = []
    streams = [torch.cuda.Stream() for _ in range(bmax)]
    for B in batches:
        while len(engines) < B:
            e = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(**shape), dtype=torch.bfloat16)
            e.reserve(ctx + tot + 1)
            engines.append(e)
        for e in engines[:B]:
            e.reset()
            e.encode_stream(Q, K, V)
        torch.cuda.synchronize()
        for t in range(tot):
            if t == warm:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
            if mode == "batched":
                decode_batch(engines[:B], qd[:B, t, 0].contiguous(), kd[:B, t, 0].contiguous(), vd[:B, t, 0].contiguous(),
                             out=out[:B, 0])
            else:
                for i in range(B):
                    engines[i].decode_step(qd[i, t], kd[i, t], vd[i, t], out=out[i], stream=streams[i])
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / steps
        m = engines[0].metrics()
        kv_bytes = B * (cfg["init_size"] + cfg["n_lookup"] * cfg["unit_size"] + cfg["local_size"] + 1) * Hkv * d * 2 * 2
        idx_bytes = B * m["units"] * cfg["n_repr"] * Hkv * d * 2
        row = dict(ctx=ctx, batch=B, mode=mode, step_ms=dt * 1e3, tokens_per_s=B / dt, units=m["units"],
                   hbm_gbs=(kv_bytes + idx_bytes) / dt / 1e9)
        rows.append(row)
        print(json.dumps(row), flush=True)
    for e in engines:
        e.close()
    return rows


if __name__ == "__main__":
    ctxs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "131072,524288").split(",")]
    bs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8,16,32").split(",")]
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    mode = sys.argv[4] if len(sys.argv) > 4 else "batched"
    for c in ctxs:
        run(c, bs, steps, mode=mode)
