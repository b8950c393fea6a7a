# Batched decode (C4): host time per infllm_decode_batch call vs device time per
# step (CUDA events on the call's stream) — is the batched step host-bound?
#   python tools/decode_host_probe.py [ctx=131072] [B=32] [steps=48]
import json
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, decode_batch  # noqa: E402
import bench  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 48
cfg, shape = bench.CFG, bench.SHAPE
H, Hkv, d = shape["n_heads"], shape["n_kv_heads"], shape["head_dim"]
g = torch.Generator(device="cuda")
g.manual_seed(7)
Q = torch.randn((ctx, H, d), generator=g, device="cuda").bfloat16()
K = torch.randn((ctx, Hkv, d), generator=g, device="cuda").bfloat16()
V = torch.randn((ctx, Hkv, d), generator=g, device="cuda").bfloat16()
qd = torch.randn((steps, B, H, d), generator=g, device="cuda").bfloat16()
kd = torch.randn((steps, B, Hkv, d), generator=g, device="cuda").bfloat16()
vd = torch.randn((steps, B, Hkv, d), generator=g, device="cuda").bfloat16()
out = torch.empty((B, H, d), device="cuda", dtype=torch.bfloat16)
engs = []
for _ in range(B):
    e = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(**shape), dtype=torch.bfloat16)
    e.reserve(ctx + steps + 1)
    e.encode_stream(Q, K, V)
    engs.append(e)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
host = []
ev[0].record()
t0 = time.perf_counter()
for t in range(steps):
    h0 = time.perf_counter()
    decode_batch(engs, qd[t], kd[t], vd[t], out=out)
    host.append(time.perf_counter() - h0)
    ev[t + 1].record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / steps
dev = [ev[t].elapsed_time(ev[t + 1]) * 1e3 for t in range(steps)]
warm = 8
print(json.dumps(dict(ctx=ctx, batch=B, wall_us=wall * 1e6, host_us_med=sorted(host[warm:])[len(host[warm:]) // 2] * 1e6,
                      dev_us_med=sorted(dev[warm:])[len(dev[warm:]) // 2], dev_us_min=min(dev[warm:]))))
for e in engs:
    e.close()
