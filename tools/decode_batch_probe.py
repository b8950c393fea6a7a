# Batched decode (infllm_decode_batch) at C4: host submission vs device time per
# step, B sequences prefilled to ctx tokens.
#   python tools/decode_batch_probe.py [ctx=131072] [B=32] [steps=50]
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, decode_batch  # noqa: E402
import bench  # noqa: E402


def main(ctx=131072, B=32, steps=50):
    cfg, shape = bench.CFG, bench.SHAPE
    H, Hkv, d = shape["n_heads"], shape["n_kv_heads"], shape["head_dim"]
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    Q = torch.randn((ctx, H, d), generator=g, device="cuda").bfloat16()
    K = torch.randn((ctx, Hkv, d), generator=g, device="cuda").bfloat16()
    V = torch.randn((ctx, Hkv, d), generator=g, device="cuda").bfloat16()
    qd = torch.randn((steps + 8, B, H, d), generator=g, device="cuda").bfloat16()
    kd = torch.randn((steps + 8, B, Hkv, d), generator=g, device="cuda").bfloat16()
    vd = torch.randn((steps + 8, B, Hkv, d), generator=g, device="cuda").bfloat16()
    out = torch.empty((B, H, d), device="cuda", dtype=torch.bfloat16)
    engs = []
    for _ in range(B):
        e = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(**shape), dtype=torch.bfloat16)
        e.reserve(ctx + steps + 16)
        e.encode_stream(Q, K, V)
        engs.append(e)
    torch.cuda.synchronize()
    for t in range(8):
        decode_batch(engs, qd[t], kd[t], vd[t], out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    for t in range(8, steps + 8):
        decode_batch(engs, qd[t], kd[t], vd[t], out=out)
    b.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"B={B} ctx={ctx}: host submit {(t1 - t0) / steps * 1e6:.1f} us/step, wall {(t2 - t0) / steps * 1e6:.1f} "
          f"us/step, device {a.elapsed_time(b) / steps * 1e3:.1f} us/step", flush=True)


if __name__ == "__main__":
    main(*(int(x) for x in sys.argv[1:]))
