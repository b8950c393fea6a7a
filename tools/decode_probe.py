# Where a single-sequence decode step's time goes (C2 shape, 128K context):
# host submission time per decode_step call vs the device time of the step
# chain, with the K4 decode kernel and with the tcgen05 path.
#   python tools/decode_probe.py [ctx=131072] [steps=200]
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine  # noqa: E402
import bench  # noqa: E402


def main(ctx=131072, steps=200, variants=(1, 0)):
    cfg, shape = bench.CFG, bench.SHAPE
    H, Hkv, d = shape["n_heads"], shape["n_kv_heads"], shape["head_dim"]
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    Q = torch.randn((ctx + steps, H, d), generator=g, device="cuda").bfloat16()
    K = torch.randn((ctx + steps, Hkv, d), generator=g, device="cuda").bfloat16()
    V = torch.randn((ctx + steps, Hkv, d), generator=g, device="cuda").bfloat16()
    out = torch.empty((1, H, d), device="cuda", dtype=torch.bfloat16)
    for dec in variants:
        eng = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(**shape), dtype=torch.bfloat16)
        eng.set_option("decode_kernel", dec)
        eng.reserve(ctx + steps + 1)
        eng.encode_stream(Q[:ctx], K[:ctx], V[:ctx])
        torch.cuda.synchronize()
        for i in range(ctx, ctx + 8):  # warm-up
            eng.decode_step(Q[i:i + 1], K[i:i + 1], V[i:i + 1], out=out)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = eng.kernel_launches()
        t0 = time.perf_counter()
        a.record()
        for i in range(ctx + 8, ctx + steps):
            eng.decode_step(Q[i:i + 1], K[i:i + 1], V[i:i + 1], out=out)
        b.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        n = steps - 8
        print(f"decode_kernel={dec}: host submit {(t1 - t0) / n * 1e6:.1f} us/step, wall {(t2 - t0) / n * 1e6:.1f} "
              f"us/step, device (events, caller stream) {a.elapsed_time(b) / n * 1e3:.1f} us/step, "
              f"{(eng.kernel_launches() - l0) / n:.1f} launches/step", flush=True)
        eng.close()


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 131072, int(sys.argv[2]) if len(sys.argv) > 2 else 200,
         tuple(int(x) for x in sys.argv[3].split(',')) if len(sys.argv) > 3 else (1, 0))
