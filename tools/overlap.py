# timing experiment: stream time when the attention does not wait for the lookup (results invalid)
import sys, time, torch
sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine
import bench
n = 131072
g = torch.Generator(device='cuda'); g.manual_seed(0)
Q = torch.randn((n, 32, 128), generator=g, device='cuda').bfloat16()
K = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
V = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
O = torch.empty_like(Q)
for skip in [0, 2, 4, 8, 16, 32]:
    eng = StreamEngine(EngineConfig.make(**bench.CFG), ModelShape.make(**bench.SHAPE), dtype=torch.bfloat16)
    eng.reserve(n)
    eng.set_option("debug_skip", skip)
    ts = []
    for it in range(4):
        eng.reset(); torch.cuda.synchronize()
        t0 = time.perf_counter(); eng.encode_stream(Q, K, V, out=O); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"skip={skip:2d} ms/stream={1000*min(ts[1:]):.2f} us/step={1e6*min(ts[1:])/256:.1f}", flush=True)
    eng.close()
