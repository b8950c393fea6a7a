# timing experiment: what the bench's timed region costs beyond the kernels
import sys, torch
sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine
import bench
n = 131072
g = torch.Generator(device='cuda'); g.manual_seed(0)
Q = torch.randn((n, 32, 128), generator=g, device='cuda').bfloat16()
K = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
V = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
O = torch.empty_like(Q)
eng = StreamEngine(EngineConfig.make(**bench.CFG), ModelShape.make(**bench.SHAPE), dtype=torch.bfloat16)
eng.reserve(n)
for prof in (True, False, True, False):
    eng.profile_begin(prof)
    for _ in range(3):
        eng.reset(); eng.encode_stream(Q, K, V, out=O)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        eng.reset(); eng.encode_stream(Q, K, V, out=O)
    e1.record(); torch.cuda.synchronize()
    print(f"prof={prof} ms/stream={e0.elapsed_time(e1)/5:.2f}", flush=True)
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record()
    for _ in range(5):
        eng.reset()
    r1.record(); torch.cuda.synchronize()
    print(f"  reset only ms={r0.elapsed_time(r1)/5:.3f}", flush=True)
