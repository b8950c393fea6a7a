# A short C2-shaped stream (n tokens, default 20480 = 40 chunk steps) for ncu captures of one kernel.
#   python tools/short_stream.py [n] [opt=val,...]
import sys, torch
sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20480
opts = dict(kv.split('=') for kv in (sys.argv[2].split(',') if len(sys.argv) > 2 else []) if kv)
g = torch.Generator(device='cuda'); g.manual_seed(0)
Q = torch.randn((n, 32, 128), generator=g, device='cuda').bfloat16()
K = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
V = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
eng = StreamEngine(EngineConfig.make(**bench.CFG), ModelShape.make(**bench.SHAPE), dtype=torch.bfloat16)
eng.reserve(n)
eng.set_option("cuda_graphs", 0)
for k, v in opts.items():
    eng.set_option(k, int(v))
eng.encode_stream(Q, K, V)
torch.cuda.synchronize()
print("ok", eng.metrics()["units"])
