import sys, ctypes as C, numpy as np, torch
sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, _lib
import bench
n = 131072
g = torch.Generator(device='cuda'); g.manual_seed(0)
Q = torch.randn((n, 32, 128), generator=g, device='cuda').bfloat16()
K = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
V = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
eng = StreamEngine(EngineConfig.make(**bench.CFG), ModelShape.make(**bench.SHAPE), dtype=torch.bfloat16)
eng.reserve(n); eng.set_option("cuda_graphs", 0)
eng.encode_stream(Q, K, V); torch.cuda.synchronize()
us = C.c_double()
_lib.check(_lib.lib().infllm_debug_kernel_bench(eng.h, int(sys.argv[1]), 5, C.byref(us)))
ts = np.zeros(64, np.uint64)
_lib.check(_lib.lib().infllm_debug_timestamps(ts.ctypes.data))
t = ts.astype(np.int64); base = t[0]
print("topk us", us.value)
idx=[int(x) for x in sys.argv[2].split(",")]; base=t[idx[0]]
for i in idx: print(i, t[i]-base)
