import os, sys, ctypes as C, numpy as np, torch
os.environ["INFLLM_TS_ATTN"] = "1"
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
_lib.check(_lib.lib().infllm_debug_kernel_bench(eng.h, 2, 3, C.byref(us)))
ts = np.zeros(64, np.uint64)
_lib.check(_lib.lib().infllm_debug_timestamps(ts.ctypes.data))
t = ts.astype(np.int64)
u = t[0:64].reshape(8, 8); base = u[0, 0]
print("tile j (WG0): pv_issued s_seen(j) k_wait_start(j+2) qk_issued(j+2) exp_done(j) k_ready(j+2) p_wait_start p_ready")
for j in range(8):
    r = [int(x - base) for x in u[j]]
    print(20 + 2 * j, r, [r[k] - r[k - 1] for k in range(1, 6)])
