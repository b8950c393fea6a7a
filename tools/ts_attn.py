# per-tile MMA-issuer timestamps of attention CTA (0,0) (build with -DATTN_TS=1; INFLLM_TS_ATTN=1)
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
t = ts.astype(np.int64).reshape(8, 8)
base = t[0, 0]
print("attention us", us.value)
names = ["qk_start", "k_ready", "p_ready", "v_ready", "qk_done", "pv_done", "sm_s_seen", "sm_p_arr"]
print("tile " + " ".join(f"{n:>9s}" for n in names))
for j in range(8):
    print(f"{18+j:4d} " + " ".join(f"{t[j,k]-base:9d}" for k in range(8)))
