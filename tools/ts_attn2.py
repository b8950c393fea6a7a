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
names = ["s_seen", "s_free", "exp_go", "exp_end", "p_arr", "qk+2_go", "qk+2_end", "pv_end"]
print("tile(WG0) " + " ".join(f"{n:>9s}" for n in names))
for j in range(8):
    print(2 * j, " ".join(f"{int(x - base):9d}" for x in u[j]))
e = t[56:63] - t[56]
print("entry->cluster_sync", e[1], " ->flag", e[2], " tile0 s_seen", t[0] - t[56], " ->all PV done", e[3], " ->epilogue end", e[4], " ->syncthreads", e[5], " ->cluster_sync", e[6])
print("all PV done -> bar.sync", t[53] - t[59], " -> O stored", t[54] - t[59], " -> masses+end", t[60] - t[59])
