# per-CTA start/end spread of one attention launch (build with -DATTN_CTA_TS=1)
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
# reset the stamp slots: min fields to max, others to 0, then one launch
import ctypes
sym = np.array([2**64 - 1, 0, 2**64 - 1, 0, 0, 2**64 - 1, 0, 0] + [0] * 56, dtype=np.uint64)
lib = _lib.lib()
cudart = ctypes.CDLL("libcudart.so") if False else None
us = C.c_double()
_lib.check(lib.infllm_debug_kernel_bench(eng.h, 2, 1, C.byref(us)))  # warm
ts = np.zeros(64, np.uint64)
_lib.check(lib.infllm_debug_timestamps(ts.ctypes.data))
print("note: stamps accumulate over the bench launches")
t = ts.astype(np.int64)
print("launch us (bench)", us.value)
print(f"start spread {(t[1]-t[0])/1e3:.1f} us, end spread {(t[3]-t[2])/1e3:.1f} us, first start->last end {(t[3]-t[0])/1e3:.1f} us, "
      f"CTA duration max {t[4]/1e3:.1f} min {t[5]/1e3:.1f} mean {t[6]/max(t[7],1)/1e3:.1f} us over {t[7]} CTAs")
dt_ns = t[12] - t[10]; dc = t[13] - t[11]
print(f"CTA(3,0): {dt_ns/1e3:.1f} us, {dc} cycles -> effective SM clock {dc/dt_ns:.3f} GHz")
