# steady-state per-kernel timing at the C2 steady state (debug entry point)
import sys, ctypes as C, torch
sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, _lib
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
g = torch.Generator(device='cuda'); g.manual_seed(0)
Q = torch.randn((n, 32, 128), generator=g, device='cuda').bfloat16()
K = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
V = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
names = ["prep", "lookup+topk", "attention", "evict+select", "lru", "lookup-scan", "topk-only", "empty-124x256", "empty-1x32"]
for which in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0","1","2","3","4"])]:
    eng = StreamEngine(EngineConfig.make(**bench.CFG), ModelShape.make(**bench.SHAPE), dtype=torch.bfloat16)
    eng.reserve(n); eng.set_option("cuda_graphs", 0)
    eng.encode_stream(Q, K, V); torch.cuda.synchronize()
    us = C.c_double()
    _lib.check(_lib.lib().infllm_debug_kernel_bench(eng.h, which, 50, C.byref(us)))
    print(f"{names[which]:14s} {us.value:8.2f} us/launch  (U={eng.metrics()['units']})", flush=True)
    eng.close()
