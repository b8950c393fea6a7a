# Isolated K1+K2 (scan + top-k) at the C2 steady state for several grid sizes
# (engine option lookup_units_per_block_decode), graph-replayed, plus the
# in-kernel phase marks of one launch from the device timeline.
import ctypes as C, sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, _lib
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
g = torch.Generator(device='cuda'); g.manual_seed(0)
Q = torch.randn((n, 32, 128), generator=g, device='cuda').bfloat16()
K = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
V = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
eng = StreamEngine(EngineConfig.make(**bench.CFG), ModelShape.make(**bench.SHAPE), dtype=torch.bfloat16)
eng.reserve(n); eng.set_option("cuda_graphs", 0)
eng.encode_stream(Q, K, V); torch.cuda.synchronize()
L = _lib.lib()
for upb in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else "4,8,16,32,64".split(","))]:
    eng.set_option("lookup_units_per_block_decode", upb)
    us = C.c_double()
    _lib.check(L.infllm_debug_kernel_bench(eng.h, 1, 50, C.byref(us)))
    cap = 1 << 16
    _lib.check(L.infllm_timeline_enable(cap))
    _lib.check(L.infllm_debug_kernel_bench(eng.h, 1, 1, C.byref(C.c_double())))
    kid = np.zeros(cap, np.uint32); sm = np.zeros(cap, np.uint32); t0 = np.zeros(cap, np.uint64); t1 = np.zeros(cap, np.uint64)
    nn = C.c_int64()
    _lib.check(L.infllm_timeline_read(kid.ctypes.data, sm.ctypes.data, t0.ctypes.data, t1.ctypes.data, cap, C.byref(nn), 1))
    _lib.check(L.infllm_timeline_enable(0))
    m = min(nn.value, cap)
    kid, t0, t1 = kid[:m], t0[:m].astype(np.int64), t1[:m].astype(np.int64)
    # the debug bench launches twice (warm + graph of 1 + replay): keep the last launch's records
    lk = np.where(kid == 4)[0]
    last0 = t0[lk].max() - 30000
    ph = {k: (t1[(kid == 100 + k) & (t0 > last0)] - t0[(kid == 100 + k) & (t0 > last0)]) / 1e3 for k in range(4)}
    span = (t1[(kid >= 100) & (t0 > last0)].max() - t0[lk][t0[lk] > last0].min()) / 1e3
    print(f"U={eng.metrics()['units']} units/block={upb:3d} blocks={(eng.metrics()['units'] + upb - 1) // upb:4d} "
          f"graph-timed {us.value:6.2f} us | phases (median us): scan {np.median(ph[0]):.2f} block-merge "
          f"{np.median(ph[1]):.2f} last-stage {np.median(ph[2]) if len(ph[2]) else 0:.2f} final "
          f"{np.median(ph[3]) if len(ph[3]) else 0:.2f}; first start->last mark {span:.2f}", flush=True)
