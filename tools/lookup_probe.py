# Standalone K1+K2 (infllm_lookup) at the C2 (991 units) and C3 (8159 units)
# index sizes: graph-timed device time per lookup and the in-kernel phase marks
# of one launch (scan / block top-32 / candidates staged / final selection).
#   python tools/lookup_probe.py [U,...]
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2402_04617_b200 import _lib

L = _lib.lib()
G, RK, D, KM = 8, 4, 128, 16
for U in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "991,8159").split(",")]:
    reprk = torch.randn(U, G, RK, D, device="cuda").bfloat16()
    qsum = torch.randn(G, D, device="cuda", dtype=torch.float64)
    rel = torch.empty(U, device="cuda", dtype=torch.float64)
    ids = torch.empty(KM, device="cuda", dtype=torch.int64)
    s = torch.cuda.Stream()

    def call():
        _lib.check(L.infllm_lookup(qsum.data_ptr(), reprk.data_ptr(), _lib.DTYPE_BF16, U, RK, G, D, KM,
                                   rel.data_ptr(), ids.data_ptr(), s.cuda_stream))

    with torch.cuda.stream(s):
        call()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                call()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1000
    b = U * G * RK * D * 2
    # phase marks of one launch
    cap = 1 << 16
    _lib.check(L.infllm_timeline_enable(cap))
    with torch.cuda.stream(s):
        call()
    torch.cuda.synchronize()
    kid = np.zeros(cap, np.uint32); sm = np.zeros(cap, np.uint32)
    t0 = np.zeros(cap, np.uint64); t1 = np.zeros(cap, np.uint64)
    nn = C.c_int64()
    _lib.check(L.infllm_timeline_read(kid.ctypes.data, sm.ctypes.data, t0.ctypes.data, t1.ctypes.data, cap,
                                      C.byref(nn), 1))
    _lib.check(L.infllm_timeline_enable(0))
    m = min(nn.value, cap)
    kid, t0, t1 = kid[:m], t0[:m].astype(np.int64), t1[:m].astype(np.int64)
    ph = {k: (t1[kid == 100 + k] - t0[kid == 100 + k]) / 1e3 for k in range(8)}
    blocks = int((kid == 4).sum())
    span = (t1.max() - t0.min()) / 1e3 if m else 0
    med = {k: (np.median(v) if len(v) else 0.0) for k, v in ph.items()}
    print(f"U={U:6d}: {us:7.2f} us per lookup (graph), {b / 1e6:6.1f} MB -> {b / us / 1e3:7.1f} GB/s; "
          f"blocks {blocks}; phase marks median us: " + " ".join(f"{k}:{v:.2f}" for k, v in med.items() if v) +
          f"; timeline span {span:.2f}", flush=True)
