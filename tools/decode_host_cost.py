# Host cost of a decode step vs batch size: engines prefilled to a short
# context (device work small), then infllm_decode_step / infllm_decode_batch
# called through the C-ABI with prepared arguments; host us per call (wall,
# no sync inside the loop) and device us per call (events).
#   python tools/decode_host_cost.py [ctx=8192]
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, _lib  # noqa: E402
import bench  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
cfg, shape = bench.CFG, bench.SHAPE
H, Hkv, d = shape["n_heads"], shape["n_kv_heads"], shape["head_dim"]
g = torch.Generator(device="cuda")
g.manual_seed(5)
Q = torch.randn((ctx, H, d), generator=g, device="cuda").bfloat16()
K = torch.randn((ctx, Hkv, d), generator=g, device="cuda").bfloat16()
V = torch.randn((ctx, Hkv, d), generator=g, device="cuda").bfloat16()
L = _lib.lib()
st = torch.cuda.current_stream().cuda_stream
for B in (1, 4, 32):
    engs = []
    for _ in range(B):
        e = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(**shape), dtype=torch.bfloat16)
        e.reserve(ctx + 256)
        e.encode_stream(Q, K, V)
        engs.append(e)
    steps = 100
    qd = torch.randn((steps + 4, B, H, d), generator=g, device="cuda").bfloat16()
    kd = torch.randn((steps + 4, B, Hkv, d), generator=g, device="cuda").bfloat16()
    vd = torch.randn((steps + 4, B, Hkv, d), generator=g, device="cuda").bfloat16()
    out = torch.empty((B, H, d), device="cuda", dtype=torch.bfloat16)
    hs = (C.c_void_p * B)(*[e.h.value for e in engs])
    args = [(qd[i].data_ptr(), kd[i].data_ptr(), vd[i].data_ptr()) for i in range(steps + 4)]

    def call(i):
        qp, kp, vp = args[i]
        if B == 1:
            _lib.check(L.infllm_decode_step(engs[0].h, 0, qp, kp, vp, out.data_ptr(), st))
        else:
            _lib.check(L.infllm_decode_batch(hs, B, 0, qp, kp, vp, out.data_ptr(), st))

    for i in range(4):
        call(i)
    torch.cuda.synchronize()
    _lib.check(L.infllm_debug_host_times(None, 1))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    for i in range(4, steps + 4):
        call(i)
    t1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    hb = (C.c_double * 6)()
    _lib.check(L.infllm_debug_host_times(C.cast(hb, C.c_void_p), 1))
    nc = max(1.0, hb[5])
    print(f"B={B:3d} ctx={ctx}: host {1e6 * (t1 - t0) / steps:7.1f} us/call, device {1e3 * a.elapsed_time(b) / steps:7.1f} us/call"
          + (f"; decode_batch host us/call: checks {hb[0] / nc:.1f} step-logic {hb[1] / nc:.1f} tables {hb[2] / nc:.1f} "
             f"slot-wait {hb[3] / nc:.1f} copies+launches {hb[4] / nc:.1f}" if B > 1 else ""), flush=True)
    for e in engs:
        e.close()
