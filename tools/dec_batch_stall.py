# Long batched decode run: per-round device time and decode_batch host-time
# breakdown, to locate periodic stalls (which round, host or device side).
#   python tools/dec_batch_stall.py [n=131072] [B=16] [rounds=20] [B_first=0]
# (B_first > 0: the first B_first engines step 152 times alone first, as the
# bench's grid does before a larger batch joins them)
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, _lib, decode_batch  # noqa: E402
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 20
b_first = int(sys.argv[4]) if len(sys.argv) > 4 else 0
steps = 48
cfg, shape = bench.CFG, bench.SHAPE
H, Hkv, d = shape["n_heads"], shape["n_kv_heads"], shape["head_dim"]
g = torch.Generator(device="cuda")
g.manual_seed(5)
Q = torch.randn((n, H, d), generator=g, device="cuda").bfloat16()
K = torch.randn((n, Hkv, d), generator=g, device="cuda").bfloat16()
V = torch.randn((n, Hkv, d), generator=g, device="cuda").bfloat16()
engs = []
for _ in range(B):
    e = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(**shape), dtype=torch.bfloat16)
    e.reserve(n + rounds * steps + 64 + 160)
    e.encode_stream(Q, K, V)
    engs.append(e)
del Q, K, V
qd = torch.randn((steps, B, H, d), generator=g, device="cuda").bfloat16()
kd = torch.randn((steps, B, Hkv, d), generator=g, device="cuda").bfloat16()
vd = torch.randn((steps, B, Hkv, d), generator=g, device="cuda").bfloat16()
out = torch.empty((B, H, d), device="cuda", dtype=torch.bfloat16)
L = _lib.lib()
st = torch.cuda.current_stream().cuda_stream
hs = (C.c_void_p * B)(*[e.h.value for e in engs])
if b_first:
    for t in range(152):
        decode_batch(engs[:b_first], qd[t % steps, :b_first].contiguous(), kd[t % steps, :b_first].contiguous(),
                     vd[t % steps, :b_first].contiguous(), out=out[:b_first])
    torch.cuda.synchronize()
for t in range(8):
    decode_batch(engs, qd[t], kd[t], vd[t], out=out)
torch.cuda.synchronize()
for r in range(rounds):
    _lib.check(L.infllm_debug_host_times(None, 1))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    for i in range(steps):
        _lib.check(L.infllm_decode_batch(hs, B, 0, qd[i].data_ptr(), kd[i].data_ptr(), vd[i].data_ptr(), out.data_ptr(), st))
    b.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    hb = (C.c_double * 6)()
    _lib.check(L.infllm_debug_host_times(C.cast(hb, C.c_void_p), 1))
    units = engs[0].metrics()["units"]
    print(f"round {r:2d} (steps {8 + r * steps}-{8 + (r + 1) * steps}, units {units}): device {1e3 * a.elapsed_time(b) / steps:8.1f} us/step, "
          f"host {1e6 * (t1 - t0) / steps:8.1f} us/call: step-logic {hb[1] / steps:.1f} tables {hb[2] / steps:.1f} "
          f"slot-wait {hb[3] / steps:.1f} copies+launches {hb[4] / steps:.1f}", flush=True)
