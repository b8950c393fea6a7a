# Batched decode (infllm_decode_batch) at the C2 shape: device us per step for
# library variants, interleaved in fresh subprocesses (B sequences after a
# prefill of n tokens, C-ABI calls with prepared arguments, median of rounds).
#   python tools/dec_batch_ab.py n B libA.so libB.so ...
import subprocess
import sys

CHILD = r'''
import ctypes as C, os, sys, torch
sys.path.insert(0, '.')
import paper_2402_04617_b200._lib as L
L.LIB_PATH = sys.argv[1]
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, _lib, decode_batch
import bench
n, B = int(sys.argv[2]), int(sys.argv[3])
cfg, shape = bench.CFG, bench.SHAPE
H, Hkv, d = shape["n_heads"], shape["n_kv_heads"], shape["head_dim"]
g = torch.Generator(device="cuda"); g.manual_seed(5)
Q = torch.randn((n, H, d), generator=g, device="cuda").bfloat16()
K = torch.randn((n, Hkv, d), generator=g, device="cuda").bfloat16()
V = torch.randn((n, Hkv, d), generator=g, device="cuda").bfloat16()
engs = []
for _ in range(B):
    e = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(**shape), dtype=torch.bfloat16)
    e.reserve(n + 600); e.encode_stream(Q, K, V); engs.append(e)
steps = 48
qd = torch.randn((4 * steps + 8, B, H, d), generator=g, device="cuda").bfloat16()
kd = torch.randn((4 * steps + 8, B, Hkv, d), generator=g, device="cuda").bfloat16()
vd = torch.randn((4 * steps + 8, B, Hkv, d), generator=g, device="cuda").bfloat16()
out = torch.empty((B, H, d), device="cuda", dtype=torch.bfloat16)
lib = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
hs = (C.c_void_p * B)(*[e.h.value for e in engs])
for t in range(8): decode_batch(engs, qd[t], kd[t], vd[t], out=out)
res = []
t = 8
for r in range(3):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(steps):
        _lib.check(lib.infllm_decode_batch(hs, B, 0, qd[t + i].data_ptr(), kd[t + i].data_ptr(), vd[t + i].data_ptr(), out.data_ptr(), st))
    b.record(); torch.cuda.synchronize(); t += steps
    res.append(1e3 * a.elapsed_time(b) / steps)
res.sort()
print(f"{sys.argv[1]:32s} n={n} B={B}: {res[1]:8.2f} us/step (rounds {', '.join(f'{x:.1f}' for x in res)})", flush=True)
'''
n, B, libs = sys.argv[1], sys.argv[2], sys.argv[3:]
for rnd in range(2):
    for lb in libs:
        subprocess.run([sys.executable, "-c", CHILD, lb, n, B])
