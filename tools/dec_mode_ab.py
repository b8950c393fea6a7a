# One-sequence decode at the C2 shape after a prefill of n tokens, engine
# option A/B: host us per call and device us per call (events) through the
# C-ABI with prepared arguments, rounds interleaved over the option values.
#   python tools/dec_mode_ab.py [n=131072] [option=decode_chain] [values=1,2] [rounds=3]
# (DEC_AB_LIB=path.so: time that library build)
import ctypes as C
import sys
import time

import os

import torch

sys.path.insert(0, '.')
import paper_2402_04617_b200._lib as _L  # noqa: E402

if os.environ.get("DEC_AB_LIB"):  # a library variant (tmp_libs/...) instead of the in-tree build
    _L.LIB_PATH = os.environ["DEC_AB_LIB"]
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, _lib  # noqa: E402
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
opt = sys.argv[2] if len(sys.argv) > 2 else "decode_chain"
vals = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "1,2").split(",")]
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 3
cfg, shape = bench.CFG, bench.SHAPE
H, Hkv, d = shape["n_heads"], shape["n_kv_heads"], shape["head_dim"]
g = torch.Generator(device="cuda")
g.manual_seed(5)
Q = torch.randn((n, H, d), generator=g, device="cuda").bfloat16()
K = torch.randn((n, Hkv, d), generator=g, device="cuda").bfloat16()
V = torch.randn((n, Hkv, d), generator=g, device="cuda").bfloat16()
L = _lib.lib()
st = torch.cuda.current_stream().cuda_stream
steps = 128
engs = {}
for v in vals:
    e = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(**shape), dtype=torch.bfloat16)
    e.reserve(n + rounds * (steps + 4) + 64)
    e.set_option(opt, v)
    e.encode_stream(Q, K, V)
    engs[v] = e
del Q, K, V
qd = torch.randn((steps + 4, H, d), generator=g, device="cuda").bfloat16()
kd = torch.randn((steps + 4, Hkv, d), generator=g, device="cuda").bfloat16()
vd = torch.randn((steps + 4, Hkv, d), generator=g, device="cuda").bfloat16()
out = torch.empty((H, d), device="cuda", dtype=torch.bfloat16)
args = [(qd[i].data_ptr(), kd[i].data_ptr(), vd[i].data_ptr()) for i in range(steps + 4)]
res = {v: [] for v in vals}
for r in range(rounds):
    for v in vals:
        h = engs[v].h
        for i in range(4):
            _lib.check(L.infllm_decode_step(h, 0, *args[i], out.data_ptr(), st))
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record()
        for i in range(4, steps + 4):
            _lib.check(L.infllm_decode_step(h, 0, *args[i], out.data_ptr(), st))
        t1 = time.perf_counter()
        b.record()
        torch.cuda.synchronize()
        res[v].append((1e6 * (t1 - t0) / steps, 1e3 * a.elapsed_time(b) / steps))
for v in vals:
    hs = sorted(x[0] for x in res[v])
    ds = sorted(x[1] for x in res[v])
    print(f"n={n} {opt}={v}: host us/call {hs[len(hs) // 2]:6.1f}  device us/step median {ds[len(ds) // 2]:6.2f} "
          f"(all {', '.join(f'{x:.2f}' for x in ds)})", flush=True)
