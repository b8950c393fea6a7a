# The bench's C4 decode-grid procedure for one context and B = 1, with an
# engine option: n_eng engines prefilled (the grid prefills 32), engine 0
# stepped through the C-ABI with prepared arguments.
#   python tools/dec_grid_probe.py [ctx=524288] [n_eng=32] [opt=val,...]
import ctypes as C
import sys

import torch

sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, _lib, decode_batch  # noqa: E402
import bench  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
n_eng = int(sys.argv[2]) if len(sys.argv) > 2 else 32
opts = [kv.split("=") for kv in (sys.argv[3].split(",") if len(sys.argv) > 3 else []) if kv]
CFG, SHAPE = bench.CFG, bench.SHAPE
H, Hkv, d = SHAPE["n_heads"], SHAPE["n_kv_heads"], SHAPE["head_dim"]
dev = torch.device("cuda")
g = torch.Generator(device=dev)
g.manual_seed(ctx)
Q = torch.randn((ctx, H, d), generator=g, device=dev).bfloat16()
K = torch.randn((ctx, Hkv, d), generator=g, device=dev).bfloat16()
V = torch.randn((ctx, Hkv, d), generator=g, device=dev).bfloat16()
steps, warm = 48, 4
engs = []
for _ in range(n_eng):
    e = StreamEngine(EngineConfig.make(**CFG), ModelShape.make(**SHAPE), dtype=torch.bfloat16)
    e.reserve(ctx + 3 * (steps + warm) + 8)
    for k_, v_ in opts:
        e.set_option(k_, int(v_))
    e.encode_stream(Q, K, V)
    engs.append(e)
del Q, K, V
qd = torch.randn((3 * (steps + warm), H, d), generator=g, device=dev).bfloat16()
kd = torch.randn((3 * (steps + warm), Hkv, d), generator=g, device=dev).bfloat16()
vd = torch.randn((3 * (steps + warm), Hkv, d), generator=g, device=dev).bfloat16()
res = torch.empty((1, H, d), device=dev, dtype=torch.bfloat16)
lib_ = _lib.lib()
st_ = torch.cuda.current_stream(dev).cuda_stream
t = 0
for rnd in range(3):
    for _ in range(warm):
        decode_batch(engs[:1], qd[t:t + 1], kd[t:t + 1], vd[t:t + 1], out=res)
        t += 1
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        _lib.check(lib_.infllm_decode_step(engs[0].h, 0, qd[t + i].data_ptr(), kd[t + i].data_ptr(),
                                           vd[t + i].data_ptr(), res.data_ptr(), st_))
    e1.record()
    torch.cuda.synchronize()
    t += steps
    print(f"ctx={ctx} engines={n_eng} {opts}: round {rnd} {1e3 * e0.elapsed_time(e1) / steps:.2f} us/step", flush=True)
