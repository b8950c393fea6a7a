# A/B of engine options on the C2 128K stream: ms per stream (CUDA events, best of N) and
# bitwise output equality against the first configuration.
#   python tools/opt_ab.py "" attn_splits=2
import sys, torch
sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine
import bench
n = 131072
g = torch.Generator(device='cuda'); g.manual_seed(0)
Q = torch.randn((n, 32, 128), generator=g, device='cuda').bfloat16()
K = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
V = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
ref = None
for spec in sys.argv[1:]:
    opts = dict(kv.split('=') for kv in spec.split(',') if kv)
    eng = StreamEngine(EngineConfig.make(**bench.CFG), ModelShape.make(**bench.SHAPE), dtype=torch.bfloat16)
    eng.reserve(n)
    for k2, v2 in opts.items():
        eng.set_option(k2, int(v2))
    O = torch.empty_like(Q)
    ts = []
    for it in range(6):
        eng.reset(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); eng.encode_stream(Q, K, V, out=O); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    same = None
    if ref is None:
        ref = O.clone()
    else:
        same = bool(torch.equal(ref, O))
    print(f"{spec:30s} ms/stream best {min(ts[1:]):.3f} median {sorted(ts[1:])[2]:.3f}  us/step {1000*min(ts[1:])/256:.1f}  bitwise_same={same}", flush=True)
    eng.close()
