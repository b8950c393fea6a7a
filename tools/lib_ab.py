# A/B of library builds on the C2 128K stream: each argument is a path to a
# libinfllm_b200.so variant (e.g. under tmp_libs/, built with a kernel change);
# runs are interleaved (A B A B ...) in fresh subprocesses, ms per stream best of 5.
# A path may carry engine options: lib.so:opt=1,opt2=0
#   python tools/lib_ab.py paper_2402_04617_b200/libinfllm_b200.so tmp_libs/libX.so
import subprocess
import sys

CHILD = r'''
import sys, torch
sys.path.insert(0, '.')
import paper_2402_04617_b200._lib as L
path, _, opts = sys.argv[1].partition(':')
L.LIB_PATH = path
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine
import bench
n = 131072
g = torch.Generator(device='cuda'); g.manual_seed(0)
Q = torch.randn((n, 32, 128), generator=g, device='cuda').bfloat16()
K = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
V = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
eng = StreamEngine(EngineConfig.make(**bench.CFG), ModelShape.make(**bench.SHAPE), dtype=torch.bfloat16)
eng.reserve(n)
for kv in filter(None, opts.split(',')):
    k2, v2 = kv.split('=')
    eng.set_option(k2, int(v2))
O = torch.empty_like(Q)
ts = []
for it in range(6):
    eng.reset(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); eng.encode_stream(Q, K, V, out=O); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
h = int(torch.sum(O.view(torch.int16).to(torch.int64) * torch.arange(O.numel(), device='cuda').view(O.shape) % 1000003).item())
print(f"{sys.argv[1]:50s} ms/stream best {min(ts[1:]):.3f} us/step {1000*min(ts[1:])/256:.1f} out_hash {h}", flush=True)
'''
libs = sys.argv[1:]
for rnd in range(2):
    for lib in libs:
        subprocess.run([sys.executable, "-c", CHILD, lib], check=False)
