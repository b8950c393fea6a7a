# A/B of library builds on the host-buffer C2 stream (infllm_encode_stream_host,
# pinned q/k/v/out, H2D/D2H inside the timed region): wall ms per 128K stream,
# best of 5, runs interleaved in fresh subprocesses.
#   python tools/e2e_ab.py paper_2402_04617_b200/libinfllm_b200.so tmp_libs/libX.so
import subprocess
import sys

CHILD = r'''
import sys, time, torch
sys.path.insert(0, '.')
import paper_2402_04617_b200._lib as L
L.LIB_PATH = sys.argv[1]
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine
import bench
n = 131072
g = torch.Generator(device='cuda'); g.manual_seed(0)
Q = torch.randn((n, 32, 128), generator=g, device='cuda').bfloat16()
K = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
V = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
eng = StreamEngine(EngineConfig.make(**bench.CFG), ModelShape.make(**bench.SHAPE), dtype=torch.bfloat16)
eng.reserve(n)
Hq, Hk, Hv = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in (Q, K, V)]
Hq.copy_(Q); Hk.copy_(K); Hv.copy_(V)
Ho = torch.empty(Q.shape, dtype=Q.dtype, pin_memory=True)
ts = []
for it in range(6):
    eng.reset(); torch.cuda.synchronize()
    t0 = time.perf_counter(); eng.encode_stream_host(Hq, Hk, Hv, Ho); torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
print(f"{sys.argv[1]:50s} host-buffer stream ms best {min(ts[1:]):.2f} median {sorted(ts[1:])[2]:.2f} -> {n / min(ts[1:]) / 1e3:.3f} Mtok/s", flush=True)
'''
for rnd in range(2):
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, "-c", CHILD, lib], check=False)
