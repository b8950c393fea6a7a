# PCIe ceiling vs the host-buffer stream path (C2 shapes)
import sys, time, torch
sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine
import bench
n = 131072
Q = torch.randn((n, 32, 128)).bfloat16().pin_memory()
K = torch.randn((n, 8, 128)).bfloat16().pin_memory()
V = torch.randn((n, 8, 128)).bfloat16().pin_memory()
O = torch.empty((n, 32, 128), dtype=torch.bfloat16).pin_memory()
dQ, dK, dV, dO = (torch.empty(x.shape, dtype=x.dtype, device="cuda") for x in (Q, K, V, O))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timeit(f, it=3):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(it): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / it * 1e3
h2d = lambda: (dQ.copy_(Q, non_blocking=True), dK.copy_(K, non_blocking=True), dV.copy_(V, non_blocking=True))
d2h = lambda: O.copy_(dO, non_blocking=True)
def both():
    with torch.cuda.stream(s1): h2d()
    with torch.cuda.stream(s2): d2h()
gb_in = (Q.numel() + K.numel() + V.numel()) * 2 / 1e9
gb_out = O.numel() * 2 / 1e9
t = timeit(h2d); print(f"H2D {gb_in:.2f} GB: {t:.1f} ms = {gb_in / t * 1e3:.1f} GB/s")
t = timeit(d2h); print(f"D2H {gb_out:.2f} GB: {t:.1f} ms = {gb_out / t * 1e3:.1f} GB/s")
t = timeit(both); print(f"both concurrently: {t:.1f} ms")
eng = StreamEngine(EngineConfig.make(**bench.CFG), ModelShape.make(**bench.SHAPE), dtype=torch.bfloat16)
eng.reserve(n)
def run():
    eng.reset(); eng.encode_stream_host(Q, K, V, O)
t = timeit(run); print(f"encode_stream_host: {t:.1f} ms = {n / t / 1e3:.2f} Mtok/s")
def dev():
    eng.reset(); eng.encode_stream(dQ, dK, dV, out=dO)
t = timeit(dev); print(f"encode_stream (device): {t:.1f} ms")
eng.set_option("cuda_graphs", 0)
t = timeit(run); print(f"encode_stream_host without graphs: {t:.1f} ms = {n / t / 1e3:.2f} Mtok/s")
C = 512
def chunked():
    for t in range(n // C):
        sl = slice(t * C, (t + 1) * C)
        with torch.cuda.stream(s1):
            dQ[sl].copy_(Q[sl], non_blocking=True); dK[sl].copy_(K[sl], non_blocking=True); dV[sl].copy_(V[sl], non_blocking=True)
        with torch.cuda.stream(s2):
            O[sl].copy_(dO[sl], non_blocking=True)
t = timeit(chunked); print(f"chunked copies both directions, no compute: {t:.1f} ms")
def chunked_h2d():
    for t in range(n // C):
        sl = slice(t * C, (t + 1) * C)
        with torch.cuda.stream(s1):
            dQ[sl].copy_(Q[sl], non_blocking=True); dK[sl].copy_(K[sl], non_blocking=True); dV[sl].copy_(V[sl], non_blocking=True)
t = timeit(chunked_h2d); print(f"chunked H2D only: {t:.1f} ms")
