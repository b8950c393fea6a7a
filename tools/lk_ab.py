# Standalone lookup timing (infllm_lookup, graph-timed) for library variants:
#   python tools/lk_ab.py lib1.so lib2.so ...
import subprocess
import sys

CHILD = r'''
import sys, torch
sys.path.insert(0, '.')
import paper_2402_04617_b200._lib as L
L.LIB_PATH = sys.argv[1]
lib = L.lib()
G, RK, D, KM = 8, 4, 128, 16
res = []
for U in (991, 8159, 131072):
    reprk = torch.randn(U, G, RK, D, device="cuda").bfloat16()
    qsum = torch.randn(G, D, device="cuda", dtype=torch.float64)
    rel = torch.empty(U, device="cuda", dtype=torch.float64)
    ids = torch.empty(KM, device="cuda", dtype=torch.int64)
    s = torch.cuda.Stream()
    def call():
        L.check(lib.infllm_lookup(qsum.data_ptr(), reprk.data_ptr(), L.DTYPE_BF16, U, RK, G, D, KM, rel.data_ptr(), ids.data_ptr(), s.cuda_stream))
    with torch.cuda.stream(s):
        call(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20): call()
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); g.replay(); e1.record(s); torch.cuda.synchronize()
    res.append(f"U={U}: {e0.elapsed_time(e1) / 20 * 1000:.2f} us")
print(f"{sys.argv[1]:40s} " + "  ".join(res), flush=True)
'''
for rnd in range(2):
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, "-c", CHILD, lib], check=False)
