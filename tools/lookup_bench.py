# standalone lookup (infllm_lookup: relevance scan + exact top-k) throughput vs unit count
import sys
sys.path.insert(0, '.')
import torch
from paper_2402_04617_b200 import lookup
G, rk, d = 8, 4, 128
km = int(sys.argv[1]) if len(sys.argv) > 1 else 16
for U in [991, 8159, 32768, 131072]:
    repr_keys = torch.randn(U, G, rk, d, device="cuda").bfloat16()
    qsum = torch.randn(G, d, device="cuda", dtype=torch.float64)
    for _ in range(3):
        lookup(qsum, repr_keys, km)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        lookup(qsum, repr_keys, km)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / n * 1000
    b = U * G * rk * d * 2
    print(f"U={U:6d}: {us:8.2f} us per lookup, index {b/1e6:7.1f} MB -> {b / us / 1e3:7.1f} GB/s", flush=True)
