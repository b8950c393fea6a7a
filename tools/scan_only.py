# one standalone relevance scan at 131072 units (for ncu)
import sys
sys.path.insert(0, '.')
import torch
from paper_2402_04617_b200 import lookup
U, G, rk, d = 131072, 8, 4, 128
reprk = torch.randn(U, G, rk, d, device="cuda").bfloat16()
qsum = torch.randn(G, d, device="cuda", dtype=torch.float64)
for _ in range(3):
    lookup(qsum, reprk, 0)
torch.cuda.synchronize()
print("ok")
