# Device timeline of batched decode steps (infllm_decode_batch) at the C2 shape:
# per-stage launch spans (front, select, lookup scan, top-k, K4, LRU) per step.
#   python tools/decode_batch_timeline.py [ctx=131072] [B=32] [steps=32] [opt=val,...]
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, _lib, decode_batch  # noqa: E402
import bench  # noqa: E402

KINDS = ["attn", "rope", "prep", "prefix", "lookup", "topk", "evict", "select", "lru", "tier", "dec", "dec_front",
         "mass"]
ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 32
opts = [kv.split("=") for kv in (sys.argv[4].split(",") if len(sys.argv) > 4 else []) if kv]
cfg, shape = bench.CFG, bench.SHAPE
H, Hkv, d = shape["n_heads"], shape["n_kv_heads"], shape["head_dim"]
g = torch.Generator(device="cuda")
g.manual_seed(3)
Q = torch.randn((ctx, H, d), generator=g, device="cuda").bfloat16()
K = torch.randn((ctx, Hkv, d), generator=g, device="cuda").bfloat16()
V = torch.randn((ctx, Hkv, d), generator=g, device="cuda").bfloat16()
qd = torch.randn((steps + 8, B, H, d), generator=g, device="cuda").bfloat16()
kd = torch.randn((steps + 8, B, Hkv, d), generator=g, device="cuda").bfloat16()
vd = torch.randn((steps + 8, B, Hkv, d), generator=g, device="cuda").bfloat16()
out = torch.empty((B, H, d), device="cuda", dtype=torch.bfloat16)
engs = []
for _ in range(B):
    e = StreamEngine(EngineConfig.make(**cfg), ModelShape.make(**shape), dtype=torch.bfloat16)
    e.reserve(ctx + steps + 16)
    for k_, v_ in opts:
        e.set_option(k_, int(v_))
    e.encode_stream(Q, K, V)
    engs.append(e)
del Q, K, V
for t in range(4):
    decode_batch(engs, qd[t], kd[t], vd[t], out=out)
torch.cuda.synchronize()
L = _lib.lib()
cap = 1 << 20
_lib.check(L.infllm_timeline_enable(cap))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
a.record()
for t in range(steps):
    decode_batch(engs, qd[4 + t], kd[4 + t], vd[4 + t], out=out)
b.record()
host = (time.perf_counter() - t0) / steps * 1e6
torch.cuda.synchronize()
dev = a.elapsed_time(b) / steps * 1e3
kid = np.zeros(cap, np.uint32); sm = np.zeros(cap, np.uint32); t0a = np.zeros(cap, np.uint64); t1a = np.zeros(cap, np.uint64)
nn = C.c_int64()
_lib.check(L.infllm_timeline_read(kid.ctypes.data, sm.ctypes.data, t0a.ctypes.data, t1a.ctypes.data, cap, C.byref(nn), 1))
_lib.check(L.infllm_timeline_enable(0))
m = min(nn.value, cap)
kid, t0a, t1a = kid[:m], t0a[:m].astype(np.int64), t1a[:m].astype(np.int64)
print(f"B={B} ctx={ctx}: host {host:.1f} us/step, device (events) {dev:.1f} us/step")
for k in range(len(KINDS)):
    s = kid == k
    if s.any():
        idx = np.where(s)[0]; idx = idx[np.argsort(t0a[idx])]
        cut = np.where(np.diff(t0a[idx]) > 5000)[0] + 1
        segs = np.split(idx, cut)
        spans = [(t1a[x].max() - t0a[x].min()) / 1e3 for x in segs]
        print(f"  {KINDS[k]:9s} launches {len(segs):4d} span us median {np.median(spans):7.2f} blocks/launch "
              f"{np.median([len(x) for x in segs]):.0f}")
# one step's launches ordered by start, offsets from that step's lookup-scan start
segs_all = []
for k in range(len(KINDS)):
    idx = np.where(kid == k)[0]
    if not len(idx):
        continue
    idx = idx[np.argsort(t0a[idx])]
    cut = np.where(np.diff(t0a[idx]) > 3000)[0] + 1
    for x in np.split(idx, cut):
        segs_all.append((t0a[x].min(), t1a[x].max(), KINDS[k], len(x)))
segs_all.sort()
lk = [s_ for s_ in segs_all if s_[2] == "lookup"]
if len(lk) > steps // 2 + 2:
    j = steps // 2
    a0, b0 = lk[j][0], lk[j + 1][0]
    print(f"step {j}: lookup-to-lookup {(b0 - a0) / 1e3:.2f} us")
    for s_ in segs_all:
        if a0 - 30000 <= s_[0] < b0:
            print(f"   {s_[2]:9s} {(s_[0] - a0) / 1e3:7.2f} .. {(s_[1] - a0) / 1e3:7.2f} us  ({s_[3]} blocks)")
