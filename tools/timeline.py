# Device timeline of the C2 128K stream (infllm_timeline_*): per attention launch,
# the CTA start spread, CTA durations and the handover gap to the next launch,
# and which side kernels held SMs while the next launch's CTAs were waiting.
#   python tools/timeline.py [n_tokens] [opt=val,...]
import ctypes as C
import sys
from collections import Counter

import numpy as np
import torch

sys.path.insert(0, '.')
import bench
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, _lib

KINDS = ["attn", "rope", "prep", "prefix", "lookup", "topk", "evict", "select", "lru", "tier", "dec", "dec_front",
         "mass"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
opts = dict(kv.split('=') for kv in (sys.argv[2].split(',') if len(sys.argv) > 2 else []) if kv)
g = torch.Generator(device='cuda')
g.manual_seed(0)
Q = torch.randn((n, 32, 128), generator=g, device='cuda').bfloat16()
K = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
V = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
eng = StreamEngine(EngineConfig.make(**bench.CFG), ModelShape.make(**bench.SHAPE), dtype=torch.bfloat16)
eng.reserve(n)
for k, v in opts.items():
    eng.set_option(k, int(v))
O = torch.empty_like(Q)
for _ in range(2):
    eng.reset()
    eng.encode_stream(Q, K, V, out=O)
torch.cuda.synchronize()
L = _lib.lib()
cap = 1 << 21
_lib.check(L.infllm_timeline_enable(cap))
eng.reset()
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
eng.encode_stream(Q, K, V, out=O)
ev1.record()
torch.cuda.synchronize()
kid = np.zeros(cap, np.uint32)
sm = np.zeros(cap, np.uint32)
t0 = np.zeros(cap, np.uint64)
t1 = np.zeros(cap, np.uint64)
nn = C.c_int64()
_lib.check(L.infllm_timeline_read(kid.ctypes.data, sm.ctypes.data, t0.ctypes.data, t1.ctypes.data, cap, C.byref(nn), 1))
_lib.check(L.infllm_timeline_enable(0))
m = min(nn.value, cap)
kid, sm, t0, t1 = kid[:m], sm[:m], t0[:m].astype(np.int64), t1[:m].astype(np.int64)
base = t0.min()
t0 -= base
t1 -= base
print(f"stream {ev0.elapsed_time(ev1):.3f} ms (timeline on), {m} block records")
for k in range(100, 120):  # kernel phase marks (kid >= 100)
    sel = kid == k
    if sel.any():
        d = (t1[sel] - t0[sel]) / 1e3
        print(f"  phase {k - 100:3d}: n {sel.sum():6d} us mean {d.mean():7.2f} median {np.median(d):7.2f} max {d.max():7.2f}")
for k in range(len(KINDS)):
    sel = kid == k
    if sel.any():
        d = (t1[sel] - t0[sel]) / 1e3
        print(f"  {KINDS[k]:10s} blocks {sel.sum():7d}  block us mean {d.mean():6.2f} max {d.max():7.2f}  "
              f"busy SM-us {d.sum():9.0f}")
att = np.where(kid == 0)[0]
att = att[np.argsort(t0[att])]
per = 128
nl = len(att) // per
rows = []
for i in range(nl):
    idx = att[i * per:(i + 1) * per]
    rows.append((t0[idx].min(), t0[idx].max(), t1[idx].min(), t1[idx].max(), ((t1[idx] - t0[idx]) / 1e3).mean()))
rows = np.array(rows, np.float64)
spread = (rows[:, 1] - rows[:, 0]) / 1e3
span = (rows[:, 3] - rows[:, 0]) / 1e3
gap = (rows[1:, 0] - rows[:-1, 3]) / 1e3
print(f"attention launches {nl}: span us mean {span.mean():.2f} (median {np.median(span):.2f}); CTA dur mean "
      f"{rows[:, 4].mean():.2f}; start spread mean {spread.mean():.2f} max {spread.max():.2f}; "
      f"gap to next launch mean {gap.mean():.2f} max {gap.max():.2f}; step period "
      f"{(rows[-1, 0] - rows[0, 0]) / 1e3 / (nl - 1):.2f} us")
# side blocks overlapping the late-start window of each launch: [first CTA start, last CTA start]
late = Counter()
late_sm = Counter()
for i in range(20, nl):
    a, b = rows[i, 0], rows[i, 1]
    if b - a < 1000:
        continue
    o = (kid != 0) & (t0 < b) & (t1 > a)
    for k in np.unique(kid[o]):
        if k >= len(KINDS):
            continue
        late[KINDS[k]] += int(((kid == k) & o).sum())
        late_sm[KINDS[k]] += len(np.unique(sm[(kid == k) & o]))
print("side blocks overlapping the attention CTA start window (launches 20+):", dict(late))
print("distinct SMs per kind summed over launches:", dict(late_sm))
# steady-state per-step sequence of one step (window of launch 100)
if nl > 101:
    a, e = rows[100, 0], rows[101, 3]
    print("launch 100..101 window: kernel blocks starting inside, relative to launch-100 start (us):")
    o = (t0 >= a - 80000) & (t0 < e)
    for k in range(1, len(KINDS)):
        s2 = o & (kid == k)
        if s2.any():
            print(f"  {KINDS[k]:10s} n={s2.sum():4d} start [{(t0[s2].min() - a) / 1e3:8.2f}, {(t0[s2].max() - a) / 1e3:8.2f}] "
                  f"end max {(t1[s2].max() - a) / 1e3:8.2f} SMs {len(np.unique(sm[s2]))}")
    print(f"  attn 100: start [0, {(rows[100, 1] - a) / 1e3:.2f}] end [{(rows[100, 2] - a) / 1e3:.2f}, "
          f"{(rows[100, 3] - a) / 1e3:.2f}]; attn 101 start [{(rows[101, 0] - a) / 1e3:.2f}, {(rows[101, 1] - a) / 1e3:.2f}]")


def launches(k, thr_ns=10000):
    """Segments the blocks of kernel kind k into launches by start-time gaps."""
    idx = np.where(kid == k)[0]
    idx = idx[np.argsort(t0[idx])]
    if len(idx) == 0:
        return np.zeros((0, 4))
    cut = np.where(np.diff(t0[idx]) > thr_ns)[0] + 1
    segs = np.split(idx, cut)
    return np.array([(t0[s].min(), t0[s].max(), t1[s].max(), len(s)) for s in segs], np.float64)


LK = {KINDS[k]: launches(k) for k in range(1, len(KINDS)) if (kid == k).any()}
print("launch counts:", {k: len(v) for k, v in LK.items()})
# for each attention launch i >= 20: the latest-ending launch of each kind that ended before A_i's first CTA start
slack = {k: [] for k in LK}
for i in range(20, nl):
    s0 = rows[i, 0]
    for k, v in LK.items():
        before = v[v[:, 2] <= s0]
        if len(before):
            slack[k].append((s0 - before[:, 2].max()) / 1e3)
prev_end = (rows[20:, 0] - rows[19:-1, 3]) / 1e3
print(f"A_i first start - A_(i-1) last end: median {np.median(prev_end):.2f} p90 {np.percentile(prev_end, 90):.2f}")
for k, v in slack.items():
    if v:
        v = np.array(v)
        print(f"A_i first start - last {k:9s} end: median {np.median(v):7.2f} p10 {np.percentile(v, 10):7.2f} "
              f"min {v.min():7.2f}")
for k, v in LK.items():
    d = (v[:, 2] - v[:, 0]) / 1e3
    sp = (v[:, 1] - v[:, 0]) / 1e3
    print(f"{k:9s} launch span us median {np.median(d):7.2f} p90 {np.percentile(d, 90):7.2f}; block start spread "
          f"median {np.median(sp):6.2f}; blocks/launch {np.median(v[:, 3]):.0f}")

# at each handoff (A_(i-1) last CTA end): side blocks resident then, and side
# blocks that started between that moment and A_i's last CTA start
res = Counter()
res_sm = []
started = Counter()
for i in range(20, nl):
    T = rows[i - 1, 3]
    o = (kid != 0) & (kid < len(KINDS)) & (t0 <= T) & (t1 > T)
    for k in np.unique(kid[o]):
        res[KINDS[k]] += int(((kid == k) & o).sum())
    res_sm.append(len(np.unique(sm[o])))
    w = (kid != 0) & (kid < len(KINDS)) & (t0 > T) & (t0 < rows[i, 1])
    for k in np.unique(kid[w]):
        started[KINDS[k]] += int(((kid == k) & w).sum())
n_h = max(1, nl - 20)
print("side blocks resident at the handoff (per handoff):", {k: round(v / n_h, 1) for k, v in res.items()},
      f"SMs with a side block: median {np.median(res_sm):.0f}")
print("side blocks started between the handoff and the last attention CTA start (per handoff):",
      {k: round(v / n_h, 1) for k, v in started.items()})
