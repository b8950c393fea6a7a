# Device timeline of single-sequence decode steps at the C2 shape after a prefill
# of n tokens: per-step kernel spans and idle gaps (is a step GPU- or host-bound?).
#   python tools/decode_timeline.py [n_tokens] [steps] [opt=val,...]
import ctypes as C, sys, time, torch, numpy as np
sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, _lib
import bench
KINDS = ["attn", "rope", "prep", "prefix", "lookup", "topk", "evict", "select", "lru", "tier", "dec", "dec_front", "mass"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 64
g = torch.Generator(device='cuda'); g.manual_seed(0)
Q = torch.randn((n, 32, 128), generator=g, device='cuda').bfloat16()
K = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
V = torch.randn((n, 8, 128), generator=g, device='cuda').bfloat16()
eng = StreamEngine(EngineConfig.make(**bench.CFG), ModelShape.make(**bench.SHAPE), dtype=torch.bfloat16)
eng.reserve(n + steps + 64)
for kv in filter(None, (sys.argv[3] if len(sys.argv) > 3 else "").split(",")):
    k_, v_ = kv.split("=")
    eng.set_option(k_, int(v_))
eng.encode_stream(Q, K, V)
qd = torch.randn((steps + 16, 1, 32, 128), generator=g, device='cuda').bfloat16()
kd = torch.randn((steps + 16, 1, 8, 128), generator=g, device='cuda').bfloat16()
vd = torch.randn((steps + 16, 1, 8, 128), generator=g, device='cuda').bfloat16()
for t in range(16):
    eng.decode_step(qd[t], kd[t], vd[t])
torch.cuda.synchronize()
L = _lib.lib()
cap = 1 << 18
_lib.check(L.infllm_timeline_enable(cap))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
a.record()
for t in range(steps):
    eng.decode_step(qd[16 + t], kd[16 + t], vd[16 + t])
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
print(f"U={eng.metrics()['units']}: host launch time {host:.1f} us/step, device (events) {dev:.1f} us/step")
# busy intervals: union of all block intervals
order = np.argsort(t0a)
busy, cur0, cur1 = 0, None, None
for i in order:
    if cur1 is None or t0a[i] > cur1:
        if cur1 is not None:
            busy += cur1 - cur0
        cur0, cur1 = t0a[i], t1a[i]
    else:
        cur1 = max(cur1, t1a[i])
busy += cur1 - cur0
span = t1a.max() - t0a.min()
print(f"device busy (any kernel running) {busy / steps / 1e3:.1f} us/step of {span / steps / 1e3:.1f} us/step span")
for k in range(len(KINDS)):
    s = kid == k
    if s.any():
        # per-launch spans by clustering starts
        idx = np.where(s)[0]; idx = idx[np.argsort(t0a[idx])]
        cut = np.where(np.diff(t0a[idx]) > 3000)[0] + 1
        segs = np.split(idx, cut)
        spans = [(t1a[x].max() - t0a[x].min()) / 1e3 for x in segs]
        print(f"  {KINDS[k]:9s} launches {len(segs):4d} span us median {np.median(spans):6.2f} blocks/launch {np.median([len(x) for x in segs]):.0f}")
for k in range(100, 160):
    s_ = kid == k
    if s_.any():
        d_ = (t1a[s_] - t0a[s_]) / 1e3
        print(f"  mark {k - 100:3d}: n {s_.sum():5d} median {np.median(d_):6.2f} us")
# one step's kernels (launch segments ordered by start), offsets from that step's lookup start
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
if len(lk) > 34:
    for j in (30, 31):
        a0, b0 = lk[j][0], lk[j + 1][0]
        print(f"step {j}: lookup-to-lookup {(b0 - a0) / 1e3:.2f} us")
        for s_ in segs_all:
            if a0 - 2000 <= s_[0] < b0:
                print(f"   {s_[2]:9s} {(s_[0] - a0) / 1e3:7.2f} .. {(s_[1] - a0) / 1e3:7.2f} us  ({s_[3]} blocks)")
        for mk_ in (120, 121, 122, 123, 150, 151, 152, 153):
            s_ = (kid == mk_) & (t0a >= a0 - 2000) & (t0a < b0)
            if s_.any():
                e_ = np.sort((t1a[s_] - a0) / 1e3)
                print(f"   mark {mk_ - 100}: ends min {e_[0]:6.2f} median {np.median(e_):6.2f} max {e_[-1]:6.2f} us (n {len(e_)})")
