import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine
C0 = dict(chunk_size=128, unit_size=128, n_repr=4, local_size=512, init_size=64, n_lookup=4, hot_capacity=32, decay=0.1)
n=2048
shape = O.ModelShape.make(n_heads=1, head_dim=64)
q, k, v = O.adapter_batch(0, shape, O.noise_ids(0, n))
oe = O.OracleEngine(O.EngineConfig.make(**C0), shape)
ge = StreamEngine(EngineConfig.make(**C0), ModelShape.make(n_heads=1, head_dim=64), dtype=torch.float32)
qt,kt,vt=[torch.from_numpy(x).cuda() for x in (q,k,v)]
for s in range(14):
    a=s*128
    r=oe.step(q[a:a+128],k[a:a+128],v[a:a+128])
    g=ge.step(qt[a:a+128].contiguous(),kt[a:a+128].contiguous(),vt[a:a+128].contiguous())
    om,gm=oe.metrics(),ge.metrics()
    print(s, r.retrieved_ids, g.retrieved_ids, om['units'], gm['units'], np.abs(r.out-g.out.cpu().numpy()).max())
    print('  state', oe.stream_state(), ge.stream_state())
    for u in range(om['units']):
        oi, gi = oe.unit_info(u), ge.unit_info(u)
        if oi != gi: print('  unit', u, oi, gi)
    es = oe.evicted_scores()
    print('  n evicted scores', len(es), es[:6])
