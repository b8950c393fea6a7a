# attention error vs the oracle for peaked softmaxes (large-norm bf16 inputs), tcgen05 vs CUDA-core path
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from oracle import oracle as O
from tests.parity_util import gaussian_inputs, run_pair, rel_err
cfg = dict(chunk_size=256, unit_size=128, n_repr=4, local_size=1024, init_size=128, n_lookup=8, hot_capacity=12)
n = 3072
for scale in [float(x) for x in sys.argv[1:]] or [3.0]:
    q, k, v = gaussian_inputs(11, n, 8, 2, 128, scale=scale, bf16=True)
    sched = O.encode_schedule(n, 256, 8)
    for tc in (True, False):
        oeng, geng, recs = run_pair(cfg, 8, 2, 128, q, k, v, sched, decode_tail=8, dtype=torch.bfloat16, tc=tc)
        errs = [rel_err(r["g_out"], r["o_out"]) for r in recs]
        worst = int(np.argmax(errs))
        r = recs[worst]
        d = np.abs(r["g_out"].astype(np.float64) - r["o_out"])
        idx = np.unravel_index(np.argmax(d), d.shape)
        print(f"scale {scale} tc={tc}: max rel err {max(errs):.3e} at step {worst} (b={r['b']}) token/head/dim {idx} "
              f"got {r['g_out'][idx]:.5f} want {r['o_out'][idx]:.5f}", flush=True)
