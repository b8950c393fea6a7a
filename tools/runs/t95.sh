timeout 900 python tools/dec_grid_probe.py 524288 32 decode_lookup_fused=1 > gpurun_out/t95_a.log 2>&1; echo rc=$?
timeout 900 python tools/dec_grid_probe.py 524288 32 decode_lookup_fused=0 > gpurun_out/t95_b.log 2>&1; echo rc=$?
timeout 900 python tools/dec_grid_probe.py 524288 1 decode_lookup_fused=1 > gpurun_out/t95_c.log 2>&1; echo rc=$?
