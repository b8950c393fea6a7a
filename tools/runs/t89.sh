timeout 600 python tools/dec_mode_ab.py 524288 decode_lookup_fused 0,1 3 > gpurun_out/t89_dec.log 2>&1; echo rc=$?
timeout 300 python tools/decode_timeline.py 524288 64 decode_lookup_fused=1 > gpurun_out/t89_tl.log 2>&1; echo rc=$?
