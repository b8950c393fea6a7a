timeout 600 python tools/dec_mode_ab.py 131072 decode_select_threshold 0,1 3 > gpurun_out/t94_dec.log 2>&1; echo rc=$?
timeout 300 python tools/decode_timeline.py 131072 64 > gpurun_out/t94_tl.log 2>&1; echo rc=$?
