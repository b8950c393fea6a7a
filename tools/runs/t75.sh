timeout 400 python tools/dec_mode_ab.py 131072 decode_chain 1,2 3 > gpurun_out/t75_ab.log 2>&1; echo rc=$?
timeout 300 python tools/decode_timeline.py 131072 64 > gpurun_out/t75_dec.log 2>&1; echo rc=$?
