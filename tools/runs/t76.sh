timeout 300 python tools/decode_timeline.py 131072 64 > gpurun_out/t76_dec.log 2>&1; echo rc=$?
timeout 300 python tools/decode_timeline.py 131072 64 decode_chain=1 > gpurun_out/t76_dec1.log 2>&1; echo rc=$?
