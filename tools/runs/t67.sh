timeout 300 python tools/decode_timeline.py 131072 64 > gpurun_out/t67_dec.log 2>&1; echo rc=$?
timeout 300 python tools/decode_timeline.py 524288 64 > gpurun_out/t67_dec512.log 2>&1; echo rc=$?
