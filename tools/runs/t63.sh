timeout 300 python tools/decode_timeline.py 131072 64 > gpurun_out/t63_dec.log 2>&1; echo rc=$?
