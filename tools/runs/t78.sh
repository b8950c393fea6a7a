timeout 300 python tools/decode_batch_timeline.py 131072 2 32 > gpurun_out/t78_b2.log 2>&1; echo rc=$?
timeout 300 python tools/decode_batch_timeline.py 131072 32 32 > gpurun_out/t78_b32.log 2>&1; echo rc=$?
