timeout 600 python tools/decode_batch_timeline.py 8192 4 32 > gpurun_out/t52_b4.log 2>&1; echo rc=$?
timeout 600 python tools/decode_batch_timeline.py 8192 32 32 > gpurun_out/t52_b32.log 2>&1; echo rc=$?
