timeout 600 python tools/decode_batch_timeline.py 131072 32 32 > gpurun_out/t42_b32.log 2>&1; echo b32_rc=$?
timeout 600 python tools/decode_batch_timeline.py 131072 4 32 > gpurun_out/t42_b4.log 2>&1; echo b4_rc=$?
