timeout 900 python tools/dec_batch_stall.py 131072 16 6 8 > gpurun_out/t111_stall.log 2>&1; echo rc=$?
