timeout 900 python tools/dec_batch_stall.py 131072 16 20 > gpurun_out/t110_stall.log 2>&1; echo rc=$?
