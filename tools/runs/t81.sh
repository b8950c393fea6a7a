timeout 600 python tools/decode_host_cost.py 131072 > gpurun_out/t81_host.log 2>&1; echo rc=$?
timeout 300 python tools/decode_batch_timeline.py 131072 4 32 > gpurun_out/t81_b4.log 2>&1; echo rc=$?
