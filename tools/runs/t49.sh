timeout 600 python tools/decode_host_cost.py 8192 > gpurun_out/t49_host.log 2>&1; echo rc=$?
timeout 600 python tools/decode_host_cost.py 131072 > gpurun_out/t49_host128.log 2>&1; echo rc=$?
