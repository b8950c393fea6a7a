timeout 600 python tools/decode_host_cost.py 8192 > gpurun_out/t50_host.log 2>&1; echo rc=$?
