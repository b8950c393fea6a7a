timeout 300 python tools/decode_timeline.py 131072 64 > gpurun_out/t65_dec.log 2>&1; echo rc=$?
timeout 300 python tools/decode_timeline.py 131072 64 decode_merge_kernel=0 > gpurun_out/t65_dec0.log 2>&1; echo rc=$?
timeout 600 python tools/decode_host_cost.py 131072 > gpurun_out/t65_host.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_streams.py tests/test_gpu_parity.py tests/test_gpu_host_tier.py -x -q > gpurun_out/t65_pytest.log 2>&1; echo pytest_rc=$?
