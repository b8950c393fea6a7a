timeout 600 python tools/decode_host_cost.py 8192 > gpurun_out/t51_host.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/t51_pytest.log 2>&1; echo pytest_rc=$?
