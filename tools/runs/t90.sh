timeout 1500 python -m pytest tests/test_gpu_decode.py tests/test_gpu_streams.py tests/test_gpu_parity.py tests/test_gpu_host_tier.py -x -q > gpurun_out/t90_pytest.log 2>&1; echo pytest_rc=$?
