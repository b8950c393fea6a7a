timeout 900 python -m pytest tests/test_gpu_host_tier.py -x -q -k c3_full > gpurun_out/t48_pytest.log 2>&1; echo pytest_rc=$?
