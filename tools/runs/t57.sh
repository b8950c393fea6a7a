timeout 900 python -m pytest tests/test_gpu_streams.py -x -q -k c4 -s > gpurun_out/t57_pytest.log 2>&1; echo pytest_rc=$?
