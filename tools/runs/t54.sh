python -m pytest tests -m gpu -x -q > gpurun_out/t54_pytest.log 2>&1; echo pytest_rc=$?
