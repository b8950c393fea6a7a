python -m pytest tests -x -q -m gpu > gpurun_out/t113_pytest.log 2>&1; echo pytest_rc=$?
