timeout 900 python tools/dec_batch_stall.py 131072 16 6 8 > gpurun_out/t112_stall.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/t112_pytest.log 2>&1; echo pytest_rc=$?
