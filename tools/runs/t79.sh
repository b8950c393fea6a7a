timeout 300 python tools/decode_batch_timeline.py 131072 2 32 > gpurun_out/t79_b2.log 2>&1; echo rc=$?
timeout 300 python tools/decode_batch_timeline.py 131072 32 32 > gpurun_out/t79_b32.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/t79_pytest.log 2>&1; echo pytest_rc=$?
