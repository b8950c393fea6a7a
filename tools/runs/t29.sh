timeout 300 python tools/decode_timeline.py 131072 64 > gpurun_out/t29_dec.log 2>&1; echo dec_rc=$?
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity.py -x -q > gpurun_out/t29_pytest.log 2>&1; echo pytest_rc=$?
