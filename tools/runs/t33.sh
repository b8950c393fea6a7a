timeout 300 python tools/decode_timeline.py 131072 64 > gpurun_out/t33_dec.log 2>&1; echo dec_rc=$?
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity.py tests/test_gpu_streams.py -x -q > gpurun_out/t33_pytest.log 2>&1; echo pytest_rc=$?
