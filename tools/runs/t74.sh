timeout 300 python tools/decode_timeline.py 131072 64 > gpurun_out/t74_dec.log 2>&1; echo rc=$?
timeout 300 python tools/decode_timeline.py 131072 64 decode_chain=1 > gpurun_out/t74_dec1.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_streams.py -x -q > gpurun_out/t74_pytest.log 2>&1; echo pytest_rc=$?
