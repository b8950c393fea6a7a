timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity.py -x -q > gpurun_out/t26_pytest.log 2>&1; echo pytest_rc=$?
timeout 300 python tools/decode_timeline.py 131072 64 > gpurun_out/t26_dec.log 2>&1; echo dec_rc=$?
timeout 300 python tools/decode_timeline.py 131072 64 decode_chain=0 > gpurun_out/t26_dec0.log 2>&1; echo dec0_rc=$?
