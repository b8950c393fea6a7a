timeout 300 python tools/decode_timeline.py 131072 64 > gpurun_out/t27_dec.log 2>&1; echo dec_rc=$?
timeout 300 python tools/decode_timeline.py 131072 64 decode_chain=0 > gpurun_out/t27_dec0.log 2>&1; echo dec0_rc=$?
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/t27_pytest.log 2>&1; echo pytest_rc=$?
