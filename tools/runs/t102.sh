timeout 900 python tools/dec_mode_ab.py 131072 decode_chain 1,2 3 > gpurun_out/t102_dec.log 2>&1; echo rc=$?
timeout 900 python tools/dec_mode_ab.py 524288 decode_chain 1,2 3 >> gpurun_out/t102_dec.log 2>&1; echo rc=$?
timeout 1200 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/t102_pytest.log 2>&1; echo pytest_rc=$?
