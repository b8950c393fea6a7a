timeout 1500 python -m pytest tests/test_gpu_decode.py tests/test_gpu_streams.py -x -q > gpurun_out/t93_pytest.log 2>&1; echo pytest_rc=$?
timeout 600 python tools/dec_mode_ab.py 131072 decode_select_threshold 0,1 3 > gpurun_out/t93_dec.log 2>&1; echo rc=$?
timeout 300 python tools/decode_timeline.py 131072 64 > gpurun_out/t93_tl.log 2>&1; echo rc=$?
