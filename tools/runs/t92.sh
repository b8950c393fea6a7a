timeout 1500 python -m pytest tests/test_gpu_streams.py tests/test_gpu_parity.py tests/test_gpu_decode.py -x -q > gpurun_out/t92_pytest.log 2>&1; echo pytest_rc=$?
timeout 600 python tools/dec_mode_ab.py 524288 decode_chain 1 3 > gpurun_out/t92_dec.log 2>&1; echo rc=$?
timeout 300 python tools/decode_timeline.py 524288 64 > gpurun_out/t92_tl.log 2>&1; echo rc=$?
timeout 900 python tools/lib_ab.py tmp_libs/librank.so tmp_libs/libtau.so > gpurun_out/t92_ab.log 2>&1; echo rc=$?
