timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t91_pytest.log 2>&1; echo pytest_rc=$?
timeout 600 python tools/dec_mode_ab.py 524288 decode_chain 1 3 > gpurun_out/t91_dec.log 2>&1; echo rc=$?
timeout 300 python tools/decode_timeline.py 524288 64 > gpurun_out/t91_tl.log 2>&1; echo rc=$?
timeout 900 python tools/lib_ab.py tmp_libs/libhead.so tmp_libs/librank.so > gpurun_out/t91_ab.log 2>&1; echo rc=$?
