timeout 1200 python tools/dec_batch_ab.py 524288 4 tmp_libs/libhead.so tmp_libs/libtk512.so > gpurun_out/t118_ab.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/t118_pytest.log 2>&1; echo pytest_rc=$?
