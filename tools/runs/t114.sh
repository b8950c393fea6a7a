timeout 900 python tools/dec_batch_ab.py 131072 4 tmp_libs/libhead.so tmp_libs/libtk256.so > gpurun_out/t114_ab.log 2>&1; echo rc=$?
timeout 1200 python tools/dec_batch_ab.py 131072 32 tmp_libs/libhead.so tmp_libs/libtk256.so >> gpurun_out/t114_ab.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/t114_pytest.log 2>&1; echo pytest_rc=$?
