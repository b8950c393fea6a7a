timeout 900 python tools/dec_batch_ab.py 131072 2 tmp_libs/libhead.so tmp_libs/libk4c.so > gpurun_out/t116_ab.log 2>&1; echo rc=$?
timeout 900 python tools/dec_batch_ab.py 131072 4 tmp_libs/libhead.so tmp_libs/libk4c.so >> gpurun_out/t116_ab.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/t116_pytest.log 2>&1; echo pytest_rc=$?
