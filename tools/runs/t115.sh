timeout 900 python tools/dec_batch_ab.py 131072 8 tmp_libs/libhead.so tmp_libs/libk4p.so > gpurun_out/t115_ab.log 2>&1; echo rc=$?
timeout 1200 python tools/dec_batch_ab.py 131072 32 tmp_libs/libhead.so tmp_libs/libk4p.so >> gpurun_out/t115_ab.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/t115_pytest.log 2>&1; echo pytest_rc=$?
