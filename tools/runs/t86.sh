timeout 900 python tools/lib_ab.py tmp_libs/libhead.so tmp_libs/libev.so > gpurun_out/t86_ab.log 2>&1; echo rc=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_streams.py -x -q > gpurun_out/t86_pytest.log 2>&1; echo pytest_rc=$?
