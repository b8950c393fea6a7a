python tools/lib_ab.py tmp_libs/libhead.so paper_2402_04617_b200/libinfllm_b200.so > gpurun_out/t25_ab.log 2>&1; echo ab_rc=$?
python -m pytest tests/test_gpu_parity.py tests/test_gpu_streams.py -x -q > gpurun_out/t25_pytest.log 2>&1; echo pytest_rc=$?
