python tools/lookup_probe.py > gpurun_out/t32_lk.log 2>&1; echo lk_rc=$?
python -m pytest tests/test_gpu_parity.py tests/test_gpu_streams.py tests/test_gpu_standalone.py -x -q > gpurun_out/t32_pytest.log 2>&1; echo pytest_rc=$?
python tools/lib_ab.py tmp_libs/libhead.so paper_2402_04617_b200/libinfllm_b200.so > gpurun_out/t32_ab.log 2>&1; echo ab_rc=$?
