python tools/lib_ab.py tmp_libs/libhead.so paper_2402_04617_b200/libinfllm_b200.so tmp_libs/libprep2.so > gpurun_out/t6_ab.log 2>&1; echo ab_rc=$?
python tools/timeline.py > gpurun_out/t6_tl.log 2>&1; echo tl_rc=$?
python -m pytest tests/test_gpu_streams.py tests/test_gpu_parity.py tests/test_gpu_decode.py tests/test_gpu_standalone.py -x -q > gpurun_out/t6_pytest.log 2>&1; echo pytest_rc=$?
