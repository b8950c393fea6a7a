python tools/lib_ab.py tmp_libs/libhead.so paper_2402_04617_b200/libinfllm_b200.so tmp_libs/libprep2.so tmp_libs/libprep1.so paper_2402_04617_b200/libinfllm_b200.so:prep_gate=1 tmp_libs/libprep2.so:prep_gate=1 > gpurun_out/t7_ab.log 2>&1; echo ab_rc=$?
python -m pytest tests/test_gpu_streams.py tests/test_gpu_parity.py -x -q > gpurun_out/t7_pytest.log 2>&1; echo pytest_rc=$?
