python tools/e2e_ab.py paper_2402_04617_b200/libinfllm_b200.so tmp_libs/libg8.so tmp_libs/libg4.so > gpurun_out/t36_e2e.log 2>&1; echo e2e_rc=$?
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q -k chain > gpurun_out/t36_pytest.log 2>&1; echo pytest_rc=$?
