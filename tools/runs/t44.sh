python tools/e2e_ab.py tmp_libs/libhead.so paper_2402_04617_b200/libinfllm_b200.so > gpurun_out/t44_e2e.log 2>&1; echo e2e_rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -k "host or stream or golden or cli" > gpurun_out/t44_pytest.log 2>&1; echo pytest_rc=$?
