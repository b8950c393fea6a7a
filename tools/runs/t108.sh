timeout 1200 python tools/dec_batch_ab.py 131072 32 tmp_libs/libfb.so paper_2402_04617_b200/libinfllm_b200.so > gpurun_out/t108_ab.log 2>&1; echo rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t108_pytest.log 2>&1; echo pytest_rc=$?
