timeout 600 python tools/decode_host_cost.py 131072 > gpurun_out/t53_host128.log 2>&1; echo rc=$?
timeout 600 python tools/decode_batch_timeline.py 131072 4 32 > gpurun_out/t53_b4.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/t53_pytest.log 2>&1; echo pytest_rc=$?
