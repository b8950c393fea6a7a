timeout 600 python tools/shard_probe.py > gpurun_out/t41_shard.log 2>&1; echo shard_rc=$?
timeout 900 python -m pytest tests/test_gpu_split.py tests/test_gpu_shard.py tests/test_nccl_shard.py -x -q > gpurun_out/t41_pytest.log 2>&1; echo pytest_rc=$?
