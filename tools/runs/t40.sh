timeout 600 python tools/shard_probe.py > gpurun_out/t40_shard.log 2>&1; echo shard_rc=$?
