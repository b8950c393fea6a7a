./tools/tail_bench > gpurun_out/t103_tail.log 2>&1; echo rc=$?
