python tools/e2e_ab.py tmp_libs/libh2d1.so paper_2402_04617_b200/libinfllm_b200.so > gpurun_out/t56_e2e.log 2>&1; echo e2e_rc=$?
