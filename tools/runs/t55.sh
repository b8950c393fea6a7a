python tools/lk_ab.py paper_2402_04617_b200/libinfllm_b200.so tmp_libs/libnocomp.so > gpurun_out/t55_lk.log 2>&1; echo lk_rc=$?
