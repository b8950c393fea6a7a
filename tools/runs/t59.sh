python tools/lib_ab.py paper_2402_04617_b200/libinfllm_b200.so tmp_libs/libtile8.so > gpurun_out/t59_ab.log 2>&1; echo ab_rc=$?
