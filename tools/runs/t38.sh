python tools/lib_ab.py paper_2402_04617_b200/libinfllm_b200.so tmp_libs/libturn0.so tmp_libs/libpoly4.so tmp_libs/libcl4.so > gpurun_out/t38_ab.log 2>&1; echo ab_rc=$?
