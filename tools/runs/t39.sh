python tools/lk_ab.py paper_2402_04617_b200/libinfllm_b200.so tmp_libs/libiw.so > gpurun_out/t39_lk.log 2>&1; echo lk_rc=$?
python tools/lib_ab.py paper_2402_04617_b200/libinfllm_b200.so tmp_libs/libiw.so > gpurun_out/t39_ab.log 2>&1; echo ab_rc=$?
