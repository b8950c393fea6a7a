python tools/lib_ab.py paper_2402_04617_b200/libinfllm_b200.so paper_2402_04617_b200/libinfllm_b200.so:prep_after_lru=1 > gpurun_out/t22_ab.log 2>&1; echo ab_rc=$?
python tools/timeline.py 131072 prep_after_lru=1 > gpurun_out/t22_tl.log 2>&1; echo tl_rc=$?
