python tools/lib_ab.py paper_2402_04617_b200/libinfllm_b200.so paper_2402_04617_b200/libinfllm_b200.so:prep_gate=1 > gpurun_out/t8_ab.log 2>&1; echo ab_rc=$?
python tools/timeline.py 131072 prep_gate=1 > gpurun_out/t8_tl.log 2>&1; echo tl_rc=$?
python tools/timeline.py 131072 > gpurun_out/t8_tl0.log 2>&1; echo tl0_rc=$?
