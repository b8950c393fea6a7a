python tools/e2e_probe.py > gpurun_out/t43_probe.log 2>&1; echo probe_rc=$?
python tools/e2e_ab.py paper_2402_04617_b200/libinfllm_b200.so tmp_libs/libnb4.so tmp_libs/libg12.so > gpurun_out/t43_e2e.log 2>&1; echo e2e_rc=$?
