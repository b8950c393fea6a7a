python tools/lib_ab.py paper_2402_04617_b200/libinfllm_b200.so tmp_libs/libprep4.so > gpurun_out/t12_ab.log 2>&1; echo ab_rc=$?
python tools/lookup_sweep.py 131072 48 > gpurun_out/t12_lk.log 2>&1; echo lk_rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_lookup_topk -s 3 -c 1 -o gpurun_out/t12_lookup python tools/lookup_sweep.py 131072 48 > gpurun_out/t12_ncu.log 2>&1; echo ncu_rc=$?
