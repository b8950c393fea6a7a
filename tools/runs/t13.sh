./tools/f64_rate > gpurun_out/t13_f64.log 2>&1; echo f64_rc=$?
python tools/lookup_probe.py > gpurun_out/t13_lk.log 2>&1; echo lk_rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_lookup_topk -s 30 -c 1 -o gpurun_out/t13_lookup991 python tools/lookup_probe.py 991 > gpurun_out/t13_ncu.log 2>&1; echo ncu_rc=$?
