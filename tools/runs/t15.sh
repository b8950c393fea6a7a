python tools/lookup_probe.py > gpurun_out/t15_lk.log 2>&1; echo lk_rc=$?
python tools/decode_timeline.py > gpurun_out/t15_dec.log 2>&1; echo dec_rc=$?
