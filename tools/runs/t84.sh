timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_prep_tok -s 20 -c 2 -o gpurun_out/t84_prep python tools/short_stream.py 20480 > gpurun_out/t84_ncu.log 2>&1; echo rc=$?
