timeout 1500 python tools/lib_ab.py tmp_libs/libfinal.so tmp_libs/libprep4.so > gpurun_out/t101_ab.log 2>&1; echo rc=$?
