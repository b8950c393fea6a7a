timeout 900 python tools/lib_ab.py tmp_libs/libhead.so tmp_libs/libtlc.so > gpurun_out/t85_ab.log 2>&1; echo rc=$?
timeout 400 python tools/dec_mode_ab.py 131072 decode_chain 1 3 > gpurun_out/t85_dec.log 2>&1; echo rc=$?
timeout 300 python tools/decode_timeline.py 131072 64 > gpurun_out/t85_tl.log 2>&1; echo rc=$?
