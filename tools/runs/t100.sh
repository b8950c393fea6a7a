timeout 900 python tools/dec_mode_ab.py 524288 lookup_units_per_block_decode 8,16,28 3 > gpurun_out/t100_dec.log 2>&1; echo rc=$?
