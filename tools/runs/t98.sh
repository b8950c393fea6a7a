for r in 1 2; do
for L in tmp_libs/libhead.so tmp_libs/libmrec.so; do
DEC_AB_LIB=$L timeout 600 python tools/dec_mode_ab.py 131072 decode_chain 1 3 2>&1 | sed "s|^|$L |" >> gpurun_out/t98_dec.log
done; done; echo done
