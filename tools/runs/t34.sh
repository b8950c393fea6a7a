for nb in 0 16 32 48 64; do timeout 300 python tools/decode_timeline.py 131072 64 decode_chain_lookup_blocks=$nb > gpurun_out/t34_dec$nb.log 2>&1; echo "nb=$nb rc=$?"; done
timeout 300 python tools/decode_timeline.py 131072 64 decode_chain=0 > gpurun_out/t34_dec_off.log 2>&1; echo off_rc=$?
