for B in 2 4 8 16 32; do
for c in 1 0; do
timeout 300 python tools/decode_batch_timeline.py 131072 $B 32 decode_chain=$c 2>&1 | head -1 >> gpurun_out/t80_ab.log
done; done; echo done
