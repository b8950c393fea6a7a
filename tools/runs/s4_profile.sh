set -x
timeout 600 python tools/decode_bench.py 131072,524288 1,2,4,8,16,32 32 batched > gpurun_out/s4_decode_grid.jsonl 2> gpurun_out/s4_decode_grid.err
timeout 300 python tools/decode_bench.py 131072,524288 1 32 streams > gpurun_out/s4_decode_single.jsonl 2>> gpurun_out/s4_decode_grid.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 4048 -c 1012 --csv --log-file gpurun_out/s4_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-extra > gpurun_out/s4_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attn_tc -s 60 -c 1 -o gpurun_out/s4_attn python tools/kbench.py 131072 2 > gpurun_out/s4_ncu_full.log 2>&1
echo done
