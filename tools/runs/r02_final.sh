set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/fin5_smi.txt
python -m pytest tests -m gpu -x -q > gpurun_out/fin5_pytest.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin5_smoke.log 2>&1; echo smoke_rc=$?
python bench.py --steps 10 --warmup 3 > gpurun_out/fin5_bench.json 2> gpurun_out/fin5_bench.err; echo bench_rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin5_bench_ref.json 2> gpurun_out/fin5_bench_ref.err; echo ref_rc=$?
python bench.py --steps 2 --warmup 3 --no-extra --no-cpu --no-e2e > gpurun_out/fin5_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 600 --csv --log-file gpurun_out/fin5_launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu --no-e2e > gpurun_out/fin5_ncu_launch.log 2>&1; echo launch_rc=$?
python tools/short_stream.py 131072 > gpurun_out/fin5_short.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_attn_tc|k_lookup_topk|k_prep_tok|k_evict_warp|k_select" -s 1200 -c 5 -o gpurun_out/fin5_kernels python tools/short_stream.py 131072 > gpurun_out/fin5_ncu_full.log 2>&1; echo full_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_lookup_reg|k_attn_dec1|k_dec_merge1|k_dec_front" -s 40 -c 4 -o gpurun_out/fin5_decode python tools/dec_mode_ab.py 131072 decode_chain 1 1 > gpurun_out/fin5_ncu_dec.log 2>&1; echo dec_rc=$?
