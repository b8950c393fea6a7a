nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/fin9_smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin9_smoke.log 2>&1; echo smoke_rc=$?
python bench.py --steps 10 --warmup 3 > gpurun_out/fin9_bench.json 2> gpurun_out/fin9_bench.err; echo bench_rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin9_bench_ref.json 2> gpurun_out/fin9_bench_ref.err; echo ref_rc=$?
python bench.py --steps 2 --warmup 3 --no-extra --no-cpu --no-e2e > gpurun_out/fin9_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 600 --csv --log-file gpurun_out/fin9_launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu --no-e2e > gpurun_out/fin9_ncu_launch.log 2>&1; echo launch_rc=$?
