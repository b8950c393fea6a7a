python bench.py --no-cpu --no-e2e > gpurun_out/t109_bench.json 2> gpurun_out/t109_bench.err; echo bench_rc=$?
