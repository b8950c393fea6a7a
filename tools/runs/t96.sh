timeout 1200 python bench.py > gpurun_out/t96_bench.json 2> gpurun_out/t96_bench.err; echo bench_rc=$?
