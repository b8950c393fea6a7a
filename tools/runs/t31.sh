python tools/lib_ab.py tmp_libs/libhead.so paper_2402_04617_b200/libinfllm_b200.so > gpurun_out/t31_ab.log 2>&1; echo ab_rc=$?
python bench.py --steps 10 --warmup 3 > gpurun_out/t31_bench.json 2> gpurun_out/t31_bench.err; echo bench_rc=$?
