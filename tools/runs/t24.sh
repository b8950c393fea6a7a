python -m pytest tests -m gpu -x -q > gpurun_out/t24_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --steps 10 --warmup 3 > gpurun_out/t24_bench.json 2> gpurun_out/t24_bench.err; echo bench_rc=$?
