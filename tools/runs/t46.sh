python -m pytest tests -m gpu -x -q > gpurun_out/t46_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --steps 10 --warmup 3 --no-extra > gpurun_out/t46_bench.json 2> gpurun_out/t46_bench.err; echo bench_rc=$?
