timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t82_pytest.log 2>&1; echo pytest_rc=$?
timeout 900 python bench.py > gpurun_out/t82_bench.json 2> gpurun_out/t82_bench.err; echo bench_rc=$?
