python -m pytest tests -m gpu -x -q > gpurun_out/t11_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --steps 10 --warmup 3 > gpurun_out/t11_bench.json 2> gpurun_out/t11_bench.err; echo bench_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t11_smoke.log 2>&1; echo smoke_rc=$?
