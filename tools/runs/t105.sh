python -m pytest tests -x -q -m gpu > gpurun_out/t105_pytest.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t105_smoke.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/t105_bench.json 2> gpurun_out/t105_bench.err; echo bench_rc=$?
