python tools/opt_ab.py "attn_streams=1" "" "attn_streams=1" "" > gpurun_out/t2_ab.log 2>&1; echo ab_rc=$?
python -m pytest tests -m gpu -x -q > gpurun_out/t2_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --steps 5 --warmup 3 --no-extra --no-cpu > gpurun_out/t2_bench.json 2> gpurun_out/t2_bench.err; echo bench_rc=$?
python tools/timeline.py > gpurun_out/t2_tl.log 2>&1; echo tl_rc=$?
