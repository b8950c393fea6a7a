python tools/opt_ab.py "" "attn_streams=1" "" > gpurun_out/t4_ab.log 2>&1; echo ab_rc=$?
python tools/timeline.py > gpurun_out/t4_tl.log 2>&1; echo tl_rc=$?
python -m pytest tests -m gpu -x -q > gpurun_out/t4_pytest.log 2>&1; echo pytest_rc=$?
