python -m pytest tests -m gpu -x -q > gpurun_out/t1_pytest.log 2>&1; echo pytest_rc=$?
python tools/opt_ab.py "" "" > gpurun_out/t1_ab.log 2>&1; echo ab_rc=$?
python tools/timeline.py > gpurun_out/t1_tl.log 2>&1; echo tl_rc=$?
