python tools/opt_ab.py "" "" > gpurun_out/t5_ab.log 2>&1; echo ab_rc=$?
python tools/timeline.py > gpurun_out/t5_tl.log 2>&1; echo tl_rc=$?
python -m pytest tests/test_gpu_streams.py tests/test_gpu_parity.py tests/test_gpu_decode.py -x -q > gpurun_out/t5_pytest.log 2>&1; echo pytest_rc=$?
