timeout 300 python tools/decode_timeline.py 131072 64 > gpurun_out/t70_dec.log 2>&1; echo rc=$?
timeout 300 python tools/decode_timeline.py 524288 64 > gpurun_out/t70_dec512.log 2>&1; echo rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t70_pytest.log 2>&1; echo pytest_rc=$?
