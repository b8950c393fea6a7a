timeout 900 python -m pytest tests/test_gpu_decode.py -x -q -k merge > gpurun_out/t66_pytest.log 2>&1; echo pytest_rc=$?
bash tools/runs/r02_final.sh
