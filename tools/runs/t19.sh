python tools/decode_timeline.py > gpurun_out/t19_dec.log 2>&1; echo dec_rc=$?
python tools/decode_timeline.py 524288 > gpurun_out/t19_dec512.log 2>&1; echo dec512_rc=$?
python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/t19_pytest.log 2>&1; echo pytest_rc=$?
