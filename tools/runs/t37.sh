timeout 900 python -m pytest tests/test_gpu_decode.py -x -q -k chain > gpurun_out/t37_pytest.log 2>&1; echo pytest_rc=$?
timeout 300 python tools/decode_timeline.py 524288 64 > gpurun_out/t37_dec512.log 2>&1; echo dec_rc=$?
timeout 300 python tools/decode_timeline.py 524288 64 decode_chain=0 > gpurun_out/t37_dec512_off.log 2>&1; echo dec0_rc=$?
timeout 300 python tools/decode_timeline.py 131072 64 > gpurun_out/t37_dec128.log 2>&1; echo dec128_rc=$?
python tools/e2e_ab.py paper_2402_04617_b200/libinfllm_b200.so tmp_libs/libg32.so > gpurun_out/t37_e2e.log 2>&1; echo e2e_rc=$?
