timeout 300 python tools/e2e_probe.py > gpurun_out/t83_probe.log 2>&1; echo rc=$?
timeout 600 python bench.py --no-extra --no-cpu > gpurun_out/t83_bench.json 2> gpurun_out/t83_bench.err; echo bench_rc=$?
nvidia-smi -q | grep -i -A3 "Link Width\|PCIe Generation" | head -20 > gpurun_out/t83_pcie.txt
