cat /sys/bus/pci/devices/*/local_cpulist 2>/dev/null | sort | uniq -c | head -5 > gpurun_out/t117_numa.txt
nproc >> gpurun_out/t117_numa.txt
python bench.py --no-extra --no-cpu > gpurun_out/t117_bench.json 2> gpurun_out/t117_bench.err; echo bench_rc=$?
