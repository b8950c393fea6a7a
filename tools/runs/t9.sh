python tools/lib_ab.py paper_2402_04617_b200/libinfllm_b200.so paper_2402_04617_b200/libinfllm_b200.so:graph_node_priority=1 paper_2402_04617_b200/libinfllm_b200.so:lookup_units_per_block=16 paper_2402_04617_b200/libinfllm_b200.so:lookup_units_per_block=24 > gpurun_out/t9_ab.log 2>&1; echo ab_rc=$?
python tools/timeline.py 131072 graph_node_priority=1 > gpurun_out/t9_tl.log 2>&1; echo tl_rc=$?
