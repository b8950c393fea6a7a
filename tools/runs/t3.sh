python tools/opt_ab.py "attn_streams=1,graph_node_priority=0" "attn_streams=2,graph_node_priority=0" "attn_streams=1,graph_node_priority=1" "attn_streams=2,graph_node_priority=1" "attn_streams=1,graph_node_priority=0" "attn_streams=2,graph_node_priority=1" > gpurun_out/t3_ab.log 2>&1; echo ab_rc=$?
python tools/timeline.py > gpurun_out/t3_tl.log 2>&1; echo tl_rc=$?
python tools/lookup_sweep.py 131072 4,8,16,48 > gpurun_out/t3_lk.log 2>&1; echo lk_rc=$?
