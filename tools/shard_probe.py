# Per-GPU step time of one KV-group shard of the C2 stream (kv_group_count = 8 / G),
# split-KV attention auto vs off. No exchange hook is set (the cross-shard partial
# sums are missing, so ids differ): this isolates the compute each GPU does at G.
import sys, torch
sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
for G in (1, 2, 4, 8):
    gs = 8 // G
    g = torch.Generator(device='cuda'); g.manual_seed(0)
    Q = torch.randn((n, 4 * gs, 128), generator=g, device='cuda').bfloat16()
    K = torch.randn((n, gs, 128), generator=g, device='cuda').bfloat16()
    V = torch.randn((n, gs, 128), generator=g, device='cuda').bfloat16()
    for splits in (1, 0):
        eng = StreamEngine(EngineConfig.make(**bench.CFG), ModelShape.make(**bench.SHAPE), dtype=torch.bfloat16,
                           kv_group_begin=0, kv_group_count=gs)
        eng.reserve(n)
        eng.set_option("attn_splits", splits)
        O = torch.empty_like(Q)
        ts = []
        for it in range(4):
            eng.reset(); torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); eng.encode_stream(Q, K, V, out=O); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        eng.profile_begin(True); eng.reset(); eng.encode_stream(Q, K, V, out=O)
        pr = eng.profile_read(); eng.profile_begin(False)
        print(f"G={G} groups/shard={gs} splits={'auto' if splits == 0 else splits}: {1000 * min(ts[1:]) / 256:.1f} us/step "
              f"(attention {1000 * pr['attn_ms'] / 256:.1f} us/step)", flush=True)
        eng.close()
