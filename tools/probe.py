import sys, ctypes as C, torch
sys.path.insert(0, '.')
from paper_2402_04617_b200 import EngineConfig, ModelShape, StreamEngine, _lib
eng = StreamEngine(EngineConfig.make(chunk_size=128, local_size=512, n_lookup=4), ModelShape.make(n_heads=8, n_kv_heads=2, head_dim=128), dtype=torch.bfloat16)
for w, name in [(9, "f64"), (10, "f32")]:
    us = C.c_double()
    _lib.check(_lib.lib().infllm_debug_kernel_bench(eng.h, w, 3, C.byref(us)))
    ops = 148 * 4 * 256 * 8 * 1000
    print(name, f"{us.value:.1f} us", f"{2 * ops / us.value / 1e6:.2f} TFLOP/s", f"{ops / (us.value * 1e-6 * 1.965e9 * 148):.1f} FMA/clk/SM")
