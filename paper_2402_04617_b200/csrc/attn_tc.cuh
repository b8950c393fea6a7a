// attn_tc.cuh — tcgen05/TMEM/TMA attention kernel interface (bf16, d = 128).
#pragma once

#include "kernels.cuh"

namespace infllm {

// true when the tensor-core kernel covers this shape/mode
bool attn_tc_supported(int d, int dv, int unit_size, bool absolute);
// true when the tc kernel reduces the per-unit masses itself (AttnParams::mass_cta)
bool attn_tc_masses_in_kernel(int n_sel);
// launches the tensor-core attention for one step; returns #kernels launched
int launch_attn_tc(const AttnParams& p, cudaStream_t st);
// building-block self-test (one 128x128x128 tile), see attn_tc.cu
void debug_read_attn_timestamps(unsigned long long* out64);
void tc_selftest(const void* q, const void* k, const void* vt, float* s_out, float* o_out, cudaStream_t st);

}  // namespace infllm
