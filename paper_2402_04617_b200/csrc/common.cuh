// common.cuh — shared device helpers for the InfLLM B200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace infllm {

using bf16 = __nv_bfloat16;

template <typename T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<bf16>(bf16 x) { return __bfloat162float(x); }

template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

// Rotary factors (rotary.hpp:19-34): angle = pos * freq in double (freq table
// computed on the host with std::pow exactly like the reference), cos/sin in
// double, narrowed to float.
struct RopeFreqs {
    double f[128];   // up to head_dim 256
    float cL[128];   // float(cos(l_L * f)), float(sin(l_L * f)): the constant
    float sL[128];   // rotation of rotate_by_constant (rotary.hpp:66-72)
};

// rotate one pair exactly like rotate_row (rotary.hpp:40-51): no FMA
// contraction, so the float result matches the reference's separate
// multiply/subtract rounding.
__device__ __forceinline__ void rope_pair(float x0, float x1, float c, float s, float& y0, float& y1) {
    y0 = __fsub_rn(__fmul_rn(x0, c), __fmul_rn(x1, s));
    y1 = __fadd_rn(__fmul_rn(x0, s), __fmul_rn(x1, c));
}

__device__ __forceinline__ void rope_cs(const RopeFreqs& fr, int a, int64_t pos, float& c, float& s) {
    const double ang = static_cast<double>(pos) * fr.f[a];
    double sd, cd;
    sincos(ang, &sd, &cd);
    c = static_cast<float>(cd);
    s = static_cast<float>(sd);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Device timeline (infllm_timeline_*): thread 0 of every block of the step
// kernels appends (kernel, SM, globaltimer start, end) to a device ring when a
// buffer is bound, so the overlap of the five step streams can be read back
// without a profiler. Unbound (the default) it costs one timer read and one
// predicated branch per block.
enum TlKernel : unsigned {
    TL_ATTN = 0, TL_ROPE, TL_PREP, TL_PREFIX, TL_LOOKUP, TL_TOPK, TL_EVICT, TL_SELECT, TL_LRU, TL_TIER,
    TL_DEC, TL_DEC_FRONT, TL_MASS, TL_KINDS
};
struct TlRec {
    unsigned long long t0, t1;
    unsigned kid, sm;
};
struct TlBuf {
    TlRec* rec;
    unsigned long long* cnt;
    unsigned long long cap;
};
static __constant__ TlBuf g_tl;  // one per translation unit, bound by tl_bind_tu (constant bank: the
                                 // enabled check in every TL_MARK is a broadcast, not a global load)
static inline cudaError_t tl_bind_tu(const TlBuf& b) { return cudaMemcpyToSymbol(g_tl, &b, sizeof(b)); }
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void tl_put(unsigned kid, unsigned long long t0) {
    const unsigned long long i = atomicAdd(g_tl.cnt, 1ull);
    if (i >= g_tl.cap) return;
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_tl.rec[i] = TlRec{t0, gtimer(), kid, sm};
}
#define TL_BEGIN() const unsigned long long tl_t0_ = threadIdx.x == 0 ? ::infllm::gtimer() : 0ull
#define TL_END(kid)                                                              \
    do {                                                                         \
        if (threadIdx.x == 0 && ::infllm::g_tl.rec) ::infllm::tl_put((kid), tl_t0_); \
    } while (0)

// phase marks inside a kernel (timeline kinds 100 + k): thread 0 of each block
// records [mark, now] and restarts `mark` (a variable holding the last mark)
#define TL_MARK(k, mark)                                    \
    do {                                                    \
        if (threadIdx.x == 0 && ::infllm::g_tl.rec) {       \
            ::infllm::tl_put(100 + (k), (mark));            \
            (mark) = ::infllm::gtimer();                    \
        }                                                   \
    } while (0)

// Device LRU/bookkeeping state of one layer's TieredStore (memory.hpp:170-323).
struct LruState {
    int64_t hot_count;
    uint64_t hits, misses, loads, evictions, requested;
    int64_t peak_hot_units;
    int64_t peak_hot_bytes;
    int64_t trace_count;
};

}  // namespace infllm
