// Microbenchmark: raw tcgen05.mma issue rate per SM (kind::f16, cta_group::1),
// SS (A and B from shared memory) and TS (A from TMEM) at M=128, K=16 and
// N in {128, 256}; operands are uninitialised (timing only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_2402_04617_b200/csrc tools/mma_rate.cu -o /tmp/mma_rate
#include <cstdio>

#include "tc_prims.cuh"

using namespace infllm::tc;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) k_rate(int iters, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 98304);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = *slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_bf16(128, N);
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                if (TS)
                    mma_ts(tb + 256, tb + 8 * kk, sdesc_sw128(b + off), idesc, 1u);
                else
                    mma_ss(tb + (it & 1) * 128, sdesc_sw128(a + off), sdesc_sw128(b + off), idesc, 1u);
            }
        }
        mma_commit(bar);
        mbar_wait(bar, 0);
        const unsigned long long t1 = clock64();
        if (blockIdx.x == 0) *cyc = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

// the attention kernel's MMA pattern per KV tile: S[j%3] = Q K^T (SS), then
// O += P V with P = S[(j-2)%3] in TMEM (TS); mode 1: PV's A from a column range no QK writes;
// mode 2: as 0 plus a tcgen05.commit after each group (to an mbarrier nobody waits on)
template <int MODE>
__global__ void __launch_bounds__(352, 1) k_attn_pattern(int iters, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 98304);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 4);
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        mbar_init(bar + 2, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = *slot;
    if (MODE >= 4) {  // random bf16 operands in [-1, 1) instead of zeros
        uint32_t* w = reinterpret_cast<uint32_t*>(smem);
        for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) {
            uint32_t x = i * 2654435761u + 12345u;
            x ^= x >> 13;
            x *= 0x5bd1e995u;
            x ^= x >> 15;
            const uint32_t lo = 0x3f80u | (x & 0x807fu), hi = 0x3f80u | ((x >> 16) & 0x807fu);
            w[i] = (lo & 0xffffu) | (hi << 16);
        }
        __syncthreads();
    }
    if (MODE >= 3 && warp >= 2 && blockDim.x > 128) {
        // spectators spinning on an mbarrier that completes only at the end
        mbar_wait(bar + 2, 0);
    }
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_bf16(128, 128);
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768), v = smem_u32(smem + 65536);
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                mma_ss(tb + 128 * (it % 3), sdesc_sw128(a + off), sdesc_sw128(b + off), idesc, kk > 0);
            }
            if (MODE == 2) mma_commit(bar + 1);
            const uint32_t pcol = MODE == 1 ? tb + 448 : tb + 128 * ((it + 1) % 3);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                mma_ts(tb + 384, pcol + 8 * (kk & (MODE == 1 ? 7 : 7)) * (MODE == 1 ? 0 : 1), sdesc_sw128(v + (kk >> 2) * 16384 + (kk & 3) * 32), idesc, 1u);
            if (MODE == 2) mma_commit(bar + 1);
        }
        mma_commit(bar);
        mbar_wait(bar, 0);
        const unsigned long long t1 = clock64();
        if (blockIdx.x == 0) *cyc = t1 - t0;
        if (MODE >= 3) mbar_arrive(bar + 2);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

// the kernel's dependency structure without softmax warps: QK_{j+2} two ahead,
// PV_j issued after waiting on the commit of QK_j (mbarrier ring of 3)
__global__ void __launch_bounds__(352, 1) k_dep_pattern(int iters, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 98304);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 8);
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 5; ++i) mbar_init(bar + i, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = *slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_bf16(128, 128);
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768), v = smem_u32(smem + 65536);
        auto qk = [&](int j) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                mma_ss(tb + 128 * (j % 3), sdesc_sw128(a + off), sdesc_sw128(b + off), idesc, kk > 0);
            }
            mma_commit(bar + j % 3);
        };
        const unsigned long long t0 = clock64();
        qk(0);
        qk(1);
        for (int j = 0; j < iters; ++j) {
            mbar_wait(bar + j % 3, (j / 3) & 1);
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                mma_ts(tb + 384, tb + 128 * (j % 3) + 8 * kk, sdesc_sw128(v + (kk >> 2) * 16384 + (kk & 3) * 32),
                       idesc, 1u);
            mma_commit(bar + 3);
            if (j + 2 < iters) qk(j + 2);
        }
        mma_commit(bar + 4);
        mbar_wait(bar + 4, 0);
        const unsigned long long t1 = clock64();
        if (blockIdx.x == 0) *cyc = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

void run_dep(int grid, int iters, int threads = 128, int smem = 98304 + 1024 + 128) {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(k_dep_pattern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_dep_pattern<<<grid, threads, smem>>>(iters, d);
    cudaDeviceSynchronize();
    unsigned long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("dependency pattern grid=%d threads=%d smem=%d: %.1f cyc per KV tile  [%s]\n", grid, threads, smem,
           (double)c / iters,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

template <int MODE>
void run_pattern(int grid, int iters) {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    const int smem = 98304 + 1024 + 64;
    cudaFuncSetAttribute(k_attn_pattern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_attn_pattern<MODE><<<grid, MODE >= 3 ? 352 : 128, smem>>>(iters, d);
    cudaDeviceSynchronize();
    unsigned long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("attention pattern mode %d grid=%d: %.1f cyc per KV tile (QK + PV = 16 MMAs)  [%s]\n", MODE, grid,
           (double)c / iters, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

template <int N, bool TS>
void run(int grid, int iters) {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    const int smem = 98304 + 1024 + 64;
    cudaFuncSetAttribute(k_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_rate<N, TS><<<grid, 128, smem>>>(iters, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_rate<N, TS><<<grid, 128, smem>>>(iters, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double flops = 2.0 * 128 * N * 128 * iters * (double)grid;
    printf("N=%d %s grid=%d: %.1f cyc per 128x%dx128 (8 MMAs), %.0f TFLOP/s  [%s]\n", N, TS ? "TS" : "SS", grid,
           (double)c / iters, N, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    run_dep(1, 2000);
    run_dep(128, 2000);
    run_dep(128, 2000, 352);
    run_dep(128, 2000, 352, 226000);
    for (int grid : {1, 128}) {
        run_pattern<0>(grid, 2000);
        run_pattern<1>(grid, 2000);
        run_pattern<2>(grid, 2000);
        run_pattern<3>(grid, 2000);
        run_pattern<4>(grid, 2000);
    }
    for (int grid : {1, 148}) {
        run<128, false>(grid, 2000);
        run<128, true>(grid, 2000);
        run<256, false>(grid, 2000);
    }
    return 0;
}
