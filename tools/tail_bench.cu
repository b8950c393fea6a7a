// Single-block latency primitives on this part (the one-block top-k tails of
// the lookup): cycles per block barrier, per dependent 64-bit compare-exchange
// stage over shuffles (bitonic network step), per contended shared atomic
// round, per dependent L2 load, and the SM clock while one block runs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tail_bench tools/tail_bench.cu && tools/tail_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_prims(const uint64_t* chase, long long* out, int n) {
    __shared__ int hist[256];
    __shared__ uint64_t sk[256];
    const int t = threadIdx.x, lane = t & 31;
    long long c0, c1;
    unsigned long long g0, g1;
    // barriers
    __syncthreads();
    c0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    c1 = clock64();
    if (t == 0) out[0] = (c1 - c0) / n;
    // dependent compare-exchange stages (64-bit key + 32-bit id), one warp
    uint64_t k = (uint64_t)(t * 2654435761u) << 20 | t;
    int id = t;
    __syncthreads();
    c0 = clock64();
    if (t < 32) {
        for (int i = 0; i < n; ++i) {
            const int j = 1 << (i % 5);
            const uint64_t pk = __shfl_xor_sync(0xffffffffu, k, j);
            const int pi = __shfl_xor_sync(0xffffffffu, id, j);
            const bool first = k > pk || (k == pk && id < pi);
            if (first != ((lane & j) == 0)) {
                k = pk;
                id = pi;
            }
        }
    }
    c1 = clock64();
    if (t == 0) out[1] = (c1 - c0) / n;
    sk[t] = k + id;
    // contended shared atomics: every thread into one of 2 bins, then a barrier
    if (t < 256) hist[t] = 0;
    __syncthreads();
    c0 = clock64();
    for (int i = 0; i < n; ++i) {
        atomicAdd(&hist[(t + i) & 1], 1);
        __syncthreads();
    }
    c1 = clock64();
    if (t == 0) out[2] = (c1 - c0) / n;
    // dependent global loads (L2-resident chain), thread 0
    __syncthreads();
    if (t == 0) {
        uint64_t p = 0;
        c0 = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
        for (int i = 0; i < n; ++i) p = __ldcg(chase + p);
        c1 = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
        out[3] = (c1 - c0) / n;
        out[4] = (long long)p;
        out[5] = (long long)(g1 - g0);  // ns for the n loads: with out[3] * n gives the clock
        out[6] = c1 - c0;
    }
    if (t == 0) out[7] = sk[5];
}

int main() {
    const int n = 512, m = 1 << 20;
    uint64_t* h = new uint64_t[m];
    for (int i = 0; i < m; ++i) h[i] = (uint64_t)((i * 7919ull + 104729ull) % m);
    uint64_t* d;
    long long* o;
    cudaMalloc(&d, m * 8);
    cudaMalloc(&o, 8 * 8);
    cudaMemcpy(d, h, m * 8, cudaMemcpyHostToDevice);
    for (int r = 0; r < 3; ++r) k_prims<<<1, 256>>>(d, o, n);
    cudaDeviceSynchronize();
    long long v[8];
    cudaMemcpy(v, o, sizeof(v), cudaMemcpyDeviceToHost);
    printf("cycles: barrier (256 thr) %lld, cmp-exchange stage (1 warp, 64-bit key) %lld, "
           "contended smem atomic + barrier %lld, dependent L2 load %lld; SM clock while one block runs %.0f MHz\n",
           v[0], v[1], v[2], v[3], v[5] > 0 ? 1e3 * (double)v[6] / (double)v[5] : 0.0);
    return 0;
}
