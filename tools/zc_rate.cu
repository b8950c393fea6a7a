// zc_rate.cu — host-tier transfer microbenchmark: device-initiated reads of
// mapped pinned host memory (the k_tier_copy pattern) vs cudaMemcpyAsync H2D
// (copy engine), for unit-page-sized pieces (512 KB = one C2 unit, K + V^T).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/zc_rate tools/zc_rate.cu && tools/zc_rate
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <int U>
__global__ void zc_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n16, int64_t per_block) {
    const int64_t base = static_cast<int64_t>(blockIdx.x) * per_block;
    for (int64_t o = 0; o < per_block; o += blockDim.x * U) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = base + o + threadIdx.x + static_cast<int64_t>(blockDim.x) * u;
            if (i < n16 && o + threadIdx.x + blockDim.x * u < per_block) r[u] = __ldg(src + i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = base + o + threadIdx.x + static_cast<int64_t>(blockDim.x) * u;
            if (i < n16 && o + threadIdx.x + blockDim.x * u < per_block) dst[i] = r[u];
        }
    }
}

int main() {
    const size_t bytes = 64ull << 20;  // 128 unit pages of 512 KB
    void *h, *d;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    cudaMalloc(&d, bytes);
    for (size_t i = 0; i < bytes / 8; ++i) static_cast<uint64_t*>(h)[i] = i;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    const int64_t n16 = bytes / 16;
    for (int blocks : {20, 40, 80, 160, 320, 640, 1280}) {
        for (int unroll : {4, 8, 16}) {
            const int64_t per_block = (n16 + blocks - 1) / blocks;
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                if (unroll == 4) zc_copy<4><<<blocks, 256>>>((const uint4*)h, (uint4*)d, n16, per_block);
                if (unroll == 8) zc_copy<8><<<blocks, 256>>>((const uint4*)h, (uint4*)d, n16, per_block);
                if (unroll == 16) zc_copy<16><<<blocks, 256>>>((const uint4*)h, (uint4*)d, n16, per_block);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
            }
            cudaEventElapsedTime(&ms, a, b);
            printf("zero-copy kernel: %5d blocks x 256 thr, %2d x 16B in flight/thr: %6.1f GB/s\n", blocks, unroll,
                   bytes / ms / 1e6);
        }
    }
    for (size_t piece : {size_t(32) << 10, size_t(256) << 10, size_t(512) << 10, size_t(8) << 20, bytes}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            for (size_t o = 0; o < bytes; o += piece)
                cudaMemcpyAsync(static_cast<char*>(d) + o, static_cast<char*>(h) + o, piece, cudaMemcpyHostToDevice);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        cudaEventElapsedTime(&ms, a, b);
        printf("cudaMemcpyAsync H2D in %8zu-byte pieces: %6.1f GB/s\n", piece, bytes / ms / 1e6);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
