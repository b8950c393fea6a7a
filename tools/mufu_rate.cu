// Microbenchmark: MUFU.EX2 and FMA-pipe throughput per SM (cycles via clock64).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mufu_rate.cu -o tools/mufu_rate.bin
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int KIND>
__global__ void k(int iters, float* out, unsigned long long* cyc) {
    float v[8];
    for (int i = 0; i < 8; ++i) v[i] = -0.001f * (threadIdx.x + i);
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (KIND == 0)
                v[i] = ex2(v[i]);
            else if (KIND == 1)
                v[i] = fmaf(v[i], 0.999f, -0.0001f);
            else if (KIND == 3) {  // ex2 + one bf16x2 pack per two elements (the softmax mix)
                v[i] = ex2(v[i]);
                if (i & 1) {
                    uint32_t pk;
                    asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(pk) : "f"(v[i]), "f"(v[i - 1]));
                    v[i - 1] = __uint_as_float(pk << 16) - 1.0f;
                }
            } else if (KIND == 4) {  // ex2.approx.f16x2: two exponentials per instruction (elements counted)
                if (i & 1) {
                    uint32_t x = __float_as_uint(v[i]), y;
                    asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
                    v[i] = __uint_as_float(y);
                }
            } else if (KIND == 5) {  // ex2.approx.ftz.bf16x2
                if (i & 1) {
                    uint32_t x = __float_as_uint(v[i]), y;
                    asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
                    v[i] = __uint_as_float(y);
                }
            } else {  // bf16x2 pack (cvt.rn.bf16x2.f32) feeding back into the chain
                uint32_t pk;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(pk) : "f"(v[i]), "f"(v[(i + 1) & 7]));
                v[i] = __uint_as_float(pk & 0xffff0000u) + 1e-30f;
            }
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    float* o;
    unsigned long long* c;
    cudaMalloc(&o, 1 << 24);
    cudaMalloc(&c, 8);
    for (int threads : {128, 256, 512, 1024}) {
        for (int kind : {0, 3, 4, 5}) {
            const int iters = 4096;
            if (kind == 0)
                k<0><<<148, threads>>>(iters, o, c);
            else if (kind == 1)
                k<1><<<148, threads>>>(iters, o, c);
            else if (kind == 2)
                k<2><<<148, threads>>>(iters, o, c);
            else if (kind == 3)
                k<3><<<148, threads>>>(iters, o, c);
            else if (kind == 4)
                k<4><<<148, threads>>>(iters, o, c);
            else
                k<5><<<148, threads>>>(iters, o, c);
            cudaDeviceSynchronize();
            unsigned long long cy;
            cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
            printf("%s threads=%d: %.2f ops/clk/SM\n", kind == 0 ? "ex2" : kind == 1 ? "ffma" : kind == 2 ? "cvt.bf16x2(+fadd,and)" : kind == 3 ? "ex2 + pack per pair (elements)" : kind == 4 ? "ex2.f16x2 (elements)" : "ex2.bf16x2 (elements)", threads,
                   (double)threads * iters * 8 / cy);
        }
    }
    return 0;
}
