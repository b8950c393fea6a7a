// Throughput of the fp64 pipe instructions the relevance scan issues per
// element: F2F.F64.F32 (bf16 -> fp64 widening) and DFMA, and of an
// integer-only bf16 -> fp64 widening, per SM (one block of 256..1024 threads per SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/f64_rate tools/f64_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_f2f(const unsigned* in, double* out, int iters) {
    unsigned x = in[threadIdx.x] | 0x3f800000u;
    double acc = 0.0;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            acc += static_cast<double>(__uint_as_float((x + j) << 16));
        }
        x += 17;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_f2f_only(const unsigned* in, double* out, int iters) {
    unsigned x = in[threadIdx.x] | 0x3f800000u;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
            a0 = static_cast<double>(__uint_as_float((x + j) << 16));
            a1 = static_cast<double>(__uint_as_float((x + j + 1) << 16));
            a2 = static_cast<double>(__uint_as_float((x + j + 2) << 16));
            a3 = static_cast<double>(__uint_as_float((x + j + 3) << 16));
            x ^= __double2hiint(a0) ^ __double2hiint(a1) ^ __double2hiint(a2) ^ __double2hiint(a3);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + x;
}
__global__ void k_dfma(const unsigned* in, double* out, int iters) {
    double q = 1.0000001 + threadIdx.x * 1e-9;
    double a[8] = {0, 1, 2, 3, 4, 5, 6, 7};
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j & 7] = fma(q, a[j & 7], 0.5);
    }
    double s = 0;
    for (int j = 0; j < 8; ++j) s += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ double widen_int(unsigned f) {
    const unsigned hi = (f & 0x80000000u) | (((f >> 3) & 0x0fffe000u) + 0x38000000u);
    return __hiloint2double(static_cast<int>(hi), 0);
}
__global__ void k_int(const unsigned* in, double* out, int iters) {
    unsigned x = in[threadIdx.x] | 0x3f800000u;
    double acc = 0.0;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += widen_int((x + j) << 16);
        x += 17;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    unsigned* in;
    double* out;
    cudaMalloc(&in, 4096 * 4);
    cudaMemset(in, 0, 4096 * 4);
    cudaMalloc(&out, 148 * 1024 * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    for (int threads : {256, 512, 1024}) {
        auto run = [&](const char* name, void (*k)(const unsigned*, double*, int), double per_iter) {
            k<<<148, threads>>>(in, out, 16);
            cudaEventRecord(a);
            k<<<148, threads>>>(in, out, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            int clk;
            cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
            const double ops = 148.0 * threads * iters * per_iter;
            printf("%-10s threads %4d: %.3f ms, %.1f Gop/s, %.2f lanes/clk/SM at the max clock\n", name, threads, ms,
                   ops / ms / 1e6, ops / (ms * 1e-3) / 148 / (clk * 1e3));
        };
        run("f2f+dadd", k_f2f, 16);
        run("f2f", k_f2f_only, 16);
        run("dfma", k_dfma, 16);
        run("int+dadd", k_int, 16);
    }
    return 0;
}
