// Probe: can a green-context stream (a subset of SMs) take part in a CUDA graph
// captured from a primary-context stream, with runtime-API launches, and do its
// kernels stay on the partition's SMs?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/green_probe.cu -o tools/green_probe -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <set>

#define CK(x)                                                                              \
    do {                                                                                   \
        auto r = (x);                                                                      \
        if (r != 0) {                                                                      \
            printf("FAIL %s -> %d (line %d)\n", #x, (int)r, __LINE__);                     \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

__global__ void k_smid(int* out) {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    const long long t0 = clock64();
    while (clock64() - t0 < 20000) {
    }
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

int main() {
    CK(cudaSetDevice(0));
    CK(cudaFree(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUdevResource all;
    CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("device SMs: %u\n", all.sm.smCount);
    CUdevResource part[2], rem;
    unsigned n = 1;
    CK(cuDevSmResourceSplitByCount(part, &n, &all, &rem, 0, 16));
    printf("groups %u, group SMs %u, remaining %u\n", n, part[0].sm.smCount, rem.sm.smCount);
    CUdevResourceDesc desc;
    CK(cuDevResourceGenerateDesc(&desc, part, 1));
    CUgreenCtx g;
    CK(cuGreenCtxCreate(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream gs;
    CK(cuGreenCtxStreamCreate(&gs, g, CU_STREAM_NON_BLOCKING, 0));
    cudaStream_t main_s;
    CK(cudaStreamCreateWithFlags(&main_s, cudaStreamNonBlocking));
    int* d;
    CK(cudaMalloc(&d, 4096 * sizeof(int)));
    // direct launch on the green stream
    k_smid<<<256, 64, 0, (cudaStream_t)gs>>>(d);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    int h[4096];
    CK(cudaMemcpy(h, d, 256 * sizeof(int), cudaMemcpyDeviceToHost));
    std::set<int> sms(h, h + 256);
    printf("direct: kernel on green stream used %zu distinct SMs\n", sms.size());
    // captured: main -> green -> main
    cudaEvent_t e1, e2;
    CK(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(main_s, cudaStreamCaptureModeThreadLocal));
    CK(cudaEventRecord(e1, main_s));
    CK(cudaStreamWaitEvent((cudaStream_t)gs, e1, 0));
    k_smid<<<256, 64, 0, (cudaStream_t)gs>>>(d + 512);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e2, (cudaStream_t)gs));
    CK(cudaStreamWaitEvent(main_s, e2, 0));
    k_smid<<<256, 64, 0, main_s>>>(d + 1024);
    CK(cudaStreamEndCapture(main_s, &graph));
    cudaGraphExec_t ex;
    CK(cudaGraphInstantiate(&ex, graph, 0));
    CK(cudaGraphLaunch(ex, main_s));
    CK(cudaStreamSynchronize(main_s));
    CK(cudaMemcpy(h, d + 512, 256 * sizeof(int), cudaMemcpyDeviceToHost));
    std::set<int> s2(h, h + 256);
    CK(cudaMemcpy(h, d + 1024, 256 * sizeof(int), cudaMemcpyDeviceToHost));
    std::set<int> s3(h, h + 256);
    printf("captured: green-stream kernel used %zu SMs, main-stream kernel used %zu SMs\n", s2.size(), s3.size());
    return 0;
}
