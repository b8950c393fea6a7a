// C++ host over include/infllm_b200.hpp, the way a user of the reference's
// blockmem::StreamEngine would drive it. Built and run by tests/test_cpp_facade.py.
//   facade_demo cpu   : host-only checks (defaults, validation errors); no GPU calls
//   facade_demo gpu   : a small fp32 stream (C0-like, 4 heads / 2 KV heads, d 64),
//                       prints the retrieved unit ids of every step and the metrics
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

#include "infllm_b200.hpp"

// deterministic inputs, restated in the Python test: value(i) in [-0.5, 0.5)
static float val(uint64_t i, uint64_t salt) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull ^ (salt * 0xD1B54A32D192ED03ull);
    x ^= x >> 31;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    return static_cast<float>(x >> 40) / 16777216.0f - 0.5f;
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    infllm::EngineConfig cfg = infllm::default_config();
    std::printf("defaults %lld %lld %lld %lld %lld %lld %lld %.2f\n", (long long)cfg.chunk_size,
                (long long)cfg.unit_size, (long long)cfg.n_repr, (long long)cfg.local_size, (long long)cfg.init_size,
                (long long)cfg.n_lookup, (long long)cfg.hot_capacity, cfg.decay);
    try {
        infllm::EngineConfig bad = cfg;
        bad.hot_capacity = 4;
        bad.n_lookup = 8;
        infllm::validate(bad);
        std::printf("no error\n");
    } catch (const infllm::ConfigError& e) {
        std::printf("ConfigError: %s\n", e.what());
    }
    if (!gpu) return 0;

    cfg.chunk_size = 128;
    cfg.unit_size = 128;
    cfg.n_repr = 4;
    cfg.local_size = 512;
    cfg.init_size = 64;
    cfg.n_lookup = 4;
    cfg.hot_capacity = 32;
    infllm::ModelShape shape{1, 4, 2, 64, 64};
    const int64_t n = 2048, H = 4, G = 2, d = 64;
    std::vector<float> q(n * H * d), k(n * G * d), v(n * G * d);
    for (size_t i = 0; i < q.size(); ++i) q[i] = val(i, 1);
    for (size_t i = 0; i < k.size(); ++i) k[i] = val(i, 2);
    for (size_t i = 0; i < v.size(); ++i) v[i] = val(i, 3) * 2.0f;
    float *dq, *dk, *dv, *dout;
    cudaMalloc(&dq, q.size() * 4);
    cudaMalloc(&dk, k.size() * 4);
    cudaMalloc(&dv, v.size() * 4);
    cudaMalloc(&dout, n * H * d * 4);
    cudaMemcpy(dq, q.data(), q.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dk, k.data(), k.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, v.data(), v.size() * 4, cudaMemcpyHostToDevice);
    infllm::StreamEngine eng(cfg, shape, infllm::Dtype::f32);
    for (int64_t off = 0; off < n; off += cfg.chunk_size) {
        eng.encode_chunk(0, dq + off * H * d, dk + off * G * d, dv + off * G * d, cfg.chunk_size, dout + off * H * d);
        std::printf("ids");
        for (int64_t id : eng.retrieved_ids(0)) std::printf(" %lld", (long long)id);
        std::printf("\n");
    }
    try {
        eng.encode_chunk(0, dq, dk, dv, cfg.chunk_size + 1, dout);
    } catch (const infllm::StreamError& e) {
        std::printf("StreamError: %s\n", e.what());
    }
    eng.finish();
    const auto m = eng.metrics(0);
    std::printf("metrics units %lld hits %llu misses %llu evictions %llu requested %llu\n", (long long)m.units,
                (unsigned long long)m.hits, (unsigned long long)m.misses, (unsigned long long)m.evictions,
                (unsigned long long)m.requested);
    std::vector<float> out(n * H * d);
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    double cs = 0;
    for (float x : out) cs += x;
    std::printf("checksum %.9g\n", cs);
    return 0;
}
