// infllm_b200.hpp — header-only C++ facade over the C-ABI (infllm_b200.h)
// with the shape of the reference's operator API, for C++ hosts that used
// blockmem::StreamEngine<Scalar> (engine.hpp:63-395) and blockmem::TieredStore
// (memory.hpp:170-323). Paths are relative to
// /root/reference/proj/include/blockmem/.
//
// Differences from the reference, by design:
//  - q/k/v are passed explicitly as DEVICE tensors (token-major, GQA) instead
//    of being produced by the synthetic token adapter from token ids;
//  - steps are asynchronous on a cudaStream_t; accessors that read device
//    state (retrieved ids, metrics, store) synchronise;
//  - one engine object serves all layers; a reference "step" is one call per
//    layer, in layer order.
// Errors: ConfigError / StreamError with the reference's messages
// (types.hpp:20-26); CudaError / ExchangeError for the device side.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <array>
#include <vector>

#include "infllm_b200.h"

namespace infllm {

struct ConfigError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct StreamError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ExchangeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == INFLLM_OK) return;
    const char* m = infllm_last_error();
    const std::string msg = m ? m : "";
    switch (rc) {
        case INFLLM_ERR_CONFIG: throw ConfigError(msg);
        case INFLLM_ERR_STREAM: throw StreamError(msg);
        case INFLLM_ERR_CUDA: throw CudaError(msg);
        case INFLLM_ERR_NCCL: throw ExchangeError(msg);
        default: throw std::invalid_argument(msg);
    }
}

using EngineConfig = infllm_engine_config;  // types.hpp:84-110, same field names
using ModelShape = infllm_model_shape;      // types.hpp:29-49 + n_kv_heads
using EngineLayerMetrics = infllm_layer_metrics;  // engine.hpp:35-41 + CacheCounters

/// EngineConfig{} (types.hpp:85-94 defaults).
inline EngineConfig default_config() {
    EngineConfig c{};
    check(infllm_config_default(&c));
    return c;
}

/// EngineConfig::validate + ModelShape::validate (types.hpp:96-109, 45-48).
inline void validate(const EngineConfig& c, const ModelShape* s = nullptr) { check(infllm_config_validate(&c, s)); }

enum class Dtype : int32_t { f32 = INFLLM_DTYPE_F32, bf16 = INFLLM_DTYPE_BF16 };

struct UnitInfo {  // MemoryUnit (memory.hpp:19-41): span + representative positions
    int64_t start_abs = 0, size = 0;
    std::vector<int64_t> repr_abs;
};

struct TraceRecord {  // TieredStore trace entry (memory.hpp:159-163)
    int64_t step, unit_id;
    bool hit;
};

struct StreamState {  // engine.hpp:77-78, 140-148
    int64_t tokens_fed, steps_done, initial_len, local_len, pending_partial;
};

class StreamEngine {
public:
    StreamEngine(const EngineConfig& config, const ModelShape& shape, Dtype dtype = Dtype::bf16, int device = 0,
                 int kv_group_begin = 0, int kv_group_count = 0)
        : config_(config), shape_(shape) {
        check(infllm_engine_create(&config_, &shape_, static_cast<int32_t>(dtype), device, kv_group_begin,
                                   kv_group_count, &h_));
    }
    ~StreamEngine() {
        if (h_) infllm_engine_destroy(h_);
    }
    StreamEngine(const StreamEngine&) = delete;
    StreamEngine& operator=(const StreamEngine&) = delete;
    StreamEngine(StreamEngine&& o) noexcept : config_(o.config_), shape_(o.shape_), h_(std::exchange(o.h_, nullptr)) {}

    const EngineConfig& config() const { return config_; }
    const ModelShape& shape() const { return shape_; }
    infllm_engine_t handle() const { return h_; }

    /// encode_chunk (engine.hpp:92-97) for one layer: l_x <= chunk_size tokens.
    void encode_chunk(int layer, const void* q, const void* k, const void* v, int64_t l_x, void* out,
                      void* stream = nullptr) {
        check(infllm_encode_chunk(h_, layer, q, k, v, l_x, out, stream));
    }
    /// decode_step (engine.hpp:100-103) for one layer.
    void decode_step(int layer, const void* q, const void* k, const void* v, void* out, void* stream = nullptr) {
        check(infllm_decode_step(h_, layer, q, k, v, out, stream));
    }
    /// feed (engine.hpp:106-112) for one layer, graph-replayed chunk schedule.
    void feed(int layer, const void* q, const void* k, const void* v, int64_t n_tokens, void* out,
              void* stream = nullptr) {
        check(infllm_encode_stream(h_, layer, q, k, v, n_tokens, out, stream));
    }
    /// feed from host buffers (pinned): per-chunk copies overlapped with compute.
    void feed_host(int layer, const void* q, const void* k, const void* v, int64_t n_tokens, void* out,
                   void* stream = nullptr) {
        check(infllm_encode_stream_host(h_, layer, q, k, v, n_tokens, out, stream));
    }
    /// finish (engine.hpp:115-119): flush held-back partial units.
    void finish(void* stream = nullptr) { check(infllm_finish(h_, stream)); }
    void reset(void* stream = nullptr) { check(infllm_engine_reset(h_, stream)); }
    void reserve(int64_t max_tokens) { check(infllm_engine_reserve(h_, max_tokens)); }
    void set_option(const std::string& key, int64_t value) { check(infllm_engine_set_option(h_, key.c_str(), value)); }
    void set_allgather(infllm_allgather_fn fn, void* user) { check(infllm_engine_set_allgather(h_, fn, user)); }

    /// LayerStepOutput::retrieved_ids of the layer's latest step (engine.hpp:26-30).
    std::vector<int64_t> retrieved_ids(int layer) const {
        std::vector<int64_t> ids(static_cast<size_t>(config_.n_lookup > 0 ? config_.n_lookup : 1));
        int64_t n = 0;
        check(infllm_retrieved_ids(h_, layer, ids.data(), static_cast<int64_t>(ids.size()), &n));
        ids.resize(static_cast<size_t>(n));
        return ids;
    }
    /// metrics().layers[layer] (engine.hpp:121-138).
    EngineLayerMetrics metrics(int layer) const {
        EngineLayerMetrics m{};
        check(infllm_get_layer_metrics(h_, layer, &m));
        return m;
    }
    StreamState stream_state(int layer) const {
        StreamState s{};
        check(infllm_stream_state(h_, layer, &s.tokens_fed, &s.steps_done, &s.initial_len, &s.local_len,
                                  &s.pending_partial));
        return s;
    }
    int64_t tokens_fed(int layer = 0) const { return stream_state(layer).tokens_fed; }
    int64_t steps_done(int layer = 0) const { return stream_state(layer).steps_done; }

    /// store(layer).unit(id) (memory.hpp:178-180).
    UnitInfo unit(int layer, int64_t unit_id) const {
        UnitInfo u;
        u.repr_abs.resize(static_cast<size_t>(config_.n_repr));
        int64_t n = 0;
        check(infllm_unit_info(h_, layer, unit_id, &u.start_abs, &u.size, u.repr_abs.data(), &n));
        u.repr_abs.resize(static_cast<size_t>(n));
        return u;
    }
    /// store(layer).trace() (memory.hpp:182).
    std::vector<TraceRecord> trace(int layer) const {
        int64_t n = 0;
        check(infllm_trace(h_, layer, nullptr, nullptr, nullptr, 0, &n));
        std::vector<int64_t> st(static_cast<size_t>(n)), un(static_cast<size_t>(n));
        std::vector<int32_t> hit(static_cast<size_t>(n));
        if (n > 0) check(infllm_trace(h_, layer, st.data(), un.data(), hit.data(), n, &n));
        std::vector<TraceRecord> out;
        out.reserve(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) out.push_back({st[i], un[i], hit[i] != 0});
        return out;
    }

    /// Engine options (infllm_engine_set_option): "host_tier_slots", "decode_kernel", ...
    void set_option(const char* key, int64_t value) { check(infllm_engine_set_option(h_, key, value)); }
    /// Host tier counters: page loads, cache hits, H2D bytes, slots (infllm_tier_stats).
    std::array<int64_t, 4> tier_stats(int layer = 0) const {
        std::array<int64_t, 4> s{};
        check(infllm_tier_stats(h_, layer, s.data()));
        return s;
    }

private:
    EngineConfig config_;
    ModelShape shape_;
    infllm_engine_t h_ = nullptr;
};

/// One decode step of engines.size() independent sequences (infllm_decode_batch):
/// q [B][H][d], k/v [B][H_kv][d], out [B][H][d_v] device pointers.
inline void decode_batch(const std::vector<StreamEngine*>& engines, int layer, const void* q, const void* k,
                         const void* v, void* out, void* stream = nullptr) {
    std::vector<infllm_engine_t> hs;
    hs.reserve(engines.size());
    for (auto* e : engines) hs.push_back(e->handle());
    check(infllm_decode_batch(hs.data(), static_cast<int32_t>(hs.size()), layer, q, k, v, out, stream));
}

}  // namespace infllm
