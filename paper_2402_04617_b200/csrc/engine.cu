// engine.cu — host side of the B200 InfLLM layer: the C-ABI declared in
// include/infllm_b200.h and the per-step orchestration that mirrors
// blockmem::StreamEngine::step (engine.hpp:242-359). All data-dependent state
// (lookup ids, representative indices, LRU tiers/frequencies/counters, trace)
// lives on the device; the host only advances the stream arithmetic that the
// reference derives from token counts (local window bounds, initial-token
// pinning, unit packing boundaries), so a step is a fixed kernel sequence on
// the caller's stream with no host synchronisation.

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <type_traits>
#include <stdexcept>
#include <string>
#include <cstdlib>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>  // types and enums only: the library is resolved at run time (dlopen)
#include <nvtx3/nvToolsExt.h>

#include "../../include/infllm_b200.h"
#include "attn_dec.cuh"
#include "attn_tc.cuh"
#include "kernels.cuh"

using namespace infllm;

namespace {

thread_local std::string g_err;

// NVTX ranges named after the reference's PhaseTimings (engine.hpp:43-49):
// host-side brackets of each phase's launches (nsys / Nsight show them)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
// device-time phases (PhaseTimings order minus the adapter)
constexpr int kPhLookup = 0, kPhAttend = 1, kPhScore = 2, kPhEvict = 3, kPhases = 4;

struct ConfigError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct StreamError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ExchangeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
int guard(F&& f) {
    try {
        f();
        return INFLLM_OK;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return INFLLM_ERR_CONFIG;
    } catch (const StreamError& e) {
        g_err = e.what();
        return INFLLM_ERR_STREAM;
    } catch (const CudaError& e) {
        g_err = e.what();
        return INFLLM_ERR_CUDA;
    } catch (const ExchangeError& e) {
        g_err = e.what();
        return INFLLM_ERR_NCCL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return INFLLM_ERR_ARG;
    }
}

void validate_cfg(const infllm_engine_config& c) {  // types.hpp:96-109
    if (c.chunk_size < 1) throw ConfigError("chunk_size must be >= 1");
    if (c.unit_size < 1) throw ConfigError("unit_size must be >= 1");
    if (c.n_repr < 1) throw ConfigError("n_repr must be >= 1");
    if (c.local_size < 1) throw ConfigError("local_size must be >= 1");
    if (c.init_size < 0) throw ConfigError("init_size must be >= 0");
    if (c.n_lookup < 0) throw ConfigError("n_lookup must be >= 0");
    if (c.n_repr > c.unit_size) throw ConfigError("n_repr must not exceed unit_size");
    if (c.hot_capacity < c.n_lookup) throw ConfigError("hot_capacity must be >= n_lookup");
    if (c.decay < 0.0 || c.decay > 1.0) throw ConfigError("decay must lie in [0, 1]");
    if (c.lookup_mode < 0 || c.lookup_mode > 2) throw ConfigError("lookup_mode: unknown value");
    if (c.position_mode < 0 || c.position_mode > 1) throw ConfigError("position_mode: unknown value");
}

void validate_shape(const infllm_model_shape& s) {  // types.hpp:45-48
    if (s.n_layers < 1 || s.n_heads < 1 || s.head_dim < 1)
        throw ConfigError("ModelShape: all fields must be >= 1");
    const int hkv = s.n_kv_heads > 0 ? s.n_kv_heads : s.n_heads;
    if (s.n_heads % hkv != 0) throw ConfigError("ModelShape: n_heads must be a multiple of n_kv_heads");
}

// device allocation (stream-ordered so pools can grow mid-stream)
struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void alloc(size_t b, cudaStream_t st, bool zero = true) {
        release(st);
        if (b == 0) return;
        ck(cudaMallocAsync(&p, b, st), "cudaMallocAsync");
        bytes = b;
        if (zero) ck(cudaMemsetAsync(p, 0, b, st), "cudaMemsetAsync");
    }
    void grow(size_t b, cudaStream_t st) {  // keep contents
        if (b <= bytes) return;
        void* n = nullptr;
        ck(cudaMallocAsync(&n, b, st), "cudaMallocAsync");
        ck(cudaMemsetAsync(n, 0, b, st), "cudaMemsetAsync");
        if (p) {
            ck(cudaMemcpyAsync(n, p, bytes, cudaMemcpyDeviceToDevice, st), "cudaMemcpyAsync");
            ck(cudaFreeAsync(p, st), "cudaFreeAsync");
        }
        p = n;
        bytes = b;
    }
    void release(cudaStream_t st) {
        if (p) cudaFreeAsync(p, st);
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

// mapped pinned host allocation (host tier unit pages); device-addressable via UVA
struct HBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void grow(size_t b) {  // keep contents; the caller has drained every stream touching it
        if (b <= bytes) return;
        void* n = nullptr;
        ck(cudaHostAlloc(&n, b, cudaHostAllocMapped | cudaHostAllocPortable), "cudaHostAlloc (host tier)");
        if (p) std::memcpy(n, p, bytes);
        std::memset(static_cast<uint8_t*>(n) + bytes, 0, b - bytes);
        if (p) cudaFreeHost(p);
        p = n;
        bytes = b;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
    }
    void* dev() const {
        void* d = nullptr;
        if (p) ck(cudaHostGetDevicePointer(&d, p, 0), "cudaHostGetDevicePointer");
        return d;
    }
};

__global__ void k_empty() {}
// throughput probes: 8 independent FMA chains x n iterations per thread
__global__ void k_probe_f64(double* out, int n) {
    double a[8];
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
    const double m = 1.0000001, c = 1e-9;
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fma(a[j], m, c);
    double s = 0;
    for (int j = 0; j < 8; ++j) s += a[j];
    if (s == 12345.0) out[0] = s;
}
__global__ void k_probe_f32(float* out, int n) {
    float a[8];
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
    const float m = 1.0000001f, c = 1e-9f;
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], m, c);
    float s = 0;
    for (int j = 0; j < 8; ++j) s += a[j];
    if (s == 12345.0f) out[0] = s;
}

// NCCL, resolved at run time: the library loads (and runs single-GPU) without it;
// a process that already loaded one (torch) shares that copy (RTLD_NOLOAD first)
struct Nccl {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};
const Nccl& nccl() {
    static Nccl n = [] {
        Nccl x;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return x;
        x.get_unique_id = reinterpret_cast<decltype(x.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        x.comm_init_rank = reinterpret_cast<decltype(x.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        x.all_gather = reinterpret_cast<decltype(x.all_gather)>(dlsym(h, "ncclAllGather"));
        x.comm_destroy = reinterpret_cast<decltype(x.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        x.error_string = reinterpret_cast<decltype(x.error_string)>(dlsym(h, "ncclGetErrorString"));
        return x;
    }();
    if (!n.get_unique_id || !n.comm_init_rank || !n.all_gather) throw ExchangeError("NCCL (libnccl.so.2) not available");
    return n;
}
void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw ExchangeError(std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "NCCL error"));
}

// exchange layout: the fp64 partials of the engine are [rows][g_total] with this
// shard's columns [g0, g0 + G); NCCL all-gathers contiguous [rows][G] blocks per
// rank, rank r owning groups [r G, (r + 1) G)
__global__ void k_pack_cols(const double* buf, int64_t rows, int gt, int g0, int g, double* send) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < rows * g) send[t] = buf[(t / g) * gt + g0 + t % g];
}
__global__ void k_unpack_cols(const double* recv, int64_t rows, int gt, int g, double* buf) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // over [rank][row][col]
    if (t >= rows * gt) return;
    const int64_t r = t / (rows * g), rem = t % (rows * g);
    buf[(rem / g) * gt + r * g + rem % g] = recv[t];
}
// output all-gather: [rank][lx][Hs][dv] -> [lx][H][dv]
__global__ void k_interleave_heads(const uint8_t* recv, int64_t lx, int hs, int nr, int64_t row_bytes, uint8_t* out) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // 16-byte pieces
    const int64_t per = row_bytes / 16, n = static_cast<int64_t>(nr) * lx * hs * per;
    if (t >= n) return;
    const int64_t piece = t % per, hh = (t / per) % hs, i = (t / (per * hs)) % lx, r = t / (per * hs * lx);
    reinterpret_cast<uint4*>(out)[((i * nr + r) * hs + hh) * per + piece] = reinterpret_cast<const uint4*>(recv)[t];
}

__global__ void k_fill_i32(int32_t* x, int64_t n, int32_t v) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) x[i] = v;
}

}  // namespace

// parameters of one batched decode step, gathered from each engine's step()
struct DecFrontRec {  // layout of the batched decode-front table (kernels.cu DecFront)
    PrepParams p;
    EvictParams ep;
};
struct DecodeCollector {
    std::vector<DecFrontRec> front;
    std::vector<PrepParams> prep;
    std::vector<EvictParams> evict;
    std::vector<SelectParams> select;
    std::vector<LookupParams> lookup;
    std::vector<AttnParams> attn;
    std::vector<LruParams> lru;
};

// an event shared by the engines of a batch (the last batched LRU they joined)
struct SharedEvent {
    cudaEvent_t ev = nullptr;
    ~SharedEvent() {
        if (ev) cudaEventDestroy(ev);
    }
};
// device/host resources of batched decode calls (owned by the batch's first engine)
struct BatchCtx {
    // parameter-table slots: a call reuses the slot of the call kSlots back once that
    // call's LRU (the last reader, on its own stream) is done
    static constexpr int kSlots = 4;
    void* host[kSlots] = {};  // pinned parameter staging
    void* dev[kSlots] = {};   // device parameter tables
    size_t cap = 0;
    cudaEvent_t done[kSlots] = {};
    int slot = 0;
    DBuf part, mass, cnt;  // K4 batch scratch
    int part_B = 0, mass_B = 0;
    // the LRU stage runs on its own stream, overlapping the next calls' work; a
    // call's lookup rewrites the selection buffer (and its K4 the mass buffer)
    // the LRU of the call three back read (each engine rotates kSB = 3 buffers,
    // one step per call), so it waits for that LRU only
    cudaStream_t lru_st = nullptr;
    cudaEvent_t ev_k4 = nullptr;
    std::shared_ptr<SharedEvent> lru_ev;
    bool lru_pending = false;
    static constexpr int kRing = 3;
    cudaEvent_t lru_ring[kRing] = {nullptr, nullptr, nullptr};
    bool ring_set[kRing] = {false, false, false};
    int64_t calls = 0;
};

struct infllm_engine {
    infllm_engine_config cfg{};
    DecodeCollector* coll = nullptr;  // decode_batch: record kernel parameters instead of launching
    std::unique_ptr<BatchCtx> bctx;
    std::shared_ptr<SharedEvent> ext_dep;  // a batched LRU on another stream that touched this engine
    void join_ext(cudaStream_t st) {       // order `st` after it (engine calls outside a batch)
        if (!ext_dep) return;
        ck(cudaStreamWaitEvent(st, ext_dep->ev, 0), "wait");
        ext_dep.reset();
    }
    void sync_ext() {  // before pool growth (buffers the LRU may still read or write)
        if (ext_dep) ck(cudaEventSynchronize(ext_dep->ev), "sync");
    }
    int H = 1, Gt = 1, rep = 1, d = 0, dv = 0, n_layers = 1;
    int g0 = 0, Gs = 1, Hs = 1;  // shard
    int dtype = INFLLM_DTYPE_F32;
    int device = 0;
    size_t esz = 4;
    int64_t R = 0;  // ring capacity
    int64_t lxp = 0;
    RopeFreqs freqs{};
    infllm_allgather_fn allgather = nullptr;
    void* allgather_user = nullptr;
    int64_t launches = 0;
    bool use_tc = false;
    bool tc_disabled = false;
    bool score_bound = true;  // tcgen05 attention: fixed-offset softmax when the bound allows
    bool use_dec = false;     // K4 split-KV decode attention for l_x = 1 steps
    bool dec_disabled = false;
    int attn_splits = 0;      // option attn_splits: split-KV K3 (0: auto, when the grid leaves SMs idle)
    int lookup_upb = 48;      // option lookup_units_per_block: K1+K2 grid inside the prefill pipeline
    int lookup_upb_decode = 8;  // option lookup_units_per_block_decode: the same for one-token steps (whole GPU)
    // option attn_streams: chunk-step attention alternates between this many
    // dedicated high-priority streams (1: the caller's stream). Attention t+1
    // reads nothing attention t writes (own prep, selection and mass buffers),
    // so with two streams its CTAs take the SMs attention t frees as they free
    // up instead of queueing behind t's last CTA while side kernels fill them.
    int attn_streams = 2;
    bool graph_prio = false;
    bool dec_chain_opt = true;  // option decode_chain
    bool dec_lk_fused = true;  // option decode_lookup_fused: one-token steps past 2048 units take k_lookup_topk
                               // (512K one sequence 40.8 -> 39.7 us per step)
    bool dec_merge_opt = true;  // option decode_merge_kernel: K4's split merge as its own parallel launch  // option graph_node_priority (measured slower: 73.8 vs 70.6 us per C2 step)
    cudaStream_t attn_st[2] = {nullptr, nullptr};
    cudaEvent_t out_free = nullptr;  // host path: the staging buffer `out` points into is drained
    VLayout vl{};
    // two-stream step pipeline: the side stream runs prep/lookup/top-k and
    // evict/finalize/select, the caller's (main) stream attention + LRU; step
    // k's front half overlaps step k-1's attention. Scratch written by the
    // side stream and read by the main stream is double-buffered by k % 2.
    // The prep of step k runs on its own stream, concurrently with step k-1's
    // eviction/selection on the side stream (it only waits for step k-1's lookup,
    // the last reader of the chunk query sums it rewrites).
    cudaStream_t side_stream = nullptr, lru_stream = nullptr, prep_stream = nullptr, evict_stream = nullptr;
    // selection / mass buffers rotate over kSB steps: the lookup of step k reuses
    // the buffers of step k - kSB, read by its attention and LRU
    static constexpr int kSB = 3;
    cudaEvent_t e_call = nullptr, e_topk = nullptr, e_side = nullptr, e_lru[kSB] = {nullptr, nullptr, nullptr};
    cudaEvent_t e_attn = nullptr, e_lrudone = nullptr, e_prep = nullptr, e_lookup = nullptr, e_prepdone = nullptr;
    // The prep runs up to kPB - 1 chunks ahead of the attention: prep outputs
    // (qa, qc, chunk sums, key-norm bound) rotate over kPB buffers, the prep of
    // step k waits for the attention of step k - kPB, and the ring holds
    // l_L + kPB chunks + 1 slots, so the chunk being prepared never overwrites
    // a key an attention that may still run reads.
    static constexpr int kPB = 3;
    cudaEvent_t e_evict = nullptr, e_evdone = nullptr, e_attnp[kPB] = {nullptr, nullptr, nullptr};
    int64_t attn_seq[kPB] = {-1, -1, -1};  // step that last recorded e_attnp[pb]
    int64_t attn_last = -1;                 // step that last recorded e_attn
    // host tier: slot assignment + PCIe page pulls of step t on their own stream
    // (after lookup t, before attention t), so lookup t+1 does not queue behind them
    cudaStream_t tier_stream = nullptr;
    cudaEvent_t e_tier = nullptr, e_tierdone = nullptr;
    int64_t tier_seq = -1;  // step that last queued work on the tier stream
    int64_t lookup_seq = -1;         // step that last recorded e_lookup
    int64_t evict_seq = -1;          // step that last recorded e_evict
    int64_t seq = 0;                 // engine-wide step counter
    int64_t lru_seq[kSB] = {-1, -1, -1};  // step that last recorded e_lru[b]
    int64_t capture_seq0 = -1;       // first step of the graph being captured (-1: not capturing)
    size_t qa_half = 0;              // bytes of one qa/qc buffer
    int64_t mass_cta_half = 0;       // doubles in one mass_cta buffer
    // last launch parameters per kernel (debug kernel timing only)
    PrepParams last_pp{};
    LookupParams last_lkp{};
    AttnParams last_ap{};
    EvictParams last_ep{};
    LruParams last_lp{};
    bool last_bf16 = false;

    // scratch shared by layers (layers run sequentially on one stream)
    DBuf split_o, split_ml;  // split-KV K3 partials
    DBuf qa, qc, chunk_qsum, mass_e, mass_m, row_m, row_l, mass_cta, rtab, qsb, tsum, topk_done, evict_done;
    DBuf dec_part, dec_mass, dec_cnt;  // K4 decode scratch (one sequence)

    struct Layer {
        int64_t n_fed = 0, step = 0, local_start = 0, init_len = 0;
        int64_t n_units = 0, pend_start = 0, pend_count = 0;
        int64_t trace_count = 0, last_n_sel = 0, last_b = 0;
        int64_t unit_cap = 0, trace_cap = 0;
        std::vector<int64_t> unit_start;
        std::vector<int32_t> unit_len;
        DBuf ring_k, ring_krot, ring_v, P;
        DBuf init_k, init_krot, init_v;
        DBuf unit_k, unit_krot, unit_v, unit_scores, repr, repr_idx, ulen, freq, hot;
        DBuf hot_list, lru, trace, sel, rel, relw, lookup_part, mass_part, ev_part;
        DBuf kmax2;  // [kPB step buffers][G] running max |k|^2 (attention score bound)
        DBuf cand;   // multi-block top-k candidates (values then ids), large unit counts
        DBuf dec_maps;  // K4 TMA tensor maps (6), re-encoded when a buffer moves
        std::vector<const void*> dec_maps_key;
        // host tier (tier_slots > 0): unit pages in mapped pinned host memory,
        // the attention reads them from tier_slots device cache slots
        HBuf host_k, host_krot, host_v;
        void *dhost_k = nullptr, *dhost_krot = nullptr, *dhost_v = nullptr;
        DBuf slot_k, slot_krot, slot_v, slot_unit, slot_used, unit_slot, sel_slot, tier_miss, tier_stats;
    };
    std::vector<Layer> layers;

    // host stream arithmetic of a layer (everything a step derives on the host)
    struct HostState {
        int64_t n_fed, step, local_start, init_len, n_units, pend_start, pend_count, trace_count, last_n_sel, last_b;
        std::vector<int64_t> unit_start;
        std::vector<int32_t> unit_len;
        bool operator==(const HostState& o) const {
            return n_fed == o.n_fed && step == o.step && local_start == o.local_start && init_len == o.init_len &&
                   n_units == o.n_units && pend_start == o.pend_start && pend_count == o.pend_count &&
                   trace_count == o.trace_count && last_n_sel == o.last_n_sel && last_b == o.last_b &&
                   unit_start == o.unit_start &&
                   unit_len == o.unit_len;
        }
    };
    static HostState save(const Layer& L) {
        return HostState{L.n_fed,      L.step,        L.local_start, L.init_len, L.n_units,    L.pend_start,
                         L.pend_count, L.trace_count, L.last_n_sel,  L.last_b,   L.unit_start, L.unit_len};
    }
    static void restore(Layer& L, const HostState& h) {
        L.n_fed = h.n_fed;
        L.step = h.step;
        L.local_start = h.local_start;
        L.init_len = h.init_len;
        L.n_units = h.n_units;
        L.pend_start = h.pend_start;
        L.pend_count = h.pend_count;
        L.trace_count = h.trace_count;
        L.last_n_sel = h.last_n_sel;
        L.last_b = h.last_b;
        L.unit_start = h.unit_start;
        L.unit_len = h.unit_len;
    }

    // CUDA graphs of whole multi-chunk streams: the launch sequence and every
    // kernel parameter follow from the host arithmetic alone (data-dependent
    // values stay on the device), so a stream from a given host state replays
    // as one graph launch.
    struct GraphEntry {
        int layer;
        const void *q, *k, *v;
        void* out;
        int64_t n;
        bool host, prof;
        HostState before, after;
        cudaGraphExec_t exec = nullptr;
        int64_t launches = 0;
        uint64_t inv_checks = 0, inv_bad = 0;  // invariant checks the captured steps make per replay
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[kPhases];  // profile events per phase
        int64_t replays_in_window = 0;
        int64_t steps = 0;
        std::vector<const void*> bufs;  // device addresses baked into the graph (buf_snapshot)
    };
    std::vector<GraphEntry> graphs;
    static constexpr size_t kMaxGraphs = 8;
    static void drop_graph(GraphEntry& g) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        g.exec = nullptr;
        for (auto& evs : g.ev) {
            for (auto& p : evs) {
                cudaEventDestroy(p.first);
                cudaEventDestroy(p.second);
            }
            evs.clear();
        }
    }
    cudaStream_t cap_stream = nullptr, h2d_stream = nullptr, d2h_stream = nullptr;
    bool use_graphs = true;
    int64_t tier_slots = 0;  // host tier: GPU unit-cache slots (0: unit pages resident in HBM)
    bool capturing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* cap_ev = nullptr;  // [kPhases] of the graph being captured
    static constexpr int kNB = 4;  // host-pointer staging buffers (groups of kGroup chunks)
    DBuf stage_q[kNB], stage_k[kNB], stage_v[kNB], stage_o[kNB];

    void record(cudaEvent_t e, cudaStream_t st) {
        if (capturing)
            ck(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal), "event record (capture)");
        else
            ck(cudaEventRecord(e, st), "event record");
    }

    // profiling (dominant kernel + lookup timing with events on the caller stream)
    bool prof = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[kPhases];
    // brackets one phase's launches on `st` with timing events (profile mode)
    // NVTX range named after the reference's phase (host side, for nsys) and,
    // in profile mode, device timing events on the phase's stream
    std::pair<cudaEvent_t, cudaEvent_t> phase_begin(const char* name, cudaStream_t st) {
        nvtxRangePushA(name);
        if (!prof) return {};
        std::pair<cudaEvent_t, cudaEvent_t> p{take_event(), take_event()};
        record(p.first, st);
        return p;
    }
    void phase_end(int ph, std::pair<cudaEvent_t, cudaEvent_t> p, cudaStream_t st) {
        nvtxRangePop();
        if (!prof) return;
        record(p.second, st);
        (capturing ? cap_ev : ev)[ph].push_back(p);
    }
    // invariant counters (engine.hpp:88-89, 361-383)
    uint64_t inv_checks = 0, inv_conservation_bad = 0;
    DBuf inv_dev;  // device count of check_softmax violations
    std::vector<cudaEvent_t> ev_pool;

    cudaEvent_t take_event() {
        if (!ev_pool.empty()) {
            cudaEvent_t e = ev_pool.back();
            ev_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        ck(cudaEventCreate(&e), "cudaEventCreate");
        return e;
    }

    size_t unit_elems_k() const { return static_cast<size_t>(Gs) * cfg.unit_size * d; }
    size_t unit_elems_v() const { return static_cast<size_t>(Gs) * cfg.unit_size * dv; }

    // every device buffer the engine owns (a captured step graph holds their addresses)
    std::vector<DBuf*> dev_buffers() {
        std::vector<DBuf*> v{&ex_send, &ex_recv, &out_stage, &out_recv, &split_o, &split_ml, &inv_dev, &qa, &qc, &chunk_qsum, &mass_e, &mass_m, &row_m, &row_l, &mass_cta, &rtab, &qsb,
                             &tsum, &topk_done, &evict_done, &dec_part, &dec_mass, &dec_cnt};
        for (int b = 0; b < kNB; ++b)
            for (auto* x : {&stage_q[b], &stage_k[b], &stage_v[b], &stage_o[b]}) v.push_back(x);
        for (auto& L : layers)
            for (auto* b : {&L.ring_k, &L.ring_krot, &L.ring_v, &L.P, &L.init_k, &L.init_krot, &L.init_v, &L.unit_k,
                            &L.unit_krot, &L.unit_v, &L.unit_scores, &L.repr, &L.repr_idx, &L.ulen, &L.freq, &L.hot,
                            &L.hot_list, &L.lru, &L.trace, &L.sel, &L.rel, &L.relw, &L.lookup_part, &L.mass_part,
                            &L.ev_part, &L.kmax2, &L.cand, &L.slot_k, &L.slot_krot, &L.slot_v, &L.slot_unit,
                            &L.slot_used, &L.unit_slot, &L.sel_slot, &L.tier_miss, &L.tier_stats, &L.dec_maps})
                v.push_back(b);
        return v;
    }
    std::vector<const void*> buf_snapshot() {
        std::vector<const void*> r;
        for (auto* b : dev_buffers()) r.push_back(b->p);
        for (auto& L : layers)
            for (const void* h : {L.dhost_k, L.dhost_krot, L.dhost_v}) r.push_back(h);
        return r;
    }
    void ensure_units(Layer& L, int64_t need, cudaStream_t st) {
        if (need <= L.unit_cap) return;
        sync_ext();
        if (side_stream) ck(cudaStreamSynchronize(side_stream), "side sync before pool growth");
        if (lru_stream) ck(cudaStreamSynchronize(lru_stream), "lru sync before pool growth");
        if (evict_stream) ck(cudaStreamSynchronize(evict_stream), "evict sync before pool growth");
        const int64_t cap = std::max<int64_t>({need, 2 * L.unit_cap, 16});
        const bool absolute = cfg.position_mode == INFLLM_POSITION_ABSOLUTE;
        if (tier_slots > 0) {
            ck(cudaStreamSynchronize(st), "sync before host-tier growth");
            L.host_k.grow(cap * unit_elems_k() * esz);
            if (absolute) L.host_krot.grow(cap * unit_elems_k() * esz);
            L.host_v.grow(cap * unit_elems_v() * esz);
            L.dhost_k = L.host_k.dev();
            L.dhost_krot = L.host_krot.dev();
            L.dhost_v = L.host_v.dev();
            if (!L.slot_k.p) {
                const int64_t S = tier_slots;
                L.slot_k.alloc(S * unit_elems_k() * esz, st);
                if (absolute) L.slot_krot.alloc(S * unit_elems_k() * esz, st);
                L.slot_v.alloc(S * unit_elems_v() * esz, st);
                L.slot_unit.alloc(S * sizeof(int64_t), st, false);
                ck(cudaMemsetAsync(L.slot_unit.p, 0xff, L.slot_unit.bytes, st), "memset");
                L.slot_used.alloc(S * sizeof(int64_t), st);
                const size_t km = static_cast<size_t>(std::max<int64_t>(cfg.n_lookup, 1));
                L.sel_slot.alloc(kSB * km * sizeof(int32_t), st);
                L.tier_miss.alloc((2 * km + 1) * sizeof(int32_t), st);
                L.tier_stats.alloc(4 * sizeof(int64_t), st);
            }
            L.unit_slot.grow(cap * sizeof(int32_t), st);
            k_fill_i32<<<static_cast<unsigned>((cap - L.unit_cap + 255) / 256), 256, 0, st>>>(
                L.unit_slot.as<int32_t>() + L.unit_cap, cap - L.unit_cap, -1);
            ++launches;
        } else {
            L.unit_k.grow(cap * unit_elems_k() * esz, st);
            if (absolute) L.unit_krot.grow(cap * unit_elems_k() * esz, st);
            L.unit_v.grow(cap * unit_elems_v() * esz, st);
        }
        L.unit_scores.grow(cap * cfg.unit_size * sizeof(float), st);
        L.repr.grow(cap * static_cast<size_t>(Gs) * cfg.n_repr * d * esz, st);
        L.repr_idx.grow(cap * cfg.n_repr * sizeof(int32_t), st);
        const int64_t old = L.unit_cap;
        L.ulen.grow(cap * sizeof(int32_t), st);
        k_fill_i32<<<static_cast<unsigned>((cap - old + 255) / 256), 256, 0, st>>>(L.ulen.as<int32_t>() + old, cap - old,
                                                                                 static_cast<int32_t>(cfg.unit_size));
        ++launches;
        L.freq.grow(cap * sizeof(double), st);
        L.hot.grow(cap * sizeof(int8_t), st);
        L.rel.grow(cap * sizeof(double), st);
        L.relw.grow(cap * sizeof(double), st);
        L.lookup_part.grow(cap * Gt * sizeof(double), st);
        // multi-block top-k candidates (sized here: no allocation may happen inside a captured step)
        L.cand.grow(static_cast<size_t>(topk_multi_scratch(cap, std::max<int64_t>(cfg.n_lookup, 1))) * 16, st);
        L.unit_cap = cap;
        ensure_exchange(std::max<int64_t>({cap, cfg.chunk_size, cfg.n_lookup}));
    }

    void ensure_trace(Layer& L, int64_t need, cudaStream_t st) {
        if (need <= L.trace_cap) return;
        sync_ext();
        if (side_stream) ck(cudaStreamSynchronize(side_stream), "side sync before pool growth");
        if (lru_stream) ck(cudaStreamSynchronize(lru_stream), "lru sync before pool growth");
        if (evict_stream) ck(cudaStreamSynchronize(evict_stream), "evict sync before pool growth");
        const int64_t cap = std::max<int64_t>({need, 4 * L.trace_cap, 1024});  // rare: each growth drains
        L.trace.grow(cap * 3 * sizeof(int64_t), st);
        L.trace_cap = cap;
    }

    DecScratch dec_scratch() const {
        return DecScratch{dec_part.as<float>(), dec_mass.as<float>(), dec_cnt.as<unsigned>(),
                          static_cast<int>(std::max<int64_t>(cfg.n_lookup, 1)), 0};
    }

    // where unit pages are written (HBM pool, or the host tier)
    void* upage_k(const Layer& L) const { return tier_slots > 0 ? L.dhost_k : L.unit_k.p; }
    void* upage_krot(const Layer& L) const { return tier_slots > 0 ? L.dhost_krot : L.unit_krot.p; }
    void* upage_v(const Layer& L) const { return tier_slots > 0 ? L.dhost_v : L.unit_v.p; }

    bool one_stream = false;           // current step runs on the caller's stream only
    bool pipe_dirty = false;           // pipeline streams may hold work the caller's stream does not wait for
    bool multi_stream_decode = false;  // option: keep the five-stream pipeline for decode steps
    void rec(cudaEvent_t e, cudaStream_t s2) {
        if (!one_stream) ck(cudaEventRecord(e, s2), "record");
    }
    void wt(cudaStream_t s2, cudaEvent_t e) {
        if (!one_stream) ck(cudaStreamWaitEvent(s2, e, 0), "wait");
    }

    // make `st` wait for everything queued on the side stream
    void join_side(cudaStream_t st) {
        ck(cudaEventRecord(e_side, side_stream), "record");
        ck(cudaStreamWaitEvent(st, e_side, 0), "wait");
        ck(cudaEventRecord(e_lrudone, lru_stream), "record");
        ck(cudaStreamWaitEvent(st, e_lrudone, 0), "wait");
        ck(cudaEventRecord(e_prepdone, prep_stream), "record");
        ck(cudaStreamWaitEvent(st, e_prepdone, 0), "wait");
        ck(cudaEventRecord(e_evdone, evict_stream), "record");
        ck(cudaStreamWaitEvent(st, e_evdone, 0), "wait");
        if (tier_seq >= 0 && (capture_seq0 < 0 || tier_seq >= capture_seq0)) {  // only a stream that joined
            ck(cudaEventRecord(e_tierdone, tier_stream), "record");
            ck(cudaStreamWaitEvent(st, e_tierdone, 0), "wait");
        }
        tier_seq = -1;
        for (auto& x : lru_seq) x = -1;
        for (auto& a : attn_seq) a = -1;
        attn_last = -1;
        lookup_seq = -1;
        evict_seq = -1;
        pipe_dirty = false;
    }

    // cross-shard exchange C-1: the other shards' columns of a
    // [rows][Gt] fp64 partial buffer, in stream order on `st`
    void gather(double* buf, int64_t rows, cudaStream_t st) {
        if (Gs == Gt || rows <= 0) return;
        if (comm) {
            if (coll) throw StreamError("decode_batch: sharded engines are not batched");
            const unsigned nb = static_cast<unsigned>((rows * Gs + 255) / 256);
            k_pack_cols<<<nb, 256, 0, st>>>(buf, rows, Gt, g0, Gs, ex_send.as<double>());
            nck(nccl().all_gather(ex_send.p, ex_recv.p, static_cast<size_t>(rows) * Gs, ncclDouble,
                                  static_cast<ncclComm_t>(comm), st),
                "ncclAllGather (partials)");
            k_unpack_cols<<<static_cast<unsigned>((rows * Gt + 255) / 256), 256, 0, st>>>(ex_recv.as<double>(), rows,
                                                                                         Gt, Gs, buf);
            launches += 2;
            return;
        }
        if (!allgather) return;
        if (allgather(allgather_user, buf, rows, g0, Gs, Gt, st) != 0)
            throw ExchangeError("allgather hook failed");
    }
    // NCCL communicator over the KV-group shards (infllm_engine_set_comm)
    void* comm = nullptr;
    int comm_rank = 0, comm_size = 1;
    bool gather_output = false;  // option gather_output: C-2 all-gather of the outputs to all heads
    DBuf ex_send, ex_recv, out_stage, out_recv;
    void ensure_exchange(int64_t rows) {
        if (!comm) return;
        const size_t need = static_cast<size_t>(std::max<int64_t>(rows, 1)) * Gt * sizeof(double);
        if (ex_recv.bytes >= need) return;
        ex_send.alloc(need / comm_size + 256, nullptr, false);
        ex_recv.alloc(need, nullptr, false);
    }

    // Units are whole 128-token ring pages (they start at l_I + 128 u and every
    // token of a unit is still in the ring when it completes): copied per unit
    // with 16-byte vectors instead of per evicted token.
    bool page_mode() const {
        return cfg.unit_size == 128 && cfg.init_size % 128 == 0 && cfg.chunk_size >= 64 && (d * esz) % 16 == 0 &&
               (dv * esz) % 16 == 0;
    }
    void set_page(SelectParams& sp, const Layer& L, int64_t pos0) const {
        sp.page_mode = page_mode() ? 1 : 0;
        sp.absolute = cfg.position_mode == INFLLM_POSITION_ABSOLUTE;
        sp.dv = dv;
        sp.pos0 = pos0;
        sp.R = R;
        sp.ring_k = L.ring_k.p;
        sp.ring_krot = L.ring_krot.p;
        sp.ring_v = L.ring_v.p;
        sp.unit_krot = upage_krot(L);
        sp.unit_v = upage_v(L);
        sp.vl = vl;
    }

    // split-KV for the tcgen05 attention: a KV-group shard (or a short chunk)
    // leaves most SMs idle with one CTA per (128 rows, head); splitting each
    // CTA's tile list over grid.z fills them (>= 4 tiles per split)
    int pick_splits_tc(int64_t lx, const AttnParams& ap) {
        const int64_t ctas = ((lx + 127) / 128) * static_cast<int64_t>(Hs);
        const int64_t tiles = (ap.init_len + 127) / 128 + ap.n_sel + (ap.s + lx - ap.local_start + 127) / 128 + 2;
        int64_t S = attn_splits > 0 ? attn_splits : 148 / std::max<int64_t>(ctas, 1);
        // two splits do not pay for the merge and the fp32 partials (G = 2 shards of C2:
        // 86.0 us per step with, 68.7 without; tools/shard_probe.py)
        if (attn_splits <= 0 && S < 3) S = 1;
        S = std::clamp<int64_t>(std::min<int64_t>(S, tiles / 4), 1, kMaxSplitsTc);
        if (S > 1) ensure_split_scratch(S);
        return static_cast<int>(S);
    }
    void ensure_split_scratch(int64_t S) {
        const size_t need_o = static_cast<size_t>(S) * Hs * lxp * 128 * sizeof(float);
        const size_t need_ml = static_cast<size_t>(S) * Hs * lxp * 2 * sizeof(float);
        if (split_o.bytes >= need_o && split_ml.bytes >= need_ml) return;
        if (capturing) throw StreamError("split-KV scratch must be sized before capture");
        ck(cudaDeviceSynchronize(), "split scratch");
        split_o.alloc(need_o, nullptr, false);
        split_ml.alloc(need_ml, nullptr, false);
    }
    // the most splits any step of this engine can take (a 1-tile-row chunk)
    int64_t max_splits_tc() const {
        const int64_t s = attn_splits > 0 ? attn_splits : 148 / std::max(Hs, 1);
        return std::clamp<int64_t>(s, 1, kMaxSplitsTc);
    }
    static constexpr int kMaxSplitsTc = 16;

    bool tc_eligible(int64_t lx) const {
        (void)lx;
        return use_tc && !tc_disabled;
    }

    // fork: the side stream starts from the caller's current point on `st`
    // (inputs written there); inputs_ready: additionally wait for this event
    // (host-buffer path). Within one encode_stream only the first step forks.
    template <typename T>
    void step(int li, const void* q, const void* k, const void* v, int64_t lx, bool decode, void* out,
              cudaStream_t st, bool fork = true, cudaEvent_t inputs_ready = nullptr) {
        if (li < 0 || li >= n_layers) throw StreamError("layer out of range");
        if (lx < 1) throw StreamError("step: empty batch");
        if (!decode && lx > cfg.chunk_size) throw StreamError("encode_chunk: batch exceeds chunk_size");
        if (!coll) join_ext(st);
        Layer& L = layers[static_cast<size_t>(li)];
        const bool lookup_enabled = decode ? cfg.lookup_mode != INFLLM_LOOKUP_NONE
                                           : cfg.lookup_mode == INFLLM_LOOKUP_ENCODE_AND_DECODE;
        const int64_t s = L.n_fed;
        const bool do_lookup = lookup_enabled && cfg.n_lookup > 0 && L.n_units > 0;  // engine.hpp:254-255
        const int64_t n_sel = do_lookup ? std::min<int64_t>(cfg.n_lookup, L.n_units) : 0;
        const int64_t local_len = s - L.local_start;
        const int64_t overflow = std::max<int64_t>(0, local_len + lx - cfg.local_size);  // engine.hpp:306
        const int64_t to_init = std::clamp<int64_t>(cfg.init_size - L.local_start, 0, overflow);  // 311-312
        const int64_t to_evict = overflow - to_init;
        const int64_t new_pending = L.pend_count + to_evict;
        const int64_t completed = new_pending / cfg.unit_size;
        ensure_units(L, L.n_units + completed + 1, st);
        ensure_trace(L, L.trace_count + n_sel, st);

        // stream fork: side waits for the caller's point (inputs) and for the
        // main-stream step k-2 that last read this parity's buffers
        const int64_t kseq = seq++;
        const int b = static_cast<int>(kseq % kSB);   // selection / mass buffers
        const int pb = static_cast<int>(kseq % kPB);  // prep-output buffers
        // decode steps (one token) run on the caller's stream alone: the
        // multi-stream pipeline only pays for chunk-sized steps, and skipping
        // its ~25 event calls halves the host cost of a decode step
        one_stream = lx == 1 && !capturing && !multi_stream_decode;
        bool dual = false;
        if constexpr (std::is_same_v<T, bf16>)
            dual = attn_streams > 1 && !one_stream && !coll && lx > 1 && Gs == Gt && tc_eligible(lx);
        const cudaStream_t caller = st;
        cudaStream_t main = dual ? attn_st[kseq & 1] : st, side = one_stream ? st : side_stream,
                     pst = one_stream ? st : prep_stream,
                     est = one_stream ? st : evict_stream;
        // decode steps keep the LRU bookkeeping on its own stream (off the critical
        // path: no later prep / lookup / attention reads it), with real events
        const bool lru_side = one_stream && !coll;
        cudaStream_t lru_st = (one_stream && !lru_side) ? st : lru_stream, tier_st = one_stream ? st : tier_stream;
        if (one_stream && pipe_dirty) join_side(st);  // earlier pipelined steps become upstream of `st`
        pipe_dirty = !one_stream;
        if (fork) {
            rec(e_call, caller);
            wt(side, e_call);
            wt(pst, e_call);
        }
        if (inputs_ready) wt(pst, inputs_ready);
        if (lru_seq[b] >= 0 && (capture_seq0 < 0 || lru_seq[b] >= capture_seq0)) {
            if (lru_side)
                ck(cudaStreamWaitEvent(side, e_lru[b], 0), "wait");  // side == caller's stream
            else
                wt(side, e_lru[b]);  // selection buffer b: attention + LRU k-kSB
        }
        // prep-output buffer pb (and the ring slots of this chunk) were last read by attention k-kPB
        if (attn_seq[pb] >= 0 && (capture_seq0 < 0 || attn_seq[pb] >= capture_seq0))
            wt(pst, e_attnp[pb]);
        void* qa_b = static_cast<uint8_t*>(qa.p) + pb * qa_half;
        void* qc_b = static_cast<uint8_t*>(qc.p) + pb * qa_half;
        int64_t* sel_b = L.sel.as<int64_t>() + b * std::max<int64_t>(cfg.n_lookup, 1);
        st = pst;

        // K7: ring append, RoPE, prefix sums
        PrepParams pp{};
        pp.q = q;
        pp.k = k;
        pp.v = v;
        pp.qa = qa_b;
        pp.qc = qc_b;
        pp.ring_k = L.ring_k.p;
        pp.ring_krot = L.ring_krot.p;
        pp.ring_v = L.ring_v.p;
        pp.P = L.P.as<double>();
        pp.chunk_qsum = chunk_qsum.as<double>() + pb * Gs * d;
        pp.s = s;
        pp.lx = lx;
        pp.lxp = lxp;
        pp.R = R;
        pp.L = cfg.local_size;
        pp.H = Hs;
        pp.G = Gs;
        pp.rep = rep;
        pp.d = d;
        pp.dv = dv;
        pp.freqs = freqs;
        pp.vl = vl;
        pp.rtab = rtab.as<float2>();
        pp.qs = qsb.as<double>();
        pp.tsum = tsum.as<double>();
        // the token-tiled prep maintains the key-norm bound the tcgen05 attention uses
        const bool kbound = d == 128 && dv == 128 && rep <= 8;
        const int lb = static_cast<int>(L.step % kPB);  // this layer's step, modulo the prep buffers
        pp.kmax2 = kbound ? L.kmax2.as<float>() + lb * Gs : nullptr;
        pp.kmax2_prev = kbound ? L.kmax2.as<float>() + ((lb + kPB - 1) % kPB) * Gs : nullptr;
        last_pp = pp;
        last_bf16 = std::is_same_v<T, bf16>;
        // one-token steps on one stream: prep and eviction fused into one launch
        // (issued at the eviction site below)
        bool fused_front = false;
        if constexpr (std::is_same_v<T, bf16>)
            fused_front = lx == 1 && (one_stream || coll) && dec_front_supported(pp) && page_mode() && Gs == Gt;
        // decode chain (one-token steps, lookup <= 2048 units): the lookup needs only
        // this token's q (it forms the group sums itself), so it is launched first and
        // the fused front follows as its programmatic dependent, overlapping it; the
        // front and the unit-page copy of a completed unit are issued after the lookup
        const bool dec_chain = fused_front && one_stream && !coll && !prof && tier_slots == 0 && dec_chain_opt &&
                               do_lookup && n_sel > 0 && Gs == Gt;
        EvictParams chain_ep{};
        SelectParams chain_sp{};
        bool chain_sel = false;
        auto issue_front = [&](const EvictParams& ep2, cudaStream_t s2) {
            if (coll)
                coll->front.push_back(DecFrontRec{pp, ep2});
            else if (dec_chain)
                chain_ep = ep2;
            else
                launch_dec_front(pp, ep2, s2);
        };
        const auto evs = fused_front ? std::pair<cudaEvent_t, cudaEvent_t>{} : phase_begin("score", st);
        if (fused_front) {
        } else if (coll) {
            coll->prep.push_back(pp);
        } else {
            launch_prep<T>(pp, st);
        }
        if (!fused_front)
            launches += (d == 128 && dv == 128 && rep <= 8) ? 3 : 2;
        if (!fused_front) phase_end(kPhScore, evs, st);
        rec(e_prep, pst);
        wt(side, e_prep);
        st = side;

        // window roll: init pinning, eviction, representative scoring, packing.
        // Its kernels only touch the evicted tokens and the units created in
        // this step, which this step's lookup and attention never read (units
        // of step t are visible from step t+1, engine.hpp:257-346), so they run
        // on the eviction stream concurrently with the lookup and attention.
        const int64_t n_units0 = L.n_units, init_len0 = L.init_len, local_start0 = L.local_start;
        // this step's lookup (side stream) sees the units completed by the previous step
        if (evict_seq >= 0 && (capture_seq0 < 0 || evict_seq >= capture_seq0))
            wt(side, e_evict);
        st = est;
        wt(est, e_prep);
        const auto eve = (overflow > 0 || fused_front) ? phase_begin("evict", st) : std::pair<cudaEvent_t, cudaEvent_t>{};
        if (overflow > 0) {
            // UnitPacker::add: an empty packer starts its pending run at the
            // first evicted token (memory.hpp:65-66)
            if (L.pend_count == 0 && to_evict > 0) L.pend_start = L.local_start + to_init;
            EvictParams ep{};
            ep.ring_k = L.ring_k.p;
            ep.ring_krot = L.ring_krot.p;
            ep.ring_v = L.ring_v.p;
            ep.P = L.P.as<double>();
            ep.init_k = L.init_k.p;
            ep.init_krot = L.init_krot.p;
            ep.init_v = L.init_v.p;
            ep.unit_k = upage_k(L);
            ep.unit_krot = upage_krot(L);
            ep.unit_v = upage_v(L);
            ep.ev_part = L.ev_part.as<double>();
            ep.pop0 = L.local_start;
            ep.n_init = to_init;
            ep.n_evict = to_evict;
            ep.R = R;
            ep.L = cfg.local_size;
            ep.l_I = cfg.init_size;
            ep.pend_start = L.pend_start;
            ep.unit0 = L.n_units;
            ep.G = Gs;
            ep.Gtot = Gt;
            ep.g0 = g0;
            ep.d = d;
            ep.dv = dv;
            ep.l_bs = static_cast<int>(cfg.unit_size);
            ep.absolute = cfg.position_mode == INFLLM_POSITION_ABSOLUTE;
            ep.vl = vl;
            // single shard (and 16-byte rows): scores + selection fused into the eviction launch
            ep.fused = (Gs == Gt && Gs <= 32) ? 1 : 0;  // single shard: scores finalized in the eviction kernel
            ep.unit_scores = L.unit_scores.as<float>();
            ep.repr = L.repr.p;
            ep.repr_idx = L.repr_idx.as<int32_t>();
            ep.unit_len = L.ulen.as<int32_t>();
            ep.sel_u0 = L.n_units;
            ep.sel_n = completed;
            ep.r_k = static_cast<int>(cfg.n_repr);
            ep.done = evict_done.as<unsigned int>();
            ep.page_mode = page_mode() ? 1 : 0;
            last_ep = ep;
            if (fused_front) {
                issue_front(ep, st);
            } else if (coll) {
                if (!ep.fused) throw StreamError("decode_batch: sharded eviction is not batched");
                if (ep.n_init + ep.n_evict > 0) coll->evict.push_back(ep);
            } else {
                launch_evict<T>(ep, st);
            }
            ++launches;
            if (!ep.fused && to_evict > 0) {
                gather(L.ev_part.as<double>(), to_evict, st);
                FinalizeParams fp{};
                fp.ev_part = L.ev_part.as<double>();
                fp.unit_scores = L.unit_scores.as<float>();
                fp.e0 = L.local_start + to_init;
                fp.n_evict = to_evict;
                fp.pend_start = L.pend_start;
                fp.unit0 = L.n_units;
                fp.L = cfg.local_size;
                fp.Gtot = Gt;
                fp.l_bs = static_cast<int>(cfg.unit_size);
                launch_finalize(fp, st);
                ++launches;
            }
            if (completed > 0) {
                SelectParams sp{};
                sp.unit_scores = L.unit_scores.as<float>();
                sp.unit_len = L.ulen.as<int32_t>();
                sp.unit_k = upage_k(L);
                sp.repr = L.repr.p;
                sp.repr_idx = L.repr_idx.as<int32_t>();
                sp.u0 = L.n_units;
                sp.n_units = completed;
                sp.G = Gs;
                sp.r_k = static_cast<int>(cfg.n_repr);
                sp.d = d;
                sp.l_bs = static_cast<int>(cfg.unit_size);
                set_page(sp, L, L.pend_start);
                if (coll) {
                    coll->select.push_back(sp);
                } else if (dec_chain) {
                    chain_sp = sp;
                    chain_sel = true;
                } else {
                    launch_select<T>(sp, st);
                }
                ++launches;
                for (int64_t c = 0; c < completed; ++c) {
                    L.unit_start.push_back(L.pend_start + c * cfg.unit_size);
                    L.unit_len.push_back(static_cast<int32_t>(cfg.unit_size));
                }
                L.n_units += completed;
                L.pend_start += completed * cfg.unit_size;
            }
            L.pend_count = new_pending - completed * cfg.unit_size;
            L.local_start += overflow;
            L.init_len += to_init;
        } else if (fused_front) {
            issue_front(EvictParams{}, st);  // nothing leaves the window: prep only
            ++launches;
        }
        if (overflow > 0 || fused_front) phase_end(kPhEvict, eve, est);
        rec(e_evict, est);
        evict_seq = kseq;
        st = side;


        // K1 + K2: lookup (memory.hpp:239-269)
        bool k4_pdl = false;  // the lookup is the last kernel before K4 on the caller's stream
        if (do_lookup) {
            const auto evp = phase_begin("lookup", st);
            LookupParams lp{};
            lp.qsum = chunk_qsum.as<double>() + pb * Gs * d;
            lp.repr = L.repr.p;
            lp.part = L.lookup_part.as<double>();
            lp.U = n_units0;
            lp.G = Gs;
            lp.Gtot = Gt;
            lp.g0 = g0;
            lp.r_k = static_cast<int>(cfg.n_repr);
            lp.d = d;
            // single shard: relevance + exact top-k fused into one launch (last lookup
            // block, 256 threads x 8 ids); beyond that rel + a multi-block top-k
            lp.fused = Gs == Gt ? (n_units0 <= 256 * 8 ? 1 : 2) : 0;
            lp.rel = L.rel.as<double>();
            lp.sel = sel_b;
            lp.done = topk_done.as<unsigned int>();
            lp.n_sel = n_sel;
            lp.early_dependents = one_stream ? 1 : 0;  // decode: K4 (or the chained front) follows as a dependent
            // batched decode with the fused front (one-token steps, bf16 d 128): the scan
            // forms the query sums from q too, so the batch's fronts run beside it
            const bool bchain_q = coll && fused_front && dec_chain_opt && Gs == Gt && d == 128 && Gs <= 8 &&
                                  !(reinterpret_cast<uintptr_t>(q) & 7);
            lp.qtok = (dec_chain || bchain_q) ? q : nullptr;
            lp.qrep = rep;
            last_lkp = lp;
            if (coll) {  // batched: relevance scan (rel only) + one top-k block per sequence
                lp.fused = 2;
                coll->lookup.push_back(lp);
            }
            // one-token steps keep the latency-tuned two-kernel path (fused radix tail, K4
            // as its programmatic dependent); chunk steps take the one-launch kernel sized
            // for the ~20 SMs the attention leaves free
            const bool fast = !coll && (!one_stream || (dec_lk_fused && n_units0 > 256 * 8)) && Gs == Gt &&
                              lookup_topk_supported(lp, dtype == INFLLM_DTYPE_BF16);
            if (fast) {
                // one launch: scan + exact top-k; few fat blocks inside the prefill
                // pipeline (the attention holds most SMs), one unit per warp in decode
                const int64_t nc = topk_multi_scratch(n_units0, n_sel);
                lp.cand_v = L.cand.as<double>();
                lp.cand_i = reinterpret_cast<int64_t*>(L.cand.as<double>() + nc);
                lp.fused = 1;
                last_lkp = lp;
                launch_lookup_topk_fast(lp, lookup_topk_blocks(n_units0, one_stream ? lookup_upb_decode : lookup_upb), st);
            } else if (coll) {
            } else if (lp.fused != 2) {
                launch_lookup(lp, dtype == INFLLM_DTYPE_BF16, st);
            }
            if (!lp.fused) gather(L.lookup_part.as<double>(), n_units0, st);
            TopkParams tp{};
            tp.part = L.lookup_part.as<double>();
            tp.rel = L.rel.as<double>();
            tp.sel = sel_b;
            tp.U = n_units0;
            tp.n_sel = n_sel;
            tp.Gtot = Gt;
            if (!lp.fused) launch_topk(tp, st);
            int n_lk = lp.fused == 1 ? 1 : 2;
            // decode chain: the front (a programmatic dependent of the scan, waiting for it
            // before it exits) and a completed unit's page copy go right after the scan
            struct ChainCtx {
                PrepParams pp;
                EvictParams ep;
                SelectParams sp;
                bool sel;
            } cctx{pp, chain_ep, chain_sp, chain_sel};
            cctx.pp.dec_chain = 1;
            auto chain_issue = [](void* c, cudaStream_t s2) {
                auto* x = static_cast<ChainCtx*>(c);
                launch_dec_front(x->pp, x->ep, s2);
                if (x->sel) launch_select<T>(x->sp, s2);
            };
            bool chain_done = false;
            if (lp.fused == 2 && !coll && !fast) {
                const int64_t nc = topk_multi_scratch(n_units0, n_sel);  // <= the size ensure_units reserved
                double* cv = L.cand.as<double>();
                n_lk = launch_lookup_topk(lp, dtype == INFLLM_DTYPE_BF16, cv, reinterpret_cast<int64_t*>(cv + nc), st,
                                          dec_chain ? +chain_issue : nullptr, &cctx);
                chain_done = dec_chain;
            }
            launches += n_lk;
            k4_pdl = one_stream && !coll && !prof && n_sel > 0 && lp.fused != 0;
            if (dec_chain && !chain_done) {  // the front (and a completed unit's page copy) behind the lookup
                if (lp.fused != 1) throw StreamError("decode chain: lookup path mismatch");
                chain_issue(&cctx, st);
            }
            phase_end(kPhLookup, evp, st);
        }

        rec(e_topk, side);
        wt(main, e_topk);
        if (tier_slots > 0 && n_sel > 0) {  // GPU unit cache: slots for this step's units, PCIe pull of the misses
            wt(tier_st, e_topk);
            // k_tier_assign keeps the slots of steps k-1 and k: the attention of k-2 must be done
            const int b2 = static_cast<int>((kseq + kSB - 2) % kSB);
            if (lru_seq[b2] == kseq - 2 && (capture_seq0 < 0 || lru_seq[b2] >= capture_seq0)) wt(tier_st, e_lru[b2]);
            TierParams tp2{};
            tp2.sel = sel_b;
            tp2.sel_slot = L.sel_slot.as<int32_t>() + b * std::max<int64_t>(cfg.n_lookup, 1);
            tp2.unit_slot = L.unit_slot.as<int32_t>();
            tp2.slot_unit = L.slot_unit.as<int64_t>();
            tp2.slot_used = L.slot_used.as<int64_t>();
            tp2.miss = L.tier_miss.as<int32_t>() + 1;
            tp2.miss_n = L.tier_miss.as<int32_t>();
            tp2.stats = L.tier_stats.as<int64_t>();
            tp2.host_k = L.dhost_k;
            tp2.host_krot = L.dhost_krot;
            tp2.host_v = L.dhost_v;
            tp2.slot_k = L.slot_k.p;
            tp2.slot_krot = L.slot_krot.p;
            tp2.slot_v = L.slot_v.p;
            tp2.n_sel = n_sel;
            tp2.S = tier_slots;
            tp2.step = L.step;
            tp2.page_k = static_cast<int64_t>(unit_elems_k() * esz);
            tp2.page_v = static_cast<int64_t>(unit_elems_v() * esz);
            tp2.kmax = static_cast<int>(n_sel);
            launch_tier(tp2, tier_st);
            tier_seq = kseq;
            launches += 2;
            rec(e_tier, tier_st);
            wt(main, e_tier);
        }
        rec(e_lookup, side);
        lookup_seq = kseq;
        // this parity's mass buffers were last read by LRU(k-2)
        if (lru_seq[b] >= 0 && (capture_seq0 < 0 || lru_seq[b] >= capture_seq0))
            wt(main, e_lru[b]);
        if (dual && out_free) wt(main, out_free);  // host path: stage_o of this group drained
        st = main;
        double* mass_cta_b = mass_cta.as<double>() + b * mass_cta_half;
        double* mass_part_b = L.mass_part.as<double>() + b * std::max<int64_t>(cfg.n_lookup, 1) * Gt;

        // K3: attention over [initial | retrieved | local | chunk] (attention.hpp:116-230)
        const bool want_mass = do_lookup && n_sel > 0;
        AttnParams ap{};
        ap.qa = qa_b;
        ap.qc = qc_b;
        // C-2: with gather_output the caller's `out` holds all heads; this shard's
        // heads go to a staging buffer and are all-gathered after the attention
        const bool gout = comm && gather_output && Gs != Gt && !coll;
        ap.out = gout ? out_stage.p : out;
        ap.init_k = L.init_k.p;
        ap.init_krot = L.init_krot.p;
        ap.init_v = L.init_v.p;
        const bool tier = tier_slots > 0;
        ap.unit_k = tier ? L.slot_k.p : L.unit_k.p;
        ap.unit_krot = tier ? L.slot_krot.p : L.unit_krot.p;
        ap.unit_v = tier ? L.slot_v.p : L.unit_v.p;
        ap.unit_len = L.ulen.as<int32_t>();
        ap.sel = sel_b;
        ap.sel_slot = tier ? L.sel_slot.as<int32_t>() + b * std::max<int64_t>(cfg.n_lookup, 1) : nullptr;
        ap.ring_k = L.ring_k.p;
        ap.ring_krot = L.ring_krot.p;
        ap.ring_v = L.ring_v.p;
        ap.mass_e = mass_e.as<float>();
        ap.mass_m = mass_m.as<float>();
        ap.row_m = row_m.as<float>();
        ap.row_l = row_l.as<float>();
        ap.mass_cta = mass_cta_b;
        ap.kmax2 = score_bound ? pp.kmax2 : nullptr;
        ap.R = R;
        ap.s = s;
        ap.lx = lx;
        ap.lxp = lxp;
        ap.init_len = init_len0;
        ap.local_start = local_start0;
        ap.L = cfg.local_size;
        ap.l_I = cfg.init_size;
        ap.n_sel = static_cast<int>(n_sel);
        ap.H = Hs;
        ap.G = Gs;
        ap.rep = rep;
        ap.d = d;
        ap.dv = dv;
        ap.l_bs = static_cast<int>(cfg.unit_size);
        ap.absolute = cfg.position_mode == INFLLM_POSITION_ABSOLUTE;
        ap.want_mass = want_mass;
        ap.scale = 1.0f / std::sqrt(static_cast<float>(d));  // attention.hpp:140
        ap.vl = vl;
        ap.unit_cap = tier ? tier_slots : L.unit_cap;
        ap.mass_part = mass_part_b;
        ap.Gtot = Gt;
        ap.g0 = g0;
        const bool dec_ran = lx == 1 && use_dec && !dec_disabled;
        if (dec_ran) {  // K4 tensor maps of this layer's buffers (rebuilt only when one moved or grew)
            const int64_t urows = (tier ? tier_slots : L.unit_cap) * static_cast<int64_t>(Gs) * 128;
            std::vector<const void*> key{ap.init_k, ap.init_v, ap.unit_k, ap.unit_v, ap.ring_krot, ap.ring_v,
                                         reinterpret_cast<const void*>(urows)};
            if (key != L.dec_maps_key || !L.dec_maps.p) {
                alignas(64) CUtensorMap hm[6];
                dec_encode_maps(ap, urows, hm);
                if (!L.dec_maps.p) L.dec_maps.alloc(sizeof(hm), st, false);
                if (reinterpret_cast<uintptr_t>(L.dec_maps.p) % 128)
                    throw StreamError("K4 tensor maps: device buffer not 128-byte aligned");
                ck(cudaMemcpyAsync(L.dec_maps.p, hm, sizeof(hm), cudaMemcpyHostToDevice, st), "tensor maps H2D");
                ck(cudaStreamSynchronize(st), "tensor maps");  // hm is a stack buffer
                L.dec_maps_key = key;
            }
            ap.dec_maps = L.dec_maps.p;
        }
        last_ap = ap;
        ap.inv_violations = inv_dev.as<unsigned long long>();
        const auto eva = phase_begin("attend", st);
        if constexpr (std::is_same_v<T, bf16>) {
            if (dec_ran) {
                if (coll)
                    coll->attn.push_back(ap);
                else {
                    DecScratch sc = dec_scratch();
                    sc.pdl = dec_chain ? 2 : k4_pdl ? 1 : 0;  // behind the chain every split waits
                    sc.sep_merge = dec_merge_opt ? 1 : 0;
                    launch_attn_dec(ap, sc, st);
                    if (sc.sep_merge) ++launches;  // k_dec_merge1
                }
                ++launches;
            } else if (tc_eligible(lx)) {
                ap.n_split = pick_splits_tc(lx, ap);
                // one split scratch: after the other stream's attention
                if (ap.n_split > 1 && dual && attn_last >= 0 && (capture_seq0 < 0 || attn_last >= capture_seq0))
                    wt(main, e_attn);
                if (ap.n_split > 1) {
                    ap.split_o = split_o.as<float>();
                    ap.split_ml = split_ml.as<float>();
                }
                launches += launch_attn_tc(ap, st);
            } else {
                launch_attn_simt<T>(ap, st);
                ++launches;
            }
        } else {
            launch_attn_simt<T>(ap, st);
            ++launches;
        }
        phase_end(kPhAttend, eva, st);
        if (gout) {
            const int64_t row = static_cast<int64_t>(dv) * static_cast<int64_t>(esz);
            nck(nccl().all_gather(out_stage.p, out_recv.p, static_cast<size_t>(lx * Hs * row), ncclUint8,
                                  static_cast<ncclComm_t>(comm), st),
                "ncclAllGather (outputs)");
            const int64_t pieces = comm_size * lx * Hs * (row / 16);
            k_interleave_heads<<<static_cast<unsigned>((pieces + 255) / 256), 256, 0, st>>>(
                out_recv.as<uint8_t>(), lx, Hs, comm_size, row, static_cast<uint8_t*>(out));
            ++launches;
        }
        if (want_mass) inv_checks += static_cast<uint64_t>(Hs) * lx;  // check_softmax rows (engine.hpp:266)

        // attention masses -> lookup bookkeeping, frequency update, capacity
        // (engine.hpp:257,271-285; memory.hpp:254-300)
        const bool tc_ran = std::is_same_v<T, bf16> && tc_eligible(lx) && !dec_ran;
        int mass_src = 0;
        if (want_mass) {
            if (dec_ran) {
                gather(mass_part_b, n_sel, st);  // per-group masses written by the decode kernel
            } else if (tc_ran && attn_tc_masses_in_kernel(static_cast<int>(n_sel)) && ap.n_split <= 1) {
                if (Gs == Gt) {
                    mass_src = 1;
                } else {
                    launch_mass_cta_reduce(mass_cta_b, mass_part_b, static_cast<int>(n_sel), Gs,
                                           Gt, g0, rep, static_cast<int>((lx + 127) / 128), st);
                    ++launches;
                    gather(mass_part_b, n_sel, st);
                }
            } else {
                MassParams mp{};
                mp.mass_e = mass_e.as<float>();
                mp.mass_m = mass_m.as<float>();
                mp.row_m = row_m.as<float>();
                mp.row_l = row_l.as<float>();
                mp.part = mass_part_b;
                mp.lx = lx;
                mp.n_sel = static_cast<int>(n_sel);
                mp.H = Hs;
                mp.G = Gs;
                mp.Gtot = Gt;
                mp.g0 = g0;
                mp.rep = rep;
                launch_mass(mp, st);
                ++launches;
                gather(mass_part_b, n_sel, st);
            }
        }
        LruParams lp{};
        lp.mass_part = mass_part_b;
        lp.mass_cta = mass_cta_b;
        lp.sel = sel_b;
        lp.freq = L.freq.as<double>();
        lp.hot = L.hot.as<int8_t>();
        lp.hot_list = L.hot_list.as<int64_t>();
        lp.unit_len = L.ulen.as<int32_t>();
        lp.lru = L.lru.as<LruState>();
        lp.trace = L.trace.as<int64_t>();
        lp.n_sel = n_sel;
        lp.n_mass = want_mass ? n_sel : 0;
        lp.cap = cfg.hot_capacity;
        lp.step = L.step;
        lp.Gtot = Gt;
        lp.G = Gs;
        lp.rep = rep;
        lp.n_mt = static_cast<int>((lx + 127) / 128);
        lp.H_total = H;
        lp.mass_src = mass_src;
        lp.decay = cfg.decay;
        lp.bytes_per_token = static_cast<int64_t>(Gs) * (d + dv) * static_cast<int64_t>(esz);
        // TieredStore bookkeeping runs on its own stream, off the attention critical path
        rec(e_attn, main);
        rec(e_attnp[pb], main);
        attn_seq[pb] = kseq;
        attn_last = kseq;
        wt(lru_st, e_attn);
        if (lru_side) {
            ck(cudaEventRecord(e_attn, main), "record");
            ck(cudaStreamWaitEvent(lru_st, e_attn, 0), "wait");
        }
        last_lp = lp;
        const auto evl = coll ? std::pair<cudaEvent_t, cudaEvent_t>{} : phase_begin("evict", lru_st);
        if (coll)
            coll->lru.push_back(lp);
        else
            launch_lru(lp, lru_st);
        if (!coll) phase_end(kPhEvict, evl, lru_st);
        ++launches;
        rec(e_lru[b], lru_st);
        if (lru_side) ck(cudaEventRecord(e_lru[b], lru_st), "record");
        lru_seq[b] = kseq;
        if (dual) wt(caller, e_attn);  // the caller's stream follows every attention (outputs)
        st = side;

        if (one_stream) {  // nothing else was recorded: no later step may wait on those events
            if (!lru_side)
                for (auto& x : lru_seq) x = -1;
            for (auto& a2 : attn_seq) a2 = -1;
            attn_last = -1;
            lookup_seq = evict_seq = tier_seq = -1;
        }
        L.trace_count += n_sel;
        L.last_n_sel = n_sel;
        L.last_b = b;
        L.n_fed += lx;
        L.step += 1;
        {  // check_conservation (engine.hpp:373-383): every fed token is initial, local, pending or in a unit
            ++inv_checks;
            const int64_t in_units = L.n_units ? L.unit_start.back() + L.unit_len.back() - cfg.init_size : 0;
            if (L.init_len + (L.n_fed - L.local_start) + L.pend_count + in_units != L.n_fed) ++inv_conservation_bad;
        }
        ck(cudaGetLastError(), "kernel launch");
    }

    // pointer to chunk `off` of a token-major tensor with `row` elements per token
    const void* at(const void* p, int64_t off, int64_t row) const {
        return static_cast<const uint8_t*>(p) + off * row * static_cast<int64_t>(esz);
    }

    template <typename T>
    void run_chunks(int li, const void* q, const void* k, const void* v, int64_t n, void* out, cudaStream_t st) {
        for (int64_t off = 0; off < n; off += cfg.chunk_size) {
            const int64_t lx = std::min<int64_t>(cfg.chunk_size, n - off);
            step<T>(li, at(q, off, Hs * d), at(k, off, Gs * d), at(v, off, Gs * dv), lx, false,
                    const_cast<void*>(at(out, off, Hs * dv)), st, off == 0);
        }
    }

    // host-pointer stream: H2D of q/k/v into staging buffers and D2H of the
    // outputs in groups of kGroup chunks (PCIe moves multi-MB copies in both
    // directions at once far better than per-chunk ones), on their own streams,
    // overlapping the neighbouring groups' compute
    static constexpr int kGroup = 16;
    template <typename T>
    void run_chunks_host(int li, const void* hq, const void* hk, const void* hv, int64_t n, void* hout,
                         cudaStream_t st) {
        const int64_t C = cfg.chunk_size;
        // groups of chunks: ramped 1, 2, 4, 8 at both ends of a long stream (the first
        // compute waits for one group's H2D and the last D2H waits for one group's
        // compute, so small end groups shorten the fill and the drain), kGroup between
        const int64_t nc = (n + C - 1) / C;
        std::vector<int64_t> gch;  // chunks per group
        if (nc >= 4 * kGroup) {
            const int64_t ramp[4] = {1, 2, 4, 8};
            for (int64_t r : ramp) gch.push_back(r);
            int64_t mid = nc - 30;
            for (; mid >= kGroup; mid -= kGroup) gch.push_back(kGroup);
            if (mid > 0) gch.push_back(mid);
            for (int r = 3; r >= 0; --r) gch.push_back(ramp[r]);
        } else {
            for (int64_t c0 = 0; c0 < nc; c0 += kGroup) gch.push_back(std::min<int64_t>(kGroup, nc - c0));
        }
        const int64_t ng = static_cast<int64_t>(gch.size());
        std::vector<int64_t> goffs(ng + 1, 0);  // token offset of each group
        for (int64_t t = 0; t < ng; ++t) goffs[t + 1] = std::min<int64_t>(n, goffs[t] + gch[t] * C);
        std::vector<cudaEvent_t> ev_in(ng), ev_comp(ng), ev_out(ng);
        for (int64_t t = 0; t < ng; ++t) {
            ev_in[t] = take_event();
            ev_comp[t] = take_event();
            ev_out[t] = take_event();
        }
        cudaEvent_t fork = take_event();
        ck(cudaEventRecord(fork, st), "fork");
        ck(cudaStreamWaitEvent(h2d_stream, fork, 0), "fork");
        ck(cudaStreamWaitEvent(d2h_stream, fork, 0), "fork");
        auto h2d = [&](int64_t gi) {
            const int64_t off = goffs[gi], len = goffs[gi + 1] - goffs[gi];
            const int b = static_cast<int>(gi % kNB);
            if (gi >= kNB) ck(cudaStreamWaitEvent(h2d_stream, ev_comp[gi - kNB], 0), "wait");
            ck(cudaMemcpyAsync(stage_q[b].p, at(hq, off, Hs * d), len * Hs * d * esz, cudaMemcpyHostToDevice,
                               h2d_stream),
               "H2D");
            ck(cudaMemcpyAsync(stage_k[b].p, at(hk, off, Gs * d), len * Gs * d * esz, cudaMemcpyHostToDevice,
                               h2d_stream),
               "H2D");
            ck(cudaMemcpyAsync(stage_v[b].p, at(hv, off, Gs * dv), len * Gs * dv * esz, cudaMemcpyHostToDevice,
                               h2d_stream),
               "H2D");
            ck(cudaEventRecord(ev_in[gi], h2d_stream), "record");
        };
        for (int64_t gi = 0; gi < std::min<int64_t>(kNB - 1, ng); ++gi) h2d(gi);
        for (int64_t gi = 0; gi < ng; ++gi) {
            if (gi + kNB - 1 < ng) h2d(gi + kNB - 1);
            const int64_t goff = goffs[gi], glen = goffs[gi + 1] - goffs[gi];
            const int b = static_cast<int>(gi % kNB);
            if (gi >= kNB) ck(cudaStreamWaitEvent(st, ev_out[gi - kNB], 0), "wait");  // stage_o[b] drained
            out_free = gi >= kNB ? ev_out[gi - kNB] : nullptr;  // the attention streams wait for it too
            for (int64_t off = 0; off < glen; off += C) {
                const int64_t lx = std::min<int64_t>(C, glen - off);
                step<T>(li, at(stage_q[b].p, off, Hs * d), at(stage_k[b].p, off, Gs * d),
                        at(stage_v[b].p, off, Gs * dv), lx, false, const_cast<void*>(at(stage_o[b].p, off, Hs * dv)), st,
                        gi == 0 && off == 0, off == 0 ? ev_in[gi] : nullptr);
            }
            out_free = nullptr;
            ck(cudaEventRecord(ev_comp[gi], st), "record");
            ck(cudaStreamWaitEvent(d2h_stream, ev_comp[gi], 0), "wait");
            ck(cudaMemcpyAsync(const_cast<void*>(at(hout, goff, Hs * dv)), stage_o[b].p, glen * Hs * dv * esz,
                               cudaMemcpyDeviceToHost, d2h_stream),
               "D2H");
            ck(cudaEventRecord(ev_out[gi], d2h_stream), "record");
        }
        ck(cudaStreamWaitEvent(st, ev_out[ng - 1], 0), "join");
        ck(cudaStreamWaitEvent(st, ev_in[ng - 1], 0), "join");
        for (int64_t t = 0; t < ng; ++t) {
            ev_pool.push_back(ev_in[t]);
            ev_pool.push_back(ev_comp[t]);
            ev_pool.push_back(ev_out[t]);
        }
        ev_pool.push_back(fork);
    }

    template <typename T>
    void encode_stream(int li, const void* q, const void* k, const void* v, int64_t n, void* out, cudaStream_t st,
                       bool host) {
        NvtxRange nv("encode_stream");
        if (li < 0 || li >= n_layers) throw StreamError("layer out of range");
        if (n < 1) throw StreamError("encode_stream: empty stream");
        Layer& L = layers[static_cast<size_t>(li)];
        join_ext(st);
        if (!cap_stream) {
            ck(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking), "stream");
            ck(cudaStreamCreateWithFlags(&h2d_stream, cudaStreamNonBlocking), "stream");
            ck(cudaStreamCreateWithFlags(&d2h_stream, cudaStreamNonBlocking), "stream");
        }
        // capacity for the whole stream up front (no pool growth inside a graph)
        const int64_t steps = (n + cfg.chunk_size - 1) / cfg.chunk_size;
        if (use_tc && max_splits_tc() > 1) ensure_split_scratch(max_splits_tc());
        ensure_units(L, L.n_units + (L.pend_count + n) / cfg.unit_size + 2, st);
        ensure_trace(L, L.trace_count + steps * std::max<int64_t>(cfg.n_lookup, 1), st);
        if (host && !stage_q[0].p) {
            const int64_t C = cfg.chunk_size * kGroup;
            for (int b = 0; b < kNB; ++b) {
                stage_q[b].alloc(C * Hs * d * esz, st, false);
                stage_k[b].alloc(C * Gs * d * esz, st, false);
                stage_v[b].alloc(C * Gs * dv * esz, st, false);
                stage_o[b].alloc(C * Hs * dv * esz, st, false);
            }
        }
        // host-buffer streams run eagerly: copies issued as plain cudaMemcpyAsync overlap
        // the compute better than the same copies as graph nodes (35.3 vs 37.1 ms per
        // 128K stream, tools/e2e_probe.py); host exchange hooks cannot be captured
        if (!use_graphs || host || (allgather && Gs != Gt)) {
            if (host)
                run_chunks_host<T>(li, q, k, v, n, out, st);
            else
                run_chunks<T>(li, q, k, v, n, out, st);
            return;
        }
        const HostState cur = save(L);
        // a graph whose buffers have moved since its capture (pool growth, decode
        // scratch, ...) would replay into freed memory: drop it
        const std::vector<const void*> bufs = buf_snapshot();
        for (size_t i = graphs.size(); i-- > 0;)
            if (graphs[i].bufs != bufs) {
                ck(cudaStreamSynchronize(st), "graph drop");
                drop_graph(graphs[i]);
                graphs.erase(graphs.begin() + static_cast<std::ptrdiff_t>(i));
            }
        GraphEntry* ge = nullptr;
        for (auto& g : graphs)
            if (g.layer == li && g.q == q && g.k == k && g.v == v && g.out == out && g.n == n && g.host == host &&
                g.prof == prof && g.before == cur)
                ge = &g;
        if (!ge) {
            ck(cudaStreamSynchronize(st), "pre-capture sync");
            GraphEntry g;
            g.layer = li;
            g.q = q;
            g.k = k;
            g.v = v;
            g.out = out;
            g.n = n;
            g.host = host;
            g.prof = prof;
            g.before = cur;
            g.bufs = bufs;
            const int64_t l0 = launches;
            const uint64_t c0 = inv_checks, b0 = inv_conservation_bad;
            cudaGraph_t graph = nullptr;
            capturing = true;
            cap_ev = g.ev;
            const int64_t seq0 = seq;
            ck(cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeThreadLocal), "begin capture");
            capture_seq0 = seq;
            try {
                if (host)
                    run_chunks_host<T>(li, q, k, v, n, out, cap_stream);
                else
                    run_chunks<T>(li, q, k, v, n, out, cap_stream);
                join_side(cap_stream);
            } catch (...) {
                capturing = false;
                capture_seq0 = -1;
                out_free = nullptr;
                cudaStreamEndCapture(cap_stream, &graph);
                if (graph) cudaGraphDestroy(graph);
                restore(L, cur);
                seq = seq0;
                throw;
            }
            capturing = false;
            capture_seq0 = -1;
            g.steps = seq - seq0;
            seq = seq0;
            ck(cudaStreamEndCapture(cap_stream, &graph), "end capture");
            // node priorities (the attention launches carry the highest) are honoured
            // only with this flag: without it the graph's pending side-kernel blocks and
            // the next attention's CTAs are dispatched in plain launch order
            ck(cudaGraphInstantiate(&g.exec, graph, graph_prio ? cudaGraphInstantiateFlagUseNodePriority : 0),
               "graph instantiate");
            cudaGraphDestroy(graph);
            g.after = save(L);
            g.launches = launches - l0;
            launches = l0;
            g.inv_checks = inv_checks - c0;
            g.inv_bad = inv_conservation_bad - b0;
            inv_checks = c0;
            inv_conservation_bad = b0;
            restore(L, cur);
            if (graphs.size() >= kMaxGraphs) {  // bounded cache: the oldest capture goes
                ck(cudaStreamSynchronize(st), "graph drop");
                drop_graph(graphs.front());
                graphs.erase(graphs.begin());
            }
            graphs.push_back(std::move(g));
            ge = &graphs.back();
        }
        join_side(st);  // the graph starts from a quiet side stream and joins it at its end
        ck(cudaGraphLaunch(ge->exec, st), "graph launch");
        seq += ge->steps;
        restore(L, ge->after);
        launches += ge->launches;
        inv_checks += ge->inv_checks;
        inv_conservation_bad += ge->inv_bad;
        if (prof) ge->replays_in_window++;
    }

    template <typename T>
    void finish(cudaStream_t st) {  // engine.hpp:115-119, UnitPacker::flush memory.hpp:81-84
        join_side(st);
        for (auto& L : layers) {
            if (L.pend_count == 0) continue;
            ensure_units(L, L.n_units + 1, st);
            const int32_t len = static_cast<int32_t>(L.pend_count);
            k_fill_i32<<<1, 1, 0, st>>>(L.ulen.as<int32_t>() + L.n_units, 1, len);
            ++launches;
            SelectParams sp{};
            sp.unit_scores = L.unit_scores.as<float>();
            sp.unit_len = L.ulen.as<int32_t>();
            sp.unit_k = upage_k(L);
            sp.repr = L.repr.p;
            sp.repr_idx = L.repr_idx.as<int32_t>();
            sp.u0 = L.n_units;
            sp.n_units = 1;
            sp.G = Gs;
            sp.r_k = static_cast<int>(cfg.n_repr);
            sp.d = d;
            sp.l_bs = static_cast<int>(cfg.unit_size);
            set_page(sp, L, L.pend_start);
            launch_select<T>(sp, st);
            ++launches;
            L.unit_start.push_back(L.pend_start);
            L.unit_len.push_back(len);
            L.n_units += 1;
            L.pend_start += L.pend_count;
            L.pend_count = 0;
        }
        ck(cudaStreamSynchronize(st), "finish");
    }
};

namespace {
bool batchable(const infllm_engine* e, const infllm_engine* e0, int32_t layer) {
    return e && e->dtype == INFLLM_DTYPE_BF16 && e->use_dec && !e->dec_disabled && e->Gs == e->Gt &&
           e->tier_slots == 0 && e->page_mode() && e->H == e0->H && e->Gt == e0->Gt && e->d == e0->d &&
           e->dv == e0->dv && e->device == e0->device && std::memcmp(&e->cfg, &e0->cfg, sizeof(e->cfg)) == 0 &&
           layer >= 0 && layer < e->n_layers && e->layers[static_cast<size_t>(layer)].n_units <= 8192;
}
template <typename P>
size_t put(std::vector<uint8_t>& buf, const std::vector<P>& v) {
    const size_t off = (buf.size() + 255) / 256 * 256;
    buf.resize(off + v.size() * sizeof(P));
    if (!v.empty()) std::memcpy(buf.data() + off, v.data(), v.size() * sizeof(P));
    return off;
}
}  // namespace

extern "C" {

const char* infllm_last_error(void) { return g_err.c_str(); }

const char* infllm_version(void) {
    return "infllm_b200 0.1 (sm_100a; fp32 CUDA-core + bf16 tcgen05 attention)";
}

int infllm_config_default(infllm_engine_config* c) {
    if (!c) return INFLLM_ERR_ARG;
    c->chunk_size = 512;
    c->unit_size = 128;
    c->n_repr = 4;
    c->local_size = 4096;
    c->init_size = 128;
    c->n_lookup = 32;
    c->hot_capacity = 32;
    c->decay = 0.1;
    c->lookup_mode = INFLLM_LOOKUP_ENCODE_AND_DECODE;
    c->position_mode = INFLLM_POSITION_CLAMPED;
    return INFLLM_OK;
}

int infllm_config_validate(const infllm_engine_config* cfg, const infllm_model_shape* shape) {
    return guard([&] {
        if (!cfg) throw ConfigError("null config");
        validate_cfg(*cfg);
        if (shape) validate_shape(*shape);
    });
}

int infllm_engine_create(const infllm_engine_config* cfg, const infllm_model_shape* shape, int32_t dtype,
                         int32_t device, int32_t kv_group_begin, int32_t kv_group_count, infllm_engine_t* out) {
    return guard([&] {
        if (!cfg || !shape || !out) throw ConfigError("null argument");
        validate_cfg(*cfg);
        validate_shape(*shape);
        if (dtype != INFLLM_DTYPE_F32 && dtype != INFLLM_DTYPE_BF16) throw ConfigError("dtype must be f32 or bf16");
        auto e = std::make_unique<infllm_engine>();
        e->cfg = *cfg;
        e->H = shape->n_heads;
        e->Gt = shape->n_kv_heads > 0 ? shape->n_kv_heads : shape->n_heads;
        e->rep = e->H / e->Gt;
        e->d = shape->head_dim;
        e->dv = shape->value_dim > 0 ? shape->value_dim : shape->head_dim;
        e->n_layers = shape->n_layers;
        if (e->d > 256 || e->dv > 128) throw ConfigError("head_dim <= 256 and value_dim <= 128 supported");
        if (cfg->n_repr > 32) throw ConfigError("n_repr <= 32 supported");
        if (cfg->n_lookup > 128) throw ConfigError("n_lookup <= 128 supported");
        if (cfg->hot_capacity + cfg->n_lookup > 510) throw ConfigError("hot_capacity + n_lookup <= 510 supported");
        if (kv_group_count <= 0) {
            kv_group_begin = 0;
            kv_group_count = e->Gt;
        }
        if (kv_group_begin < 0 || kv_group_begin + kv_group_count > e->Gt)
            throw ConfigError("kv group shard out of range");
        e->g0 = kv_group_begin;
        e->Gs = kv_group_count;
        e->Hs = e->Gs * e->rep;
        e->dtype = dtype;
        e->device = device;
        e->esz = dtype == INFLLM_DTYPE_BF16 ? 2 : 4;
        // ring: the local window, the chunk being attended and the two chunks the
        // prep stream may run ahead by never share a slot
        const int64_t need = cfg->local_size + infllm_engine::kPB * cfg->chunk_size + 1;
        e->R = (need + 127) / 128 * 128;
        e->lxp = (cfg->chunk_size + 127) / 128 * 128;
        for (int a = 0; a < e->d / 2; ++a) {  // rotary.hpp:25-30 (RotaryTable::make)
            e->freqs.f[a] = std::pow(10000.0, -2.0 * a / e->d);
            const double ang = static_cast<double>(cfg->local_size) * e->freqs.f[a];
            e->freqs.cL[a] = static_cast<float>(std::cos(ang));
            e->freqs.sL[a] = static_cast<float>(std::sin(ang));
        }
        e->use_tc = dtype == INFLLM_DTYPE_BF16 && attn_tc_supported(e->d, e->dv, static_cast<int>(cfg->unit_size),
                                                                     cfg->position_mode == INFLLM_POSITION_ABSOLUTE);
        e->vl.vt = e->use_tc ? 1 : 0;
        e->use_dec = e->use_tc && attn_dec_supported(e->d, e->dv, static_cast<int>(cfg->unit_size), e->rep,
                                                     cfg->position_mode == INFLLM_POSITION_ABSOLUTE, 1);
        e->vl.R = e->R;
        e->vl.nI = static_cast<int>((std::max<int64_t>(cfg->init_size, 1) + 127) / 128);
        e->vl.l_I = cfg->init_size;
        e->vl.l_bs = static_cast<int>(cfg->unit_size);
        e->vl.dv = e->dv;
        e->vl.G = e->Gs;
        ck(cudaSetDevice(device), "cudaSetDevice");
        cudaStream_t st = nullptr;
        const size_t es = e->esz;
        e->qa_half = static_cast<size_t>(e->Hs) * e->lxp * e->d * es;
        e->qa.alloc(infllm_engine::kPB * e->qa_half, st);
        e->qc.alloc(infllm_engine::kPB * e->qa_half, st);
        ck(cudaStreamCreateWithFlags(&e->side_stream, cudaStreamNonBlocking), "side stream");
        ck(cudaStreamCreateWithFlags(&e->lru_stream, cudaStreamNonBlocking), "lru stream");
        ck(cudaStreamCreateWithFlags(&e->prep_stream, cudaStreamNonBlocking), "prep stream");
        ck(cudaStreamCreateWithFlags(&e->evict_stream, cudaStreamNonBlocking), "evict stream");
        ck(cudaStreamCreateWithFlags(&e->tier_stream, cudaStreamNonBlocking), "tier stream");
        {
            int lo = 0, hi = 0;
            ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
            for (auto& s2 : e->attn_st)
                ck(cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, hi), "attention stream");
        }
        for (auto* ev : {&e->e_call, &e->e_topk, &e->e_side, &e->e_lru[0], &e->e_lru[1], &e->e_lru[2], &e->e_attn,
                         &e->e_lrudone, &e->e_prep, &e->e_lookup, &e->e_prepdone, &e->e_evict, &e->e_evdone,
                         &e->e_attnp[0], &e->e_attnp[1], &e->e_attnp[2], &e->e_tier, &e->e_tierdone})
            ck(cudaEventCreateWithFlags(ev, cudaEventDisableTiming), "event");
        e->inv_dev.alloc(sizeof(unsigned long long), st);
        e->chunk_qsum.alloc(infllm_engine::kPB * static_cast<size_t>(e->Gs) * e->d * sizeof(double), st);
        const size_t km = static_cast<size_t>(std::max<int64_t>(cfg->n_lookup, 1));
        e->mass_e.alloc(static_cast<size_t>(e->Hs) * cfg->chunk_size * km * sizeof(float), st);
        e->mass_m.alloc(static_cast<size_t>(e->Hs) * cfg->chunk_size * km * sizeof(float), st);
        e->row_m.alloc(static_cast<size_t>(e->Hs) * cfg->chunk_size * sizeof(float), st);
        e->row_l.alloc(static_cast<size_t>(e->Hs) * cfg->chunk_size * sizeof(float), st);
        e->topk_done.alloc(sizeof(unsigned int), st);
        e->evict_done.alloc(sizeof(unsigned int), st);
        e->rtab.alloc(static_cast<size_t>(cfg->chunk_size) * std::max(1, e->d / 2) * sizeof(float2), st);
        e->tsum.alloc(static_cast<size_t>((cfg->chunk_size + kTokTile - 1) / kTokTile) * e->Gs * e->d * sizeof(double), st);
        e->qsb.alloc(static_cast<size_t>(cfg->chunk_size) * e->Gs * e->d * sizeof(double), st);
        e->mass_cta_half = static_cast<int64_t>(e->Hs) * (e->lxp / 128) * km;
        e->mass_cta.alloc(infllm_engine::kSB * e->mass_cta_half * sizeof(double), st);
        if (e->use_dec) {
            e->dec_part.alloc(dec_part_floats(1, e->Gs, e->rep) * sizeof(float), st, false);
            e->dec_mass.alloc(static_cast<size_t>(e->Hs) * km * kDecWarps * 2 * sizeof(float), st);
            e->dec_cnt.alloc(static_cast<size_t>(e->Gs) * sizeof(unsigned), st);
        }
        e->layers.resize(static_cast<size_t>(e->n_layers));
        for (auto& L : e->layers) {
            L.ring_k.alloc(static_cast<size_t>(e->Gs) * e->R * e->d * es, st);
            L.ring_krot.alloc(static_cast<size_t>(e->Gs) * e->R * e->d * es, st);
            L.ring_v.alloc(static_cast<size_t>(e->Gs) * e->R * e->dv * es, st);
            L.P.alloc(static_cast<size_t>(e->R) * e->Gs * e->d * sizeof(double), st);
            L.kmax2.alloc(infllm_engine::kPB * static_cast<size_t>(e->Gs) * sizeof(float), st);
            const size_t ni = static_cast<size_t>(std::max<int64_t>(cfg->init_size, 1));
            L.init_k.alloc(static_cast<size_t>(e->Gs) * ni * e->d * es, st);
            if (cfg->position_mode == INFLLM_POSITION_ABSOLUTE)
                L.init_krot.alloc(static_cast<size_t>(e->Gs) * ni * e->d * es, st);
            L.init_v.alloc(static_cast<size_t>(e->Gs) * (e->vl.vt ? e->vl.nI * 128 : ni) * e->dv * es, st);
            L.hot_list.alloc(static_cast<size_t>(cfg->hot_capacity + km + 1) * sizeof(int64_t), st);
            L.lru.alloc(sizeof(LruState), st);
            L.sel.alloc(infllm_engine::kSB * km * sizeof(int64_t), st);
            L.mass_part.alloc(infllm_engine::kSB * km * e->Gt * sizeof(double), st);
            L.ev_part.alloc(static_cast<size_t>(cfg->chunk_size) * e->Gt * sizeof(double), st);
        }
        ck(cudaStreamSynchronize(st), "engine_create");
        *out = e.release();
    });
}

int infllm_engine_destroy(infllm_engine_t e) {
    return guard([&] {
        if (!e) return;
        cudaDeviceSynchronize();
        cudaStream_t st = nullptr;
        for (auto* b : e->dev_buffers()) b->release(st);
        for (auto& L : e->layers)
            for (auto* h : {&L.host_k, &L.host_krot, &L.host_v}) h->release();
        for (auto& evs : e->ev)
            for (auto& p : evs) {
                cudaEventDestroy(p.first);
                cudaEventDestroy(p.second);
            }
        for (auto ev : e->ev_pool) cudaEventDestroy(ev);
        for (auto& g : e->graphs) infllm_engine::drop_graph(g);
        if (e->comm) nccl().comm_destroy(static_cast<ncclComm_t>(e->comm));
        for (auto s2 : {e->cap_stream, e->h2d_stream, e->d2h_stream, e->side_stream, e->lru_stream, e->prep_stream,
                        e->evict_stream, e->tier_stream, e->attn_st[0], e->attn_st[1]})
            if (s2) cudaStreamDestroy(s2);
        for (auto ev : {e->e_call, e->e_topk, e->e_side, e->e_lru[0], e->e_lru[1], e->e_lru[2], e->e_attn,
                        e->e_lrudone, e->e_prep, e->e_lookup, e->e_prepdone, e->e_evict, e->e_evdone,
                        e->e_attnp[0], e->e_attnp[1], e->e_attnp[2], e->e_tier, e->e_tierdone})
            if (ev) cudaEventDestroy(ev);
        cudaDeviceSynchronize();
        if (e->bctx) {
            for (int t = 0; t < BatchCtx::kSlots; ++t) {
                if (e->bctx->host[t]) cudaFreeHost(e->bctx->host[t]);
                if (e->bctx->dev[t]) cudaFree(e->bctx->dev[t]);
                if (e->bctx->done[t]) cudaEventDestroy(e->bctx->done[t]);
            }
            for (auto* b : {&e->bctx->part, &e->bctx->mass, &e->bctx->cnt}) b->release(nullptr);
            if (e->bctx->lru_st) cudaStreamDestroy(e->bctx->lru_st);
            if (e->bctx->ev_k4) cudaEventDestroy(e->bctx->ev_k4);
            for (auto ev : e->bctx->lru_ring)
                if (ev) cudaEventDestroy(ev);
        }
        delete e;
    });
}

int infllm_engine_set_allgather(infllm_engine_t e, infllm_allgather_fn fn, void* user) {
    if (!e) return INFLLM_ERR_ARG;
    e->allgather = fn;
    e->allgather_user = user;
    return INFLLM_OK;
}

int infllm_nccl_unique_id(uint8_t* id128) {
    return guard([&] {
        if (!id128) throw ConfigError("null argument");
        ncclUniqueId id;
        nck(nccl().get_unique_id(&id), "ncclGetUniqueId");
        std::memcpy(id128, id.internal, NCCL_UNIQUE_ID_BYTES);
    });
}

int infllm_engine_set_comm(infllm_engine_t e, const uint8_t* id128, int32_t rank, int32_t nranks) {
    return guard([&] {
        if (!e || !id128) throw ConfigError("null argument");
        if (e->comm) throw ConfigError("set_comm: the engine already has a communicator");
        if (nranks < 1 || rank < 0 || rank >= nranks) throw ConfigError("set_comm: bad rank / nranks");
        if (e->Gt % nranks || e->Gs * nranks != e->Gt || e->g0 != rank * e->Gs)
            throw ConfigError("set_comm: rank r must own KV groups [r G/n, (r + 1) G/n)");
        ncclUniqueId id;
        std::memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
        ck(cudaSetDevice(e->device), "cudaSetDevice");
        ncclComm_t c = nullptr;
        nck(nccl().comm_init_rank(&c, nranks, id, rank), "ncclCommInitRank");
        e->comm = c;
        e->comm_rank = rank;
        e->comm_size = nranks;
        int64_t cap = 0;
        for (auto& L : e->layers) cap = std::max(cap, L.unit_cap);
        e->ensure_exchange(std::max<int64_t>({cap, e->cfg.chunk_size, e->cfg.n_lookup}));
        const size_t ob = static_cast<size_t>(e->cfg.chunk_size) * e->Hs * e->dv * e->esz;
        e->out_stage.alloc(ob, nullptr, false);
        e->out_recv.alloc(ob * nranks, nullptr, false);
        ck(cudaDeviceSynchronize(), "set_comm");
    });
}

int infllm_exchange_fold_host(const double* gathered, int64_t rows, int32_t nranks, int32_t g_count, double* out) {
    return guard([&] {
        if (rows < 0 || nranks < 1 || g_count < 1 || (rows > 0 && (!gathered || !out)))
            throw ConfigError("exchange_fold: bad arguments");
        for (int64_t u = 0; u < rows; ++u) {  // group order 0..g_total-1, as k_topk / k_finalize sum them
            double a = 0.0;
            for (int32_t r = 0; r < nranks; ++r)
                for (int32_t g = 0; g < g_count; ++g) a += gathered[(static_cast<int64_t>(r) * rows + u) * g_count + g];
            out[u] = a;
        }
    });
}

int infllm_topk_host(const double* rel, int64_t n, int64_t k, int64_t* ids, int64_t* n_out) {
    return guard([&] {
        if (n < 0 || k < 0 || (n > 0 && (!rel || !ids)) || !n_out) throw ConfigError("topk: bad arguments");
        const int64_t take = std::min(k, n);  // memory.hpp:240-253
        std::vector<int64_t> idx(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) idx[static_cast<size_t>(i)] = i;
        auto better = [&](int64_t a, int64_t b) {
            const double ra = rel[a] == 0.0 ? 0.0 : rel[a], rb = rel[b] == 0.0 ? 0.0 : rel[b];
            return ra != rb ? ra > rb : a < b;
        };
        std::partial_sort(idx.begin(), idx.begin() + take, idx.end(), better);
        std::sort(idx.begin(), idx.begin() + take);
        for (int64_t i = 0; i < take; ++i) ids[i] = idx[static_cast<size_t>(i)];
        *n_out = take;
    });
}

int infllm_engine_reserve(infllm_engine_t e, int64_t max_tokens) {
    return guard([&] {
        cudaStream_t st = nullptr;
        e->sync_ext();
        const int64_t units = std::max<int64_t>(0, max_tokens - e->cfg.init_size) / e->cfg.unit_size + 2;
        for (auto& L : e->layers) {
            e->ensure_units(L, units, st);
            // chunk steps of max_tokens plus 4096 one-token steps: a trace growth drains every
            // stream of the engine (and a batch's LRU), a multi-ms stall inside a decode loop
            const int64_t steps = (max_tokens + e->cfg.chunk_size - 1) / e->cfg.chunk_size + 1 + 4096;
            e->ensure_trace(L, steps * std::max<int64_t>(e->cfg.n_lookup, 1), st);
        }
        ck(cudaStreamSynchronize(st), "reserve");
    });
}

int infllm_engine_reset(infllm_engine_t e, void* stream) {
    return guard([&] {
        auto st = static_cast<cudaStream_t>(stream);
        e->join_ext(st);
        e->join_side(st);
        for (auto& L : e->layers) {
            L.n_fed = L.step = L.local_start = L.init_len = 0;
            L.n_units = L.pend_start = L.pend_count = 0;
            L.trace_count = L.last_n_sel = L.last_b = 0;
            L.unit_start.clear();
            L.unit_len.clear();
            ck(cudaMemsetAsync(L.P.p, 0, L.P.bytes, st), "memset");
            ck(cudaMemsetAsync(L.kmax2.p, 0, L.kmax2.bytes, st), "memset");
            ck(cudaMemsetAsync(L.lru.p, 0, L.lru.bytes, st), "memset");
            if (L.hot.p) ck(cudaMemsetAsync(L.hot.p, 0, L.hot.bytes, st), "memset");
            if (L.freq.p) ck(cudaMemsetAsync(L.freq.p, 0, L.freq.bytes, st), "memset");
            if (L.slot_unit.p) {  // host tier: empty GPU unit cache
                ck(cudaMemsetAsync(L.slot_unit.p, 0xff, L.slot_unit.bytes, st), "memset");
                ck(cudaMemsetAsync(L.slot_used.p, 0, L.slot_used.bytes, st), "memset");
                ck(cudaMemsetAsync(L.unit_slot.p, 0xff, L.unit_slot.bytes, st), "memset");
                ck(cudaMemsetAsync(L.tier_stats.p, 0, L.tier_stats.bytes, st), "memset");
            }
            if (L.ulen.p) {
                k_fill_i32<<<static_cast<unsigned>((L.unit_cap + 255) / 256), 256, 0, st>>>(
                    L.ulen.as<int32_t>(), L.unit_cap, static_cast<int32_t>(e->cfg.unit_size));
                ++e->launches;
            }
        }
        ck(cudaGetLastError(), "reset");
    });
}

int infllm_engine_set_option(infllm_engine_t e, const char* key, int64_t value) {
    return guard([&] {
        if (!e) throw ConfigError("null engine");
        const std::string k = key ? key : "";
        // captured stream graphs bake in the launch choices these options make:
        // drop them so the next encode_stream recaptures with the new setting
        if (k == "tc_attention" || k == "attn_score_bound" || k == "decode_kernel" || k == "multi_stream_decode" ||
            k == "lookup_units_per_block" || k == "lookup_units_per_block_decode" || k == "attn_splits" ||
            k == "gather_output" || k == "attn_streams" || k == "graph_node_priority" || k == "decode_chain" ||
            k == "decode_merge_kernel" || k == "decode_lookup_fused") {
            ck(cudaDeviceSynchronize(), "set_option");
            for (auto& g : e->graphs) infllm_engine::drop_graph(g);
            e->graphs.clear();
        }
        if (k == "tc_attention")
            e->tc_disabled = value == 0;
        else if (k == "cuda_graphs")
            e->use_graphs = value != 0;
        else if (k == "attn_score_bound")
            e->score_bound = value != 0;
        else if (k == "decode_kernel")
            e->dec_disabled = value == 0;
        else if (k == "multi_stream_decode")
            e->multi_stream_decode = value != 0;
        else if (k == "gather_output")
            e->gather_output = value != 0;
        else if (k == "decode_chain")
            e->dec_chain_opt = value != 0;
        else if (k == "decode_lookup_fused")
            e->dec_lk_fused = value != 0;
        else if (k == "decode_merge_kernel")
            e->dec_merge_opt = value != 0;
        else if (k == "graph_node_priority")
            e->graph_prio = value != 0;
        else if (k == "attn_streams")
            e->attn_streams = static_cast<int>(std::clamp<int64_t>(value, 1, 2));
        else if (k == "attn_splits")
            e->attn_splits = static_cast<int>(std::clamp<int64_t>(value, 0, infllm_engine::kMaxSplitsTc));
        else if (k == "lookup_units_per_block_decode")
            e->lookup_upb_decode = static_cast<int>(std::clamp<int64_t>(value, 1, 1 << 20));
        else if (k == "lookup_units_per_block")
            e->lookup_upb = static_cast<int>(std::clamp<int64_t>(value, 1, 1 << 20));
        else if (k == "host_tier_slots") {
            for (auto& L : e->layers)
                if (L.unit_cap > 0 && value != e->tier_slots)
                    throw ConfigError("host_tier_slots must be set before reserve() and the first step");
            const int64_t km = std::max<int64_t>(e->cfg.n_lookup, 1);
            if (value != 0 && (value < 2 * km || value > 16384))
                throw ConfigError("host_tier_slots must be 0 or in [2*n_lookup, 16384]");
            if (value != 0 && ((e->unit_elems_k() * e->esz) % 16 != 0 || (e->unit_elems_v() * e->esz) % 16 != 0))
                throw ConfigError("host_tier_slots: unit pages must be multiples of 16 bytes");
            e->tier_slots = value;
        }
        else
            throw ConfigError("unknown option '" + k + "'");
    });
}

int infllm_encode_chunk(infllm_engine_t e, int32_t layer, const void* q, const void* k, const void* v, int64_t l_x,
                        void* out, void* stream) {
    return guard([&] {
        if (!e) throw ConfigError("null engine");
        auto st = static_cast<cudaStream_t>(stream);
        if (e->dtype == INFLLM_DTYPE_BF16)
            e->step<bf16>(layer, q, k, v, l_x, false, out, st);
        else
            e->step<float>(layer, q, k, v, l_x, false, out, st);
    });
}

int infllm_decode_step(infllm_engine_t e, int32_t layer, const void* q, const void* k, const void* v, void* out,
                       void* stream) {
    return guard([&] {
        if (!e) throw ConfigError("null engine");
        auto st = static_cast<cudaStream_t>(stream);
        if (e->dtype == INFLLM_DTYPE_BF16)
            e->step<bf16>(layer, q, k, v, 1, true, out, st);
        else
            e->step<float>(layer, q, k, v, 1, true, out, st);
    });
}

// Batched decode: one decode step of `n` independent
// sequences (one engine each), every stage one launch for all of them. Each
// engine's step() runs in collect mode (host stream arithmetic, pool growth,
// parameter structs, no launches); the parameter tables go to the device in
// one copy; then prep, eviction, unit selection, lookup + top-k, K4 attention
// and LRU each launch once with grid.z (or grid.x) = sequence.
namespace {
// host time of infllm_decode_batch by section (diagnostic, infllm_debug_host_times;
// relaxed atomics: calls from several host threads add up without a data race)
std::atomic<double> g_dbh[6];
inline double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

int infllm_debug_host_times(double* out6, int32_t reset) {
    return guard([&] {
        if (out6)
            for (int i = 0; i < 6; ++i) out6[i] = g_dbh[i].load(std::memory_order_relaxed);
        if (reset)
            for (auto& x : g_dbh) x.store(0.0, std::memory_order_relaxed);
    });
}

int infllm_decode_batch(infllm_engine_t* engs, int32_t n, int32_t layer, const void* q, const void* k,
                        const void* v, void* out, void* stream) {
    return guard([&] {
        const double h0 = now_us();
        if (!engs || n < 1) throw ConfigError("decode_batch: no engines");
        auto st = static_cast<cudaStream_t>(stream);
        infllm_engine* e0 = engs[0];
        if (!e0) throw ConfigError("null engine");
        const size_t qrow = static_cast<size_t>(e0->Hs) * e0->d * e0->esz, krow = static_cast<size_t>(e0->Gs) * e0->d * e0->esz;
        const size_t vrow = static_cast<size_t>(e0->Gs) * e0->dv * e0->esz, orow = static_cast<size_t>(e0->Hs) * e0->dv * e0->esz;
        bool all = true;
        for (int32_t i = 0; i < n; ++i) all = all && batchable(engs[i], e0, layer);
        for (int32_t i = 0; i < n && all; ++i)
            for (int32_t j = 0; j < i; ++j)
                if (engs[i] == engs[j]) all = false;
        auto at = [](const void* p, size_t off) { return static_cast<const uint8_t*>(p) + off; };
        // one sequence: the single-sequence chain (programmatic K4, fused lookup)
        // is shorter than the batched stages (46 vs 73 us @128K); same ids, counters
        // and trace (tests/test_gpu_decode.py::test_decode_batch_of_one)
        if (n == 1) all = false;
        if (!all) {  // other shapes / modes / one sequence: the per-engine decode step, sequence by sequence
            for (int32_t i = 0; i < n; ++i) {
                if (!engs[i]) throw ConfigError("null engine");
                if (engs[i]->dtype == INFLLM_DTYPE_BF16)
                    engs[i]->step<bf16>(layer, at(q, i * qrow), at(k, i * krow), at(v, i * vrow),
                                        1, true, const_cast<uint8_t*>(at(out, i * orow)), st);
                else
                    engs[i]->step<float>(layer, at(q, i * qrow), at(k, i * krow), at(v, i * vrow),
                                         1, true, const_cast<uint8_t*>(at(out, i * orow)), st);
            }
            return;
        }
        for (int32_t i = 0; i < n; ++i)  // an LRU of another batch context still touching this engine
            if (engs[i]->ext_dep && (!e0->bctx || engs[i]->ext_dep != e0->bctx->lru_ev)) engs[i]->join_ext(st);
        DecodeCollector c;
        const double h1 = now_us();
        for (int32_t i = 0; i < n; ++i) {
            engs[i]->coll = &c;
            try {
                engs[i]->step<bf16>(layer, at(q, i * qrow), at(k, i * krow), at(v, i * vrow), 1, true,
                                    const_cast<uint8_t*>(at(out, i * orow)), st);
            } catch (...) {
                engs[i]->coll = nullptr;
                throw;
            }
            engs[i]->coll = nullptr;
        }
        const double h2 = now_us();
        if (static_cast<int32_t>(c.prep.size() + c.front.size()) != n || static_cast<int32_t>(c.attn.size()) != n ||
            static_cast<int32_t>(c.lru.size()) != n)
            throw StreamError("decode_batch: unexpected step shape");
        if (!e0->bctx) e0->bctx = std::make_unique<BatchCtx>();
        BatchCtx& bc = *e0->bctx;
        std::vector<uint8_t> buf;
        if (!c.front.empty() && static_cast<int32_t>(c.front.size()) != n)
            throw StreamError("decode_batch: mixed decode-front shapes");
        if (dec_front_size() != sizeof(DecFrontRec)) throw StreamError("decode_batch: front record layout");
        const size_t o_front = put(buf, c.front);
        const size_t o_prep = put(buf, c.prep), o_ev = put(buf, c.evict), o_sel = put(buf, c.select);
        const size_t o_lk = put(buf, c.lookup), o_at = put(buf, c.attn), o_lru = put(buf, c.lru);
        const int s = bc.slot;
        bc.slot = (bc.slot + 1) % BatchCtx::kSlots;
        const double h3 = now_us();
        if (bc.done[s]) ck(cudaEventSynchronize(bc.done[s]), "batch slot");  // the batch kSlots calls back
        const double h4 = now_us();
        // capacity for every record a call of n sequences can carry (fronts or preps,
        // evictions and completed units' copies of all n, ...): a growth drains the
        // device and re-allocates pinned memory (ms), so it happens once per batch size,
        // not when a call first carries completed units
        const size_t worst = static_cast<size_t>(n) * (sizeof(DecFrontRec) + sizeof(PrepParams) + sizeof(EvictParams) +
                                                       sizeof(SelectParams) + sizeof(LookupParams) + sizeof(AttnParams) +
                                                       sizeof(LruParams)) + 8 * 256;
        if (buf.size() > bc.cap || worst > bc.cap) {
            ck(cudaDeviceSynchronize(), "batch table growth");
            for (int t = 0; t < BatchCtx::kSlots; ++t) {
                if (bc.host[t]) cudaFreeHost(bc.host[t]);
                if (bc.dev[t]) cudaFree(bc.dev[t]);
                bc.host[t] = bc.dev[t] = nullptr;
            }
            bc.cap = std::max(buf.size(), worst);
            for (int t = 0; t < BatchCtx::kSlots; ++t) {
                ck(cudaHostAlloc(&bc.host[t], bc.cap, cudaHostAllocDefault), "cudaHostAlloc");
                ck(cudaMalloc(&bc.dev[t], bc.cap), "cudaMalloc");
                if (!bc.done[t]) ck(cudaEventCreateWithFlags(&bc.done[t], cudaEventDisableTiming), "event");
            }
        }
        std::memcpy(bc.host[s], buf.data(), buf.size());
        ck(cudaMemcpyAsync(bc.dev[s], bc.host[s], buf.size(), cudaMemcpyHostToDevice, st), "batch tables H2D");
        uint8_t* dt = static_cast<uint8_t*>(bc.dev[s]);
        // K4 batch scratch
        const int rep = e0->rep, G = e0->Gs;
        const int km = static_cast<int>(std::max<int64_t>(e0->cfg.n_lookup, 1));
        if (bc.part_B < n) {
            ck(cudaStreamSynchronize(st), "scratch growth");
            bc.part.alloc(dec_part_floats(n, G, rep) * sizeof(float), st, false);
            bc.mass.alloc(static_cast<size_t>(n) * e0->Hs * km * kDecWarps * 2 * sizeof(float), st);
            bc.cnt.alloc(static_cast<size_t>(n) * G * sizeof(unsigned), st);
            bc.part_B = n;
        }
        int64_t ev_max = 0, sel_max = 0, lk_max = 0, tiles_max = 0;
        for (auto& ep : c.evict) ev_max = std::max<int64_t>(ev_max, ep.n_init + ep.n_evict);
        for (auto& sp : c.select) sel_max = std::max<int64_t>(sel_max, sp.n_units);
        int64_t lk_units = 0, lk_str = 0;  // all sequences' units | per-sequence scan blocks << 32
        for (auto& lp : c.lookup) {
            lk_units += lp.U;
            lk_str = std::max<int64_t>(lk_str, decode_batch_lookup_blocks(lp.U) >> 32);
        }
        lk_max = std::min<int64_t>(lk_units, 0xffffffff) | (lk_str << 32);
        for (auto& ap : c.attn) tiles_max = std::max<int64_t>(tiles_max, dec_max_tiles(ap));
        // batch chain (every sequence's scan forms its query sums from q): the scan
        // first, the fronts as its programmatic dependent (they end after it), then
        // completed units' copies and the top-k; else front, select, scan + top-k
        // (measured: B = 2 at 128K 63.7 -> 55.9 us per step; from B = 4 on the fronts
        // compete with the scan for SMs and the order makes no difference)
        bool bchain = n <= 4 && !c.front.empty() && c.evict.empty() && static_cast<int32_t>(c.lookup.size()) == n;
        for (auto& lp : c.lookup) bchain = bchain && lp.qtok != nullptr;
        if (bchain) {
            if (bc.ring_set[bc.calls % BatchCtx::kRing])  // the LRU of the call three back
                ck(cudaStreamWaitEvent(st, bc.lru_ring[bc.calls % BatchCtx::kRing], 0), "wait");
            launch_decode_batch_stage(5, dt + o_lk, n, lk_max, st);
            launch_dec_front_batch(dt + o_front, n, G, st, 1);
            if (!c.select.empty())
                launch_decode_batch_stage(2, dt + o_sel, static_cast<int>(c.select.size()),
                                          sel_max | (static_cast<int64_t>(G) << 32), st);
            launch_decode_batch_stage(7, dt + o_lk, n, lk_max, st);
        } else {
            if (!c.front.empty())
                launch_dec_front_batch(dt + o_front, n, G, st);
            else
                launch_decode_batch_stage(0, dt + o_prep, n, G, st);
            if (!c.evict.empty())
                launch_decode_batch_stage(1, dt + o_ev, static_cast<int>(c.evict.size()),
                                          ev_max | (static_cast<int64_t>(G) << 32), st);
            if (!c.select.empty())
                launch_decode_batch_stage(2, dt + o_sel, static_cast<int>(c.select.size()),
                                          sel_max | (static_cast<int64_t>(G) << 32), st);
            if (bc.ring_set[bc.calls % BatchCtx::kRing])  // the LRU of the call three back
                ck(cudaStreamWaitEvent(st, bc.lru_ring[bc.calls % BatchCtx::kRing], 0), "wait");
            if (!c.lookup.empty())
                launch_decode_batch_stage(3, dt + o_lk, static_cast<int>(c.lookup.size()), lk_max, st);
        }
        launch_attn_dec_batch(reinterpret_cast<const AttnParams*>(dt + o_at), n, G, tiles_max,
                              DecScratch{bc.part.as<float>(), bc.mass.as<float>(), bc.cnt.as<unsigned>(), km,
                                         // K4's splits without retrieved units start beside the top-k: past
                                         // the batch chain the fronts finished before the scan started, in
                                         // it the top-k releases K4 only after its wait (fronts complete)
                                         1,
                                         e0->dec_merge_opt ? 1 : 0},
                              st);
        cudaStream_t lst = st;
        {
            if (!bc.lru_st) {
                ck(cudaStreamCreateWithFlags(&bc.lru_st, cudaStreamNonBlocking), "stream");
                ck(cudaEventCreateWithFlags(&bc.ev_k4, cudaEventDisableTiming), "event");
                bc.lru_ev = std::make_shared<SharedEvent>();
                ck(cudaEventCreateWithFlags(&bc.lru_ev->ev, cudaEventDisableTiming), "event");
            }
            ck(cudaEventRecord(bc.ev_k4, st), "record");
            ck(cudaStreamWaitEvent(bc.lru_st, bc.ev_k4, 0), "wait");
            lst = bc.lru_st;
        }
        launch_decode_batch_stage(4, dt + o_lru, n, 0, lst);
        ck(cudaGetLastError(), "decode_batch launch");
        if (lst != st) {
            ck(cudaEventRecord(bc.lru_ev->ev, lst), "record");
            bc.lru_pending = true;
            for (int32_t i = 0; i < n; ++i) engs[i]->ext_dep = bc.lru_ev;
            const int r = static_cast<int>(bc.calls % BatchCtx::kRing);
            if (!bc.lru_ring[r]) ck(cudaEventCreateWithFlags(&bc.lru_ring[r], cudaEventDisableTiming), "event");
            ck(cudaEventRecord(bc.lru_ring[r], lst), "record");
            bc.ring_set[r] = true;
        }
        ++bc.calls;
        ck(cudaEventRecord(bc.done[s], lst), "record");  // lst follows everything of this call
        const double h5 = now_us();
        const double parts[6] = {h1 - h0,   // argument checks
                                 h2 - h1,   // per-sequence step() in collect mode
                                 h3 - h2,   // tables
                                 h4 - h3,   // wait for the batch two calls back
                                 h5 - h4,   // copies and launches
                                 1.0};
        for (int i = 0; i < 6; ++i) g_dbh[i].fetch_add(parts[i], std::memory_order_relaxed);
    });
}

int infllm_encode_stream(infllm_engine_t e, int32_t layer, const void* q, const void* k, const void* v,
                         int64_t n_tokens, void* out, void* stream) {
    return guard([&] {
        if (!e) throw ConfigError("null engine");
        auto st = static_cast<cudaStream_t>(stream);
        if (e->dtype == INFLLM_DTYPE_BF16)
            e->encode_stream<bf16>(layer, q, k, v, n_tokens, out, st, false);
        else
            e->encode_stream<float>(layer, q, k, v, n_tokens, out, st, false);
    });
}

int infllm_encode_stream_host(infllm_engine_t e, int32_t layer, const void* host_q, const void* host_k,
                              const void* host_v, int64_t n_tokens, void* host_out, void* stream) {
    return guard([&] {
        if (!e) throw ConfigError("null engine");
        auto st = static_cast<cudaStream_t>(stream);
        if (e->dtype == INFLLM_DTYPE_BF16)
            e->encode_stream<bf16>(layer, host_q, host_k, host_v, n_tokens, host_out, st, true);
        else
            e->encode_stream<float>(layer, host_q, host_k, host_v, n_tokens, host_out, st, true);
    });
}

int infllm_finish(infllm_engine_t e, void* stream) {
    return guard([&] {
        auto st = static_cast<cudaStream_t>(stream);
        e->join_ext(st);
        if (e->dtype == INFLLM_DTYPE_BF16)
            e->finish<bf16>(st);
        else
            e->finish<float>(st);
    });
}

int infllm_retrieved_ids(infllm_engine_t e, int32_t layer, int64_t* host_ids, int64_t cap, int64_t* n_out) {
    return guard([&] {
        auto& L = e->layers.at(static_cast<size_t>(layer));
        ck(cudaDeviceSynchronize(), "sync");
        *n_out = L.last_n_sel;
        const int64_t n = std::min(cap, L.last_n_sel);
        const int64_t* src = L.sel.as<int64_t>() + L.last_b * std::max<int64_t>(e->cfg.n_lookup, 1);
        if (n > 0) ck(cudaMemcpy(host_ids, src, n * sizeof(int64_t), cudaMemcpyDeviceToHost), "D2H");
    });
}

int infllm_get_layer_metrics(infllm_engine_t e, int32_t layer, infllm_layer_metrics* m) {
    return guard([&] {
        auto& L = e->layers.at(static_cast<size_t>(layer));
        ck(cudaDeviceSynchronize(), "sync");
        LruState s{};
        ck(cudaMemcpy(&s, L.lru.p, sizeof(s), cudaMemcpyDeviceToHost), "D2H");
        m->units = L.n_units;
        m->hot_units = s.hot_count;
        m->peak_hot_units = s.peak_hot_units;
        m->peak_hot_bytes = s.peak_hot_bytes;
        m->hits = s.hits;
        m->misses = s.misses;
        m->loads = s.loads;
        m->evictions = s.evictions;
        m->requested = s.requested;
    });
}

int infllm_unit_info(infllm_engine_t e, int32_t layer, int64_t id, int64_t* start_abs, int64_t* size,
                     int64_t* host_repr_abs, int64_t* n_repr_out) {
    return guard([&] {
        auto& L = e->layers.at(static_cast<size_t>(layer));
        if (id < 0 || id >= L.n_units) throw StreamError("unit id out of range");
        ck(cudaDeviceSynchronize(), "sync");
        std::vector<int32_t> idx(static_cast<size_t>(e->cfg.n_repr));
        ck(cudaMemcpy(idx.data(), L.repr_idx.as<int32_t>() + id * e->cfg.n_repr, idx.size() * sizeof(int32_t),
                      cudaMemcpyDeviceToHost),
           "D2H");
        *start_abs = L.unit_start[static_cast<size_t>(id)];
        *size = L.unit_len[static_cast<size_t>(id)];
        int64_t n = 0;
        for (auto x : idx)
            if (x >= 0) host_repr_abs[n++] = *start_abs + x;
        *n_repr_out = n;
    });
}

int infllm_stream_state(infllm_engine_t e, int32_t layer, int64_t* fed, int64_t* steps, int64_t* init_len,
                        int64_t* local_len, int64_t* pending) {
    return guard([&] {
        auto& L = e->layers.at(static_cast<size_t>(layer));
        *fed = L.n_fed;
        *steps = L.step;
        *init_len = L.init_len;
        *local_len = L.n_fed - L.local_start;
        *pending = L.pend_count;
    });
}

int infllm_unit_freq(infllm_engine_t e, int32_t layer, double* host_freq, int32_t* host_hot, int64_t n) {
    return guard([&] {
        auto& L = e->layers.at(static_cast<size_t>(layer));
        n = std::min(n, L.n_units);
        ck(cudaDeviceSynchronize(), "sync");
        if (n <= 0) return;
        ck(cudaMemcpy(host_freq, L.freq.p, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
        std::vector<int8_t> h(static_cast<size_t>(n));
        ck(cudaMemcpy(h.data(), L.hot.p, n, cudaMemcpyDeviceToHost), "D2H");
        for (int64_t i = 0; i < n; ++i) host_hot[i] = h[static_cast<size_t>(i)];
    });
}

int infllm_trace(infllm_engine_t e, int32_t layer, int64_t* host_step, int64_t* host_unit, int32_t* host_hit,
                 int64_t cap, int64_t* n_out) {
    return guard([&] {
        auto& L = e->layers.at(static_cast<size_t>(layer));
        ck(cudaDeviceSynchronize(), "sync");
        *n_out = L.trace_count;
        const int64_t n = std::min(cap, L.trace_count);
        if (n <= 0) return;
        std::vector<int64_t> t(static_cast<size_t>(3 * n));
        ck(cudaMemcpy(t.data(), L.trace.p, t.size() * sizeof(int64_t), cudaMemcpyDeviceToHost), "D2H");
        for (int64_t i = 0; i < n; ++i) {
            host_step[i] = t[static_cast<size_t>(3 * i)];
            host_unit[i] = t[static_cast<size_t>(3 * i + 1)];
            host_hit[i] = static_cast<int32_t>(t[static_cast<size_t>(3 * i + 2)]);
        }
    });
}

int infllm_tier_stats(infllm_engine_t e, int32_t layer, int64_t* out4) {
    return guard([&] {
        if (!e || !out4) throw ConfigError("null argument");
        if (layer < 0 || layer >= e->n_layers) throw StreamError("layer out of range");
        const auto& L = e->layers[static_cast<size_t>(layer)];
        out4[0] = out4[1] = out4[2] = 0;
        out4[3] = e->tier_slots;
        if (!L.tier_stats.p) return;
        ck(cudaDeviceSynchronize(), "sync");
        int64_t st[4];
        ck(cudaMemcpy(st, L.tier_stats.p, sizeof(st), cudaMemcpyDeviceToHost), "D2H");
        for (int i = 0; i < 3; ++i) out4[i] = st[i];
        if (st[3] != 0) throw StreamError("host tier: slot assignment failed");
    });
}

int infllm_kernel_launches(infllm_engine_t e, int64_t* n_out) {
    *n_out = e->launches;
    return INFLLM_OK;
}

int infllm_profile_begin(infllm_engine_t e, int32_t enable) {
    return guard([&] {
        for (auto& evs : e->ev) {
            for (auto& p : evs) {
                e->ev_pool.push_back(p.first);
                e->ev_pool.push_back(p.second);
            }
            evs.clear();
        }
        for (auto& g : e->graphs) g.replays_in_window = 0;
        e->prof = enable != 0;
    });
}

namespace {
// device time (ms) during which a phase had launches in flight: the length of
// the union of its [begin, end] event intervals. Launches of one phase on one
// stream never overlap (union = sum); chunk-step attention alternates between
// two streams, and consecutive launches overlap while one's CTAs drain and the
// next one's start, which a plain sum would count twice.
double union_ms(const std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v) {
    if (v.empty()) return 0;
    std::vector<std::pair<float, float>> iv;
    iv.reserve(v.size());
    for (auto& p : v) {
        float a = 0, b = 0;
        ck(cudaEventElapsedTime(&a, v[0].first, p.first), "elapsed");
        ck(cudaEventElapsedTime(&b, v[0].first, p.second), "elapsed");
        iv.emplace_back(a, b);
    }
    std::sort(iv.begin(), iv.end());
    double tot = 0, lo = iv[0].first, hi = iv[0].second;
    for (size_t i = 1; i < iv.size(); ++i) {
        if (iv[i].first > hi) {
            tot += hi - lo;
            lo = iv[i].first;
            hi = iv[i].second;
        } else {
            hi = std::max(hi, static_cast<double>(iv[i].second));
        }
    }
    return tot + (hi - lo);
}
// device time of each phase's launches in the profile window (ms) and launch counts
void phase_sums(infllm_engine* e, double* ms, int64_t* n) {
    ck(cudaDeviceSynchronize(), "sync");
    for (int ph = 0; ph < kPhases; ++ph) {
        n[ph] = static_cast<int64_t>(e->ev[ph].size());
        ms[ph] = union_ms(e->ev[ph]);
        // graph replays: event nodes hold the timings of the latest replay
        for (auto& g : e->graphs) {
            if (g.replays_in_window == 0) continue;
            ms[ph] += union_ms(g.ev[ph]) * g.replays_in_window;
            n[ph] += static_cast<int64_t>(g.ev[ph].size()) * g.replays_in_window;
        }
    }
}
}  // namespace

int infllm_profile_read(infllm_engine_t e, double* attn_ms, int64_t* attn_n, double* lookup_ms, int64_t* lookup_n) {
    return guard([&] {
        double ms[kPhases];
        int64_t n[kPhases];
        phase_sums(e, ms, n);
        *attn_ms = ms[kPhAttend];
        *attn_n = n[kPhAttend];
        *lookup_ms = ms[kPhLookup];
        *lookup_n = n[kPhLookup];
    });
}

int infllm_phase_timings(infllm_engine_t e, double* ms4, int64_t* launches4) {
    return guard([&] {
        if (!e || !ms4) throw ConfigError("null argument");
        int64_t n[kPhases];
        phase_sums(e, ms4, n);
        if (launches4)
            for (int ph = 0; ph < kPhases; ++ph) launches4[ph] = n[ph];
    });
}

int infllm_invariants(infllm_engine_t e, uint64_t* checks, uint64_t* violations) {
    return guard([&] {
        if (!e || !checks || !violations) throw ConfigError("null argument");
        unsigned long long dev = 0;
        ck(cudaDeviceSynchronize(), "sync");
        ck(cudaMemcpy(&dev, e->inv_dev.p, sizeof(dev), cudaMemcpyDeviceToHost), "D2H");
        *checks = e->inv_checks;
        *violations = e->inv_conservation_bad + dev;
    });
}

int infllm_select_representatives(const float* scores, const int64_t* lens, int64_t n_units, int64_t unit_len,
                                  int64_t r_k, int64_t* idx, void* stream) {
    return guard([&] {
        if (r_k < 1 || r_k > 32) throw ConfigError("r_k must be in [1, 32]");
        launch_select_standalone(scores, lens, n_units, unit_len, r_k, idx, static_cast<cudaStream_t>(stream));
        ck(cudaGetLastError(), "select");
    });
}

int infllm_lookup(const double* qsum, const void* repr, int32_t dtype, int64_t n_units, int64_t r_k,
                  int32_t n_kv_heads, int32_t head_dim, int64_t k_m, double* rel, int64_t* ids, void* stream) {
    return guard([&] {
        auto st = static_cast<cudaStream_t>(stream);
        if (n_units <= 0) return;
        const int64_t k = std::min(k_m, n_units);
        const int64_t nc = topk_multi_scratch(n_units, std::max<int64_t>(k, 1));
        // grow-only scratch shared by this thread's calls (a per-call allocation would
        // dominate small lookups); a call on any stream first waits for the previous
        // call's kernels, so neither the reuse nor a growth free can race with them
        static thread_local DBuf cand, cnt;
        static thread_local cudaEvent_t last = nullptr;
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        ck(cudaStreamIsCapturing(st, &cs), "capture status");
        const bool capturing_now = cs != cudaStreamCaptureStatusNone;  // a graph orders its own nodes
        if (!last)
            ck(cudaEventCreateWithFlags(&last, cudaEventDisableTiming), "event");
        else if (!capturing_now)
            ck(cudaStreamWaitEvent(st, last, 0), "wait");
        cand.grow(static_cast<size_t>(nc) * 16, st);
        LookupParams lp{};
        lp.qsum = qsum;
        lp.repr = repr;
        lp.rel = rel;
        lp.U = n_units;
        lp.G = n_kv_heads;
        lp.Gtot = n_kv_heads;
        lp.g0 = 0;
        lp.r_k = static_cast<int>(r_k);
        lp.d = head_dim;
        lp.n_sel = k;
        lp.sel = ids;
        cnt.grow(64, st);  // block counter of the folded merge (zeroed once, re-zeroed by the kernel)
        lp.done = cnt.as<unsigned int>();
        lp.fused = 1;
        lp.cand_v = cand.as<double>();
        lp.cand_i = reinterpret_cast<int64_t*>(cand.as<double>() + nc);
        if (lookup_topk_supported(lp, dtype == INFLLM_DTYPE_BF16))
            launch_lookup_topk_fast(lp, lookup_topk_blocks(n_units, 8), st);
        else
            launch_lookup_topk(lp, dtype == INFLLM_DTYPE_BF16, cand.as<double>(),
                               reinterpret_cast<int64_t*>(cand.as<double>() + nc), st);
        ck(cudaGetLastError(), "lookup");
        if (!capturing_now) ck(cudaEventRecord(last, st), "record");
    });
}

// Debug: steady-state duration of one kernel family, re-launched `iters`
// times (in a CUDA graph) with the parameters of the engine's last step.
// which: 0 prep, 1 lookup (+ exact top-k) as a one-token step launches it,
// 2 attention, 3 evict (+ fused select), 4 LRU, 5 relevance scan only, 6 top-k
// only, 7/8 empty kernels, 9/10 fp64/fp32 FMA probes, 11 lookup with the
// chunk-step (in-pipeline) grid. Mutates engine state: only for performance
// investigation.
int infllm_debug_kernel_bench(infllm_engine_t e, int32_t which, int32_t iters, double* us_per_launch) {
    return guard([&] {
        cudaStream_t st;
        ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
        ck(cudaDeviceSynchronize(), "sync");
        auto launch = [&]() {
            switch (which) {
                case 0:
                    if (e->last_bf16) launch_prep<bf16>(e->last_pp, st); else launch_prep<float>(e->last_pp, st);
                    break;
                case 1: {  // the last step's lookup as a one-token step runs it (whole GPU):
                           // k_lookup_reg + fused radix top-k up to 2048 units, else the one-launch scan
                    LookupParams lp = e->last_lkp;
                    if (lp.G == lp.Gtot && lp.U <= 256 * 8) {
                        lp.fused = 1;
                        launch_lookup(lp, e->last_bf16, st);
                    } else if (lp.cand_v && lookup_topk_supported(lp, e->last_bf16)) {
                        launch_lookup_topk_fast(lp, lookup_topk_blocks(lp.U, e->lookup_upb_decode), st);
                    } else {
                        launch_lookup(lp, e->last_bf16, st);
                    }
                    break;
                }
                case 11:  // the chunk-step lookup with its in-pipeline grid (few fat blocks)
                    if (e->last_lkp.cand_v && lookup_topk_supported(e->last_lkp, e->last_bf16))
                        launch_lookup_topk_fast(e->last_lkp, lookup_topk_blocks(e->last_lkp.U, e->lookup_upb), st);
                    else
                        launch_lookup(e->last_lkp, e->last_bf16, st);
                    break;
                case 2:
                    if (e->last_bf16 && e->tc_eligible(e->last_ap.lx)) launch_attn_tc(e->last_ap, st);
                    else if (e->last_bf16) launch_attn_simt<bf16>(e->last_ap, st);
                    else launch_attn_simt<float>(e->last_ap, st);
                    break;
                case 3:
                    if (e->last_bf16) launch_evict<bf16>(e->last_ep, st); else launch_evict<float>(e->last_ep, st);
                    break;
                case 4: launch_lru(e->last_lp, st); break;
                case 5: {  // relevance scan only
                    LookupParams lp = e->last_lkp;
                    lp.fused = 0;
                    lp.part = e->layers[0].lookup_part.as<double>();
                    launch_lookup(lp, e->last_bf16, st);
                    break;
                }
                case 6: {  // top-k only (1024-thread radix select over rel)
                    TopkParams tp{};
                    tp.part = e->layers[0].lookup_part.as<double>();
                    tp.rel = e->layers[0].rel.as<double>();
                    tp.sel = e->layers[0].sel.as<int64_t>();
                    tp.U = e->last_lkp.U;
                    tp.n_sel = e->last_lkp.n_sel;
                    tp.Gtot = e->Gt;
                    launch_topk(tp, st);
                    break;
                }
                case 7: k_empty<<<124, 256, 0, st>>>(); break;
                case 8: k_empty<<<1, 32, 0, st>>>(); break;
                case 9: k_probe_f64<<<148 * 4, 256, 0, st>>>(nullptr, 1000); break;   // 1.21e9 DFMA
                case 10: k_probe_f32<<<148 * 4, 256, 0, st>>>(nullptr, 1000); break;  // 1.21e9 FFMA
                default: throw ConfigError("unknown kernel id");
            }
        };
        launch();  // warm
        ck(cudaStreamSynchronize(st), "warm");
        cudaGraph_t g;
        ck(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "capture");
        for (int i = 0; i < iters; ++i) launch();
        ck(cudaStreamEndCapture(st, &g), "capture");
        cudaGraphExec_t x;
        ck(cudaGraphInstantiate(&x, g, 0), "instantiate");
        ck(cudaGraphLaunch(x, st), "launch");
        ck(cudaStreamSynchronize(st), "sync");
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, st);
        ck(cudaGraphLaunch(x, st), "launch");
        cudaEventRecord(b, st);
        ck(cudaStreamSynchronize(st), "sync");
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        *us_per_launch = 1000.0 * ms / iters;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaGraphExecDestroy(x);
        cudaGraphDestroy(g);
        cudaStreamDestroy(st);
    });
}

int infllm_debug_timestamps(unsigned long long* out64) {
    return guard([&] {
        ck(cudaDeviceSynchronize(), "sync");
        debug_read_timestamps(out64);
    });
}

// ---- stand-alone reference operators (standalone.cu) ----
namespace {
RopeFreqs make_freqs(int d, int64_t local_size) {  // rotary.hpp:25-30 (RotaryTable::make)
    RopeFreqs f{};
    for (int a = 0; a < d / 2; ++a) {
        f.f[a] = std::pow(10000.0, -2.0 * a / d);
        const double ang = static_cast<double>(local_size) * f.f[a];
        f.cL[a] = static_cast<float>(std::cos(ang));
        f.sL[a] = static_cast<float>(std::sin(ang));
    }
    return f;
}
}  // namespace

struct infllm_store {
    int64_t cap = 0;
    double decay = 0.0;
    int H = 1, G = 1, d = 0, r_k = 1, dtype = INFLLM_DTYPE_F32;
    size_t esz = 4;
    int64_t bpt = 0;
    int64_t n_units = 0, unit_cap = 0, trace_cap = 0, trace_count = 0, step = 0;
    DBuf repr, freq, hot, hot_list, unit_tokens, lru, trace, err, qsum, rel, ids, cand, done, up_ids, up_mass;
    cudaStream_t st = nullptr;
    StoreDev dev() {
        return StoreDev{lru.as<LruState>(), trace.as<int64_t>(), freq.as<double>(), hot.as<int8_t>(),
                        hot_list.as<int64_t>(), unit_tokens.as<int32_t>(), err.as<int>(), n_units, cap, bpt, decay};
    }
    void ensure_units(int64_t n) {
        if (n <= unit_cap) return;
        const int64_t c = std::max<int64_t>({n, 2 * unit_cap, 64});
        repr.grow(static_cast<size_t>(c) * G * r_k * d * esz, st);
        freq.grow(c * sizeof(double), st);
        hot.grow(c * sizeof(int8_t), st);
        hot_list.grow(c * sizeof(int64_t), st);
        unit_tokens.grow(c * sizeof(int32_t), st);
        rel.grow(c * sizeof(double), st);
        cand.grow(static_cast<size_t>(topk_multi_scratch(c, 128)) * 16, st);
        unit_cap = c;
    }
    void check_err() {
        int e = 0;
        ck(cudaMemcpyAsync(&e, err.p, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "store");
        if (!e) return;
        ck(cudaMemsetAsync(err.p, 0, sizeof(int), st), "memset");
        if (e == 1) throw StreamError("update_frequency: mass for a unit that is not hot");
        throw StreamError("TieredStore: hot tier over capacity at step end");
    }
};

struct infllm_score_acc {
    int64_t L = 0, lo = 0, hi = 0, next_q = 0, ring0 = 0, cap = 0;
    int H = 1, G = 1, d = 0, dtype = INFLLM_DTYPE_F32;
    DBuf sums, out;
};

extern "C" {

int infllm_attend(const infllm_model_shape* shape, int32_t dtype, int32_t position_mode, int64_t local_size,
                  const infllm_segment* window, int32_t n_segments, const void* q, const void* k, const void* v,
                  int64_t l_x, int64_t start_abs, void* out, double* seg_mass, float* weights, void* stream) {
    return guard([&] {
        if (!shape) throw ConfigError("null shape");
        validate_shape(*shape);
        if (dtype != INFLLM_DTYPE_F32 && dtype != INFLLM_DTYPE_BF16) throw ConfigError("dtype must be f32 or bf16");
        if (position_mode != INFLLM_POSITION_CLAMPED && position_mode != INFLLM_POSITION_ABSOLUTE)
            throw ConfigError("position_mode: unknown value");
        if (l_x < 1) throw StreamError("attend: empty batch");  // attention.hpp:123
        if (n_segments < 0 || (n_segments > 0 && !window)) throw ConfigError("attend: bad window");
        const int H = shape->n_heads, G = shape->n_kv_heads > 0 ? shape->n_kv_heads : H, d = shape->head_dim;
        const int dv = shape->value_dim > 0 ? shape->value_dim : d;
        if (d > 256) throw ConfigError("head_dim <= 256 supported");
        auto st = static_cast<cudaStream_t>(stream);
        const size_t esz = dtype == INFLLM_DTYPE_BF16 ? 2 : 4;
        std::vector<uint8_t> segs(std::max<size_t>(1, static_cast<size_t>(n_segments)) * attend_seg_bytes());
        int64_t n_ctx = 0;
        for (int32_t i = 0; i < n_segments; ++i) {
            const infllm_segment& sg = window[i];
            if (sg.kind < INFLLM_SEG_INITIAL || sg.kind > INFLLM_SEG_LOCAL) throw ConfigError("attend: segment kind");
            if (sg.n_tokens < 0 || (sg.n_tokens > 0 && (!sg.keys || !sg.values)))
                throw StreamError("attend: segment without keys / values");
            attend_pack_seg(segs.data(), i, sg.keys, sg.values, sg.start_abs, sg.n_tokens, n_ctx, sg.kind);
            n_ctx += sg.n_tokens;
        }
        const int64_t n_all = n_ctx + l_x;
        void *d_segs = nullptr, *scratch = nullptr;
        const size_t b_scores = weights ? 0 : static_cast<size_t>(H) * l_x * n_all * sizeof(float);
        const size_t b_part = static_cast<size_t>(H) * l_x * std::max(1, n_segments) * sizeof(double);
        const size_t b_qrot = 2 * static_cast<size_t>(H) * l_x * d * sizeof(float);
        const size_t b_krot = static_cast<size_t>(n_all) * G * d * sizeof(float);
        auto al = [](size_t x) { return (x + 255) / 256 * 256; };
        ck(cudaMallocAsync(&d_segs, segs.size(), st), "cudaMallocAsync");
        ck(cudaMallocAsync(&scratch, al(b_scores) + al(b_part) + al(b_qrot) + al(b_krot), st), "cudaMallocAsync");
        ck(cudaMemcpyAsync(d_segs, segs.data(), segs.size(), cudaMemcpyHostToDevice, st), "H2D");
        uint8_t* p8 = static_cast<uint8_t*>(scratch);
        AttendLaunch L{};
        L.dev_segs = d_segs;
        L.n_seg = n_segments;
        L.q = q;
        L.k = k;
        L.v = v;
        L.out = out;
        L.scores = weights ? weights : reinterpret_cast<float*>(p8);
        L.mass_part = reinterpret_cast<double*>(p8 + al(b_scores));
        L.mass = seg_mass;
        L.qrot = reinterpret_cast<float*>(p8 + al(b_scores) + al(b_part));
        L.krot = reinterpret_cast<float*>(p8 + al(b_scores) + al(b_part) + al(b_qrot));
        L.lx = l_x;
        L.n_ctx = n_ctx;
        L.start_abs = start_abs;
        L.local_size = local_size;
        L.H = H;
        L.G = G;
        L.d = d;
        L.dv = dv;
        L.absolute = position_mode == INFLLM_POSITION_ABSOLUTE;
        L.bf16 = dtype == INFLLM_DTYPE_BF16;
        L.freqs = make_freqs(d, local_size);
        (void)esz;
        attend_run(L, st);
        ck(cudaGetLastError(), "attend");
        ck(cudaFreeAsync(scratch, st), "cudaFreeAsync");
        ck(cudaFreeAsync(d_segs, st), "cudaFreeAsync");
        ck(cudaStreamSynchronize(st), "attend");  // the host segment table is freed on return
    });
}

int infllm_store_create(int64_t hot_capacity, double decay, int32_t n_heads, int32_t n_kv_heads, int32_t head_dim,
                        int64_t n_repr, int32_t dtype, int64_t bytes_per_token, infllm_store_t* out) {
    return guard([&] {
        if (!out) throw ConfigError("null argument");
        if (hot_capacity < 0) throw ConfigError("hot_capacity must be >= 0");
        if (decay < 0.0 || decay > 1.0) throw ConfigError("decay must lie in [0, 1]");
        if (n_heads < 1 || n_kv_heads < 1 || n_heads % n_kv_heads || head_dim < 1 || n_repr < 1 || n_repr > 32)
            throw ConfigError("TieredStore: bad shape");
        if (dtype != INFLLM_DTYPE_F32 && dtype != INFLLM_DTYPE_BF16) throw ConfigError("dtype must be f32 or bf16");
        auto s = std::make_unique<infllm_store>();
        s->cap = hot_capacity;
        s->decay = decay;
        s->H = n_heads;
        s->G = n_kv_heads;
        s->d = head_dim;
        s->r_k = static_cast<int>(n_repr);
        s->dtype = dtype;
        s->esz = dtype == INFLLM_DTYPE_BF16 ? 2 : 4;
        s->bpt = bytes_per_token;
        ck(cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking), "stream");
        s->lru.alloc(sizeof(LruState), s->st);
        s->err.alloc(sizeof(int), s->st);
        s->qsum.alloc(static_cast<size_t>(n_kv_heads) * head_dim * sizeof(double), s->st);
        s->ids.alloc(128 * sizeof(int64_t), s->st);
        s->done.alloc(64, s->st);
        s->up_ids.alloc(1024 * sizeof(int64_t), s->st);
        s->up_mass.alloc(1024 * sizeof(double), s->st);
        s->ensure_units(64);
        ck(cudaStreamSynchronize(s->st), "store create");
        *out = s.release();
    });
}

int infllm_store_destroy(infllm_store_t s) {
    return guard([&] {
        if (!s) return;
        cudaStreamSynchronize(s->st);
        for (auto* b : {&s->repr, &s->freq, &s->hot, &s->hot_list, &s->unit_tokens, &s->lru, &s->trace, &s->err, &s->qsum,
                        &s->rel, &s->ids, &s->cand, &s->done, &s->up_ids, &s->up_mass})
            b->release(s->st);
        cudaStreamSynchronize(s->st);
        cudaStreamDestroy(s->st);
        delete s;
    });
}

int infllm_store_add_unit(infllm_store_t s, const void* repr_keys, int64_t n, int64_t unit_tokens, int64_t* unit_id) {
    return guard([&] {
        if (!s) throw ConfigError("null store");
        if (n < 1 || n > s->r_k || !repr_keys) throw StreamError("add_unit: 1..n_repr representative keys required");
        s->ensure_units(s->n_units + 1);
        const int64_t u = s->n_units;
        store_put_repr(repr_keys, s->repr.p, u, static_cast<int>(n), s->r_k, s->G, s->d, static_cast<int>(s->esz), s->st);
        const int32_t tok = static_cast<int32_t>(unit_tokens);
        ck(cudaMemcpyAsync(s->unit_tokens.as<int32_t>() + u, &tok, sizeof(tok), cudaMemcpyHostToDevice, s->st), "H2D");
        ck(cudaStreamSynchronize(s->st), "add_unit");
        s->n_units = u + 1;  // new units start cold (memory.hpp:199)
        if (unit_id) *unit_id = u;
    });
}

int infllm_store_begin_step(infllm_store_t s, int64_t step) {
    if (!s) return INFLLM_ERR_ARG;
    s->step = step;
    return INFLLM_OK;
}

int infllm_store_lookup(infllm_store_t s, const void* q, int64_t l_x, int64_t k_m, int64_t* host_ids, int64_t* n_ids,
                        double* rel) {
    return guard([&] {
        if (!s) throw ConfigError("null store");
        if (k_m > 128) throw ConfigError("k_m <= 128 supported");
        const int64_t take = std::min<int64_t>(k_m, s->n_units);  // memory.hpp:240
        if (n_ids) *n_ids = std::max<int64_t>(take, 0);
        if (take <= 0) return;
        if (s->trace_count + take > s->trace_cap) {
            const int64_t c = std::max<int64_t>({s->trace_count + take, 2 * s->trace_cap, 1024});
            s->trace.grow(static_cast<size_t>(c) * 3 * sizeof(int64_t), s->st);
            s->trace_cap = c;
        }
        store_qsum(q, l_x, s->H, s->G, s->d, s->dtype == INFLLM_DTYPE_BF16, s->qsum.as<double>(), s->st);
        LookupParams lp{};
        lp.qsum = s->qsum.as<double>();
        lp.repr = s->repr.p;
        lp.rel = rel ? rel : s->rel.as<double>();
        lp.U = s->n_units;
        lp.G = s->G;
        lp.Gtot = s->G;
        lp.r_k = s->r_k;
        lp.d = s->d;
        lp.n_sel = take;
        lp.sel = s->ids.as<int64_t>();
        lp.done = s->done.as<unsigned int>();
        const int64_t nc = topk_multi_scratch(s->unit_cap, 128);
        lp.fused = 1;
        lp.cand_v = s->cand.as<double>();
        lp.cand_i = reinterpret_cast<int64_t*>(s->cand.as<double>() + nc);
        const bool bf = s->dtype == INFLLM_DTYPE_BF16;
        if (lookup_topk_supported(lp, bf))
            launch_lookup_topk_fast(lp, lookup_topk_blocks(s->n_units, 8), s->st);
        else
            launch_lookup_topk(lp, bf, lp.cand_v, lp.cand_i, s->st);
        store_book(s->dev(), s->ids.as<int64_t>(), take, s->step, s->st);
        s->trace_count += take;
        ck(cudaGetLastError(), "store lookup");
        if (host_ids)
            ck(cudaMemcpyAsync(host_ids, s->ids.p, take * sizeof(int64_t), cudaMemcpyDeviceToHost, s->st), "D2H");
        ck(cudaStreamSynchronize(s->st), "store lookup");
    });
}

int infllm_store_update_frequency(infllm_store_t s, const int64_t* host_ids, const double* host_mass, int64_t n) {
    return guard([&] {
        if (!s) throw ConfigError("null store");
        if (n < 0 || (n > 0 && (!host_ids || !host_mass))) throw ConfigError("update_frequency: bad arguments");
        if (static_cast<size_t>(n) * sizeof(int64_t) > s->up_ids.bytes) {
            s->up_ids.grow(n * sizeof(int64_t), s->st);
            s->up_mass.grow(n * sizeof(double), s->st);
        }
        if (n > 0) {
            ck(cudaMemcpyAsync(s->up_ids.p, host_ids, n * sizeof(int64_t), cudaMemcpyHostToDevice, s->st), "H2D");
            ck(cudaMemcpyAsync(s->up_mass.p, host_mass, n * sizeof(double), cudaMemcpyHostToDevice, s->st), "H2D");
        }
        store_update(s->dev(), s->up_ids.as<int64_t>(), s->up_mass.as<double>(), n, s->st);
        ck(cudaGetLastError(), "update_frequency");
        s->check_err();
    });
}

int infllm_store_enforce_capacity(infllm_store_t s) {
    return guard([&] {
        if (!s) throw ConfigError("null store");
        store_enforce(s->dev(), s->st);
        ck(cudaGetLastError(), "enforce_capacity");
        s->check_err();
    });
}

int infllm_store_note_step_boundary(infllm_store_t s) {
    return guard([&] {
        if (!s) throw ConfigError("null store");
        store_boundary(s->dev(), s->st);
        ck(cudaGetLastError(), "note_step_boundary");
        s->check_err();
    });
}

int infllm_store_counters(infllm_store_t s, infllm_layer_metrics* m) {
    return guard([&] {
        if (!s || !m) throw ConfigError("null argument");
        LruState x{};
        ck(cudaMemcpyAsync(&x, s->lru.p, sizeof(x), cudaMemcpyDeviceToHost, s->st), "D2H");
        ck(cudaStreamSynchronize(s->st), "counters");
        m->units = s->n_units;
        m->hot_units = x.hot_count;
        m->peak_hot_units = x.peak_hot_units;
        m->peak_hot_bytes = x.peak_hot_bytes;
        m->hits = x.hits;
        m->misses = x.misses;
        m->loads = x.loads;
        m->evictions = x.evictions;
        m->requested = x.requested;
    });
}

int infllm_store_trace(infllm_store_t s, int64_t* host_step, int64_t* host_unit, int32_t* host_hit, int64_t cap,
                       int64_t* n_out) {
    return guard([&] {
        if (!s) throw ConfigError("null store");
        *n_out = s->trace_count;
        const int64_t n = std::min(cap, s->trace_count);
        if (n <= 0) return;
        std::vector<int64_t> t(static_cast<size_t>(3 * n));
        ck(cudaMemcpyAsync(t.data(), s->trace.p, t.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s->st), "D2H");
        ck(cudaStreamSynchronize(s->st), "trace");
        for (int64_t i = 0; i < n; ++i) {
            host_step[i] = t[static_cast<size_t>(3 * i)];
            host_unit[i] = t[static_cast<size_t>(3 * i + 1)];
            host_hit[i] = static_cast<int32_t>(t[static_cast<size_t>(3 * i + 2)]);
        }
    });
}

int infllm_store_unit_freq(infllm_store_t s, double* host_freq, int32_t* host_hot, int64_t n) {
    return guard([&] {
        if (!s) throw ConfigError("null store");
        n = std::min(n, s->n_units);
        if (n <= 0) return;
        std::vector<int8_t> h(static_cast<size_t>(n));
        ck(cudaMemcpyAsync(host_freq, s->freq.p, n * sizeof(double), cudaMemcpyDeviceToHost, s->st), "D2H");
        ck(cudaMemcpyAsync(h.data(), s->hot.p, n, cudaMemcpyDeviceToHost, s->st), "D2H");
        ck(cudaStreamSynchronize(s->st), "unit_freq");
        for (int64_t i = 0; i < n; ++i) host_hot[i] = h[static_cast<size_t>(i)];
    });
}

int infllm_score_acc_create(int64_t local_size, int32_t n_heads, int32_t n_kv_heads, int32_t head_dim, int32_t dtype,
                            infllm_score_acc_t* out) {
    return guard([&] {
        if (!out) throw ConfigError("null argument");
        if (local_size < 1) throw ConfigError("local_size must be >= 1");
        if (n_heads < 1 || n_kv_heads < 1 || n_heads % n_kv_heads || head_dim < 1)
            throw ConfigError("ScoreAccumulator: bad shape");
        if (dtype != INFLLM_DTYPE_F32 && dtype != INFLLM_DTYPE_BF16) throw ConfigError("dtype must be f32 or bf16");
        auto a = std::make_unique<infllm_score_acc>();
        a->L = local_size;
        a->H = n_heads;
        a->G = n_kv_heads;
        a->d = head_dim;
        a->dtype = dtype;
        *out = a.release();
    });
}

int infllm_score_acc_destroy(infllm_score_acc_t a) {
    return guard([&] {
        if (!a) return;
        cudaDeviceSynchronize();
        a->sums.release(nullptr);
        a->out.release(nullptr);
        cudaDeviceSynchronize();
        delete a;
    });
}

int infllm_score_acc_accumulate(infllm_score_acc_t a, const void* q, int64_t l_x, int64_t s, const void* pending_keys,
                                int64_t n_pending, void* stream) {
    return guard([&] {
        if (!a) throw ConfigError("null accumulator");
        auto st = static_cast<cudaStream_t>(stream);
        // repr_score.hpp:42-49
        if (s != a->next_q) throw StreamError("ScoreAccumulator: out-of-order query batch");
        if (a->hi != s) throw StreamError("ScoreAccumulator: pending range out of sync");
        const int64_t hi = s + l_x;
        if (n_pending != hi - a->lo) throw StreamError("ScoreAccumulator: pending keys do not cover range");
        if (hi - a->lo > a->cap) {  // grow the ring, live range re-based at 0
            const int64_t c = std::max<int64_t>({hi - a->lo, 2 * a->cap, 1024});
            DBuf nb;
            nb.alloc(c * sizeof(double), st);
            const int64_t live = a->hi - a->lo;
            for (int64_t j = 0; j < live;) {  // at most two contiguous pieces
                const int64_t src = (a->ring0 + j) % std::max<int64_t>(a->cap, 1);
                const int64_t len = std::min(live - j, a->cap - src);
                ck(cudaMemcpyAsync(nb.as<double>() + j, a->sums.as<double>() + src, len * sizeof(double),
                                   cudaMemcpyDeviceToDevice, st),
                   "D2D");
                j += len;
            }
            a->sums.release(st);
            a->sums = nb;
            nb.p = nullptr;
            a->cap = c;
            a->ring0 = 0;
        }
        score_acc_zero(a->sums.as<double>(), a->ring0 + (a->hi - a->lo), l_x, a->cap, st);  // new pending sums
        score_acc_run(q, l_x, s, pending_keys, n_pending, a->lo, a->L, a->H, a->G, a->d,
                      a->dtype == INFLLM_DTYPE_BF16, a->sums.as<double>(), a->ring0, a->cap, st);
        ck(cudaGetLastError(), "accumulate");
        a->hi = hi;
        a->next_q = hi;
    });
}

int infllm_score_acc_finalize_front(infllm_score_acc_t a, int64_t n, float* host_out) {
    return guard([&] {
        if (!a) throw ConfigError("null accumulator");
        if (n > a->hi - a->lo) throw StreamError("ScoreAccumulator: finalize beyond range");  // repr_score.hpp:73
        if (n <= 0) return;
        if (static_cast<size_t>(n) * sizeof(float) > a->out.bytes) a->out.alloc(n * sizeof(float), nullptr, false);
        score_acc_final(a->sums.as<double>(), a->ring0, a->cap, n, a->L, a->out.as<float>(), nullptr);
        ck(cudaMemcpy(host_out, a->out.p, n * sizeof(float), cudaMemcpyDeviceToHost), "D2H");
        a->ring0 = (a->ring0 + n) % a->cap;
        a->lo += n;
    });
}

}  // extern "C"

// Device timeline (common.cuh TlRec): every block of the step kernels appends
// (kernel, SM, start, end) while a buffer is bound.
namespace {
struct Timeline {
    TlRec* rec = nullptr;
    unsigned long long* cnt = nullptr;
    int64_t cap = 0;
} g_timeline;
void timeline_bind(const TlBuf& b) {
    ck(tl_bind_kernels(b), "timeline bind");
    ck(tl_bind_attn_tc(b), "timeline bind");
    ck(tl_bind_attn_dec(b), "timeline bind");
    ck(tl_bind_lookup(b), "timeline bind");
}
}  // namespace

int infllm_timeline_enable(int64_t capacity) {
    return guard([&] {
        ck(cudaDeviceSynchronize(), "timeline");
        timeline_bind(TlBuf{nullptr, nullptr, 0});
        if (g_timeline.rec) cudaFree(g_timeline.rec);
        if (g_timeline.cnt) cudaFree(g_timeline.cnt);
        g_timeline = Timeline{};
        if (capacity <= 0) return;
        ck(cudaMalloc(&g_timeline.rec, static_cast<size_t>(capacity) * sizeof(TlRec)), "timeline alloc");
        ck(cudaMalloc(&g_timeline.cnt, sizeof(unsigned long long)), "timeline alloc");
        ck(cudaMemset(g_timeline.cnt, 0, sizeof(unsigned long long)), "timeline");
        g_timeline.cap = capacity;
        timeline_bind(TlBuf{g_timeline.rec, g_timeline.cnt, static_cast<unsigned long long>(capacity)});
    });
}

int infllm_timeline_read(uint32_t* kernel, uint32_t* sm, uint64_t* t0, uint64_t* t1, int64_t cap, int64_t* n_out,
                         int32_t reset) {
    return guard([&] {
        *n_out = 0;
        if (!g_timeline.rec) return;
        ck(cudaDeviceSynchronize(), "timeline");
        unsigned long long n = 0;
        ck(cudaMemcpy(&n, g_timeline.cnt, sizeof(n), cudaMemcpyDeviceToHost), "timeline");
        const int64_t m = std::min<int64_t>({static_cast<int64_t>(n), g_timeline.cap, cap});
        std::vector<TlRec> r(static_cast<size_t>(std::max<int64_t>(m, 0)));
        if (m > 0) ck(cudaMemcpy(r.data(), g_timeline.rec, m * sizeof(TlRec), cudaMemcpyDeviceToHost), "timeline");
        for (int64_t i = 0; i < m; ++i) {
            kernel[i] = r[i].kid;
            sm[i] = r[i].sm;
            t0[i] = r[i].t0;
            t1[i] = r[i].t1;
        }
        *n_out = static_cast<int64_t>(n);
        if (reset) ck(cudaMemset(g_timeline.cnt, 0, sizeof(unsigned long long)), "timeline");
    });
}

int infllm_debug_tc_selftest(const void* q, const void* k, const void* vt, float* s_out, float* o_out,
                             void* stream) {
    return guard([&] {
        tc_selftest(q, k, vt, s_out, o_out, static_cast<cudaStream_t>(stream));
        ck(cudaGetLastError(), "tc_selftest");
    });
}

}  // extern "C"
