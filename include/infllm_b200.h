/*
 * infllm_b200.h — C-ABI drop-in boundary for the InfLLM block-memory attention
 * layer (arXiv 2402.04617), B200-native (sm_100a).
 *
 * The reference exposes its hot path as a header-only C++ template API in
 * namespace `blockmem` (see /root/reference/proj/include/blockmem/). This
 * header is the flat C boundary a C++/cgo/ctypes host binds instead. Every
 * entry point below names the reference interface it replaces (file:line,
 * paths relative to proj/include/blockmem/).
 *
 * Conventions
 *  - Return value: INFLLM_OK (0) or an error code; infllm_last_error() gives a
 *    thread-local one-line message. INFLLM_ERR_CONFIG mirrors blockmem::
 *    ConfigError (types.hpp:20-22), INFLLM_ERR_STREAM mirrors
 *    blockmem::StreamError (types.hpp:24-26).
 *  - Tensor arguments are DEVICE pointers (unless the name says host_), dense
 *    row-major, element type = the engine dtype (fp32 or bf16):
 *        q   [l_x][n_heads][head_dim]
 *        k   [l_x][n_kv_heads][head_dim]
 *        v   [l_x][n_kv_heads][value_dim]
 *        out [l_x][n_heads][value_dim]
 *    n_heads must be a multiple of n_kv_heads (GQA); with n_kv_heads ==
 *    n_heads this is the reference's MHA layout transposed from per-head
 *    matrices (types.hpp:158-169) to token-major.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream). All compute
 *    entry points are asynchronous on it; nothing data-dependent is read back
 *    to the host inside a step (lookup ids, representative indices and LRU
 *    state live on the device).
 *  - One host thread per engine at a time (reference: SPEC.md "Concurrency
 *    Model"; no internal locking, like blockmem::StreamEngine).
 */
#ifndef INFLLM_B200_H
#define INFLLM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define INFLLM_OK 0
#define INFLLM_ERR_CONFIG 1 /* blockmem::ConfigError   (types.hpp:20-22) */
#define INFLLM_ERR_STREAM 2 /* blockmem::StreamError   (types.hpp:24-26) */
#define INFLLM_ERR_CUDA 3
#define INFLLM_ERR_NCCL 4
#define INFLLM_ERR_ARG 5

/* blockmem::LookupMode (types.hpp:51) */
#define INFLLM_LOOKUP_ENCODE_AND_DECODE 0
#define INFLLM_LOOKUP_DECODE_ONLY 1
#define INFLLM_LOOKUP_NONE 2

/* blockmem::PositionMode (types.hpp:52) */
#define INFLLM_POSITION_CLAMPED 0
#define INFLLM_POSITION_ABSOLUTE 1

/* engine element type; the reference's Real is float (real.hpp:7-11) */
#define INFLLM_DTYPE_F32 0
#define INFLLM_DTYPE_BF16 1

/* blockmem::EngineConfig (types.hpp:84-110); same field names and defaults */
typedef struct infllm_engine_config {
    int64_t chunk_size;   /* l_C  (default 512)  */
    int64_t unit_size;    /* l_bs (default 128)  */
    int64_t n_repr;       /* r_k  (default 4)    */
    int64_t local_size;   /* l_L  (default 4096) */
    int64_t init_size;    /* l_I  (default 128)  */
    int64_t n_lookup;     /* k_m  (default 32)   */
    int64_t hot_capacity; /* default 32          */
    double decay;         /* d    (default 0.1)  */
    int32_t lookup_mode;   /* INFLLM_LOOKUP_*    */
    int32_t position_mode; /* INFLLM_POSITION_*  */
} infllm_engine_config;

/* blockmem::ModelShape (types.hpp:29-49) + the GQA KV-head count the
 * reference lacks. */
typedef struct infllm_model_shape {
    int32_t n_layers;
    int32_t n_heads;    /* query heads */
    int32_t n_kv_heads; /* key/value heads; n_heads % n_kv_heads == 0 */
    int32_t head_dim;
    int32_t value_dim;  /* <= 0: same as head_dim */
} infllm_model_shape;

/* blockmem::CacheCounters (memory.hpp:151-157) + EngineLayerMetrics
 * (engine.hpp:35-41) */
typedef struct infllm_layer_metrics {
    int64_t units;
    int64_t hot_units;
    int64_t peak_hot_units;
    int64_t peak_hot_bytes;
    uint64_t hits;
    uint64_t misses;
    uint64_t loads;
    uint64_t evictions;
    uint64_t requested;
} infllm_layer_metrics;

typedef struct infllm_engine* infllm_engine_t;

/* Thread-local message of the last failed call on this thread. */
const char* infllm_last_error(void);
/* Library build string (arch, dtype support). */
const char* infllm_version(void);

/* EngineConfig{} defaults (types.hpp:84-94). */
int infllm_config_default(infllm_engine_config* cfg);
/* EngineConfig::validate (types.hpp:96-109) + ModelShape::validate
 * (types.hpp:45-48); shape may be NULL. */
int infllm_config_validate(const infllm_engine_config* cfg, const infllm_model_shape* shape);

/* StreamEngine<Scalar>(EngineConfig, ModelShape, seed) (engine.hpp:66-73),
 * minus the synthetic adapter: q/k/v are supplied per call. `device` is the
 * CUDA ordinal. kv_group_begin/kv_group_count select the KV heads this engine
 * owns (multi-GPU KV-group sharding; pass 0 / n_kv_heads for the whole
 * layer); its q/k/v/out pointers then hold only the owned heads. */
int infllm_engine_create(const infllm_engine_config* cfg, const infllm_model_shape* shape,
                         int32_t dtype, int32_t device, int32_t kv_group_begin,
                         int32_t kv_group_count, infllm_engine_t* out);
int infllm_engine_destroy(infllm_engine_t eng);

/* Cross-shard exchange hook for KV-group sharding.
 * Relevance, representative scores and attention masses are sums over ALL
 * heads (memory.hpp:221-228, repr_score.hpp:55-57, engine.hpp:278-281), so
 * each shard computes fp64 partials per KV group into a [rows][g_total]
 * device buffer (its own columns [g0, g0 + g_count)); the hook must fill the
 * other columns in place (an all-gather, on `stream`) before the engine sums
 * the groups in fixed order 0..g_total-1, which keeps ids bit-identical for
 * any number of shards. NULL (the default) = single shard. Return 0 on
 * success. */
typedef int (*infllm_allgather_fn)(void* user, double* buf, int64_t rows, int32_t g0,
                                   int32_t g_count, int32_t g_total, void* stream);
int infllm_engine_set_allgather(infllm_engine_t eng, infllm_allgather_fn fn, void* user);

/* KV-group sharding over NCCL: the same exchange as the hook
 * above, done by the library itself with ncclAllGather on the engine's streams
 * (graph-capturable, so sharded streams stay CUDA-graph replayed). Rank 0
 * makes an id with infllm_nccl_unique_id and the host broadcasts its 128
 * bytes; every rank then calls infllm_engine_set_comm with its engine, which
 * must own KV groups [rank G/n, (rank + 1) G/n). NCCL is loaded at run time
 * (libnccl.so.2); INFLLM_ERR_NCCL when it is missing. Option "gather_output"
 * = 1 makes the step's `out` the full [l_x][n_heads][value_dim] tensor,
 * all-gathered over the shards after the attention (C-2). */
int infllm_nccl_unique_id(uint8_t* id128);
int infllm_engine_set_comm(infllm_engine_t eng, const uint8_t* id128, int32_t rank, int32_t nranks);

/* The exchange arithmetic on the host (no GPU): gathered [nranks][rows]
 * [g_count] fp64 per-group partials as an all-gather delivers them -> out
 * [rows], each row summed over all groups in group order (exactly the
 * association the device uses after the exchange); and the lookup's top-k
 * (memory.hpp:240-253: rel desc, id asc, returned ascending). */
int infllm_exchange_fold_host(const double* gathered, int64_t rows, int32_t nranks, int32_t g_count, double* out);
int infllm_topk_host(const double* rel, int64_t n, int64_t k, int64_t* ids, int64_t* n_out);

/* Pre-size the unit pool and trace for a stream of max_tokens tokens plus
 * 4096 one-token steps of trace (the reference grows its std::vectors on
 * demand; the engine grows its device pools too, draining its streams, this
 * only moves the growth out of the timed region). */
int infllm_engine_reserve(infllm_engine_t eng, int64_t max_tokens);
/* Return every layer to the empty-stream state (tokens_fed = 0), keeping the
 * device pools; asynchronous on `stream`. */
int infllm_engine_reset(infllm_engine_t eng, void* stream);
/* Engine options: "tc_attention" (1 = tcgen05 attention when the shape
 * allows, 0 = CUDA-core attention), "cuda_graphs" (1 = graph-replayed
 * encode_stream, default), "attn_score_bound" (1 = the tcgen05 attention may
 * use the per-row score bound |q| |k|_max as a fixed softmax offset, default;
 * 0 = always the online-max path), "host_tier_slots" (S > 0: unit pages live
 * in a pinned-host tier and the attention reads them from an S-slot GPU unit
 * cache filled on demand over PCIe on a side stream -- the north star's
 * host-offloaded store; TieredStore's hot/cold tiers (memory.hpp:165-168) are
 * bookkeeping only in the reference, outputs are identical either way;
 * 2*n_lookup <= S <= 16384; set before reserve() and the first step),
 * "decode_kernel" (1 = split-KV decode attention for one-token steps,
 * default; 0 = the prefill attention kernel), "multi_stream_decode" (1 = run
 * decode steps through the five-stream pipeline; default 0 = caller's stream),
 * "attn_splits" (split-KV tcgen05 attention: 0 = automatic when the grid leaves
 * SMs idle, else the split count, <= 16), "attn_streams" (2 = chunk-step
 * attention alternates between two dedicated streams so consecutive launches
 * overlap at the handoff, default; 1 = the caller's stream),
 * "graph_node_priority" (1 = instantiate stream graphs honouring the
 * attention's launch priority; default 0), "decode_chain" (1 = a one-token
 * step launches the lookup first, forming the query sums from q itself, with
 * the decode front as its programmatic dependent and K4 behind both, and a
 * decode_batch of <= 4 sequences runs its fronts beside its relevance scan;
 * default; 0 = front, lookup, K4 in sequence), "decode_lookup_fused" (1 =
 * one-token steps past 2048 units take the one-launch scan + top-k of chunk
 * steps, default; 0 = the streaming scan + a top-k launch), "decode_merge_kernel" (1 = the
 * decode attention's split merge as its own parallel launch, default; 0 = in
 * each group's last split), "lookup_units_per_block" /
 * "lookup_units_per_block_decode" (K1+K2 grid: units per block in chunk /
 * one-token steps), "gather_output" (sharded engines: all-gather every head's
 * output into `out`). Options that change launches drop captured graphs. */
int infllm_engine_set_option(infllm_engine_t eng, const char* key, int64_t value);

/* StreamEngine::encode_chunk (engine.hpp:92-97) for one layer: lookup (if
 * lookup_mode == encode_and_decode), attention over [initial | retrieved
 * units | local | causal chunk], frequency update + capacity, representative
 * scoring, window roll and unit packing (engine.hpp:242-359). Requires
 * 1 <= l_x <= chunk_size. Layers advance independently; a step of the
 * reference engine is one call per layer in order 0..n_layers-1. */
int infllm_encode_chunk(infllm_engine_t eng, int32_t layer, const void* q, const void* k,
                        const void* v, int64_t l_x, void* out, void* stream);

/* StreamEngine::feed (engine.hpp:106-112) for one layer: n_tokens of
 * device q/k/v [n_tokens][heads][dim] as consecutive encode_chunk steps of
 * chunk_size tokens, outputs into out [n_tokens][n_heads][value_dim]. The
 * whole chunk schedule is captured once into a CUDA graph (keyed by
 * pointers, length and the starting stream state) and replayed; option
 * "cuda_graphs" = 0 launches the steps directly. */
int infllm_encode_stream(infllm_engine_t eng, int32_t layer, const void* q, const void* k, const void* v,
                         int64_t n_tokens, void* out, void* stream);
/* Same with HOST (preferably pinned) q/k/v/out: per-chunk H2D into device
 * staging buffers and D2H of each output chunk, on copy streams overlapped
 * with the neighbouring chunks' compute. */
int infllm_encode_stream_host(infllm_engine_t eng, int32_t layer, const void* host_q, const void* host_k,
                              const void* host_v, int64_t n_tokens, void* host_out, void* stream);

/* StreamEngine::decode_step (engine.hpp:100-103): l_x = 1, lookup unless
 * lookup_mode == none. */
int infllm_decode_step(infllm_engine_t eng, int32_t layer, const void* q, const void* k,
                       const void* v, void* out, void* stream);

/* Batched decode (BASELINE configs[4]): one
 * StreamEngine::decode_step (engine.hpp:100-103) for each of n independent
 * sequences, engine i owning sequence i. q [n][H][d], k/v [n][H_kv][d], out
 * [n][H][d_v], device memory. Every stage (prep, eviction, unit selection,
 * lookup + top-k, attention, LRU) is one launch for all n sequences when the
 * engines share config and shape (bf16, d = 128, unit 128, single shard, no
 * host tier) and n > 1; otherwise (and for one sequence, whose single-sequence
 * chain is shorter) the engines step one after another. Results equal n
 * decode_step calls. */
int infllm_decode_batch(infllm_engine_t* engs, int32_t n, int32_t layer, const void* q,
                        const void* k, const void* v, void* out, void* stream);

/* StreamEngine::finish (engine.hpp:115-119): flushes each layer's held-back
 * partial unit. Synchronous. */
int infllm_finish(infllm_engine_t eng, void* stream);

/* ---- diagnostics (synchronous: they wait for the engine's queued work) ---- */

/* LayerStepOutput::retrieved_ids of the most recent step of `layer`
 * (engine.hpp:26-30), ascending unit ids. */
int infllm_retrieved_ids(infllm_engine_t eng, int32_t layer, int64_t* host_ids, int64_t cap,
                         int64_t* n_out);
/* StreamEngine::metrics() per layer (engine.hpp:121-138). */
int infllm_get_layer_metrics(infllm_engine_t eng, int32_t layer, infllm_layer_metrics* out);
/* TieredStore::unit(id) (memory.hpp:178-180): span and representative
 * positions (MemoryUnit::repr_abs, memory.hpp:25). host_repr_abs holds
 * n_repr entries. */
int infllm_unit_info(infllm_engine_t eng, int32_t layer, int64_t unit_id, int64_t* start_abs,
                     int64_t* size, int64_t* host_repr_abs, int64_t* n_repr_out);
/* Stream bookkeeping: tokens fed, steps done, initial_len, local_len,
 * pending_partial (engine.hpp:77-78,140-148). */
int infllm_stream_state(infllm_engine_t eng, int32_t layer, int64_t* tokens_fed,
                        int64_t* steps_done, int64_t* initial_len, int64_t* local_len,
                        int64_t* pending_partial);
/* Per-unit decayed-frequency scores s_b (MemoryUnit::freq_score,
 * memory.hpp:27) and tiers (1 = hot) for units [0, n). */
int infllm_unit_freq(infllm_engine_t eng, int32_t layer, double* host_freq, int32_t* host_hot,
                     int64_t n);
/* Engine trace (TieredStore::trace, memory.hpp:159-163,182): up to cap
 * records (step, unit_id, hit). */
int infllm_trace(infllm_engine_t eng, int32_t layer, int64_t* host_step, int64_t* host_unit,
                 int32_t* host_hit, int64_t cap, int64_t* n_out);
/* Host tier counters of `layer` since the last reset: out[0] unit pages
 * copied host -> GPU cache, out[1] retrieved units already resident in the
 * cache, out[2] H2D bytes, out[3] slot count (0: host tier off). */
int infllm_tier_stats(infllm_engine_t eng, int32_t layer, int64_t* out4);
/* Number of kernels this engine launched so far (all layers). */
int infllm_kernel_launches(infllm_engine_t eng, int64_t* n_out);
/* Fill host_out with the dominant attention kernel's average device time of
 * the last timed window (ms) and the number of launches in it;
 * infllm_profile_begin starts the window (events on the engine stream). */
int infllm_profile_begin(infllm_engine_t eng, int32_t enable);
int infllm_profile_read(infllm_engine_t eng, double* attn_ms_total, int64_t* attn_launches,
                        double* lookup_ms_total, int64_t* lookup_launches);

/* Device timeline (tracing; the reference's PhaseTimings, engine.hpp:43-49,
 * at kernel granularity): while enabled, thread 0 of every block of the step
 * kernels appends (kernel kind, SM id, globaltimer start / end in ns) to a
 * device ring of `capacity` records. Kernel kinds: 0 attention (K3), 1 RoPE
 * table, 2 prep, 3 prefix, 4 lookup scan, 5 top-k, 6 eviction + scoring,
 * 7 representative selection, 8 LRU, 9 host-tier copy, 10 decode attention
 * (K4), 11 decode front, 12 mass reduction. capacity 0 disables (the
 * default). Process-wide; synchronous. */
int infllm_timeline_enable(int64_t capacity);
/* Copy up to cap records out; *n_out = records written since the last reset
 * (may exceed the capacity: the ring keeps the first `capacity`). reset != 0
 * clears the ring. Synchronous. */
int infllm_timeline_read(uint32_t* kernel, uint32_t* sm, uint64_t* t0, uint64_t* t1, int64_t cap,
                         int64_t* n_out, int32_t reset);

/* StreamEngine::metrics().timings (PhaseTimings, engine.hpp:43-49; cli.cpp
 * timings_ms) measured on the device: summed event time of each phase's
 * launches over the profile window (infllm_profile_begin), in ms, in the
 * order lookup, attend, score (query sums / prefix for the representative
 * scores, ring append, RoPE), evict (eviction scoring, unit packing,
 * representative selection, frequency update and capacity); launches4 (may
 * be NULL) gets the number of timed launch groups per phase. Phases overlap
 * on the engine's streams, so the sum exceeds the wall time. */
int infllm_phase_timings(infllm_engine_t eng, double* ms4, int64_t* launches4);
/* StreamEngine::invariant_checks / invariant_violations (engine.hpp:88-89):
 * check_softmax (361-371) counts one check per head and row of every step
 * that attended retrieved units (a violation: a row whose softmax
 * denominator is not a positive finite number, checked on the device) and
 * check_conservation (373-383) one per layer step. Synchronous. */
int infllm_invariants(infllm_engine_t eng, uint64_t* checks, uint64_t* violations);

/* ---- standalone operators (device pointers, async on stream) ---- */

/* select_representatives (repr_score.hpp:94-112) for `n_units` units at
 * once: scores [n_units][unit_len] fp32 (row u has lens[u] valid entries,
 * lens may be NULL = all unit_len); writes min(r_k, len) ascending indices
 * per unit into idx [n_units][r_k] (unused slots = -1). */
int infllm_select_representatives(const float* scores, const int64_t* lens, int64_t n_units,
                                  int64_t unit_len, int64_t r_k, int64_t* idx, void* stream);

/* TieredStore::relevance_all + lookup's top-k (memory.hpp:217-253) over an
 * explicit representative index: qsum [n_kv_heads][head_dim] fp64 (sum of
 * the chunk's queries over the heads of each KV group), repr
 * [n_units][n_kv_heads][r_k][head_dim] (dtype), -> rel [n_units] fp64 and
 * ids [min(k_m, n_units)] ascending. */
int infllm_lookup(const double* qsum, const void* repr, int32_t dtype, int64_t n_units,
                  int64_t r_k, int32_t n_kv_heads, int32_t head_dim, int64_t k_m, double* rel,
                  int64_t* ids, void* stream);

/* ---- stand-alone reference operators (the pieces StreamEngine::step composes) ---- */

/* blockmem::Segment kinds (attention.hpp:14-26) */
#define INFLLM_SEG_INITIAL 0
#define INFLLM_SEG_RETRIEVED 1
#define INFLLM_SEG_LOCAL 2

/* blockmem::SegmentView (attention.hpp:28-51): one window segment; keys are
 * raw (un-rotated, rotary.hpp is applied at attention time). Device pointers,
 * token-major, element type = dtype. */
typedef struct infllm_segment {
    int32_t kind;        /* INFLLM_SEG_* */
    int64_t start_abs;   /* absolute position of the first token */
    int64_t n_tokens;
    const void* keys;    /* [n_tokens][n_kv_heads][head_dim] */
    const void* values;  /* [n_tokens][n_kv_heads][value_dim] */
} infllm_segment;

/* blockmem::attend (attention.hpp:116-230): the batch q/k/v [l_x][heads][dim]
 * (device) at absolute positions start_abs.. attends over the window
 * segments in order, then causally over itself; clamped or absolute
 * positions per position_mode with l_L = local_size. out [l_x][n_heads][dv].
 * seg_mass (device, may be NULL): per segment sum over heads, rows and its
 * columns of the softmax weights / n_heads (the unit mass of
 * engine.hpp:271-283, for retrieved segments). weights (device, may be NULL):
 * the full weights [n_heads][l_x][n_ctx + l_x] (emit_weights,
 * attention.hpp:227). Asynchronous on stream except for a small parameter
 * upload. */
int infllm_attend(const infllm_model_shape* shape, int32_t dtype, int32_t position_mode, int64_t local_size,
                  const infllm_segment* window, int32_t n_segments, const void* q, const void* k,
                  const void* v, int64_t l_x, int64_t start_abs, void* out, double* seg_mass, float* weights,
                  void* stream);

/* blockmem::TieredStore (memory.hpp:170-323) on the device: the
 * representative index ([units][n_kv_heads][r_k][head_dim], dtype), decayed
 * frequency scores, hot tier, counters and trace. Store calls are
 * synchronous (they return the reference's StreamError conditions). */
typedef struct infllm_store* infllm_store_t;
/* TieredStore(hot_capacity, decay, n_heads) (memory.hpp:172-175) + the
 * index shape; bytes_per_token feeds hot_bytes (MemoryUnit::bytes). */
int infllm_store_create(int64_t hot_capacity, double decay, int32_t n_heads, int32_t n_kv_heads, int32_t head_dim,
                        int64_t n_repr, int32_t dtype, int64_t bytes_per_token, infllm_store_t* out);
int infllm_store_destroy(infllm_store_t s);
/* add_unit (memory.hpp:196-212): the next unit id; repr_keys [n][n_kv][d]
 * (device, n <= n_repr representative keys); the unit holds unit_tokens
 * tokens; it starts cold. */
int infllm_store_add_unit(infllm_store_t s, const void* repr_keys, int64_t n, int64_t unit_tokens,
                          int64_t* unit_id);
/* begin_step (memory.hpp:214): the step id the next lookup records. */
int infllm_store_begin_step(infllm_store_t s, int64_t step);
/* relevance_all + lookup (memory.hpp:217-269): batch queries q
 * [l_x][n_heads][d] (device) -> ids (host, ascending, min(k_m, units)),
 * hit/miss bookkeeping and trace; rel (device, may be NULL) [units] fp64. */
int infllm_store_lookup(infllm_store_t s, const void* q, int64_t l_x, int64_t k_m, int64_t* host_ids, int64_t* n_ids,
                        double* rel);
/* update_frequency (memory.hpp:273-281): host (id, mass) pairs. */
int infllm_store_update_frequency(infllm_store_t s, const int64_t* host_ids, const double* host_mass, int64_t n);
/* enforce_capacity (memory.hpp:285-300) and note_step_boundary (303-308). */
int infllm_store_enforce_capacity(infllm_store_t s);
int infllm_store_note_step_boundary(infllm_store_t s);
/* counters (memory.hpp:151-157,181): units, hot_units, peaks, hits, misses,
 * loads, evictions, requested. */
int infllm_store_counters(infllm_store_t s, infllm_layer_metrics* m);
/* trace (memory.hpp:159-163,182) and per-unit s_b / tier (memory.hpp:27). */
int infllm_store_trace(infllm_store_t s, int64_t* host_step, int64_t* host_unit, int32_t* host_hit, int64_t cap,
                       int64_t* n_out);
int infllm_store_unit_freq(infllm_store_t s, double* host_freq, int32_t* host_hot, int64_t n);

/* blockmem::ScoreAccumulator (repr_score.hpp:21-89): fp64 band sums of the
 * queries each pending key will see before it leaves the local window. */
typedef struct infllm_score_acc* infllm_score_acc_t;
int infllm_score_acc_create(int64_t local_size, int32_t n_heads, int32_t n_kv_heads, int32_t head_dim,
                            int32_t dtype, infllm_score_acc_t* out);
int infllm_score_acc_destroy(infllm_score_acc_t a);
/* accumulate (repr_score.hpp:39-69): batch q [l_x][n_heads][d] (device) at
 * absolute position s; pending_keys [n_pending][n_kv][d] (device) covering
 * every pending token [lo, s + l_x). Errors as the reference's StreamError. */
int infllm_score_acc_accumulate(infllm_score_acc_t a, const void* q, int64_t l_x, int64_t s,
                                const void* pending_keys, int64_t n_pending, void* stream);
/* finalize_front (repr_score.hpp:72-82): the first n scores (sum / l_L as
 * float) into host_out, and drops them. Synchronous. */
int infllm_score_acc_finalize_front(infllm_score_acc_t a, int64_t n, float* host_out);

/* Diagnostic: steady-state per-launch time (us) of one kernel family
 * (0 prep, 1 lookup + exact top-k as a one-token step launches it, 2
 * attention, 3 evict + fused select, 4 LRU, 5 relevance scan only, 6 top-k
 * only, 11 lookup with the chunk-step in-pipeline grid) re-launched with the
 * parameters of the engine's last step.
 * Corrupts the engine's stream state: performance investigation only. */
int infllm_debug_kernel_bench(infllm_engine_t eng, int32_t which, int32_t iters, double* us_per_launch);
/* Diagnostic: accumulated host time (us) of infllm_decode_batch by section:
 * [0] argument checks, [1] per-sequence step logic, [2] parameter tables,
 * [3] wait for the parameter-table slot (the batch four calls back),
 * [4] copies + launches, [5] calls. */
int infllm_debug_host_times(double* out6, int32_t reset);
/* Diagnostic: 64 clock64 phase stamps written by instrumented kernels. */
int infllm_debug_timestamps(unsigned long long* out64);
/* Diagnostic: tcgen05 building-block self-test on one 128x128x128 bf16 tile
 * (q, k, vt row-major [128][128] device bf16): s_out = q k^T, o_out =
 * bf16(s_out) vt^T, both fp32 [128][128]. */
int infllm_debug_tc_selftest(const void* q, const void* k, const void* vt, float* s_out, float* o_out,
                             void* stream);

#ifdef __cplusplus
}
#endif

#endif /* INFLLM_B200_H */
