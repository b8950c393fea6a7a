/*
 * infllm_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference InfLLM engine (/root/reference/proj,
 * header-only C++20/Eigen, namespace blockmem) used as the parity checker for
 * the B200 path. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it. The product library
 * (paper_2402_04617_b200/libinfllm_b200.so) never links or calls it.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * proj/include/blockmem/). Differences from the reference are deliberate and
 * documented: (1) q/k/v are injected per step instead of coming from the
 * SyntheticAdapter (engine.hpp:251), (2) GQA is emulated by
 * replicating each KV head across its query heads, (3) Eigen's
 * dense products are restated as plain sequential-k loops (Eigen is an
 * unpinned dependency, proj/CMakeLists.txt:12).
 */
#ifndef INFLLM_ORACLE_H
#define INFLLM_ORACLE_H

#include <stdint.h>

#include "../include/infllm_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_engine oracle_engine;

const char* oracle_last_error(void);

/* StreamEngine<float> without the adapter (engine.hpp:66-73). n_threads > 1
 * parallelises over heads (the reference is single-threaded per stream). */
oracle_engine* oracle_engine_create(const infllm_engine_config* cfg,
                                    const infllm_model_shape* shape, int32_t n_threads);
void oracle_engine_destroy(oracle_engine* e);
/* fuzz support: StreamEngine::set_always_emit_weights (engine.hpp:84-86) */
void oracle_set_always_emit_weights(oracle_engine* e, int32_t v);

/* One StreamEngine::step for one layer (engine.hpp:242-359) with explicit
 * token-major q [l_x][H][d], k [l_x][Hkv][d], v [l_x][Hkv][dv] (fp32).
 * is_decode selects decode_step (engine.hpp:100-103) vs encode_chunk
 * (92-97) lookup semantics. out [l_x][H][dv]. ids_out receives the retrieved
 * unit ids (capacity ids_cap), masses_out (may be NULL) the per-retrieved-unit
 * masses (engine.hpp:271-283). Returns 0 or an INFLLM_ERR_* code. */
int32_t oracle_step(oracle_engine* e, int32_t layer, const float* q, const float* k,
                    const float* v, int64_t l_x, int32_t is_decode, float* out,
                    int64_t* ids_out, int64_t ids_cap, int64_t* n_ids, double* masses_out);
int32_t oracle_finish(oracle_engine* e);
/* CPU-baseline harness: stream n tokens through the window/packing/score
 * bookkeeping only (no lookup, no attention) to reach a steady state. */
int32_t oracle_warm_start(oracle_engine* e, int32_t layer, const float* q, const float* k, const float* v,
                          int64_t n);

int32_t oracle_layer_metrics(oracle_engine* e, int32_t layer, infllm_layer_metrics* m);
int32_t oracle_stream_state(oracle_engine* e, int32_t layer, int64_t* tokens_fed,
                            int64_t* steps_done, int64_t* initial_len, int64_t* local_len,
                            int64_t* pending_partial);
int32_t oracle_unit_info(oracle_engine* e, int32_t layer, int64_t unit_id, int64_t* start_abs,
                         int64_t* size, int64_t* repr_abs, int64_t* n_repr_out);
int32_t oracle_unit_freq(oracle_engine* e, int32_t layer, double* freq, int32_t* hot, int64_t n);
int32_t oracle_trace(oracle_engine* e, int32_t layer, int64_t* step, int64_t* unit,
                     int32_t* hit, int64_t cap, int64_t* n_out);
/* invariant counters (engine.hpp:88-89,361-383) */
int32_t oracle_invariants(oracle_engine* e, uint64_t* checks, uint64_t* violations);
/* phase timings in ms (engine.hpp:43-49): adapter(=0), lookup, attend, score, evict */
int32_t oracle_timings(oracle_engine* e, double* ms5);
/* Representative-score accumulator state for layer: the finalized scores of
 * every token evicted so far (abs positions [init_size, init_size + n)). */
int32_t oracle_evicted_scores(oracle_engine* e, int32_t layer, float* scores, int64_t cap,
                              int64_t* n_out);
/* Representative keys of unit `unit_id`, [n_repr][Hkv][d]. */
int32_t oracle_unit_repr_keys(oracle_engine* e, int32_t layer, int64_t unit_id, float* keys);

/* ---- standalone restatements ---- */
/* select_representatives (repr_score.hpp:94-112) */
int32_t oracle_select_representatives(const float* scores, int64_t n, int64_t r_k,
                                      int64_t* idx, int64_t* n_out);
/* oracle::argsort_topk (oracle.hpp:187-195) */
int32_t oracle_argsort_topk(const double* values, int64_t n, int64_t k, int64_t* idx,
                            int64_t* n_out);
/* TieredStore::relevance_all (memory.hpp:217-234) on an explicit index:
 * q [l_x][H][d] fp32, repr [U][r_k][Hkv][d] fp32 -> rel [U] */
int32_t oracle_relevance_all(const float* q, int64_t l_x, int32_t H, int32_t Hkv, int32_t d,
                             const float* repr, int64_t U, int64_t r_k, double* rel);
/* relevance(batch, unit) single unit (memory.hpp:141-149) */
double oracle_relevance_unit(const float* q, int64_t l_x, int32_t H, int32_t Hkv, int32_t d,
                             const float* repr_keys, int64_t n_repr);
/* oracle::mean_repr_relevance (oracle.hpp:199-207): unit_keys [n][Hkv][d],
 * queries [l_x][H][d] (double) */
double oracle_mean_repr_relevance(const double* unit_keys, int64_t n, const double* q,
                                  int64_t l_x, int32_t H, int32_t Hkv, int32_t d);

/* ---- stand-alone operators, mirroring the C-ABI's infllm_attend /
 * infllm_store_* / infllm_score_acc_* ---- */
typedef struct oracle_store oracle_store;
oracle_store* oracle_store_create(int64_t hot_capacity, double decay, int32_t H, int32_t Hkv, int32_t d,
                                  int64_t bytes_per_token);
void oracle_store_destroy(oracle_store* x);
int32_t oracle_store_add_unit(oracle_store* x, const float* repr_keys, int64_t n, int64_t unit_tokens, int64_t* id);
int32_t oracle_store_begin_step(oracle_store* x, int64_t step);
int32_t oracle_store_lookup(oracle_store* x, const float* q, int64_t l_x, int64_t k_m, int64_t* ids, int64_t* n);
int32_t oracle_store_update_frequency(oracle_store* x, const int64_t* ids, const double* mass, int64_t n);
int32_t oracle_store_enforce_capacity(oracle_store* x);
int32_t oracle_store_note_step_boundary(oracle_store* x);
int32_t oracle_store_counters(oracle_store* x, infllm_layer_metrics* m);
int32_t oracle_store_trace(oracle_store* x, int64_t* step, int64_t* unit, int32_t* hit, int64_t cap, int64_t* n_out);
int32_t oracle_store_unit_freq(oracle_store* x, double* freq, int32_t* hot, int64_t n);
typedef struct oracle_score_acc oracle_score_acc;
oracle_score_acc* oracle_score_acc_create(int64_t local_size, int32_t H, int32_t Hkv, int32_t d);
void oracle_score_acc_destroy(oracle_score_acc* x);
int32_t oracle_score_acc_accumulate(oracle_score_acc* x, const float* q, int64_t l_x, int64_t s, const float* keys,
                                    int64_t n_pending);
int32_t oracle_score_acc_finalize_front(oracle_score_acc* x, int64_t n, float* out);
int32_t oracle_attend(int32_t H, int32_t Hkv, int32_t d, int32_t dv, int32_t position_mode, int64_t local_size,
                      const int32_t* seg_kind, const int64_t* seg_start, const int64_t* seg_n,
                      const float* const* seg_keys, const float* const* seg_values, int32_t n_seg, const float* q,
                      const float* k, const float* v, int64_t l_x, int64_t start_abs, float* out, double* seg_mass,
                      float* weights);

/* ---- double-precision brute-force oracles (oracle.hpp) ---- */
/* dense_attention (oracle.hpp:64-97); token-major double tensors */
int32_t oracle_dense_attention(const double* q, const double* k, const double* v, int64_t n,
                               int32_t H, int32_t Hkv, int32_t d, int32_t dv,
                               int32_t position_mode, int64_t local_size, double* out);
/* windowed_attention_reference (oracle.hpp:103-168) */
int32_t oracle_windowed_attention(const double* q, const double* k, const double* v, int64_t n,
                                  int32_t H, int32_t Hkv, int32_t d, int32_t dv,
                                  const int64_t* schedule, int64_t n_sched, int64_t init_size,
                                  int64_t local_size, int64_t unit_size, int32_t position_mode,
                                  double* out);
/* batch_repr_scores (oracle.hpp:173-184) */
int32_t oracle_batch_repr_scores(const double* q, const double* k, int64_t n, int32_t H,
                                 int32_t Hkv, int32_t d, int64_t local_size, double* out);

/* ---- input generators (harness) ---- */
/* cli.cpp:30-36 noise_ids */
int32_t oracle_noise_ids(uint64_t seed, int64_t n, int64_t* ids);
/* SyntheticAdapter::batch (adapter.hpp:45-69): token-major q/k/v [n][H][d]. */
int32_t oracle_adapter_batch(uint64_t seed, int32_t n_layers, int32_t n_heads, int32_t head_dim,
                             int32_t value_dim, int32_t layer, const int64_t* ids, int64_t n,
                             float* q, float* k, float* v);
/* Counter-based N(0,1) generator for the C1-C4 synthetic tensors
 * (SURVEY §8d): value(seed, tensor, token, head, dim) via splitmix64 +
 * Box-Muller. Fills x[n_tok][n_head][dim] for tokens [tok0, tok0+n_tok). */
int32_t oracle_gaussian_fill(uint64_t seed, uint64_t tensor, int64_t tok0, int64_t n_tok,
                             int32_t n_head, int32_t dim, float* x);
/* workload::gen_planted (workload.hpp:35-76); returns plant_start, plant_id,
 * expected unit range, token ids [length]. */
int32_t oracle_gen_planted(uint64_t seed, int64_t length, int64_t plant_len,
                           const infllm_engine_config* cfg, int64_t probe_len,
                           int32_t align_to_units, int64_t* plant_start, int64_t* plant_id,
                           int64_t* first_unit, int64_t* last_unit, int64_t* ids);

#ifdef __cplusplus
}
#endif

#endif
