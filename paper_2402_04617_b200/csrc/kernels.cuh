// kernels.cuh — device-side layer state layout and kernel launch interfaces.
//
// HBM layout of one layer (G = KV groups owned by this engine, R = ring
// capacity, a multiple of 128 >= local_size + chunk_size + 1):
//   ring_k / ring_krot / ring_v  [G][R][d]       raw keys, RoPE'd keys
//                                                 (rotated once at append by
//                                                 their absolute position), values
//   P                            [R][G][d] f64   prefix sums of qs_t = sum of
//                                                 the group's query heads
//   init_k / init_krot / init_v  [G][l_I][d]     pinned initial tokens
//   unit_k / unit_krot / unit_v  [U][G][l_bs][d] unit pages (krot only in
//                                                 absolute position mode)
//   repr                         [U][G][r_k][d]  representative keys (lookup index)
//   unit_scores                  [U][l_bs] f32   finalized r_m per token
#pragma once

#include <stdint.h>

#include "common.cuh"
#include "../../include/infllm_b200.h"

namespace infllm {

// Value pages are stored either row-major ([token][dv]) or, when the tcgen05
// attention is used (unit_size == 128), as transposed 128-token pages
// ([dv][128 tokens]) so V^T tiles are K-major UMMA B operands.
struct VLayout {
    int vt;      // 1: transposed pages
    int64_t R;   // ring capacity (multiple of 128)
    int nI;      // init pages (ceil(l_I / 128))
    int64_t l_I;
    int l_bs, dv, G;
    __device__ __forceinline__ int64_t ring(int g, int64_t pos, int c) const {
        const int64_t sl = pos % R;
        return vt ? ((g * (R / 128) + sl / 128) * dv + c) * 128 + sl % 128 : (g * R + sl) * dv + c;
    }
    __device__ __forceinline__ int64_t init(int g, int64_t pos, int c) const {
        return vt ? ((static_cast<int64_t>(g) * nI + pos / 128) * dv + c) * 128 + pos % 128 : (g * l_I + pos) * dv + c;
    }
    __device__ __forceinline__ int64_t unit(int64_t u, int g, int64_t off, int c) const {
        return vt ? ((u * G + g) * dv + c) * l_bs + off : ((u * G + g) * l_bs + off) * dv + c;
    }
};

// tokens per k_prep_tok block (x 16 threads: one per 8-dim chunk of a token)
constexpr int kTokTile = 16;
struct PrepParams {
    const void* q;  // [lx][H][d]
    const void* k;  // [lx][G][d]
    const void* v;  // [lx][G][dv]
    void* qa;       // [H][lxp][d]  rope(q, pos)
    void* qc;       // [H][lxp][d]  rope(q, L)
    void* ring_k;
    void* ring_krot;
    void* ring_v;
    double* P;           // [R][G][d]
    double* chunk_qsum;  // [G][d]
    float2* rtab;        // [lx][d/2] rotation factors of the chunk positions (scratch)
    double* qs;          // [lx][G][d] per-token group query sums (scratch)
    double* tsum;        // [lx/16][G][d] per-16-token-tile sums of qs (scratch)
    float* kmax2;             // [G] running max of |k|^2 over every key fed so far (this step's copy)
    const float* kmax2_prev;  // [G] the previous step's copy
    int dec_chain;  // decode front launched as the lookup's programmatic dependent: lets K4 launch at
                    // entry, waits for the lookup grid before it exits (K4 waits for the front)
    int64_t s, lx, lxp, R, L;
    int H, G, rep, d, dv;
    VLayout vl;
    RopeFreqs freqs;
};

struct LookupParams {
    const double* qsum;  // [G][d]
    const void* repr;    // [U][G][r_k][d]
    double* part;        // [U][Gtot] (writes columns g0..g0+G)    (sharded mode)
    double* rel;         // [U] relevance (fused single-shard mode)
    int64_t* sel;        // [n_sel] ascending ids           (fused single-shard mode)
    unsigned int* done;  // block counter for the fused top-k (zeroed, re-zeroed by the last block)
    int64_t U, n_sel;
    int G, Gtot, g0, r_k, d;
    int fused;           // 1: single shard: rel + top-k in this launch; 2: rel only (multi-block top-k follows)
    double* cand_v;      // fused 2, streaming scan: per-block top-k candidates [gridDim][n_sel]
    int64_t* cand_i;
    int early_dependents;  // 1: let a programmatic dependent (decode K4) launch at kernel entry
    // decode: the query sums are formed from the token's q [H][d] (bf16) in the
    // order the decode front forms them (heads of the group in order from 0.0),
    // so the lookup does not wait for the front; nullptr: read qsum
    const void* qtok;
    int qrep;
};
// fp64 query sum of (group, dim) t = g * d + c
__device__ __forceinline__ double lk_qsum(const LookupParams& p, int t) {
    if (!p.qtok) return p.qsum[t];
    const int g = t / p.d, c = t % p.d;
    const __nv_bfloat16* q = static_cast<const __nv_bfloat16*>(p.qtok) + static_cast<int64_t>(g) * p.qrep * p.d + c;
    double a = 0.0;
    for (int hh = 0; hh < p.qrep; ++hh) a += static_cast<double>(__bfloat162float(q[hh * p.d]));
    return a;
}

// The token's per-group query sums into shared memory s[G * d] (decode chain)
// or a copy of p.qsum: every head load of a slice is issued before its first
// add, and the adds run in head order as in lk_qsum (same fp64 sums).
__device__ __forceinline__ void lk_stage_qsums(const LookupParams& p, double* s) {
    const int n = p.G * p.d;
    if (!p.qtok || (p.d & 3) || (reinterpret_cast<uintptr_t>(p.qtok) & 7)) {
        for (int t = threadIdx.x; t < n; t += blockDim.x) s[t] = lk_qsum(p, t);
        return;
    }
    const int nq = p.d / 4;  // 4-element slices per head row
    for (int t = threadIdx.x; t < p.G * nq; t += blockDim.x) {
        const int g = t / nq, c = (t % nq) * 4;
        const uint2* q = reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(p.qtok) +
                                                        static_cast<int64_t>(g) * p.qrep * p.d + c);
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        for (int h0 = 0; h0 < p.qrep; h0 += 8) {
            uint2 v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (h0 + j < p.qrep) v[j] = q[static_cast<int64_t>(h0 + j) * nq];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (h0 + j < p.qrep) {
                    a0 += static_cast<double>(__uint_as_float(v[j].x << 16));
                    a1 += static_cast<double>(__uint_as_float(v[j].x & 0xffff0000u));
                    a2 += static_cast<double>(__uint_as_float(v[j].y << 16));
                    a3 += static_cast<double>(__uint_as_float(v[j].y & 0xffff0000u));
                }
        }
        double* o = s + g * p.d + c;
        o[0] = a0;
        o[1] = a1;
        o[2] = a2;
        o[3] = a3;
    }
}

struct TopkParams {
    const double* part;  // [U][Gtot]
    double* rel;         // [U]
    int64_t* sel;        // [n_sel] ascending
    int64_t U, n_sel;
    int Gtot;
};

struct AttnParams {
    const void* qa;
    const void* qc;
    void* out;  // [lx][H][dv]
    const void* init_k;
    const void* init_krot;
    const void* init_v;
    const void* unit_k;
    const void* unit_krot;
    const void* unit_v;
    const int32_t* unit_len;
    const int64_t* sel;
    const int32_t* sel_slot;  // host tier: GPU cache slot of each retrieved unit (unit_k/v are slot pages), or null
    const void* ring_k;
    const void* ring_krot;
    const void* ring_v;
    float* mass_e;  // [H][lx][n_sel]
    float* mass_m;
    float* row_m;   // [H][lx]
    float* row_l;
    double* mass_cta;  // [H][n_mt][n_sel] (tcgen05 path)
    const float* kmax2;  // [G] max |k|^2 over all keys (score bound), or null
    double* mass_part;   // decode kernel (K4): per-group unit masses [n_sel][Gtot], or null
    const void* dec_maps;  // decode kernel (K4): 6 TMA tensor maps in device memory (see attn_dec.cu)
    int Gtot, g0;
    int64_t R, s, lx, lxp, init_len, local_start, L, l_I, unit_cap;
    int n_sel, H, G, rep, d, dv, l_bs;
    int absolute, want_mass;
    // check_softmax (engine.hpp:361-371) on the device: rows whose softmax
    // denominator is not a positive finite number add one here (or null)
    unsigned long long* inv_violations;
    // split-KV K3 (n_split > 1): grid.z = split, each CTA a contiguous share of the
    // window's tiles; partials O [split][H][lxp][128] and (m, l) [split][H][lxp][2]
    // (fp32, exp2 domain), merged by k_attn_merge; masses then go through k_mass
    int n_split;
    float* split_o;
    float* split_ml;
    float scale;
    VLayout vl;
};

struct MassParams {
    const float* mass_e;
    const float* mass_m;
    const float* row_m;
    const float* row_l;
    double* part;  // [n_sel][Gtot]
    int64_t lx;
    int n_sel, H, G, Gtot, g0, rep;
};

// One step of TieredStore bookkeeping after the attention: the lookup's
// tier transfers/counters/trace (memory.hpp:254-267), update_frequency
// (273-281), enforce_capacity (285-300) and note_step_boundary (303-308).
struct LruParams {
    const double* mass_part;  // [n_sel][Gtot]            (mass_src 0)
    const double* mass_cta;   // [H][n_mt][n_sel] per CTA (mass_src 1)
    const int64_t* sel;
    double* freq;       // [U]
    int8_t* hot;        // [U]
    int64_t* hot_list;
    const int32_t* unit_len;
    LruState* lru;
    int64_t* trace;     // [trace_cap][3]
    int64_t n_sel, n_mass, cap, step;
    int Gtot, G, rep, n_mt, H_total, mass_src;
    double decay;
    int64_t bytes_per_token;
};

// Host tier (north star: pinned-host unit store + GPU-resident LRU unit
// cache). Unit pages live in mapped pinned host memory ([U][G][l_bs][d] K,
// V^T pages as in HBM mode); the attention reads them from S device slots.
// k_tier_assign maps this step's retrieved ids to slots (hits keep theirs;
// misses take the least-recently-used slot not read by this layer's previous
// or current step) and k_tier_copy pulls the missing pages over PCIe with
// device-initiated loads, so the lookup -> copy -> attention chain needs no
// host synchronisation and stays graph-capturable.
struct TierParams {
    const int64_t* sel;   // [n_sel] retrieved ids (ascending)
    int32_t* sel_slot;    // [n_sel] out: slot of each
    int32_t* unit_slot;   // [Ucap] slot holding the unit, -1 if not resident
    int64_t* slot_unit;   // [S] unit in the slot, -1 if empty
    int64_t* slot_used;   // [S] (layer step of the last use) + 2, 0 = never used
    int32_t* miss;        // [2][n_sel]: slot and selection index of each unit to copy
    int32_t* miss_n;      // [1]
    int64_t* stats;       // [4] page loads, slot hits, H2D bytes, assignment failures
    const void* host_k;
    const void* host_krot;  // absolute position mode only
    const void* host_v;
    void* slot_k;
    void* slot_krot;
    void* slot_v;
    int64_t n_sel, S, step;
    int64_t page_k, page_v;  // bytes of one unit's K (and K_rot) / V page, all groups
    int kmax;                // grid.x of the copy (max misses)
};

struct EvictParams {
    const void* ring_k;
    const void* ring_krot;
    const void* ring_v;
    const double* P;
    void* init_k;
    void* init_krot;
    void* init_v;
    void* unit_k;
    void* unit_krot;
    void* unit_v;
    double* ev_part;  // [n_evict][Gtot]
    int64_t pop0, n_init, n_evict, R, L, l_I;
    int64_t pend_start, unit0;  // token pend_start belongs to unit id unit0 at offset 0
    int G, Gtot, g0, d, dv, l_bs, absolute;
    VLayout vl;
    // fused single-shard mode: finalize_front + select_representatives in the same launch
    int fused;
    float* unit_scores;   // [U][l_bs]
    void* repr;           // [U][G][r_k][d]
    int32_t* repr_idx;    // [U][r_k]
    const int32_t* unit_len;
    int64_t sel_u0, sel_n;  // units completed by this step
    int r_k;
    unsigned int* done;
    int page_mode;  // 1: units are whole ring pages, copied per unit by k_select (not per token here)
};

struct FinalizeParams {
    const double* ev_part;
    float* unit_scores;  // [U][l_bs]
    int64_t e0, n_evict, pend_start, unit0, L;
    int Gtot, l_bs;
};

struct SelectParams {
    const float* unit_scores;
    const int32_t* unit_len;
    const void* unit_k;
    void* repr;        // [U][G][r_k][d]
    int32_t* repr_idx; // [U][r_k]
    int64_t u0, n_units;
    int G, r_k, d, l_bs;
    // page mode (unit_size 128, units aligned to 128-token ring pages): grid
    // (unit, group); each block copies its unit page K / V (/ K_rot) from the
    // ring and gathers the representative rows from there
    int page_mode, absolute, dv;
    int64_t pos0, R;  // first token of unit u0; ring capacity
    const void* ring_k;
    const void* ring_krot;
    const void* ring_v;
    void* unit_krot;
    void* unit_v;
    VLayout vl;
};

void debug_read_timestamps(unsigned long long* out);

// standalone.cu: the reference's stand-alone operators (attend, TieredStore, ScoreAccumulator)
struct AttendLaunch {
    const void* dev_segs;  // AttendSeg[n_seg] in device memory (attend_pack_seg)
    int n_seg;
    const void *q, *k, *v;
    void* out;
    float* scores;       // [H][lx][n_ctx + lx] (the weights)
    double* mass_part;   // [H][lx][n_seg] scratch
    double* mass;        // [n_seg] or null
    float* qrot;         // [2][H][lx][d] scratch
    float* krot;         // [n_ctx + lx][G][d] scratch
    int64_t lx, n_ctx, start_abs, local_size;
    int H, G, d, dv, absolute, bf16;
    RopeFreqs freqs;
};
size_t attend_seg_bytes();
void attend_pack_seg(void* dst, int idx, const void* keys, const void* values, int64_t start_abs, int64_t n,
                     int64_t col0, int kind);
void attend_run(const AttendLaunch& L, cudaStream_t st);
struct StoreDev {
    LruState* lru;
    int64_t* trace;
    double* freq;
    int8_t* hot;
    int64_t* hot_list;
    int32_t* unit_tokens;
    int* err;
    int64_t n_units, cap, bytes_per_token;
    double decay;
};
void store_qsum(const void* q, int64_t lx, int H, int G, int d, bool bf16, double* qsum, cudaStream_t st);
void store_put_repr(const void* src, void* repr, int64_t u, int n_repr, int r_k, int G, int d, int esz, cudaStream_t st);
void store_book(const StoreDev& s, const int64_t* ids, int64_t n, int64_t step, cudaStream_t st);
void store_update(const StoreDev& s, const int64_t* ids, const double* mass, int64_t n, cudaStream_t st);
void store_enforce(const StoreDev& s, cudaStream_t st);
void store_boundary(const StoreDev& s, cudaStream_t st);
void score_acc_run(const void* q, int64_t lx, int64_t s, const void* keys, int64_t n_pending, int64_t lo, int64_t L,
                   int H, int G, int d, bool bf16, double* sums, int64_t ring0, int64_t cap, cudaStream_t st);
void score_acc_final(const double* sums, int64_t ring0, int64_t cap, int64_t n, int64_t L, float* out, cudaStream_t st);
void score_acc_zero(double* sums, int64_t from, int64_t n, int64_t cap, cudaStream_t st);


// bind the device timeline buffer in each translation unit (kernels.cu, attn_tc.cu, attn_dec.cu)
cudaError_t tl_bind_kernels(const TlBuf& b);
cudaError_t tl_bind_attn_tc(const TlBuf& b);
cudaError_t tl_bind_attn_dec(const TlBuf& b);
cudaError_t tl_bind_lookup(const TlBuf& b);
template <typename T> void launch_prep(const PrepParams& p, cudaStream_t st);
void launch_lookup(const LookupParams& p, int dtype_bf16, cudaStream_t st);
void launch_topk(const TopkParams& p, cudaStream_t st);
// exact top-k (rel desc, id asc) over rel[U] for large U; scratch of topk_multi_scratch(U, k) entries each
// lookup (fused == 2) + exact top-k for a single shard; cand_v / cand_i scratch as above
// returns the number of kernels launched
// between(ctx, st), when given, is issued right after the relevance scan and
// before the top-k kernels (the decode chain puts its front there)
int launch_lookup_topk(LookupParams p, int dtype_bf16, double* cand_v, int64_t* cand_i, cudaStream_t st,
                       void (*between)(void*, cudaStream_t) = nullptr, void* ctx = nullptr);
int64_t topk_multi_scratch(int64_t U, int64_t k);
// lookup.cu: relevance scan + exact top-k (k_m <= 32) in one launch; candidates
// p.cand_v / p.cand_i hold blocks x 32 entries (within topk_multi_scratch)
bool lookup_topk_supported(const LookupParams& p, int dtype_bf16);
int lookup_topk_blocks(int64_t U, int units_per_block);
void launch_lookup_topk_fast(const LookupParams& p, int blocks, cudaStream_t st);
int launch_topk_multi(const double* rel, int64_t U, int64_t k, double* cand_v, int64_t* cand_i, int64_t* sel,
                       cudaStream_t st);
template <typename T> void launch_attn_simt(const AttnParams& p, cudaStream_t st);
void launch_mass(const MassParams& p, cudaStream_t st);
void launch_mass_cta_reduce(const double* mass_cta, double* part, int n_sel, int G, int Gtot, int g0, int rep, int n_mt,
                            cudaStream_t st);
void launch_lru(const LruParams& p, cudaStream_t st);
void launch_tier(const TierParams& p, cudaStream_t st);  // k_tier_assign + k_tier_copy
template <typename T> void launch_evict(const EvictParams& p, cudaStream_t st);
void launch_finalize(const FinalizeParams& p, cudaStream_t st);
template <typename T> void launch_select(const SelectParams& p, cudaStream_t st);

// batched decode stages (grid.z / grid.x = sequence; tab = device array of B params):
// 0 prep (PrepParams), 1 evict (EvictParams, gx = max tokens | G << 32), 2 select
// (SelectParams, gx = max units | G << 32), 3 lookup + top-k (LookupParams,
// gx = max scan blocks), 4 LRU (LruParams), 5 / 6 the scan / the top-k of stage 3
// launched apart (batch chain: the front runs beside the scan), 7 = 6 with the
// top-k's dependents (K4) released after its wait
void launch_decode_batch_stage(int stage, const void* tab, int B, int64_t gx, cudaStream_t st);
int64_t decode_batch_lookup_blocks(int64_t U);
// decode front (one token): prep + eviction in one launch; batched: tab = B x {PrepParams, EvictParams}
bool dec_front_supported(const PrepParams& p);
void launch_dec_front(const PrepParams& p, const EvictParams& ep, cudaStream_t st);
void launch_dec_front_batch(const void* tab, int B, int G, cudaStream_t st, int chain = 0);
size_t dec_front_size();

// standalone select (C ABI infllm_select_representatives)
void launch_select_standalone(const float* scores, const int64_t* lens, int64_t n_units, int64_t unit_len,
                              int64_t r_k, int64_t* idx, cudaStream_t st);
// standalone relevance reduce + top-k (C ABI infllm_lookup)

}  // namespace infllm
