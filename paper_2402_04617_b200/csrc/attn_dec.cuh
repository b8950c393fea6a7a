// attn_dec.cuh — K4 decode attention (l_x = 1), single sequence or batched.
#pragma once

#include "kernels.cuh"

namespace infllm {

constexpr int kDecMaxRep = 8;      // query heads per KV group
constexpr int kDecMaxSplits = 64;  // KV splits per (sequence, group)
constexpr int kDecMaxSel = 128;    // retrieved units (n_lookup)
constexpr int kDecWarps = 8;       // warps per CTA (per-warp unit mass records)

// scratch of one launch: split partials (m, l, O[128]) per head, per-unit
// (mass, running max) records, and per-(sequence, group) arrival counters
// (zero-initialised once; the merging CTA resets its counter)
struct DecScratch {
    float* part;    // [B][G][splits][rep][130]
    float* mass;    // [B][H][max_sel][kDecWarps][2] per-warp (mass, running max)
    unsigned* cnt;  // [B][G]
    int max_sel;
    int pdl;  // 1: the kernel right before K4 on its stream is the lookup (or its top-k), whose
              // inputs were complete before it started: K4 may launch as its programmatic dependent;
              // 2: it is the decode front running as the lookup's dependent: every split waits
    int sep_merge;  // 1: the splits only publish their partials; k_dec_merge (launched right
                    // after K4, its programmatic dependent) merges every (sequence, group, head)
                    // in parallel instead of the group's last split alone
};
inline size_t dec_part_floats(int B, int G, int rep) {
    return static_cast<size_t>(B) * G * kDecMaxSplits * rep * 130;
}

// host: the K4 tensor maps of one layer (6 x CUtensorMap, 64-byte aligned
// host buffer) for its current buffers; unit_rows = unit (or slot) pages x G x 128
void dec_encode_maps(const AttnParams& a, int64_t unit_rows, void* host6);
bool attn_dec_supported(int d, int dv, int unit_size, int rep, bool absolute, int dtype_bf16);
int64_t dec_max_tiles(const AttnParams& a);
void launch_attn_dec(const AttnParams& a, const DecScratch& sc, cudaStream_t st);
// dev_params: B AttnParams in device memory; G KV groups per sequence (all equal)
void launch_attn_dec_batch(const AttnParams* dev_params, int B, int G, int64_t max_tiles, const DecScratch& sc,
                           cudaStream_t st);

}  // namespace infllm
