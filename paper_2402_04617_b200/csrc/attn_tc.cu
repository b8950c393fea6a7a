// attn_tc.cu — tcgen05 / TMEM / TMA attention for the InfLLM window
// (bf16, head_dim = value_dim = 128, 128-token memory units).
#include <cuda.h>

#include <vector>

#include "attn_tc.cuh"
#include "tc_prims.cuh"
#include "tmap.cuh"

__device__ unsigned long long g_attn_ts[64];
namespace infllm {
cudaError_t tl_bind_attn_tc(const TlBuf& b) { return tl_bind_tu(b); }
void debug_read_attn_timestamps(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, g_attn_ts, sizeof(unsigned long long) * 64);
}
}  // namespace infllm
#define ATS(k, jj)                                                                          \
    if (ATTN_TS && blockIdx.x == ATTN_TS_M && blockIdx.y == 0 && (jj) >= ATTN_TS_J0 && (jj) < ATTN_TS_J0 + 16) \
        g_attn_ts[((jj) - ATTN_TS_J0) / 2 * 8 + (k)] = clock64();
#define ATS1(idx)                                                                           \
    if (ATTN_TS && blockIdx.x == ATTN_TS_M && blockIdx.y == 0) g_attn_ts[idx] = clock64();
#ifndef ATTN_CTA_TS
#define ATTN_CTA_TS 0
#endif
// clusters of 2 query heads share each K/V tile by TMA multicast; 4 measured
// slower in-stream (65.6 vs 66.1 us per C2 step): a 4-CTA cluster needs 4 free
// SMs of one GPC at once, which the handoff between consecutive attentions rarely has
#ifndef ATTN_MAX_CLUSTER
#define ATTN_MAX_CLUSTER 2
#endif
#ifndef ATTN_TS_J0
#define ATTN_TS_J0 20
#endif
#ifndef ATTN_TS_M
#define ATTN_TS_M 0
#endif
#ifndef ATTN_TS
#define ATTN_TS 0
#endif


namespace infllm {

using namespace tc;

// ---------------------------------------------------------------------------
// Self-test of the building blocks on one 128x128x128 tile:
//   S = Q K^T      (SS MMA, both operands TMA-loaded K-major SW128)
//   P = bf16(S)    (stored back into TMEM, packed pairs)
//   O = P V        (TS MMA: A = P from TMEM, B = V^T tile K-major)
__global__ void __launch_bounds__(192, 1)
    k_tc_selftest(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                  const __grid_constant__ CUtensorMap tv, float* s_out, float* o_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = smem + 32768;
    uint8_t* sV = smem + 65536;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 98304);
    uint64_t* tma_bar = bars;
    uint64_t* mma_bar = bars + 1;
    uint64_t* p_bar = bars + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0 && lane == 0) {
        mbar_init(tma_bar, 1);
        mbar_init(mma_bar, 1);
        mbar_init(p_bar, 128);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    if (warp == 0 && lane == 0) {
        mbar_expect_tx(tma_bar, 6 * 16384);
        tma_load_2d(&tq, tma_bar, sQ, 0, 0);
        tma_load_2d(&tq, tma_bar, sQ + 16384, 64, 0);
        tma_load_2d(&tk, tma_bar, sK, 0, 0);
        tma_load_2d(&tk, tma_bar, sK + 16384, 64, 0);
        tma_load_2d(&tv, tma_bar, sV, 0, 0);
        tma_load_2d(&tv, tma_bar, sV + 16384, 64, 0);
    }
    const uint32_t idesc = idesc_bf16(128, 128);
    if (warp == 1 && lane == 0) {
        mbar_wait(tma_bar, 0);
        tc_fence_after();
        for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            mma_ss(tbase, sdesc_sw128(smem_u32(sQ) + off), sdesc_sw128(smem_u32(sK) + off), idesc, kk > 0);
        }
        mma_commit(mma_bar);
    }
    if (warp >= 2) {
        const int q = warp & 3;
        const int row = 32 * q + lane;
        mbar_wait(mma_bar, 0);
        tc_fence_after();
        uint32_t pk[64];
        for (int c = 0; c < 4; ++c) {
            uint32_t r[32];
            tmem_ld32(tbase + ((32u * q) << 16) + 32 * c, r);
            tmem_wait_ld();
            for (int j = 0; j < 32; ++j) s_out[row * 128 + 32 * c + j] = __uint_as_float(r[j]);
            for (int j = 0; j < 16; ++j) pk[16 * c + j] = pack_bf16(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
        }
        uint32_t a[32], b[32];
        for (int j = 0; j < 32; ++j) {
            a[j] = pk[j];
            b[j] = pk[32 + j];
        }
        tmem_st32(tbase + ((32u * q) << 16) + 128, a);
        tmem_st32(tbase + ((32u * q) << 16) + 160, b);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(p_bar);
    }
    if (warp == 1 && lane == 0) {
        mbar_wait(p_bar, 0);
        tc_fence_after();
        for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            mma_ts(tbase + 256, tbase + 128 + 8 * kk, sdesc_sw128(smem_u32(sV) + off), idesc, kk > 0);
        }
        mma_commit(mma_bar);
    }
    if (warp >= 2) {
        const int q = warp & 3;
        const int row = 32 * q + lane;
        mbar_wait(mma_bar, 1);
        tc_fence_after();
        for (int c = 0; c < 4; ++c) {
            uint32_t r[32];
            tmem_ld32(tbase + ((32u * q) << 16) + 256 + 32 * c, r);
            tmem_wait_ld();
            for (int j = 0; j < 32; ++j) o_out[row * 128 + 32 * c + j] = __uint_as_float(r[j]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tbase, 512);
}

void tc_selftest(const void* q, const void* k, const void* vt, float* s_out, float* o_out, cudaStream_t st) {
    const CUtensorMap tq = make_tmap_bf16_sw128(q, 128, 128, 128);
    const CUtensorMap tk = make_tmap_bf16_sw128(k, 128, 128, 128);
    const CUtensorMap tv = make_tmap_bf16_sw128(vt, 128, 128, 128);
    const int smem = 98304 + 64 + 1024;
    cudaFuncSetAttribute(k_tc_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_tc_selftest<<<1, 192, smem, st>>>(tq, tk, tv, s_out, o_out);
}

// ---------------------------------------------------------------------------
// InfLLM window attention on tcgen05 (attention.hpp:116-230 semantics).
//
// CTA = (128 query tokens) x (one query head h of KV group g). KV tiles of
// 128 keys in window order: initial tokens, the k_m retrieved units (unit id
// from the device-side lookup result), then the local window + causal chunk
// (ring pages). Per tile: S = Q K^T into TMEM (SS MMA, K-major SW128 operands
// staged by TMA), the softmax warps read S rows from TMEM (one thread per
// query row), apply the clamped-position / causal masks, online softmax in
// the exp2 domain with lazy (thresholded) rescaling of the TMEM O
// accumulator, write P (bf16) back into TMEM over S, and O += P V^T runs as a
// TS MMA (A = P from TMEM, B = V^T page from smem).
// Position modes per tile (SURVEY Appendix A rules 1-3):
//   CLAMP: far tiles (initial / retrieved) and local keys beyond l_L:
//          S = rope(q, l_L) . k_raw
//   ABS  : near keys: S = rope(q, pos_q) . rope(k, pos_k)
//   MIXED: tiles straddling the l_L staircase: both products, selected per
//          element by pos_q - pos_k > l_L (attention.hpp:96-108,179-187).
// Warp roles: warp 0 TMA producer, warp 1 MMA issuer (+TMEM owner),
// warps 2-5 softmax/epilogue (TMEM lane quarter = warp % 4).

constexpr int kKS = 2;                 // K stages (32 KB each: one 128-key x 128-dim tile)
constexpr int kVS = 2;                 // V^T stages (32 KB each: one 128-dim x 128-key page)
constexpr int kTcThreads = 384;        // 3 warpgroups: control (producers + MMA), softmax 0, softmax 1
constexpr uint32_t kStageBytes = 32768;
constexpr uint32_t kQBytes = 65536;    // rope(q, pos) and rope(q, l_L) tiles, K-major SW128
constexpr uint32_t kSmemBytes = kQBytes + (kKS + kVS) * kStageBytes + 256 + 1024;
constexpr int kMassSlots = 16;  // retrieved units whose masses are reduced in-kernel
constexpr int kMaxSel = 128;    // n_lookup limit (infllm_engine_create)
// TMEM columns: softmax warpgroup w owns S_w (P overwrites S in place as
// packed bf16) and its own O_w accumulator; the two partial softmaxes are
// merged in the epilogue.
__device__ __forceinline__ constexpr uint32_t col_s(int w) { return 128u * static_cast<uint32_t>(w); }
__device__ __forceinline__ constexpr uint32_t col_o(int w) { return 256u + 128u * static_cast<uint32_t>(w); }
// fast path: O is col_o(0) for both warpgroups and P_w (packed bf16, 64 columns) sits in col_o(1)'s range
__device__ __forceinline__ constexpr uint32_t col_p(int w) { return 384u + 64u * static_cast<uint32_t>(w); }

enum { SRC_INIT = 0, SRC_UNIT = 1, SRC_RING = 2 };
// CLAMP_PART / ABS_PART: the two halves of a tile straddling the l_L
// staircase, each attended as its own tile with the other half masked
enum { MODE_CLAMP = 0, MODE_ABS = 1, MODE_CLAMP_PART = 2, MODE_ABS_PART = 3 };

__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

struct TcParams {
    CUtensorMap tm_qa, tm_qc, tm_rk, tm_rkr, tm_rv, tm_ik, tm_iv, tm_uk, tm_uv;
    AttnParams a;
    int csize;  // CTAs per cluster: query heads of one KV group sharing every K/V tile
};

struct Tile {
    int src, mode, lo, hi, slot;
    int64_t key0, id;
};

// Window order (engine.hpp:187-221): initial tiles, retrieved units by
// ascending id, then local-window/chunk ring pages; ring pages whose keys
// straddle the l_L distance threshold for this CTA's 128 rows appear twice.
struct TileSched {
    int n_init, n_units, n_near, n_mixed, r_mixed, T;
    int j0;  // split-KV: this CTA's tiles are [j0, j0 + T) of the window's T_all
    int64_t near0, near_end, qp_lo, qp_hi;
    const int32_t* sel;  // retrieved unit ids and lengths, staged in shared memory
    const int32_t* len;
    __device__ int near_mode(const AttnParams& a, int64_t P, int lo, int hi) const {
        const int64_t max_dist = qp_hi - (P + lo);
        const int64_t min_dist = qp_lo - (P + hi - 1);
        return max_dist <= a.L ? MODE_ABS : (min_dist > a.L ? MODE_CLAMP : -1);
    }
    __device__ void near_range(const AttnParams& a, int64_t P, int& lo, int& hi) const {
        lo = static_cast<int>(imax64(0, a.local_start - P));
        hi = static_cast<int>(imin64(128, near_end - P));
    }
    __device__ void init(const AttnParams& a, int m) {
        n_init = static_cast<int>((a.init_len + 127) / 128);
        n_units = a.n_sel;
        const int64_t rows = imin64(a.lx, 128 * m + 128);
        near0 = (a.local_start / 128) * 128;
        near_end = a.s + rows;
        n_near = static_cast<int>((near_end - near0 + 127) / 128);
        qp_lo = a.s + 128 * m;
        qp_hi = a.s + rows - 1;
        // the staircase pages are consecutive (two at most for 128 consecutive rows)
        n_mixed = 0;
        r_mixed = n_near;
        for (int r = 0; r < n_near; ++r) {
            int lo, hi;
            const int64_t P = near0 + 128 * static_cast<int64_t>(r);
            near_range(a, P, lo, hi);
            if (near_mode(a, P, lo, hi) < 0) {
                if (n_mixed == 0) r_mixed = r;
                ++n_mixed;
            }
        }
        const int T_all = n_init + n_units + n_near + n_mixed;
        // split-KV (AttnParams::n_split > 1): a contiguous share of the tile list
        const int ns = a.n_split > 1 ? a.n_split : 1, sp = a.n_split > 1 ? static_cast<int>(blockIdx.z) : 0;
        j0 = static_cast<int>(static_cast<int64_t>(T_all) * sp / ns);
        T = static_cast<int>(static_cast<int64_t>(T_all) * (sp + 1) / ns) - j0;
    }
    __device__ Tile get(const AttnParams& a, int jl) const {
        const int j = jl + j0;
        Tile t;
        t.slot = -1;
        if (j < n_init) {
            t.src = SRC_INIT;
            t.mode = MODE_CLAMP;
            t.key0 = 128 * j;
            t.id = j;
            t.lo = 0;
            t.hi = static_cast<int>(imin64(128, a.init_len - 128 * j));
        } else if (j < n_init + n_units) {
            const int u = j - n_init;
            t.src = SRC_UNIT;
            t.mode = MODE_CLAMP;
            t.id = sel[u];
            t.key0 = 0;
            t.lo = 0;
            t.hi = len[u];
            t.slot = u;
        } else {
            const int jn = j - n_init - n_units;
            int r, part = -1;
            if (jn < r_mixed) {
                r = jn;
            } else if (jn < r_mixed + 2 * n_mixed) {
                r = r_mixed + (jn - r_mixed) / 2;
                part = (jn - r_mixed) % 2;
            } else {
                r = jn - n_mixed;
            }
            const int64_t P = near0 + 128 * static_cast<int64_t>(r);
            t.src = SRC_RING;
            t.key0 = P;
            t.id = 0;
            near_range(a, P, t.lo, t.hi);
            t.mode = part < 0 ? near_mode(a, P, t.lo, t.hi) : (part == 0 ? MODE_CLAMP_PART : MODE_ABS_PART);
        }
        return t;
    }
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 2^x on the FMA/ALU pipes (round-to-nearest split x = n + f, |f| <= 1/2,
// degree-3 polynomial for 2^f, n added to the exponent field). Relative error
// < 1e-4: far below the bf16 rounding P goes through; x is clamped at -127.
__device__ __forceinline__ float ex2_poly(float x) {
    x = fmaxf(x, -127.f);
    const float t = x + 12582912.f;  // 1.5 * 2^23: round(x) in the low mantissa bits
    const float f = x - (t - 12582912.f);
    float p = fmaf(f, 0.0555041086648216f, 0.240226506959101f);
    p = fmaf(p, f, 0.693147180559945f);
    p = fmaf(p, f, 1.0f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

#ifndef ATTN_TURN
#define ATTN_TURN 1
#endif
#ifndef ATTN_POLY_EVERY
#define ATTN_POLY_EVERY 0  // 4: a quarter of the exp2 on the FMA pipe instead of MUFU, 2: half, 0: none
#endif

// Blackwell packed fp32 pairs (FFMA2 / FADD2) and 3-input max (FMNMX3): the
// softmax is issue-bound next to MUFU, so pairs halve its FP32 instruction count
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0,
                                      float c1) {
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mov.b64 rc, {%6, %7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void fadd2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
// ex2_poly on a pair, FP32 work in FFMA2 / FADD2
__device__ __forceinline__ void ex2_poly2(float& y0, float& y1, float x0, float x1) {
    x0 = fmaxf(x0, -127.f);
    x1 = fmaxf(x1, -127.f);
    float t0, t1, r0, r1, f0, f1, p0, p1;
    fadd2(t0, t1, x0, x1, 12582912.f, 12582912.f);
    fadd2(r0, r1, t0, t1, -12582912.f, -12582912.f);
    fadd2(f0, f1, x0, x1, -r0, -r1);
    ffma2(p0, p1, f0, f1, 0.0555041086648216f, 0.0555041086648216f, 0.240226506959101f, 0.240226506959101f);
    ffma2(p0, p1, p0, p1, f0, f1, 0.693147180559945f, 0.693147180559945f);
    ffma2(p0, p1, p0, p1, f0, f1, 1.0f, 1.0f);
    y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
    y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

__device__ __forceinline__ bool clamped_operand(int mode) { return mode == MODE_CLAMP || mode == MODE_CLAMP_PART; }

__device__ __forceinline__ void tmem_ld32_x(uint32_t taddr, float* x) {
    uint32_t r[32];
    tmem_ld32(taddr, r);
    tmem_wait_ld_r(r);
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = __uint_as_float(r[i]);
}

// Warpgroup roles. WG0 (warps 0-3, 56 registers): warp 0 K producer, warp 2
// V^T producer (TMA, multicast across the cluster), warp 1 the P V issuer
// (+TMEM owner), warp 3 the Q K issuer. WG1 / WG2 (224 registers): softmax
// warpgroups 0 / 1 taking alternate KV tiles; thread = one query row (TMEM
// lane = row), all 128 key columns of the tile.
// Fast path (every row's score bound |q| |k|_max <= 60 in the exp2 domain):
// both warpgroups use that bound as a fixed softmax offset, so they share one
// O accumulator, P goes to its own TMEM columns and Q K of tile j + 2 is
// issued as soon as S_j has been read into registers; P V products are issued
// by one thread in tile order, so O is summed in a fixed order (deterministic).
// Slow path: per-warpgroup online max with lazy rescaling of its own O_w, P
// over S_w, merged in the epilogue.
__global__ void __launch_bounds__(kTcThreads, 1) k_attn_tc(const __grid_constant__ TcParams P) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQa = smem;
    uint8_t* sQc = smem + kQBytes / 2;
    uint8_t* sK = smem + kQBytes;
    uint8_t* sV = sK + kKS * kStageBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kVS * kStageBytes);
    uint64_t* q_full = bars;
    uint64_t* k_full = bars + 1;
    uint64_t* k_empty = k_full + kKS;
    uint64_t* v_full = k_empty + kKS;
    uint64_t* v_empty = v_full + kVS;
    uint64_t* s_full = v_empty + kVS;
    uint64_t* p_full = s_full + 2;
    uint64_t* o_done = p_full + 2;
    uint64_t* s_free = o_done + 2;  // fast path: S_w read into registers, Q K of tile j+2 may overwrite it
    uint64_t* flag_bar = s_free + 2;
    uint64_t* o_zero = flag_bar + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_zero + 1);
    int* sSlow = reinterpret_cast<int*>(tmem_slot + 1);
    float* sMassE = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);  // [slot][128 rows]
    float* sMassM = sMassE + kMassSlots * 128;                                         // [slot][128 rows]
    double* sRed = reinterpret_cast<double*>(sMassM + kMassSlots * 128);               // [slot][4]
    float* sML = reinterpret_cast<float*>(sRed + kMassSlots * 4);                      // [wg][m, l][128]
    int32_t* sSel = reinterpret_cast<int32_t*>(sML + 4 * 128);                         // [k_m] unit ids
    int32_t* sLen = sSel + kMaxSel;                                                    // [k_m] unit lengths

    TL_BEGIN();
    if (threadIdx.x == 0) ATS1(56);
    uint64_t cta_t0 = 0;
    if (ATTN_CTA_TS && threadIdx.x == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(cta_t0));
        if (blockIdx.x == 3 && blockIdx.y == 0) {
            g_attn_ts[10] = cta_t0;
            g_attn_ts[11] = clock64();
        }
        atomicMin(reinterpret_cast<unsigned long long*>(g_attn_ts) + 0, cta_t0);
        atomicMax(reinterpret_cast<unsigned long long*>(g_attn_ts) + 1, cta_t0);
    }
    const AttnParams& a = P.a;
    const bool split = a.n_split > 1;
    const bool mass_in_kernel = a.want_mass && a.n_sel <= kMassSlots && !split;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int m = blockIdx.x, h = blockIdx.y, g = h / a.rep;
    TileSched ts;
    ts.init(a, m);
    ts.sel = sSel;
    ts.len = sLen;
    if (threadIdx.x < a.n_sel) {
        const int64_t id = a.sel[threadIdx.x];
        sSel[threadIdx.x] = a.sel_slot ? a.sel_slot[threadIdx.x] : static_cast<int32_t>(id);  // page index
        sLen[threadIdx.x] = a.unit_len[id];
    }

    if (warp == 0 && lane == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < kKS; ++i) {
            mbar_init(k_full + i, 1);
            mbar_init(k_empty + i, P.csize);  // one MMA-commit arrival from each CTA of the cluster
        }
        for (int i = 0; i < kVS; ++i) {
            mbar_init(v_full + i, 1);
            mbar_init(v_empty + i, P.csize);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(s_full + i, 1);
            mbar_init(p_full + i, 4);  // one arrival per warp of the softmax warpgroup
            mbar_init(o_done + i, 1);
            mbar_init(s_free + i, 4);
        }
        mbar_init(flag_bar, 4);
        mbar_init(o_zero, 8);
        *sSlow = a.kmax2 ? 0 : 1;
        fence_barrier_init();
        prefetch_tmap(&P.tm_qa);
        prefetch_tmap(&P.tm_qc);
        prefetch_tmap(&P.tm_rk);
        prefetch_tmap(&P.tm_rkr);
        prefetch_tmap(&P.tm_uk);
        prefetch_tmap(&P.tm_ik);
    }
    if (warp == 2 && lane == 0) {
        prefetch_tmap(&P.tm_rv);
        prefetch_tmap(&P.tm_uv);
        prefetch_tmap(&P.tm_iv);
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // every CTA's barriers are initialised before any multicast targets them
    tc_fence_after();
    if (threadIdx.x == 0) ATS1(57);
    const uint32_t tbase = *tmem_slot;
    const uint32_t idesc = idesc_bf16(128, 128);
    const uint16_t cmask = static_cast<uint16_t>((1u << P.csize) - 1u);
    const int slice = 128 / P.csize;  // K/V rows this CTA fetches for the whole cluster
    const int soff = static_cast<int>(cluster_ctarank()) * slice;
    const int R128 = static_cast<int>(a.R / 128);

    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
        if ((warp == 0 || warp == 2) && lane == 0) {
            // ---------------- TMA producers (K on warp 0, V^T on warp 2)
            const bool is_k = warp == 0;
            uint8_t* ring = is_k ? sK : sV;
            uint64_t* full = is_k ? k_full : v_full;
            uint64_t* empty = is_k ? k_empty : v_empty;
            const int NS = is_k ? kKS : kVS;
            if (is_k) {
                const int qrow = static_cast<int>(h * a.lxp + 128 * m);
                mbar_expect_tx(q_full, kQBytes);
                tma_load_2d(&P.tm_qa, q_full, sQa, 0, qrow);
                tma_load_2d(&P.tm_qa, q_full, sQa + 16384, 64, qrow);
                tma_load_2d(&P.tm_qc, q_full, sQc, 0, qrow);
                tma_load_2d(&P.tm_qc, q_full, sQc + 16384, 64, qrow);
            }
            for (int j = 0; j < ts.T; ++j) {
                const Tile t = ts.get(a, j);
                const CUtensorMap* map;
                int row;
                if (t.src == SRC_INIT) {
                    map = is_k ? &P.tm_ik : &P.tm_iv;
                    row = is_k ? static_cast<int>(g * a.l_I + t.key0) : static_cast<int>((g * a.vl.nI + t.id) * a.dv);
                } else if (t.src == SRC_UNIT) {
                    map = is_k ? &P.tm_uk : &P.tm_uv;
                    row = static_cast<int>((t.id * a.G + g) * (is_k ? 128 : a.dv));
                } else {
                    const int slot = static_cast<int>(t.key0 % a.R);
                    map = is_k ? (clamped_operand(t.mode) ? &P.tm_rk : &P.tm_rkr) : &P.tm_rv;
                    row = is_k ? g * static_cast<int>(a.R) + slot : (g * R128 + slot / 128) * a.dv;
                }
                const int s = j % NS;
                if (j >= NS) mbar_wait(empty + s, ((j / NS) - 1) & 1);
                uint8_t* dst = ring + s * kStageBytes;
                mbar_expect_tx(full + s, kStageBytes);  // all slices, from every CTA of the cluster
                tma_load_2d_mc(map, full + s, dst + soff * 128, 0, row + soff, cmask);
                tma_load_2d_mc(map, full + s, dst + 16384 + soff * 128, 64, row + soff, cmask);
            }
        } else if ((warp == 1 || warp == 3) && lane == 0) {
            // ---------------- MMA issuer. Tile j belongs to softmax warpgroup w = j % 2:
            // S_w = Q K_j^T, then O += P_j V_j. Fast path (score bound known, see
            // the softmax): one shared O, P_w in its own TMEM columns, so Q K of
            // tile j + 2 is issued as soon as S_j has been read. Slow path: O_w per
            // warpgroup (online max), P_w over S_w, Q K of j + 2 after P V of j.
            mbar_wait(q_full, 0);
            tc_fence_after();
            bool fast = false;  // set after the first two Q K (flag_bar)
            const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aQa = smem_u32(sQa), aQc = smem_u32(sQc);
            auto qk = [&](int jj) {
                const Tile t = ts.get(a, jj);
                const int s = jj % kKS;
                mbar_wait(k_full + s, (jj / kKS) & 1);
                tc_fence_after();
                const uint32_t qb = clamped_operand(t.mode) ? aQc : aQa;
                const uint32_t kb = aK + s * kStageBytes;
                const uint32_t d = tbase + col_s(jj & 1);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                    mma_ss(d, sdesc_sw128(qb + off), sdesc_sw128(kb + off), idesc, kk > 0 ? 1u : 0u);
                }
                mma_commit_mc(k_empty + s, cmask);
                mma_commit(s_full + (jj & 1));
            };
            auto pv = [&](int jj) {
                const int w = jj & 1;
                mbar_wait(p_full + w, (jj >> 1) & 1);
                const int s = jj % kVS;
                mbar_wait(v_full + s, (jj / kVS) & 1);
                tc_fence_after();
                const uint32_t vb = aV + s * kStageBytes;
                const uint32_t pcol = tbase + (fast ? col_p(w) : col_s(w));
                const uint32_t d = tbase + (fast ? col_o(0) : col_o(w));
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ts(d, pcol + 8 * kk, sdesc_sw128(vb + (kk >> 2) * 16384 + (kk & 3) * 32), idesc,
                           (fast || jj > 1 || kk > 0) ? 1u : 0u);
                mma_commit_mc(v_empty + s, cmask);
                mma_commit(o_done + w);
            };
            // Three issuers (MMA issue is nearly synchronous: one thread cannot keep
            // the tensor pipe busy): warp 1 every P V in tile order (O sums in a
            // fixed order), warps 2 / 3 the Q K of even / odd tiles, each as soon as
            // its warpgroup has read the previous S. The slow path keeps Q K of
            // tile j + 2 behind P V of tile j on warp 1.
            const bool pv_issuer = warp == 1;
            if (!pv_issuer)
                for (int j = 0; j < ts.T && j < 2; ++j) qk(j);
            mbar_wait(flag_bar, 0);
            fast = *sSlow == 0;
            if (fast) {
                if (pv_issuer) {
                    mbar_wait(o_zero, 0);
                    for (int j = 0; j < ts.T; ++j) {
                        pv(j);
                        if (!(j & 1)) ATS(7, j);
                    }
                } else {
                    for (int j = 0; j + 2 < ts.T; ++j) {
                        mbar_wait(s_free + (j & 1), (j >> 1) & 1);
                        if (!(j & 1)) ATS(5, j);
                        qk(j + 2);
                        if (!(j & 1)) ATS(6, j);
                    }
                }
            } else if (pv_issuer) {
                for (int j = 0; j < ts.T; ++j) {
                    pv(j);
                    if (j + 2 < ts.T) qk(j + 2);
                }
            }
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
        // ---------------- softmax warpgroups: wg takes tiles j = wg, wg + 2, ...
        const int wg = (warp >> 2) - 1;
        const int q4 = warp & 3;
        const int row = 32 * q4 + lane;
        const int64_t i = 128 * static_cast<int64_t>(m) + row;
        const bool row_ok = i < a.lx;
        const int64_t qp = row_ok ? a.s + i : ts.qp_hi;
        const uint32_t tl = tbase + ((32u * q4) << 16);
        const uint32_t tS = tl + col_s(wg), tO = tl + col_o(wg);
        const float sl2 = a.scale * 1.4426950408889634f;
        // Score bound: |s| <= |q| |k|_max (Cauchy-Schwarz, same bf16 values the
        // MMA multiplies; rope keeps norms). With m_row = that bound in the exp2
        // domain, 2^(s*scale*log2e - m_row) lies in [2^(-2 m_row), 1], so for
        // m_row <= 60 a fixed per-row offset replaces the running max exactly
        // (no overflow, no underflow, the softmax is shift-invariant). CTAs with
        // a larger bound anywhere take the online-max path.
        float m_row = INFINITY;
        if (a.kmax2) {
            const uint4* q4p = reinterpret_cast<const uint4*>(static_cast<const bf16*>(a.qa) +
                                                              (static_cast<size_t>(h) * a.lxp + 128 * static_cast<size_t>(m) + row) * 128);
            float n2 = 0.f;
#pragma unroll
            for (int v4 = 0; v4 < 16; ++v4) {
                const uint4 u = q4p[v4];
                const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float lo = __uint_as_float(w4[e] << 16), hi = __uint_as_float(w4[e] & 0xffff0000u);
                    n2 = fmaf(lo, lo, fmaf(hi, hi, n2));
                }
            }
            m_row = sqrtf(n2 * a.kmax2[g]) * (a.scale * 1.4426950408889634f) * 1.001f + 1e-3f;
        }
        if (wg == 0) {
            if (row_ok && !(m_row <= 60.f)) atomicOr(sSlow, 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(flag_bar);
        }
        mbar_wait(flag_bar, 0);
        const bool fast = *sSlow == 0;
        if (fast) {
            // zero the shared O (this warpgroup's 64 value columns of each row)
            uint32_t z[32];
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) z[jj] = 0u;
            tmem_st32(tl + col_o(0) + 64 * wg, z);
            tmem_st32(tl + col_o(0) + 64 * wg + 32, z);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(o_zero);
        }
        if (warp == 4 && lane == 0) ATS1(58);
        const uint32_t tP = fast ? tl + col_p(wg) : tS;  // where P_j goes
        float m_run = fast ? m_row : -INFINITY, l_run = 0.f;
        int n_mine = 0;
        for (int j = wg; j < ts.T; j += 2, ++n_mine) {
            const Tile t = ts.get(a, j);
            // valid key columns [klo, kmax): page range, causal limit, staircase part
            int klo = t.lo, kmax = t.hi;
            if (t.src == SRC_RING) {
                kmax = static_cast<int>(imax64(t.lo, imin64(t.hi, qp - t.key0 + 1)));
                if (t.mode >= MODE_CLAMP_PART) {
                    // columns c < cmax are farther than l_L from this row: clamped product
                    const int cmax = static_cast<int>(imax64(0, imin64(128, qp - a.L - t.key0)));
                    if (t.mode == MODE_CLAMP_PART)
                        kmax = min(kmax, cmax);
                    else
                        klo = max(klo, cmax);
                }
            }
            const bool edge = __any_sync(0xffffffffu, klo > 0 || kmax < 128);
            mbar_wait(s_full + wg, n_mine & 1);
            tc_fence_after();
            if (wg == 0 && warp == 4 && lane == 0) ATS(0, j);
            float x[128];
            {
                uint32_t r0[32], r1[32], r2[32], r3[32];
                tmem_ld32(tS, r0);
                tmem_ld32(tS + 32, r1);
                tmem_ld32(tS + 64, r2);
                tmem_ld32(tS + 96, r3);
                tmem_wait_ld_r(r0);
                tmem_wait_ld_r(r1);
                tmem_wait_ld_r(r2);
                tmem_wait_ld_r(r3);
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) {
                    x[jj] = __uint_as_float(r0[jj]);
                    x[32 + jj] = __uint_as_float(r1[jj]);
                    x[64 + jj] = __uint_as_float(r2[jj]);
                    x[96 + jj] = __uint_as_float(r3[jj]);
                }
            }
            if (fast) {  // S_w is in registers: Q K of tile j + 2 may overwrite it
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(s_free + wg);
            }
            if (wg == 0 && warp == 4 && lane == 0) ATS(1, j);
            if (edge) {
#pragma unroll
                for (int c = 0; c < 128; ++c)
                    if (c < klo || c >= kmax) x[c] = -INFINITY;
            }
            float m_new = m_run;
            if (!fast) {
                float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
                for (int c = 0; c < 128; c += 8) {
                    mx0 = fmax3(mx0, x[c], x[c + 1]);
                    mx1 = fmax3(mx1, x[c + 2], x[c + 3]);
                    mx2 = fmax3(mx2, x[c + 4], x[c + 5]);
                    mx3 = fmax3(mx3, x[c + 6], x[c + 7]);
                }
                m_new = fmaxf(m_run, fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * sl2);
            }
            if (!fast && __any_sync(0xffffffffu, m_new > m_run + 8.0f)) {  // lazy rescale of this warpgroup's O
                const float corr = (m_run == -INFINITY) ? 0.f : ex2(m_run - m_new);
                l_run *= corr;
                if (n_mine > 0) {
                    mbar_wait(o_done + wg, (n_mine - 1) & 1);  // the previous P V into O_wg is complete
                    tc_fence_after();
#pragma unroll
                    for (int c4 = 0; c4 < 4; ++c4) {
                        uint32_t r[32];
                        tmem_ld32(tO + 32 * c4, r);
                        tmem_wait_ld_r(r);
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) r[jj] = __float_as_uint(__uint_as_float(r[jj]) * corr);
                        tmem_st32(tO + 32 * c4, r);
                    }
                    tmem_wait_st();
                }
                m_run = m_new;
            }
            // p = 2^(s * scale * log2e - m): one FFMA + one exp2 per score
            const float neg = (m_run == -INFINITY) ? 0.f : -m_run;
            // the exp sections of the two warpgroups take turns (named barriers 3/4):
            // they share the MUFU pipes of every SMSP, so overlapping them only
            // stretches both, while alternating keeps the tensor pipe fed
            if (ATTN_TURN && j > 0) asm volatile("bar.sync %0, 256;" ::"r"(3 + wg) : "memory");
            if (wg == 0 && warp == 4 && lane == 0) ATS(2, j);
            if (fast && n_mine > 0) {  // P_w is free once the previous P V of this warpgroup completed
                mbar_wait(o_done + wg, (n_mine - 1) & 1);
                tc_fence_after();
            }
            float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t pk[16];
#pragma unroll
                for (int c = 32 * ch; c < 32 * ch + 32; c += 4) {
                    ffma2(x[c], x[c + 1], x[c], x[c + 1], sl2, sl2, neg, neg);
                    ffma2(x[c + 2], x[c + 3], x[c + 2], x[c + 3], sl2, sl2, neg, neg);
                    x[c] = ex2(x[c]);
                    x[c + 1] = ex2(x[c + 1]);
                    if ((ATTN_POLY_EVERY == 4 && (c & 4)) || ATTN_POLY_EVERY == 2) {
                        ex2_poly2(x[c + 2], x[c + 3], x[c + 2], x[c + 3]);  // every 4th pair: FMA pipe
                    } else {
                        x[c + 2] = ex2(x[c + 2]);
                        x[c + 3] = ex2(x[c + 3]);
                    }
                    fadd2(s0, s1, s0, s1, x[c], x[c + 1]);
                    fadd2(s2, s3, s2, s3, x[c + 2], x[c + 3]);
                    pk[(c - 32 * ch) / 2] = pack_bf16(x[c], x[c + 1]);
                    pk[(c - 32 * ch) / 2 + 1] = pack_bf16(x[c + 2], x[c + 3]);
                }
                tmem_st16(tP + 16 * ch, pk);  // keys 32*ch.. packed two per column
            }
            if (ATTN_TURN && j + 1 < ts.T) asm volatile("bar.arrive %0, 256;" ::"r"(4 - wg) : "memory");
            if (wg == 0 && warp == 4 && lane == 0) ATS(3, j);
            const float rs = (s0 + s1) + (s2 + s3);
            l_run += rs;
            if (t.slot >= 0 && a.want_mass) {
                if (mass_in_kernel) {
                    sMassE[t.slot * 128 + row] = row_ok ? rs : 0.f;
                    sMassM[t.slot * 128 + row] = m_run;
                } else if (row_ok) {
                    const int64_t o = (static_cast<int64_t>(h) * a.lx + i) * a.n_sel + t.slot;
                    a.mass_e[o] = rs;
                    a.mass_m[o] = m_run * 0.6931471805599453f;
                }
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full + wg);
            if (wg == 0 && warp == 4 && lane == 0) ATS(4, j);
        }
        // ---------------- epilogue: merge the two partial softmaxes, O / l -> bf16
        sML[(wg * 2) * 128 + row] = m_run;
        sML[(wg * 2 + 1) * 128 + row] = l_run;
        // both accumulators complete: the last P V of each warpgroup
        const int n0 = (ts.T + 1) / 2, n1 = ts.T / 2;
        if (n0 > 0) mbar_wait(o_done, (n0 - 1) & 1);
        if (n1 > 0) mbar_wait(o_done + 1, (n1 - 1) & 1);
        tc_fence_after();
        if (warp == 4 && lane == 0) ATS1(59);
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (warp == 4 && lane == 0) ATS1(53);
        const float m0 = sML[row], l0 = sML[128 + row], m1 = sML[256 + row], l1 = sML[384 + row];
        const float mf = fmaxf(m0, m1);
        const float a0 = l0 > 0.f ? ex2(m0 - mf) : 0.f;
        const float a1 = l1 > 0.f ? ex2(m1 - mf) : 0.f;
        const float lf = fast ? l0 + l1 : l0 * a0 + l1 * a1;
        const float inv = split ? 1.f : 1.f / lf;  // split-KV: unnormalised partials, merged by k_attn_merge
        if (a.inv_violations && row_ok && wg == 0 && !split && !(lf > 0.f && isfinite(lf) && isfinite(inv)))
            atomicAdd(a.inv_violations, 1ull);  // check_softmax (engine.hpp:361-371)
        if (split && row_ok && wg == 0) {
            float* ml = a.split_ml + ((static_cast<int64_t>(blockIdx.z) * a.H + h) * a.lxp + i) * 2;
            ml[0] = mf;
            ml[1] = lf;
        }
        // fast path: one O holding both warpgroups' sums, both at the same fixed offset
        const float w0 = fast ? inv : a0 * inv, w1 = fast ? 0.f : a1 * inv;
        // warpgroup wg writes value dims [64 wg, 64 wg + 64)
        bf16* out = static_cast<bf16*>(a.out) + (i * a.H + h) * a.dv + 64 * wg;
        float* pout = split ? a.split_o + ((static_cast<int64_t>(blockIdx.z) * a.H + h) * a.lxp + i) * 128 + 64 * wg
                            : nullptr;
#pragma unroll
        for (int c4 = 0; c4 < 2; ++c4) {
            const int col = 64 * wg + 32 * c4;
            uint32_t r0[32], r1[32];
            tmem_ld32(tl + col_o(0) + col, r0);
            if (!fast) tmem_ld32(tl + col_o(1) + col, r1);  // fast path: col_o(1) holds P, one shared O
            tmem_wait_ld_r(r0);
            if (!fast) tmem_wait_ld_r(r1);
            if (row_ok && split) {
#pragma unroll
                for (int jj = 0; jj < 32; jj += 4) {
                    float4 o4;
                    o4.x = w0 != 0.f ? __uint_as_float(r0[jj]) * w0 : 0.f;
                    o4.y = w0 != 0.f ? __uint_as_float(r0[jj + 1]) * w0 : 0.f;
                    o4.z = w0 != 0.f ? __uint_as_float(r0[jj + 2]) * w0 : 0.f;
                    o4.w = w0 != 0.f ? __uint_as_float(r0[jj + 3]) * w0 : 0.f;
                    if (w1 != 0.f) {
                        o4.x += __uint_as_float(r1[jj]) * w1;
                        o4.y += __uint_as_float(r1[jj + 1]) * w1;
                        o4.z += __uint_as_float(r1[jj + 2]) * w1;
                        o4.w += __uint_as_float(r1[jj + 3]) * w1;
                    }
                    *reinterpret_cast<float4*>(pout + 32 * c4 + jj) = o4;
                }
            } else if (row_ok) {
                uint32_t wv[16];
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                    // an accumulator that saw no tile holds garbage: weight 0 must not meet NaN
                    const float o0a = w0 != 0.f ? __uint_as_float(r0[2 * jj]) * w0 : 0.f;
                    const float o0b = w0 != 0.f ? __uint_as_float(r0[2 * jj + 1]) * w0 : 0.f;
                    const float o1a = w1 != 0.f ? __uint_as_float(r1[2 * jj]) * w1 : 0.f;
                    const float o1b = w1 != 0.f ? __uint_as_float(r1[2 * jj + 1]) * w1 : 0.f;
                    wv[jj] = pack_bf16(o0a + o1a, o0b + o1b);
                }
                uint4* dst = reinterpret_cast<uint4*>(out + 32 * c4);
#pragma unroll
                for (int v4 = 0; v4 < 4; ++v4)
                    dst[v4] = make_uint4(wv[4 * v4], wv[4 * v4 + 1], wv[4 * v4 + 2], wv[4 * v4 + 3]);
            }
        }
        if (warp == 4 && lane == 0) ATS1(54);
        if (mass_in_kernel) {
            // per-unit attention mass of this CTA's rows: sum_rows e_u 2^(m_u - m) / l
            // (engine.hpp:271-283) in fp64. Warpgroup w reduces units 8w..8w+7: each
            // lane holds its row's 8 values, a transposing butterfly (masks 16, 8, 4,
            // then 2, 1) leaves lane l with one unit's warp sum; quarters are added
            // in order 0..3. Fixed order, so bitwise reproducible.
            double v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int u = 8 * wg + k;
                const float e = u < a.n_sel ? sMassE[u * 128 + row] : 0.f;
                const float mu = u < a.n_sel ? sMassM[u * 128 + row] : 0.f;
                v[k] = (row_ok && e > 0.f) ? static_cast<double>(e * ex2(mu - mf) * inv) : 0.0;
            }
#pragma unroll
            for (int lvl = 0; lvl < 3; ++lvl) {
                const int mask = 16 >> lvl, half = 4 >> lvl;
                const bool upper = (lane & mask) != 0;
#pragma unroll
                for (int k = 0; k < half; ++k) {
                    const double send = upper ? v[k] : v[k + half];
                    const double keep = upper ? v[k + half] : v[k];
                    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
                }
            }
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
            const int slot = 8 * wg + ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
            if ((lane & 3) == 0) sRed[slot * 4 + q4] = v[0];
            asm volatile("bar.sync 1, 256;" ::: "memory");
            const int tid = threadIdx.x - 128;
            if (tid < a.n_sel) {
                const double* r4 = sRed + tid * 4;
                a.mass_cta[(static_cast<int64_t>(h) * gridDim.x + m) * a.n_sel + tid] = ((r4[0] + r4[1]) + r4[2]) + r4[3];
            }
        } else if (row_ok && a.want_mass && wg == 0 && !split) {
            a.row_m[static_cast<int64_t>(h) * a.lx + i] = mf * 0.6931471805599453f;
            a.row_l[static_cast<int64_t>(h) * a.lx + i] = lf;
        }
    }
    tc_fence_before();
    if (threadIdx.x == 128) ATS1(60);
    __syncthreads();
    if (threadIdx.x == 128) ATS1(61);
    cluster_sync();  // no CTA leaves while cluster peers may still signal its barriers
    if (threadIdx.x == 128) ATS1(62);
    if (ATTN_CTA_TS && threadIdx.x == 0) {
        uint64_t t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        atomicMin(reinterpret_cast<unsigned long long*>(g_attn_ts) + 2, t1);
        atomicMax(reinterpret_cast<unsigned long long*>(g_attn_ts) + 3, t1);
        atomicMax(reinterpret_cast<unsigned long long*>(g_attn_ts) + 4, t1 - cta_t0);
        atomicMin(reinterpret_cast<unsigned long long*>(g_attn_ts) + 5, t1 - cta_t0);
        atomicAdd(reinterpret_cast<unsigned long long*>(g_attn_ts) + 6, t1 - cta_t0);
        atomicAdd(reinterpret_cast<unsigned long long*>(g_attn_ts) + 7, 1ull);
        if (blockIdx.x == 3 && blockIdx.y == 0) {
            g_attn_ts[12] = t1;
            g_attn_ts[13] = clock64();
        }
    }
    if (warp == 1) tmem_dealloc(tbase, 512);
    TL_END(TL_ATTN);
}

bool attn_tc_masses_in_kernel(int n_sel) { return n_sel <= kMassSlots; }

// split-KV merge: out = sum_s O_s 2^(m_s - M) / sum_s l_s 2^(m_s - M), splits in
// order (deterministic); the row's (M ln 2, L) feed the unit-mass reduction
// (k_mass). Fast-path splits share the fixed offset, so the weights are 1.
__global__ void __launch_bounds__(128) k_attn_merge(AttnParams a) {
    const int64_t i = blockIdx.x;
    const int h = blockIdx.y, c = threadIdx.x;
    const int S = a.n_split;
    const float* ml = a.split_ml + (static_cast<int64_t>(h) * a.lxp + i) * 2;
    const int64_t sstride = static_cast<int64_t>(a.H) * a.lxp;
    float M = -INFINITY;
    for (int sp = 0; sp < S; ++sp) {
        const float l = ml[sp * sstride * 2 + 1];
        if (l > 0.f) M = fmaxf(M, ml[sp * sstride * 2]);
    }
    float L = 0.f, o = 0.f;
    for (int sp = 0; sp < S; ++sp) {
        const float l = ml[sp * sstride * 2 + 1];
        if (!(l > 0.f)) continue;
        const float w = ex2(ml[sp * sstride * 2] - M);
        L = fmaf(l, w, L);
        o = fmaf(a.split_o[((sp * sstride) + static_cast<int64_t>(h) * a.lxp + i) * 128 + c], w, o);
    }
    const float inv = 1.f / L;
    static_cast<bf16*>(a.out)[(i * a.H + h) * a.dv + c] = __float2bfloat16_rn(o * inv);
    if (c == 0) {
        if (a.inv_violations && !(L > 0.f && isfinite(L) && isfinite(inv))) atomicAdd(a.inv_violations, 1ull);
        if (a.want_mass) {
            a.row_m[static_cast<int64_t>(h) * a.lx + i] = M * 0.6931471805599453f;
            a.row_l[static_cast<int64_t>(h) * a.lx + i] = L;
        }
    }
}

bool attn_tc_supported(int d, int dv, int unit_size, bool absolute) {
    return d == 128 && dv == 128 && unit_size == 128 && !absolute;
}

// Tensor maps depend only on buffer pointers/extents: cache them so a step
// costs no host-side re-encoding (a handful of layers x engines in flight).
struct TmapKey {
    const void* p[9];
    uint64_t n[4];
    bool operator==(const TmapKey& o) const {
        for (int i = 0; i < 9; ++i)
            if (p[i] != o.p[i]) return false;
        for (int i = 0; i < 4; ++i)
            if (n[i] != o.n[i]) return false;
        return true;
    }
};
struct TmapEntry {
    TmapKey key;
    CUtensorMap m[9];
};

int launch_attn_tc(const AttnParams& a, cudaStream_t st) {
    TcParams P;
    P.a = a;
    const uint64_t R = static_cast<uint64_t>(a.R);
    const uint64_t ucap = static_cast<uint64_t>(a.unit_cap > 0 ? a.unit_cap : 1);
    int csize = 1;
    while (csize * 2 <= ATTN_MAX_CLUSTER && a.rep % (csize * 2) == 0) csize *= 2;
    const int box = 128 / csize;
    TmapKey key{{a.qa, a.qc, a.ring_k, a.ring_krot, a.ring_v, a.init_k, a.init_v, a.unit_k, a.unit_v},
                {static_cast<uint64_t>(a.H) * a.lxp, a.G * R, ucap,
                 static_cast<uint64_t>(a.G) * a.l_I + (static_cast<uint64_t>(csize) << 48)}};
    static thread_local std::vector<TmapEntry> cache;
    TmapEntry* hit = nullptr;
    for (auto& e : cache)
        if (e.key == key) hit = &e;
    if (!hit) {
        if (cache.size() >= 32) cache.erase(cache.begin());
        TmapEntry e;
        e.key = key;
        e.m[0] = make_tmap_bf16_sw128(a.qa, static_cast<uint64_t>(a.H) * a.lxp, 128, 128);
        e.m[1] = make_tmap_bf16_sw128(a.qc, static_cast<uint64_t>(a.H) * a.lxp, 128, 128);
        e.m[2] = make_tmap_bf16_sw128(a.ring_k, a.G * R, 128, box);
        e.m[3] = make_tmap_bf16_sw128(a.ring_krot, a.G * R, 128, box);
        e.m[4] = make_tmap_bf16_sw128(a.ring_v, a.G * (R / 128) * 128, 128, box);
        e.m[5] = make_tmap_bf16_sw128(a.init_k, static_cast<uint64_t>(a.G) * a.l_I, 128, box);
        e.m[6] = make_tmap_bf16_sw128(a.init_v, static_cast<uint64_t>(a.G) * a.vl.nI * 128, 128, box);
        e.m[7] = make_tmap_bf16_sw128(a.unit_k ? a.unit_k : a.ring_k, a.unit_k ? ucap * a.G * 128 : 128, 128, box);
        e.m[8] = make_tmap_bf16_sw128(a.unit_v ? a.unit_v : a.ring_v, a.unit_v ? ucap * a.G * 128 : 128, 128, box);
        cache.push_back(e);
        hit = &cache.back();
    }
    P.tm_qa = hit->m[0];
    P.tm_qc = hit->m[1];
    P.tm_rk = hit->m[2];
    P.tm_rkr = hit->m[3];
    P.tm_rv = hit->m[4];
    P.tm_ik = hit->m[5];
    P.tm_iv = hit->m[6];
    P.tm_uk = hit->m[7];
    P.tm_uv = hit->m[8];
    P.csize = csize;
    const uint32_t smem = kSmemBytes + kMassSlots * 2 * 128 * sizeof(float) + kMassSlots * 4 * sizeof(double) +
                          4 * 128 * sizeof(float) + 2 * kMaxSel * sizeof(int32_t);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_attn_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    dim3 grid(static_cast<unsigned>((a.lx + 127) / 128), a.H, a.n_split > 1 ? a.n_split : 1);
    // highest launch priority: the side-stream kernels of the next step must
    // not hold SMs the attention CTAs (one per SM) are waiting for
    static int prio_hi = 1;
    if (prio_hi > 0) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        prio_hi = hi;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kTcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute la[2];
    la[0].id = cudaLaunchAttributePriority;
    la[0].val.priority = prio_hi;
    la[1].id = cudaLaunchAttributeClusterDimension;  // the csize query heads of one KV group
    la[1].val.clusterDim.x = 1;
    la[1].val.clusterDim.y = static_cast<unsigned>(csize);
    la[1].val.clusterDim.z = 1;
    cfg.attrs = la;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, k_attn_tc, P);
    if (a.n_split > 1) {
        k_attn_merge<<<dim3(static_cast<unsigned>(a.lx), a.H), 128, 0, st>>>(a);
        return 2;
    }
    return 1;
}

}  // namespace infllm
