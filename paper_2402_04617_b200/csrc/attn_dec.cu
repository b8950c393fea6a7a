// attn_dec.cu — K4: decode attention (l_x = 1) for one or a batch of
// sequences, bf16, d = d_v = 128, 128-token units (V^T pages).
//
// Reference: attend (attention.hpp:116-230) with a single query row, as
// StreamEngine::decode_step runs it (engine.hpp:100-103): window = [initial |
// retrieved units | local window | the token itself], clamped positions
// (far keys: rope(q, l_L) . k_raw, near keys: rope(q, pos) . rope(k, pos),
// attention.hpp:165-201), scale 1/sqrt(d), max-subtracted softmax, plus the
// per-unit attention masses for the LRU (engine.hpp:271-283).
//
// One query row reads every key once: the step is HBM-bound (K + V^T of the
// ~6.3K-key window = 25.7 MB per C2 sequence), so it is split-KV
// ("flash-decoding") on CUDA cores: grid (splits, KV groups, sequences); a
// CTA streams a contiguous run of 128-key tiles of its (sequence, group) and
// keeps an online softmax for the group's query heads; the last CTA of a
// (sequence, group) merges the splits (log-sum-exp) and finishes the masses.
#include "attn_dec.cuh"
#include "tc_prims.cuh"
#include "tmap.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>

namespace infllm {

namespace {

constexpr int kW = kDecWarps;  // warps: 16 keys each for S = QK^T and for P V
constexpr int kThr = 32 * kW;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct DecTile {
    int src;  // 0 init, 1 unit, 2 ring
    int lo, hi;
    int64_t key0, page;
};

// window tile t (window order, engine.hpp:187-221)
__device__ __forceinline__ DecTile dec_tile(const AttnParams& a, int t, int n_init, int64_t near0,
                                            const int32_t* s_page, const int32_t* s_len) {
    DecTile r;
    if (t < n_init) {
        r.src = 0;
        r.key0 = 128 * static_cast<int64_t>(t);
        r.page = t;
        r.lo = 0;
        r.hi = static_cast<int>(min(static_cast<int64_t>(128), a.init_len - r.key0));
    } else if (t < n_init + a.n_sel) {
        const int u = t - n_init;
        r.src = 1;
        r.key0 = 0;
        r.page = s_page[u];  // unit page (or host-tier cache slot), staged in shared memory
        r.lo = 0;
        r.hi = s_len[u];
    } else {
        const int64_t P = near0 + 128 * static_cast<int64_t>(t - n_init - a.n_sel);
        r.src = 2;
        r.key0 = P;
        r.page = 0;
        r.lo = static_cast<int>(max(static_cast<int64_t>(0), a.local_start - P));
        r.hi = static_cast<int>(min(static_cast<int64_t>(128), a.s + 1 - P));
    }
    return r;
}

__device__ __forceinline__ int dec_tiles(const AttnParams& a, int& n_init, int64_t& near0) {
    n_init = static_cast<int>((a.init_len + 127) / 128);
    near0 = (a.local_start / 128) * 128;
    return n_init + a.n_sel + static_cast<int>((a.s + 1 - near0 + 127) / 128);
}

// shared-memory stage of one 128-key tile: K rows and V^T rows with 272-byte
// rows (256 + 16 pad: ldmatrix conflict-free). Decode keys of the ring are
// always within l_L of the query (the local window holds l_L tokens), so a
// ring page is attended with rotated keys only; init / unit pages are far
// (clamped: rope(q, l_L) . k_raw, attention.hpp:165-173).
// stage = K tile then V^T tile, each two TMA boxes of [128 rows][64 cols] bf16
// with the 128-byte swizzle (16-byte chunk c of row r at chunk c ^ (r & 7))
constexpr int kBoxB = 128 * 128;    // 16 KB
constexpr int kMatB = 2 * kBoxB;    // 32 KB
constexpr int kStageB = 2 * kMatB;
constexpr int kStages = 3;
constexpr int kDecSmem = kStages * kStageB + 1024;  // + alignment slack (SW128 boxes: 1024 B)

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
// D += A(16x16 bf16; rows >= 8 are zero: the <= 8 query heads of a group) * B(16x8)
__device__ __forceinline__ void mma16816(float* d, uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
using tc::pack_bf16;

// tile `tl` into stage `sb`: four TMA boxes (K cols 0-63 / 64-127, V^T keys
// 0-63 / 64-127) issued by one thread, completion counted in bytes on `bar`.
// Tensor maps (device memory, one set per engine): 0 init K, 1 init V^T,
// 2 unit K, 3 unit V^T, 4 ring K_rot, 5 ring V^T.
__device__ __forceinline__ void dec_load(const AttnParams& a, const DecTile& tl, int g, uint8_t* sb, uint64_t* bar) {
    if (threadIdx.x != 0) return;
    const CUtensorMap* tm = static_cast<const CUtensorMap*>(a.dec_maps);
    int mk, mv, rk, rv;
    if (tl.src == 0) {
        mk = 0, mv = 1;
        rk = static_cast<int>(g * a.l_I + tl.key0);
        rv = static_cast<int>((g * a.vl.nI + tl.page) * 128);
    } else if (tl.src == 1) {
        mk = 2, mv = 3;
        rk = rv = static_cast<int>((tl.page * a.G + g) * 128);
    } else {
        const int64_t sl = tl.key0 % a.R;
        mk = 4, mv = 5;
        rk = static_cast<int>(g * a.R + sl);
        rv = static_cast<int>((g * (a.R / 128) + sl / 128) * 128);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the stage was last read by ldmatrix
    tc::mbar_expect_tx(bar, kStageB);
    tc::tma_load_2d(tm + mk, bar, sb, 0, rk);
    tc::tma_load_2d(tm + mk, bar, sb + kBoxB, 64, rk);
    tc::tma_load_2d(tm + mv, bar, sb + kMatB, 0, rv);
    tc::tma_load_2d(tm + mv, bar, sb + kMatB + kBoxB, 64, rv);
}

__device__ __forceinline__ void dec_body(const AttnParams& a, const DecScratch& sc, int b, int x, int nsplit,
                                         unsigned long long& mark) {
    extern __shared__ __align__(1024) uint8_t dsm_raw[];
    uint8_t* dsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ float sred[kW][kDecMaxRep], sl_red[kW][kDecMaxRep];
    __shared__ float s_m[kDecMaxRep], s_M[kDecMaxRep], s_L[kDecMaxRep];
    __shared__ bool s_last;
    __shared__ int32_t s_page[kDecMaxSel], s_len[kDecMaxSel];
    __shared__ __align__(8) uint64_t s_bar[kStages];

    const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
    const int gq = lane >> 2, tq = lane & 3;  // mma fragment row (query head) / column pair
    int n_init;
    int64_t near0;
    const int T = dec_tiles(a, n_init, near0);
    const int tps = (T + nsplit - 1) / nsplit;
    const int t0 = x * tps, t1 = min(T, t0 + tps);
    const bool units = t0 < n_init + a.n_sel && t1 > n_init;
    // a split attending retrieved units waits for the lookup grid when launched as its
    // programmatic dependent (no-op otherwise); behind the decode chain's front
    // (pdl 2) every split waits: the front writes this token's rotated query and ring row
    const int g = blockIdx.y, rep = a.rep;
    if (threadIdx.x == 0) {  // before any wait: the maps were written before this launch
        for (int i = 0; i < kStages; ++i) tc::mbar_init(&s_bar[i], 1);
        tc::fence_barrier_init();
        // the maps are rewritten in place when a buffer of the layer moves
        for (int i = 0; i < 6; ++i) tc::acquire_tmap(static_cast<const CUtensorMap*>(a.dec_maps) + i);
    }
    unsigned pre = 0;  // stages whose tile was requested before the wait
    if (units || sc.pdl == 2) {
        // first tiles that neither the front nor the lookup writes or selects (initial
        // pages; ring pages wholly before this token, whose page the front writes) are
        // requested now, so their loads overlap the wait (thread 0 issues: its own
        // barrier initialisation is ordered before them)
        for (int st = 0; st < kStages - 1; ++st) {
            const int t = t0 + st;
            if (t >= t1 || (t >= n_init && t < n_init + a.n_sel)) continue;
            const DecTile tl = dec_tile(a, t, n_init, near0, s_page, s_len);
            if (tl.src == 0 || a.s - tl.key0 >= 128) {
                dec_load(a, tl, g, dsm + st * kStageB, &s_bar[st]);
                pre |= 1u << st;
            }
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    if (units) {
        for (int u = tid; u < a.n_sel; u += kThr) {  // the retrieved units' pages and lengths
            const int64_t id = a.sel[u];
            s_page[u] = a.sel_slot ? a.sel_slot[u] : static_cast<int32_t>(id);
            s_len[u] = a.unit_len[id];
        }
    }
    __syncthreads();
    const float sl2 = a.scale * kLog2e;
    TL_MARK(50, mark);  // dependencies met, stages initialised
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(dsm));  // 1024-aligned

    for (int st = 0; st < kStages - 1; ++st)  // prefetch the first tiles
        if (t0 + st < t1 && !((pre >> st) & 1u))
            dec_load(a, dec_tile(a, t0 + st, n_init, near0, s_page, s_len), g, dsm + st * kStageB, &s_bar[st]);
    // query fragments (A operand, row = query head of the group, zero beyond rep):
    // rope(q, pos) for ring pages, rope(q, l_L) for init / unit pages; 8 k-steps of 16 dims
    uint32_t qa[8][2], qc[8][2];
    {
        const bool hv = gq < rep;
        const int64_t qrow = static_cast<int64_t>(g * rep + (hv ? gq : 0)) * a.lxp * 128;
        const bf16* pa = static_cast<const bf16*>(a.qa) + qrow;
        const bf16* pc = static_cast<const bf16*>(a.qc) + qrow;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            qa[kk][0] = hv ? *reinterpret_cast<const uint32_t*>(pa + 16 * kk + 2 * tq) : 0u;
            qa[kk][1] = hv ? *reinterpret_cast<const uint32_t*>(pa + 16 * kk + 8 + 2 * tq) : 0u;
            qc[kk][0] = hv ? *reinterpret_cast<const uint32_t*>(pc + 16 * kk + 2 * tq) : 0u;
            qc[kk][1] = hv ? *reinterpret_cast<const uint32_t*>(pc + 16 * kk + 8 + 2 * tq) : 0u;
        }
    }
    float mw = -INFINITY;  // this warp's running max of row gq (log2 domain): online softmax per warp
    float o[16][4];  // O fragments of this warp's keys: 16 n-tiles of 8 dims (rows gq)
#pragma unroll
    for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float lsum = 0.f;  // this thread's share of the softmax denominator of row gq
    const int k0 = 16 * warp;  // this warp's keys of every tile

    for (int t = t0; t < t1; ++t) {
        const int st = (t - t0) % kStages;
        const DecTile tl = dec_tile(a, t, n_init, near0, s_page, s_len);
        __syncthreads();  // every warp is done with tile t-1
        // refill the stage of tile t-1 with tile t+kStages-1 (one barrier per tile)
        if (t + kStages - 1 < t1) {
            const int sn = (t - t0 + kStages - 1) % kStages;
            dec_load(a, dec_tile(a, t + kStages - 1, n_init, near0, s_page, s_len), g, dsm + sn * kStageB, &s_bar[sn]);
        }
        tc::mbar_wait(&s_bar[st], static_cast<uint32_t>(((t - t0) / kStages) & 1));
        const uint32_t sk = sbase + st * kStageB, sv = sk + kMatB;
        // ---- S = Q K^T for keys k0..k0+15 (2 n-tiles) ----
        float s2[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        const bool far = tl.src != 2;
        const int krow = k0 + (lane & 7) + ((lane >> 4) & 1) * 8, khalf = (lane >> 3) & 1;
        const uint32_t kbase = sk + krow * 128;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            uint32_t b0, b1, b2, b3;
            const int chunk = 2 * (kk & 3) + khalf;  // 16-byte chunk within the 128-byte swizzled row
            ldsm_x4(kbase + (kk >> 2) * kBoxB + ((chunk ^ (krow & 7)) << 4), b0, b1, b2, b3);
            const uint32_t A0 = far ? qc[kk][0] : qa[kk][0], A2 = far ? qc[kk][1] : qa[kk][1];
            mma16816(s2[0], A0, A2, b0, b1);
            mma16816(s2[1], A0, A2, b2, b3);
        }
        // mask + scale (log2 domain): row gq, key k0 + 8 j + 2 tq + e
        float sv2[2][2];
        float tmax = -INFINITY;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = k0 + 8 * j + 2 * tq + e;
                const float v = (col >= tl.lo && col < tl.hi) ? s2[j][e] * sl2 : -INFINITY;
                sv2[j][e] = v;
                tmax = fmaxf(tmax, v);
            }
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
        const float mn = fmaxf(mw, tmax);
        const float al = mn == -INFINITY ? 1.f : (mw == -INFINITY ? 0.f : ex2f(mw - mn));
        mw = mn;
        float p[2][2], psum = 0.f;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                p[j][e] = sv2[j][e] == -INFINITY ? 0.f : ex2f(sv2[j][e] - mn);
                psum += p[j][e];
            }
        lsum = lsum * al + psum;
        if (tl.src == 1 && a.want_mass) {  // this warp's share of the unit's mass, relative to its running max
            float e2 = psum;
            e2 += __shfl_xor_sync(0xffffffffu, e2, 1);
            e2 += __shfl_xor_sync(0xffffffffu, e2, 2);
            if (tq == 0 && gq < rep) {
                float* mr = sc.mass + (((static_cast<int64_t>(b) * a.H + g * rep + gq) * sc.max_sel + (t - n_init)) * kW + warp) * 2;
                mr[0] = e2;
                mr[1] = mn;
            }
        }
        // ---- O = O alpha + P V over this warp's 16 keys (one k-step; P from the S fragments) ----
        if (__any_sync(0xffffffffu, al != 1.f)) {  // the max moved for some row of this warp
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                o[j][0] *= al;
                o[j][1] *= al;
            }
        }
        const uint32_t A0 = pack_bf16(p[0][0], p[0][1]), A2 = pack_bf16(p[1][0], p[1][1]);
        const int vkey = k0 + ((lane >> 3) & 1) * 8;  // first key of this lane's 8-key chunk
        const int vchunk = (vkey & 63) >> 3;
        const uint32_t vbase = sv + (vkey >> 6) * kBoxB;
#pragma unroll
        for (int jp = 0; jp < 8; ++jp) {
            uint32_t b0, b1, b2, b3;
            const int vrow = 16 * jp + (lane & 7) + ((lane >> 4) & 1) * 8;  // value dim
            ldsm_x4(vbase + vrow * 128 + ((vchunk ^ (vrow & 7)) << 4), b0, b1, b2, b3);
            mma16816(o[2 * jp], A0, A2, b0, b1);
            mma16816(o[2 * jp + 1], A0, A2, b2, b3);
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    TL_MARK(51, mark);  // tiles attended
    // ---- this split's partial (m, l, O) per head: the warps' online softmaxes merged ----
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
    if (tq == 0 && gq < kDecMaxRep) {
        sred[warp][gq] = mw;
        sl_red[warp][gq] = lsum;
    }
    float* so = reinterpret_cast<float*>(dsm);  // [kW][rep][128] (the stages are free now)
    __syncthreads();
    if (tid < rep) {
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kW; ++w) M = fmaxf(M, sred[w][tid]);
        float l = 0.f;
#pragma unroll
        for (int w = 0; w < kW; ++w) {
            const float f = sred[w][tid] == -INFINITY ? 0.f : ex2f(sred[w][tid] - M);
            sred[w][tid] = f;  // the warp's scale factor
            l += sl_red[w][tid] * f;
        }
        s_m[tid] = M;
        s_L[tid] = l;
    }
    if (gq < rep) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            *reinterpret_cast<float2*>(&so[(warp * rep + gq) * 128 + 8 * j + 2 * tq]) = make_float2(o[j][0], o[j][1]);
    }
    __syncthreads();
    const int64_t stride = static_cast<int64_t>(rep) * 130;
    float* part = sc.part + ((static_cast<int64_t>(b) * a.G + g) * nsplit + x) * stride;
    if (tid < rep) {
        part[tid * 130 + 0] = s_m[tid];
        part[tid * 130 + 1] = s_L[tid];
    }
    for (int i = tid; i < rep * 128; i += kThr) {
        const int h = i / 128, c = i % 128;
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < kW; ++w) v = fmaf(so[(w * rep + h) * 128 + c], sred[w][h], v);
        part[h * 130 + 2 + c] = v;
    }
    if (sc.sep_merge) {  // k_dec_merge combines the splits
        TL_MARK(52, mark);  // partial published
        return;
    }
    // ---- the last split of (sequence, group) merges ----
    __threadfence();
    __syncthreads();
    unsigned* cnt = sc.cnt + static_cast<int64_t>(b) * a.G + g;
    if (tid == 0) s_last = atomicAdd(cnt, 1u) == static_cast<unsigned>(nsplit - 1);
    __syncthreads();
    TL_MARK(52, mark);  // partial published
    if (!s_last) {
        if (s_last && tid == 0) *cnt = 0;
        return;
    }
    __threadfence();
    const float* p0 = sc.part + (static_cast<int64_t>(b) * a.G + g) * nsplit * stride;
    __shared__ float s_w[kDecMaxSplits][kDecMaxRep], s_ls[kDecMaxSplits][kDecMaxRep];
    // mass records of the retrieved units, loaded up front (one round trip)
    const bool mass_thread = a.want_mass && a.mass_part && tid < a.n_sel;
    for (int i = tid; i < nsplit * rep; i += kThr) {
        const int xs = i / rep, h = i % rep;
        s_w[xs][h] = __ldcg(p0 + xs * stride + h * 130);
        s_ls[xs][h] = __ldcg(p0 + xs * stride + h * 130 + 1);
    }
    // this thread's O values: (split, head, dim) with dim = tid % 128, heads split over the two halves
    const int c = tid & 127, hh = tid >> 7;
    __syncthreads();
    if (tid < rep) {
        float M = -INFINITY;
        for (int xs = 0; xs < nsplit; ++xs) M = fmaxf(M, s_w[xs][tid]);
        float L = 0.f;
        for (int xs = 0; xs < nsplit; ++xs) {
            const float mx = s_w[xs][tid];
            if (mx != -INFINITY) L += s_ls[xs][tid] * ex2f(mx - M);
        }
        s_M[tid] = M;
        s_L[tid] = L;
        if (a.inv_violations && !(L > 0.f && isfinite(L))) atomicAdd(a.inv_violations, 1ull);  // check_softmax
    }
    __syncthreads();
    for (int i = tid; i < nsplit * rep; i += kThr) {
        const int xs = i / rep, h = i % rep;
        const float mx = s_w[xs][h];
        s_w[xs][h] = mx == -INFINITY ? 0.f : ex2f(mx - s_M[h]) / s_L[h];
    }
    __syncthreads();
    for (int h = hh; h < rep; h += 2) {
        float acc = 0.f;
        for (int x0 = 0; x0 < nsplit; x0 += 32) {
            float ov[32];
#pragma unroll
            for (int u = 0; u < 32; ++u) ov[u] = x0 + u < nsplit ? __ldcg(p0 + (x0 + u) * stride + h * 130 + 2 + c) : 0.f;
#pragma unroll
            for (int u = 0; u < 32; ++u)
                if (x0 + u < nsplit) acc = fmaf(ov[u], s_w[x0 + u][h], acc);
        }
        static_cast<bf16*>(a.out)[static_cast<int64_t>(g * rep + h) * a.dv + c] = __float2bfloat16_rn(acc);
    }
    // masses of the retrieved units: this group's heads' normalised weights of
    // the unit's keys, summed (engine.hpp:271-283; the LRU divides by H)
    if (mass_thread) {
        double msum = 0.0;
        for (int h = 0; h < rep; ++h) {
            const float* mr = sc.mass + ((static_cast<int64_t>(b) * a.H + g * rep + h) * sc.max_sel + tid) * kW * 2;
            float rec[2 * kW];
#pragma unroll
            for (int i = 0; i < 2 * kW; ++i) rec[i] = __ldcg(mr + i);
            float e = 0.f;
#pragma unroll
            for (int w = 0; w < kW; ++w) e += rec[2 * w + 1] == -INFINITY ? 0.f : rec[2 * w] * ex2f(rec[2 * w + 1] - s_M[h]);
            msum += static_cast<double>(e / s_L[h]);
        }
        a.mass_part[static_cast<int64_t>(tid) * a.Gtot + a.g0 + g] = msum;
    }
    if (tid == 0) *cnt = 0;
    TL_MARK(53, mark);  // splits merged (the group's last split)
}

// Split merge as its own launch (sep_merge): block (head h < rep, group, sequence)
// with thread = value dim combines that head's nsplit partials, block h = rep
// the group's retrieved-unit masses; the arithmetic and its order are the last
// split's merge below (max and denominator over splits in order, weights, then
// one fma per split in order), so the outputs are bitwise the same.
__device__ __forceinline__ void dec_merge_body(const AttnParams& a, const DecScratch& sc, int b, int g, int hsel,
                                               int nsplit) {
    const int tid = threadIdx.x, rep = a.rep;
    const int64_t stride = static_cast<int64_t>(rep) * 130;
    const float* p0 = sc.part + (static_cast<int64_t>(b) * a.G + g) * nsplit * stride;
    __shared__ float s_w[kDecMaxSplits][kDecMaxRep], s_ls[kDecMaxSplits][kDecMaxRep];
    __shared__ float s_M[kDecMaxRep], s_L[kDecMaxRep];
    const bool masses = hsel == rep;
    const int h_lo = masses ? 0 : hsel, h_n = masses ? rep : 1;
    for (int i = tid; i < nsplit * h_n; i += blockDim.x) {
        const int xs = i / h_n, h = h_lo + i % h_n;
        s_w[xs][h] = __ldcg(p0 + xs * stride + h * 130);
        s_ls[xs][h] = __ldcg(p0 + xs * stride + h * 130 + 1);
    }
    // this thread's O values (all splits of its dim), issued with the (m, l) loads
    constexpr int kPre = 32;
    float ov[kPre];
    if (!masses) {
#pragma unroll
        for (int u = 0; u < kPre; ++u) ov[u] = u < nsplit ? __ldcg(p0 + u * stride + hsel * 130 + 2 + tid) : 0.f;
    }
    __syncthreads();
    if (tid < h_n) {
        const int h = h_lo + tid;
        float M = -INFINITY;
        for (int xs = 0; xs < nsplit; ++xs) M = fmaxf(M, s_w[xs][h]);
        float L = 0.f;
        for (int xs = 0; xs < nsplit; ++xs) {
            const float mx = s_w[xs][h];
            if (mx != -INFINITY) L += s_ls[xs][h] * ex2f(mx - M);
        }
        s_M[h] = M;
        s_L[h] = L;
        if (!masses && a.inv_violations && !(L > 0.f && isfinite(L))) atomicAdd(a.inv_violations, 1ull);
    }
    __syncthreads();
    if (masses) {  // the group's heads' normalised weights of each unit's keys, summed (engine.hpp:271-283)
        if (a.want_mass && a.mass_part) {
            // one thread per (unit, head) record, then per unit the heads summed in order
            __shared__ float s_e[128];
            for (int u0 = 0; u0 < a.n_sel; u0 += blockDim.x / rep) {
                const int u = u0 + tid / rep, h = tid % rep;
                const bool on = tid < (blockDim.x / rep) * rep && u < a.n_sel;
                if (on) {
                    const float* mr = sc.mass + ((static_cast<int64_t>(b) * a.H + g * rep + h) * sc.max_sel + u) * kW * 2;
                    float rec[2 * kW];
#pragma unroll
                    for (int i = 0; i < 2 * kW; ++i) rec[i] = __ldcg(mr + i);
                    float e = 0.f;
#pragma unroll
                    for (int w = 0; w < kW; ++w)
                        e += rec[2 * w + 1] == -INFINITY ? 0.f : rec[2 * w] * ex2f(rec[2 * w + 1] - s_M[h]);
                    s_e[tid] = e / s_L[h];
                }
                __syncthreads();
                if (on && h == 0) {
                    double msum = 0.0;
                    for (int hh = 0; hh < rep; ++hh) msum += static_cast<double>(s_e[tid + hh]);
                    a.mass_part[static_cast<int64_t>(u) * a.Gtot + a.g0 + g] = msum;
                }
                __syncthreads();
            }
        }
        return;
    }
    for (int xs = tid; xs < nsplit; xs += blockDim.x) {
        const float mx = s_w[xs][hsel];
        s_w[xs][hsel] = mx == -INFINITY ? 0.f : ex2f(mx - s_M[hsel]) / s_L[hsel];
    }
    __syncthreads();
    float acc = 0.f;
    for (int x0 = 0; x0 < nsplit; x0 += 32) {
        float o2[32];
#pragma unroll
        for (int u = 0; u < 32; ++u)
            o2[u] = x0 == 0 ? ov[u] : (x0 + u < nsplit ? __ldcg(p0 + (x0 + u) * stride + hsel * 130 + 2 + tid) : 0.f);
#pragma unroll
        for (int u = 0; u < 32; ++u)
            if (x0 + u < nsplit) acc = fmaf(o2[u], s_w[x0 + u][hsel], acc);
    }
    static_cast<bf16*>(a.out)[static_cast<int64_t>(g * rep + hsel) * a.dv + tid] = __float2bfloat16_rn(acc);
}
__global__ void __launch_bounds__(128) k_dec_merge1(AttnParams a, DecScratch sc, int nsplit) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // K4's partials
    TL_BEGIN();
    dec_merge_body(a, sc, 0, blockIdx.y, blockIdx.x, nsplit);
    TL_END(TL_MASS);
}
__global__ void __launch_bounds__(128) k_dec_mergeb(const AttnParams* __restrict__ ps, DecScratch sc, int nsplit) {
    // this sequence's parameters into shared memory while K4 drains (the table was
    // uploaded before K4 launched), then the wait for K4's partials
    __shared__ __align__(16) AttnParams sa;
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(AttnParams) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t*>(&sa)[i] = reinterpret_cast<const uint32_t*>(ps + blockIdx.z)[i];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    if (static_cast<int>(blockIdx.x) > sa.rep) return;
    TL_BEGIN();
    dec_merge_body(sa, sc, blockIdx.z, blockIdx.y, blockIdx.x, nsplit);
    TL_END(TL_MASS);
}
void launch_dec_merge(const AttnParams* host_a, const AttnParams* dev_params, int B, int G, int rep, int nsplit,
                      const DecScratch& sc, cudaStream_t st) {
    cudaLaunchConfig_t cfg{};  // programmatic dependent of K4 (which lets it launch on entry)
    cfg.gridDim = dim3(rep + 1, G, B);
    cfg.blockDim = dim3(128);
    cfg.stream = st;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = la;
    cfg.numAttrs = 1;
    if (host_a)
        cudaLaunchKernelEx(&cfg, k_dec_merge1, *host_a, sc, nsplit);
    else
        cudaLaunchKernelEx(&cfg, k_dec_mergeb, dev_params, sc, nsplit);
}

__global__ void __launch_bounds__(kThr, 1) k_attn_dec1(AttnParams a, DecScratch sc) {
    if (sc.sep_merge) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // k_dec_merge1
    TL_BEGIN();
    unsigned long long mark = tl_t0_;
    dec_body(a, sc, 0, blockIdx.x, gridDim.x, mark);
    TL_END(TL_DEC);
}

__global__ void __launch_bounds__(kThr, 1) k_attn_decb(const AttnParams* __restrict__ ps, DecScratch sc) {
    if (sc.sep_merge) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // k_dec_mergeb
    // this sequence's parameters in shared memory (read all through the tile loop)
    __shared__ __align__(16) AttnParams sa;
    static_assert(sizeof(AttnParams) % 4 == 0, "word copy");
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(AttnParams) / 4); i += kThr)
        reinterpret_cast<uint32_t*>(&sa)[i] = reinterpret_cast<const uint32_t*>(ps + blockIdx.z)[i];
    __syncthreads();
    TL_BEGIN();
    unsigned long long mark = tl_t0_;
    dec_body(sa, sc, blockIdx.z, blockIdx.x, gridDim.x, mark);
    TL_END(TL_DEC);
}

int pick_splits(int64_t max_tiles, int G, int B) {
    const int64_t items = static_cast<int64_t>(G) * B;
    if (items < 148) {  // few sequences: one wave of CTAs (<= 148, one per SM), short splits
        const int64_t want = 148 / items;
        return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>({want, max_tiles, kDecMaxSplits})));
    }
    // a batch (1 CTA per SM): the split count whose CTA total fills its last wave
    // best (the per-CTA prologue and the merge favour fewer splits on ties)
    int best = 1;
    double best_eff = 0.0;
    for (int sp = 1; sp <= 8 && sp * 4 <= max_tiles; ++sp) {
        const double waves = static_cast<double>(items * sp) / 148.0;
        const double eff = waves / std::ceil(waves);
        if (eff > best_eff + 1e-3) {
            best_eff = eff;
            best = sp;
        }
    }
    return best;
}

}  // namespace

bool attn_dec_supported(int d, int dv, int unit_size, int rep, bool absolute, int dtype_bf16) {
    return dtype_bf16 && d == 128 && dv == 128 && unit_size == 128 && rep <= kDecMaxRep && !absolute;
}

void dec_encode_maps(const AttnParams& a, int64_t unit_rows, void* host6) {
    CUtensorMap* m = static_cast<CUtensorMap*>(host6);
    const uint64_t G = static_cast<uint64_t>(a.G);
    m[0] = make_tmap_bf16_sw128(a.init_k, G * static_cast<uint64_t>(a.l_I), 128, 128);
    m[1] = make_tmap_bf16_sw128(a.init_v, G * a.vl.nI * 128, 128, 128);
    m[2] = make_tmap_bf16_sw128(a.unit_k ? a.unit_k : a.ring_k, a.unit_k ? static_cast<uint64_t>(unit_rows) : 128, 128, 128);
    m[3] = make_tmap_bf16_sw128(a.unit_v ? a.unit_v : a.ring_v, a.unit_v ? static_cast<uint64_t>(unit_rows) : 128, 128, 128);
    m[4] = make_tmap_bf16_sw128(a.ring_krot, G * static_cast<uint64_t>(a.R), 128, 128);
    m[5] = make_tmap_bf16_sw128(a.ring_v, G * static_cast<uint64_t>(a.R), 128, 128);
}

cudaError_t tl_bind_attn_dec(const TlBuf& b) { return tl_bind_tu(b); }

int64_t dec_max_tiles(const AttnParams& a) {
    const int64_t n_init = (a.init_len + 127) / 128, near0 = (a.local_start / 128) * 128;
    return n_init + a.n_sel + (a.s + 1 - near0 + 127) / 128;
}

void launch_attn_dec(const AttnParams& a, const DecScratch& sc0, cudaStream_t st) {
    const DecScratch& sc = sc0;
    const int ns = pick_splits(dec_max_tiles(a), a.G, 1);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_attn_dec1, cudaFuncAttributeMaxDynamicSharedMemorySize, kDecSmem);
        cudaFuncSetAttribute(k_attn_decb, cudaFuncAttributeMaxDynamicSharedMemorySize, kDecSmem);
        attr = true;
    }
    // programmatic dependent launch after the lookup (sc.pdl)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ns, a.G, 1);
    cfg.blockDim = dim3(kThr);
    cfg.dynamicSmemBytes = kDecSmem;
    cfg.stream = st;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = la;
    cfg.numAttrs = sc.pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_attn_dec1, a, sc);
    if (sc.sep_merge) launch_dec_merge(&a, nullptr, 1, a.G, a.rep, ns, sc, st);
}

void launch_attn_dec_batch(const AttnParams* dev_params, int B, int G, int64_t max_tiles, const DecScratch& sc,
                           cudaStream_t st) {
    const DecScratch& s2 = sc;
    const int ns = pick_splits(max_tiles, G, B);
    cudaFuncSetAttribute(k_attn_decb, cudaFuncAttributeMaxDynamicSharedMemorySize, kDecSmem);
    // programmatic dependent of the top-k: splits without retrieved units start early
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ns, G, B);
    cfg.blockDim = dim3(kThr);
    cfg.dynamicSmemBytes = kDecSmem;
    cfg.stream = st;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = la;
    cfg.numAttrs = sc.pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_attn_decb, dev_params, s2);
    if (sc.sep_merge) launch_dec_merge(nullptr, dev_params, B, G, kDecMaxRep, ns, sc, st);
}

}  // namespace infllm
