// kernels.cu — the per-step kernels of the InfLLM layer other than the
// tensor-core attention: RoPE/append/prefix (K7), unit lookup (K1), top-k +
// LRU bookkeeping (K2), eviction + representative scoring (K5/K8),
// representative selection (K6), attention-mass reduction and the
// frequency-decayed LRU update, plus a CUDA-core attention kernel used for
// the fp32 parity mode and for shapes the tcgen05 kernel does not cover.
// Reference citations are relative to /root/reference/proj/include/blockmem/.

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <stdexcept>
#include <string>

#include "kernels.cuh"
#include "tc_prims.cuh"

namespace infllm {

// debug phase timestamps (clock64 of one thread), read by infllm_debug_timestamps
__device__ unsigned long long g_dbg_ts[64];
#define DBG_TS(i)                                   \
    do {                                            \
        if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) g_dbg_ts[(i)] = clock64(); \
    } while (0)

cudaError_t tl_bind_kernels(const TlBuf& b) { return tl_bind_tu(b); }


void debug_read_timestamps(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, g_dbg_ts, sizeof(unsigned long long) * 64);
}

// --------------------------------------------------------------------------
// K7 prep: append k/v to the ring, K_rot = rope(k, pos), q_abs = rope(q, pos),
// q_clamp = rope(q, L)  (rotary.hpp:55-72; attention.hpp:166-167).
// Block = 4 tokens; the (cos, sin) factors of each (token, pair) are computed
// once (fp64 angle, rotary.hpp:25-30) and shared by all heads.
constexpr int kPrepTok = 4;
template <typename T>
__global__ void __launch_bounds__(256) k_prep(PrepParams p) {
    __shared__ float2 cs[kPrepTok][128];
    const int pairs = p.d / 2;
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kPrepTok;
    const int nt = static_cast<int>(min(static_cast<int64_t>(kPrepTok), p.lx - i0));
    for (int t = threadIdx.x; t < nt * pairs; t += blockDim.x) {
        const int tok = t / pairs, a = t % pairs;
        float c, sn;
        rope_cs(p.freqs, a, p.s + i0 + tok, c, sn);
        cs[tok][a] = make_float2(c, sn);
    }
    __syncthreads();
    const T* q = static_cast<const T*>(p.q);
    const T* k = static_cast<const T*>(p.k);
    const T* v = static_cast<const T*>(p.v);
    T* qa = static_cast<T*>(p.qa);
    T* qc = static_cast<T*>(p.qc);
    T* rk = static_cast<T*>(p.ring_k);
    T* rkr = static_cast<T*>(p.ring_krot);
    T* rv = static_cast<T*>(p.ring_v);
    const int dh = (p.d + 1) / 2;  // pairs + odd tail slot
    for (int t = threadIdx.x; t < nt * p.H * dh; t += blockDim.x) {
        const int tok = t / (p.H * dh), rem = t % (p.H * dh), h = rem / dh, a = rem % dh;
        const int64_t i = i0 + tok;
        const T* src = q + (i * p.H + h) * p.d;
        T* da = qa + (static_cast<int64_t>(h) * p.lxp + i) * p.d;
        T* dc = qc + (static_cast<int64_t>(h) * p.lxp + i) * p.d;
        if (a == pairs) {  // odd trailing component is left as is (rotary.hpp:36-37)
            da[p.d - 1] = src[p.d - 1];
            dc[p.d - 1] = src[p.d - 1];
            continue;
        }
        const float x0 = to_f(src[2 * a]), x1 = to_f(src[2 * a + 1]);
        float y0, y1;
        const float2 f = cs[tok][a];
        rope_pair(x0, x1, f.x, f.y, y0, y1);
        da[2 * a] = from_f<T>(y0);
        da[2 * a + 1] = from_f<T>(y1);
        rope_pair(x0, x1, p.freqs.cL[a], p.freqs.sL[a], y0, y1);
        dc[2 * a] = from_f<T>(y0);
        dc[2 * a + 1] = from_f<T>(y1);
    }
    for (int t = threadIdx.x; t < nt * p.G * dh; t += blockDim.x) {
        const int tok = t / (p.G * dh), rem = t % (p.G * dh), g = rem / dh, a = rem % dh;
        const int64_t i = i0 + tok, pos = p.s + i;
        const T* src = k + (i * p.G + g) * p.d;
        const int64_t o = (static_cast<int64_t>(g) * p.R + pos % p.R) * p.d;
        if (a == pairs) {
            rk[o + p.d - 1] = src[p.d - 1];
            rkr[o + p.d - 1] = src[p.d - 1];
            continue;
        }
        const T x0r = src[2 * a], x1r = src[2 * a + 1];
        float y0, y1;
        const float2 f = cs[tok][a];
        rope_pair(to_f(x0r), to_f(x1r), f.x, f.y, y0, y1);
        rk[o + 2 * a] = x0r;
        rk[o + 2 * a + 1] = x1r;
        rkr[o + 2 * a] = from_f<T>(y0);
        rkr[o + 2 * a + 1] = from_f<T>(y1);
    }
    // values: consecutive threads take consecutive tokens so transposed pages
    // get adjacent 2-byte stores
    for (int t = threadIdx.x; t < nt * p.G * p.dv; t += blockDim.x) {
        const int tok = t % nt, rem = t / nt, g = rem / p.dv, c = rem % p.dv;
        const int64_t i = i0 + tok;
        rv[p.vl.ring(g, p.s + i, c)] = v[(i * p.G + g) * p.dv + c];
    }
}

// prefix of qs_t[g][c] = sum_{h in g} q[t][h][c] (fp64) into the P ring, and
// the chunk total (the lookup's query sum, memory.hpp:224-225). Block = one
// group x 32 columns; 32 token segments scanned in parallel, then combined.
// (bf16 inputs make every fp64 partial exact, so the association does not
// change the values.)
constexpr int kScanSegs = 32;
template <typename T>
__global__ void __launch_bounds__(1024) k_prefix(PrepParams p) {
    __shared__ double tot[kScanSegs][33];
    const int g = blockIdx.x;
    const int c = blockIdx.y * 32 + threadIdx.x;
    const int seg = threadIdx.y;
    const bool live = c < p.d;
    const T* q = static_cast<const T*>(p.q);
    const int64_t len = (p.lx + kScanSegs - 1) / kScanSegs;
    const int64_t i0 = seg * len, i1 = min(p.lx, i0 + len);
    auto qs = [&](int64_t i) {
        double a = 0.0;
        for (int hh = 0; hh < p.rep; ++hh) a += static_cast<double>(to_f(q[(i * p.H + g * p.rep + hh) * p.d + c]));
        return a;
    };
    double t = 0.0;
    if (live)
        for (int64_t i = i0; i < i1; ++i) t += qs(i);
    tot[seg][threadIdx.x] = t;
    __syncthreads();
    if (!live) return;
    double run = p.P[((p.s % p.R) * p.G + g) * p.d + c];
    for (int j = 0; j < seg; ++j) run += tot[j][threadIdx.x];
    for (int64_t i = i0; i < i1; ++i) {
        run += qs(i);
        p.P[(((p.s + i + 1) % p.R) * p.G + g) * p.d + c] = run;
    }
    if (seg == 0) {
        double all = 0.0;
        for (int j = 0; j < kScanSegs; ++j) all += tot[j][threadIdx.x];
        p.chunk_qsum[g * p.d + c] = all;
    }
}

// ---- vectorised prep path (head_dim, value_dim multiples of 8) ----------------
// (1) per-step rotation-factor table: one fp64 sincos per (token, pair)
__device__ __forceinline__ void rope_table_body(const PrepParams& p, int64_t t) {
    const int pairs = p.d / 2;
    if (p.kmax2 && t < p.G) p.kmax2[t] = p.kmax2_prev[t];  // k_prep_tok raises it with this chunk's keys
    if (t >= p.lx * pairs) return;
    const int64_t i = t / pairs;
    const int a = static_cast<int>(t % pairs);
    float c, s;
    rope_cs(p.freqs, a, p.s + i, c, s);
    p.rtab[t] = make_float2(c, s);
}
__global__ void k_rope_table(PrepParams p) {
    TL_BEGIN();
    const int64_t n = p.lx * (p.d / 2), stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < (n > p.G ? n : p.G); t += stride)
        rope_table_body(p, t);
    TL_END(TL_ROPE);
}

template <typename T>
struct V8 {
    T v[8];
};
template <typename T>
__device__ __forceinline__ V8<T> ld8(const T* p) {
    V8<T> r;
    if constexpr (sizeof(T) == 2) {
        *reinterpret_cast<uint4*>(&r) = *reinterpret_cast<const uint4*>(p);
    } else {
        reinterpret_cast<uint4*>(&r)[0] = reinterpret_cast<const uint4*>(p)[0];
        reinterpret_cast<uint4*>(&r)[1] = reinterpret_cast<const uint4*>(p)[1];
    }
    return r;
}
template <typename T>
__device__ __forceinline__ void st8(T* p, const V8<T>& r) {
    if constexpr (sizeof(T) == 2) {
        *reinterpret_cast<uint4*>(p) = *reinterpret_cast<const uint4*>(&r);
    } else {
        reinterpret_cast<uint4*>(p)[0] = reinterpret_cast<const uint4*>(&r)[0];
        reinterpret_cast<uint4*>(p)[1] = reinterpret_cast<const uint4*>(&r)[1];
    }
}

// (5) token-tiled prep with coalesced stores: block = 16 tokens x one KV
// group, thread = (token, 8-dim chunk) for head_dim 128 (16 chunks). Rows of
// q_abs / q_clamp / ring k / k_rot are written by 16 consecutive threads
// (256 B each); value pages are transposed through shared memory; the fp64
// group query sums go to qs[token][g][:] plus a per-tile column sum.
// RP: query heads per KV group when known at compile time (0: p.rep <= 8).
template <typename T, int RP>
__device__ __forceinline__ void prep_tok_body(const PrepParams& p, int bx, int g, unsigned long long& mark) {
    __shared__ double sqs[kTokTile][128 + 2];
    __shared__ T svt[128][kTokTile + 2];
    const int tt = threadIdx.x / 16, c8 = threadIdx.x % 16;  // token in tile, dim chunk
    const int64_t i = static_cast<int64_t>(bx) * kTokTile + tt;
    const bool live = i < p.lx;
    const int64_t pos = p.s + i;
    const T* qg = static_cast<const T*>(p.q);
    double qs[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    float kn2 = 0.f;  // this thread's part of |k|^2
    if (live) {
        constexpr int kMaxRep = RP > 0 ? RP : 8;
        const int nrep = RP > 0 ? RP : p.rep;
        V8<T> qv[kMaxRep];
#pragma unroll
        for (int hh = 0; hh < kMaxRep; ++hh)
            if (hh < nrep) qv[hh] = ld8(qg + (i * p.H + g * nrep + hh) * p.d + 8 * c8);
        const V8<T> kv = ld8(static_cast<const T*>(p.k) + (i * p.G + g) * p.d + 8 * c8);
        const V8<T> vv = ld8(static_cast<const T*>(p.v) + (i * p.G + g) * p.dv + 8 * c8);
        float2 f[4];
        {
            const float4* rt = reinterpret_cast<const float4*>(p.rtab + i * (p.d / 2) + 4 * c8);
            const float4 a = rt[0], b = rt[1];
            f[0] = make_float2(a.x, a.y);
            f[1] = make_float2(a.z, a.w);
            f[2] = make_float2(b.x, b.y);
            f[3] = make_float2(b.z, b.w);
        }
        V8<T> kr;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float y0, y1;
            rope_pair(to_f(kv.v[2 * j]), to_f(kv.v[2 * j + 1]), f[j].x, f[j].y, y0, y1);
            kr.v[2 * j] = from_f<T>(y0);
            kr.v[2 * j + 1] = from_f<T>(y1);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) kn2 = fmaf(to_f(kv.v[e]), to_f(kv.v[e]), kn2);
        const int64_t ro = (static_cast<int64_t>(g) * p.R + pos % p.R) * p.d + 8 * c8;
        st8(static_cast<T*>(p.ring_k) + ro, kv);
        st8(static_cast<T*>(p.ring_krot) + ro, kr);
#pragma unroll
        for (int hh = 0; hh < kMaxRep; ++hh) {
            if (hh >= nrep) break;
            V8<T> qa, qc;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float x0 = to_f(qv[hh].v[2 * j]), x1 = to_f(qv[hh].v[2 * j + 1]);
                float y0, y1;
                rope_pair(x0, x1, f[j].x, f[j].y, y0, y1);
                qa.v[2 * j] = from_f<T>(y0);
                qa.v[2 * j + 1] = from_f<T>(y1);
                const int a = 4 * c8 + j;
                rope_pair(x0, x1, p.freqs.cL[a], p.freqs.sL[a], y0, y1);
                qc.v[2 * j] = from_f<T>(y0);
                qc.v[2 * j + 1] = from_f<T>(y1);
                qs[2 * j] += static_cast<double>(x0);
                qs[2 * j + 1] += static_cast<double>(x1);
            }
            const int64_t qo = (static_cast<int64_t>(g * nrep + hh) * p.lxp + i) * p.d + 8 * c8;
            st8(static_cast<T*>(p.qa) + qo, qa);
            st8(static_cast<T*>(p.qc) + qo, qc);
        }
        double2* qd = reinterpret_cast<double2*>(p.qs + (i * p.G + g) * p.d + 8 * c8);
#pragma unroll
        for (int e = 0; e < 4; ++e) qd[e] = make_double2(qs[2 * e], qs[2 * e + 1]);
        TL_MARK(10, mark);  // rows loaded, rotated, stored
        if (!p.vl.vt) {
            st8(static_cast<T*>(p.ring_v) + p.vl.ring(g, pos, 8 * c8), vv);
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) svt[8 * c8 + e][tt] = vv.v[e];
        }
    }
    if (p.kmax2) {
        // |k|^2 per token (the attention kernel's score bound), max into the running value
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) kn2 += __shfl_xor_sync(0xffffffffu, kn2, o);
        kn2 = fmaxf(kn2, __shfl_xor_sync(0xffffffffu, kn2, 16));  // the warp's two tokens
        if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int*>(p.kmax2) + g, __float_as_int(kn2));
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) sqs[tt][8 * c8 + e] = qs[e];
    __syncthreads();
    TL_MARK(11, mark);  // key-norm bound, tile staged
    // per-tile column sums (token order)
    if (threadIdx.x < 128) {
        const int c = threadIdx.x;
        double a = 0.0;
        for (int t = 0; t < kTokTile; ++t) a += sqs[t][c];
        p.tsum[(static_cast<int64_t>(bx) * p.G + g) * p.d + c] = a;
    }
    TL_MARK(12, mark);  // tile column sums
    if (p.vl.vt) {
        // transposed value page rows: 16 consecutive positions of one dim
        const int64_t i0 = static_cast<int64_t>(bx) * kTokTile;
        const int nt = static_cast<int>(min(static_cast<int64_t>(kTokTile), p.lx - i0));
        T* rv = static_cast<T*>(p.ring_v);
        const int R = static_cast<int>(p.R);
        const int sl0 = static_cast<int>((p.s + i0) % p.R);  // one 64-bit division per block
        if (sizeof(T) == 2 && nt == kTokTile && sl0 % kTokTile == 0 && p.dv == 128) {
            // whole aligned tile: the kTokTile positions of a dim are contiguous bytes
            // of one page row, written as 16-byte vectors of 8 (thread = dim, eighth)
            constexpr int hs = kTokTile / 8;
            const int c = threadIdx.x / hs, h = threadIdx.x % hs;
            if (c < 128) {
                uint4 w;
                uint16_t* wv = reinterpret_cast<uint16_t*>(&w);
#pragma unroll
                for (int e = 0; e < 8; ++e) wv[e] = reinterpret_cast<const uint16_t*>(&svt[c][8 * h + e])[0];
                *reinterpret_cast<uint4*>(rv + ((static_cast<int64_t>(g) * (R / 128) + sl0 / 128) * p.dv + c) * 128 +
                                          sl0 % 128 + 8 * h) = w;
            }
        } else {
            for (int t = threadIdx.x; t < 128 * kTokTile; t += blockDim.x) {
                const int c = t / kTokTile, j = t % kTokTile;
                const int sl = sl0 + j >= R ? sl0 + j - R : sl0 + j;
                // [G][R/128][dv][128] pages (VLayout::ring with vt)
                if (j < nt) rv[((static_cast<int64_t>(g) * (R / 128) + sl / 128) * p.dv + c) * 128 + sl % 128] = svt[c][j];
            }
        }
        TL_MARK(13, mark);  // value pages
    }
}

template <typename T, int RP>
__global__ void __launch_bounds__(kTokTile * 16, RP == 4 ? 48 / kTokTile : 1) k_prep_tok(PrepParams p) {
    TL_BEGIN();
    unsigned long long mark = tl_t0_;
    const int tiles = static_cast<int>((p.lx + kTokTile - 1) / kTokTile);
    for (int item = blockIdx.x; item < tiles * p.G; item += gridDim.x) {
        prep_tok_body<T, RP>(p, item % tiles, item / tiles, mark);
        __syncthreads();  // shared tiles are reused by the next item
    }
    TL_END(TL_PREP);
}

// (6) fp64 prefix into the P ring from the per-token sums and the tile sums:
// block = (tile, group), thread = dim; rows of P written whole (coalesced).
template <typename T>
__device__ __forceinline__ void prefix_tiles_body(const PrepParams& p, int tile, int g, int ntiles) {
    const int c = threadIdx.x;
    if (c >= p.d) return;
    const int64_t stride = static_cast<int64_t>(p.G) * p.d;
    double run = p.P[((p.s % p.R) * p.G + g) * p.d + c];
    // earlier tiles' sums: loads issued together, added in tile order (same rounding)
    for (int t0 = 0; t0 < tile; t0 += 16) {
        double ts[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) ts[k] = t0 + k < tile ? p.tsum[(t0 + k) * stride + g * p.d + c] : 0.0;
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (t0 + k < tile) run += ts[k];
    }
    const int64_t i0 = static_cast<int64_t>(tile) * kTokTile;
    const int nt = static_cast<int>(min(static_cast<int64_t>(kTokTile), p.lx - i0));
    double v[kTokTile];
#pragma unroll
    for (int j = 0; j < kTokTile; ++j) v[j] = j < nt ? p.qs[(i0 + j) * stride + g * p.d + c] : 0.0;
    const int R = static_cast<int>(p.R);
    int sl = static_cast<int>((p.s + i0 + 1) % p.R);  // one 64-bit division, then wrap by hand
#pragma unroll
    for (int j = 0; j < kTokTile; ++j) {
        if (j >= nt) break;
        run += v[j];
        p.P[(static_cast<int64_t>(sl) * p.G + g) * p.d + c] = run;
        if (++sl == R) sl = 0;
    }
    if (tile == ntiles - 1) {  // chunk total = sum of the tile sums, in order
        double all = 0.0;
        for (int t = 0; t < ntiles; ++t) all += p.tsum[t * stride + g * p.d + c];
        p.chunk_qsum[g * p.d + c] = all;
    }
}
template <typename T>
__global__ void __launch_bounds__(128) k_prefix_tiles(PrepParams p) {
    TL_BEGIN();
    const int tiles = static_cast<int>((p.lx + kTokTile - 1) / kTokTile);
    for (int item = blockIdx.x; item < tiles * p.G; item += gridDim.x)
        prefix_tiles_body<T>(p, item % tiles, item / tiles, tiles);
    TL_END(TL_PREFIX);
}

template <typename T>
void launch_prep(const PrepParams& p, cudaStream_t st) {
    if (p.d == 128 && p.dv == 128 && p.rep <= 8 && p.rtab && p.tsum) {
        const int64_t nt = p.lx * (p.d / 2);
        const unsigned tiles = static_cast<unsigned>((p.lx + kTokTile - 1) / kTokTile);
        const unsigned items = tiles * static_cast<unsigned>(p.G);
        k_rope_table<<<static_cast<unsigned>((nt + 255) / 256), 256, 0, st>>>(p);
        if (p.rep == 4)
            k_prep_tok<T, 4><<<items, kTokTile * 16, 0, st>>>(p);
        else
            k_prep_tok<T, 0><<<items, kTokTile * 16, 0, st>>>(p);
        k_prefix_tiles<T><<<items, 128, 0, st>>>(p);
        return;
    }
    k_prep<T><<<static_cast<unsigned>((p.lx + kPrepTok - 1) / kPrepTok), 256, 0, st>>>(p);
    dim3 grid(p.G, (p.d + 31) / 32);
    k_prefix<T><<<grid, dim3(32, kScanSegs), 0, st>>>(p);
}
template void launch_prep<float>(const PrepParams&, cudaStream_t);
template void launch_prep<bf16>(const PrepParams&, cudaStream_t);

// --------------------------------------------------------------------------
// K1 lookup score: per (unit, group) the fp64 dot of the chunk's group query
// sum with the unit's r_k representative keys (TieredStore::relevance_all,
// memory.hpp:217-234). One warp per unit; per group, lane L owns the fixed
// contiguous run [L*per, (L+1)*per) of the group's r_k*d elements, then an
// xor-tree: the association does not depend on how groups are sharded. In the
// single-shard (fused) mode the warp sums the groups in order 0..G-1 into
// rel[u] and the last block to finish runs the exact top-k (K2) over all units.
__device__ void block_topk_radix(const double* rel, int64_t U, int64_t K, int64_t* out, unsigned long long* mk = nullptr);

__device__ __forceinline__ int qpad(int c);
template <typename T, int kPer>
__device__ __forceinline__ double group_dot(const T* src, const double* qg, int lane, int d) {
    // elements e = lane*kPer + j of the [r_k][d] run; dim = e % d
    double a = 0.0;
    const int e0 = lane * kPer;
    int c = e0 % d;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        a += qg[qpad(c)] * static_cast<double>(to_f(src[e0 + j]));
        if (++c == d) c = 0;
    }
    return warp_sum_d(a);
}

// qsum is staged in shared memory with 2 doubles of padding per 16 dims so
// the 8 distinct dims read together (16 apart) fall in distinct banks
__device__ __forceinline__ int qpad(int c) { return c + 2 * (c >> 4); }

template <typename T>
__global__ void __launch_bounds__(256) k_lookup(LookupParams p) {
    extern __shared__ double sq[];  // [G][qpad(d)]
    const int dp = qpad(p.d);
    for (int t = threadIdx.x; t < p.G * p.d; t += blockDim.x) sq[(t / p.d) * dp + qpad(t % p.d)] = lk_qsum(p, t);
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t u = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + warp;
    if (u < p.U) {
        const int E = p.r_k * p.d;
        const T* base = static_cast<const T*>(p.repr) + u * p.G * E;
        double rel = 0.0;
        if (E == 512 && sizeof(T) == 2) {
            // 16 bf16 per lane, all groups' loads in flight before the math
            uint4 buf[16];
#pragma unroll
            for (int g = 0; g < 8; ++g)
                if (g < p.G) {
                    buf[2 * g] = __ldcs(reinterpret_cast<const uint4*>(base + g * 512) + lane * 2);
                    buf[2 * g + 1] = __ldcs(reinterpret_cast<const uint4*>(base + g * 512) + lane * 2 + 1);
                }
            const int c0 = (lane * 16) % p.d;  // 16 | d: the run stays inside one key row
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                if (g >= p.G) break;
                const double* qg = sq + g * dp + qpad(c0);
                const bf16* e = reinterpret_cast<const bf16*>(&buf[2 * g]);
                double a = 0.0;
#pragma unroll
                for (int j = 0; j < 16; ++j) a += qg[j] * static_cast<double>(__bfloat162float(e[j]));
                a = warp_sum_d(a);
                if (p.fused) rel += a;
                else if (lane == 0) p.part[u * p.Gtot + p.g0 + g] = a;
            }
            for (int g = 8; g < p.G; ++g) {
                const double a = group_dot<T, 16>(base + g * E, sq + g * dp, lane, p.d);
                if (p.fused) rel += a;
                else if (lane == 0) p.part[u * p.Gtot + p.g0 + g] = a;
            }
        } else {
            const int per = (E + 31) / 32;
            for (int g = 0; g < p.G; ++g) {
                const T* src = base + g * E;
                const double* qg = sq + g * dp;
                double a = 0.0;
                for (int j = 0; j < per; ++j) {
                    const int e = lane * per + j;
                    if (e < E) a += qg[qpad(e % p.d)] * static_cast<double>(to_f(src[e]));
                }
                a = warp_sum_d(a);
                if (p.fused) rel += a;
                else if (lane == 0) p.part[u * p.Gtot + p.g0 + g] = a;
            }
        }
        if (p.fused && lane == 0) p.rel[u] = rel;
    }
    if (p.fused != 1) return;  // 2: rel only, the multi-block top-k follows
    // last block to finish selects the top-k over all units
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(p.done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    block_topk_radix(p.rel, p.U, p.n_sel, p.sel);
    if (threadIdx.x == 0) *p.done = 0;
}

// bf16, head_dim 128, r_k 4, <= 8 KV groups (the C1-C3 shapes): lane l owns
// dims [4l, 4l+4) of every representative row, so its slice of the chunk query
// sums stays in registers (no shared-memory traffic per unit); warps stride
// over units and keep all 32 row loads of a unit in flight before the math.
// Single shard: per lane the groups are summed in order 0..G-1, then one warp
// tree; sharded: one warp tree per group (partials exchanged by the caller).
__device__ __forceinline__ void lookup_reg_body(const LookupParams& p, int nblocks) {
    unsigned long long mark = threadIdx.x == 0 ? gtimer() : 0ull;
    const int lane = threadIdx.x % 32;
    const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
    const int64_t nwarps = static_cast<int64_t>(nblocks) * blockDim.x / 32;
    uint2 x[32];
    auto load_unit = [&](int64_t u) {
        const bf16* base = static_cast<const bf16*>(p.repr) + u * p.G * 512 + 4 * lane;
#pragma unroll
        for (int r = 0; r < 32; ++r)
            if (r < 4 * p.G) x[r] = __ldcs(reinterpret_cast<const uint2*>(base + r * 128));
    };
    // decode chain: this thread's slice of the token's query rows is requested
    // before the first unit, so it is not queued behind 64 KB of unit loads
    uint2 qv[8];
    const bool qpre = p.qtok && p.qrep <= 8 && p.G * 32 <= static_cast<int>(blockDim.x) &&
                      !(reinterpret_cast<uintptr_t>(p.qtok) & 7);
    const int qg = threadIdx.x / 32, qc = lane * 4;
    if (qpre && qg < p.G) {
        const uint2* qq = reinterpret_cast<const uint2*>(static_cast<const bf16*>(p.qtok) +
                                                         static_cast<int64_t>(qg) * p.qrep * 128 + qc);
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < p.qrep) qv[j] = qq[j * 32];
    }
    if (warp0 < p.U) load_unit(warp0);  // in flight while the query sums are formed
    double q[8][4];
    if (p.qtok) {  // decode chain: the token's group query sums, formed once per block
        __shared__ double s_qs[8 * 128];
        if (!qpre) {
            lk_stage_qsums(p, s_qs);
        } else if (qg < p.G) {  // head order, as lk_qsum
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j < p.qrep) {
                    a0 += static_cast<double>(__uint_as_float(qv[j].x << 16));
                    a1 += static_cast<double>(__uint_as_float(qv[j].x & 0xffff0000u));
                    a2 += static_cast<double>(__uint_as_float(qv[j].y << 16));
                    a3 += static_cast<double>(__uint_as_float(qv[j].y & 0xffff0000u));
                }
            double* o = s_qs + qg * 128 + qc;
            o[0] = a0;
            o[1] = a1;
            o[2] = a2;
            o[3] = a3;
        }
        __syncthreads();
#pragma unroll
        for (int g = 0; g < 8; ++g)
#pragma unroll
            for (int j = 0; j < 4; ++j) q[g][j] = g < p.G ? s_qs[g * 128 + 4 * lane + j] : 0.0;
    } else {
#pragma unroll
        for (int g = 0; g < 8; ++g)
#pragma unroll
            for (int j = 0; j < 4; ++j) q[g][j] = g < p.G ? p.qsum[g * 128 + 4 * lane + j] : 0.0;
    }
    TL_MARK(20, mark);  // query sums in registers
    for (int64_t u = warp0; u < p.U; u += nwarps) {
        if (u != warp0) load_unit(u);
        double rel = 0.0;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            if (g >= p.G) break;
            double a = 0.0;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint2 v = x[4 * g + r];
                a = fma(q[g][0], static_cast<double>(__uint_as_float(v.x << 16)), a);
                a = fma(q[g][1], static_cast<double>(__uint_as_float(v.x & 0xffff0000u)), a);
                a = fma(q[g][2], static_cast<double>(__uint_as_float(v.y << 16)), a);
                a = fma(q[g][3], static_cast<double>(__uint_as_float(v.y & 0xffff0000u)), a);
            }
            if (p.fused) {
                rel += a;
            } else {
                a = warp_sum_d(a);
                if (lane == 0) p.part[u * p.Gtot + p.g0 + g] = a;
            }
        }
        if (p.fused) {
            rel = warp_sum_d(rel);
            if (lane == 0) p.rel[u] = rel;
        }
    }
    if (p.fused != 1) return;
    // arrival: the barrier orders the block's relevance stores before thread 0's
    // gpu-scope fence + counter update (cumulativity), the last block's thread 0
    // fences again before the barrier that releases its readers
    __shared__ bool last;
    __syncthreads();
    TL_MARK(21, mark);  // units scored
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(p.done, 1u) == static_cast<unsigned>(nblocks - 1);
        if (last) __threadfence();
    }
    __syncthreads();
    if (!last) return;
    TL_MARK(22, mark);  // last block: arrival counted
    block_topk_radix(p.rel, p.U, p.n_sel, p.sel, &mark);
    TL_MARK(23, mark);  // top-k written
    if (threadIdx.x == 0) *p.done = 0;
}
__global__ void __launch_bounds__(256, 1) k_lookup_reg(LookupParams p) {
    // a decode step's K4 may start its CTAs that do not read the selection now
    // (programmatic dependent launch; those that do wait for this grid)
    if (p.early_dependents) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    TL_BEGIN();
    lookup_reg_body(p, gridDim.x);
    TL_END(TL_LOOKUP);
}

// Large indices: the same math fed by cp.async (16-byte LDGSTS) into a
// 3-deep per-warp shared-memory ring, so each warp keeps the next two units
// (16 KB) in flight while it computes one; 8 warps x 3 x 8 KB per SM.
constexpr int kScanStages = 3;
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void lookup_stream_body(const LookupParams& p, int nblocks) {
    extern __shared__ __align__(16) uint8_t scan_smem[];
    const int lane = threadIdx.x % 32, wib = threadIdx.x / 32;
    uint8_t* ring = scan_smem + static_cast<size_t>(wib) * kScanStages * 8192;
    // contiguous slice per block (its candidates then come out in unit order)
    const int64_t S = (p.U + nblocks - 1) / nblocks;
    const int64_t s0 = static_cast<int64_t>(blockIdx.x) * S, s1 = s0 + S < p.U ? s0 + S : p.U;
    const int64_t warp0 = s0 + wib;
    const int64_t nwarps = blockDim.x / 32;
    const int64_t bytes_u = static_cast<int64_t>(p.G) * 512 * 2;  // one unit's repr rows
    double q[8][4];
    if (p.qtok) {  // decode chain: the token's group query sums, formed once per block
        __shared__ double s_qs[8 * 128];
        lk_stage_qsums(p, s_qs);
        __syncthreads();
#pragma unroll
        for (int g = 0; g < 8; ++g)
#pragma unroll
            for (int j = 0; j < 4; ++j) q[g][j] = g < p.G ? s_qs[g * 128 + 4 * lane + j] : 0.0;
    } else {
#pragma unroll
        for (int g = 0; g < 8; ++g)
#pragma unroll
            for (int j = 0; j < 4; ++j) q[g][j] = g < p.G ? p.qsum[g * 128 + 4 * lane + j] : 0.0;
    }
    // one bulk copy (TMA engine) per unit row block, completion on a per-(warp, stage) mbarrier
    __shared__ __align__(8) uint64_t sbar[8][kScanStages];
    if (lane == 0)
        for (int st = 0; st < kScanStages; ++st) tc::mbar_init(&sbar[wib][st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    auto issue = [&](int64_t u, int stage) {
        if (u < s1 && lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the stage was read by this warp
            tc::mbar_expect_tx(&sbar[wib][stage], static_cast<uint32_t>(bytes_u));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             tc::smem_u32(ring + stage * 8192)),
                         "l"(static_cast<const uint8_t*>(p.repr) + u * bytes_u), "r"(static_cast<uint32_t>(bytes_u)),
                         "r"(tc::smem_u32(&sbar[wib][stage]))
                         : "memory");
        }
    };
#pragma unroll
    for (int st = 0; st < kScanStages - 1; ++st) issue(warp0 + st * nwarps, st);
    int stage = 0;
    int64_t it = 0;
    for (int64_t u = warp0; u < s1; u += nwarps, ++it) {
        issue(u + (kScanStages - 1) * nwarps, (stage + kScanStages - 1) % kScanStages);
        tc::mbar_wait(&sbar[wib][stage], static_cast<uint32_t>((it / kScanStages) & 1));
        const uint8_t* buf = ring + stage * 8192 + 8 * lane;
        double rel = 0.0;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            if (g >= p.G) break;
            double a = 0.0;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint2 v = *reinterpret_cast<const uint2*>(buf + (4 * g + r) * 256);
                a = fma(q[g][0], static_cast<double>(__uint_as_float(v.x << 16)), a);
                a = fma(q[g][1], static_cast<double>(__uint_as_float(v.x & 0xffff0000u)), a);
                a = fma(q[g][2], static_cast<double>(__uint_as_float(v.y << 16)), a);
                a = fma(q[g][3], static_cast<double>(__uint_as_float(v.y & 0xffff0000u)), a);
            }
            if (p.fused) {
                rel += a;
            } else {
                a = warp_sum_d(a);
                if (lane == 0) p.part[u * p.Gtot + p.g0 + g] = a;
            }
        }
        if (p.fused) {
            rel = warp_sum_d(rel);
            if (lane == 0) p.rel[u] = rel;
        }
        __syncwarp();  // the stage is refilled next iteration
        stage = (stage + 1) % kScanStages;
    }
    if (!p.cand_v) return;
    // this block's slice: top n_sel candidates for the final merge (k_topk_final)
    __shared__ int64_t loc[128];
    __threadfence_block();
    __syncthreads();
    const int64_t len = s1 > s0 ? s1 - s0 : 0;
    const int64_t kk = p.n_sel < len ? p.n_sel : len;
    if (kk > 0) block_topk_radix(p.rel + s0, len, kk, loc);
    __syncthreads();
    for (int r = threadIdx.x; r < p.n_sel; r += blockDim.x) {
        const bool ok = r < kk;
        p.cand_v[blockIdx.x * p.n_sel + r] = ok ? p.rel[s0 + loc[r]] : -INFINITY;
        p.cand_i[blockIdx.x * p.n_sel + r] = ok ? s0 + loc[r] : -1;
    }
}

void launch_lookup(const LookupParams& p, int dtype_bf16, cudaStream_t st) {
    const int warps = 8;
    if (dtype_bf16 && p.d == 128 && p.r_k == 4 && p.G <= 8) {
        // one unit per warp up to two waves of resident blocks, then warps stride
        const int64_t want = (p.U + warps - 1) / warps;
        const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(want, 148 * 4));
        k_lookup_reg<<<blocks, warps * 32, 0, st>>>(p);
        return;
    }
    const unsigned blocks = static_cast<unsigned>((p.U + warps - 1) / warps);
    const size_t smem = sizeof(double) * p.G * (p.d + 2 * ((p.d + 15) / 16));
    if (dtype_bf16)
        k_lookup<bf16><<<blocks, warps * 32, smem, st>>>(p);
    else
        k_lookup<float><<<blocks, warps * 32, smem, st>>>(p);
}

// --------------------------------------------------------------------------
// K2 top-k: rel[u] = sum_g part[u][g] (group order 0..Gtot-1), then the top
// n_sel by (rel desc, id asc), returned ascending (memory.hpp:240-253).
// Two-level warp selection over shared memory: each warp extracts the top
// n_sel of its slice, warp 0 merges the candidates; ids are placed by rank.
__device__ __forceinline__ bool better(double va, int ia, double vb, int ib) {
    return ia >= 0 && (ib < 0 || va > vb || (va == vb && ia < ib));
}
__device__ __forceinline__ void warp_argmax(double& v, int& i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i, o);
        if (better(ov, oi, v, i)) {
            v = ov;
            i = oi;
        }
    }
}

constexpr int kTopkMax = 128;  // max k_m
constexpr int kTopkWarps = 16;
constexpr int kTopkSmemU = 12288;  // units kept in shared memory (else global)
// rel: [U] values (read only); work: scratch [U] (global, used when U > kTopkSmemU)
__device__ void block_topk(const double* rel, double* work, int64_t U, int64_t n_sel, int64_t* out) {
    extern __shared__ double sh_rel[];
    __shared__ double cv[kTopkWarps][kTopkMax];
    __shared__ int ci[kTopkWarps][kTopkMax];
    const int lane = threadIdx.x % 32, warp = threadIdx.x / 32, nw = blockDim.x / 32;
    double* w = U <= kTopkSmemU ? sh_rel : work;
    for (int64_t u = threadIdx.x; u < U; u += blockDim.x) w[u] = rel[u];
    __syncthreads();
    const int64_t S = (U + nw - 1) / nw;
    const int b0 = static_cast<int>(warp * S), b1 = static_cast<int>(min(U, warp * S + S));
    for (int64_t r = 0; r < n_sel; ++r) {
        double bv = -INFINITY;
        int bi = -1;
        for (int u = b0 + lane; u < b1; u += 32) {
            const double x = w[u];
            if (x != -INFINITY && better(x, u, bv, bi)) {
                bv = x;
                bi = u;
            }
        }
        warp_argmax(bv, bi);
        if (lane == 0) {
            cv[warp][r] = bv;
            ci[warp][r] = bi;
        }
        if (bi >= 0 && (bi - b0) % 32 == lane) w[bi] = -INFINITY;
        __syncwarp();
    }
    __syncthreads();
    if (warp == 0) {
        int mine[kTopkMax / 32];
#pragma unroll
        for (int k = 0; k < kTopkMax / 32; ++k) mine[k] = -1;
        const int ns = static_cast<int>(n_sel);
        for (int r = 0; r < ns; ++r) {
            double bv = -INFINITY;
            int bi = -1, bt = -1;
            for (int t = lane; t < nw * ns; t += 32) {
                const int ww = t / ns, rr = t % ns;
                if (better(cv[ww][rr], ci[ww][rr], bv, bi)) {
                    bv = cv[ww][rr];
                    bi = ci[ww][rr];
                    bt = t;
                }
            }
            const int mybi = bi;
            warp_argmax(bv, bi);
            if (mybi == bi && bi >= 0) ci[bt / ns][bt % ns] = -1;  // unique id -> unique owner
            __syncwarp();
#pragma unroll
            for (int kk = 0; kk < kTopkMax / 32; ++kk)
                if (kk == r / 32 && r % 32 == lane) mine[kk] = bi;
        }
        // place by rank (ids are distinct); every lane joins every shuffle
#pragma unroll
        for (int k = 0; k < kTopkMax / 32; ++k) {
            if (32 * k >= ns) break;
            const int id = mine[k];
            int rank = 0;
            for (int r = 0; r < ns; ++r) {
                int o = 0x7fffffff;
#pragma unroll
                for (int kk = 0; kk < kTopkMax / 32; ++kk)
                    if (kk == r / 32) o = __shfl_sync(0xffffffffu, mine[kk], r % 32);
                rank += o < id;
            }
            if (id >= 0) out[rank] = id;
        }
    }
    __syncthreads();
}

// Exact top-K by (value desc, id asc) with an MSB-first 8-bit radix select
// on order-preserving 64-bit keys: 8 histogram passes find the K-th key T;
// ids with key > T are taken, and the lowest ids among key == T fill the
// rest. Output ids ascending. Thread t owns the contiguous id range
// [t*E, t*E+E) so block scans give id order. Works for any blockDim
// (multiple of 32) with U <= blockDim * kRadixE.
constexpr int kRadixE = 8;
__device__ __forceinline__ uint64_t order_key(double v) {
    if (v == 0.0) v = 0.0;  // -0.0 == +0.0 for the reference's comparator (memory.hpp:245-252): one key
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ int block_excl_scan(int v, int* wsum, int* total) {
    const int lane = threadIdx.x % 32, warp = threadIdx.x / 32, nw = blockDim.x / 32;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < nw ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < nw) wsum[lane] = w;  // inclusive
    }
    __syncthreads();
    const int before = (warp > 0 ? wsum[warp - 1] : 0) + x - v;
    if (total) *total = wsum[nw - 1];
    __syncthreads();
    return before;
}

__device__ void block_topk_radix(const double* rel, int64_t U, int64_t K, int64_t* out, unsigned long long* mk) {
    __shared__ int hist[2][256];  // pass p counts into hist[p & 1] while hist[(p + 1) & 1] is cleared
    __shared__ int wsum[32];
    __shared__ uint64_t s_prefix, s_mask;
    __shared__ int s_remaining, s_done;
    const int T = blockDim.x, lane = threadIdx.x % 32;
    const int E = static_cast<int>((U + T - 1) / T);
    const int64_t u0 = static_cast<int64_t>(threadIdx.x) * E;
    uint64_t key[kRadixE];
#pragma unroll
    for (int e = 0; e < kRadixE; ++e) key[e] = (e < E && u0 + e < U) ? order_key(rel[u0 + e]) : 0ull;
    if (mk) TL_MARK(24, *mk);  // keys loaded (thread 0)
    for (int i = threadIdx.x; i < 256; i += T) hist[0][i] = 0;
    if (threadIdx.x == 0) {
        s_prefix = 0;
        s_mask = 0;
        s_remaining = static_cast<int>(K);
        s_done = 0;
    }
    __syncthreads();
    for (int pass = 0; pass < 8; ++pass) {
        if (s_done) break;  // uniform: written before the last barrier
        const int shift = 56 - 8 * pass;
        int* h = hist[pass & 1];
        const uint64_t prefix = s_prefix, mask = s_mask;
#pragma unroll
        for (int e = 0; e < kRadixE; ++e)
            if (e < E && u0 + e < U && (key[e] & mask) == prefix) atomicAdd(&h[(key[e] >> shift) & 255], 1);
        for (int i = threadIdx.x; i < 256; i += T) hist[(pass + 1) & 1][i] = 0;
        __syncthreads();
        if (threadIdx.x < 32) {
            // bins high -> low: lane l owns bins 255-8l .. 248-8l
            int c[8], sum = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                c[j] = h[255 - 8 * lane - j];
                sum += c[j];
            }
            int incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int rem = s_remaining;
            int run = incl - sum;  // count in higher bins
            int found = -1, above = 0, cnt = 0;
            if (run < rem && incl >= rem) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (found < 0 && run + c[j] >= rem) {
                        found = 255 - 8 * lane - j;
                        above = run;
                        cnt = c[j];
                    }
                    run += c[j];
                }
            }
            const unsigned m = __ballot_sync(0xffffffffu, found >= 0);
            const int src = __ffs(m) - 1;
            found = __shfl_sync(0xffffffffu, found, src);
            above = __shfl_sync(0xffffffffu, above, src);
            cnt = __shfl_sync(0xffffffffu, cnt, src);
            if (lane == 0) {
                s_prefix = prefix | (static_cast<uint64_t>(found) << shift);
                s_mask = mask | (0xFFull << shift);
                s_remaining = rem - above;
                // the boundary bin is taken whole: no need to resolve further digits
                if (cnt == rem - above) s_done = 1;
            }
        }
        __syncthreads();
    }
    if (mk) TL_MARK(25, *mk);  // digit passes done
    const uint64_t Tk = s_prefix, Tm = s_mask;
    const int need_eq = s_remaining;  // how many of the (key & Tm) == Tk ids to take, lowest first
    // one scan of (above, equal) counts, packed: a thread's first output slot is
    // the ids above T before it plus the equal ids before it that are taken
    int n_gt = 0, n_eq = 0;
#pragma unroll
    for (int e = 0; e < kRadixE; ++e) {
        if (!(e < E && u0 + e < U)) continue;
        const uint64_t km = key[e] & Tm;
        n_gt += km > Tk ? 1 : 0;
        n_eq += km == Tk ? 1 : 0;
    }
    const int ex = block_excl_scan(n_gt | (n_eq << 16), wsum, nullptr);
    int eq_before = ex >> 16;
    int pos = (ex & 0xffff) + (eq_before < need_eq ? eq_before : need_eq);
#pragma unroll
    for (int e = 0; e < kRadixE; ++e) {
        if (!(e < E && u0 + e < U)) continue;
        const uint64_t km = key[e] & Tm;
        bool take = km > Tk;
        if (km == Tk) take = eq_before++ < need_eq;
        if (take) out[pos++] = u0 + e;
    }
}

// Multi-block exact top-k for large unit counts: each block selects the top
// k of a 2048-unit slice (radix select), then one block selects the top k of
// the candidates. Candidates are laid out in slice order with ascending ids
// inside a slice, so candidate index order is unit id order and the
// (rel desc, id asc) tie rule carries over (memory.hpp:245-253).
constexpr int kSliceU = 256 * kRadixE;
constexpr int kTopkMaxSel = 128;  // n_lookup limit
__global__ void __launch_bounds__(256) k_topk_local(const double* rel, int64_t U, int64_t k, double* cand_v,
                                                    int64_t* cand_i) {
    __shared__ int64_t loc[kTopkMaxSel];
    const int64_t s0 = static_cast<int64_t>(blockIdx.x) * kSliceU;
    const int64_t len = U - s0 < kSliceU ? U - s0 : kSliceU;
    const int64_t kk = k < len ? k : len;
    block_topk_radix(rel + s0, len, kk, loc);
    __syncthreads();
    for (int r = threadIdx.x; r < k; r += blockDim.x) {
        const bool ok = r < kk;
        cand_v[blockIdx.x * k + r] = ok ? rel[s0 + loc[r]] : -INFINITY;
        cand_i[blockIdx.x * k + r] = ok ? s0 + loc[r] : -1;
    }
}
__global__ void __launch_bounds__(256, 1) k_lookup_stream(LookupParams p) {
    if (p.early_dependents) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // merge block / K4 (PDL)
    TL_BEGIN();
    lookup_stream_body(p, gridDim.x);
    TL_END(TL_LOOKUP);
}
__global__ void __launch_bounds__(1024) k_topk_final(const double* cand_v, const int64_t* cand_i, int64_t n, int64_t k,
                                                     int64_t* sel) {
    // as a programmatic dependent of the scan: let a decode step's K4 launch,
    // then wait for the scan's candidates (both no-ops on a plain launch)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    TL_BEGIN();
    __shared__ int64_t loc[kTopkMaxSel];
    block_topk_radix(cand_v, n, k, loc);
    __syncthreads();
    for (int r = threadIdx.x; r < k; r += blockDim.x) sel[r] = cand_i[loc[r]];
    TL_END(TL_TOPK);
}
constexpr int kScanBlocks = 148;  // streaming scan: one block per SM, one slice each
int64_t topk_multi_scratch(int64_t U, int64_t k) {
    const int64_t nb = (U + kSliceU - 1) / kSliceU;
    const int64_t n = (nb > kScanBlocks ? nb : kScanBlocks) * k;
    const int64_t m = n > 148 * 32 ? n : 148 * 32;  // also the block lists of k_lookup_topk (lookup.cu)
    return (m + 1) / 2 * 2;  // the id half starts 16-byte aligned (bulk copies)
}
int launch_lookup_topk(LookupParams p, int dtype_bf16, double* cand_v, int64_t* cand_i, cudaStream_t st,
                       void (*between)(void*, cudaStream_t), void* ctx) {
    p.fused = 2;
    constexpr int64_t stream_min = 2049;  // past the fused last-block top-k
    if (dtype_bf16 && p.d == 128 && p.r_k == 4 && p.G <= 8 && p.U >= stream_min &&
        p.U <= static_cast<int64_t>(kScanBlocks) * kSliceU && p.n_sel >= 0 &&
        kScanBlocks * p.n_sel <= 1024 * kRadixE) {
        // large index: streaming scan with the per-slice top-k fused, then one merge block
        const size_t smem = static_cast<size_t>(8) * kScanStages * 8192;
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_lookup_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            attr = true;
        }
        p.cand_v = p.n_sel > 0 ? cand_v : nullptr;
        p.cand_i = p.n_sel > 0 ? cand_i : nullptr;
        // the merge block follows as a programmatic dependent (a decode step's K4 may launch from it)
        k_lookup_stream<<<kScanBlocks, 256, smem, st>>>(p);
        if (between) between(ctx, st);
        if (p.n_sel > 0) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(1);
            cfg.blockDim = dim3(1024);
            cfg.stream = st;
            cudaLaunchAttribute la[1];
            la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            la[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = la;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_topk_final, static_cast<const double*>(cand_v), static_cast<const int64_t*>(cand_i),
                               static_cast<int64_t>(kScanBlocks) * p.n_sel, p.n_sel, p.sel);
            return 2;
        }
        return 1;
    }
    p.cand_v = nullptr;
    p.cand_i = nullptr;
    launch_lookup(p, dtype_bf16, st);
    if (between) between(ctx, st);
    if (p.n_sel > 0 && p.U > 0) return 1 + launch_topk_multi(p.rel, p.U, p.n_sel, cand_v, cand_i, p.sel, st);
    return 1;
}
// up to 1024 * kRadixE units one block selects directly (ids are the indices)
__global__ void __launch_bounds__(1024) k_topk_one(const double* rel, int64_t U, int64_t k, int64_t* sel) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    TL_BEGIN();
    block_topk_radix(rel, U, k, sel);
    TL_END(TL_TOPK);
}
int launch_topk_multi(const double* rel, int64_t U, int64_t k, double* cand_v, int64_t* cand_i, int64_t* sel,
                      cudaStream_t st) {
    if (U <= 0 || k <= 0) return 0;
    if (U <= 1024 * kRadixE) {
        k_topk_one<<<1, 1024, 0, st>>>(rel, U, std::min<int64_t>(k, U), sel);
        return 1;
    }
    const int64_t nb = (U + kSliceU - 1) / kSliceU;
    // the final block holds at most 1024 * kRadixE candidates (block_topk_radix)
    if (nb * k > 1024 * kRadixE)
        throw std::invalid_argument("lookup: n_units * n_lookup beyond the top-k capacity (U <= " +
                                    std::to_string(1024 * kRadixE / k * kSliceU) + " units at this n_lookup)");
    k_topk_local<<<static_cast<unsigned>(nb), 256, 0, st>>>(rel, U, k, cand_v, cand_i);
    k_topk_final<<<1, 1024, 0, st>>>(cand_v, cand_i, nb * k, std::min<int64_t>(k, U), sel);
    return 2;
}

__global__ void __launch_bounds__(1024) k_topk(TopkParams p) {
    for (int64_t u = threadIdx.x; u < p.U; u += blockDim.x) {
        double v[16];
#pragma unroll
        for (int g = 0; g < 16; ++g) v[g] = g < p.Gtot ? p.part[u * p.Gtot + g] : 0.0;
        double a = 0.0;
#pragma unroll
        for (int g = 0; g < 16; ++g)
            if (g < p.Gtot) a += v[g];
        for (int g = 16; g < p.Gtot; ++g) a += p.part[u * p.Gtot + g];
        p.rel[u] = a;
    }
    __syncthreads();
    if (p.U <= static_cast<int64_t>(blockDim.x) * kRadixE)
        block_topk_radix(p.rel, p.U, p.n_sel, p.sel);
    else
        block_topk(p.rel, p.rel, p.U, p.n_sel, p.sel);
}

static size_t topk_smem(int64_t U) { return U <= kTopkSmemU ? static_cast<size_t>(U) * sizeof(double) : 0; }

void launch_topk(const TopkParams& p, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_topk, cudaFuncAttributeMaxDynamicSharedMemorySize, kTopkSmemU * sizeof(double));
        attr = true;
    }
    // radix select with 1024 threads x kRadixE ids, else the two-level warp selection
    const bool radix = p.U <= 1024 * kRadixE;
    k_topk<<<1, radix ? 1024 : 32 * kTopkWarps, radix ? 0 : topk_smem(p.U), st>>>(p);
}

// --------------------------------------------------------------------------
// CUDA-core attention (attention.hpp:116-230) with online softmax, staircase
// clamp, causal chunk, and per-unit attention mass partials (engine.hpp:271-283).
constexpr int kBQ = 32, kBK = 64, kThreads = 256;

template <typename T>
__device__ __forceinline__ const T* row_ptr(const AttnParams& p, int kind, int g, int64_t id, int64_t pos_or_off,
                                            const void* init, const void* unit, const void* ring, int dim) {
    // kind 0: init (pos), 1: unit (id, offset), 2: ring (pos)
    if (kind == 0) return static_cast<const T*>(init) + (static_cast<int64_t>(g) * p.l_I + pos_or_off) * dim;
    if (kind == 1) return static_cast<const T*>(unit) + ((id * p.G + g) * p.l_bs + pos_or_off) * dim;
    return static_cast<const T*>(ring) + (static_cast<int64_t>(g) * p.R + (pos_or_off % p.R)) * dim;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_attn_simt(AttnParams p) {
    extern __shared__ float sm[];
    const int d = p.d, dv = p.dv;
    const int dp = d + 1, dvp = dv + 1;
    float* sqa = sm;                   // [BQ][dp]
    float* sqc = sqa + kBQ * dp;       // [BQ][dp]
    float* skr = sqc + kBQ * dp;       // [BK][dp] raw
    float* skt = skr + kBK * dp;       // [BK][dp] rotated
    float* sv = skt + kBK * dp;        // [BK][dvp]
    float* sp = sv + kBK * dvp;        // [BQ][BK+1]
    __shared__ int64_t kpos[kBK];

    const int h = blockIdx.y, g = h / p.rep;
    const int64_t q0 = static_cast<int64_t>(blockIdx.x) * kBQ;
    const int tid = threadIdx.x, r = tid / 8, sub = tid % 8;
    const int64_t qi = q0 + r;
    const bool qvalid = qi < p.lx;
    const int64_t qp = p.s + qi;

    const T* qa = static_cast<const T*>(p.qa) + static_cast<int64_t>(h) * p.lxp * d;
    const T* qc = static_cast<const T*>(p.qc) + static_cast<int64_t>(h) * p.lxp * d;
    for (int t = tid; t < kBQ * d; t += kThreads) {
        const int rr = t / d, c = t % d;
        const bool ok = q0 + rr < p.lx;
        sqa[rr * dp + c] = ok ? to_f(qa[(q0 + rr) * d + c]) : 0.f;
        sqc[rr * dp + c] = ok ? to_f(qc[(q0 + rr) * d + c]) : 0.f;
    }

    float m = -INFINITY, l = 0.f;
    float acc[16];  // dv <= 128
#pragma unroll
    for (int t = 0; t < 16; ++t) acc[t] = 0.f;
    float unit_e = 0.f, unit_m = -INFINITY;

    const int64_t near_end = min(p.s + p.lx, p.s + q0 + kBQ);  // causal: keys beyond the last row are masked
    const int n_segs = 1 + p.n_sel + 1;
    for (int seg = 0; seg < n_segs; ++seg) {
        int kind;
        int64_t seg_len, seg_start, id = -1;
        if (seg == 0) {
            kind = 0;
            seg_len = p.init_len;
            seg_start = 0;
        } else if (seg <= p.n_sel) {
            kind = 1;
            id = p.sel[seg - 1];
            seg_len = p.unit_len[id];
            if (p.sel_slot) id = p.sel_slot[seg - 1];  // host tier: the unit's GPU cache slot page
            seg_start = 0;
        } else {
            kind = 2;
            seg_start = p.local_start;
            seg_len = near_end - p.local_start;
        }
        const bool far = kind != 2;
        for (int64_t t0 = 0; t0 < seg_len; t0 += kBK) {
            const int nk = static_cast<int>((seg_len - t0 < kBK ? seg_len - t0 : (int64_t)kBK));
            __syncthreads();
            // load tile rows
            for (int t = tid; t < kBK; t += kThreads) kpos[t] = kind == 2 ? seg_start + t0 + t : -1;
            const bool need_raw = !p.absolute;
            const bool need_rot = p.absolute || !far;
            for (int t = tid; t < nk * d; t += kThreads) {
                const int rr = t / d, c = t % d;
                const int64_t off = seg_start + t0 + rr;
                if (need_raw)
                    skr[rr * dp + c] = to_f(row_ptr<T>(p, kind, g, id, off, p.init_k, p.unit_k, p.ring_k, d)[c]);
                if (need_rot)
                    skt[rr * dp + c] = to_f(row_ptr<T>(p, kind, g, id, off, p.init_krot, p.unit_krot, p.ring_krot, d)[c]);
            }
            for (int t = tid; t < nk * dv; t += kThreads) {
                const int rr = t / dv, c = t % dv;
                const int64_t off = seg_start + t0 + rr;
                const int64_t vi = kind == 0 ? p.vl.init(g, off, c) : (kind == 1 ? p.vl.unit(id, g, off, c) : p.vl.ring(g, off, c));
                const T* vb = static_cast<const T*>(kind == 0 ? p.init_v : (kind == 1 ? p.unit_v : p.ring_v));
                sv[rr * dvp + c] = to_f(vb[vi]);
            }
            __syncthreads();
            // scores
            float sc[kBK / 8];
            float tmax = -INFINITY;
#pragma unroll
            for (int j8 = 0; j8 < kBK / 8; ++j8) {
                const int j = sub + 8 * j8;
                float x = -INFINITY;
                if (qvalid && j < nk) {
                    bool use_clamp, masked = false;
                    if (p.absolute) {
                        use_clamp = false;
                        if (!far) masked = kpos[j] > qp;
                    } else if (far) {
                        use_clamp = true;
                    } else {
                        masked = kpos[j] > qp;
                        use_clamp = qp - kpos[j] > p.L;
                    }
                    if (!masked) {
                        const float* qv = use_clamp ? sqc + r * dp : sqa + r * dp;
                        const float* kv = use_clamp ? skr + j * dp : skt + j * dp;
                        float a = 0.f;
                        for (int c = 0; c < d; ++c) a = fmaf(qv[c], kv[c], a);
                        x = a * p.scale;
                    }
                }
                sc[j8] = x;
                tmax = fmaxf(tmax, x);
            }
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 4));
            const float m_new = fmaxf(m, tmax);
            float tsum = 0.f;
#pragma unroll
            for (int j8 = 0; j8 < kBK / 8; ++j8) {
                const float e = (m_new == -INFINITY || sc[j8] == -INFINITY) ? 0.f : expf(sc[j8] - m_new);
                sp[r * (kBK + 1) + sub + 8 * j8] = e;
                tsum += e;
            }
            tsum += __shfl_xor_sync(0xffffffffu, tsum, 1);
            tsum += __shfl_xor_sync(0xffffffffu, tsum, 2);
            tsum += __shfl_xor_sync(0xffffffffu, tsum, 4);
            const float corr = (m == -INFINITY) ? 0.f : expf(m - m_new);
            l = l * corr + tsum;
#pragma unroll
            for (int t = 0; t < 16; ++t) acc[t] *= corr;
            if (kind == 1 && p.want_mass) {
                const float uc = (unit_m == -INFINITY) ? 0.f : expf(unit_m - m_new);
                unit_e = (t0 == 0 ? 0.f : unit_e * uc) + tsum;
                unit_m = m_new;
            }
            m = m_new;
            __syncthreads();
            for (int j = 0; j < nk; ++j) {
                const float pj = sp[r * (kBK + 1) + j];
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                    const int c = sub + 8 * t;
                    if (c < dv) acc[t] = fmaf(pj, sv[j * dvp + c], acc[t]);
                }
            }
        }
        if (kind == 1 && p.want_mass && qvalid && sub == 0) {
            const int64_t o = (static_cast<int64_t>(h) * p.lx + qi) * p.n_sel + (seg - 1);
            p.mass_e[o] = seg_len > 0 ? unit_e : 0.f;
            p.mass_m[o] = unit_m;
            unit_e = 0.f;
            unit_m = -INFINITY;
        }
    }
    if (qvalid) {
        T* out = static_cast<T*>(p.out) + (qi * p.H + h) * dv;
        const float inv = 1.f / l;
        if (p.inv_violations && sub == 0 && !(l > 0.f && isfinite(l) && isfinite(inv)))
            atomicAdd(p.inv_violations, 1ull);  // check_softmax (engine.hpp:361-371)
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            const int c = sub + 8 * t;
            if (c < dv) out[c] = from_f<T>(acc[t] * inv);
        }
        if (sub == 0 && p.want_mass) {
            p.row_m[static_cast<int64_t>(h) * p.lx + qi] = m;
            p.row_l[static_cast<int64_t>(h) * p.lx + qi] = l;
        }
    }
}

template <typename T>
void launch_attn_simt(const AttnParams& p, cudaStream_t st) {
    const int dp = p.d + 1, dvp = p.dv + 1;
    const size_t smem = sizeof(float) * (2 * kBQ * dp + 2 * kBK * dp + kBK * dvp + kBQ * (kBK + 1));
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_attn_simt<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    dim3 grid(static_cast<unsigned>((p.lx + kBQ - 1) / kBQ), p.H);
    k_attn_simt<T><<<grid, kThreads, smem, st>>>(p);
}
template void launch_attn_simt<float>(const AttnParams&, cudaStream_t);
template void launch_attn_simt<bf16>(const AttnParams&, cudaStream_t);

// --------------------------------------------------------------------------
// per-unit attention mass: sum over the group's heads and the chunk's rows of
// the normalised weights of the unit's columns (engine.hpp:271-283), fp64,
// fixed association (thread-strided partials + tree).
__global__ void k_mass(MassParams p) {
    __shared__ double red[256];
    const int j = blockIdx.x;
    for (int g = 0; g < p.G; ++g) {
        double a = 0.0;
        const int64_t n = static_cast<int64_t>(p.rep) * p.lx;
        for (int64_t t = threadIdx.x; t < n; t += blockDim.x) {
            const int hh = static_cast<int>(t / p.lx);
            const int64_t i = t % p.lx;
            const int h = g * p.rep + hh;
            const int64_t o = static_cast<int64_t>(h) * p.lx + i;
            const float e = p.mass_e[o * p.n_sel + j];
            if (e > 0.f) a += static_cast<double>(e) * exp(static_cast<double>(p.mass_m[o * p.n_sel + j]) - static_cast<double>(p.row_m[o])) /
                              static_cast<double>(p.row_l[o]);
        }
        red[threadIdx.x] = a;
        __syncthreads();
        for (int w = blockDim.x / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) p.part[j * p.Gtot + p.g0 + g] = red[0];
        __syncthreads();
    }
}

// mass_part[j][g0+g] = sum_{hh, m-tile} mass_cta (sharded runs exchange per-group partials)
__global__ void k_mass_cta_reduce(const double* mass_cta, double* part, int n_sel, int G, int Gtot, int g0, int rep,
                                  int n_mt) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_sel) return;
    for (int g = 0; g < G; ++g) {
        double mg = 0.0;
        for (int hh = 0; hh < rep; ++hh)
            for (int mt = 0; mt < n_mt; ++mt) mg += mass_cta[((static_cast<int64_t>(g) * rep + hh) * n_mt + mt) * n_sel + j];
        part[static_cast<int64_t>(j) * Gtot + g0 + g] = mg;
    }
}

void launch_mass_cta_reduce(const double* mass_cta, double* part, int n_sel, int G, int Gtot, int g0, int rep, int n_mt,
                            cudaStream_t st) {
    if (n_sel > 0) k_mass_cta_reduce<<<(n_sel + 63) / 64, 64, 0, st>>>(mass_cta, part, n_sel, G, Gtot, g0, rep, n_mt);
}

void launch_mass(const MassParams& p, cudaStream_t st) {
    if (p.n_sel > 0) k_mass<<<p.n_sel, 256, 0, st>>>(p);
}

// TieredStore bookkeeping for one step: lookup tier transfers + counters +
// trace (memory.hpp:254-267), decay of every hot unit then + attention mass
// (273-281), capacity eviction of the min-(s_b, id) unit (285-300),
// residency peaks (303-308). All global reads are issued up front by 8
// warps; the sequential logic then runs in warp 0 over shared memory.
constexpr int kLruMax = 512;  // hot_capacity + k_m bound
__device__ __forceinline__ void lru_body(const LruParams& p) {
    __shared__ int64_t ids[kLruMax];
    __shared__ double fr[kLruMax];
    __shared__ int64_t sel[kTopkMax];
    __shared__ int8_t sel_hot[kTopkMax];
    __shared__ double sel_f[kTopkMax];
    __shared__ double mass[kTopkMax];
    __shared__ LruState st;
    const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
    if (threadIdx.x == 0) st = *p.lru;
    __syncthreads();
    const int64_t n0 = st.hot_count;
    for (int64_t a = threadIdx.x; a < n0; a += blockDim.x) {
        const int64_t id = p.hot_list[a];
        ids[a] = id;
        fr[a] = p.freq[id];
    }
    for (int64_t j = threadIdx.x; j < p.n_sel; j += blockDim.x) {
        const int64_t id = p.sel[j];
        sel[j] = id;
        sel_hot[j] = p.hot[id];
        sel_f[j] = p.freq[id];
    }
    // attention masses of the retrieved units (engine.hpp:271-283)
    for (int64_t j = warp; j < p.n_mass; j += blockDim.x / 32) {
        double m = 0.0;
        if (p.mass_src == 0) {
            if (lane == 0)
                for (int g = 0; g < p.Gtot; ++g) m += p.mass_part[j * p.Gtot + g];
        } else {
            const int nt = p.G * p.rep * p.n_mt;  // flattened (g, hh, m-tile) in order
            for (int t = lane; t < nt; t += 32) m += p.mass_cta[static_cast<int64_t>(t) * p.n_sel + j];
            m = warp_sum_d(m);
        }
        if (lane == 0) mass[j] = m / static_cast<double>(p.H_total);
    }
    __syncthreads();
    if (warp != 0) return;
    // 1. lookup bookkeeping, ids ascending as returned by lookup
    int64_t n = n0;
    if (lane == 0) {
        for (int64_t j = 0; j < p.n_sel; ++j) {
            const int64_t id = sel[j];
            st.requested++;
            int64_t* tr = p.trace + 3 * st.trace_count;
            tr[0] = p.step;
            tr[1] = id;
            tr[2] = sel_hot[j] ? 1 : 0;
            st.trace_count++;
            if (sel_hot[j]) {
                st.hits++;
            } else {
                st.misses++;
                st.loads++;
                p.hot[id] = 1;
                ids[n] = id;
                fr[n] = sel_f[j];
                ++n;
            }
        }
    }
    n = __shfl_sync(0xffffffffu, n, 0);
    __syncwarp();
    // 2. decay every hot unit, 3. add this step's masses
    for (int64_t a = lane; a < n; a += 32) {
        double f = fr[a] * p.decay;
        for (int64_t j = 0; j < p.n_mass; ++j)
            if (sel[j] == ids[a]) f += mass[j];
        fr[a] = f;
    }
    __syncwarp();
    // 4. capacity
    int64_t cnt = n;
    while (cnt > p.cap) {
        double bv = INFINITY;
        int64_t bi = INT64_MAX, ba = -1;
        for (int64_t a = lane; a < cnt; a += 32)
            if (fr[a] < bv || (fr[a] == bv && ids[a] < bi)) {
                bv = fr[a];
                bi = ids[a];
                ba = a;
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            const int64_t oa = __shfl_xor_sync(0xffffffffu, ba, o);
            if (ov < bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
                ba = oa;
            }
        }
        if (lane == 0) {
            p.hot[bi] = 0;
            p.freq[bi] = bv;  // s_b persists in the cold tier
            ids[ba] = ids[cnt - 1];
            fr[ba] = fr[cnt - 1];
            st.evictions++;
        }
        --cnt;
        __syncwarp();
    }
    // 5. write back + peaks
    int64_t bytes = 0;
    for (int64_t a = lane; a < cnt; a += 32) {
        p.hot_list[a] = ids[a];
        p.freq[ids[a]] = fr[a];
        bytes += p.bytes_per_token * p.unit_len[ids[a]];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
    if (lane == 0) {
        st.hot_count = cnt;
        if (cnt > st.peak_hot_units) st.peak_hot_units = cnt;
        if (bytes > st.peak_hot_bytes) st.peak_hot_bytes = bytes;
        *p.lru = st;
    }
}

__global__ void __launch_bounds__(256) k_lru(LruParams p) {
    TL_BEGIN();
    lru_body(p);
    TL_END(TL_LRU);
}
void launch_lru(const LruParams& p, cudaStream_t st) { k_lru<<<1, 256, 0, st>>>(p); }

// ---- host tier: GPU unit-cache slot assignment + PCIe page pull ----
// One warp. Slot stamps (layer step + 2) live in shared memory for the whole
// assignment; hits are stamped first so no miss can take them, then each miss
// takes the least-recently-stamped slot (tie: lower slot) whose last use is
// older than the previous step of this layer (that attention may still be
// reading it: the lookup of step t overlaps the attention of step t-1).
__global__ void __launch_bounds__(32) k_tier_assign(TierParams p) {
    extern __shared__ int64_t s_used[];  // [S]
    __shared__ int32_t s_slot[kTopkMax];
    const int lane = threadIdx.x;
    const int64_t stamp = p.step + 2;
    for (int64_t s = lane; s < p.S; s += 32) s_used[s] = p.slot_used[s];
    for (int64_t j = lane; j < p.n_sel; j += 32) s_slot[j] = p.unit_slot[p.sel[j]];
    __syncwarp();
    int64_t hits = 0;
    for (int64_t j = lane; j < p.n_sel; j += 32)
        if (s_slot[j] >= 0) {
            s_used[s_slot[j]] = stamp;
            ++hits;
        }
    __syncwarp();
    int nm = 0, fail = 0;
    for (int64_t j = 0; j < p.n_sel; ++j) {
        if (s_slot[j] >= 0) continue;
        int64_t bv = INT64_MAX;
        int bs = -1;
        for (int s = lane; s < p.S; s += 32)
            if (s_used[s] <= p.step && s_used[s] < bv) {
                bv = s_used[s];
                bs = s;
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int64_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int os = __shfl_xor_sync(0xffffffffu, bs, o);
            if (os >= 0 && (bs < 0 || ov < bv || (ov == bv && os < bs))) {
                bv = ov;
                bs = os;
            }
        }
        if (bs < 0) {  // cannot happen with S >= 2 k_m (checked on the host)
            ++fail;
            continue;
        }
        if (lane == 0) {
            const int64_t id = p.sel[j];
            const int64_t old = p.slot_unit[bs];
            if (old >= 0) p.unit_slot[old] = -1;
            p.unit_slot[id] = bs;
            p.slot_unit[bs] = id;
            s_used[bs] = stamp;
            s_slot[j] = bs;
            p.miss[nm] = bs;
            p.miss[p.n_sel + nm] = static_cast<int32_t>(j);
        }
        ++nm;
        __syncwarp();
    }
    __syncwarp();
    for (int64_t s = lane; s < p.S; s += 32) p.slot_used[s] = s_used[s];
    for (int64_t j = lane; j < p.n_sel; j += 32) p.sel_slot[j] = s_slot[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) hits += __shfl_xor_sync(0xffffffffu, hits, o);
    if (lane == 0) {
        *p.miss_n = nm;
        p.stats[0] += nm;
        p.stats[1] += hits;
        p.stats[2] += static_cast<int64_t>(nm) * (p.page_k * (p.host_krot ? 2 : 1) + p.page_v);
        p.stats[3] += fail;
    }
}

// grid (max misses, chunks of 32 KB over the unit's K | K_rot | V pages):
// 8 independent 16-byte loads in flight per thread from mapped host memory.
constexpr int kTierChunk = 256 * 8 * 16;
__global__ void __launch_bounds__(256) k_tier_copy(TierParams p) {
    const int j = blockIdx.x;
    if (j >= *p.miss_n) return;
    const int64_t slot = p.miss[j];
    const int64_t id = p.sel[p.miss[p.n_sel + j]];
    // chunk c of the K page, then of the V page, then of the K_rot page
    const int64_t ck = (p.page_k + kTierChunk - 1) / kTierChunk, cv = (p.page_v + kTierChunk - 1) / kTierChunk;
    int64_t c = blockIdx.y;
    const uint8_t* src;
    uint8_t* dst;
    int64_t page;
    if (c < ck) {
        src = static_cast<const uint8_t*>(p.host_k);
        dst = static_cast<uint8_t*>(p.slot_k);
        page = p.page_k;
    } else if ((c -= ck) < cv) {
        src = static_cast<const uint8_t*>(p.host_v);
        dst = static_cast<uint8_t*>(p.slot_v);
        page = p.page_v;
    } else {
        c -= cv;
        if (!p.host_krot || c >= ck) return;
        src = static_cast<const uint8_t*>(p.host_krot);
        dst = static_cast<uint8_t*>(p.slot_krot);
        page = p.page_k;
    }
    const int64_t off = c * kTierChunk, len = page - off;
    src += id * page + off;
    dst += slot * page + off;
    const int64_t n16 = (len < kTierChunk ? len : kTierChunk) / 16;
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    uint4 r[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int64_t i = threadIdx.x + 256 * u;
        if (i < n16) r[u] = __ldg(s4 + i);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int64_t i = threadIdx.x + 256 * u;
        if (i < n16) d4[i] = r[u];
    }
}

void launch_tier(const TierParams& p, cudaStream_t st) {
    const size_t smem = static_cast<size_t>(p.S) * sizeof(int64_t);
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
        cudaFuncSetAttribute(k_tier_assign, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        attr = smem;
    }
    k_tier_assign<<<1, 32, smem, st>>>(p);
    const int64_t ck = (p.page_k + kTierChunk - 1) / kTierChunk, cv = (p.page_v + kTierChunk - 1) / kTierChunk;
    dim3 grid(static_cast<unsigned>(p.kmax), static_cast<unsigned>(ck * (p.host_krot ? 2 : 1) + cv));
    k_tier_copy<<<grid, 256, 0, st>>>(p);
}

__device__ void warp_select(const float* sc, int len, int r_k, int* out);

// --------------------------------------------------------------------------
// K8 evict + K5 representative-score partials. Popped positions
// [pop0, pop0 + n_init) are pinned as initial tokens (engine.hpp:311-322);
// the rest are evicted into unit pages (engine.hpp:323-340, UnitPacker::add
// memory.hpp:59-78). r_m partial per group: k_m . (P[m+L+1] - P[m+1]), i.e.
// sum over the L following queries of the group's q . k_m (repr_score.hpp:53-67).
// Eviction with all loads in flight at once: block = one popped token, warp
// = one KV group. Copies k (and k_rot in absolute mode) and v into the
// initial-token buffer or the token's unit page; for evicted tokens computes
// the per-group r_m partial k_m . (P[m+L+1] - P[m+1]) with lane-contiguous
// dims + xor tree, and either stores it (sharded: exchanged, then
// k_finalize) or sums the groups in order 0..G-1 in-block and writes the
// finalized score (finalize_front, repr_score.hpp:72-82).
template <typename T>
__device__ __forceinline__ void evict_tok_body(const EvictParams& p) {
    __shared__ double part[32];
    const int g = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t idx = blockIdx.x;
    const int64_t pos = p.pop0 + idx;
    const int64_t slot = pos % p.R;
    const bool to_init = idx < p.n_init;
    int64_t u = 0, off = 0;
    if (!to_init) {
        const int64_t rel = pos - p.pend_start;
        u = p.unit0 + rel / p.l_bs;
        off = rel % p.l_bs;
    }
    const T* rk = static_cast<const T*>(p.ring_k) + (static_cast<int64_t>(g) * p.R + slot) * p.d;
    const int per = (p.d + 31) / 32;  // contiguous dims per lane
    const int c0 = lane * per;
    // issue the score loads first (evictees only)
    double acc = 0.0;
    if (!to_init) {
        const int64_t slo = slot + 1 == p.R ? 0 : slot + 1;
        int64_t shi = slot + 1 + p.L;  // l_L < R: at most one wrap
        if (shi >= p.R) shi -= p.R;
        const double* Phi = p.P + (shi * p.G + g) * p.d;
        const double* Plo = p.P + (slo * p.G + g) * p.d;
        for (int j = 0; j < per; ++j) {
            const int c = c0 + j;
            if (c < p.d) acc += static_cast<double>(to_f(rk[c])) * (Phi[c] - Plo[c]);
        }
    }
    // copies
    if (!(p.page_mode && !to_init)) {  // page mode: k_select copies whole unit pages
    const int nvec = (p.d * static_cast<int>(sizeof(T))) % 16 == 0 ? p.d * static_cast<int>(sizeof(T)) / 16 : 0;
    T* dk = to_init ? static_cast<T*>(p.init_k) + (static_cast<int64_t>(g) * p.l_I + pos) * p.d
                    : static_cast<T*>(p.unit_k) + ((u * p.G + g) * p.l_bs + off) * p.d;
    T* dkr = !p.absolute ? nullptr
             : to_init ? static_cast<T*>(p.init_krot) + (static_cast<int64_t>(g) * p.l_I + pos) * p.d
                       : static_cast<T*>(p.unit_krot) + ((u * p.G + g) * p.l_bs + off) * p.d;
    const T* rkr = static_cast<const T*>(p.ring_krot) + (static_cast<int64_t>(g) * p.R + slot) * p.d;
    if (nvec) {
        for (int t = lane; t < nvec; t += 32) {
            reinterpret_cast<uint4*>(dk)[t] = reinterpret_cast<const uint4*>(rk)[t];
            if (dkr) reinterpret_cast<uint4*>(dkr)[t] = reinterpret_cast<const uint4*>(rkr)[t];
        }
    } else {
        for (int c = lane; c < p.d; c += 32) {
            dk[c] = rk[c];
            if (dkr) dkr[c] = rkr[c];
        }
    }
    const T* rv = static_cast<const T*>(p.ring_v);
    T* dvb = static_cast<T*>(to_init ? p.init_v : p.unit_v);
    for (int c = lane; c < p.dv; c += 32) {
        const T x = rv[p.vl.ring(g, pos, c)];
        if (to_init)
            dvb[p.vl.init(g, pos, c)] = x;
        else
            dvb[p.vl.unit(u, g, off, c)] = x;
    }
    }
    if (to_init) return;
    acc = warp_sum_d(acc);
    if (!p.fused) {
        if (lane == 0) p.ev_part[(idx - p.n_init) * p.Gtot + p.g0 + g] = acc;
        return;
    }
    if (lane == 0) part[g] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int gg = 0; gg < p.G; ++gg) tot += part[gg];
        p.unit_scores[u * p.l_bs + off] = static_cast<float>(tot / static_cast<double>(p.L));
    }
}

template <typename T>
__global__ void __launch_bounds__(256) k_evict_tok(EvictParams p) {
    TL_BEGIN();
    evict_tok_body<T>(p);
    TL_END(TL_EVICT);
}

// Chunk steps: one warp per departing token, all of its KV groups (the
// per-group dots are the same lane slices and xor trees as evict_tok_body,
// summed in group order, so scores are bitwise identical); eight tokens per
// block. A chunk's 512 evictions take 64 short blocks instead of 512, so the
// launch leaves the SMs the attention is about to take after a few
// microseconds (SM occupancy, not bandwidth, is what it costs the step).
constexpr int kEvWarps = 8;
template <typename T>
__global__ void __launch_bounds__(kEvWarps * 32) k_evict_warp(EvictParams p) {
    TL_BEGIN();
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kEvWarps;
    const int64_t idx = i0 + w;
    const int R = static_cast<int>(p.R);
    const int sl0 = static_cast<int>((p.pop0 + i0) % p.R);  // one 64-bit division per block
    if (idx < p.n_init + p.n_evict) {
        const int64_t pos = p.pop0 + idx;
        const int slot = sl0 + w >= R ? sl0 + w - R : sl0 + w;
        const bool to_init = idx < p.n_init;
        int64_t u = 0;
        int off = 0;
        if (!to_init) {
            const int rel = static_cast<int>(pos - p.pend_start);  // < l_L + l_C: 32-bit division
            u = p.unit0 + rel / p.l_bs;
            off = rel % p.l_bs;
        }
        const int per = (p.d + 31) / 32;
        const int c0 = lane * per;
        int slo = slot + 1 == R ? 0 : slot + 1;
        int shi = slot + 1 + static_cast<int>(p.L);  // l_L < R: at most one wrap
        if (shi >= R) shi -= R;
        double tot = 0.0;
        for (int g = 0; g < p.G; ++g) {
            const T* rk = static_cast<const T*>(p.ring_k) + (static_cast<int64_t>(g) * R + slot) * p.d;
            double acc = 0.0;
            if (!to_init) {
                const double* Phi = p.P + (static_cast<int64_t>(shi) * p.G + g) * p.d;
                const double* Plo = p.P + (static_cast<int64_t>(slo) * p.G + g) * p.d;
                if (per == 4 && sizeof(T) == 2) {  // d = 128: 8-byte key slice, two 16-byte loads per P row
                    const uint2 kb = *reinterpret_cast<const uint2*>(rk + c0);
                    const double2 h0 = *reinterpret_cast<const double2*>(Phi + c0);
                    const double2 h1 = *reinterpret_cast<const double2*>(Phi + c0 + 2);
                    const double2 l0 = *reinterpret_cast<const double2*>(Plo + c0);
                    const double2 l1 = *reinterpret_cast<const double2*>(Plo + c0 + 2);
                    const T* kk = reinterpret_cast<const T*>(&kb);
                    acc += static_cast<double>(to_f(kk[0])) * (h0.x - l0.x);
                    acc += static_cast<double>(to_f(kk[1])) * (h0.y - l0.y);
                    acc += static_cast<double>(to_f(kk[2])) * (h1.x - l1.x);
                    acc += static_cast<double>(to_f(kk[3])) * (h1.y - l1.y);
                } else {
                    for (int j = 0; j < per; ++j) {
                        const int c = c0 + j;
                        if (c < p.d) acc += static_cast<double>(to_f(rk[c])) * (Phi[c] - Plo[c]);
                    }
                }
            }
            if (!(p.page_mode && !to_init)) {  // page mode: k_select copies whole unit pages
                T* dk = to_init ? static_cast<T*>(p.init_k) + (static_cast<int64_t>(g) * p.l_I + pos) * p.d
                                : static_cast<T*>(p.unit_k) + ((u * p.G + g) * p.l_bs + off) * p.d;
                T* dkr = !p.absolute ? nullptr
                         : to_init   ? static_cast<T*>(p.init_krot) + (static_cast<int64_t>(g) * p.l_I + pos) * p.d
                                     : static_cast<T*>(p.unit_krot) + ((u * p.G + g) * p.l_bs + off) * p.d;
                const T* rkr = static_cast<const T*>(p.ring_krot) + (static_cast<int64_t>(g) * R + slot) * p.d;
                for (int c = lane; c < p.d; c += 32) {
                    dk[c] = rk[c];
                    if (dkr) dkr[c] = rkr[c];
                }
                const T* rv = static_cast<const T*>(p.ring_v);
                T* dvb = static_cast<T*>(to_init ? p.init_v : p.unit_v);
                for (int c = lane; c < p.dv; c += 32) {
                    const T x = rv[p.vl.ring(g, pos, c)];
                    if (to_init)
                        dvb[p.vl.init(g, pos, c)] = x;
                    else
                        dvb[p.vl.unit(u, g, off, c)] = x;
                }
            }
            if (to_init) continue;
            acc = warp_sum_d(acc);
            if (!p.fused) {
                if (lane == 0) p.ev_part[(idx - p.n_init) * p.Gtot + p.g0 + g] = acc;
            } else {
                tot += acc;
            }
        }
        if (!to_init && p.fused && lane == 0)
            p.unit_scores[u * p.l_bs + off] = static_cast<float>(tot / static_cast<double>(p.L));
    }
    TL_END(TL_EVICT);
}

template <typename T>
void launch_evict(const EvictParams& p, cudaStream_t st) {
    const int64_t n = p.n_init + p.n_evict;
    if (n <= 0) return;
    k_evict_warp<T><<<static_cast<unsigned>((n + kEvWarps - 1) / kEvWarps), kEvWarps * 32, 0, st>>>(p);
}
template void launch_evict<float>(const EvictParams&, cudaStream_t);
template void launch_evict<bf16>(const EvictParams&, cudaStream_t);

// finalize_front (repr_score.hpp:72-82): r_m = (sum_g part) / l_L, narrowed to float
__global__ void k_finalize(FinalizeParams p) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= p.n_evict) return;
    double a = 0.0;
    for (int g = 0; g < p.Gtot; ++g) a += p.ev_part[e * p.Gtot + g];
    const int64_t rel = p.e0 + e - p.pend_start;
    const int64_t u = p.unit0 + rel / p.l_bs, off = rel % p.l_bs;
    p.unit_scores[u * p.l_bs + off] = static_cast<float>(a / static_cast<double>(p.L));
}

void launch_finalize(const FinalizeParams& p, cudaStream_t st) {
    if (p.n_evict > 0) k_finalize<<<static_cast<unsigned>((p.n_evict + 127) / 128), 128, 0, st>>>(p);
}

// K6 select_representatives (repr_score.hpp:94-112) + repr-key gather
// (memory.hpp:111-123, 200-208): warp per unit, r_k rounds of warp argmax
// over (score desc, index asc), output ascending.
__device__ void warp_select(const float* sc, int len, int r_k, int* out) {
    const int lane = threadIdx.x % 32;
    const int take = min(r_k, len);
    unsigned long long taken[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // per-lane bitmask of taken slots (len <= 32*64)
    for (int r = 0; r < take; ++r) {
        float bv = -INFINITY;
        int bi = INT32_MAX;
        for (int j = lane, t = 0; j < len; j += 32, ++t) {
            if (taken[t >> 6] >> (t & 63) & 1ull) continue;
            const float x = sc[j];
            if (bi == INT32_MAX || x > bv || (x == bv && j < bi)) {
                bv = x;
                bi = j;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (oi != INT32_MAX && (bi == INT32_MAX || ov > bv || (ov == bv && oi < bi))) {
                bv = ov;
                bi = oi;
            }
        }
        if (bi % 32 == lane) {
            const int t = bi / 32;
            taken[t >> 6] |= 1ull << (t & 63);
        }
        out[r] = bi;
    }
    // ascending
    for (int a = 1; a < take; ++a) {
        const int x = out[a];
        int b = a - 1;
        while (b >= 0 && out[b] > x) {
            out[b + 1] = out[b];
            --b;
        }
        out[b + 1] = x;
    }
}

// page mode: block = (unit, group): the unit's K (and K_rot) rows and its V
// page are contiguous 32 KB blocks of the ring (slots pos0 + 128 i .. + 127,
// no wrap since R is a multiple of 128): copied with 16-byte vectors by
// threads [32, blockDim) while warp 0 selects the representatives
template <typename T>
__device__ __forceinline__ int64_t select_page_slot(const SelectParams& p, int64_t u) {
    return (p.pos0 + 128 * (u - p.u0)) % p.R;
}
template <typename T>
__device__ void select_page_copy(const SelectParams& p, int64_t u, int g, int tid, int nthr) {
    const int64_t slot = select_page_slot<T>(p, u);
    const int64_t rowb = static_cast<int64_t>(128) * p.d * static_cast<int64_t>(sizeof(T)) / 16;  // uint4 per K page
    const uint4* sk = reinterpret_cast<const uint4*>(static_cast<const T*>(p.ring_k) + (g * p.R + slot) * p.d);
    uint4* dk = reinterpret_cast<uint4*>(static_cast<T*>(const_cast<void*>(p.unit_k)) + ((u * p.G + g) * 128) * p.d);
    const int64_t vb = static_cast<int64_t>(128) * p.dv * static_cast<int64_t>(sizeof(T)) / 16;
    const T* rv = static_cast<const T*>(p.ring_v);
    T* uv = static_cast<T*>(p.unit_v);
    // both layouts keep a unit's values contiguous: V^T page [dv][128] or rows [128][dv]
    const uint4* sv = reinterpret_cast<const uint4*>(rv + (p.vl.vt ? p.vl.ring(g, slot, 0) : (g * p.R + slot) * p.dv));
    uint4* dv = reinterpret_cast<uint4*>(uv + p.vl.unit(u, g, 0, 0));
    // K and V pages: 8 + 8 independent 16-byte loads in flight per thread, then the stores
    for (int64_t t0 = 0; t0 < rowb || t0 < vb; t0 += 8 * static_cast<int64_t>(nthr)) {
        uint4 rk4[8], rv4[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int64_t t = t0 + tid + i * static_cast<int64_t>(nthr);
            if (t < rowb) rk4[i] = sk[t];
            if (t < vb) rv4[i] = sv[t];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int64_t t = t0 + tid + i * static_cast<int64_t>(nthr);
            if (t < rowb) dk[t] = rk4[i];
            if (t < vb) dv[t] = rv4[i];
        }
    }
    if (p.absolute) {
        const uint4* skr = reinterpret_cast<const uint4*>(static_cast<const T*>(p.ring_krot) + (g * p.R + slot) * p.d);
        uint4* dkr = reinterpret_cast<uint4*>(static_cast<T*>(p.unit_krot) + ((u * p.G + g) * 128) * p.d);
        for (int64_t t = tid; t < rowb; t += nthr) dkr[t] = skr[t];
    }
}
// representative rows of this group straight from the ring (memory.hpp:111-123)
template <typename T>
__device__ void select_page_repr(const SelectParams& p, int64_t u, int g, const int* idx, int take) {
    const int64_t slot = select_page_slot<T>(p, u);
    const T* rk = static_cast<const T*>(p.ring_k) + (g * p.R + slot) * p.d;
    T* rp = static_cast<T*>(p.repr) + ((u * p.G + g) * p.r_k) * p.d;
    const int nv = p.d * static_cast<int>(sizeof(T)) / 16;
    for (int t = threadIdx.x; t < p.r_k * nv; t += blockDim.x) {
        const int r = t / nv, c = t % nv;
        uint4 x = make_uint4(0, 0, 0, 0);
        if (r < take) x = reinterpret_cast<const uint4*>(rk + idx[r] * p.d)[c];
        reinterpret_cast<uint4*>(rp + r * p.d)[c] = x;
    }
}

template <typename T>
__device__ __forceinline__ void select_body(const SelectParams& p) {
    __shared__ int idx[32];
    const int64_t u = p.u0 + blockIdx.x;
    const int len = p.unit_len[u];
    const int take = min(p.r_k, len);
    if (threadIdx.x < 32) {
        int r[32];
        warp_select(p.unit_scores + u * p.l_bs, len, p.r_k, r);
        if (threadIdx.x == 0)
            for (int k = 0; k < take; ++k) idx[k] = r[k];
        if (threadIdx.x < p.r_k && blockIdx.y == 0)
            p.repr_idx[u * p.r_k + threadIdx.x] = threadIdx.x < take ? r[threadIdx.x] : -1;
    } else if (p.page_mode) {
        select_page_copy<T>(p, u, static_cast<int>(blockIdx.y), threadIdx.x - 32, blockDim.x - 32);
    }
    __syncthreads();
    if (p.page_mode) {
        select_page_repr<T>(p, u, static_cast<int>(blockIdx.y), idx, take);
        return;
    }
    const T* uk = static_cast<const T*>(p.unit_k);
    T* rp = static_cast<T*>(p.repr);
    // repr[u][g][r][:] = key row idx[r] of the unit (memory.hpp:111-123);
    // units shorter than r_k (final flush) get zero rows, which add 0 to relevance
    if ((p.d * sizeof(T)) % 16 == 0) {
        const int nv = p.d * static_cast<int>(sizeof(T)) / 16;
        const int n = p.G * p.r_k * nv;
        for (int t = threadIdx.x; t < n; t += blockDim.x) {
            const int g = t / (p.r_k * nv), rem = t % (p.r_k * nv), r = rem / nv, c = rem % nv;
            uint4 x = make_uint4(0, 0, 0, 0);
            if (r < take) x = reinterpret_cast<const uint4*>(uk + ((u * p.G + g) * p.l_bs + idx[r]) * p.d)[c];
            reinterpret_cast<uint4*>(rp + ((u * p.G + g) * p.r_k + r) * p.d)[c] = x;
        }
        return;
    }
    const int n = p.G * p.r_k * p.d;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        const int g = t / (p.r_k * p.d), rem = t % (p.r_k * p.d), r = rem / p.d, c = rem % p.d;
        rp[((u * p.G + g) * p.r_k + r) * p.d + c] =
            r < take ? uk[((u * p.G + g) * p.l_bs + idx[r]) * p.d + c] : from_f<T>(0.f);
    }
}

template <typename T>
__global__ void __launch_bounds__(512) k_select(SelectParams p) {
    TL_BEGIN();
    select_body<T>(p);
    TL_END(TL_SELECT);
}

template <typename T>
void launch_select(const SelectParams& p, cudaStream_t st) {
    if (p.n_units <= 0) return;
    k_select<T><<<dim3(static_cast<unsigned>(p.n_units), p.page_mode ? p.G : 1), p.page_mode ? 512 : 128, 0, st>>>(p);
}
template void launch_select<float>(const SelectParams&, cudaStream_t);
template void launch_select<bf16>(const SelectParams&, cudaStream_t);

__global__ void k_select_standalone(const float* scores, const int64_t* lens, int64_t n_units, int64_t unit_len,
                                    int64_t r_k, int64_t* out) {
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t u = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + warp;
    if (u >= n_units) return;
    const int len = static_cast<int>(lens ? lens[u] : unit_len);
    int idx[32];
    warp_select(scores + u * unit_len, len, static_cast<int>(r_k), idx);
    const int take = static_cast<int>((r_k < len ? r_k : (int64_t)len));
    if (lane < r_k) out[u * r_k + lane] = lane < take ? idx[lane] : -1;
}

void launch_select_standalone(const float* scores, const int64_t* lens, int64_t n_units, int64_t unit_len,
                              int64_t r_k, int64_t* idx, cudaStream_t st) {
    if (n_units <= 0) return;
    k_select_standalone<<<static_cast<unsigned>((n_units + 3) / 4), 128, 0, st>>>(scores, lens, n_units, unit_len,
                                                                                  r_k, idx);
}

}  // namespace infllm

namespace infllm {

// ---- decode front: K7 prep of one token + eviction of the token leaving the
// local window, one block of 32 x G threads per sequence (warp = KV group).
// Same arithmetic as k_rope_table + k_prep_tok + k_prefix_tiles +
// k_evict_tok at l_x = 1 (rope factors from fp64 angles, query sums in head
// order, P[s+1] = P[s] + qs, r_m from the prefix difference), in one launch.
__device__ __forceinline__ void dec_front_body(const PrepParams& p, const EvictParams& ep,
                                               unsigned long long mark = 0) {
    const int g = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t pos = p.s;
    // the d/2 rotation factors of this position, one fp64 sincos per thread in
    // parallel (rotary.hpp:25-30; the large-argument reduction is the slow part)
    __shared__ float2 s_rc[128], s_cl[128];
    for (int a = threadIdx.x; a < p.d / 2; a += blockDim.x) {
        float c, sn;
        rope_cs(p.freqs, a, pos, c, sn);
        s_rc[a] = make_float2(c, sn);
        s_cl[a] = make_float2(p.freqs.cL[a], p.freqs.sL[a]);  // lanes index it by dim: no divergent constant loads
    }
    __syncthreads();
    TL_MARK(40, mark);  // rotation factors
    // ring slots of this position and the next, computed once (64-bit division
    // is a subroutine on the GPU)
    const int R = static_cast<int>(p.R);
    const int slot = static_cast<int>(pos % p.R), slot1 = slot + 1 == R ? 0 : slot + 1;
    if (lane < 16) {
        const int c8 = lane;
        // this position's prefix row, loaded with the inputs
        const double* Pin = p.P + (static_cast<int64_t>(slot) * p.G + g) * p.d + 8 * c8;
        double pin[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) pin[e] = Pin[e];
        const bf16* qg = static_cast<const bf16*>(p.q);
        constexpr int kMaxRep = 8;
        V8<bf16> qv[kMaxRep];
#pragma unroll
        for (int hh = 0; hh < kMaxRep; ++hh)
            if (hh < p.rep) qv[hh] = ld8(qg + (g * p.rep + hh) * p.d + 8 * c8);
        const V8<bf16> kv = ld8(static_cast<const bf16*>(p.k) + g * p.d + 8 * c8);
        const V8<bf16> vv = ld8(static_cast<const bf16*>(p.v) + g * p.dv + 8 * c8);
        float2 f[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) f[j] = s_rc[4 * c8 + j];
        V8<bf16> kr;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float y0, y1;
            rope_pair(to_f(kv.v[2 * j]), to_f(kv.v[2 * j + 1]), f[j].x, f[j].y, y0, y1);
            kr.v[2 * j] = from_f<bf16>(y0);
            kr.v[2 * j + 1] = from_f<bf16>(y1);
        }
        float kn2 = 0.f;  // |k|^2, as k_prep_tok
#pragma unroll
        for (int e = 0; e < 8; ++e) kn2 = fmaf(to_f(kv.v[e]), to_f(kv.v[e]), kn2);
        const int64_t ro = (static_cast<int64_t>(g) * R + slot) * p.d + 8 * c8;
        st8(static_cast<bf16*>(p.ring_k) + ro, kv);
        st8(static_cast<bf16*>(p.ring_krot) + ro, kr);
        double qs[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int hh = 0; hh < kMaxRep; ++hh) {
            if (hh >= p.rep) break;
            V8<bf16> qa, qc;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float x0 = to_f(qv[hh].v[2 * j]), x1 = to_f(qv[hh].v[2 * j + 1]);
                float y0, y1;
                rope_pair(x0, x1, f[j].x, f[j].y, y0, y1);
                qa.v[2 * j] = from_f<bf16>(y0);
                qa.v[2 * j + 1] = from_f<bf16>(y1);
                const int a = 4 * c8 + j;
                rope_pair(x0, x1, s_cl[a].x, s_cl[a].y, y0, y1);
                qc.v[2 * j] = from_f<bf16>(y0);
                qc.v[2 * j + 1] = from_f<bf16>(y1);
                qs[2 * j] += static_cast<double>(x0);
                qs[2 * j + 1] += static_cast<double>(x1);
            }
            const int64_t qo = (static_cast<int64_t>(g * p.rep + hh) * p.lxp) * p.d + 8 * c8;
            st8(static_cast<bf16*>(p.qa) + qo, qa);
            st8(static_cast<bf16*>(p.qc) + qo, qc);
        }
        bf16* rv = static_cast<bf16*>(p.ring_v);
        if (p.vl.vt) {  // transposed value pages [G][R/128][dv][128]
            const int64_t vb = ((static_cast<int64_t>(g) * (R / 128) + slot / 128) * p.dv + 8 * c8) * 128 + slot % 128;
#pragma unroll
            for (int e = 0; e < 8; ++e) rv[vb + 128 * e] = vv.v[e];
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) rv[p.vl.ring(g, pos, 8 * c8 + e)] = vv.v[e];
        }
        // prefix ring and chunk query sum (k_prefix_tiles at l_x = 1)
        double* Pout = p.P + (static_cast<int64_t>(slot1) * p.G + g) * p.d + 8 * c8;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            Pout[e] = pin[e] + qs[e];
            p.chunk_qsum[g * p.d + 8 * c8 + e] = 0.0 + (qs[e] + 0.0);
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) kn2 += __shfl_xor_sync(0x0000ffffu, kn2, o);
        if (lane == 0 && p.kmax2) p.kmax2[g] = fmaxf(p.kmax2_prev[g], kn2);
    }
    if (ep.n_init + ep.n_evict == 0) return;  // uniform: nothing leaves the window this step
    __syncthreads();  // this step's P row is read by the eviction score
    TL_MARK(41, mark);  // prep of the token
    evict_tok_body<bf16>(ep);
    TL_MARK(42, mark);  // eviction of the token leaving the window
}
__global__ void __launch_bounds__(256) k_dec_front(PrepParams p, EvictParams ep) {
    // decode chain: K4 may launch now (it waits for this grid); this grid ends
    // only after the lookup it overlaps, so K4's wait covers both
    if (p.dec_chain) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    TL_BEGIN();
    dec_front_body(p, ep, tl_t0_);
    if (p.dec_chain) asm volatile("griddepcontrol.wait;" ::: "memory");
    TL_END(TL_DEC_FRONT);
}
struct DecFront {
    PrepParams p;
    EvictParams ep;
};
__global__ void __launch_bounds__(256) k_dec_front_b(const DecFront* __restrict__ fs, int chain) {
    TL_BEGIN();
    // this sequence's parameters (rotation constants included) in shared memory:
    // the body reads them all through its phases
    __shared__ __align__(16) DecFront sf;
    static_assert(sizeof(DecFront) % 4 == 0, "word copy");
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(DecFront) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t*>(&sf)[i] = reinterpret_cast<const uint32_t*>(fs + blockIdx.z)[i];
    __syncthreads();
    dec_front_body(sf.p, sf.ep);
    // batch chain: launched as the relevance scan's programmatic dependent, it ends
    // after the scan, so the launches that follow see both
    if (chain) asm volatile("griddepcontrol.wait;" ::: "memory");
    TL_END(TL_DEC_FRONT);
}
bool dec_front_supported(const PrepParams& p) {
    return p.d == 128 && p.dv == 128 && p.rep <= 8 && p.G <= 8 && p.lx == 1 && p.vl.vt;  // one warp per group
}
void launch_dec_front(const PrepParams& p, const EvictParams& ep, cudaStream_t st) {
    if (!p.dec_chain) {
        k_dec_front<<<1, 32 * p.G, 0, st>>>(p, ep);
        return;
    }
    cudaLaunchConfig_t cfg{};  // programmatic dependent of the lookup launched just before
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32 * p.G);
    cfg.stream = st;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = la;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_dec_front, p, ep);
}
void launch_dec_front_batch(const void* tab, int B, int G, cudaStream_t st, int chain) {
    if (!chain) {
        k_dec_front_b<<<dim3(1, 1, B), 32 * G, 0, st>>>(static_cast<const DecFront*>(tab), 0);
        return;
    }
    cudaLaunchConfig_t cfg{};  // programmatic dependent of the scan launched just before
    cfg.gridDim = dim3(1, 1, B);
    cfg.blockDim = dim3(32 * G);
    cfg.stream = st;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = la;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_dec_front_b, static_cast<const DecFront*>(tab), 1);
}
size_t dec_front_size() { return sizeof(DecFront); }

// ---- batched decode: one launch per stage for B sequences (grid.z = sequence;
// per-sequence parameter tables in device memory) -------------------------------
__global__ void k_rope_table_b(const PrepParams* __restrict__ ps) {
    rope_table_body(ps[blockIdx.z], static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x);
}
__global__ void __launch_bounds__(kTokTile * 16) k_prep_tok_b(const PrepParams* __restrict__ ps) {
    unsigned long long mark = 0;
    prep_tok_body<bf16, 0>(ps[blockIdx.z], blockIdx.x, blockIdx.y, mark);
}
__global__ void __launch_bounds__(128) k_prefix_tiles_b(const PrepParams* __restrict__ ps) {
    prefix_tiles_body<bf16>(ps[blockIdx.z], blockIdx.x, blockIdx.y, gridDim.x);
}
__global__ void __launch_bounds__(256) k_evict_tok_b(const EvictParams* __restrict__ ps) {
    const EvictParams& p = ps[blockIdx.z];
    if (blockIdx.x >= p.n_init + p.n_evict) return;
    evict_tok_body<bf16>(p);
}
__global__ void __launch_bounds__(256) k_select_b(const SelectParams* __restrict__ ps) {
    const SelectParams& p = ps[blockIdx.z];
    if (blockIdx.x >= p.n_units) return;
    TL_BEGIN();
    select_body<bf16>(p);
    TL_END(TL_SELECT);
}
// streaming relevance scan per sequence slice (8 warps, bulk-copy ring per warp); rel[u] only
__device__ __forceinline__ int stream_blocks(int64_t U) { return static_cast<int>((U + 255) / 256); }
__global__ void __launch_bounds__(256, 1) k_lookup_stream_b(const LookupParams* __restrict__ ps) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the top-k (or front) may launch (PDL)
    const LookupParams& p = ps[blockIdx.z];
    const int nb = stream_blocks(p.U);
    if (static_cast<int>(blockIdx.x) >= nb) return;
    lookup_stream_body(p, nb);
}
// balanced variant: one block per SM over the concatenated unit ranges of all
// sequences (contiguous share per block, warps strided inside it), so a batch
// of long indices has no partial last wave; same per-unit arithmetic and order
// as lookup_stream_body (bit-identical rel[u]).
constexpr int kScanMaxB = 256;
__global__ void __launch_bounds__(256, 1) k_lookup_stream_bal(const LookupParams* __restrict__ ps, int B) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the top-k blocks may launch (PDL)
    TL_BEGIN();
    extern __shared__ __align__(16) uint8_t scan_smem[];
    __shared__ int64_t s_off[kScanMaxB + 1];
    __shared__ const uint8_t* s_repr[kScanMaxB];
    __shared__ const double* s_q[kScanMaxB];
    __shared__ const uint2* s_qt[kScanMaxB];  // batch chain: the token's q rows (query sums formed here)
    __shared__ double* s_rel[kScanMaxB];
    __shared__ __align__(8) uint64_t sbar[8][kScanStages];
    const int lane = threadIdx.x % 32, wib = threadIdx.x / 32;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        s_repr[b] = static_cast<const uint8_t*>(ps[b].repr);
        s_q[b] = ps[b].qsum;
        s_qt[b] = static_cast<const uint2*>(ps[b].qtok);
        s_rel[b] = ps[b].rel;
    }
    if (threadIdx.x == 0) {
        int64_t o = 0;
        for (int b = 0; b < B; ++b) {
            s_off[b] = o;
            o += ps[b].U;
        }
        s_off[B] = o;
    }
    const int G = ps[0].G, qrep = ps[0].qrep;
    if (lane == 0)
        for (int st = 0; st < kScanStages; ++st) tc::mbar_init(&sbar[wib][st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const int64_t total = s_off[B];
    const int64_t S = (total + gridDim.x - 1) / gridDim.x;
    const int64_t s0 = static_cast<int64_t>(blockIdx.x) * S, s1 = s0 + S < total ? s0 + S : total;
    const int64_t nwarps = blockDim.x / 32;
    const int64_t bytes_u = static_cast<int64_t>(G) * 512 * 2;
    uint8_t* ring = scan_smem + static_cast<size_t>(wib) * kScanStages * 8192;
    int ib = 0, cb = -1;  // sequence cursors of the issue side and the compute side (t only grows)
    auto seq_of = [&](int64_t t, int& c) {
        while (c + 1 < B && t >= s_off[c + 1]) ++c;
        return c;
    };
    auto issue = [&](int64_t t, int stage) {
        if (t < s1 && lane == 0) {
            const int b = seq_of(t, ib);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tc::mbar_expect_tx(&sbar[wib][stage], static_cast<uint32_t>(bytes_u));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             tc::smem_u32(ring + stage * 8192)),
                         "l"(s_repr[b] + (t - s_off[b]) * bytes_u), "r"(static_cast<uint32_t>(bytes_u)),
                         "r"(tc::smem_u32(&sbar[wib][stage]))
                         : "memory");
        }
    };
    const int64_t warp0 = s0 + wib;
#pragma unroll
    for (int st = 0; st < kScanStages - 1; ++st) issue(warp0 + st * nwarps, st);
    double q[8][4];
    int stage = 0;
    int64_t it = 0;
    for (int64_t t = warp0; t < s1; t += nwarps, ++it) {
        issue(t + (kScanStages - 1) * nwarps, (stage + kScanStages - 1) % kScanStages);
        int b = cb;
        if (b < 0 || t >= s_off[b + 1]) {  // first unit of a sequence for this warp: its query sums
            if (cb < 0) cb = 0;
            b = seq_of(t, cb);
            if (s_qt[b]) {  // sums over the group's heads in head order from 0.0 (as lk_qsum)
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
                    if (g < G) {
                        const uint2* qq = s_qt[b] + static_cast<int64_t>(g) * qrep * 32 + lane;
                        uint2 v[8];
#pragma unroll
                        for (int hh = 0; hh < 8; ++hh)
                            if (hh < qrep) v[hh] = qq[hh * 32];
#pragma unroll
                        for (int hh = 0; hh < 8; ++hh)
                            if (hh < qrep) {
                                a0 += static_cast<double>(__uint_as_float(v[hh].x << 16));
                                a1 += static_cast<double>(__uint_as_float(v[hh].x & 0xffff0000u));
                                a2 += static_cast<double>(__uint_as_float(v[hh].y << 16));
                                a3 += static_cast<double>(__uint_as_float(v[hh].y & 0xffff0000u));
                            }
                    }
                    q[g][0] = a0;
                    q[g][1] = a1;
                    q[g][2] = a2;
                    q[g][3] = a3;
                }
            } else {
#pragma unroll
                for (int g = 0; g < 8; ++g)
#pragma unroll
                    for (int j = 0; j < 4; ++j) q[g][j] = g < G ? s_q[b][g * 128 + 4 * lane + j] : 0.0;
            }
        }
        tc::mbar_wait(&sbar[wib][stage], static_cast<uint32_t>((it / kScanStages) & 1));
        const uint8_t* buf = ring + stage * 8192 + 8 * lane;
        double rel = 0.0;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            if (g >= G) break;
            double a = 0.0;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint2 v = *reinterpret_cast<const uint2*>(buf + (4 * g + r) * 256);
                a = fma(q[g][0], static_cast<double>(__uint_as_float(v.x << 16)), a);
                a = fma(q[g][1], static_cast<double>(__uint_as_float(v.x & 0xffff0000u)), a);
                a = fma(q[g][2], static_cast<double>(__uint_as_float(v.y << 16)), a);
                a = fma(q[g][3], static_cast<double>(__uint_as_float(v.y & 0xffff0000u)), a);
            }
            rel += a;
        }
        rel = warp_sum_d(rel);
        if (lane == 0) s_rel[b][t - s_off[b]] = rel;
        __syncwarp();  // the stage is refilled next iteration
        stage = (stage + 1) % kScanStages;
    }
    TL_END(TL_LOOKUP);
}
__global__ void __launch_bounds__(1024) k_topk_b(const LookupParams* __restrict__ ps, int late) {
    // programmatic dependent of the scan: K4 may launch now; the relevance must be complete.
    // late (batch chain, the fronts between the scan and this launch): K4 launches only
    // once the fronts (which end after the scan) are complete
    if (!late) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (late) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    TL_BEGIN();
    const LookupParams& p = ps[blockIdx.x];
    block_topk_radix(p.rel, p.U, p.n_sel, p.sel);
    TL_END(TL_TOPK);
}
__global__ void __launch_bounds__(256) k_lru_b(const LruParams* __restrict__ ps) {
    TL_BEGIN();
    lru_body(ps[blockIdx.x]);
    TL_END(TL_LRU);
}

void launch_decode_batch_stage(int stage, const void* tab, int B, int64_t gx, cudaStream_t st) {
    switch (stage) {
        case 0: {  // K7 prep of one token per sequence (the chunk-path kernels, l_x = 1)
            const PrepParams* ps = static_cast<const PrepParams*>(tab);
            k_rope_table_b<<<dim3(1, 1, B), 256, 0, st>>>(ps);
            k_prep_tok_b<<<dim3(1, static_cast<unsigned>(gx), B), kTokTile * 16, 0, st>>>(ps);
            k_prefix_tiles_b<<<dim3(1, static_cast<unsigned>(gx), B), 128, 0, st>>>(ps);
            break;
        }
        case 1:  // eviction of the token(s) leaving the local window (gx = max tokens; block = 32 x G)
            k_evict_tok_b<<<dim3(static_cast<unsigned>(gx & 0xffffffff), 1, B), static_cast<unsigned>(32 * (gx >> 32)), 0, st>>>(
                static_cast<const EvictParams*>(tab));
            break;
        case 2:  // completed units: representative selection + page copy (gx = max units; grid.y = G)
            k_select_b<<<dim3(static_cast<unsigned>(gx & 0xffffffff), static_cast<unsigned>(gx >> 32), B), 256, 0, st>>>(
                static_cast<const SelectParams*>(tab));
            break;
        case 3:    // relevance scan + exact top-k (rel desc, id asc)
        case 5: {  // the scan alone (6: the top-k alone)
            const LookupParams* ps = static_cast<const LookupParams*>(tab);
            const size_t smem = static_cast<size_t>(8) * kScanStages * 8192;
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(k_lookup_stream_b, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
                attr = true;
            }
            if (B <= kScanMaxB) {
                static bool attr2 = false;
                if (!attr2) {
                    cudaFuncSetAttribute(k_lookup_stream_bal, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
                    attr2 = true;
                }
                // one block per SM (fewer when the batch's units are few: >= 8 units per block,
                // one per warp; with >= 64 per block, B = 4 at 128K scanned in 61 blocks: 20.3
                // vs 13.3 us)
                const int64_t units = (gx & 0xffffffff);
                const unsigned nb = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(148, units / 8)));
                k_lookup_stream_bal<<<nb, 256, smem, st>>>(ps, B);
            } else {
                k_lookup_stream_b<<<dim3(static_cast<unsigned>(gx >> 32), 1, B), 256, smem, st>>>(ps);
            }
            if (stage == 5) break;  // batch chain: the front (and a completed unit's copy) come between
            [[fallthrough]];
        }
        case 6:
        case 7: {  // 7: the top-k alone, its dependents released after its wait (batch chain)
            const LookupParams* ps = static_cast<const LookupParams*>(tab);
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(static_cast<unsigned>(B));
            // one block per sequence, 8 keys per thread where they fit (fewer warps per
            // barrier): 256 threads up to 2048 units, 512 up to 4096, else 1024
            cfg.blockDim = dim3((gx >> 32) <= 8 ? 256 : (gx >> 32) <= 16 ? 512 : 1024);
            cfg.stream = st;
            cudaLaunchAttribute la[1];
            la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            la[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = la;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_topk_b, ps, stage == 7 ? 1 : 0);
            break;
        }
        case 4:  // LRU / tier bookkeeping
            k_lru_b<<<B, 256, 0, st>>>(static_cast<const LruParams*>(tab));
            break;
        default:
            break;
    }
}
int64_t decode_batch_lookup_blocks(int64_t U) {  // per-sequence stream-scan blocks << 32
    return ((U + 255) / 256) << 32;
}
}  // namespace infllm
