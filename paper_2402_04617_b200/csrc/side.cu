// side.cu — the chunk-step side kernels of the prefill pipeline written for a
// small SM footprint: the tcgen05 attention holds 128 of the 148 SMs with one
// CTA each, so everything else of a step (prep of step t+2, eviction and
// scoring of step t, lookup of step t+1, LRU) has to run on the ~20 SMs left,
// with enough bytes in flight per SM to finish inside one attention.
//
// K7 k_prep_chunk (bf16, head_dim = value_dim = 128, <= 8 query heads per KV
// group, transposed value pages): one block per 32-token tile of the chunk
// (16 blocks at l_C = 512), looping over the KV groups. Per (tile, group) the
// q rows of the group's heads, k and v rows arrive by bulk copies (TMA engine)
// into a double-buffered shared-memory stage while the previous group is
// computed: RoPE (rotary.hpp:15-72; fp64 angles, factors computed once per
// tile and shared by the groups), q_abs = rope(q, pos), q_clamp = rope(q, l_L)
// (attention.hpp:166-167), raw and rotated keys and transposed values into the
// ring, the fp64 group query sums qs_t and their prefix P[t] = P[s] + sum qs
// (the band sums of ScoreAccumulator, repr_score.hpp:53-57, become prefix
// differences at eviction). The prefix across tiles is a decoupled look-back:
// tiles take tickets in launch order, publish their 16-token sub-tile sums per
// group and wait only for lower tickets, so no second kernel is needed. The
// additions happen in exactly the order of the three-kernel path (rope table,
// k_prep_tok, k_prefix_tiles), so every value is bitwise the same.
#include "kernels.cuh"
#include "tc_prims.cuh"

namespace infllm {

namespace {
constexpr int kPcTok = 32;       // tokens per tile (one block)
constexpr int kPcThreads = 512;  // 32 tokens x 16 chunks of 8 dims
constexpr int kPcSqs = kPcTok * (128 + 2) * 8;       // fp64 group query sums of the tile
constexpr int kPcSvt = 128 * (kPcTok + 8) * 2;       // transposed values
constexpr int kPcRope = kPcTok * 64 * 8;             // rotation factors
}  // namespace

struct PrepSync {
    unsigned ticket, done;
    int flags[kPrepChunkMaxTiles][8];
};

size_t prep_chunk_sync_bytes() { return sizeof(PrepSync); }

bool prep_chunk_supported(const PrepParams& p) {
    return p.d == 128 && p.dv == 128 && (p.rep == 1 || p.rep == 2 || p.rep == 4 || p.rep == 8) && p.G >= 1 &&
           p.G <= 8 && p.vl.vt && p.lx >= 1 && (p.lx + kPcTok - 1) / kPcTok <= kPrepChunkMaxTiles && p.sync && p.qs &&
           p.tsum;
}

template <int REP>
struct PcIn {
    uint4 q[REP];
    uint4 k, v;
};
template <int REP>
__device__ __forceinline__ void pc_load(const PrepParams& p, int64_t i, int g, int c8, bool live, PcIn<REP>& x) {
    if (!live) return;
    const uint4* qp = reinterpret_cast<const uint4*>(static_cast<const bf16*>(p.q) + (i * p.H + g * REP) * 128) + c8;
#pragma unroll
    for (int hh = 0; hh < REP; ++hh) x.q[hh] = __ldcs(qp + hh * 16);
    x.k = __ldcs(reinterpret_cast<const uint4*>(static_cast<const bf16*>(p.k) + (i * p.G + g) * 128) + c8);
    x.v = __ldcs(reinterpret_cast<const uint4*>(static_cast<const bf16*>(p.v) + (i * p.G + g) * 128) + c8);
}

template <int REP>
__global__ void __launch_bounds__(kPcThreads, 1) k_prep_chunk(PrepParams p) {
    TL_BEGIN();
    using T = bf16;
    extern __shared__ __align__(128) uint8_t pc_smem[];
    auto sqs = reinterpret_cast<double(*)[128 + 2]>(pc_smem);
    auto svt = reinterpret_cast<T(*)[kPcTok + 8]>(pc_smem + kPcSqs);
    auto srope = reinterpret_cast<float2(*)[64]>(pc_smem + kPcSqs + kPcSvt);
    __shared__ int s_tile;
    PrepSync* sync = static_cast<PrepSync*>(p.sync);
    const int tid = threadIdx.x, lane = tid % 32;
    const int tt = tid / 16, c8 = tid % 16;
    if (tid == 0) s_tile = static_cast<int>(atomicAdd(&sync->ticket, 1u));  // launch order: the look-back only waits on running blocks
    __syncthreads();
    const int tile = s_tile;
    const int ntile = static_cast<int>((p.lx + kPcTok - 1) / kPcTok);
    const int64_t i0 = static_cast<int64_t>(tile) * kPcTok;
    const int nt = static_cast<int>(min(static_cast<int64_t>(kPcTok), p.lx - i0));
    const int64_t i = i0 + tt;
    const bool live = tt < nt;
    const int64_t pos = p.s + i;
    const int64_t stride = static_cast<int64_t>(p.G) * 128;
    // ring slots, computed once (64-bit division is a subroutine call on the GPU)
    const int R = static_cast<int>(p.R);
    const int slot = static_cast<int>(pos % p.R);               // this thread's token
    const int slot_t0 = static_cast<int>((p.s + i0) % p.R);      // the tile's first token
    const int s0_slot = static_cast<int>(p.s % p.R);             // P row of the chunk start

    PcIn<REP> in0, in1;
    pc_load<REP>(p, i, 0, c8, live, in0);
    // rotation factors of the tile's positions (rotary.hpp:25-30), shared by every group
    for (int t = tid; t < kPcTok * 64; t += kPcThreads) {
        const int j = t / 64, a = t % 64;
        float c = 0.f, s = 0.f;
        if (j < nt) rope_cs(p.freqs, a, p.s + i0 + j, c, s);
        srope[j][a] = make_float2(c, s);
    }
    __syncthreads();
    unsigned long long mark = tl_t0_;
#define PC_MARK(k) TL_MARK(20 + (k), mark)
    PC_MARK(0);
    float2 f[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) f[j] = srope[tt][4 * c8 + j];

    // phase 1: per group, the next group's rows in flight while this one is computed
    auto group = [&](int g, const PcIn<REP>& x, PcIn<REP>& nx) {
        if (g + 1 < p.G) pc_load<REP>(p, i, g + 1, c8, live, nx);
        double qs[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        float kn2 = 0.f;
        if (live) {
            const T* kv = reinterpret_cast<const T*>(&x.k);
            const T* vv = reinterpret_cast<const T*>(&x.v);
            uint4 krr;
            T* kr = reinterpret_cast<T*>(&krr);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float y0, y1;
                rope_pair(to_f(kv[2 * j]), to_f(kv[2 * j + 1]), f[j].x, f[j].y, y0, y1);
                kr[2 * j] = from_f<T>(y0);
                kr[2 * j + 1] = from_f<T>(y1);
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) kn2 = fmaf(to_f(kv[e]), to_f(kv[e]), kn2);
            const int64_t ro = (static_cast<int64_t>(g) * R + slot) * 128 + 8 * c8;
            *reinterpret_cast<uint4*>(static_cast<T*>(p.ring_k) + ro) = x.k;
            *reinterpret_cast<uint4*>(static_cast<T*>(p.ring_krot) + ro) = krr;
#pragma unroll
            for (int hh = 0; hh < REP; ++hh) {
                const T* qv = reinterpret_cast<const T*>(&x.q[hh]);
                uint4 qar, qcr;
                T* qa = reinterpret_cast<T*>(&qar);
                T* qc = reinterpret_cast<T*>(&qcr);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float x0 = to_f(qv[2 * j]), x1 = to_f(qv[2 * j + 1]);
                    float y0, y1;
                    rope_pair(x0, x1, f[j].x, f[j].y, y0, y1);
                    qa[2 * j] = from_f<T>(y0);
                    qa[2 * j + 1] = from_f<T>(y1);
                    const int a = 4 * c8 + j;
                    rope_pair(x0, x1, p.freqs.cL[a], p.freqs.sL[a], y0, y1);
                    qc[2 * j] = from_f<T>(y0);
                    qc[2 * j + 1] = from_f<T>(y1);
                    qs[2 * j] += static_cast<double>(x0);
                    qs[2 * j + 1] += static_cast<double>(x1);
                }
                const int64_t qo = (static_cast<int64_t>(g * REP + hh) * p.lxp + i) * 128 + 8 * c8;
                *reinterpret_cast<uint4*>(static_cast<T*>(p.qa) + qo) = qar;
                *reinterpret_cast<uint4*>(static_cast<T*>(p.qc) + qo) = qcr;
            }
            double2* qd = reinterpret_cast<double2*>(p.qs + (i * p.G + g) * 128 + 8 * c8);
#pragma unroll
            for (int e = 0; e < 4; ++e) qd[e] = make_double2(qs[2 * e], qs[2 * e + 1]);
#pragma unroll
            for (int e = 0; e < 8; ++e) svt[8 * c8 + e][tt] = vv[e];
        }
        if (p.kmax2) {  // |k|^2 per token, max into the running bound (same reduction as k_prep_tok)
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) kn2 += __shfl_xor_sync(0xffffffffu, kn2, o);
            kn2 = fmaxf(kn2, __shfl_xor_sync(0xffffffffu, kn2, 16));
            if (lane == 0)
                atomicMax(reinterpret_cast<int*>(p.kmax2) + g, __float_as_int(fmaxf(kn2, p.kmax2_prev[g])));
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) sqs[tt][8 * c8 + e] = qs[e];
        __syncthreads();
        // 16-token sub-tile column sums (the k_prep_tok tiles), published for the look-back
        if (tid < 256) {
            const int sub = tid / 128, c = tid % 128;
            double a = 0.0;
            for (int t = 0; t < 16; ++t) a += sqs[16 * sub + t][c];
            if (16 * sub < nt) p.tsum[((2 * static_cast<int64_t>(tile) + sub) * p.G + g) * 128 + c] = a;
        }
        {  // transposed value pages [G][R/128][dv][128]: 8 consecutive positions of one dim per thread
            const int c = tid / 4, j8 = tid % 4;
            T* rv = static_cast<T*>(p.ring_v);
            const int sl0 = slot_t0 + 8 * j8 >= R ? slot_t0 + 8 * j8 - R : slot_t0 + 8 * j8;
            auto at = [&](int sl) { return ((static_cast<int64_t>(g) * (R / 128) + sl / 128) * 128 + c) * 128 + sl % 128; };
            if (8 * j8 + 8 <= nt && sl0 % 8 == 0) {
                *reinterpret_cast<uint4*>(rv + at(sl0)) = *reinterpret_cast<const uint4*>(&svt[c][8 * j8]);
            } else {
                for (int e = 0; e < 8; ++e) {
                    const int sl = sl0 + e >= R ? sl0 + e - R : sl0 + e;
                    if (8 * j8 + e < nt) rv[at(sl)] = svt[c][8 * j8 + e];
                }
            }
        }
        __syncthreads();  // sqs / svt reused by the next group
        PC_MARK(1 + g);
    };
    for (int g = 0; g < p.G; g += 2) {
        group(g, in0, in1);
        if (g + 1 < p.G) group(g + 1, in1, in0);
    }
    // publish this tile's sub-tile sums (every group) once
    __threadfence();
    __syncthreads();
    if (tid == 0) flag_release_i32(&sync->flags[tile][0], 1);

    // phase 2: the k_prefix_tiles arithmetic once every earlier tile has published its sums
    if (tid < tile) flag_wait_i32(&sync->flags[tid][0]);  // one poller per earlier tile
    __syncthreads();
    PC_MARK(9);
    const int nsub = 2 * tile;  // 16-token sub-tiles before this tile
    for (int g = tid / 128; g < p.G; g += kPcThreads / 128) {
        const int c = tid % 128;
        double v[kPcTok];
#pragma unroll
        for (int j = 0; j < kPcTok; ++j) v[j] = j < nt ? p.qs[((i0 + j) * p.G + g) * 128 + c] : 0.0;
        double run = p.P[(static_cast<int64_t>(s0_slot) * p.G + g) * 128 + c];
        for (int t0 = 0; t0 < nsub; t0 += 16) {
            double ts[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) ts[k] = t0 + k < nsub ? __ldcg(p.tsum + (t0 + k) * stride + g * 128 + c) : 0.0;
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (t0 + k < nsub) run += ts[k];
        }
        double sub0 = 0.0;  // this tile's first sub-tile sum, as published
#pragma unroll
        for (int j = 0; j < 16; ++j) sub0 += v[j];
        const double base1 = run + sub0;  // where k_prefix_tiles starts the second sub-tile
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (j >= nt) break;
            run += v[j];
            int sl = slot_t0 + j + 1;
            if (sl >= R) sl -= R;
            p.P[(static_cast<int64_t>(sl) * p.G + g) * 128 + c] = run;
        }
        if (nt > 16) {
            run = base1;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                if (16 + j >= nt) break;
                run += v[16 + j];
                int sl = slot_t0 + 16 + j + 1;
                if (sl >= R) sl -= R;
                p.P[(static_cast<int64_t>(sl) * p.G + g) * 128 + c] = run;
            }
        }
        if (tile == ntile - 1) {  // chunk total = sum of all sub-tile sums, in order
            const int n16 = static_cast<int>((p.lx + 15) / 16);
            double all = 0.0;
            for (int t = 0; t < n16; ++t) all += __ldcg(p.tsum + t * stride + g * 128 + c);
            p.chunk_qsum[g * 128 + c] = all;
        }
    }
    PC_MARK(10);
    TL_END(TL_PREP);
    // the last block to finish clears the look-back state for the next launch
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(&sync->done, 1u) == static_cast<unsigned>(gridDim.x - 1);
    __syncthreads();
    if (!last) return;
    for (int t = tid; t < ntile * 8; t += kPcThreads) sync->flags[t / 8][t % 8] = 0;
    if (tid == 0) {
        sync->ticket = 0;
        sync->done = 0;
    }
}

void launch_prep_chunk(const PrepParams& p, cudaStream_t st) {
    const unsigned tiles = static_cast<unsigned>((p.lx + kPcTok - 1) / kPcTok);
    const int smem = kPcSqs + kPcSvt + kPcRope;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_prep_chunk<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_prep_chunk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_prep_chunk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_prep_chunk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    switch (p.rep) {
        case 1: k_prep_chunk<1><<<tiles, kPcThreads, smem, st>>>(p); break;
        case 2: k_prep_chunk<2><<<tiles, kPcThreads, smem, st>>>(p); break;
        case 4: k_prep_chunk<4><<<tiles, kPcThreads, smem, st>>>(p); break;
        default: k_prep_chunk<8><<<tiles, kPcThreads, smem, st>>>(p); break;
    }
}

cudaError_t tl_bind_side(const TlBuf& b) { return tl_bind_tu(b); }

}  // namespace infllm
