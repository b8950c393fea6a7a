// lookup.cu — K1 + K2 in one launch: relevance of every memory unit against
// the chunk's query sums (TieredStore::relevance_all, memory.hpp:217-234) and
// the exact top-k_m selection (TieredStore::lookup, memory.hpp:239-253).
//
// Shape: bf16 representative index [U][G][r_k = 4][d = 128], G <= 8, one
// shard, k_m <= 32 (the C1-C4 configurations). Each block owns a contiguous
// slice of units; each warp streams whole units (G x 4 x 128 bf16 = 8 KB at
// G = 8) through a 3-stage shared-memory ring filled by bulk copies (TMA
// engine, one mbarrier per stage), and lane l owns dims [4l, 4l + 4) of every
// representative row: the fp64 dot of the group's query-sum slice with the
// unit's rows, groups summed in order 0..G-1, then one xor tree. The block's
// slice then goes through a warp-level bitonic top-32 (key = order-preserving
// bits of rel, tie to the lower unit id, memory.hpp:245-252), the block list
// is published, and the last block to finish merges the per-block lists
// (bitonic merges of sorted 32-lists) and writes the k_m ids ascending.
// The grid is sized by the caller: few fat blocks inside the prefill pipeline
// (the attention holds most SMs), one unit per warp for a decode step.
#include "kernels.cuh"
#include "tc_prims.cuh"

namespace infllm {

namespace {
constexpr int kLkWarps = 8;
constexpr int kLkStages = 3;
constexpr int kLkStageBytes = 8192;  // one unit at G = 8
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint64_t lk_key(double v) {
    if (v == 0.0) v = 0.0;  // -0.0 and +0.0 compare equal in the reference comparator: one key
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
// (rel desc, id asc); invalid entries are (0, -1): worse than every unit
__device__ __forceinline__ bool lk_better(uint64_t ka, int ia, uint64_t kb, int ib) {
    return ka > kb || (ka == kb && static_cast<unsigned>(ia) < static_cast<unsigned>(ib));
}
// bitonic sort of one entry per lane: lane 0 ends with the best
__device__ __forceinline__ void warp_sort_desc(uint64_t& k, int& i, int lane) {
#pragma unroll
    for (int kk = 2; kk <= 32; kk <<= 1)
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
            const uint64_t ok = __shfl_xor_sync(kFull, k, j);
            const int oi = __shfl_xor_sync(kFull, i, j);
            const bool desc = (lane & kk) == 0, lower = (lane & j) == 0;
            const bool ob = lk_better(ok, oi, k, i);
            if ((desc == lower) == ob) {
                k = ok;
                i = oi;
            }
        }
}
// (k, i) sorted desc across the warp, (bk, bi) another sorted list: keep the best 32, sorted
__device__ __forceinline__ void warp_merge(uint64_t& k, int& i, uint64_t bk, int bi, int lane) {
    const uint64_t rk = __shfl_sync(kFull, bk, 31 - lane);
    const int ri = __shfl_sync(kFull, bi, 31 - lane);
    if (lk_better(rk, ri, k, i)) {
        k = rk;
        i = ri;
    }
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
        const uint64_t ok = __shfl_xor_sync(kFull, k, j);
        const int oi = __shfl_xor_sync(kFull, i, j);
        const bool lower = (lane & j) == 0;
        if (lower == lk_better(ok, oi, k, i)) {
            k = ok;
            i = oi;
        }
    }
}
}  // namespace

constexpr int kLkMaxSlice = 1024;  // units per block (keys staged in shared memory)
constexpr int kLkSurv = 1024;      // survivors of the threshold filter kept for the final sort

// the best 32 of n (key, id) pairs in shared memory, sorted desc, in warp `lane`s registers
__device__ __forceinline__ void warp_top32(const uint64_t* key, const int* id, int n, uint64_t& bk, int& bi,
                                           int lane) {
    bk = 0;
    bi = -1;
    for (int c = 0; c < n; c += 32) {
        uint64_t k = c + lane < n ? key[c + lane] : 0ull;
        int i = c + lane < n ? id[c + lane] : -1;
        warp_sort_desc(k, i, lane);
        if (c == 0) {
            bk = k;
            bi = i;
        } else {
            warp_merge(bk, bi, k, i, lane);
        }
    }
}

__global__ void __launch_bounds__(kLkWarps * 32, 1) k_lookup_topk(LookupParams p) {
    if (p.early_dependents) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // decode K4 (PDL)
    TL_BEGIN();
    extern __shared__ __align__(128) uint8_t lk_smem[];
    __shared__ __align__(8) uint64_t sbar[kLkWarps][kLkStages];
    __shared__ __align__(8) uint64_t cbar;
    __shared__ double sq[8 * 128];
    __shared__ uint64_t skey[kLkMaxSlice];
    __shared__ int sid[kLkMaxSlice];
    __shared__ uint64_t slk[kLkWarps][32];
    __shared__ int sli[kLkWarps][32];
    __shared__ uint64_t s_tau;
    __shared__ int s_cnt;
    __shared__ bool last;
    const int lane = threadIdx.x % 32, wib = threadIdx.x / 32;
    const int nb = static_cast<int>(gridDim.x);
    const int64_t S = (p.U + nb - 1) / nb;
    const int64_t s0 = min(static_cast<int64_t>(blockIdx.x) * S, p.U), s1 = min(s0 + S, p.U);
    const int ns = static_cast<int>(s1 - s0);
    const int64_t bytes_u = static_cast<int64_t>(p.G) * 512 * 2;
    uint8_t* ring = lk_smem + static_cast<size_t>(wib) * kLkStages * kLkStageBytes;
    auto issue = [&](int64_t u, int stage) {
        if (u < s1 && lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the stage was read by this warp
            tc::mbar_expect_tx(&sbar[wib][stage], static_cast<uint32_t>(bytes_u));
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    tc::smem_u32(ring + stage * kLkStageBytes)),
                "l"(static_cast<const uint8_t*>(p.repr) + u * bytes_u), "r"(static_cast<uint32_t>(bytes_u)),
                "r"(tc::smem_u32(&sbar[wib][stage]))
                : "memory");
        }
    };
    // each warp's first units are in flight before anything else happens
    if (lane == 0) {
        for (int st = 0; st < kLkStages; ++st) tc::mbar_init(&sbar[wib][st], 1);
        if (wib == 0) tc::mbar_init(&cbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t u0 = s0 + wib;
#pragma unroll
    for (int st = 0; st < kLkStages - 1; ++st) issue(u0 + st * kLkWarps, st);
    lk_stage_qsums(p, sq);
    __syncthreads();
    unsigned long long mark = tl_t0_;
    double q[8][4];
#pragma unroll
    for (int g = 0; g < 8; ++g)
#pragma unroll
        for (int j = 0; j < 4; ++j) q[g][j] = g < p.G ? sq[g * 128 + 4 * lane + j] : 0.0;

    int stage = 0;
    int64_t it = 0;
    for (int64_t u = u0; u < s1; u += kLkWarps, ++it) {
        issue(u + (kLkStages - 1) * kLkWarps, (stage + kLkStages - 1) % kLkStages);
        tc::mbar_wait(&sbar[wib][stage], static_cast<uint32_t>((it / kLkStages) & 1));
        const uint8_t* buf = ring + stage * kLkStageBytes + 8 * lane;
        double rel = 0.0;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            if (g >= p.G) break;
            double a = 0.0;
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
                const uint2 v = *reinterpret_cast<const uint2*>(buf + (4 * g + rr) * 256);
                a = fma(q[g][0], static_cast<double>(__uint_as_float(v.x << 16)), a);
                a = fma(q[g][1], static_cast<double>(__uint_as_float(v.x & 0xffff0000u)), a);
                a = fma(q[g][2], static_cast<double>(__uint_as_float(v.y << 16)), a);
                a = fma(q[g][3], static_cast<double>(__uint_as_float(v.y & 0xffff0000u)), a);
            }
            rel += a;
        }
        rel = warp_sum_d(rel);
        if (lane == 0) {
            if (p.rel) p.rel[u] = rel;
            skey[u - s0] = lk_key(rel);
            sid[u - s0] = static_cast<int>(u);
        }
        __syncwarp();  // the stage is refilled next iteration
        stage = (stage + 1) % kLkStages;
    }
    __syncthreads();
    TL_MARK(0, mark);  // scan
    if (p.n_sel <= 0) return;
    // this block's best 32 (rel desc, id asc), published for the last block
    if (wib == 0) {
        uint64_t bk;
        int bi;
        warp_top32(skey, sid, ns, bk, bi, lane);
        p.cand_v[blockIdx.x * 32 + lane] = __longlong_as_double(static_cast<long long>(bk));
        reinterpret_cast<int64_t*>(p.cand_i)[blockIdx.x * 32 + lane] = bi;
        __syncwarp();
        if (lane == 0) {
            unsigned prev = 0;
            if (nb > 1) {
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                prev = atomicAdd(p.done, 1u);
            }
            last = prev == static_cast<unsigned>(nb - 1);
        }
    }
    __syncthreads();
    TL_MARK(1, mark);  // block list published
    TL_END(TL_LOOKUP);
    if (!last) return;
    if (nb > 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    // last block: every block list into shared memory with two bulk copies
    uint64_t* ck_all = reinterpret_cast<uint64_t*>(lk_smem);
    int64_t* ci_all = reinterpret_cast<int64_t*>(lk_smem + static_cast<size_t>(nb) * 32 * sizeof(uint64_t));
    uint64_t* sv = reinterpret_cast<uint64_t*>(lk_smem + static_cast<size_t>(nb) * 32 * 16);  // survivors
    int* si = reinterpret_cast<int*>(sv + kLkSurv);
    if (threadIdx.x == 0) {
        const uint32_t nbytes = static_cast<uint32_t>(nb) * 32 * 8;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc::mbar_expect_tx(&cbar, 2 * nbytes);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         tc::smem_u32(ck_all)),
                     "l"(p.cand_v), "r"(nbytes), "r"(tc::smem_u32(&cbar))
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         tc::smem_u32(ci_all)),
                     "l"(p.cand_i), "r"(nbytes), "r"(tc::smem_u32(&cbar))
                     : "memory");
        s_cnt = 0;
        s_tau = 0;
    }
    tc::mbar_wait(&cbar, 0);
    __syncthreads();
    TL_MARK(2, mark);  // candidates staged
    // threshold: the k-th best of any block list is a lower bound of the global k-th best
    const int k = static_cast<int>(p.n_sel < 32 ? p.n_sel : 32);
    {
        uint64_t t = 0;
        for (int b = threadIdx.x; b < nb; b += blockDim.x) t = max(t, ck_all[b * 32 + k - 1]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t = max(t, __shfl_xor_sync(kFull, t, o));
        if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(&s_tau), static_cast<unsigned long long>(t));
        // so is the k-th best of the block bests (k distinct units at least that good):
        // the tighter bound when blocks hold few units (one-token steps, one unit per warp)
        if (nb >= k)
            for (int b = threadIdx.x; b < nb; b += blockDim.x) {
                const uint64_t kb = ck_all[b * 32];
                const int ib = static_cast<int>(ci_all[b * 32]);
                int r = 0;
                for (int j = 0; j < nb; ++j) r += lk_better(ck_all[j * 32], static_cast<int>(ci_all[j * 32]), kb, ib) ? 1 : 0;
                if (r == k - 1)
                    atomicMax(reinterpret_cast<unsigned long long*>(&s_tau), static_cast<unsigned long long>(kb));
            }
    }
    __syncthreads();
    const uint64_t tau = s_tau;
    for (int t = threadIdx.x; t < nb * 32; t += blockDim.x) {
        const int id = static_cast<int>(ci_all[t]);
        if (id >= 0 && ck_all[t] >= tau) {
            const int slot = atomicAdd(&s_cnt, 1);
            if (slot < kLkSurv) {
                sv[slot] = ck_all[t];
                si[slot] = id;
            }
        }
    }
    __syncthreads();
    const int cnt = s_cnt;
    if (cnt >= k && cnt <= static_cast<int>(blockDim.x)) {
        // few survivors (the usual case): each one's rank among them by direct
        // comparison, then the selected ids' ascending slots the same way; exact and
        // order-free, so the same k ids as the merge below, without its ~80
        // dependent shuffle stages in one warp
        __shared__ int s_take[kLkWarps * 32];
        const bool have = static_cast<int>(threadIdx.x) < cnt;
        const uint64_t mk = have ? sv[threadIdx.x] : 0ull;
        const int mi = have ? si[threadIdx.x] : -1;
        int rank = 0;
        if (have)
            for (int j = 0; j < cnt; ++j) rank += lk_better(sv[j], si[j], mk, mi) ? 1 : 0;
        const bool take = have && rank < k;
        s_take[threadIdx.x] = take ? mi : -1;
        __syncthreads();
        if (take) {
            int pos = 0;
            for (int j = 0; j < cnt; ++j) pos += (s_take[j] >= 0 && s_take[j] < mi) ? 1 : 0;
            p.sel[pos] = static_cast<int64_t>(mi);
        }
        if (threadIdx.x == 0) {
            if (nb > 1) *p.done = 0;
            TL_MARK(3, mark);  // final selection
        }
        return;
    }
    uint64_t bk = 0;
    int bi = -1;
    if (cnt <= kLkSurv) {
        const int per = (cnt + kLkWarps - 1) / kLkWarps;  // each warp the best 32 of its share, then warp 0
        const int a0 = min(cnt, wib * per), a1 = min(cnt, a0 + per);
        if (cnt <= 32) {
            if (wib == 0) warp_top32(sv, si, cnt, bk, bi, lane);
        } else {
            warp_top32(sv + a0, si + a0, a1 - a0, bk, bi, lane);
            slk[wib][lane] = bk;
            sli[wib][lane] = bi;
            __syncthreads();
            if (wib == 0)
                for (int w = 1; w < kLkWarps; ++w) warp_merge(bk, bi, slk[w][lane], sli[w][lane], lane);
        }
    } else {  // more than kLkSurv keys tie at the threshold: merge every block list
        for (int b = wib; b < nb; b += kLkWarps)
            warp_merge(bk, bi, ck_all[b * 32 + lane], static_cast<int>(ci_all[b * 32 + lane]), lane);
        slk[wib][lane] = bk;
        sli[wib][lane] = bi;
        __syncthreads();
        if (wib == 0)
            for (int w = 1; w < kLkWarps; ++w) warp_merge(bk, bi, slk[w][lane], sli[w][lane], lane);
    }
    if (wib == 0) {
        // the k_m best, returned ascending by id (memory.hpp:253): sort by ~id descending
        uint64_t id_key = lane < k ? ~static_cast<uint64_t>(static_cast<unsigned>(bi)) : 0ull;
        int dummy = lane;
        warp_sort_desc(id_key, dummy, lane);
        if (lane < k) p.sel[lane] = static_cast<int64_t>(static_cast<unsigned>(~id_key));
        if (lane == 0 && nb > 1) *p.done = 0;
        TL_MARK(3, mark);  // final selection
    }
}

bool lookup_topk_supported(const LookupParams& p, int dtype_bf16) {
    return dtype_bf16 && p.d == 128 && p.r_k == 4 && p.G >= 1 && p.G <= 8 && p.G == p.Gtot && p.n_sel <= 32 &&
           p.U > 0 && p.U <= 148ll * kLkMaxSlice;
}

int lookup_topk_blocks(int64_t U, int units_per_block) {
    int64_t nb = (U + units_per_block - 1) / units_per_block;
    nb = nb < (U + kLkMaxSlice - 1) / kLkMaxSlice ? (U + kLkMaxSlice - 1) / kLkMaxSlice : nb;
    return static_cast<int>(nb < 1 ? 1 : nb > 148 ? 148 : nb);
}

void launch_lookup_topk_fast(const LookupParams& p, int blocks, cudaStream_t st) {
    const size_t ring = static_cast<size_t>(kLkWarps) * kLkStages * kLkStageBytes;
    const size_t merge = static_cast<size_t>(blocks) * 32 * 16 + kLkSurv * (sizeof(uint64_t) + sizeof(int));
    const size_t smem = ring > merge ? ring : merge;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_lookup_topk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kLkWarps * kLkStages * kLkStageBytes));
        attr = true;
    }
    k_lookup_topk<<<blocks, kLkWarps * 32, smem, st>>>(p);
}

cudaError_t tl_bind_lookup(const TlBuf& b) { return tl_bind_tu(b); }

}  // namespace infllm
