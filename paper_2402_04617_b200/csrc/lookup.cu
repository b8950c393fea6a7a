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

__global__ void __launch_bounds__(kLkWarps * 32, 1) k_lookup_topk(LookupParams p) {
    if (p.early_dependents) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // decode K4 (PDL)
    TL_BEGIN();
    extern __shared__ __align__(128) uint8_t lk_smem[];
    __shared__ __align__(8) uint64_t sbar[kLkWarps][kLkStages];
    __shared__ double sq[8 * 128];
    __shared__ uint64_t slk[kLkWarps][32];
    __shared__ int sli[kLkWarps][32];
    __shared__ bool last;
    const int lane = threadIdx.x % 32, wib = threadIdx.x / 32;
    const int nb = static_cast<int>(gridDim.x);
    const int64_t S = (p.U + nb - 1) / nb;
    const int64_t s0 = min(static_cast<int64_t>(blockIdx.x) * S, p.U), s1 = min(s0 + S, p.U);
    const int64_t bytes_u = static_cast<int64_t>(p.G) * 512 * 2;
    uint8_t* ring = lk_smem + static_cast<size_t>(wib) * kLkStages * kLkStageBytes;
    for (int t = threadIdx.x; t < p.G * 128; t += blockDim.x) sq[t] = p.qsum[t];
    if (lane == 0)
        for (int st = 0; st < kLkStages; ++st) tc::mbar_init(&sbar[wib][st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    double q[8][4];
#pragma unroll
    for (int g = 0; g < 8; ++g)
#pragma unroll
        for (int j = 0; j < 4; ++j) q[g][j] = g < p.G ? sq[g * 128 + 4 * lane + j] : 0.0;

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
    const int64_t u0 = s0 + wib;
#pragma unroll
    for (int st = 0; st < kLkStages - 1; ++st) issue(u0 + st * kLkWarps, st);
    int stage = 0;
    int64_t it = 0;
    // running top-32 of this warp's units
    uint64_t bk = 0;
    int bi = -1;
    for (int64_t base = s0; base < s1; base += 32 * kLkWarps) {
        // up to 32 units of this warp per batch: unit u = base + wib + 8 * r, r < 32
        uint64_t ck = 0;
        int ci = -1;
#pragma unroll 1
        for (int r = 0; r < 32; ++r) {
            const int64_t u = base + wib + static_cast<int64_t>(kLkWarps) * r;
            if (u >= s1) break;
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
            if (lane == 0 && p.rel) p.rel[u] = rel;
            if (lane == r) {
                ck = lk_key(rel);
                ci = static_cast<int>(u);
            }
            __syncwarp();  // the stage is refilled next iteration
            stage = (stage + 1) % kLkStages;
            ++it;
        }
        warp_sort_desc(ck, ci, lane);
        warp_merge(bk, bi, ck, ci, lane);
    }
    // block list: warp 0 merges the 8 warp lists
    slk[wib][lane] = bk;
    sli[wib][lane] = bi;
    __syncthreads();
    if (wib == 0) {
        for (int w = 1; w < kLkWarps; ++w) warp_merge(bk, bi, slk[w][lane], sli[w][lane], lane);
        p.cand_v[blockIdx.x * 32 + lane] = __longlong_as_double(static_cast<long long>(bk));
        p.cand_i[blockIdx.x * 32 + lane] = bi;
    }
    TL_END(TL_LOOKUP);
    if (nb == 1) {
        last = true;
    } else {
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) last = atomicAdd(p.done, 1u) == static_cast<unsigned>(nb - 1);
        __syncthreads();
        if (!last) return;
        __threadfence();
    }
    // last block: merge the nb block lists (staged in the now idle stage ring)
    uint64_t* ck_all = reinterpret_cast<uint64_t*>(lk_smem);
    int* ci_all = reinterpret_cast<int*>(lk_smem + static_cast<size_t>(nb) * 32 * sizeof(uint64_t));
    for (int t = threadIdx.x; t < nb * 32; t += blockDim.x) {
        ck_all[t] = static_cast<uint64_t>(__double_as_longlong(__ldcg(p.cand_v + t)));
        ci_all[t] = static_cast<int>(__ldcg(p.cand_i + t));
    }
    __syncthreads();
    bk = 0;
    bi = -1;
    for (int b = wib; b < nb; b += kLkWarps) warp_merge(bk, bi, ck_all[b * 32 + lane], ci_all[b * 32 + lane], lane);
    __syncthreads();
    slk[wib][lane] = bk;
    sli[wib][lane] = bi;
    __syncthreads();
    if (wib == 0) {
        for (int w = 1; w < kLkWarps; ++w) warp_merge(bk, bi, slk[w][lane], sli[w][lane], lane);
        // the k_m best, returned ascending by id (memory.hpp:253)
        const int k = static_cast<int>(p.n_sel);
        uint64_t id_key = lane < k ? static_cast<uint64_t>(static_cast<unsigned>(bi)) : ~0ull;
        int dummy = lane;
        // ascending by id = descending by ~id
        id_key = ~id_key;
        warp_sort_desc(id_key, dummy, lane);
        if (lane < k) p.sel[lane] = static_cast<int64_t>(static_cast<unsigned>(~id_key));
        if (lane == 0 && nb > 1) *p.done = 0;
        if (p.ready_flag) {  // the attention of this step may read sel now
            __threadfence();
            __syncwarp();
            if (lane == 0) flag_release(p.ready_flag, p.ready_val);
        }
    }
}

cudaError_t tl_bind_lookup(const TlBuf& b) { return tl_bind_tu(b); }

bool lookup_topk_supported(const LookupParams& p, int dtype_bf16) {
    return dtype_bf16 && p.d == 128 && p.r_k == 4 && p.G >= 1 && p.G <= 8 && p.G == p.Gtot && p.n_sel <= 32 &&
           p.U > 0 && p.U < (1ll << 31);
}

int lookup_topk_blocks(int64_t U, int units_per_block) {
    const int64_t nb = (U + units_per_block - 1) / units_per_block;
    return static_cast<int>(nb < 1 ? 1 : nb > 148 ? 148 : nb);
}

void launch_lookup_topk_fast(const LookupParams& p, int blocks, cudaStream_t st) {
    const size_t ring = static_cast<size_t>(kLkWarps) * kLkStages * kLkStageBytes;
    const size_t merge = static_cast<size_t>(blocks) * 32 * (sizeof(uint64_t) + sizeof(int));
    const size_t smem = ring > merge ? ring : merge;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_lookup_topk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kLkWarps * kLkStages * kLkStageBytes));
        attr = true;
    }
    k_lookup_topk<<<blocks, kLkWarps * 32, smem, st>>>(p);
}

}  // namespace infllm
