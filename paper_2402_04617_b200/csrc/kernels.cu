// kernels.cu — the per-step kernels of the InfLLM layer other than the
// tensor-core attention: RoPE/append/prefix (K7), unit lookup (K1), top-k +
// LRU bookkeeping (K2), eviction + representative scoring (K5/K8),
// representative selection (K6), attention-mass reduction and the
// frequency-decayed LRU update, plus a CUDA-core attention kernel used for
// the fp32 parity mode and for shapes the tcgen05 kernel does not cover.
// Reference citations are relative to /root/reference/proj/include/blockmem/.

#include <cfloat>
#include <cmath>

#include "kernels.cuh"

namespace infllm {

// --------------------------------------------------------------------------
// K7 prep: append k/v to the ring, K_rot = rope(k, pos), q_abs = rope(q, pos),
// q_clamp = rope(q, L)  (rotary.hpp:55-72; attention.hpp:166-167)
template <typename T>
__global__ void k_prep(PrepParams p) {
    const int64_t i = blockIdx.x;
    const int64_t pos = p.s + i;
    const int pairs = p.d / 2;
    const int64_t slot = pos % p.R;
    const T* q = static_cast<const T*>(p.q);
    const T* k = static_cast<const T*>(p.k);
    const T* v = static_cast<const T*>(p.v);
    T* qa = static_cast<T*>(p.qa);
    T* qc = static_cast<T*>(p.qc);
    T* rk = static_cast<T*>(p.ring_k);
    T* rkr = static_cast<T*>(p.ring_krot);
    T* rv = static_cast<T*>(p.ring_v);
    // queries: H heads x pairs
    for (int t = threadIdx.x; t < p.H * pairs; t += blockDim.x) {
        const int h = t / pairs, a = t % pairs;
        const T* src = q + (i * p.H + h) * p.d;
        const float x0 = to_f(src[2 * a]), x1 = to_f(src[2 * a + 1]);
        float c, s, y0, y1;
        rope_cs(p.freqs, a, pos, c, s);
        rope_pair(x0, x1, c, s, y0, y1);
        T* da = qa + (static_cast<int64_t>(h) * p.lxp + i) * p.d;
        da[2 * a] = from_f<T>(y0);
        da[2 * a + 1] = from_f<T>(y1);
        rope_cs(p.freqs, a, p.L, c, s);
        rope_pair(x0, x1, c, s, y0, y1);
        T* dc = qc + (static_cast<int64_t>(h) * p.lxp + i) * p.d;
        dc[2 * a] = from_f<T>(y0);
        dc[2 * a + 1] = from_f<T>(y1);
    }
    if (p.d & 1) {  // odd trailing component is left as is (rotary.hpp:36-37)
        for (int h = threadIdx.x; h < p.H; h += blockDim.x) {
            const T x = q[(i * p.H + h) * p.d + p.d - 1];
            qa[(static_cast<int64_t>(h) * p.lxp + i) * p.d + p.d - 1] = x;
            qc[(static_cast<int64_t>(h) * p.lxp + i) * p.d + p.d - 1] = x;
        }
    }
    // keys: raw copy + rotated copy
    for (int t = threadIdx.x; t < p.G * pairs; t += blockDim.x) {
        const int g = t / pairs, a = t % pairs;
        const T* src = k + (i * p.G + g) * p.d;
        const T x0r = src[2 * a], x1r = src[2 * a + 1];
        float c, s, y0, y1;
        rope_cs(p.freqs, a, pos, c, s);
        rope_pair(to_f(x0r), to_f(x1r), c, s, y0, y1);
        const int64_t o = (static_cast<int64_t>(g) * p.R + slot) * p.d;
        rk[o + 2 * a] = x0r;
        rk[o + 2 * a + 1] = x1r;
        rkr[o + 2 * a] = from_f<T>(y0);
        rkr[o + 2 * a + 1] = from_f<T>(y1);
    }
    if (p.d & 1) {
        for (int g = threadIdx.x; g < p.G; g += blockDim.x) {
            const int64_t o = (static_cast<int64_t>(g) * p.R + slot) * p.d + p.d - 1;
            rk[o] = k[(i * p.G + g) * p.d + p.d - 1];
            rkr[o] = rk[o];
        }
    }
    for (int t = threadIdx.x; t < p.G * p.dv; t += blockDim.x) {
        const int g = t / p.dv, c = t % p.dv;
        rv[p.vl.ring(g, pos, c)] = v[(i * p.G + g) * p.dv + c];
    }
}

// prefix of qs_t[g][c] = sum_{h in g} q[t][h][c] (fp64) into the P ring, and
// the chunk total (the lookup's query sum, memory.hpp:224-225).
constexpr int kScanSegs = 16;
template <typename T>
__global__ void k_prefix(PrepParams p) {
    __shared__ double tot[kScanSegs][32];
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

template <typename T>
void launch_prep(const PrepParams& p, cudaStream_t st) {
    k_prep<T><<<static_cast<unsigned>(p.lx), 256, 0, st>>>(p);
    dim3 grid(p.G, (p.d + 31) / 32);
    k_prefix<T><<<grid, dim3(32, kScanSegs), 0, st>>>(p);
}
template void launch_prep<float>(const PrepParams&, cudaStream_t);
template void launch_prep<bf16>(const PrepParams&, cudaStream_t);

// --------------------------------------------------------------------------
// K1 lookup score: part[u][g] = sum_{r,c} qsum[g][c] * repr[u][g][r][c] in
// fp64 (TieredStore::relevance_all, memory.hpp:217-234). One warp per unit;
// per group, lane L owns a fixed contiguous run of the group's r_k*d
// elements, then an xor-tree: the association is independent of how groups
// are sharded across GPUs.
template <typename T>
__global__ void k_lookup(LookupParams p) {
    extern __shared__ double sq[];  // [G][d]
    for (int t = threadIdx.x; t < p.G * p.d; t += blockDim.x) sq[t] = p.qsum[t];
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t u = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + warp;
    if (u >= p.U) return;
    const int E = p.r_k * p.d;
    const int per = (E + 31) / 32;
    const T* base = static_cast<const T*>(p.repr) + u * p.G * E;
    for (int g = 0; g < p.G; ++g) {
        const T* src = base + g * E;
        const double* qg = sq + g * p.d;
        double a = 0.0;
        for (int j = 0; j < per; ++j) {
            const int e = lane * per + j;
            if (e < E) a += qg[e % p.d] * static_cast<double>(to_f(src[e]));
        }
        a = warp_sum_d(a);
        if (lane == 0) p.part[u * p.Gtot + p.g0 + g] = a;
    }
}

// specialised: r_k*d == 512 bf16 (16 elements = 2 x 16B per lane)
__global__ void k_lookup_bf16_512(LookupParams p) {
    extern __shared__ double sq[];
    for (int t = threadIdx.x; t < p.G * p.d; t += blockDim.x) sq[t] = p.qsum[t];
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t u = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + warp;
    if (u >= p.U) return;
    const uint4* base = reinterpret_cast<const uint4*>(static_cast<const bf16*>(p.repr) + u * p.G * 512);
    uint4 buf[16];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        if (g < p.G) {
            buf[2 * g] = __ldcs(base + g * 64 + lane * 2);
            buf[2 * g + 1] = __ldcs(base + g * 64 + lane * 2 + 1);
        }
    }
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        if (g >= p.G) break;
        const double* qg = sq + g * p.d;
        const bf16* e = reinterpret_cast<const bf16*>(&buf[2 * g]);
        double a = 0.0;
#pragma unroll
        for (int j = 0; j < 16; ++j) a += qg[(lane * 16 + j) % p.d] * static_cast<double>(__bfloat162float(e[j]));
        a = warp_sum_d(a);
        if (lane == 0) p.part[u * p.Gtot + p.g0 + g] = a;
    }
    for (int g = 8; g < p.G; ++g) {  // G > 8: generic tail
        const bf16* src = static_cast<const bf16*>(p.repr) + (u * p.G + g) * 512;
        const double* qg = sq + g * p.d;
        double a = 0.0;
        for (int j = 0; j < 16; ++j) a += qg[(lane * 16 + j) % p.d] * static_cast<double>(__bfloat162float(src[lane * 16 + j]));
        a = warp_sum_d(a);
        if (lane == 0) p.part[u * p.Gtot + p.g0 + g] = a;
    }
}

void launch_lookup(const LookupParams& p, int dtype_bf16, cudaStream_t st) {
    const int warps = 8;
    const unsigned blocks = static_cast<unsigned>((p.U + warps - 1) / warps);
    const size_t smem = sizeof(double) * p.G * p.d;
    if (dtype_bf16 && p.r_k * p.d == 512)
        k_lookup_bf16_512<<<blocks, warps * 32, smem, st>>>(p);
    else if (dtype_bf16)
        k_lookup<bf16><<<blocks, warps * 32, smem, st>>>(p);
    else
        k_lookup<float><<<blocks, warps * 32, smem, st>>>(p);
}

// --------------------------------------------------------------------------
// K2 top-k: rel[u] = sum_g part[u][g] (group order), then top n_sel by
// (rel desc, id asc), ids ascending (memory.hpp:240-253), then the lookup's
// tier bookkeeping (memory.hpp:254-267).
__device__ __forceinline__ bool better(double va, int64_t ia, double vb, int64_t ib) {
    return va > vb || (va == vb && ia < ib);
}

__device__ void block_topk(const double* rel_in, double* relw, int64_t U, int64_t n_sel, int64_t* out_sorted) {
    __shared__ double wv[32];
    __shared__ int64_t wi[32];
    int64_t* picked = out_sorted;  // written by thread 0 only, sorted in place at the end
    const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32, nw = blockDim.x / 32;
    for (int64_t u = tid; u < U; u += blockDim.x) relw[u] = rel_in[u];
    __syncthreads();
    for (int64_t r = 0; r < n_sel; ++r) {
        double bv = -INFINITY;
        int64_t bi = INT64_MAX;
        for (int64_t u = tid; u < U; u += blockDim.x) {
            const double x = relw[u];
            if (x != -INFINITY && (bi == INT64_MAX || better(x, u, bv, bi))) {
                bv = x;
                bi = u;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (oi != INT64_MAX && (bi == INT64_MAX || better(ov, oi, bv, bi))) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            wv[warp] = bv;
            wi[warp] = bi;
        }
        __syncthreads();
        if (tid == 0) {
            double v = wv[0];
            int64_t id = wi[0];
            for (int w = 1; w < nw; ++w)
                if (wi[w] != INT64_MAX && (id == INT64_MAX || better(wv[w], wi[w], v, id))) {
                    v = wv[w];
                    id = wi[w];
                }
            picked[r] = id;
            relw[id] = -INFINITY;
        }
        __syncthreads();
    }
    if (tid == 0) {
        for (int64_t a = 1; a < n_sel; ++a) {  // ascending ids
            const int64_t x = picked[a];
            int64_t b = a - 1;
            while (b >= 0 && picked[b] > x) {
                picked[b + 1] = picked[b];
                --b;
            }
            picked[b + 1] = x;
        }
    }
    __syncthreads();
}

__global__ void k_topk(TopkParams p) {
    for (int64_t u = threadIdx.x; u < p.U; u += blockDim.x) {
        double a = 0.0;
        for (int g = 0; g < p.Gtot; ++g) a += p.part[u * p.Gtot + g];
        p.rel[u] = a;
    }
    __syncthreads();
    block_topk(p.rel, p.relw, p.U, p.n_sel, p.sel);
    if (threadIdx.x == 0) {
        LruState& s = *p.lru;
        for (int64_t a = 0; a < p.n_sel; ++a) {
            const int64_t id = p.sel[a];
            s.requested++;
            int64_t* tr = p.trace + 3 * s.trace_count;
            tr[0] = p.step;
            tr[1] = id;
            if (p.hot[id]) {
                s.hits++;
                tr[2] = 1;
            } else {
                s.misses++;
                s.loads++;
                p.hot[id] = 1;
                p.hot_list[s.hot_count++] = id;
                tr[2] = 0;
            }
            s.trace_count++;
        }
    }
}

void launch_topk(const TopkParams& p, cudaStream_t st) { k_topk<<<1, 1024, 0, st>>>(p); }

__global__ void k_rel_topk_standalone(const double* part, int64_t U, int Gtot, int64_t k, double* rel, double* relw,
                                      int64_t* ids) {
    for (int64_t u = threadIdx.x; u < U; u += blockDim.x) {
        double a = 0.0;
        for (int g = 0; g < Gtot; ++g) a += part[u * Gtot + g];
        rel[u] = a;
    }
    __syncthreads();
    block_topk(rel, relw, U, k, ids);
}

void launch_rel_topk_standalone(const double* part, int64_t U, int Gtot, int64_t k, double* rel, double* relw,
                                int64_t* ids, cudaStream_t st) {
    k_rel_topk_standalone<<<1, 1024, 0, st>>>(part, U, Gtot, k, rel, relw, ids);
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

void launch_mass(const MassParams& p, cudaStream_t st) {
    if (p.n_sel > 0) k_mass<<<p.n_sel, 256, 0, st>>>(p);
}

// frequency decay + masses + capacity (memory.hpp:273-300) + step-boundary
// peaks (memory.hpp:303-308). Single thread: |hot| <= cap + k_m.
__global__ void k_lru(LruParams p) {
    LruState& s = *p.lru;
    for (int64_t a = 0; a < s.hot_count; ++a) p.freq[p.hot_list[a]] *= p.decay;
    for (int64_t j = 0; j < p.n_sel; ++j) {
        double m = 0.0;
        for (int g = 0; g < p.Gtot; ++g) m += p.mass_part[j * p.Gtot + g];
        p.freq[p.sel[j]] += m / static_cast<double>(p.H_total);
    }
    while (s.hot_count > p.cap) {
        int64_t worst = 0;
        for (int64_t a = 1; a < s.hot_count; ++a) {
            const int64_t ia = p.hot_list[a], iw = p.hot_list[worst];
            if (p.freq[ia] < p.freq[iw] || (p.freq[ia] == p.freq[iw] && ia < iw)) worst = a;
        }
        p.hot[p.hot_list[worst]] = 0;
        p.hot_list[worst] = p.hot_list[s.hot_count - 1];
        s.hot_count--;
        s.evictions++;
    }
    if (s.hot_count > s.peak_hot_units) s.peak_hot_units = s.hot_count;
    int64_t bytes = 0;
    for (int64_t a = 0; a < s.hot_count; ++a) bytes += p.bytes_per_token * p.unit_len[p.hot_list[a]];
    if (bytes > s.peak_hot_bytes) s.peak_hot_bytes = bytes;
}

void launch_lru(const LruParams& p, cudaStream_t st) { k_lru<<<1, 1, 0, st>>>(p); }

// --------------------------------------------------------------------------
// K8 evict + K5 representative-score partials. Popped positions
// [pop0, pop0 + n_init) are pinned as initial tokens (engine.hpp:311-322);
// the rest are evicted into unit pages (engine.hpp:323-340, UnitPacker::add
// memory.hpp:59-78). r_m partial per group: k_m . (P[m+L+1] - P[m+1]), i.e.
// sum over the L following queries of the group's q . k_m (repr_score.hpp:53-67).
template <typename T>
__global__ void k_evict(EvictParams p) {
    const int64_t idx = blockIdx.x;
    const int64_t pos = p.pop0 + idx;
    const int64_t slot = pos % p.R;
    const T* rk = static_cast<const T*>(p.ring_k);
    const T* rkr = static_cast<const T*>(p.ring_krot);
    const T* rv = static_cast<const T*>(p.ring_v);
    if (idx < p.n_init) {
        T* ik = static_cast<T*>(p.init_k);
        T* ikr = static_cast<T*>(p.init_krot);
        T* iv = static_cast<T*>(p.init_v);
        for (int t = threadIdx.x; t < p.G * p.d; t += blockDim.x) {
            const int g = t / p.d, c = t % p.d;
            ik[(static_cast<int64_t>(g) * p.l_I + pos) * p.d + c] = rk[(static_cast<int64_t>(g) * p.R + slot) * p.d + c];
            if (p.absolute) ikr[(static_cast<int64_t>(g) * p.l_I + pos) * p.d + c] = rkr[(static_cast<int64_t>(g) * p.R + slot) * p.d + c];
        }
        for (int t = threadIdx.x; t < p.G * p.dv; t += blockDim.x) {
            const int g = t / p.dv, c = t % p.dv;
            iv[p.vl.init(g, pos, c)] = rv[p.vl.ring(g, pos, c)];
        }
        return;
    }
    const int64_t e = idx - p.n_init;
    const int64_t rel = pos - p.pend_start;
    const int64_t u = p.unit0 + rel / p.l_bs, off = rel % p.l_bs;
    T* uk = static_cast<T*>(p.unit_k);
    T* ukr = static_cast<T*>(p.unit_krot);
    T* uv = static_cast<T*>(p.unit_v);
    for (int t = threadIdx.x; t < p.G * p.d; t += blockDim.x) {
        const int g = t / p.d, c = t % p.d;
        const int64_t o = ((u * p.G + g) * p.l_bs + off) * p.d + c;
        uk[o] = rk[(static_cast<int64_t>(g) * p.R + slot) * p.d + c];
        if (p.absolute) ukr[o] = rkr[(static_cast<int64_t>(g) * p.R + slot) * p.d + c];
    }
    for (int t = threadIdx.x; t < p.G * p.dv; t += blockDim.x) {
        const int g = t / p.dv, c = t % p.dv;
        uv[p.vl.unit(u, g, off, c)] = rv[p.vl.ring(g, pos, c)];
    }
    // score partials: warp w handles groups w, w + nwarps, ...
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
    const int64_t hi = ((pos + p.L + 1) % p.R) * p.G, lo = ((pos + 1) % p.R) * p.G;
    for (int g = warp; g < p.G; g += nw) {
        double a = 0.0;
        for (int c = lane; c < p.d; c += 32) {
            const double w = p.P[(hi + g) * p.d + c] - p.P[(lo + g) * p.d + c];
            a += static_cast<double>(to_f(rk[(static_cast<int64_t>(g) * p.R + slot) * p.d + c])) * w;
        }
        a = warp_sum_d(a);
        if (lane == 0) p.ev_part[e * p.Gtot + p.g0 + g] = a;
    }
}

template <typename T>
void launch_evict(const EvictParams& p, cudaStream_t st) {
    const int64_t n = p.n_init + p.n_evict;
    if (n > 0) k_evict<T><<<static_cast<unsigned>(n), 256, 0, st>>>(p);
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

template <typename T>
__global__ void k_select(SelectParams p) {
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t u = p.u0 + static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + warp;
    if (u >= p.u0 + p.n_units) return;
    const int len = p.unit_len[u];
    int idx[32];
    warp_select(p.unit_scores + u * p.l_bs, len, p.r_k, idx);
    const int take = min(p.r_k, len);
    if (lane < p.r_k) p.repr_idx[u * p.r_k + lane] = lane < take ? idx[lane] : -1;
    const T* uk = static_cast<const T*>(p.unit_k);
    T* rp = static_cast<T*>(p.repr);
    for (int g = 0; g < p.G; ++g)
        for (int r = 0; r < p.r_k; ++r)
            for (int c = lane; c < p.d; c += 32) {
                // units shorter than r_k (final flush) repeat their last representative row with zero keys
                const T x = r < take ? uk[((u * p.G + g) * p.l_bs + idx[r]) * p.d + c] : from_f<T>(0.f);
                rp[((u * p.G + g) * p.r_k + r) * p.d + c] = x;
            }
}

template <typename T>
void launch_select(const SelectParams& p, cudaStream_t st) {
    if (p.n_units <= 0) return;
    const int warps = 4;
    k_select<T><<<static_cast<unsigned>((p.n_units + warps - 1) / warps), warps * 32, 0, st>>>(p);
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
