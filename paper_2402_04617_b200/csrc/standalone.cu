// standalone.cu — the reference's stand-alone operators behind the C-ABI,
// for hosts that drive the pieces themselves instead of StreamEngine::step:
//
//  * infllm_attend: blockmem::attend (attention.hpp:116-230) over an explicit
//    window of segments (initial / retrieved / local, attention.hpp:14-51)
//    plus the causal batch, with the per-segment attention masses of
//    engine.hpp:271-283 and, optionally, the full softmax weights
//    (emit_weights, attention.hpp:227).
//  * infllm_store_*: blockmem::TieredStore (memory.hpp:170-323): add_unit,
//    begin_step, lookup (relevance_all + top-k + hit/miss bookkeeping),
//    update_frequency, enforce_capacity, note_step_boundary, counters, trace.
//  * infllm_score_acc_*: blockmem::ScoreAccumulator (repr_score.hpp:21-89):
//    accumulate and finalize_front.
//
// These are the operator API, not the hot path: the engine (engine.cu) runs
// the same arithmetic through its fused step kernels. Numerics: fp32 scores
// and softmax like the reference's Scalar = float; fp64 relevance, masses,
// band sums and frequency scores.
#include <algorithm>
#include <cmath>
#include <vector>

#include "kernels.cuh"

namespace infllm {

// ------------------------------------------------------------------ attend
struct AttendSeg {  // device copy of one window segment + its first column
    const void* keys;
    const void* values;
    int64_t start_abs, n, col0;
    int kind;
};

struct AttendParams {
    const AttendSeg* segs;
    int n_seg;
    const void* q;  // [lx][H][d]
    const void* k;  // [lx][G][d]
    const void* v;  // [lx][G][dv]
    void* out;      // [lx][H][dv]
    float* scores;  // [H][lx][n_all] scratch (the weights when emitted)
    double* mass_part;  // [H][lx][n_seg]
    float* qrot;    // [2][H][lx][d]: rope(q, start + i), rope(q, L)
    float* krot;    // [n_all][G][d] rope(k, pos) (absolute mode, local segments, batch)
    int64_t lx, n_ctx, n_all, start_abs, L;
    int H, G, rep, d, dv, absolute;
    RopeFreqs freqs;
};

template <typename T>
__device__ __forceinline__ float ld_f(const void* p, int64_t i) {
    return to_f(static_cast<const T*>(p)[i]);
}

// column j -> (segment, row) by linear search over the (few) segments
__device__ __forceinline__ int seg_of(const AttendParams& a, int64_t j) {
    int s = 0;
    while (s + 1 < a.n_seg && a.segs[s + 1].col0 <= j) ++s;
    return s;
}

// rotate one key/query row by an absolute position (rotary.hpp:40-51, fp64 angles)
template <typename T>
__device__ void rot_row(const RopeFreqs& fr, const void* src, int64_t off, int d, int64_t pos, float* dst, int tid,
                        int nthr) {
    for (int a = tid; a < d / 2; a += nthr) {
        float c, s;
        rope_cs(fr, a, pos, c, s);
        float y0, y1;
        rope_pair(ld_f<T>(src, off + 2 * a), ld_f<T>(src, off + 2 * a + 1), c, s, y0, y1);
        dst[2 * a] = y0;
        dst[2 * a + 1] = y1;
    }
    if ((d & 1) && tid == 0) dst[d - 1] = ld_f<T>(src, off + d - 1);  // odd last dim untouched
}

// (1) rotated queries and the keys whose rotation depends on their position
template <typename T>
__global__ void k_attend_rotate(AttendParams a) {
    const int64_t r = blockIdx.x;  // query rows first ([H][lx] x 2), then context + batch keys ([n_all][G])
    const int64_t nq = static_cast<int64_t>(a.H) * a.lx;
    if (r < nq) {
        const int h = static_cast<int>(r / a.lx);
        const int64_t i = r % a.lx;
        const int64_t off = (i * a.H + h) * a.d;
        rot_row<T>(a.freqs, a.q, off, a.d, a.start_abs + i, a.qrot + r * a.d, threadIdx.x, blockDim.x);
        // rotate_by_constant(q, L) (rotary.hpp:66-72)
        float* dc = a.qrot + (nq + r) * a.d;
        for (int c2 = threadIdx.x; c2 < a.d / 2; c2 += blockDim.x) {
            float y0, y1;
            rope_pair(ld_f<T>(a.q, off + 2 * c2), ld_f<T>(a.q, off + 2 * c2 + 1), a.freqs.cL[c2], a.freqs.sL[c2], y0, y1);
            dc[2 * c2] = y0;
            dc[2 * c2 + 1] = y1;
        }
        if ((a.d & 1) && threadIdx.x == 0) dc[a.d - 1] = ld_f<T>(a.q, off + a.d - 1);
        return;
    }
    const int64_t kr = r - nq;
    const int64_t j = kr / a.G;
    const int g = static_cast<int>(kr % a.G);
    if (j >= a.n_ctx) {  // batch key
        const int64_t i = j - a.n_ctx;
        rot_row<T>(a.freqs, a.k, (i * a.G + g) * a.d, a.d, a.start_abs + i, a.krot + kr * a.d, threadIdx.x, blockDim.x);
        return;
    }
    const int s = seg_of(a, j);
    const AttendSeg& sg = a.segs[s];
    const int64_t row = j - sg.col0;
    if (a.absolute || sg.kind == INFLLM_SEG_LOCAL)
        rot_row<T>(a.freqs, sg.keys, (row * a.G + g) * a.d, a.d, sg.start_abs + row, a.krot + kr * a.d, threadIdx.x,
                   blockDim.x);
}

// (2) one block per (query row, head): scores (attention.hpp:153-205), softmax
// (207-216), out = sum w V (218-225), per-segment mass partials (engine.hpp:271-283)
template <typename T>
__global__ void __launch_bounds__(256) k_attend_rows(AttendParams a) {
    extern __shared__ float sm[];  // qa | qc
    const int64_t i = blockIdx.x;
    const int h = blockIdx.y, g = h / a.rep;
    const int64_t r = static_cast<int64_t>(h) * a.lx + i;
    const int64_t nq = static_cast<int64_t>(a.H) * a.lx;
    float* qa = sm;
    float* qc = sm + a.d;
    for (int c = threadIdx.x; c < a.d; c += blockDim.x) {
        qa[c] = a.qrot[r * a.d + c];
        qc[c] = a.qrot[(nq + r) * a.d + c];
    }
    __syncthreads();
    const float scale = 1.0f / sqrtf(static_cast<float>(a.d));  // attention.hpp:140
    const float neg_inf = -INFINITY;
    float* srow = a.scores + r * a.n_all;
    const int64_t qpos = a.start_abs + i;
    const int64_t valid = a.n_ctx + i + 1;  // causal within the batch (204-205)
    for (int64_t j = threadIdx.x; j < a.n_all; j += blockDim.x) {
        if (j >= valid) {
            srow[j] = neg_inf;
            continue;
        }
        const float* qv;
        const void* kp;
        int64_t koff;
        bool rotated;
        if (j >= a.n_ctx) {
            const int64_t bi = j - a.n_ctx;
            rotated = true;
            kp = nullptr;
            koff = 0;
            // batch keys are near unless farther than l_L (clamped mode, 190-200)
            if (!a.absolute && qpos - (a.start_abs + bi) > a.L) {
                rotated = false;
                kp = a.k;
                koff = (bi * a.G + g) * a.d;
            }
        } else {
            const AttendSeg& sg = a.segs[seg_of(a, j)];
            const int64_t row = j - sg.col0;
            if (a.absolute) {
                rotated = true;
            } else if (sg.kind != INFLLM_SEG_LOCAL) {
                rotated = false;  // initial / retrieved: clamped distance l_L (166-173)
            } else {
                rotated = qpos - (sg.start_abs + row) <= a.L;  // local: switch to the clamp beyond l_L
            }
            kp = sg.keys;
            koff = (row * a.G + g) * a.d;
        }
        float acc = 0.f;
        if (rotated) {
            qv = qa;
            const float* kr = a.krot + (j * a.G + g) * a.d;
            for (int c = 0; c < a.d; ++c) acc = fmaf(qv[c], kr[c], acc);
        } else {
            qv = qc;
            for (int c = 0; c < a.d; ++c) acc = fmaf(qv[c], ld_f<T>(kp, koff + c), acc);
        }
        srow[j] = acc * scale;
    }
    __syncthreads();
    // softmax over the valid columns (max-subtracted, attention.hpp:207-216)
    __shared__ float red[32];
    float m = neg_inf;
    for (int64_t j = threadIdx.x; j < valid; j += blockDim.x) m = fmaxf(m, srow[j]);
    m = warp_max_f(m);
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        float x = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : neg_inf;
        x = warp_max_f(x);
        if (threadIdx.x == 0) red[0] = x;
    }
    __syncthreads();
    m = red[0];
    __syncthreads();
    float sum = 0.f;
    for (int64_t j = threadIdx.x; j < a.n_all; j += blockDim.x) {
        const float e = j < valid ? expf(srow[j] - m) : 0.f;
        srow[j] = e;
        sum += e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) t += red[w];
        red[0] = t;
    }
    __syncthreads();
    const float inv = 1.0f / red[0];
    for (int64_t j = threadIdx.x; j < a.n_all; j += blockDim.x) srow[j] *= inv;
    __syncthreads();
    // per-segment mass partials of this (row, head), in column order
    if (a.mass_part)
        for (int s = threadIdx.x; s < a.n_seg; s += blockDim.x) {
            double ms = 0.0;
            for (int64_t j = a.segs[s].col0; j < a.segs[s].col0 + a.segs[s].n; ++j) ms += static_cast<double>(srow[j]);
            a.mass_part[r * a.n_seg + s] = ms;
        }
    // out = sum_j w_j v_j
    for (int c = threadIdx.x; c < a.dv; c += blockDim.x) {
        float o = 0.f;
        for (int64_t j = 0; j < valid; ++j) {
            float vj;
            if (j >= a.n_ctx)
                vj = ld_f<T>(a.v, ((j - a.n_ctx) * a.G + g) * a.dv + c);
            else {
                const AttendSeg& sg = a.segs[seg_of(a, j)];
                vj = ld_f<T>(sg.values, ((j - sg.col0) * a.G + g) * a.dv + c);
            }
            o = fmaf(srow[j], vj, o);
        }
        static_cast<T*>(a.out)[(i * a.H + h) * a.dv + c] = from_f<T>(o);
    }
}

// (3) mass_u = sum_h sum_rows sum_cols w / H, reduced in (head, row) order
__global__ void k_attend_mass(const double* part, int64_t rows, int n_seg, int H, double* mass) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    double m = 0.0;
    for (int64_t r = 0; r < rows; ++r) m += part[r * n_seg + s];
    mass[s] = m / static_cast<double>(H);
}

void attend_run(const AttendLaunch& L, cudaStream_t st) {
    AttendParams a{};
    a.segs = static_cast<const AttendSeg*>(L.dev_segs);
    a.n_seg = L.n_seg;
    a.q = L.q;
    a.k = L.k;
    a.v = L.v;
    a.out = L.out;
    a.scores = L.scores;
    a.mass_part = L.mass_part;
    a.qrot = L.qrot;
    a.krot = L.krot;
    a.lx = L.lx;
    a.n_ctx = L.n_ctx;
    a.n_all = L.n_ctx + L.lx;
    a.start_abs = L.start_abs;
    a.L = L.local_size;
    a.H = L.H;
    a.G = L.G;
    a.rep = L.H / L.G;
    a.d = L.d;
    a.dv = L.dv;
    a.absolute = L.absolute;
    a.freqs = L.freqs;
    const int64_t nrot = static_cast<int64_t>(L.H) * L.lx + a.n_all * L.G;  // query rows, then keys
    const size_t smem = 2 * static_cast<size_t>(L.d) * sizeof(float);
    if (L.bf16) {
        k_attend_rotate<bf16><<<static_cast<unsigned>(nrot), 64, 0, st>>>(a);
        k_attend_rows<bf16><<<dim3(static_cast<unsigned>(L.lx), L.H), 256, smem, st>>>(a);
    } else {
        k_attend_rotate<float><<<static_cast<unsigned>(nrot), 64, 0, st>>>(a);
        k_attend_rows<float><<<dim3(static_cast<unsigned>(L.lx), L.H), 256, smem, st>>>(a);
    }
    if (L.mass && L.n_seg > 0)
        k_attend_mass<<<(L.n_seg + 127) / 128, 128, 0, st>>>(L.mass_part, static_cast<int64_t>(L.H) * L.lx, L.n_seg,
                                                             L.H, L.mass);
}

size_t attend_seg_bytes() { return sizeof(AttendSeg); }
void attend_pack_seg(void* dst, int idx, const void* keys, const void* values, int64_t start_abs, int64_t n,
                     int64_t col0, int kind) {
    static_cast<AttendSeg*>(dst)[idx] = AttendSeg{keys, values, start_abs, n, col0, kind};
}

// ------------------------------------------------------------ TieredStore
// repr [U][G][r_k][d] (the lookup index layout of the engine), freq [U] fp64,
// hot [U] int8, hot_list, LruState, trace [3] int64 per record.
__global__ void k_store_put_repr(const void* src, void* repr, int64_t u, int n_repr, int r_k, int G, int d, int esz) {
    // src [n_repr][G][d] -> repr[u][g][r][d]; rows r >= n_repr are zero (they add 0.0 to the relevance)
    const int64_t n = static_cast<int64_t>(G) * r_k * d;
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int g = static_cast<int>(t / (static_cast<int64_t>(r_k) * d));
        const int r = static_cast<int>((t / d) % r_k);
        const int c = static_cast<int>(t % d);
        uint8_t* dst = static_cast<uint8_t*>(repr) + ((u * G + g) * r_k + r) * static_cast<int64_t>(d) * esz +
                       static_cast<int64_t>(c) * esz;
        if (r < n_repr) {
            const uint8_t* s = static_cast<const uint8_t*>(src) + ((static_cast<int64_t>(r) * G + g) * d + c) * esz;
            for (int b = 0; b < esz; ++b) dst[b] = s[b];
        } else {
            for (int b = 0; b < esz; ++b) dst[b] = 0;
        }
    }
}

// lookup bookkeeping (memory.hpp:254-267): ids ascending
__global__ void k_store_book(StoreDev s, const int64_t* ids, int64_t n, int64_t step) {
    if (threadIdx.x != 0) return;
    LruState st = *s.lru;
    for (int64_t j = 0; j < n; ++j) {
        const int64_t id = ids[j];
        st.requested++;
        int64_t* tr = s.trace + 3 * st.trace_count;
        tr[0] = step;
        tr[1] = id;
        if (s.hot[id]) {
            st.hits++;
            tr[2] = 1;
        } else {
            st.misses++;
            st.loads++;
            s.hot[id] = 1;
            s.hot_list[st.hot_count++] = id;
            tr[2] = 0;
        }
        st.trace_count++;
    }
    *s.lru = st;
}

// update_frequency (memory.hpp:273-281): decay every hot unit, then add the masses in order
__global__ void k_store_update(StoreDev s, const int64_t* ids, const double* mass, int64_t n) {
    if (threadIdx.x != 0) return;
    const LruState st = *s.lru;
    for (int64_t a = 0; a < st.hot_count; ++a) s.freq[s.hot_list[a]] *= s.decay;
    for (int64_t j = 0; j < n; ++j) {
        const int64_t id = ids[j];
        if (id < 0 || id >= s.n_units || !s.hot[id]) {
            *s.err = 1;  // "update_frequency: mass for a unit that is not hot"
            return;
        }
        s.freq[id] += mass[j];
    }
}

// enforce_capacity (memory.hpp:285-300): evict min (s_b, id) while over capacity
__global__ void k_store_enforce(StoreDev s) {
    if (threadIdx.x != 0) return;
    LruState st = *s.lru;
    while (st.hot_count > s.cap) {
        int64_t w = 0;
        for (int64_t a = 1; a < st.hot_count; ++a) {
            const int64_t ia = s.hot_list[a], iw = s.hot_list[w];
            if (s.freq[ia] < s.freq[iw] || (s.freq[ia] == s.freq[iw] && ia < iw)) w = a;
        }
        s.hot[s.hot_list[w]] = 0;
        s.hot_list[w] = s.hot_list[st.hot_count - 1];
        st.hot_count--;
        st.evictions++;
    }
    *s.lru = st;
}

// note_step_boundary (memory.hpp:303-308)
__global__ void k_store_boundary(StoreDev s) {
    if (threadIdx.x != 0) return;
    LruState st = *s.lru;
    if (st.hot_count > s.cap) {
        *s.err = 2;  // "TieredStore: hot tier over capacity at step end"
        return;
    }
    int64_t bytes = 0;
    for (int64_t a = 0; a < st.hot_count; ++a) bytes += s.bytes_per_token * s.unit_tokens[s.hot_list[a]];
    if (st.hot_count > st.peak_hot_units) st.peak_hot_units = st.hot_count;
    if (bytes > st.peak_hot_bytes) st.peak_hot_bytes = bytes;
    *s.lru = st;
}

// per KV group query sums of a batch, fp64 (memory.hpp:224-225 summed over the group's heads)
template <typename T>
__global__ void k_store_qsum(const void* q, int64_t lx, int H, int G, int d, double* qsum) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= G * d) return;
    const int g = t / d, c = t % d, rep = H / G;
    double a = 0.0;
    for (int hh = 0; hh < rep; ++hh)
        for (int64_t i = 0; i < lx; ++i) a += static_cast<double>(to_f(static_cast<const T*>(q)[(i * H + g * rep + hh) * d + c]));
    qsum[t] = a;
}
void store_qsum(const void* q, int64_t lx, int H, int G, int d, bool is_bf16, double* qsum, cudaStream_t st) {
    const unsigned b = static_cast<unsigned>((G * d + 127) / 128);
    if (is_bf16)
        k_store_qsum<bf16><<<b, 128, 0, st>>>(q, lx, H, G, d, qsum);
    else
        k_store_qsum<float><<<b, 128, 0, st>>>(q, lx, H, G, d, qsum);
}

void store_put_repr(const void* src, void* repr, int64_t u, int n_repr, int r_k, int G, int d, int esz,
                    cudaStream_t st) {
    k_store_put_repr<<<8, 256, 0, st>>>(src, repr, u, n_repr, r_k, G, d, esz);
}
void store_book(const StoreDev& s, const int64_t* ids, int64_t n, int64_t step, cudaStream_t st) {
    k_store_book<<<1, 32, 0, st>>>(s, ids, n, step);
}
void store_update(const StoreDev& s, const int64_t* ids, const double* mass, int64_t n, cudaStream_t st) {
    k_store_update<<<1, 32, 0, st>>>(s, ids, mass, n);
}
void store_enforce(const StoreDev& s, cudaStream_t st) { k_store_enforce<<<1, 32, 0, st>>>(s); }
void store_boundary(const StoreDev& s, cudaStream_t st) { k_store_boundary<<<1, 32, 0, st>>>(s); }

// ------------------------------------------------------- ScoreAccumulator
// accumulate (repr_score.hpp:39-69): sums[m] += sum over the batch rows i with
// m + 1 <= s + i <= m + l_L of sum_h q_{i,h} . k_m, in fp64. Per pending key
// one block: B[g][c] = sum_i sum_{h in g} q (rows in order), then the dot with k.
template <typename T>
__global__ void __launch_bounds__(256) k_score_acc(const void* q, int64_t lx, int64_t s, const void* keys,
                                                   int64_t n_pending, int64_t lo, int64_t L, int H, int G, int d,
                                                   double* sums, int64_t ring0, int64_t cap) {
    const int64_t j = blockIdx.x;
    const int64_t m = lo + j;
    const int64_t first = m + 1 - s > 0 ? m + 1 - s : 0, last = m + L - s < lx - 1 ? m + L - s : lx - 1;
    if (first > last) return;
    const int rep = H / G;
    double part = 0.0;
    for (int t = threadIdx.x; t < G * d; t += blockDim.x) {
        const int g = t / d, c = t % d;
        double b = 0.0;
        for (int64_t i = first; i <= last; ++i)
            for (int hh = 0; hh < rep; ++hh)
                b += static_cast<double>(to_f(static_cast<const T*>(q)[(i * H + g * rep + hh) * d + c]));
        part += b * static_cast<double>(to_f(static_cast<const T*>(keys)[(j * G + g) * d + c]));
    }
    __shared__ double red[8];
    part = warp_sum_d(part);
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) a += red[w];
        sums[(ring0 + j) % cap] += a;
    }
}
__global__ void k_score_final(const double* sums, int64_t ring0, int64_t cap, int64_t n, int64_t L, float* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = static_cast<float>(sums[(ring0 + i) % cap] / static_cast<double>(L));  // 72-82
}
__global__ void k_score_zero(double* sums, int64_t from, int64_t n, int64_t cap) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) sums[(from + i) % cap] = 0.0;
}

void score_acc_run(const void* q, int64_t lx, int64_t s, const void* keys, int64_t n_pending, int64_t lo, int64_t L,
                   int H, int G, int d, bool is_bf16, double* sums, int64_t ring0, int64_t cap, cudaStream_t st) {
    if (n_pending <= 0) return;
    if (is_bf16)
        k_score_acc<bf16><<<static_cast<unsigned>(n_pending), 256, 0, st>>>(q, lx, s, keys, n_pending, lo, L, H, G, d,
                                                                           sums, ring0, cap);
    else
        k_score_acc<float><<<static_cast<unsigned>(n_pending), 256, 0, st>>>(q, lx, s, keys, n_pending, lo, L, H, G, d,
                                                                            sums, ring0, cap);
}
void score_acc_final(const double* sums, int64_t ring0, int64_t cap, int64_t n, int64_t L, float* out, cudaStream_t st) {
    if (n > 0) k_score_final<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(sums, ring0, cap, n, L, out);
}
void score_acc_zero(double* sums, int64_t from, int64_t n, int64_t cap, cudaStream_t st) {
    if (n > 0) k_score_zero<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(sums, from, n, cap);
}

}  // namespace infllm
