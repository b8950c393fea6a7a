// infllm_oracle.cpp — TEST INFRASTRUCTURE ONLY (see infllm_oracle.h).
//
// Plain C++20 restatement of the reference engine, in reference step order.
// Scalar = float like the reference default build (real.hpp:7-11); all score
// bookkeeping is double exactly where the reference uses double.
// Paths in citations are relative to /root/reference/proj/include/blockmem/.

#include "infllm_oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

using Index = std::int64_t;
using Scalar = float;

struct ConfigError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct StreamError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

thread_local std::string g_err;

template <typename F>
int32_t guard(F&& f) {
    try {
        f();
        return INFLLM_OK;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return INFLLM_ERR_CONFIG;
    } catch (const StreamError& e) {
        g_err = e.what();
        return INFLLM_ERR_STREAM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return INFLLM_ERR_ARG;
    }
}

// ---------------------------------------------------------------- rng.hpp:11-64
inline std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
inline std::uint64_t hash_mix(std::uint64_t a, std::uint64_t b) { return splitmix64(a ^ splitmix64(b)); }

struct Rng {
    explicit Rng(std::uint64_t seed) : state(splitmix64(seed)) {}
    std::uint64_t next_u64() {
        state += 0x9e3779b97f4a7c15ULL;
        std::uint64_t x = state;
        x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
        x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
        return x ^ (x >> 31);
    }
    double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    std::uint64_t next_below(std::uint64_t n) {
        return static_cast<std::uint64_t>(next_double() * static_cast<double>(n)) % n;
    }
    double next_gaussian() {
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        double u1 = next_double();
        double u2 = next_double();
        while (u1 <= 1e-300) u1 = next_double();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double theta = 6.283185307179586476925286766559 * u2;
        spare = r * std::sin(theta);
        have_spare = true;
        return r * std::cos(theta);
    }
    std::uint64_t state;
    bool have_spare = false;
    double spare = 0.0;
};

// ------------------------------------------------------------ dense helpers
// Row-major matrix; the reference's Mat<Scalar> (types.hpp:12-13).
template <typename T>
struct Mat {
    Index rows = 0, cols = 0;
    std::vector<T> a;
    Mat() = default;
    Mat(Index r, Index c) : rows(r), cols(c), a(static_cast<size_t>(r * c), T(0)) {}
    T* row(Index i) { return a.data() + i * cols; }
    const T* row(Index i) const { return a.data() + i * cols; }
    T& operator()(Index i, Index j) { return a[static_cast<size_t>(i * cols + j)]; }
    T operator()(Index i, Index j) const { return a[static_cast<size_t>(i * cols + j)]; }
    void append_rows(const T* src, Index n) {  // engine.hpp:173-181
        a.insert(a.end(), src, src + n * cols);
        rows += n;
    }
    void drop_front(Index n) {  // engine.hpp:183-185
        a.erase(a.begin(), a.begin() + n * cols);
        rows -= n;
    }
    Mat slice_rows(Index r0, Index n) const {
        Mat m(n, cols);
        std::memcpy(m.a.data(), row(r0), sizeof(T) * static_cast<size_t>(n * cols));
        return m;
    }
};

// C[m][n] = A[m][k] * B[n][k]^T, accumulated sequentially over k in T
// (restates the Eigen products at attention.hpp:157-200; vectorisable order).
template <typename T>
void gemm_nt(const T* A, Index m, Index k, const T* B, Index n, T* C) {
    std::vector<T> bt(static_cast<size_t>(k * n));
    for (Index j = 0; j < n; ++j)
        for (Index kk = 0; kk < k; ++kk) bt[static_cast<size_t>(kk * n + j)] = B[j * k + kk];
    for (Index i = 0; i < m; ++i) {
        T* c = C + i * n;
        for (Index j = 0; j < n; ++j) c[j] = T(0);
        const T* a = A + i * k;
        for (Index kk = 0; kk < k; ++kk) {
            const T av = a[kk];
            const T* b = bt.data() + kk * n;
            for (Index j = 0; j < n; ++j) c[j] += av * b[j];
        }
    }
}

// ------------------------------------------------------------ rotary.hpp:15-72
constexpr double kRotaryBase = 10000.0;

// RotaryTable::make + rotate_row applied to each row (rotary.hpp:19-51,55-62).
Mat<Scalar> rotate_by_positions(const Mat<Scalar>& x, Index start_pos) {
    Mat<Scalar> out = x;
    const int d = static_cast<int>(x.cols);
    const int pairs = d / 2;
    for (int a = 0; a < pairs; ++a) {
        const double freq = std::pow(kRotaryBase, -2.0 * a / d);
        for (Index i = 0; i < x.rows; ++i) {
            const double angle = static_cast<double>(start_pos + i) * freq;
            const Scalar c = static_cast<Scalar>(std::cos(angle));
            const Scalar s = static_cast<Scalar>(std::sin(angle));
            const Scalar x0 = x(i, 2 * a), x1 = x(i, 2 * a + 1);
            out(i, 2 * a) = x0 * c - x1 * s;
            out(i, 2 * a + 1) = x0 * s + x1 * c;
        }
    }
    return out;
}

// rotate_by_constant (rotary.hpp:66-72)
Mat<Scalar> rotate_by_constant(const Mat<Scalar>& x, Index pos) {
    Mat<Scalar> out = x;
    const int d = static_cast<int>(x.cols);
    const int pairs = d / 2;
    for (int a = 0; a < pairs; ++a) {
        const double freq = std::pow(kRotaryBase, -2.0 * a / d);
        const double angle = static_cast<double>(pos) * freq;
        const Scalar c = static_cast<Scalar>(std::cos(angle));
        const Scalar s = static_cast<Scalar>(std::sin(angle));
        for (Index i = 0; i < x.rows; ++i) {
            const Scalar x0 = x(i, 2 * a), x1 = x(i, 2 * a + 1);
            out(i, 2 * a) = x0 * c - x1 * s;
            out(i, 2 * a + 1) = x0 * s + x1 * c;
        }
    }
    return out;
}

// ------------------------------------------------------------ config (types.hpp:84-110)
void validate(const infllm_engine_config& c) {
    if (c.chunk_size < 1) throw ConfigError("chunk_size must be >= 1");
    if (c.unit_size < 1) throw ConfigError("unit_size must be >= 1");
    if (c.n_repr < 1) throw ConfigError("n_repr must be >= 1");
    if (c.local_size < 1) throw ConfigError("local_size must be >= 1");
    if (c.init_size < 0) throw ConfigError("init_size must be >= 0");
    if (c.n_lookup < 0) throw ConfigError("n_lookup must be >= 0");
    if (c.n_repr > c.unit_size) throw ConfigError("n_repr must not exceed unit_size");
    if (c.hot_capacity < c.n_lookup) throw ConfigError("hot_capacity must be >= n_lookup");
    if (c.decay < 0.0 || c.decay > 1.0) throw ConfigError("decay must lie in [0, 1]");
    if (c.lookup_mode < 0 || c.lookup_mode > 2) throw ConfigError("lookup_mode: unknown value");
    if (c.position_mode < 0 || c.position_mode > 1)
        throw ConfigError("position_mode: unknown value");
}

// ------------------------------------------------------------ memory.hpp:19-41
struct MemoryUnit {
    std::int64_t unit_id = 0;
    Index start_abs = 0;
    std::vector<Mat<Scalar>> keys, values;  // per KV head [size][d]
    std::vector<Index> repr_abs;
    std::vector<Mat<Scalar>> repr_keys;  // per KV head [n_repr][d]
    double freq_score = 0.0;
    bool hot = false;
    Index size() const { return keys.empty() ? 0 : keys.front().rows; }
    Index end_abs() const { return start_abs + size(); }
};

// select_representatives (repr_score.hpp:94-112)
std::vector<Index> select_representatives(const Scalar* scores, Index n, Index r_k) {
    if (n == 0) throw StreamError("select_representatives: empty unit");
    std::vector<Index> idx(static_cast<size_t>(n));
    std::iota(idx.begin(), idx.end(), Index(0));
    const Index take = std::min(r_k, n);
    std::partial_sort(idx.begin(), idx.begin() + take, idx.end(), [&](Index a, Index b) {
        if (scores[a] != scores[b]) return scores[a] > scores[b];
        return a < b;
    });
    idx.resize(static_cast<size_t>(take));
    std::sort(idx.begin(), idx.end());
    return idx;
}

// ScoreAccumulator (repr_score.hpp:21-89)
struct ScoreAccumulator {
    Index local_size;
    Index lo = 0, hi = 0, next_query_abs = 0;
    std::deque<double> sums;
    int n_threads = 1;

    // accumulate (repr_score.hpp:39-69). q: per expanded head [l_x][d];
    // pending keys: per KV head [n_pending][d]; head h uses group h / rep.
    void accumulate(Index s, const std::vector<Mat<Scalar>>& q,
                    const std::vector<Mat<Scalar>>& pending_keys, int rep) {
        const Index l_x = q.front().rows;
        if (s != next_query_abs) throw StreamError("ScoreAccumulator: out-of-order query batch");
        if (hi != s) throw StreamError("ScoreAccumulator: pending range out of sync");
        hi = s + l_x;
        sums.resize(sums.size() + static_cast<size_t>(l_x), 0.0);
        const Index n_pending = hi - lo;
        if (pending_keys.front().rows != n_pending)
            throw StreamError("ScoreAccumulator: pending keys do not cover range");
        const Index d = q.front().cols;
        // dots += q_h(double) * pending_h(double)^T, head by head (repr_score.hpp:53-57).
        // Per-thread partial dots over disjoint head ranges, merged in head order.
        const int H = static_cast<int>(q.size());
        const int nt = std::max(1, std::min(n_threads, H));
        std::vector<std::vector<double>> part(static_cast<size_t>(nt));
        auto work = [&](int t) {
            auto& dots = part[static_cast<size_t>(t)];
            dots.assign(static_cast<size_t>(l_x * n_pending), 0.0);
            std::vector<double> tmp(static_cast<size_t>(l_x * n_pending));
            std::vector<double> qd(static_cast<size_t>(l_x * d)), kd(static_cast<size_t>(n_pending * d));
            for (int h = t; h < H; h += nt) {
                const auto& qh = q[static_cast<size_t>(h)];
                const auto& kh = pending_keys[static_cast<size_t>(h / rep)];
                for (size_t i = 0; i < qd.size(); ++i) qd[i] = qh.a[i];
                for (size_t i = 0; i < kd.size(); ++i) kd[i] = kh.a[i];
                gemm_nt<double>(qd.data(), l_x, d, kd.data(), n_pending, tmp.data());
                for (size_t i = 0; i < tmp.size(); ++i) dots[i] += tmp[i];
            }
        };
        run_threads(nt, work);
        std::vector<double>& dots = part[0];
        for (int t = 1; t < nt; ++t)
            for (size_t i = 0; i < dots.size(); ++i) dots[i] += part[static_cast<size_t>(t)][i];
        for (Index j = 0; j < n_pending; ++j) {
            const Index m = lo + j;
            const Index first = std::max<Index>(0, m + 1 - s);
            const Index last = std::min<Index>(l_x - 1, m + local_size - s);
            if (first > last) continue;
            double acc = 0.0;
            for (Index i = first; i <= last; ++i) acc += dots[static_cast<size_t>(i * n_pending + j)];
            sums[static_cast<size_t>(j)] += acc;
        }
        next_query_abs = hi;
    }

    // finalize_front (repr_score.hpp:72-82)
    std::vector<Scalar> finalize_front(Index n) {
        if (n > hi - lo) throw StreamError("ScoreAccumulator: finalize beyond range");
        std::vector<Scalar> out;
        out.reserve(static_cast<size_t>(n));
        for (Index i = 0; i < n; ++i)
            out.push_back(static_cast<Scalar>(sums[static_cast<size_t>(i)] /
                                              static_cast<double>(local_size)));
        sums.erase(sums.begin(), sums.begin() + n);
        lo += n;
        return out;
    }

    template <typename F>
    static void run_threads(int nt, F&& f) {
        if (nt <= 1) {
            f(0);
            return;
        }
        std::vector<std::thread> th;
        for (int t = 1; t < nt; ++t) th.emplace_back(f, t);
        f(0);
        for (auto& x : th) x.join();
    }
};

// UnitPacker (memory.hpp:46-135)
struct UnitPacker {
    Index unit_size, n_repr;
    Index pending_start = 0;
    std::vector<Mat<Scalar>> keys, values;  // per KV head pending rows
    std::vector<Scalar> scores;
    std::int64_t next_unit_id = 0;

    UnitPacker(Index us, Index nr, int hkv, Index d, Index dv) : unit_size(us), n_repr(nr) {
        for (int g = 0; g < hkv; ++g) {
            keys.emplace_back(0, d);
            values.emplace_back(0, dv);
        }
    }
    Index pending_tokens() const { return static_cast<Index>(scores.size()); }

    // add (memory.hpp:59-78)
    std::vector<MemoryUnit> add(Index start_abs, const std::vector<Mat<Scalar>>& k,
                                const std::vector<Mat<Scalar>>& v, const Scalar* sc, Index n) {
        if (n == 0) return {};
        if (pending_tokens() == 0)
            pending_start = start_abs;
        else if (pending_start + pending_tokens() != start_abs)
            throw StreamError("UnitPacker: non-contiguous eviction");
        for (size_t g = 0; g < keys.size(); ++g) {
            keys[g].append_rows(k[g].a.data(), k[g].rows);
            values[g].append_rows(v[g].a.data(), v[g].rows);
        }
        scores.insert(scores.end(), sc, sc + n);
        std::vector<MemoryUnit> done;
        while (pending_tokens() >= unit_size) done.push_back(cut_front(unit_size));
        return done;
    }

    // flush (memory.hpp:81-84)
    bool flush(MemoryUnit& u) {
        if (pending_tokens() == 0) return false;
        u = cut_front(pending_tokens());
        return true;
    }

    // cut_front (memory.hpp:97-127)
    MemoryUnit cut_front(Index n) {
        MemoryUnit u;
        u.unit_id = next_unit_id++;
        u.start_abs = pending_start;
        for (size_t g = 0; g < keys.size(); ++g) {
            u.keys.push_back(keys[g].slice_rows(0, n));
            u.values.push_back(values[g].slice_rows(0, n));
            keys[g].drop_front(n);
            values[g].drop_front(n);
        }
        const auto repr = select_representatives(scores.data(), n, n_repr);
        for (size_t g = 0; g < keys.size(); ++g) {
            Mat<Scalar> rk(static_cast<Index>(repr.size()), u.keys[g].cols);
            for (size_t r = 0; r < repr.size(); ++r)
                std::memcpy(rk.row(static_cast<Index>(r)), u.keys[g].row(repr[r]),
                            sizeof(Scalar) * static_cast<size_t>(rk.cols));
            u.repr_keys.push_back(std::move(rk));
        }
        for (auto r : repr) u.repr_abs.push_back(pending_start + r);
        scores.erase(scores.begin(), scores.begin() + n);
        pending_start += n;
        return u;
    }
};

struct TraceRecord {
    Index step;
    std::int64_t unit_id;
    bool hit;
};

// TieredStore (memory.hpp:170-323)
struct TieredStore {
    Index hot_capacity;
    double decay;
    int H, rep;  // expanded heads, heads per KV group
    std::vector<MemoryUnit> units;
    std::vector<std::int64_t> hot;
    std::vector<Mat<double>> repr_index;  // per KV head [rows][d] (double, memory.hpp:207)
    std::vector<std::pair<Index, Index>> repr_spans;
    Index repr_rows = 0;
    infllm_layer_metrics counters{};
    std::vector<TraceRecord> trace;
    Index step = 0;
    Index peak_hot_units = 0;
    std::size_t peak_hot_bytes = 0;
    std::size_t unit_bytes_per_token = 0;

    Index total_units() const { return static_cast<Index>(units.size()); }

    // add_unit (memory.hpp:196-212)
    void add_unit(MemoryUnit u) {
        if (u.unit_id != static_cast<std::int64_t>(units.size()))
            throw StreamError("TieredStore: unit ids must be sequential");
        u.hot = false;
        const Index add = u.repr_keys.front().rows;
        for (size_t g = 0; g < repr_index.size(); ++g) {
            auto& idx = repr_index[g];
            if (idx.cols == 0) idx.cols = u.repr_keys[g].cols;
            for (Index r = 0; r < add; ++r)
                for (Index c = 0; c < idx.cols; ++c)
                    idx.a.push_back(static_cast<double>(u.repr_keys[g](r, c)));
            idx.rows += add;
        }
        repr_spans.emplace_back(repr_rows, add);
        repr_rows += add;
        units.push_back(std::move(u));
    }

    // relevance_all (memory.hpp:217-234); q per expanded head [l_x][d]
    std::vector<double> relevance_all(const std::vector<Mat<Scalar>>& q) const {
        std::vector<double> rel(units.size(), 0.0);
        if (units.empty()) return rel;
        std::vector<double> per_repr(static_cast<size_t>(repr_rows), 0.0);
        const Index d = q.front().cols;
        std::vector<double> qsum(static_cast<size_t>(d));
        for (int h = 0; h < H; ++h) {
            const auto& qh = q[static_cast<size_t>(h)];
            std::fill(qsum.begin(), qsum.end(), 0.0);
            for (Index i = 0; i < qh.rows; ++i)
                for (Index c = 0; c < d; ++c) qsum[static_cast<size_t>(c)] += static_cast<double>(qh(i, c));
            const auto& idx = repr_index[static_cast<size_t>(h / rep)];
            for (Index r = 0; r < repr_rows; ++r) {
                double acc = 0.0;
                const double* row = idx.row(r);
                for (Index c = 0; c < d; ++c) acc += row[c] * qsum[static_cast<size_t>(c)];
                per_repr[static_cast<size_t>(r)] += acc;
            }
        }
        for (size_t u = 0; u < units.size(); ++u) {
            const auto [off, len] = repr_spans[u];
            double s = 0.0;
            for (Index r = 0; r < len; ++r) s += per_repr[static_cast<size_t>(off + r)];
            rel[u] = s;
        }
        return rel;
    }

    // lookup (memory.hpp:239-269)
    std::vector<std::int64_t> lookup(const std::vector<Mat<Scalar>>& q, Index k_m) {
        const Index take = std::min<Index>(k_m, total_units());
        if (take <= 0) return {};
        const auto rel = relevance_all(q);
        std::vector<std::int64_t> ids(units.size());
        std::iota(ids.begin(), ids.end(), std::int64_t(0));
        std::partial_sort(ids.begin(), ids.begin() + take, ids.end(),
                          [&](std::int64_t a, std::int64_t b) {
                              const double ra = rel[static_cast<size_t>(a)];
                              const double rb = rel[static_cast<size_t>(b)];
                              if (ra != rb) return ra > rb;
                              return a < b;
                          });
        ids.resize(static_cast<size_t>(take));
        std::sort(ids.begin(), ids.end());
        for (auto id : ids) {
            auto& u = units[static_cast<size_t>(id)];
            counters.requested++;
            if (u.hot) {
                counters.hits++;
                trace.push_back({step, id, true});
            } else {
                counters.misses++;
                counters.loads++;
                u.hot = true;
                hot.push_back(id);
                trace.push_back({step, id, false});
            }
        }
        return ids;
    }

    // update_frequency (memory.hpp:273-281)
    void update_frequency(const std::vector<std::pair<std::int64_t, double>>& masses) {
        for (auto id : hot) units[static_cast<size_t>(id)].freq_score *= decay;
        for (const auto& [id, mass] : masses) {
            auto& u = units[static_cast<size_t>(id)];
            if (!u.hot) throw StreamError("update_frequency: mass for a unit that is not hot");
            u.freq_score += mass;
        }
    }

    // enforce_capacity (memory.hpp:285-300)
    void enforce_capacity() {
        while (static_cast<Index>(hot.size()) > hot_capacity) {
            size_t worst = 0;
            for (size_t i = 1; i < hot.size(); ++i) {
                const auto& a = units[static_cast<size_t>(hot[i])];
                const auto& b = units[static_cast<size_t>(hot[worst])];
                if (a.freq_score < b.freq_score ||
                    (a.freq_score == b.freq_score && hot[i] < hot[worst]))
                    worst = i;
            }
            units[static_cast<size_t>(hot[worst])].hot = false;
            hot[worst] = hot.back();
            hot.pop_back();
            counters.evictions++;
        }
    }

    std::size_t hot_bytes() const {
        std::size_t b = 0;
        for (auto id : hot)
            b += unit_bytes_per_token * static_cast<std::size_t>(units[static_cast<size_t>(id)].size());
        return b;
    }

    // note_step_boundary (memory.hpp:303-308)
    void note_step_boundary() {
        if (static_cast<Index>(hot.size()) > hot_capacity)
            throw StreamError("TieredStore: hot tier over capacity at step end");
        peak_hot_units = std::max<Index>(peak_hot_units, static_cast<Index>(hot.size()));
        peak_hot_bytes = std::max(peak_hot_bytes, hot_bytes());
    }
};

enum class Seg { initial, retrieved, local };

struct SegmentView {  // attention.hpp:29-38 (per KV head matrices)
    Seg kind;
    Index start_abs;
    std::int64_t unit_id;
    std::vector<const Mat<Scalar>*> keys, values;
    Index size() const { return keys.empty() ? 0 : keys.front()->rows; }
};

}  // namespace

// ------------------------------------------------------------------ engine
struct oracle_engine {
    infllm_engine_config cfg{};
    int H = 1, Hkv = 1, rep = 1, d = 0, dv = 0, n_layers = 1;
    int n_threads = 1;
    bool always_emit = false;
    std::uint64_t checks = 0, violations = 0;
    double t_ms[5] = {0, 0, 0, 0, 0};

    struct Layer {
        std::vector<Mat<Scalar>> init_keys, init_values, local_keys, local_values;  // per KV head
        Index local_start = 0;
        ScoreAccumulator acc;
        UnitPacker packer;
        TieredStore store;
        Index n_fed = 0, step = 0;
        std::vector<Scalar> evicted_scores;  // finalized r_m of every evicted token (diagnostic)
        Layer(const infllm_engine_config& c, int Hkv, int d, int dv)
            : acc{c.local_size, 0, 0, 0, {}, 1}, packer(c.unit_size, c.n_repr, Hkv, d, dv) {}
        Index initial_len() const { return init_keys.front().rows; }
        Index local_len() const { return local_keys.front().rows; }
    };
    std::vector<Layer> layers;

    // attend (attention.hpp:116-230) for expanded head h. q: [l_x][d] this
    // head; window segments; batch k/v for this head's group.
    void attend_head(int h, const Mat<Scalar>& q, Index start_abs, const std::vector<SegmentView>& segs,
                     const Mat<Scalar>& bk, const Mat<Scalar>& bv, Mat<Scalar>& out,
                     Mat<Scalar>* weights_out) const {
        const int g = h / rep;
        const Index l_x = q.rows;
        Index n_ctx = 0;
        for (const auto& s : segs) n_ctx += s.size();
        const Index n_all = n_ctx + l_x;
        const Index L = cfg.local_size;
        const Scalar scale = Scalar(1) / std::sqrt(Scalar(d));
        const Scalar neg_inf = -std::numeric_limits<Scalar>::infinity();
        Mat<Scalar> scores(l_x, n_all);
        std::vector<Scalar> tmp;
        auto put_cols = [&](const Mat<Scalar>& a, const Mat<Scalar>& keys, Index col) {
            tmp.resize(static_cast<size_t>(l_x * keys.rows));
            gemm_nt<Scalar>(a.a.data(), l_x, d, keys.a.data(), keys.rows, tmp.data());
            for (Index i = 0; i < l_x; ++i)
                std::memcpy(scores.row(i) + col, tmp.data() + i * keys.rows,
                            sizeof(Scalar) * static_cast<size_t>(keys.rows));
        };
        // apply_distance_cap (attention.hpp:96-108)
        auto cap = [&](const Mat<Scalar>& qc, const Mat<Scalar>& keys, Index col, Index col0_abs) {
            tmp.resize(static_cast<size_t>(l_x * keys.rows));
            gemm_nt<Scalar>(qc.a.data(), l_x, d, keys.a.data(), keys.rows, tmp.data());
            for (Index j = 0; j < keys.rows; ++j) {
                const Index key_abs = col0_abs + j;
                const Index first = std::max<Index>(0, L + key_abs - start_abs + 1);
                for (Index i = first; i < l_x; ++i) scores(i, col + j) = tmp[static_cast<size_t>(i * keys.rows + j)];
            }
        };
        if (cfg.position_mode == INFLLM_POSITION_ABSOLUTE) {
            const Mat<Scalar> q_abs = rotate_by_positions(q, start_abs);
            Index col = 0;
            for (const auto& s : segs) {
                put_cols(q_abs, rotate_by_positions(*s.keys[static_cast<size_t>(g)], s.start_abs), col);
                col += s.size();
            }
            put_cols(q_abs, rotate_by_positions(bk, start_abs), col);
        } else {
            const Mat<Scalar> q_clamp = rotate_by_constant(q, L);
            const Mat<Scalar> q_abs = rotate_by_positions(q, start_abs);
            Index col = 0;
            for (const auto& s : segs) {
                const Mat<Scalar>& keys = *s.keys[static_cast<size_t>(g)];
                if (s.kind != Seg::local) {
                    put_cols(q_clamp, keys, col);
                } else {
                    put_cols(q_abs, rotate_by_positions(keys, s.start_abs), col);
                    const Index max_dist = (start_abs + l_x - 1) - s.start_abs;
                    if (max_dist > L) cap(q_clamp, keys, col, s.start_abs);
                }
                col += s.size();
            }
            put_cols(q_abs, rotate_by_positions(bk, start_abs), col);
            if (l_x - 1 > L) cap(q_clamp, bk, col, start_abs);
        }
        for (auto& x : scores.a) x *= scale;
        for (Index i = 0; i < l_x; ++i)
            for (Index j = i + 1; j < l_x; ++j) scores(i, n_ctx + j) = neg_inf;
        Mat<Scalar> w(l_x, n_all);
        for (Index i = 0; i < l_x; ++i) {
            const Index valid = n_ctx + i + 1;
            Scalar m = scores(i, 0);
            for (Index j = 1; j < valid; ++j) m = std::max(m, scores(i, j));
            Scalar sum = 0;
            for (Index j = 0; j < valid; ++j) {
                w(i, j) = std::exp(scores(i, j) - m);
                sum += w(i, j);
            }
            for (Index j = 0; j < n_all; ++j) w(i, j) /= sum;
        }
        // out = sum_seg W_seg V_seg + W_batch V_batch (attention.hpp:218-225)
        out = Mat<Scalar>(l_x, dv);
        std::vector<Scalar> acc(static_cast<size_t>(dv));
        auto add_pv = [&](Index col, const Mat<Scalar>& vals) {
            for (Index i = 0; i < l_x; ++i) {
                std::fill(acc.begin(), acc.end(), Scalar(0));
                const Scalar* wr = w.row(i) + col;
                for (Index j = 0; j < vals.rows; ++j) {
                    const Scalar wj = wr[j];
                    const Scalar* vr = vals.row(j);
                    for (Index c = 0; c < dv; ++c) acc[static_cast<size_t>(c)] += wj * vr[c];
                }
                Scalar* o = out.row(i);
                for (Index c = 0; c < dv; ++c) o[c] += acc[static_cast<size_t>(c)];
            }
        };
        Index col = 0;
        for (const auto& s : segs) {
            add_pv(col, *s.values[static_cast<size_t>(g)]);
            col += s.size();
        }
        add_pv(col, bv);
        if (weights_out) *weights_out = std::move(w);
    }

    // compose_window (engine.hpp:187-231)
    std::vector<SegmentView> compose_window(Layer& layer, const std::vector<std::int64_t>& ids) {
        std::vector<SegmentView> w;
        auto ptrs = [](const std::vector<Mat<Scalar>>& v) {
            std::vector<const Mat<Scalar>*> p;
            for (auto& m : v) p.push_back(&m);
            return p;
        };
        if (layer.initial_len() > 0)
            w.push_back({Seg::initial, 0, -1, ptrs(layer.init_keys), ptrs(layer.init_values)});
        for (auto id : ids) {
            const auto& u = layer.store.units[static_cast<size_t>(id)];
            w.push_back({Seg::retrieved, u.start_abs, id, ptrs(u.keys), ptrs(u.values)});
        }
        if (layer.local_len() > 0)
            w.push_back({Seg::local, layer.local_start, -1, ptrs(layer.local_keys), ptrs(layer.local_values)});
        Index prev_end = 0, prev_start = -1;
        for (const auto& s : w) {
            if (s.start_abs < prev_end || s.start_abs < prev_start)
                throw StreamError("compose_window: overlapping or unordered segments");
            prev_start = s.start_abs;
            prev_end = s.start_abs + s.size();
        }
        return w;
    }

    static double ms_since(std::chrono::steady_clock::time_point& mark) {
        const auto now = std::chrono::steady_clock::now();
        const double ms = std::chrono::duration<double, std::milli>(now - mark).count();
        mark = now;
        return ms;
    }

    // step (engine.hpp:242-359) for one layer with explicit q/k/v.
    void step(int li, const float* q, const float* k, const float* v, Index l_x, bool decode,
              float* out, std::vector<std::int64_t>& retrieved,
              std::vector<std::pair<std::int64_t, double>>& masses) {
        if (l_x < 1) throw StreamError("step: empty batch");
        if (!decode && l_x > cfg.chunk_size) throw StreamError("encode_chunk: batch exceeds chunk_size");
        if (decode && l_x != 1) throw StreamError("decode_step: exactly one token");
        const bool lookup_enabled = decode ? cfg.lookup_mode != INFLLM_LOOKUP_NONE
                                           : cfg.lookup_mode == INFLLM_LOOKUP_ENCODE_AND_DECODE;
        Layer& layer = layers[static_cast<size_t>(li)];
        layer.store.step = layer.step;
        auto mark = std::chrono::steady_clock::now();
        // TokenBatch per head from token-major arrays (types.hpp:158-169)
        const Index s = layer.n_fed;
        std::vector<Mat<Scalar>> bq(static_cast<size_t>(H)), bk(static_cast<size_t>(Hkv)),
            bv(static_cast<size_t>(Hkv));
        for (int h = 0; h < H; ++h) {
            bq[static_cast<size_t>(h)] = Mat<Scalar>(l_x, d);
            for (Index i = 0; i < l_x; ++i)
                std::memcpy(bq[static_cast<size_t>(h)].row(i), q + (i * H + h) * d, sizeof(float) * static_cast<size_t>(d));
        }
        for (int g = 0; g < Hkv; ++g) {
            bk[static_cast<size_t>(g)] = Mat<Scalar>(l_x, d);
            bv[static_cast<size_t>(g)] = Mat<Scalar>(l_x, dv);
            for (Index i = 0; i < l_x; ++i) {
                std::memcpy(bk[static_cast<size_t>(g)].row(i), k + (i * Hkv + g) * d, sizeof(float) * static_cast<size_t>(d));
                std::memcpy(bv[static_cast<size_t>(g)].row(i), v + (i * Hkv + g) * dv, sizeof(float) * static_cast<size_t>(dv));
            }
        }
        t_ms[0] += ms_since(mark);

        const bool do_lookup = lookup_enabled && cfg.n_lookup > 0 && layer.store.total_units() > 0;
        retrieved.clear();
        if (do_lookup) retrieved = layer.store.lookup(bq, cfg.n_lookup);
        t_ms[1] += ms_since(mark);

        auto window = compose_window(layer, retrieved);
        const bool emit = (do_lookup && !retrieved.empty()) || always_emit;
        std::vector<Mat<Scalar>> outs(static_cast<size_t>(H));
        std::vector<Mat<Scalar>> weights(emit ? static_cast<size_t>(H) : 0);
        {
            const int nt = std::max(1, std::min(n_threads, H));
            ScoreAccumulator::run_threads(nt, [&](int t) {
                for (int h = t; h < H; h += nt)
                    attend_head(h, bq[static_cast<size_t>(h)], s, window, bk[static_cast<size_t>(h / rep)],
                                bv[static_cast<size_t>(h / rep)], outs[static_cast<size_t>(h)],
                                emit ? &weights[static_cast<size_t>(h)] : nullptr);
            });
        }
        t_ms[2] += ms_since(mark);
        if (emit) {  // check_softmax (engine.hpp:361-371)
            for (const auto& w : weights)
                for (Index i = 0; i < w.rows; ++i) {
                    ++checks;
                    double sum = 0.0;
                    Scalar mn = w(i, 0);
                    for (Index j = 0; j < w.cols; ++j) {
                        sum += static_cast<double>(w(i, j));
                        mn = std::min(mn, w(i, j));
                    }
                    if (!(mn >= Scalar(0) && std::abs(sum - 1.0) <= 1e-6)) ++violations;
                }
        }
        // masses (engine.hpp:271-283)
        masses.clear();
        if (do_lookup && emit) {
            Index col = 0;
            for (const auto& seg : window) {
                if (seg.kind == Seg::retrieved) {
                    double mass = 0.0;
                    for (const auto& w : weights) {
                        double ms = 0.0;
                        for (Index i = 0; i < w.rows; ++i)
                            for (Index j = 0; j < seg.size(); ++j) ms += static_cast<double>(w(i, col + j));
                        mass += ms;
                    }
                    masses.emplace_back(seg.unit_id, mass / H);
                }
                col += seg.size();
            }
        }
        layer.store.update_frequency(masses);
        layer.store.enforce_capacity();
        t_ms[4] += ms_since(mark);

        // score accumulation over local + batch (engine.hpp:289-299)
        {
            std::vector<Mat<Scalar>> merged(static_cast<size_t>(Hkv));
            for (int g = 0; g < Hkv; ++g) {
                merged[static_cast<size_t>(g)] = layer.local_keys[static_cast<size_t>(g)];
                merged[static_cast<size_t>(g)].append_rows(bk[static_cast<size_t>(g)].a.data(), l_x);
            }
            layer.acc.n_threads = n_threads;
            layer.acc.accumulate(s, bq, merged, rep);
        }
        t_ms[3] += ms_since(mark);
        for (int g = 0; g < Hkv; ++g) {
            layer.local_keys[static_cast<size_t>(g)].append_rows(bk[static_cast<size_t>(g)].a.data(), l_x);
            layer.local_values[static_cast<size_t>(g)].append_rows(bv[static_cast<size_t>(g)].a.data(), l_x);
        }
        // eviction (engine.hpp:306-346)
        const Index overflow = std::max<Index>(0, layer.local_len() - cfg.local_size);
        if (overflow > 0) {
            const auto scores = layer.acc.finalize_front(overflow);
            const Index pop_start = layer.local_start;
            const Index to_init = std::clamp<Index>(cfg.init_size - pop_start, 0, overflow);
            for (int g = 0; g < Hkv; ++g) {
                if (to_init > 0) {
                    layer.init_keys[static_cast<size_t>(g)].append_rows(layer.local_keys[static_cast<size_t>(g)].row(0), to_init);
                    layer.init_values[static_cast<size_t>(g)].append_rows(layer.local_values[static_cast<size_t>(g)].row(0), to_init);
                }
            }
            const Index to_evict = overflow - to_init;
            if (to_evict > 0) {
                std::vector<Mat<Scalar>> ek, ev;
                for (int g = 0; g < Hkv; ++g) {
                    ek.push_back(layer.local_keys[static_cast<size_t>(g)].slice_rows(to_init, to_evict));
                    ev.push_back(layer.local_values[static_cast<size_t>(g)].slice_rows(to_init, to_evict));
                }
                layer.evicted_scores.insert(layer.evicted_scores.end(), scores.begin() + to_init, scores.end());
                auto units = layer.packer.add(pop_start + to_init, ek, ev, scores.data() + to_init, to_evict);
                for (auto& u : units) layer.store.add_unit(std::move(u));
            }
            for (int g = 0; g < Hkv; ++g) {
                layer.local_keys[static_cast<size_t>(g)].drop_front(overflow);
                layer.local_values[static_cast<size_t>(g)].drop_front(overflow);
            }
            layer.local_start += overflow;
        }
        layer.store.note_step_boundary();
        // check_conservation (engine.hpp:373-383)
        {
            ++checks;
            const Index in_units = layer.store.total_units() == 0
                                       ? 0
                                       : layer.store.units.back().end_abs() - cfg.init_size;
            const Index total = layer.initial_len() + layer.local_len() + layer.packer.pending_tokens() + in_units;
            if (total != s + l_x) ++violations;
        }
        t_ms[4] += ms_since(mark);
        for (Index i = 0; i < l_x; ++i)
            for (int h = 0; h < H; ++h)
                std::memcpy(out + (i * H + h) * dv, outs[static_cast<size_t>(h)].row(i), sizeof(float) * static_cast<size_t>(dv));
        layer.n_fed += l_x;
        layer.step += 1;
    }
};

// Bookkeeping-only streaming (CPU-baseline harness, not a reference
// function): advances init/local/packer/store exactly like step() but skips
// lookup and attention, and accumulates representative-score sums through
// per-group query prefix sums (same definition as repr_score.hpp:53-67).
void oracle_engine_warm(oracle_engine* e, int li, const float* q, const float* k, const float* v, Index n) {
    auto& layer = e->layers.at(static_cast<size_t>(li));
    const int H = e->H, Hkv = e->Hkv, d = e->d, dv = e->dv, rep = e->rep;
    const auto& cfg = e->cfg;
    for (Index off = 0; off < n; off += cfg.chunk_size) {
        const Index lx = std::min<Index>(cfg.chunk_size, n - off);
        const Index s = layer.n_fed;
        auto& acc = layer.acc;
        acc.hi = s + lx;
        acc.sums.resize(acc.sums.size() + static_cast<size_t>(lx), 0.0);
        const Index n_pending = acc.hi - acc.lo;
        // prefix over the chunk of qs[g][c]
        std::vector<double> pre(static_cast<size_t>((lx + 1) * Hkv * d), 0.0);
        for (Index i = 0; i < lx; ++i)
            for (int g = 0; g < Hkv; ++g)
                for (int c = 0; c < d; ++c) {
                    double a = 0.0;
                    for (int hh = 0; hh < rep; ++hh) a += q[((off + i) * H + g * rep + hh) * d + c];
                    pre[static_cast<size_t>(((i + 1) * Hkv + g) * d + c)] = pre[static_cast<size_t>((i * Hkv + g) * d + c)] + a;
                }
        for (Index j = 0; j < n_pending; ++j) {
            const Index m = acc.lo + j;
            const Index first = std::max<Index>(0, m + 1 - s);
            const Index last = std::min<Index>(lx - 1, m + cfg.local_size - s);
            if (first > last) continue;
            const float* km = m < s ? nullptr : k + (off + (m - s)) * Hkv * d;
            double tot = 0.0;
            for (int g = 0; g < Hkv; ++g) {
                const float* kr = km ? km + g * d : layer.local_keys[static_cast<size_t>(g)].row(m - layer.local_start);
                for (int c = 0; c < d; ++c)
                    tot += static_cast<double>(kr[c]) * (pre[static_cast<size_t>(((last + 1) * Hkv + g) * d + c)] -
                                                         pre[static_cast<size_t>((first * Hkv + g) * d + c)]);
            }
            acc.sums[static_cast<size_t>(j)] += tot;
        }
        acc.next_query_abs = acc.hi;
        std::vector<Mat<Scalar>> bk, bv;
        for (int g = 0; g < Hkv; ++g) {
            Mat<Scalar> mk(lx, d), mv(lx, dv);
            for (Index i = 0; i < lx; ++i) {
                std::memcpy(mk.row(i), k + ((off + i) * Hkv + g) * d, sizeof(float) * static_cast<size_t>(d));
                std::memcpy(mv.row(i), v + ((off + i) * Hkv + g) * dv, sizeof(float) * static_cast<size_t>(dv));
            }
            layer.local_keys[static_cast<size_t>(g)].append_rows(mk.a.data(), lx);
            layer.local_values[static_cast<size_t>(g)].append_rows(mv.a.data(), lx);
        }
        const Index overflow = std::max<Index>(0, layer.local_len() - cfg.local_size);
        if (overflow > 0) {
            const auto scores = acc.finalize_front(overflow);
            const Index pop_start = layer.local_start;
            const Index to_init = std::clamp<Index>(cfg.init_size - pop_start, 0, overflow);
            for (int g = 0; g < Hkv; ++g)
                if (to_init > 0) {
                    layer.init_keys[static_cast<size_t>(g)].append_rows(layer.local_keys[static_cast<size_t>(g)].row(0), to_init);
                    layer.init_values[static_cast<size_t>(g)].append_rows(layer.local_values[static_cast<size_t>(g)].row(0), to_init);
                }
            const Index to_evict = overflow - to_init;
            if (to_evict > 0) {
                std::vector<Mat<Scalar>> ek, ev;
                for (int g = 0; g < Hkv; ++g) {
                    ek.push_back(layer.local_keys[static_cast<size_t>(g)].slice_rows(to_init, to_evict));
                    ev.push_back(layer.local_values[static_cast<size_t>(g)].slice_rows(to_init, to_evict));
                }
                auto units = layer.packer.add(pop_start + to_init, ek, ev, scores.data() + to_init, to_evict);
                for (auto& u : units) layer.store.add_unit(std::move(u));
            }
            for (int g = 0; g < Hkv; ++g) {
                layer.local_keys[static_cast<size_t>(g)].drop_front(overflow);
                layer.local_values[static_cast<size_t>(g)].drop_front(overflow);
            }
            layer.local_start += overflow;
        }
        layer.n_fed += lx;
        layer.step += 1;
    }
}

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

oracle_engine* oracle_engine_create(const infllm_engine_config* cfg, const infllm_model_shape* shape,
                                    int32_t n_threads) {
    oracle_engine* e = nullptr;
    int32_t rc = guard([&] {
        validate(*cfg);
        if (shape->n_layers < 1 || shape->n_heads < 1 || shape->head_dim < 1)
            throw ConfigError("ModelShape: all fields must be >= 1");
        const int hkv = shape->n_kv_heads > 0 ? shape->n_kv_heads : shape->n_heads;
        if (shape->n_heads % hkv != 0) throw ConfigError("ModelShape: n_heads % n_kv_heads != 0");
        auto* x = new oracle_engine();
        x->cfg = *cfg;
        x->H = shape->n_heads;
        x->Hkv = hkv;
        x->rep = shape->n_heads / hkv;
        x->d = shape->head_dim;
        x->dv = shape->value_dim > 0 ? shape->value_dim : shape->head_dim;
        x->n_layers = shape->n_layers;
        x->n_threads = std::max(1, n_threads);
        for (int l = 0; l < x->n_layers; ++l) {
            oracle_engine::Layer layer(*cfg, hkv, x->d, x->dv);
            for (int g = 0; g < hkv; ++g) {
                layer.init_keys.emplace_back(0, x->d);
                layer.init_values.emplace_back(0, x->dv);
                layer.local_keys.emplace_back(0, x->d);
                layer.local_values.emplace_back(0, x->dv);
            }
            layer.store.hot_capacity = cfg->hot_capacity;
            layer.store.decay = cfg->decay;
            layer.store.H = x->H;
            layer.store.rep = x->rep;
            layer.store.repr_index.resize(static_cast<size_t>(hkv));
            // MemoryUnit::bytes (memory.hpp:33-40) for the GQA-expanded MHA form
            layer.store.unit_bytes_per_token =
                static_cast<size_t>(x->H) * static_cast<size_t>(x->d + x->dv) * sizeof(Scalar);
            x->layers.push_back(std::move(layer));
        }
        e = x;
    });
    return rc == INFLLM_OK ? e : nullptr;
}

void oracle_engine_destroy(oracle_engine* e) { delete e; }

int32_t oracle_warm_start(oracle_engine* e, int32_t layer, const float* q, const float* k, const float* v, int64_t n) {
    return guard([&] { oracle_engine_warm(e, layer, q, k, v, n); });
}
void oracle_set_always_emit_weights(oracle_engine* e, int32_t v) { e->always_emit = v != 0; }

int32_t oracle_step(oracle_engine* e, int32_t layer, const float* q, const float* k, const float* v,
                    int64_t l_x, int32_t is_decode, float* out, int64_t* ids_out, int64_t ids_cap,
                    int64_t* n_ids, double* masses_out) {
    return guard([&] {
        if (layer < 0 || layer >= e->n_layers) throw StreamError("layer out of range");
        std::vector<std::int64_t> ids;
        std::vector<std::pair<std::int64_t, double>> masses;
        e->step(layer, q, k, v, l_x, is_decode != 0, out, ids, masses);
        if (n_ids) *n_ids = static_cast<int64_t>(ids.size());
        for (size_t i = 0; i < ids.size() && static_cast<int64_t>(i) < ids_cap; ++i) {
            if (ids_out) ids_out[i] = ids[i];
            if (masses_out) masses_out[i] = i < masses.size() ? masses[i].second : 0.0;
        }
    });
}

int32_t oracle_finish(oracle_engine* e) {
    return guard([&] {
        for (auto& layer : e->layers) {  // engine.hpp:115-119
            MemoryUnit u;
            if (layer.packer.flush(u)) layer.store.add_unit(std::move(u));
        }
    });
}

int32_t oracle_layer_metrics(oracle_engine* e, int32_t li, infllm_layer_metrics* m) {
    return guard([&] {
        const auto& st = e->layers.at(static_cast<size_t>(li)).store;
        *m = st.counters;
        m->units = st.total_units();
        m->hot_units = static_cast<int64_t>(st.hot.size());
        m->peak_hot_units = st.peak_hot_units;
        m->peak_hot_bytes = static_cast<int64_t>(st.peak_hot_bytes);
    });
}

int32_t oracle_stream_state(oracle_engine* e, int32_t li, int64_t* fed, int64_t* steps, int64_t* init_len,
                            int64_t* local_len, int64_t* pending) {
    return guard([&] {
        const auto& l = e->layers.at(static_cast<size_t>(li));
        *fed = l.n_fed;
        *steps = l.step;
        *init_len = l.initial_len();
        *local_len = l.local_len();
        *pending = l.packer.pending_tokens();
    });
}

int32_t oracle_unit_info(oracle_engine* e, int32_t li, int64_t id, int64_t* start_abs, int64_t* size,
                         int64_t* repr_abs, int64_t* n_repr_out) {
    return guard([&] {
        const auto& st = e->layers.at(static_cast<size_t>(li)).store;
        if (id < 0 || id >= st.total_units()) throw StreamError("unit id out of range");
        const auto& u = st.units[static_cast<size_t>(id)];
        *start_abs = u.start_abs;
        *size = u.size();
        *n_repr_out = static_cast<int64_t>(u.repr_abs.size());
        for (size_t r = 0; r < u.repr_abs.size(); ++r) repr_abs[r] = u.repr_abs[r];
    });
}

int32_t oracle_unit_freq(oracle_engine* e, int32_t li, double* freq, int32_t* hot, int64_t n) {
    return guard([&] {
        const auto& st = e->layers.at(static_cast<size_t>(li)).store;
        for (int64_t i = 0; i < n && i < st.total_units(); ++i) {
            freq[i] = st.units[static_cast<size_t>(i)].freq_score;
            hot[i] = st.units[static_cast<size_t>(i)].hot ? 1 : 0;
        }
    });
}

int32_t oracle_trace(oracle_engine* e, int32_t li, int64_t* step, int64_t* unit, int32_t* hit, int64_t cap,
                     int64_t* n_out) {
    return guard([&] {
        const auto& tr = e->layers.at(static_cast<size_t>(li)).store.trace;
        *n_out = static_cast<int64_t>(tr.size());
        for (size_t i = 0; i < tr.size() && static_cast<int64_t>(i) < cap; ++i) {
            step[i] = tr[i].step;
            unit[i] = tr[i].unit_id;
            hit[i] = tr[i].hit ? 1 : 0;
        }
    });
}

int32_t oracle_invariants(oracle_engine* e, uint64_t* c, uint64_t* v) {
    *c = e->checks;
    *v = e->violations;
    return INFLLM_OK;
}

int32_t oracle_timings(oracle_engine* e, double* ms5) {
    for (int i = 0; i < 5; ++i) ms5[i] = e->t_ms[i];
    return INFLLM_OK;
}

int32_t oracle_evicted_scores(oracle_engine* e, int32_t li, float* scores, int64_t cap, int64_t* n_out) {
    return guard([&] {
        const auto& s = e->layers.at(static_cast<size_t>(li)).evicted_scores;
        *n_out = static_cast<int64_t>(s.size());
        for (size_t i = 0; i < s.size() && static_cast<int64_t>(i) < cap; ++i) scores[i] = s[i];
    });
}

int32_t oracle_unit_repr_keys(oracle_engine* e, int32_t li, int64_t id, float* keys) {
    return guard([&] {
        const auto& st = e->layers.at(static_cast<size_t>(li)).store;
        if (id < 0 || id >= st.total_units()) throw StreamError("unit id out of range");
        const auto& u = st.units[static_cast<size_t>(id)];
        const Index nr = u.repr_keys.front().rows;
        for (Index r = 0; r < nr; ++r)
            for (int g = 0; g < e->Hkv; ++g)
                std::memcpy(keys + (r * e->Hkv + g) * e->d, u.repr_keys[static_cast<size_t>(g)].row(r),
                            sizeof(float) * static_cast<size_t>(e->d));
    });
}

int32_t oracle_select_representatives(const float* scores, int64_t n, int64_t r_k, int64_t* idx, int64_t* n_out) {
    return guard([&] {
        const auto r = select_representatives(scores, n, r_k);
        *n_out = static_cast<int64_t>(r.size());
        for (size_t i = 0; i < r.size(); ++i) idx[i] = r[i];
    });
}

int32_t oracle_argsort_topk(const double* values, int64_t n, int64_t k, int64_t* idx, int64_t* n_out) {
    return guard([&] {  // oracle.hpp:187-195
        std::vector<Index> id(static_cast<size_t>(n));
        std::iota(id.begin(), id.end(), Index(0));
        std::stable_sort(id.begin(), id.end(), [&](Index a, Index b) { return values[a] > values[b]; });
        id.resize(std::min<size_t>(id.size(), static_cast<size_t>(k)));
        *n_out = static_cast<int64_t>(id.size());
        for (size_t i = 0; i < id.size(); ++i) idx[i] = id[i];
    });
}

int32_t oracle_relevance_all(const float* q, int64_t l_x, int32_t H, int32_t Hkv, int32_t d, const float* repr,
                             int64_t U, int64_t r_k, double* rel) {
    return guard([&] {
        TieredStore st;
        st.H = H;
        st.rep = H / Hkv;
        st.repr_index.resize(static_cast<size_t>(Hkv));
        for (int64_t u = 0; u < U; ++u) {
            MemoryUnit mu;
            mu.unit_id = u;
            for (int g = 0; g < Hkv; ++g) {
                Mat<Scalar> rk(r_k, d);
                for (int64_t r = 0; r < r_k; ++r)
                    std::memcpy(rk.row(r), repr + ((u * r_k + r) * Hkv + g) * d, sizeof(float) * static_cast<size_t>(d));
                mu.repr_keys.push_back(std::move(rk));
                mu.keys.emplace_back(0, d);
            }
            st.add_unit(std::move(mu));
        }
        std::vector<Mat<Scalar>> bq(static_cast<size_t>(H));
        for (int h = 0; h < H; ++h) {
            bq[static_cast<size_t>(h)] = Mat<Scalar>(l_x, d);
            for (int64_t i = 0; i < l_x; ++i)
                std::memcpy(bq[static_cast<size_t>(h)].row(i), q + (i * H + h) * d, sizeof(float) * static_cast<size_t>(d));
        }
        const auto r = st.relevance_all(bq);
        for (int64_t u = 0; u < U; ++u) rel[u] = r[static_cast<size_t>(u)];
    });
}

double oracle_relevance_unit(const float* q, int64_t l_x, int32_t H, int32_t Hkv, int32_t d, const float* rk,
                             int64_t n_repr) {
    // relevance (memory.hpp:141-149): sum over heads of (q_h * repr_h^T).sum()
    if (n_repr < 1) {
        g_err = "relevance: unit has no representatives";
        return std::nan("");
    }
    const int rep = H / Hkv;
    double total = 0.0;
    for (int h = 0; h < H; ++h) {
        const int g = h / rep;
        double s = 0.0;
        for (int64_t i = 0; i < l_x; ++i)
            for (int64_t r = 0; r < n_repr; ++r) {
                double acc = 0.0;
                for (int c = 0; c < d; ++c)
                    acc += static_cast<double>(q[(i * H + h) * d + c]) * static_cast<double>(rk[(r * Hkv + g) * d + c]);
                s += acc;
            }
        total += s;
    }
    return total;
}

double oracle_mean_repr_relevance(const double* uk, int64_t n, const double* q, int64_t l_x, int32_t H,
                                  int32_t Hkv, int32_t d) {
    // oracle.hpp:199-207 (per expanded head: mean of the unit's keys)
    const int rep = H / Hkv;
    double total = 0.0;
    std::vector<double> mean(static_cast<size_t>(d));
    for (int h = 0; h < H; ++h) {
        const int g = h / rep;
        std::fill(mean.begin(), mean.end(), 0.0);
        for (int64_t j = 0; j < n; ++j)
            for (int c = 0; c < d; ++c) mean[static_cast<size_t>(c)] += uk[(j * Hkv + g) * d + c];
        for (auto& m : mean) m /= static_cast<double>(n);
        for (int64_t i = 0; i < l_x; ++i) {
            double acc = 0.0;
            for (int c = 0; c < d; ++c) acc += q[(i * H + h) * d + c] * mean[static_cast<size_t>(c)];
            total += acc;
        }
    }
    return total;
}

}  // extern "C"

// ------------------------------------------------------------ oracle.hpp:64-184
namespace {

// detail::rotate (oracle.hpp:129-143), double
void rotate_d(const double* x, int d, Index pos, double* out) {
    for (int c = 0; c < d; ++c) out[c] = x[c];
    const int pairs = d / 2;
    for (int a = 0; a < pairs; ++a) {
        const double angle = static_cast<double>(pos) * std::pow(10000.0, -2.0 * a / static_cast<double>(d));
        const double c = std::cos(angle), s = std::sin(angle);
        const double x0 = x[2 * a], x1 = x[2 * a + 1];
        out[2 * a] = x0 * c - x1 * s;
        out[2 * a + 1] = x0 * s + x1 * c;
    }
}

void softmax_inplace(std::vector<double>& logits) {  // oracle.hpp:145-154
    double m = logits.front();
    for (double v : logits) m = std::max(m, v);
    double sum = 0.0;
    for (double& v : logits) {
        v = std::exp(v - m);
        sum += v;
    }
    for (double& v : logits) v /= sum;
}

double dotd(const double* a, const double* b, int d) {
    double s = 0.0;
    for (int c = 0; c < d; ++c) s += a[c] * b[c];
    return s;
}

}  // namespace

extern "C" {

int32_t oracle_dense_attention(const double* q, const double* k, const double* v, int64_t n, int32_t H,
                               int32_t Hkv, int32_t d, int32_t dv, int32_t position_mode, int64_t local_size,
                               double* out) {
    return guard([&] {  // oracle.hpp:64-97
        const int rep = H / Hkv;
        const double scale = 1.0 / std::sqrt(static_cast<double>(d));
        const bool clamped = position_mode == INFLLM_POSITION_CLAMPED;
        // pre-rotate keys by their positions
        std::vector<double> krot(static_cast<size_t>(n * Hkv * d));
        for (int64_t j = 0; j < n; ++j)
            for (int g = 0; g < Hkv; ++g) rotate_d(k + (j * Hkv + g) * d, d, j, krot.data() + (j * Hkv + g) * d);
        std::vector<double> qa(static_cast<size_t>(d)), qc(static_cast<size_t>(d)), acc(static_cast<size_t>(dv));
        for (int h = 0; h < H; ++h) {
            const int g = h / rep;
            for (int64_t i = 0; i < n; ++i) {
                rotate_d(q + (i * H + h) * d, d, i, qa.data());
                if (clamped) rotate_d(q + (i * H + h) * d, d, local_size, qc.data());
                std::vector<double> logits(static_cast<size_t>(i + 1));
                for (int64_t j = 0; j <= i; ++j) {
                    const bool cap = clamped && i - j > local_size;
                    const double s = cap ? dotd(qc.data(), k + (j * Hkv + g) * d, d)
                                         : dotd(qa.data(), krot.data() + (j * Hkv + g) * d, d);
                    logits[static_cast<size_t>(j)] = s * scale;
                }
                softmax_inplace(logits);
                std::fill(acc.begin(), acc.end(), 0.0);
                for (int64_t j = 0; j <= i; ++j)
                    for (int c = 0; c < dv; ++c) acc[static_cast<size_t>(c)] += logits[static_cast<size_t>(j)] * v[(j * Hkv + g) * dv + c];
                for (int c = 0; c < dv; ++c) out[(i * H + h) * dv + c] = acc[static_cast<size_t>(c)];
            }
        }
    });
}

int32_t oracle_windowed_attention(const double* q, const double* k, const double* v, int64_t n, int32_t H,
                                  int32_t Hkv, int32_t d, int32_t dv, const int64_t* schedule, int64_t n_sched,
                                  int64_t init_size, int64_t local_size, int64_t unit_size, int32_t position_mode,
                                  double* out) {
    return guard([&] {  // oracle.hpp:103-168
        const int rep = H / Hkv;
        const double scale = 1.0 / std::sqrt(static_cast<double>(d));
        const bool clamped = position_mode == INFLLM_POSITION_CLAMPED;
        std::vector<double> krot(static_cast<size_t>(n * Hkv * d));
        for (int64_t j = 0; j < n; ++j)
            for (int g = 0; g < Hkv; ++g) rotate_d(k + (j * Hkv + g) * d, d, j, krot.data() + (j * Hkv + g) * d);
        std::vector<double> qa(static_cast<size_t>(d)), qc(static_cast<size_t>(d)), acc(static_cast<size_t>(dv));
        Index fed = 0;
        for (int64_t si = 0; si < n_sched; ++si) {
            const Index batch = schedule[si];
            const Index local_begin = std::max<Index>(0, fed - local_size);
            const Index init_len = std::min(init_size, local_begin);
            const Index evicted = std::max<Index>(0, local_begin - init_size);
            const Index packed = evicted - evicted % unit_size;
            std::vector<Index> visible;
            for (Index j = 0; j < init_len; ++j) visible.push_back(j);
            for (Index j = init_size; j < init_size + packed; ++j) visible.push_back(j);
            for (Index j = local_begin; j < fed; ++j) visible.push_back(j);
            for (int h = 0; h < H; ++h) {
                const int g = h / rep;
                for (Index bi = 0; bi < batch; ++bi) {
                    const Index i = fed + bi;
                    rotate_d(q + (i * H + h) * d, d, i, qa.data());
                    rotate_d(q + (i * H + h) * d, d, local_size, qc.data());
                    std::vector<double> logits;
                    std::vector<Index> cols;
                    auto score = [&](Index j, bool far) {
                        if (clamped && (far || i - j > local_size)) return dotd(qc.data(), k + (j * Hkv + g) * d, d);
                        return dotd(qa.data(), krot.data() + (j * Hkv + g) * d, d);
                    };
                    for (Index j : visible) {
                        logits.push_back(score(j, j < local_begin) * scale);
                        cols.push_back(j);
                    }
                    for (Index j = fed; j <= i; ++j) {
                        logits.push_back(score(j, false) * scale);
                        cols.push_back(j);
                    }
                    softmax_inplace(logits);
                    std::fill(acc.begin(), acc.end(), 0.0);
                    for (size_t t = 0; t < cols.size(); ++t)
                        for (int c = 0; c < dv; ++c) acc[static_cast<size_t>(c)] += logits[t] * v[(cols[t] * Hkv + g) * dv + c];
                    for (int c = 0; c < dv; ++c) out[(i * H + h) * dv + c] = acc[static_cast<size_t>(c)];
                }
            }
            fed += batch;
        }
    });
}

int32_t oracle_batch_repr_scores(const double* q, const double* k, int64_t n, int32_t H, int32_t Hkv, int32_t d,
                                 int64_t local_size, double* out) {
    return guard([&] {  // oracle.hpp:173-184
        const int rep = H / Hkv;
        for (int64_t m = 0; m < n; ++m) {
            double sum = 0.0;
            for (int64_t j = 1; j <= local_size && m + j < n; ++j)
                for (int h = 0; h < H; ++h)
                    sum += dotd(q + ((m + j) * H + h) * d, k + (m * Hkv + h / rep) * d, d);
            out[m] = sum / static_cast<double>(local_size);
        }
    });
}

int32_t oracle_noise_ids(uint64_t seed, int64_t n, int64_t* ids) {
    Rng rng(hash_mix(seed, 0x6e6f697365ULL));  // cli.cpp:30-36
    for (int64_t i = 0; i < n; ++i) ids[i] = static_cast<int64_t>(rng.next_below(1 << 20));
    return INFLLM_OK;
}

int32_t oracle_adapter_batch(uint64_t seed, int32_t n_layers, int32_t n_heads, int32_t head_dim, int32_t value_dim,
                             int32_t layer, const int64_t* ids, int64_t n, float* q, float* k, float* v) {
    return guard([&] {  // adapter.hpp:24-69, 76-89
        if (layer < 0 || layer >= n_layers) throw StreamError("adapter: layer out of range");
        if (n < 1) throw StreamError("adapter: token batch must be non-empty");
        constexpr int E = 256;
        constexpr std::uint64_t kEmbedTag = 0x6d62656b6f74ULL;
        const int dv = value_dim > 0 ? value_dim : head_dim;
        auto mix_tag = [&](int l, int h, std::uint64_t role) {
            std::uint64_t x = hash_mix(seed, role);
            x = hash_mix(x, static_cast<std::uint64_t>(l) + 1);
            return hash_mix(x, static_cast<std::uint64_t>(h) + 1);
        };
        auto random_matrix = [&](int rows, std::uint64_t s) {
            Rng rng(s);
            std::vector<float> m(static_cast<size_t>(rows * E));
            for (auto& x : m) x = static_cast<float>(rng.next_gaussian());
            return m;
        };
        std::vector<float> emb(static_cast<size_t>(n * E));
        for (int64_t i = 0; i < n; ++i) {
            Rng rng(hash_mix(seed ^ kEmbedTag, static_cast<std::uint64_t>(ids[i])));
            for (int c = 0; c < E; ++c) emb[static_cast<size_t>(i * E + c)] = static_cast<float>(rng.next_gaussian());
        }
        const float norm = 1.0f / std::sqrt(static_cast<float>(E));
        for (int h = 0; h < n_heads; ++h) {
            // projections depend only on (layer, head); regenerate like the ctor does
            const auto kp = random_matrix(head_dim, mix_tag(layer, h, 1));
            const auto vp = random_matrix(dv, mix_tag(layer, h, 2));
            std::vector<float> kk(static_cast<size_t>(n * head_dim)), vv(static_cast<size_t>(n * dv));
            gemm_nt<float>(emb.data(), n, E, kp.data(), head_dim, kk.data());
            gemm_nt<float>(emb.data(), n, E, vp.data(), dv, vv.data());
            for (int64_t i = 0; i < n; ++i) {
                for (int c = 0; c < head_dim; ++c) {
                    const float x = kk[static_cast<size_t>(i * head_dim + c)] * norm;
                    q[(i * n_heads + h) * head_dim + c] = x;
                    k[(i * n_heads + h) * head_dim + c] = x;
                }
                for (int c = 0; c < dv; ++c) v[(i * n_heads + h) * dv + c] = vv[static_cast<size_t>(i * dv + c)] * norm;
            }
        }
    });
}

int32_t oracle_gaussian_fill(uint64_t seed, uint64_t tensor, int64_t tok0, int64_t n_tok, int32_t n_head,
                             int32_t dim, float* x) {
    for (int64_t t = 0; t < n_tok; ++t)
        for (int h = 0; h < n_head; ++h) {
            const std::uint64_t base =
                hash_mix(hash_mix(hash_mix(seed, tensor), static_cast<std::uint64_t>(tok0 + t)), static_cast<std::uint64_t>(h));
            Rng rng(base);
            for (int c = 0; c < dim; ++c) x[(t * n_head + h) * dim + c] = static_cast<float>(rng.next_gaussian());
        }
    return INFLLM_OK;
}

int32_t oracle_gen_planted(uint64_t seed, int64_t length, int64_t plant_len, const infllm_engine_config* cfg,
                           int64_t probe_len, int32_t align_to_units, int64_t* plant_start, int64_t* plant_id,
                           int64_t* first_unit, int64_t* last_unit, int64_t* ids) {
    return guard([&] {  // workload.hpp:35-76
        if (plant_len < 1 || probe_len < 1) throw ConfigError("gen_planted: plant_len and probe_len must be >= 1");
        const Index probe_pos = length - probe_len;
        const Index a_max = probe_pos - cfg->local_size - cfg->unit_size - plant_len;
        const Index a_min = cfg->init_size;
        if (a_max < a_min) throw ConfigError("gen_planted: length too small for init + local + unit margin");
        Rng rng(hash_mix(seed, 0x706c616e74ULL));
        Index a = a_min + static_cast<Index>(rng.next_below(static_cast<std::uint64_t>(a_max - a_min + 1)));
        if (align_to_units) a = cfg->init_size + ((a - cfg->init_size) / cfg->unit_size) * cfg->unit_size;
        *plant_start = a;
        *plant_id = (1 << 20) + static_cast<int64_t>(rng.next_below(1 << 20));
        for (int64_t i = 0; i < length; ++i) ids[i] = static_cast<int64_t>(rng.next_below(1 << 20));
        for (Index i = 0; i < plant_len; ++i) ids[a + i] = *plant_id;
        for (Index i = 0; i < probe_len; ++i) ids[probe_pos + i] = *plant_id;
        *first_unit = (a - cfg->init_size) / cfg->unit_size;
        *last_unit = (a + plant_len - 1 - cfg->init_size) / cfg->unit_size;
    });
}


// ---- stand-alone operators (the C-ABI's infllm_attend / infllm_store_* / infllm_score_acc_*) ----

struct oracle_store {
    TieredStore s;
    int Hkv = 1, d = 0;
};

oracle_store* oracle_store_create(int64_t hot_capacity, double decay, int32_t H, int32_t Hkv, int32_t d,
                                  int64_t bytes_per_token) {
    auto* x = new oracle_store();
    x->s.hot_capacity = hot_capacity;  // TieredStore(hot_capacity, decay, n_heads) (memory.hpp:172-175)
    x->s.decay = decay;
    x->s.H = H;
    x->s.rep = H / Hkv;
    x->s.repr_index.resize(static_cast<size_t>(Hkv));
    x->s.unit_bytes_per_token = static_cast<std::size_t>(bytes_per_token);
    x->Hkv = Hkv;
    x->d = d;
    return x;
}
void oracle_store_destroy(oracle_store* x) { delete x; }

// add_unit (memory.hpp:196-212); repr_keys [n][Hkv][d]
int32_t oracle_store_add_unit(oracle_store* x, const float* repr_keys, int64_t n, int64_t unit_tokens, int64_t* id) {
    return guard([&] {
        MemoryUnit u;
        u.unit_id = x->s.total_units();
        for (int g = 0; g < x->Hkv; ++g) {
            u.keys.emplace_back(unit_tokens, 0);  // only the size matters here (hot_bytes)
            Mat<Scalar> rk(n, x->d);
            for (Index r = 0; r < n; ++r)
                std::memcpy(rk.row(r), repr_keys + (r * x->Hkv + g) * x->d, sizeof(Scalar) * static_cast<size_t>(x->d));
            u.repr_keys.push_back(std::move(rk));
        }
        if (id) *id = u.unit_id;
        x->s.add_unit(std::move(u));
    });
}
int32_t oracle_store_begin_step(oracle_store* x, int64_t step) {
    x->s.step = step;
    return 0;
}
// lookup (memory.hpp:239-269); q [l_x][H][d]
int32_t oracle_store_lookup(oracle_store* x, const float* q, int64_t l_x, int64_t k_m, int64_t* ids, int64_t* n) {
    return guard([&] {
        std::vector<Mat<Scalar>> qh;
        for (int h = 0; h < x->s.H; ++h) {
            Mat<Scalar> m(l_x, x->d);
            for (Index i = 0; i < l_x; ++i)
                std::memcpy(m.row(i), q + (i * x->s.H + h) * x->d, sizeof(Scalar) * static_cast<size_t>(x->d));
            qh.push_back(std::move(m));
        }
        const auto r = x->s.lookup(qh, k_m);
        for (size_t i = 0; i < r.size(); ++i) ids[i] = r[i];
        *n = static_cast<int64_t>(r.size());
    });
}
int32_t oracle_store_update_frequency(oracle_store* x, const int64_t* ids, const double* mass, int64_t n) {
    return guard([&] {
        std::vector<std::pair<std::int64_t, double>> m;
        for (int64_t i = 0; i < n; ++i) m.emplace_back(ids[i], mass[i]);
        x->s.update_frequency(m);
    });
}
int32_t oracle_store_enforce_capacity(oracle_store* x) {
    return guard([&] { x->s.enforce_capacity(); });
}
int32_t oracle_store_note_step_boundary(oracle_store* x) {
    return guard([&] { x->s.note_step_boundary(); });
}
int32_t oracle_store_counters(oracle_store* x, infllm_layer_metrics* m) {
    *m = x->s.counters;
    m->units = x->s.total_units();
    m->hot_units = static_cast<int64_t>(x->s.hot.size());
    m->peak_hot_units = x->s.peak_hot_units;
    m->peak_hot_bytes = static_cast<int64_t>(x->s.peak_hot_bytes);
    return 0;
}
int32_t oracle_store_trace(oracle_store* x, int64_t* step, int64_t* unit, int32_t* hit, int64_t cap, int64_t* n_out) {
    const auto& t = x->s.trace;
    *n_out = static_cast<int64_t>(t.size());
    for (int64_t i = 0; i < std::min<int64_t>(cap, static_cast<int64_t>(t.size())); ++i) {
        step[i] = t[static_cast<size_t>(i)].step;
        unit[i] = t[static_cast<size_t>(i)].unit_id;
        hit[i] = t[static_cast<size_t>(i)].hit ? 1 : 0;
    }
    return 0;
}
int32_t oracle_store_unit_freq(oracle_store* x, double* freq, int32_t* hot, int64_t n) {
    for (int64_t i = 0; i < std::min<int64_t>(n, x->s.total_units()); ++i) {
        freq[i] = x->s.units[static_cast<size_t>(i)].freq_score;
        hot[i] = x->s.units[static_cast<size_t>(i)].hot ? 1 : 0;
    }
    return 0;
}

struct oracle_score_acc {
    ScoreAccumulator a;
    int H = 1, Hkv = 1, d = 0;
};
oracle_score_acc* oracle_score_acc_create(int64_t local_size, int32_t H, int32_t Hkv, int32_t d) {
    auto* x = new oracle_score_acc{ScoreAccumulator{local_size, 0, 0, 0, {}, 1}, H, Hkv, d};
    return x;
}
void oracle_score_acc_destroy(oracle_score_acc* x) { delete x; }
// accumulate (repr_score.hpp:39-69): q [l_x][H][d], keys [n_pending][Hkv][d]
int32_t oracle_score_acc_accumulate(oracle_score_acc* x, const float* q, int64_t l_x, int64_t s, const float* keys,
                                    int64_t n_pending) {
    return guard([&] {
        std::vector<Mat<Scalar>> qh, kh;
        for (int h = 0; h < x->H; ++h) {
            Mat<Scalar> m(l_x, x->d);
            for (Index i = 0; i < l_x; ++i)
                std::memcpy(m.row(i), q + (i * x->H + h) * x->d, sizeof(Scalar) * static_cast<size_t>(x->d));
            qh.push_back(std::move(m));
        }
        for (int g = 0; g < x->Hkv; ++g) {
            Mat<Scalar> m(n_pending, x->d);
            for (Index i = 0; i < n_pending; ++i)
                std::memcpy(m.row(i), keys + (i * x->Hkv + g) * x->d, sizeof(Scalar) * static_cast<size_t>(x->d));
            kh.push_back(std::move(m));
        }
        x->a.accumulate(s, qh, kh, x->H / x->Hkv);
    });
}
int32_t oracle_score_acc_finalize_front(oracle_score_acc* x, int64_t n, float* out) {
    return guard([&] {
        const auto r = x->a.finalize_front(n);
        for (size_t i = 0; i < r.size(); ++i) out[i] = r[i];
    });
}

// attend (attention.hpp:116-230) over explicit segments; token-major host tensors
int32_t oracle_attend(int32_t H, int32_t Hkv, int32_t d, int32_t dv, int32_t position_mode, int64_t local_size,
                      const int32_t* seg_kind, const int64_t* seg_start, const int64_t* seg_n,
                      const float* const* seg_keys, const float* const* seg_values, int32_t n_seg, const float* q,
                      const float* k, const float* v, int64_t l_x, int64_t start_abs, float* out, double* seg_mass,
                      float* weights) {
    return guard([&] {
        oracle_engine e;
        e.cfg.local_size = local_size;
        e.cfg.position_mode = position_mode;
        e.H = H;
        e.Hkv = Hkv;
        e.rep = H / Hkv;
        e.d = d;
        e.dv = dv;
        auto per_group = [&](const float* src, Index n, int cols) {
            std::vector<Mat<Scalar>> m;
            for (int g = 0; g < Hkv; ++g) {
                Mat<Scalar> x(n, cols);
                for (Index i = 0; i < n; ++i)
                    std::memcpy(x.row(i), src + (i * Hkv + g) * cols, sizeof(Scalar) * static_cast<size_t>(cols));
                m.push_back(std::move(x));
            }
            return m;
        };
        std::vector<std::vector<Mat<Scalar>>> sk, sv;
        for (int s2 = 0; s2 < n_seg; ++s2) {
            sk.push_back(per_group(seg_keys[s2], seg_n[s2], d));
            sv.push_back(per_group(seg_values[s2], seg_n[s2], dv));
        }
        std::vector<SegmentView> segs;
        Index n_ctx = 0;
        for (int s2 = 0; s2 < n_seg; ++s2) {
            SegmentView sg;
            sg.kind = seg_kind[s2] == INFLLM_SEG_INITIAL ? Seg::initial
                      : seg_kind[s2] == INFLLM_SEG_RETRIEVED ? Seg::retrieved
                                                              : Seg::local;
            sg.start_abs = seg_start[s2];
            sg.unit_id = -1;
            for (int g = 0; g < Hkv; ++g) {
                sg.keys.push_back(&sk[static_cast<size_t>(s2)][static_cast<size_t>(g)]);
                sg.values.push_back(&sv[static_cast<size_t>(s2)][static_cast<size_t>(g)]);
            }
            n_ctx += seg_n[s2];
            segs.push_back(std::move(sg));
        }
        const auto bk = per_group(k, l_x, d), bv = per_group(v, l_x, dv);
        const Index n_all = n_ctx + l_x;
        std::vector<double> mass(static_cast<size_t>(n_seg), 0.0);
        for (int h = 0; h < H; ++h) {
            Mat<Scalar> qh(l_x, d), oh, wh;
            for (Index i = 0; i < l_x; ++i)
                std::memcpy(qh.row(i), q + (i * H + h) * d, sizeof(Scalar) * static_cast<size_t>(d));
            e.attend_head(h, qh, start_abs, segs, bk[static_cast<size_t>(h / e.rep)], bv[static_cast<size_t>(h / e.rep)],
                          oh, &wh);
            for (Index i = 0; i < l_x; ++i)
                for (int c = 0; c < dv; ++c) out[(i * H + h) * dv + c] = oh(i, c);
            if (weights)
                for (Index i = 0; i < l_x; ++i)
                    std::memcpy(weights + (static_cast<int64_t>(h) * l_x + i) * n_all, wh.row(i),
                                sizeof(Scalar) * static_cast<size_t>(n_all));
            Index col = 0;  // engine.hpp:271-283
            for (int s2 = 0; s2 < n_seg; ++s2) {
                double m = 0.0;
                for (Index i = 0; i < l_x; ++i)
                    for (Index j = 0; j < seg_n[s2]; ++j) m += static_cast<double>(wh(i, col + j));
                mass[static_cast<size_t>(s2)] += m;
                col += seg_n[s2];
            }
        }
        if (seg_mass)
            for (int s2 = 0; s2 < n_seg; ++s2) seg_mass[s2] = mass[static_cast<size_t>(s2)] / H;
    });
}

}  // extern "C"
