// TEST INFRASTRUCTURE ONLY — flat C entry points over the reference engine,
// compiled from the reference headers where they lie (/root/reference/proj/
// include, see oracle/Makefile) against oracle/eigen_shim. Two builds:
//   REF_INJECT=1: q/k/v injected through the shadow adapter (ref_inject/);
//   REF_INJECT=0: the reference's own SyntheticAdapter (C0 inputs from ids).
// Nothing here re-implements the reference: it only marshals arguments, like
// cli.cpp's run_engine_collect (cli.cpp:89-119).

#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <vector>

#include "blockmem/engine.hpp"
#include "blockmem/oracle.hpp"
#include "blockmem/repr_score.hpp"
#include "blockmem/workload.hpp"

using namespace blockmem;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const StreamError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

struct RefCfg {  // same layout as infllm_engine_config
    int64_t chunk_size, unit_size, n_repr, local_size, init_size, n_lookup, hot_capacity;
    double decay;
    int32_t lookup_mode, position_mode;
};

EngineConfig to_cfg(const RefCfg* c) {
    EngineConfig e;
    e.chunk_size = c->chunk_size;
    e.unit_size = c->unit_size;
    e.n_repr = c->n_repr;
    e.local_size = c->local_size;
    e.init_size = c->init_size;
    e.n_lookup = c->n_lookup;
    e.hot_capacity = c->hot_capacity;
    e.decay = c->decay;
    e.lookup_mode = c->lookup_mode == 0 ? LookupMode::encode_and_decode
                                        : (c->lookup_mode == 1 ? LookupMode::decode_only : LookupMode::none);
    e.position_mode = c->position_mode == 0 ? PositionMode::clamped : PositionMode::absolute;
    return e;
}

oracle::SequenceData seq_from(const double* q, const double* k, const double* v, int64_t n, int H, int d, int dv) {
    oracle::SequenceData s;
    for (int h = 0; h < H; ++h) {
        Mat<double> mq(n, d), mk(n, d), mv(n, dv);
        for (int64_t i = 0; i < n; ++i) {
            for (int c = 0; c < d; ++c) {
                mq(i, c) = q[(i * H + h) * d + c];
                mk(i, c) = k[(i * H + h) * d + c];
            }
            for (int c = 0; c < dv; ++c) mv(i, c) = v[(i * H + h) * dv + c];
        }
        s.q.push_back(std::move(mq));
        s.k.push_back(std::move(mk));
        s.v.push_back(std::move(mv));
    }
    return s;
}

void to_token_major(const std::vector<Mat<double>>& per_head, int64_t n, int H, int dv, double* out) {
    for (int h = 0; h < H; ++h)
        for (int64_t i = 0; i < n; ++i)
            for (int c = 0; c < dv; ++c) out[(i * H + h) * dv + c] = per_head[static_cast<size_t>(h)](i, c);
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_injected() { return REF_INJECT; }

#if REF_INJECT
int ref_set_inputs(int layer, const float* q, const float* k, const float* v, int64_t n, int H, int d, int dv) {
    return guard([&] {
        auto& t = inject::tables();
        if (static_cast<int>(t.size()) <= layer) t.resize(static_cast<size_t>(layer) + 1);
        auto& x = t[static_cast<size_t>(layer)];
        x.n = n;
        x.H = H;
        x.d = d;
        x.dv = dv;
        x.q.assign(q, q + n * H * d);
        x.k.assign(k, k + n * H * d);
        x.v.assign(v, v + n * H * dv);
    });
}
#endif

void* ref_engine_create(const RefCfg* c, int n_layers, int H, int d, int dv, uint64_t seed) {
    StreamEngine<float>* e = nullptr;
    if (guard([&] { e = new StreamEngine<float>(to_cfg(c), ModelShape::make(n_layers, H, d, dv), seed); }) != 0)
        return nullptr;
    return e;
}

void ref_engine_destroy(void* e) { delete static_cast<StreamEngine<float>*>(e); }

void ref_set_always_emit_weights(void* e, int v) { static_cast<StreamEngine<float>*>(e)->set_always_emit_weights(v != 0); }

// One engine step (encode_chunk or decode_step) over token ids (ignored by
// the injecting adapter). out: [n_layers][l_x][H][dv]; ids: [n_layers][ids_cap].
int ref_step(void* ep, const int64_t* ids, int64_t l_x, int is_decode, float* out, int64_t* ids_out,
             int64_t ids_cap, int64_t* n_ids) {
    return guard([&] {
        auto* e = static_cast<StreamEngine<float>*>(ep);
        std::vector<std::int64_t> tok(static_cast<size_t>(l_x), 0);
        if (ids) tok.assign(ids, ids + l_x);
        StepOutput<float> so = is_decode ? e->decode_step(tok.front()) : e->encode_chunk(std::span<const std::int64_t>(tok));
        const int H = e->shape().n_heads, dv = e->shape().value_dim;
        for (size_t l = 0; l < so.size(); ++l) {
            for (int h = 0; h < H; ++h)
                for (int64_t i = 0; i < l_x; ++i)
                    for (int c = 0; c < dv; ++c)
                        out[((static_cast<int64_t>(l) * l_x + i) * H + h) * dv + c] = so[l].attn.out[static_cast<size_t>(h)](i, c);
            const auto& r = so[l].retrieved_ids;
            n_ids[l] = static_cast<int64_t>(r.size());
            for (size_t j = 0; j < r.size() && static_cast<int64_t>(j) < ids_cap; ++j) ids_out[static_cast<int64_t>(l) * ids_cap + static_cast<int64_t>(j)] = r[j];
        }
    });
}

int ref_finish(void* e) { return guard([&] { static_cast<StreamEngine<float>*>(e)->finish(); }); }

// [units, hot_units, peak_hot_units, peak_hot_bytes, hits, misses, loads, evictions, requested]
int ref_metrics(void* ep, int layer, int64_t* m9) {
    return guard([&] {
        const auto m = static_cast<StreamEngine<float>*>(ep)->metrics();
        const auto& l = m.layers.at(static_cast<size_t>(layer));
        const int64_t v[9] = {l.units, l.hot_units, l.peak_hot_units, static_cast<int64_t>(l.peak_hot_bytes),
                              static_cast<int64_t>(l.cache.hits), static_cast<int64_t>(l.cache.misses),
                              static_cast<int64_t>(l.cache.loads), static_cast<int64_t>(l.cache.evictions),
                              static_cast<int64_t>(l.cache.requested)};
        std::memcpy(m9, v, sizeof(v));
    });
}

int ref_invariants(void* ep, uint64_t* checks, uint64_t* violations) {
    auto* e = static_cast<StreamEngine<float>*>(ep);
    *checks = e->invariant_checks();
    *violations = e->invariant_violations();
    return 0;
}

int ref_stream_state(void* ep, int layer, int64_t* s5) {
    return guard([&] {
        auto* e = static_cast<StreamEngine<float>*>(ep);
        s5[0] = e->tokens_fed();
        s5[1] = e->steps_done();
        s5[2] = e->initial_len(layer);
        s5[3] = e->local_len(layer);
        s5[4] = e->pending_partial(layer);
    });
}

int ref_unit_info(void* ep, int layer, int64_t id, int64_t* start_abs, int64_t* size, int64_t* repr_abs,
                  int64_t* n_repr, double* freq, int* hot) {
    return guard([&] {
        const auto& st = static_cast<StreamEngine<float>*>(ep)->store(layer);
        if (id < 0 || id >= st.total_units()) throw StreamError("unit id out of range");
        const auto& u = st.unit(id);
        *start_abs = u.start_abs;
        *size = u.size();
        *n_repr = static_cast<int64_t>(u.repr_abs.size());
        for (size_t r = 0; r < u.repr_abs.size(); ++r) repr_abs[r] = u.repr_abs[r];
        *freq = u.freq_score;
        *hot = u.tier == Tier::hot ? 1 : 0;
    });
}

int ref_trace(void* ep, int layer, int64_t* step, int64_t* unit, int* hit, int64_t cap, int64_t* n_out) {
    return guard([&] {
        const auto& tr = static_cast<StreamEngine<float>*>(ep)->store(layer).trace();
        *n_out = static_cast<int64_t>(tr.size());
        for (size_t i = 0; i < tr.size() && static_cast<int64_t>(i) < cap; ++i) {
            step[i] = tr[i].step;
            unit[i] = tr[i].unit_id;
            hit[i] = tr[i].hit ? 1 : 0;
        }
    });
}

int ref_select_representatives(const float* scores, int64_t n, int64_t r_k, int64_t* idx, int64_t* n_out) {
    return guard([&] {
        const auto r = select_representatives<float>(std::span<const float>(scores, static_cast<size_t>(n)), r_k);
        *n_out = static_cast<int64_t>(r.size());
        for (size_t i = 0; i < r.size(); ++i) idx[i] = r[i];
    });
}

int ref_argsort_topk(const double* v, int64_t n, int64_t k, int64_t* idx, int64_t* n_out) {
    return guard([&] {
        const auto r = oracle::argsort_topk(std::vector<double>(v, v + n), k);
        *n_out = static_cast<int64_t>(r.size());
        for (size_t i = 0; i < r.size(); ++i) idx[i] = r[i];
    });
}

int ref_dense_attention(const double* q, const double* k, const double* v, int64_t n, int H, int d, int dv,
                        int position_mode, int64_t local_size, double* out) {
    return guard([&] {
        const auto s = seq_from(q, k, v, n, H, d, dv);
        to_token_major(oracle::dense_attention(s, position_mode == 0 ? PositionMode::clamped : PositionMode::absolute,
                                               local_size),
                       n, H, dv, out);
    });
}

int ref_windowed_attention(const double* q, const double* k, const double* v, int64_t n, int H, int d, int dv,
                           const int64_t* sched, int64_t n_sched, int64_t init_size, int64_t local_size,
                           int64_t unit_size, int position_mode, double* out) {
    return guard([&] {
        const auto s = seq_from(q, k, v, n, H, d, dv);
        std::vector<Index> schedule(sched, sched + n_sched);
        to_token_major(oracle::windowed_attention_reference(
                           s, schedule, init_size, local_size, unit_size,
                           position_mode == 0 ? PositionMode::clamped : PositionMode::absolute),
                       n, H, dv, out);
    });
}

int ref_batch_repr_scores(const double* q, const double* k, int64_t n, int H, int d, int64_t local_size, double* out) {
    return guard([&] {
        std::vector<double> zero(static_cast<size_t>(n * H * d), 0.0);
        const auto s = seq_from(q, k, zero.data(), n, H, d, d);
        const auto r = oracle::batch_repr_scores(s, local_size);
        for (int64_t i = 0; i < n; ++i) out[i] = r[static_cast<size_t>(i)];
    });
}

// ScoreAccumulator driven chunk by chunk over one head set (cli.cpp:302-327):
// returns finalize_front(n) of the whole stream.
int ref_accumulator_scores(const float* q, const float* k, int64_t n, int H, int d, int64_t local_size,
                           int64_t chunk, float* out) {
    return guard([&] {
        ScoreAccumulator<float> acc(local_size);
        std::vector<Mat<float>> seen(static_cast<size_t>(H));
        for (auto& m : seen) m.resize(0, d);
        int64_t fed = 0;
        while (fed < n) {
            const int64_t b = std::min(chunk, n - fed);
            TokenBatch<float> batch;
            batch.start_abs = fed;
            for (int h = 0; h < H; ++h) {
                Mat<float> mq(b, d), mk(b, d);
                for (int64_t i = 0; i < b; ++i)
                    for (int c = 0; c < d; ++c) {
                        mq(i, c) = q[((fed + i) * H + h) * d + c];
                        mk(i, c) = k[((fed + i) * H + h) * d + c];
                    }
                batch.q.push_back(mq);
                batch.k.push_back(mk);
                batch.v.push_back(mk);
                auto& m = seen[static_cast<size_t>(h)];
                const Index old = m.rows();
                m.conservativeResize(old + b, d);
                m.bottomRows(b) = mk;
            }
            std::vector<Eigen::Ref<const Mat<float>>> pending;
            for (auto& m : seen) pending.emplace_back(m);
            acc.accumulate(batch, pending);
            fed += b;
        }
        const auto got = acc.finalize_front(n);
        for (int64_t i = 0; i < n; ++i) out[i] = got[static_cast<size_t>(i)];
    });
}

// TieredStore relevance through the reference's own store: builds units with
// the given representative keys ([U][r_k][H][d]) and returns relevance_all for
// the batch q [l_x][H][d], plus lookup(k_m) ids.
int ref_store_lookup(const float* q, int64_t l_x, int H, int d, const float* repr, int64_t U, int64_t r_k,
                     int64_t k_m, double* rel, int64_t* ids, int64_t* n_ids) {
    return guard([&] {
        TieredStore<float> st(std::max<int64_t>(k_m, 1), 0.1, H);
        for (int64_t u = 0; u < U; ++u) {
            MemoryUnit<float> mu;
            mu.unit_id = u;
            mu.start_abs = u * r_k;
            for (int h = 0; h < H; ++h) {
                Mat<float> rk(r_k, d);
                for (int64_t r = 0; r < r_k; ++r)
                    for (int c = 0; c < d; ++c) rk(r, c) = repr[((u * r_k + r) * H + h) * d + c];
                mu.keys.push_back(rk);
                mu.values.push_back(rk);
                mu.repr_keys.push_back(rk);
            }
            for (int64_t r = 0; r < r_k; ++r) mu.repr_abs.push_back(u * r_k + r);
            st.add_unit(std::move(mu));
        }
        TokenBatch<float> b;
        for (int h = 0; h < H; ++h) {
            Mat<float> mq(l_x, d);
            for (int64_t i = 0; i < l_x; ++i)
                for (int c = 0; c < d; ++c) mq(i, c) = q[(i * H + h) * d + c];
            b.q.push_back(mq);
        }
        const auto r = st.relevance_all(b);
        for (int64_t u = 0; u < U; ++u) rel[u] = r[static_cast<size_t>(u)];
        const auto got = st.lookup(b, k_m);
        *n_ids = static_cast<int64_t>(got.size());
        for (size_t i = 0; i < got.size(); ++i) ids[i] = got[i];
    });
}

}  // extern "C"
