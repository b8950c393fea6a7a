// TEST INFRASTRUCTURE ONLY — shadow of blockmem/adapter.hpp used by
// oracle/_ref/libblockmem_ref.so. The reference engine takes q/k/v only from
// its SyntheticAdapter (engine.hpp:251, adapter.hpp:45-69). This
// header keeps the adapter's interface (ctor, shape(), seed(), batch()) but
// serves rows of caller-injected per-layer tables indexed by absolute
// position, so every other reference header compiles and runs unmodified.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "blockmem/types.hpp"

namespace blockmem {

namespace inject {
struct Table {
    std::vector<float> q, k, v;  // token-major [n][H][d] / [n][H][dv]
    Index n = 0;
    int H = 0, d = 0, dv = 0;
};
inline std::vector<Table>& tables() {
    static std::vector<Table> t;
    return t;
}
}  // namespace inject

template <typename Scalar>
class SyntheticAdapter {
public:
    SyntheticAdapter(std::uint64_t seed, ModelShape shape) : seed_(seed), shape_(shape) {
        shape.validate();
    }
    const ModelShape& shape() const { return shape_; }
    std::uint64_t seed() const { return seed_; }

    TokenBatch<Scalar> batch(int layer, std::span<const std::int64_t> ids, Index start_abs) const {
        if (ids.empty()) throw StreamError("adapter: token batch must be non-empty");
        const auto& t = inject::tables().at(static_cast<size_t>(layer));
        const Index n = static_cast<Index>(ids.size());
        if (start_abs + n > t.n) throw StreamError("inject adapter: positions beyond table");
        TokenBatch<Scalar> out;
        out.start_abs = start_abs;
        for (int h = 0; h < shape_.n_heads; ++h) {
            Mat<Scalar> q(n, t.d), k(n, t.d), v(n, t.dv);
            for (Index i = 0; i < n; ++i) {
                const Index p = start_abs + i;
                for (int c = 0; c < t.d; ++c) {
                    q(i, c) = static_cast<Scalar>(t.q[static_cast<size_t>((p * t.H + h) * t.d + c)]);
                    k(i, c) = static_cast<Scalar>(t.k[static_cast<size_t>((p * t.H + h) * t.d + c)]);
                }
                for (int c = 0; c < t.dv; ++c)
                    v(i, c) = static_cast<Scalar>(t.v[static_cast<size_t>((p * t.H + h) * t.dv + c)]);
            }
            out.q.push_back(std::move(q));
            out.k.push_back(std::move(k));
            out.v.push_back(std::move(v));
        }
        return out;
    }

private:
    std::uint64_t seed_;
    ModelShape shape_;
};

}  // namespace blockmem
