// saap_b200.hpp — header-only C++ host API over the C ABI, mirroring the
// reference's hot-path interface (/root/reference/proj/core/include/saap/
// {partition,attention,qmodel}.hpp): same function names, argument meaning
// and error behaviour (std::invalid_argument with the reference's message),
// in namespace saap_b200.  Functions are templates over any type with the
// reference's field names, so the reference's own structs can be passed.
//
// This header is for code written against the B200 library.  To run an
// existing program that calls saap:: unchanged, link libsaap_dropin.so
// (paper_2502_08246_b200/dropin/) ahead of the reference core instead: it
// defines the reference's own symbols.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "saap_b200.h"

namespace saap_b200 {

class Error : public std::runtime_error {
public:
    Error(int code, const std::string& m) : std::runtime_error(m), code(code) {}
    int code;
};

inline void check(int rc) {
    if (rc == SAAP_OK) return;
    const std::string msg = saap_last_error();
    if (rc == SAAP_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw Error(rc, msg);
}

// ---------------------------------------------------------------- stand-ins
struct TensorBlock {
    std::size_t rows = 0, dim = 0;
    std::vector<float> data;
    TensorBlock() = default;
    TensorBlock(std::size_t r, std::size_t d) : rows(r), dim(d), data(r * d, 0.f) {}
    const float* row(std::size_t i) const { return data.data() + i * dim; }
};
struct Partition {
    TensorBlock centroids;
};
struct KeyAssignment {
    std::vector<std::uint32_t> bucket_of;
};
struct IVFIndex {
    std::vector<std::uint64_t> off, idx;
};
struct DenseWindow {
    std::size_t sink_count = 1, recent_count = 2047;
};
struct SparseAttnConfig {
    std::size_t probes = 16, block_size = 128;
    DenseWindow dense;
};
struct AttnResult {
    TensorBlock output;
    std::size_t keys_scored = 0, max_visited_bucket = 0;
    bool empty_attention = false;
};

// ---------------------------------------------------------------- device state
class Context {
public:
    explicit Context(int device = 0) {
        saap_ctx* c = nullptr;
        check(saap_ctx_create(device, &c));
        h_.reset(c);
    }
    saap_ctx* get() const { return h_.get(); }
    static Context& current() {
        static Context ctx(0);
        return ctx;
    }

private:
    struct Del {
        void operator()(saap_ctx* c) const { saap_ctx_destroy(c); }
    };
    std::unique_ptr<saap_ctx, Del> h_;
};

class DevicePartition {
public:
    template <typename P>
    explicit DevicePartition(const P& p, Context& ctx = Context::current()) : ctx_(&ctx) {
        saap_partition* h = nullptr;
        check(saap_partition_create(ctx.get(), p.centroids.data.data(), p.centroids.rows,
                                    p.centroids.dim, &h));
        h_.reset(h);
        C_ = p.centroids.rows;
        d_ = p.centroids.dim;
    }
    saap_partition* get() const { return h_.get(); }
    Context& ctx() const { return *ctx_; }
    std::size_t n_buckets() const { return C_; }
    std::size_t dim() const { return d_; }

private:
    struct Del {
        void operator()(saap_partition* p) const { saap_partition_destroy(p); }
    };
    Context* ctx_;
    std::unique_ptr<saap_partition, Del> h_;
    std::size_t C_, d_;
};

// BucketRouter plugin (attention.hpp:102-108)
class BucketRouter {
public:
    virtual ~BucketRouter() { saap_router_destroy(h_); }
    template <typename TB>
    std::vector<std::uint32_t> select(const TB& q_roped, const TB& q_deroped, std::size_t l) const {
        std::vector<std::uint32_t> out(l);
        check(saap_router_select(ctx_->get(), h_, q_roped.data.data(), q_deroped.data.data(),
                                 q_roped.rows, q_roped.dim, l, out.data()));
        return out;
    }
    saap_router* get() const { return h_; }

protected:
    Context* ctx_ = nullptr;
    saap_router* h_ = nullptr;
};

class CentroidRouter : public BucketRouter {
public:
    template <typename P>
    CentroidRouter(const P& partition, bool use_deroped, Context& ctx = Context::current())
            : part_(partition, ctx) {
        ctx_ = &ctx;
        check(saap_router_create_centroid(ctx.get(), part_.get(), use_deroped ? 1 : 0, &h_));
    }

private:
    DevicePartition part_;
};

// ---------------------------------------------------------------- functions
template <typename TB, typename P>
KeyAssignment assign_keys(const TB& keys, const P& p) {
    DevicePartition dp(p);
    KeyAssignment a;
    a.bucket_of.resize(keys.rows);
    check(saap_assign_keys(dp.ctx().get(), dp.get(), keys.data.data(), keys.rows, keys.dim,
                           a.bucket_of.data()));
    return a;
}

// PartialAccumulator (attention.hpp:30-39) on the device; the operations
// below mirror pattn_absorb[_range], merge_into, merge_partials,
// pattn_finalize and attention_over_ids (attention.cpp:85-203), bit-exact.
class PartialAccumulator {
public:
    PartialAccumulator(std::size_t heads, std::size_t value_dim, Context& ctx = Context::current())
            : ctx_(&ctx), heads_(heads), dv_(value_dim) {
        saap_accum* a = nullptr;
        check(saap_accum_create(ctx.get(), heads, value_dim, &a));
        h_.reset(a);
    }
    std::size_t heads() const { return heads_; }
    std::size_t value_dim() const { return dv_; }
    saap_accum* get() const { return h_.get(); }
    Context& ctx() const { return *ctx_; }

private:
    struct Del {
        void operator()(saap_accum* a) const { saap_accum_destroy(a); }
    };
    Context* ctx_;
    std::size_t heads_, dv_;
    std::unique_ptr<saap_accum, Del> h_;
};

template <typename TB, typename Ids>
void pattn_absorb(PartialAccumulator& acc, const TB& q, const TB& keys, const TB& values, const Ids& ids) {
    const std::vector<std::uint64_t> v(ids.begin(), ids.end());
    check(saap_pattn_absorb(acc.ctx().get(), acc.get(), q.data.data(), q.rows, q.dim, keys.data.data(),
                            values.data.data(), keys.rows, keys.dim, values.rows, values.dim, v.data(),
                            v.size()));
}
template <typename TB>
void pattn_absorb_range(PartialAccumulator& acc, const TB& q, const TB& keys, const TB& values,
                        std::size_t begin, std::size_t end) {
    check(saap_pattn_absorb_range(acc.ctx().get(), acc.get(), q.data.data(), q.rows, q.dim,
                                  keys.data.data(), values.data.data(), keys.rows, keys.dim,
                                  values.rows, values.dim, begin, end));
}
inline void merge_into(PartialAccumulator& acc, const PartialAccumulator& part) {
    check(saap_merge_into(acc.ctx().get(), acc.get(), part.get()));
}
inline TensorBlock pattn_finalize(const PartialAccumulator& acc, bool* any_empty = nullptr) {
    TensorBlock out(acc.heads(), acc.value_dim());
    int e = 0;
    check(saap_pattn_finalize(acc.ctx().get(), acc.get(), out.data.data(), &e));
    if (any_empty) *any_empty = e != 0;
    return out;
}
template <typename TB, typename Ids>
TensorBlock attention_over_ids(const TB& q, const TB& keys, const TB& values, const Ids& ids,
                               bool* any_empty = nullptr) {
    const std::vector<std::uint64_t> v(ids.begin(), ids.end());
    TensorBlock out(q.rows, values.dim);
    int e = 0;
    check(saap_attention_over_ids(Context::current().get(), q.data.data(), q.rows, q.dim,
                                  keys.data.data(), values.data.data(), keys.rows, keys.dim,
                                  values.rows, values.dim, v.data(), v.size(), out.data.data(), &e));
    if (any_empty) *any_empty = e != 0;
    return out;
}

// Stand-in for saap::Rng (tensor.hpp:87-131): only the draws kmeans_train
// makes.  With the reference headers, pass saap::Rng itself.
class Rng {
public:
    explicit Rng(std::uint64_t seed) : seed_(seed), state_(seed) {}
    std::uint64_t next_u64() {
        std::uint64_t z = (state_ += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    std::uint64_t below(std::uint64_t n) {
        if (n == 0) throw std::invalid_argument("Rng::below: n must be >= 1");
        const std::uint64_t threshold = (0 - n) % n;
        for (;;) {
            const std::uint64_t r = next_u64();
            if (r >= threshold) return r % n;
        }
    }
    Rng child(std::uint64_t stream) const {
        Rng mixer(seed_ ^ (0xD1342543DE82EF95ull * (stream + 1)));
        return Rng(mixer.next_u64());
    }
    std::vector<std::uint64_t> sample_without_replacement(std::uint64_t n, std::uint64_t m) {
        if (m > n) throw std::invalid_argument("sample_without_replacement: m > n");
        std::vector<std::uint64_t> out;
        out.reserve(m);
        std::vector<bool> taken(n, false);
        for (std::uint64_t j = n - m; j < n; ++j) {
            std::uint64_t t = below(j + 1);
            if (taken[t]) t = j;
            taken[t] = true;
            out.push_back(t);
        }
        std::sort(out.begin(), out.end());
        return out;
    }
    template <typename T>
    void shuffle(std::vector<T>& v) {
        for (std::size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[(std::size_t)below(i)]);
    }

private:
    std::uint64_t seed_, state_;
};

struct KMeansStats {
    std::vector<double> objective_per_iter;
    std::size_t zero_vector_keys = 0;
    std::size_t empty_cluster_repairs = 0;
};

// kmeans_train (partition.cpp:52-179), bit-exact on the device.  The caller's
// Rng draws the seed rows here, as in the reference; any Rng/stats types with
// the reference's member names work (saap::Rng, saap::KMeansStats).
template <typename TB, typename RngT, typename StatsT = KMeansStats>
Partition kmeans_train(const TB& keys, std::size_t n_buckets, std::size_t iters, RngT& rng,
                       StatsT* stats = nullptr) {
    if (n_buckets < 1) throw std::invalid_argument("kmeans_train: need at least 1 bucket");
    if (keys.rows < n_buckets)
        throw std::invalid_argument("kmeans_train: " + std::to_string(keys.rows) +
                                    " keys cannot seed " + std::to_string(n_buckets) + " buckets");
    if (iters < 1) throw std::invalid_argument("kmeans_train: iters must be >= 1");
    auto seeds = rng.sample_without_replacement(keys.rows, n_buckets);
    rng.shuffle(seeds);
    std::vector<std::uint64_t> rows(seeds.begin(), seeds.end());
    Partition p;
    p.centroids = TensorBlock(n_buckets, keys.dim);
    std::vector<double> obj(iters);
    std::uint64_t zk = 0, rep = 0;
    check(saap_kmeans_train(Context::current().get(), keys.data.data(), keys.rows, keys.dim,
                            n_buckets, iters, rows.data(), p.centroids.data.data(), obj.data(),
                            &zk, &rep));
    if (stats) {
        stats->objective_per_iter.assign(obj.begin(), obj.end());
        stats->zero_vector_keys = zk;
        stats->empty_cluster_repairs = rep;
    }
    return p;
}

template <typename KA>
IVFIndex build_ivf(const KA& assignment, std::size_t n_buckets) {
    IVFIndex ix;
    ix.off.resize(n_buckets + 1);
    ix.idx.resize(assignment.bucket_of.size());
    check(saap_build_ivf(Context::current().get(), assignment.bucket_of.data(),
                         assignment.bucket_of.size(), n_buckets, ix.off.data(), ix.idx.data()));
    return ix;
}

template <typename TB>
TensorBlock full_attention(const TB& q, const TB& keys, const TB& values) {
    if (keys.rows != values.rows)
        throw std::invalid_argument("attention: " + std::to_string(keys.rows) + " keys vs " +
                                    std::to_string(values.rows) + " values");
    TensorBlock out(q.rows, values.dim);
    check(saap_full_attention(Context::current().get(), q.data.data(), q.rows, keys.data.data(),
                              values.data.data(), keys.rows, keys.dim, out.data.data()));
    return out;
}

// One ContextStore on the device (attention.hpp:76-86).
class ContextStore {
public:
    // build_context_store(keys_roped, values, rope, partition, sink), with the
    // partition's pre-RoPE keys passed explicitly (or nullptr: de-rope on device)
    template <typename TB, typename P>
    ContextStore(const TB& keys_roped, const TB& values, double rope_base, const P& partition,
                 std::size_t sink, const TB* keys_deroped = nullptr, std::size_t recent_hint = 2047,
                 Context& ctx = Context::current())
            : ctx_(&ctx), part_(partition, ctx), sink_(sink), n_(keys_roped.rows) {
        if (keys_roped.rows != values.rows)
            throw std::invalid_argument("attention: " + std::to_string(keys_roped.rows) +
                                        " keys vs " + std::to_string(values.rows) + " values");
        const std::uint64_t n = keys_roped.rows;
        saap_layer* L = nullptr;
        check(saap_layer_create(ctx.get(), 1, keys_roped.dim, part_.n_buckets(), &n, sink,
                                recent_hint, &L));
        h_.reset(L);
        const saap_partition* pp = part_.get();
        check(saap_layer_build(ctx.get(), L, &pp, keys_roped.data.data(), values.data.data(),
                               keys_deroped ? keys_deroped->data.data() : nullptr, rope_base));
    }
    std::size_t n_keys() const { return n_; }
    std::size_t id_offset() const { return sink_; }
    saap_layer* get() const { return h_.get(); }
    Context& ctx() const { return *ctx_; }
    KeyAssignment assignment() const {
        KeyAssignment a;
        a.bucket_of.resize(n_ - sink_);
        check(saap_layer_read_index(ctx_->get(), h_.get(), 0, a.bucket_of.data(), nullptr, nullptr));
        return a;
    }
    IVFIndex index() const {
        IVFIndex ix;
        ix.off.resize(part_.n_buckets() + 1);
        ix.idx.resize(n_ - sink_);
        check(saap_layer_read_index(ctx_->get(), h_.get(), 0, nullptr, ix.off.data(), ix.idx.data()));
        return ix;
    }

private:
    struct Del {
        void operator()(saap_layer* L) const { saap_layer_destroy(L); }
    };
    Context* ctx_;
    DevicePartition part_;
    std::size_t sink_, n_;
    std::unique_ptr<saap_layer, Del> h_;
};

// sparse_attention(q_roped, q_deroped, store, router, cfg) attention.cpp:317-376
template <typename TB, typename CFG>
AttnResult sparse_attention(const TB& q_roped, const TB& q_deroped, const ContextStore& store,
                            const BucketRouter& router, const CFG& cfg) {
    AttnResult r;
    r.output = TensorBlock(q_roped.rows, q_roped.dim);
    saap_sparse_cfg c{cfg.probes, cfg.block_size, cfg.dense.sink_count, cfg.dense.recent_count};
    saap_attn_stats st{};
    const saap_router* rt = router.get();
    check(saap_sparse_attention(store.ctx().get(), store.get(), &rt, q_roped.data.data(),
                                q_deroped.data.data(), q_roped.rows, &c, r.output.data.data(), &st,
                                nullptr));
    r.keys_scored = st.keys_scored;
    r.max_visited_bucket = st.max_visited_bucket;
    r.empty_attention = st.empty_attention != 0;
    return r;
}

inline double selectivity(const AttnResult& r, std::size_t n_keys) {
    if (n_keys == 0) throw std::invalid_argument("selectivity: empty context");
    return static_cast<double>(r.keys_scored) / static_cast<double>(n_keys);
}

// QModelRouter(model) (attention.hpp:127-140): Q-model parameters in the
// reference's fp64 layout (any type with QModel's Mat members).
class QModelRouter : public BucketRouter {
public:
    template <typename QM>
    explicit QModelRouter(const QM& m, Context& ctx = Context::current()) {
        ctx_ = &ctx;
        check(saap_qmodel_create(ctx.get(), m.w1.rows, m.w1.cols, m.w2.cols, m.w1.data.data(),
                                 m.b1.data.data(), m.bn_gamma.data.data(), m.bn_beta.data.data(),
                                 m.bn_run_mean.data.data(), m.bn_run_var.data.data(),
                                 m.w2.data.data(), m.b2.data.data(), &qm_));
        check(saap_router_create_qmodel(ctx.get(), qm_, &h_));
    }
    ~QModelRouter() override {
        saap_router_destroy(h_);
        h_ = nullptr;
        saap_qmodel_destroy(qm_);
    }
    saap_qmodel* model() const { return qm_; }

private:
    saap_qmodel* qm_ = nullptr;
};

// batched_bucket_select(model, q_group, l)   qmodel.cpp:485-511
template <typename TB>
std::vector<std::uint32_t> batched_bucket_select(const QModelRouter& r, const TB& q, std::size_t l) {
    std::vector<std::uint32_t> out(l);
    check(saap_batched_bucket_select(Context::current().get(), r.model(), q.data.data(), q.rows,
                                     q.dim, l, out.data()));
    return out;
}

// merge_partials(parts)   attention.cpp:130-139 (bit-exact fp64 on the device)
inline PartialAccumulator merge_partials(const std::vector<const PartialAccumulator*>& parts) {
    if (parts.empty()) throw std::invalid_argument("merge_partials: empty list");
    PartialAccumulator out(parts[0]->heads(), parts[0]->value_dim(), parts[0]->ctx());
    std::vector<const saap_accum*> hs;
    for (auto* p : parts) hs.push_back(p->get());
    check(saap_merge_partials(out.ctx().get(), hs.data(), hs.size(), out.get()));
    return out;
}

// mse(approx, exact)   attention.cpp:385-399 (bit-identical sequential fp64 sum)
template <typename TB>
double mse(const TB& approx, const TB& exact) {
    double out = 0.0;
    check(saap_mse(approx.data.data(), approx.rows, approx.dim, exact.data.data(), exact.rows,
                   exact.dim, &out));
    return out;
}

// attention_mass_coverage(q_roped, store, selected, dense)  attention.cpp:427-462
template <typename TB, typename Sel, typename DW>
double attention_mass_coverage(const TB& q_roped, const ContextStore& store, const Sel& selected,
                               const DW& dense) {
    const std::vector<std::uint32_t> sel(selected.begin(), selected.end());
    double out = 0.0;
    check(saap_attention_mass_coverage(store.ctx().get(), store.get(), q_roped.data.data(),
                                       q_roped.rows, sel.data(), sel.size(), dense.sink_count,
                                       dense.recent_count, &out));
    return out;
}

// build_context_store(keys_roped, values, rope, partition, sink)  attention.cpp:249-255,
// RopeConfig-shaped `rope` ({dim, base_theta}); the de-rope runs on the device
template <typename TB, typename Rope, typename P>
std::unique_ptr<ContextStore> build_context_store(const TB& keys_roped, const TB& values,
                                                  const Rope& rope, const P& partition,
                                                  std::size_t sink_count) {
    if (keys_roped.rows <= sink_count)
        throw std::invalid_argument("build_context_store: no keys left to index after " +
                                    std::to_string(sink_count) + " sink keys");
    if (rope.dim == 0 || rope.dim % 2 != 0)
        throw std::invalid_argument("RopeConfig: dim must be even and positive, got " +
                                    std::to_string(rope.dim));
    if (keys_roped.dim != rope.dim)
        throw std::invalid_argument("rope: block dim " + std::to_string(keys_roped.dim) +
                                    " does not match configured dim " + std::to_string(rope.dim));
    return std::make_unique<ContextStore>(keys_roped, values, rope.base_theta, partition,
                                          sink_count);
}

// build_context_store(keys_roped, values, rope, C, kmeans_iters, sink, rng, stats)
// attention.cpp:238-246: device de-rope, device k-means (the caller's Rng
// draws the seeds), then the store under the trained partition.
template <typename TB, typename Rope, typename RngT, typename StatsT = KMeansStats>
std::unique_ptr<ContextStore> build_context_store(const TB& keys_roped, const TB& values,
                                                  const Rope& rope, std::size_t n_buckets,
                                                  std::size_t kmeans_iters, std::size_t sink_count,
                                                  RngT& rng, StatsT* stats = nullptr) {
    if (keys_roped.rows <= sink_count)
        throw std::invalid_argument("build_context_store: no keys left to index after " +
                                    std::to_string(sink_count) + " sink keys");
    const std::size_t n = keys_roped.rows - sink_count, d = keys_roped.dim;
    TensorBlock de(n, d);
    std::vector<std::uint64_t> pos(n);
    for (std::size_t i = 0; i < n; ++i) pos[i] = sink_count + i;
    check(saap_rope_remove(Context::current().get(), keys_roped.data.data() + sink_count * d, n, d,
                           pos.data(), rope.base_theta, de.data.data()));
    Partition p = kmeans_train(de, n_buckets, kmeans_iters, rng, stats);
    return build_context_store(keys_roped, values, rope, p, sink_count);
}

}  // namespace saap_b200
