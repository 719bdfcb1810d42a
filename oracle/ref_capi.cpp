// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" veneer over the *unmodified* reference library (the sources under
// /root/reference/proj/core/src are compiled as-is by oracle/Makefile into
// oracle/_ref/libsaap_ref.so together with this file).  It exists so pytest,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm
// can drive the reference's own C++ API through ctypes:
//
//   generate_prompt        synthdata.cpp:169-281      (input generator)
//   train_head_partition   experiments.cpp:284-295    (k-means, offline)
//   assign_keys            partition.cpp:191-198
//   build_ivf              partition.cpp:200-223
//   CentroidRouter::select attention.cpp:275-306
//   batched_bucket_select  qmodel.cpp:485-511
//   sparse_attention       attention.cpp:317-376
//   full_attention         attention.cpp:163-195
//   attention_mass_coverage attention.cpp:427-462, mse attention.cpp:385-399
//   build_context_store    attention.cpp:249-255 (de-rope + assign + ivf)
//
// Every entry point returns 0 on success, 1 on std::invalid_argument, 2 on any
// other exception; the message is kept in a thread-local buffer readable via
// ref_last_error().  Nothing here re-implements reference arithmetic.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "saap/attention.hpp"
#include "saap/experiments.hpp"
#include "saap/partition.hpp"
#include "saap/qmodel.hpp"
#include "saap/rope.hpp"
#include "saap/synthdata.hpp"
#include "saap/tensor.hpp"
#include "saap/tensor_io.hpp"

using namespace saap;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

TensorBlock block(const float* p, std::size_t rows, std::size_t dim) {
    TensorBlock t(rows, dim);
    if (rows * dim) std::memcpy(t.data.data(), p, rows * dim * sizeof(float));
    return t;
}

void put(const TensorBlock& t, float* out) {
    if (!t.data.empty()) std::memcpy(out, t.data.data(), t.data.size() * sizeof(float));
}

Mat mat(const double* p, std::size_t rows, std::size_t cols) {
    Mat m(rows, cols);
    std::memcpy(m.data.data(), p, rows * cols * sizeof(double));
    return m;
}

struct RefSpec {
    // mirrors the HeadSpec fields the harness varies; everything else stays
    // at its reference default (synthdata.hpp:24-56)
    std::uint64_t dim;
    std::uint64_t seed;
    double drift_rate;
    std::uint64_t lowfreq_pairs;
    std::uint64_t n_clusters;
    std::uint64_t n_targets;
    std::uint64_t local_range;
    std::uint64_t longrange_threshold;
    std::uint64_t window_guard;
    double planted_longrange_fraction;
    double rope_base;
};

HeadSpec make_spec(const RefSpec* s) {
    HeadSpec h;
    h.dim = s->dim;
    h.seed = s->seed;
    h.drift_rate = s->drift_rate;
    h.lowfreq_pairs = s->lowfreq_pairs;
    h.n_clusters = s->n_clusters;
    h.n_targets = s->n_targets;
    h.local_range = s->local_range;
    h.longrange_threshold = s->longrange_threshold;
    h.window_guard = s->window_guard;
    h.planted_longrange_fraction = s->planted_longrange_fraction;
    h.rope_base = s->rope_base;
    return h;
}

QModel make_qmodel(std::size_t d, std::size_t h, std::size_t C, const double* w1,
                   const double* b1, const double* gamma, const double* beta,
                   const double* mean, const double* var, const double* w2, const double* b2) {
    QModel m;
    m.w1 = mat(w1, d, h);
    m.b1 = mat(b1, 1, h);
    m.bn_gamma = mat(gamma, 1, h);
    m.bn_beta = mat(beta, 1, h);
    m.bn_run_mean = mat(mean, 1, h);
    m.bn_run_var = mat(var, 1, h);
    m.w2 = mat(w2, h, C);
    m.b2 = mat(b2, 1, C);
    return m;
}

// A store assembled field by field (attention_test.cpp:418-432 does the same),
// so assignment parity is defined on the caller's pre-RoPE keys.
struct RefStore {
    ContextStore store;
};

struct RefRouter {
    std::unique_ptr<BucketRouter> router;
};

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_generate_prompt(const RefSpec* spec, std::uint64_t n_keys, std::uint64_t n_q,
                        std::uint64_t prompt_seed, float* keys_deroped, float* keys_roped,
                        float* values, float* q_deroped, float* q_roped) {
    return guard([&] {
        SyntheticPrompt p = generate_prompt(make_spec(spec), n_keys, n_q, prompt_seed);
        put(p.keys_deroped, keys_deroped);
        put(p.keys_roped, keys_roped);
        put(p.values, values);
        put(p.queries_deroped, q_deroped);
        put(p.queries_roped, q_roped);
    });
}

int ref_train_head_partition(const RefSpec* spec, std::uint64_t n_keys, std::uint64_t n_buckets,
                             std::uint64_t iters, std::uint64_t sink, float* centroids) {
    return guard([&] {
        Partition p = train_head_partition(make_spec(spec), n_keys, n_buckets, iters, sink);
        put(p.centroids, centroids);
    });
}

int ref_kmeans_train(const float* keys, std::uint64_t n, std::uint64_t d, std::uint64_t n_buckets,
                     std::uint64_t iters, std::uint64_t seed, float* centroids) {
    return guard([&] {
        Rng rng(seed);
        Partition p = kmeans_train(block(keys, n, d), n_buckets, iters, rng);
        put(p.centroids, centroids);
    });
}

// kmeans_train with its KMeansStats; the Rng is Rng(seed), or
// Rng(seed).child(stream) when stream != ~0 (train_head_partition's stream).
// rng_state_after receives the Rng's next draw after training (stream check).
int ref_kmeans_train_stats(const float* keys, std::uint64_t n, std::uint64_t d,
                           std::uint64_t n_buckets, std::uint64_t iters, std::uint64_t seed,
                           std::uint64_t stream, float* centroids, double* objective,
                           std::uint64_t* zero_keys, std::uint64_t* repairs,
                           std::uint64_t* next_draw) {
    return guard([&] {
        Rng rng = stream == ~0ull ? Rng(seed) : Rng(seed).child(stream);
        KMeansStats st;
        Partition p = kmeans_train(block(keys, n, d), n_buckets, iters, rng, &st);
        put(p.centroids, centroids);
        std::copy(st.objective_per_iter.begin(), st.objective_per_iter.end(), objective);
        *zero_keys = st.zero_vector_keys;
        *repairs = st.empty_cluster_repairs;
        *next_draw = rng.next_u64();
    });
}

// The seed rows kmeans_train draws (partition.cpp:80-82) for Rng(seed).
int ref_kmeans_seed_rows(std::uint64_t seed, std::uint64_t n, std::uint64_t m,
                         std::uint64_t* out) {
    return guard([&] {
        Rng rng(seed);
        auto s = rng.sample_without_replacement(n, m);
        rng.shuffle(s);
        std::copy(s.begin(), s.end(), out);
    });
}

int ref_assign_keys(const float* keys, std::uint64_t n, std::uint64_t d, const float* centroids,
                    std::uint64_t C, std::uint32_t* out) {
    return guard([&] {
        Partition p;
        p.centroids = block(centroids, C, d);
        KeyAssignment a = assign_keys(block(keys, n, d), p);
        std::copy(a.bucket_of.begin(), a.bucket_of.end(), out);
    });
}

// Threaded over disjoint key ranges; assign_keys is a pure per-key map
// (partition.cpp:191-198) so the result is identical to one call.
int ref_assign_keys_mt(const float* keys, std::uint64_t n, std::uint64_t d,
                       const float* centroids, std::uint64_t C, std::uint32_t* out,
                       std::uint64_t threads) {
    return guard([&] {
        Partition p;
        p.centroids = block(centroids, C, d);
        const std::size_t T = std::max<std::uint64_t>(1, threads);
        std::vector<std::thread> pool;
        std::atomic<int> failed{0};
        for (std::size_t t = 0; t < T; ++t) {
            pool.emplace_back([&, t] {
                const std::size_t lo = n * t / T, hi = n * (t + 1) / T;
                try {
                    KeyAssignment a = assign_keys(block(keys + lo * d, hi - lo, d), p);
                    std::copy(a.bucket_of.begin(), a.bucket_of.end(), out + lo);
                } catch (...) {
                    failed = 1;
                }
            });
        }
        for (auto& th : pool) th.join();
        if (failed) throw std::runtime_error("ref_assign_keys_mt: worker failed");
    });
}

int ref_build_ivf(const std::uint32_t* assignment, std::uint64_t n, std::uint64_t C,
                  std::uint64_t* off, std::uint64_t* idx) {
    return guard([&] {
        KeyAssignment a;
        a.bucket_of.assign(assignment, assignment + n);
        IVFIndex ix = build_ivf(a, C);
        std::copy(ix.off.begin(), ix.off.end(), off);
        std::copy(ix.idx.begin(), ix.idx.end(), idx);
    });
}

int ref_rope_remove_block(const float* x, std::uint64_t rows, std::uint64_t d,
                          const std::uint64_t* positions, double base, float* out) {
    return guard([&] {
        RopeConfig cfg{d, base};
        TensorBlock r = rope_remove_block(block(x, rows, d),
                                          std::span<const std::uint64_t>(positions, rows), cfg);
        put(r, out);
    });
}

int ref_build_context_store(const float* keys_roped, const float* values, std::uint64_t n,
                            std::uint64_t d, double rope_base, const float* centroids,
                            std::uint64_t C, std::uint64_t sink, std::uint32_t* assignment,
                            std::uint64_t* off, std::uint64_t* idx) {
    return guard([&] {
        Partition p;
        p.centroids = block(centroids, C, d);
        ContextStore s = build_context_store(block(keys_roped, n, d), block(values, n, d),
                                             RopeConfig{d, rope_base}, p, sink);
        std::copy(s.assignment.bucket_of.begin(), s.assignment.bucket_of.end(), assignment);
        std::copy(s.index.off.begin(), s.index.off.end(), off);
        std::copy(s.index.idx.begin(), s.index.idx.end(), idx);
    });
}

int ref_centroid_select(const float* centroids, std::uint64_t C, std::uint64_t d, int use_deroped,
                        const float* q_roped, const float* q_deroped, std::uint64_t G,
                        std::uint64_t l, std::uint32_t* out) {
    return guard([&] {
        Partition p;
        p.centroids = block(centroids, C, d);
        CentroidRouter r(p, use_deroped != 0);
        auto ids = r.select(block(q_roped, G, d), block(q_deroped, G, d), l);
        std::copy(ids.begin(), ids.end(), out);
    });
}

int ref_qmodel_init(std::uint64_t d, std::uint64_t h, std::uint64_t C, std::uint64_t seed,
                    double* w1, double* b1, double* gamma, double* beta, double* mean, double* var,
                    double* w2, double* b2) {
    return guard([&] {
        Rng rng(seed);
        QModel m = qmodel_init(d, h, C, rng);
        auto cp = [](const Mat& s, double* o) { std::copy(s.data.begin(), s.data.end(), o); };
        cp(m.w1, w1);
        cp(m.b1, b1);
        cp(m.bn_gamma, gamma);
        cp(m.bn_beta, beta);
        cp(m.bn_run_mean, mean);
        cp(m.bn_run_var, var);
        cp(m.w2, w2);
        cp(m.b2, b2);
    });
}

int ref_qmodel_select(std::uint64_t d, std::uint64_t h, std::uint64_t C, const double* w1,
                      const double* b1, const double* gamma, const double* beta,
                      const double* mean, const double* var, const double* w2, const double* b2,
                      const float* q_deroped, std::uint64_t G, std::uint64_t l,
                      std::uint32_t* out) {
    return guard([&] {
        QModelRouter r(make_qmodel(d, h, C, w1, b1, gamma, beta, mean, var, w2, b2));
        TensorBlock q = block(q_deroped, G, d);
        auto ids = r.select(q, q, l);
        std::copy(ids.begin(), ids.end(), out);
    });
}

int ref_qmodel_forward(std::uint64_t d, std::uint64_t h, std::uint64_t C, const double* w1,
                       const double* b1, const double* gamma, const double* beta,
                       const double* mean, const double* var, const double* w2, const double* b2,
                       const float* q_deroped, std::uint64_t G, float* probs) {
    return guard([&] {
        QModel m = make_qmodel(d, h, C, w1, b1, gamma, beta, mean, var, w2, b2);
        put(qmodel_forward(m, block(q_deroped, G, d)), probs);
    });
}

int ref_full_attention(const float* q, std::uint64_t G, const float* keys, const float* values,
                       std::uint64_t n, std::uint64_t d, float* out) {
    return guard([&] { put(full_attention(block(q, G, d), block(keys, n, d), block(values, n, d)), out); });
}

// ---- persistent store / router handles (used for timing the reference) ----

int ref_store_create(const float* keys_roped, const float* values, std::uint64_t n,
                     std::uint64_t d, const float* centroids, std::uint64_t C, std::uint64_t sink,
                     const std::uint32_t* assignment, void** out) {
    return guard([&] {
        auto* s = new RefStore;
        s->store.keys = block(keys_roped, n, d);
        s->store.values = block(values, n, d);
        s->store.id_offset = sink;
        s->store.partition.centroids = block(centroids, C, d);
        s->store.assignment.bucket_of.assign(assignment, assignment + (n - sink));
        s->store.index = build_ivf(s->store.assignment, C);
        *out = s;
    });
}

void ref_store_destroy(void* s) { delete static_cast<RefStore*>(s); }

int ref_router_centroid_create(const float* centroids, std::uint64_t C, std::uint64_t d,
                               int use_deroped, void** out) {
    return guard([&] {
        Partition p;
        p.centroids = block(centroids, C, d);
        auto* r = new RefRouter;
        r->router = std::make_unique<CentroidRouter>(p, use_deroped != 0);
        *out = r;
    });
}

int ref_router_qmodel_create(std::uint64_t d, std::uint64_t h, std::uint64_t C,
                             const double* w1, const double* b1, const double* gamma,
                             const double* beta, const double* mean, const double* var,
                             const double* w2, const double* b2, void** out) {
    return guard([&] {
        auto* r = new RefRouter;
        r->router = std::make_unique<QModelRouter>(
                make_qmodel(d, h, C, w1, b1, gamma, beta, mean, var, w2, b2));
        *out = r;
    });
}

void ref_router_destroy(void* r) { delete static_cast<RefRouter*>(r); }

int ref_router_select(void* router, const float* q_roped, const float* q_deroped,
                      std::uint64_t G, std::uint64_t d, std::uint64_t l, std::uint32_t* out) {
    return guard([&] {
        auto ids = static_cast<RefRouter*>(router)->router->select(block(q_roped, G, d),
                                                                   block(q_deroped, G, d), l);
        std::copy(ids.begin(), ids.end(), out);
    });
}

int ref_store_sparse_attention(void* store, void* router, const float* q_roped,
                               const float* q_deroped, std::uint64_t G, std::uint64_t probes,
                               std::uint64_t block_size, std::uint64_t sink, std::uint64_t recent,
                               float* out, std::uint64_t* keys_scored,
                               std::uint64_t* max_visited, int* empty) {
    return guard([&] {
        const ContextStore& s = static_cast<RefStore*>(store)->store;
        SparseAttnConfig cfg;
        cfg.probes = probes;
        cfg.block_size = block_size;
        cfg.dense = DenseWindow{sink, recent};
        const std::size_t d = s.keys.dim;
        AttnResult r = sparse_attention(block(q_roped, G, d), block(q_deroped, G, d), s,
                                        *static_cast<RefRouter*>(router)->router, cfg);
        put(r.output, out);
        *keys_scored = r.keys_scored;
        *max_visited = r.max_visited_bucket;
        *empty = r.empty_attention ? 1 : 0;
    });
}

int ref_store_full_attention(void* store, const float* q, std::uint64_t G, float* out) {
    return guard([&] {
        const ContextStore& s = static_cast<RefStore*>(store)->store;
        put(full_attention(block(q, G, s.keys.dim), s.keys, s.values), out);
    });
}

int ref_store_coverage(void* store, const float* q_roped, std::uint64_t G,
                       const std::uint32_t* selected, std::uint64_t l, std::uint64_t sink,
                       std::uint64_t recent, double* out) {
    return guard([&] {
        const ContextStore& s = static_cast<RefStore*>(store)->store;
        *out = attention_mass_coverage(block(q_roped, G, s.keys.dim), s,
                                       std::span<const std::uint32_t>(selected, l),
                                       DenseWindow{sink, recent});
    });
}

int ref_mse(const float* a, const float* b, std::uint64_t rows, std::uint64_t d, double* out) {
    return guard([&] { *out = mse(block(a, rows, d), block(b, rows, d)); });
}

// One decode step of many (store, router, query group) triples on a thread
// pool: the stores and routers are read-only, so groups
// are independent.  Used to time the reference on the bench workload.
int ref_sparse_attention_batch(std::uint64_t n_groups, void* const* stores,
                               void* const* routers, const float* q_roped,
                               const float* q_deroped, std::uint64_t G, std::uint64_t d,
                               std::uint64_t probes, std::uint64_t block_size,
                               std::uint64_t sink, std::uint64_t recent, int dense,
                               std::uint64_t threads, float* out, std::uint64_t* keys_scored) {
    return guard([&] {
        const std::size_t T = std::max<std::uint64_t>(1, threads);
        std::atomic<std::uint64_t> next{0};
        std::atomic<int> failed{0};
        std::string first_err;
        std::vector<std::thread> pool;
        for (std::size_t t = 0; t < T; ++t) {
            pool.emplace_back([&] {
                for (;;) {
                    const std::uint64_t g = next.fetch_add(1);
                    if (g >= n_groups) return;
                    try {
                        const ContextStore& s = static_cast<RefStore*>(stores[g])->store;
                        TensorBlock qr = block(q_roped + g * G * d, G, d);
                        if (dense) {
                            put(full_attention(qr, s.keys, s.values), out + g * G * d);
                            if (keys_scored) keys_scored[g] = s.n_keys();
                        } else {
                            SparseAttnConfig cfg;
                            cfg.probes = probes;
                            cfg.block_size = block_size;
                            cfg.dense = DenseWindow{sink, recent};
                            AttnResult r = sparse_attention(
                                    qr, block(q_deroped + g * G * d, G, d), s,
                                    *static_cast<RefRouter*>(routers[g])->router, cfg);
                            put(r.output, out + g * G * d);
                            if (keys_scored) keys_scored[g] = r.keys_scored;
                        }
                    } catch (const std::exception& e) {
                        failed = 1;
                        return;
                    }
                }
            });
        }
        for (auto& th : pool) th.join();
        if (failed) throw std::runtime_error("ref_sparse_attention_batch: a group failed");
    });
}

// The parity pass of the bench (tests too): per (store, router, group) on
// a thread pool, everything the GPU step is compared with -- the routed list
// (router.select), sparse_attention (output + counters), full_attention (the
// exact output, for mse) and attention_mass_coverage of the routed list.
int ref_parity_batch(std::uint64_t n_groups, void* const* stores, void* const* routers,
                     const float* q_roped, const float* q_deroped, std::uint64_t G,
                     std::uint64_t d, std::uint64_t probes, std::uint64_t block_size,
                     std::uint64_t sink, std::uint64_t recent, std::uint64_t threads,
                     float* out_sparse, float* out_full, std::uint32_t* selected,
                     std::uint64_t* keys_scored, std::uint64_t* max_visited, int* empty,
                     double* coverage) {
    return guard([&] {
        const std::size_t T = std::max<std::uint64_t>(1, threads);
        std::atomic<std::uint64_t> next{0};
        std::atomic<int> failed{0};
        std::vector<std::thread> pool;
        for (std::size_t t = 0; t < T; ++t) {
            pool.emplace_back([&] {
                for (;;) {
                    const std::uint64_t g = next.fetch_add(1);
                    if (g >= n_groups) return;
                    try {
                        const ContextStore& s = static_cast<RefStore*>(stores[g])->store;
                        const BucketRouter& r = *static_cast<RefRouter*>(routers[g])->router;
                        TensorBlock qr = block(q_roped + g * G * d, G, d);
                        TensorBlock qd = block(q_deroped + g * G * d, G, d);
                        auto ids = r.select(qr, qd, probes);
                        std::copy(ids.begin(), ids.end(), selected + g * probes);
                        SparseAttnConfig cfg;
                        cfg.probes = probes;
                        cfg.block_size = block_size;
                        cfg.dense = DenseWindow{sink, recent};
                        AttnResult a = sparse_attention(qr, qd, s, r, cfg);
                        put(a.output, out_sparse + g * G * d);
                        keys_scored[g] = a.keys_scored;
                        max_visited[g] = a.max_visited_bucket;
                        empty[g] = a.empty_attention ? 1 : 0;
                        put(full_attention(qr, s.keys, s.values), out_full + g * G * d);
                        coverage[g] = attention_mass_coverage(
                                qr, s, std::span<const std::uint32_t>(ids.data(), ids.size()),
                                DenseWindow{sink, recent});
                    } catch (const std::exception&) {
                        failed = 1;
                        return;
                    }
                }
            });
        }
        for (auto& th : pool) th.join();
        if (failed) throw std::runtime_error("ref_parity_batch: a group failed");
    });
}

// generate_prompt for many (spec seed, prompt seed) pairs on a thread pool
// (the reference generator is single-threaded; prompts are independent).
int ref_generate_prompts(const RefSpec* spec, std::uint64_t n_prompts, const std::uint64_t* seeds,
                         const std::uint64_t* prompt_seeds, std::uint64_t n_keys, std::uint64_t n_q,
                         std::uint64_t threads, float* const* keys_deroped,
                         float* const* keys_roped, float* const* values, float* q_deroped,
                         float* q_roped) {
    return guard([&] {
        const std::size_t T = std::max<std::uint64_t>(1, threads);
        std::atomic<std::uint64_t> next{0};
        std::atomic<int> failed{0};
        std::vector<std::thread> pool;
        const std::size_t d = spec->dim;
        for (std::size_t t = 0; t < T; ++t) {
            pool.emplace_back([&] {
                for (;;) {
                    const std::uint64_t i = next.fetch_add(1);
                    if (i >= n_prompts) return;
                    try {
                        RefSpec sp = *spec;
                        sp.seed = seeds[i];
                        SyntheticPrompt p = generate_prompt(make_spec(&sp), n_keys, n_q, prompt_seeds[i]);
                        if (keys_deroped && keys_deroped[i]) put(p.keys_deroped, keys_deroped[i]);
                        if (keys_roped && keys_roped[i]) put(p.keys_roped, keys_roped[i]);
                        if (values && values[i]) put(p.values, values[i]);
                        if (q_deroped) put(p.queries_deroped, q_deroped + i * n_q * d);
                        if (q_roped) put(p.queries_roped, q_roped + i * n_q * d);
                    } catch (const std::exception&) {
                        failed = 1;
                        return;
                    }
                }
            });
        }
        for (auto& th : pool) th.join();
        if (failed) throw std::runtime_error("ref_generate_prompts: a prompt failed");
    });
}

} // extern "C"

// ---------------------------------------------------------------- artifacts
// tensor_io.cpp / partition.cpp:260-296 / qmodel.cpp:530-589.  ref_io_kind()
// is the IoErrorKind of the last IoError (-1 otherwise).
namespace {
thread_local int g_io_kind = -1;
template <typename F>
int io_guard(F&& f) {
    g_io_kind = -1;
    try {
        f();
        return 0;
    } catch (const IoError& e) {
        g_err = e.what();
        g_io_kind = static_cast<int>(e.kind());
        return 3;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}
}  // namespace

extern "C" {
int ref_io_kind() { return g_io_kind; }

int ref_tensor_write(const char* path, const float* data, std::uint64_t rows, std::uint64_t dim) {
    return io_guard([&] { tensor_write(block(data, rows, dim), path); });
}

int ref_tensor_read(const char* path, float* out, std::uint64_t cap, std::uint64_t* rows,
                    std::uint64_t* dim) {
    return io_guard([&] {
        TensorBlock t = tensor_read(path);
        *rows = t.rows;
        *dim = t.dim;
        if (out && cap >= t.data.size()) put(t, out);
    });
}

int ref_u64_write(const char* path, const std::uint64_t* v, std::uint64_t n) {
    return io_guard([&] { u64_write(std::vector<std::uint64_t>(v, v + n), path); });
}

int ref_u64_read(const char* path, std::uint64_t* out, std::uint64_t cap, std::uint64_t* n) {
    return io_guard([&] {
        auto v = u64_read(path);
        *n = v.size();
        if (out && cap >= v.size()) std::copy(v.begin(), v.end(), out);
    });
}

int ref_partition_load(const char* path, float* out, std::uint64_t cap, std::uint64_t* C,
                       std::uint64_t* d) {
    return io_guard([&] {
        Partition p = partition_load(path);
        *C = p.n_buckets();
        *d = p.dim();
        if (out && cap >= p.centroids.data.size()) put(p.centroids, out);
    });
}

int ref_ivf_load(const char* off_path, const char* idx_path, std::uint64_t* n_off,
                 std::uint64_t* n_idx) {
    return io_guard([&] {
        IVFIndex ix = ivf_load(off_path, idx_path);
        *n_off = ix.off.size();
        *n_idx = ix.idx.size();
    });
}

// qmodel_save of qmodel_init(d, h, C, Rng(seed)) (the params come back via
// ref_qmodel_init with the same seed).
int ref_qmodel_save_init(const char* dir, std::uint64_t d, std::uint64_t h, std::uint64_t C,
                         std::uint64_t seed) {
    return io_guard([&] {
        Rng rng(seed);
        qmodel_save(qmodel_init(d, h, C, rng), dir);
    });
}

int ref_qmodel_load(const char* dir, std::uint64_t* dims, double* w1, double* b1, double* gamma,
                    double* beta, double* mean, double* var, double* w2, double* b2) {
    return io_guard([&] {
        QModel m = qmodel_load(dir);
        dims[0] = m.dim();
        dims[1] = m.hidden();
        dims[2] = m.n_buckets();
        if (!w1) return;
        auto cp = [](const Mat& s, double* o) { std::copy(s.data.begin(), s.data.end(), o); };
        cp(m.w1, w1);
        cp(m.b1, b1);
        cp(m.bn_gamma, gamma);
        cp(m.bn_beta, beta);
        cp(m.bn_run_mean, mean);
        cp(m.bn_run_var, var);
        cp(m.w2, w2);
        cp(m.b2, b2);
    });
}
}  // extern "C"

// ---------------------------------------------------------------- Q-model training
extern "C" {
// K train_step_on_target calls (qmodel.cpp:419-433) from the given params
// (checkpoint order) with TrainerState{lr, ...defaults}; batches q [K][n x d]
// f32 and targets [K][n x C] fp64.  Params are updated in place; losses [K].
int ref_qtrain_steps(std::uint64_t d, std::uint64_t h, std::uint64_t C, double* w1, double* b1,
                     double* gamma, double* beta, double* mean, double* var, double* w2,
                     double* b2, double lr, std::uint64_t K, std::uint64_t n, const float* q,
                     const double* targets, double* losses) {
    return guard([&] {
        QModel m = make_qmodel(d, h, C, w1, b1, gamma, beta, mean, var, w2, b2);
        TrainerState st;
        st.lr = lr;
        for (std::uint64_t k = 0; k < K; ++k) {
            TensorBlock qb = block(q + k * n * d, n, d);
            Mat t = mat(targets + k * n * C, n, C);
            losses[k] = train_step_on_target(m, st, qb, t);
        }
        auto cp = [](const Mat& s, double* o) { std::copy(s.data.begin(), s.data.end(), o); };
        cp(m.w1, w1);
        cp(m.b1, b1);
        cp(m.bn_gamma, gamma);
        cp(m.bn_beta, beta);
        cp(m.bn_run_mean, mean);
        cp(m.bn_run_var, var);
        cp(m.w2, w2);
        cp(m.b2, b2);
    });
}

int ref_attention_target(const float* q, std::uint64_t n, std::uint64_t d, const float* keys,
                         std::uint64_t n_keys, const std::uint32_t* assignment, std::uint64_t C,
                         double* out) {
    return guard([&] {
        KeyAssignment a;
        a.bucket_of.assign(assignment, assignment + n_keys);
        Mat t = attention_target_rows(block(q, n, d), block(keys, n_keys, d), a, C);
        std::copy(t.data.begin(), t.data.end(), out);
    });
}
}  // extern "C"

// ---------------------------------------------------------------- accumulators
// PartialAccumulator state as flat arrays (out_acc [H x dv], sumexp, runmax),
// in/out, so tests can drive the reference and the device in lockstep.
namespace {
PartialAccumulator acc_from(std::uint64_t H, std::uint64_t dv, const double* out, const double* se,
                            const double* rm) {
    PartialAccumulator a(H, dv);
    std::copy(out, out + H * dv, a.out_acc.data.begin());
    std::copy(se, se + H, a.sumexp.begin());
    std::copy(rm, rm + H, a.runmax.begin());
    return a;
}
void acc_to(const PartialAccumulator& a, double* out, double* se, double* rm) {
    std::copy(a.out_acc.data.begin(), a.out_acc.data.end(), out);
    std::copy(a.sumexp.begin(), a.sumexp.end(), se);
    std::copy(a.runmax.begin(), a.runmax.end(), rm);
}
}  // namespace

extern "C" {
int ref_pattn_absorb_state(const float* q, std::uint64_t G, std::uint64_t d, const float* K,
                           const float* V, std::uint64_t n, std::uint64_t dv, const std::uint64_t* ids,
                           std::uint64_t count, std::uint64_t begin, std::uint64_t end, int range,
                           double* out, double* se, double* rm) {
    return guard([&] {
        PartialAccumulator a = acc_from(G, dv, out, se, rm);
        if (range) pattn_absorb_range(a, block(q, G, d), block(K, n, d), block(V, n, dv), begin, end);
        else pattn_absorb(a, block(q, G, d), block(K, n, d), block(V, n, dv),
                          std::span<const std::uint64_t>(ids, count));
        acc_to(a, out, se, rm);
    });
}

int ref_merge_state(std::uint64_t H, std::uint64_t dv, double* out, double* se, double* rm,
                    const double* pout, const double* pse, const double* prm) {
    return guard([&] {
        PartialAccumulator a = acc_from(H, dv, out, se, rm);
        merge_into(a, acc_from(H, dv, pout, pse, prm));
        acc_to(a, out, se, rm);
    });
}

int ref_finalize_state(std::uint64_t H, std::uint64_t dv, const double* out, const double* se,
                       const double* rm, float* res, int* any_empty) {
    return guard([&] {
        bool e = false;
        TensorBlock t = pattn_finalize(acc_from(H, dv, out, se, rm), &e);
        put(t, res);
        *any_empty = e ? 1 : 0;
    });
}
}  // extern "C"

extern "C" {
// build_context_store(keys_roped, values, rope, C, iters, sink, Rng(seed), &stats)
// (attention.cpp:238-246) -> trained centroids + the store's index
int ref_build_context_store_kmeans(const float* keys_roped, const float* values, std::uint64_t n,
                                   std::uint64_t d, double rope_base, std::uint64_t C,
                                   std::uint64_t iters, std::uint64_t sink, std::uint64_t seed,
                                   float* centroids, std::uint32_t* assignment, std::uint64_t* off,
                                   std::uint64_t* idx, double* objective) {
    return guard([&] {
        Rng rng(seed);
        KMeansStats st;
        ContextStore s = build_context_store(block(keys_roped, n, d), block(values, n, d),
                                             RopeConfig{d, rope_base}, C, iters, sink, rng, &st);
        put(s.partition.centroids, centroids);
        std::copy(s.assignment.bucket_of.begin(), s.assignment.bucket_of.end(), assignment);
        std::copy(s.index.off.begin(), s.index.off.end(), off);
        std::copy(s.index.idx.begin(), s.index.idx.end(), idx);
        std::copy(st.objective_per_iter.begin(), st.objective_per_iter.end(), objective);
    });
}
}  // extern "C"
