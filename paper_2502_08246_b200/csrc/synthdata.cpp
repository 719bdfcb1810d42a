// synthdata.cpp — the reference's synthetic head generator (the benchmark
// input contract) as host C++ in the library, so bench and
// serving-style callers get the reference's exact inputs without linking
// the reference:
//
//   Rng                       tensor.cpp:92-159   (splitmix64, Box-Muller)
//   build_basis & helpers     synthdata.cpp:33-131
//   generate_prompt           synthdata.cpp:169-281
//   rope_apply_block          rope.cpp:20-41, 59-90
//   train_head_partition      experiments.cpp:284-295 (+ the device k-means)
//
// Bit-exactness: the same operation order as the reference, compiled
// without FP contraction against the same glibc libm (tests/test_synth.py
// compares every output word with the compiled reference).  The per-row
// random draws are fixed (one `below` + dim normals per key row, dim normals
// per value row), and splitmix64 is a counter, so rows are generated in
// parallel by jumping the counter; any variable-length draw (a rejected
// `below` or a zero uniform in Box-Muller, probability ~2^-53 per draw) is
// detected and the whole pass is redone sequentially.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "saap_b200.h"

namespace saap_b200 {
void set_error(const std::string& m);  // capi.cu: saap_last_error's thread-local text
}

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kStructureStream = 0;   // synthdata.cpp:17
constexpr uint64_t kPromptStreamBase = 1;  // synthdata.cpp:18
constexpr uint64_t kPartitionPromptSeed = uint64_t{1} << 20;  // experiments.cpp:21
constexpr uint64_t kKmeansStream = uint64_t{2} << 32;         // experiments.cpp:23
constexpr double kTwoPi = 2.0 * 3.141592653589793238462643383279502884;

struct Rng {  // tensor.cpp:92-159
    uint64_t seed, state;
    bool has_spare = false;
    double spare = 0.0;
    uint64_t draws = 0;  // next_u64 calls (for the parallel skip-ahead check)

    explicit Rng(uint64_t s) : seed(s), state(s) {}
    uint64_t next_u64() {
        ++draws;
        uint64_t z = (state += kGolden);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double normal() {
        if (has_spare) {
            has_spare = false;
            return spare;
        }
        double u1 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        double u2 = uniform();
        double r = std::sqrt(-2.0 * std::log(u1));
        double t = kTwoPi * u2;
        spare = r * std::sin(t);
        has_spare = true;
        return r * std::cos(t);
    }
    uint64_t below(uint64_t n) {
        if (n == 0) throw std::invalid_argument("Rng::below: n must be >= 1");
        const uint64_t threshold = (0 - n) % n;
        for (;;) {
            const uint64_t r = next_u64();
            if (r >= threshold) return r % n;
        }
    }
    Rng child(uint64_t stream) const {
        Rng mixer(seed ^ (0xD1342543DE82EF95ull * (stream + 1)));
        return Rng(mixer.next_u64());
    }
    std::vector<uint64_t> sample_without_replacement(uint64_t n, uint64_t m) {
        if (m > n) throw std::invalid_argument("sample_without_replacement: m > n");
        std::vector<uint64_t> out;
        out.reserve(m);
        std::vector<bool> taken(n, false);
        for (uint64_t j = n - m; j < n; ++j) {
            uint64_t t = below(j + 1);
            if (taken[t]) t = j;
            taken[t] = true;
            out.push_back(t);
        }
        std::sort(out.begin(), out.end());
        return out;
    }
    void shuffle(std::vector<uint64_t>& v) {
        for (size_t i = v.size(); i > 1; --i) {
            const size_t j = static_cast<size_t>(below(i));
            std::swap(v[i - 1], v[j]);
        }
    }
    // the generator `k` draws ahead of this one (fresh Box-Muller state)
    Rng ahead(uint64_t k) const {
        Rng r(seed);
        r.state = state + k * kGolden;
        return r;
    }
};

struct HeadBasis {  // synthdata.cpp:21-31
    std::vector<float> m;
    std::vector<std::vector<float>> codes, beacons, centers;
    std::vector<float> drift_dir, shift_dir;
    size_t mid_lo = 0, stable_lo = 0;
};

std::vector<float> unit_in_range(Rng& rng, size_t dim, size_t lo, size_t hi) {  // :33-49
    std::vector<float> v(dim, 0.0f);
    double norm = 0.0;
    while (norm == 0.0) {
        norm = 0.0;
        for (size_t j = lo; j < hi; ++j) {
            double x = rng.normal();
            v[j] = static_cast<float>(x);
            norm += x * x;
        }
        norm = std::sqrt(norm);
    }
    for (size_t j = lo; j < hi; ++j) v[j] = static_cast<float>(v[j] / norm);
    return v;
}

std::vector<std::vector<float>> orthonormal_set(Rng& rng, size_t dim, size_t lo, size_t hi,
                                                size_t count) {  // :53-91
    std::vector<std::vector<double>> basis;
    basis.reserve(count);
    while (basis.size() < count) {
        std::vector<double> v(hi - lo);
        for (double& x : v) x = rng.normal();
        for (const auto& b : basis) {
            double dot = 0.0;
            for (size_t j = 0; j < v.size(); ++j) dot += v[j] * b[j];
            for (size_t j = 0; j < v.size(); ++j) v[j] -= dot * b[j];
        }
        double norm = 0.0;
        for (double x : v) norm += x * x;
        norm = std::sqrt(norm);
        if (norm < 1e-6) continue;
        for (double& x : v) x /= norm;
        basis.push_back(std::move(v));
    }
    std::vector<std::vector<float>> out(count, std::vector<float>(dim, 0.0f));
    for (size_t i = 0; i < count; ++i)
        for (size_t j = 0; j < hi - lo; ++j) out[i][lo + j] = static_cast<float>(basis[i][j]);
    return out;
}

HeadBasis build_basis(const saap_head_spec& sp) {  // :93-112
    Rng rng = Rng(sp.seed).child(kStructureStream);
    HeadBasis b;
    const size_t dim = (size_t)sp.dim;
    b.stable_lo = dim - 2 * (size_t)sp.lowfreq_pairs;
    b.mid_lo = dim / 2;
    auto stable = orthonormal_set(rng, dim, b.stable_lo, dim, 1 + sp.n_clusters + sp.n_targets);
    b.m = std::move(stable[0]);
    b.codes.assign(stable.begin() + 1, stable.begin() + 1 + (ptrdiff_t)sp.n_clusters);
    b.beacons.assign(stable.begin() + 1 + (ptrdiff_t)sp.n_clusters, stable.end());
    for (size_t z = 0; z < sp.n_clusters; ++z) b.centers.push_back(unit_in_range(rng, dim, 0, b.stable_lo));
    b.drift_dir = unit_in_range(rng, dim, 0, b.stable_lo);
    b.shift_dir = unit_in_range(rng, dim, 0, b.stable_lo);
    return b;
}

inline void add_scaled(float* row, const std::vector<float>& dir, double scale) {  // :114-118
    for (size_t j = 0; j < dir.size(); ++j) row[j] += static_cast<float>(scale * dir[j]);
}

void base_query_row(const saap_head_spec& sp, const HeadBasis& basis, Rng& rng, double shift,
                    float* row) {  // :120-131
    const size_t y = static_cast<size_t>(rng.below(sp.n_clusters));
    add_scaled(row, basis.m, -sp.query_offset);
    add_scaled(row, basis.centers[y], sp.query_pull);
    if (shift != 0.0) add_scaled(row, basis.shift_dir, shift);
    for (size_t j = 0; j < sp.dim; ++j) row[j] += static_cast<float>(sp.query_noise * rng.normal());
}

void validate(const saap_head_spec& s) {  // synthdata.cpp:135-167
    auto bad = [](const std::string& m) { throw std::invalid_argument(m); };
    if (s.dim < 8 || s.dim % 2 != 0) bad("HeadSpec: dim must be even and >= 8");
    if (s.lowfreq_pairs < 1 || 4 * s.lowfreq_pairs > s.dim) bad("HeadSpec: lowfreq_pairs must be in [1, dim/4]");
    if (s.n_clusters < 1) bad("HeadSpec: need at least one cluster");
    if (1 + s.n_clusters + s.n_targets > 2 * s.lowfreq_pairs)
        bad("HeadSpec: stable pairs cannot hold " + std::to_string(s.n_clusters) + " cluster codes + " +
            std::to_string(s.n_targets) + " target beacons; raise lowfreq_pairs or shrink them");
    if (s.planted_longrange_fraction < 0.0 || s.planted_longrange_fraction > 1.0)
        bad("HeadSpec: planted_longrange_fraction outside [0,1]");
    if (s.planted_longrange_fraction > 0.0 && s.n_targets < 1) bad("HeadSpec: planting requires n_targets >= 1");
    if (s.key_noise < 0 || s.stable_noise < 0 || s.query_noise < 0 || s.key_center_scale < 0 ||
        s.sink_norm < 0 || s.drift_rate < 0)
        bad("HeadSpec: scales must be nonnegative");
    if (s.local_range < 1) bad("HeadSpec: local_range must be >= 1");
    if (s.rope_base <= 1.0) bad("HeadSpec: rope_base must exceed 1");
}

std::vector<double> pair_frequencies(size_t dim, double base) {  // rope.cpp:20-27
    std::vector<double> th(dim / 2);
    const double inv_dim = 1.0 / static_cast<double>(dim);
    for (size_t j = 0; j < th.size(); ++j) th[j] = std::pow(base, -2.0 * static_cast<double>(j) * inv_dim);
    return th;
}

// rope.cpp:29-41 with sign = +1 (rope_apply)
void rotate_with(float* x, uint64_t position, const std::vector<double>& thetas) {
    const double p = static_cast<double>(position);
    for (size_t j = 0; j < thetas.size(); ++j) {
        double angle = 1.0 * p * thetas[j];
        double c = std::cos(angle);
        double s = std::sin(angle);
        double x0 = x[2 * j];
        double x1 = x[2 * j + 1];
        x[2 * j] = static_cast<float>(x0 * c - x1 * s);
        x[2 * j + 1] = static_cast<float>(x0 * s + x1 * c);
    }
}

inline uint16_t bf16_rne(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

// one output block: f32 or bf16 (RNE), row-major [rows x d]; null = not wanted
struct Sink {
    void* p;
    int bf16;
    size_t d;
    void put(size_t row, const float* v) const {
        if (!p) return;
        if (bf16) {
            uint16_t* o = static_cast<uint16_t*>(p) + row * d;
            for (size_t j = 0; j < d; ++j) o[j] = bf16_rne(v[j]);
        } else {
            std::memcpy(static_cast<float*>(p) + row * d, v, d * 4);
        }
    }
};

template <typename F>
void parallel_rows(size_t begin, size_t end, int threads, F&& f) {
    const size_t n = end > begin ? end - begin : 0;
    const size_t T = std::max<size_t>(1, std::min<size_t>((size_t)threads, n / 256 + 1));
    if (T == 1) {
        f(begin, end);
        return;
    }
    std::vector<std::thread> ts;
    const size_t per = (n + T - 1) / T;
    for (size_t t = 0; t < T; ++t) {
        const size_t a = begin + t * per, b = std::min(end, a + per);
        if (a < b) ts.emplace_back([&f, a, b] { f(a, b); });
    }
    for (auto& t : ts) t.join();
}

struct Outputs {
    Sink kd, kr, v, qd, qr;
    int64_t* planted;
};

// generate_prompt (synthdata.cpp:169-281)
void generate(const saap_head_spec& sp, size_t n_keys, size_t n_q, uint64_t prompt_seed,
              const Outputs& out, int threads) {
    validate(sp);
    if (n_q < 1) throw std::invalid_argument("generate_prompt: need at least one query");
    if (n_keys < n_q + sp.local_range + 2)
        throw std::invalid_argument("generate_prompt: context of " + std::to_string(n_keys) +
                                    " keys cannot host " + std::to_string(n_q) +
                                    " queries with local range " + std::to_string(sp.local_range));
    const bool plant = sp.planted_longrange_fraction > 0.0;
    size_t target_hi = 0;
    if (plant) {
        const size_t guard_hi = n_keys > sp.window_guard ? n_keys - sp.window_guard : 0;
        const size_t gap_needed = n_q + sp.longrange_threshold;
        const size_t gap_hi = n_keys > gap_needed ? n_keys - gap_needed : 0;
        target_hi = std::min(guard_hi, gap_hi);
        if (target_hi < 1 + sp.n_targets)
            throw std::invalid_argument("generate_prompt: context too short to plant " +
                                        std::to_string(sp.n_targets) + " long-range targets beyond gap " +
                                        std::to_string(sp.longrange_threshold));
    }
    const size_t d = (size_t)sp.dim;
    const HeadBasis basis = build_basis(sp);
    const std::vector<double> thetas = pair_frequencies(d, sp.rope_base);
    Rng rng = Rng(sp.seed).child(kPromptStreamBase + prompt_seed);

    std::vector<uint64_t> target_ids;
    std::vector<size_t> target_of_key;  // (key id, slot) pairs, few
    if (plant) {
        target_ids = rng.sample_without_replacement(target_hi - 1, sp.n_targets);
        for (auto& t : target_ids) t += 1;  // never the sink
    }
    auto target_slot = [&](size_t i) -> size_t {
        for (size_t t = 0; t < target_ids.size(); ++t)
            if (target_ids[t] == i) return t;  // later duplicates cannot occur (distinct ids)
        return SIZE_MAX;
    };

    // rows the query pass reads back (local lookups point <= local_range back)
    const size_t tail0 = n_keys - n_q - std::min<size_t>(n_keys - n_q, sp.local_range);
    std::vector<float> tail((n_keys - tail0) * d);
    std::vector<uint32_t> cluster_of_target(target_ids.size(), 0);

    // key row i >= 1 draws below(n_clusters) + d normals; d is even, so the
    // Box-Muller spare never crosses a row
    const uint64_t per_key = 1 + d;
    auto key_rows = [&](Rng& r, size_t a, size_t b) {
        std::vector<float> row(d), rr(d);
        for (size_t i = a; i < b; ++i) {
            std::fill(row.begin(), row.end(), 0.0f);
            if (i == 0) {
                add_scaled(row.data(), basis.m, -sp.sink_norm);
            } else {
                const size_t z = static_cast<size_t>(r.below(sp.n_clusters));
                add_scaled(row.data(), basis.m, sp.key_offset);
                add_scaled(row.data(), basis.centers[z], sp.key_center_scale);
                add_scaled(row.data(), basis.codes[z], sp.cluster_code_scale);
                if (sp.drift_rate > 0.0)
                    add_scaled(row.data(), basis.drift_dir, sp.drift_rate * static_cast<double>(i));
                for (size_t j = 0; j < basis.stable_lo; ++j)
                    row[j] += static_cast<float>(sp.key_noise * r.normal());
                for (size_t j = basis.stable_lo; j < d; ++j)
                    row[j] += static_cast<float>(sp.stable_noise * r.normal());
                const size_t ts = plant ? target_slot(i) : SIZE_MAX;
                if (ts != SIZE_MAX) {
                    add_scaled(row.data(), basis.beacons[ts], sp.target_beacon);
                    cluster_of_target[ts] = (uint32_t)z;
                }
            }
            out.kd.put(i, row.data());
            if (i >= tail0) std::memcpy(&tail[(i - tail0) * d], row.data(), d * 4);
            if (out.kr.p) {
                rr = row;
                rotate_with(rr.data(), i, thetas);  // key_positions[i] = i
                out.kr.put(i, rr.data());
            }
        }
    };
    const Rng keys0 = rng;
    bool exact = true;
    if (threads > 1 && n_keys > 1) {
        std::vector<uint64_t> used(n_keys, 0);
        parallel_rows(0, n_keys, threads, [&](size_t a, size_t b) {
            Rng r = keys0.ahead(a == 0 ? 0 : (a - 1) * per_key);
            key_rows(r, a, b);
            used[a] = r.draws;
        });
        uint64_t total = 0;
        for (uint64_t u : used) total += u;
        exact = total == (n_keys - 1) * per_key;
    }
    if (threads <= 1 || n_keys <= 1 || !exact) {
        rng = keys0;
        key_rows(rng, 0, n_keys);
    } else {
        rng = keys0.ahead((n_keys - 1) * per_key);
    }

    // values: rng.fill_normal(values), n*d normals, d per row
    const Rng vals0 = rng;
    auto value_rows = [&](Rng& r, size_t a, size_t b) {
        std::vector<float> row(d);
        for (size_t i = a; i < b; ++i) {
            for (size_t j = 0; j < d; ++j) row[j] = static_cast<float>(r.normal() * 1.0);
            out.v.put(i, row.data());
        }
    };
    exact = true;
    if (threads > 1) {
        std::vector<uint64_t> used(n_keys, 0);
        parallel_rows(0, n_keys, threads, [&](size_t a, size_t b) {
            Rng r = vals0.ahead(a * d);
            value_rows(r, a, b);
            used[a] = r.draws;
        });
        uint64_t total = 0;
        for (uint64_t u : used) total += u;
        exact = total == n_keys * d;
    }
    if (threads <= 1 || !exact) {
        rng = vals0;
        value_rows(rng, 0, n_keys);
    } else {
        rng = vals0.ahead(n_keys * d);
    }

    // queries (sequential; few rows)
    const double inv_sqrt2 = 1.0 / std::sqrt(2.0);
    std::vector<float> row(d), rr(d);
    for (size_t qi = 0; qi < n_q; ++qi) {
        const size_t pos = n_keys - n_q + qi;
        std::fill(row.begin(), row.end(), 0.0f);
        base_query_row(sp, basis, rng, sp.ood_shift, row.data());
        int64_t planted = -1;
        if (plant && rng.uniform() < sp.planted_longrange_fraction) {
            const size_t t = static_cast<size_t>(rng.below(sp.n_targets));
            const uint64_t tid = target_ids[t];
            add_scaled(row.data(), basis.codes[cluster_of_target[t]], sp.query_boost * inv_sqrt2);
            add_scaled(row.data(), basis.beacons[t], sp.query_boost * inv_sqrt2);
            planted = (int64_t)tid;
        } else {
            const size_t gap = 1 + static_cast<size_t>(rng.below(sp.local_range));
            const float* target_row = &tail[(pos - gap - tail0) * d];
            double norm = 0.0;
            for (size_t j = basis.mid_lo; j < basis.stable_lo; ++j)
                norm += static_cast<double>(target_row[j]) * target_row[j];
            norm = std::sqrt(norm);
            if (norm > 0.0) {
                const double scale = sp.local_boost / norm;
                for (size_t j = basis.mid_lo; j < basis.stable_lo; ++j)
                    row[j] += static_cast<float>(scale * target_row[j]);
            }
        }
        if (out.planted) out.planted[qi] = planted;
        out.qd.put(qi, row.data());
        rr = row;
        rotate_with(rr.data(), pos, thetas);
        out.qr.put(qi, rr.data());
    }
}

struct Passthrough {  // an error already recorded by another entry point
    int code;
};

template <typename F>
int synth_guard(F&& f) {
    try {
        f();
        return SAAP_OK;
    } catch (const Passthrough& e) {
        return e.code;
    } catch (const std::invalid_argument& e) {
        saap_b200::set_error(e.what());
        return SAAP_ERR_INVALID_ARGUMENT;
    } catch (const std::bad_alloc&) {
        saap_b200::set_error("host allocation failed");
        return SAAP_ERR_RUNTIME;
    } catch (const std::exception& e) {
        saap_b200::set_error(e.what());
        return SAAP_ERR_RUNTIME;
    }
}

int default_threads(int t) {
    if (t > 0) return t;
    const unsigned h = std::thread::hardware_concurrency();
    return h ? (int)h : 1;
}

}  // namespace

extern "C" {

void saap_head_spec_default(saap_head_spec* s) {
    // synthdata.hpp:24-56
    s->dim = 64;
    s->n_clusters = 8;
    s->key_offset = 3.0;
    s->query_offset = 3.0;
    s->key_center_scale = 4.0;
    s->cluster_code_scale = 1.0;
    s->key_noise = 1.0;
    s->stable_noise = 0.05;
    s->sink_norm = 8.0;
    s->drift_rate = 5e-4;
    s->query_noise = 0.3;
    s->query_pull = 4.0;
    s->query_boost = 140.0;
    s->local_boost = 0.0;
    s->target_beacon = 1.0;
    s->ood_shift = 0.0;
    s->planted_longrange_fraction = 0.25;
    s->n_targets = 4;
    s->local_range = 64;
    s->longrange_threshold = 1024;
    s->window_guard = 2112;
    s->lowfreq_pairs = 8;
    s->rope_base = 500000.0;
    s->seed = 1;
}

int saap_generate_prompt(const saap_head_spec* spec, uint64_t n_keys, uint64_t n_q,
                         uint64_t prompt_seed, int out_bf16, void* keys_deroped, void* keys_roped,
                         void* values, float* q_deroped, float* q_roped, int64_t* planted_target,
                         int threads) {
    return synth_guard([&] {
        if (!spec) throw std::invalid_argument("generate_prompt: null spec");
        const size_t d = (size_t)spec->dim;
        Outputs o{{keys_deroped, out_bf16, d}, {keys_roped, out_bf16, d}, {values, out_bf16, d},
                  {q_deroped, 0, d}, {q_roped, 0, d}, planted_target};
        generate(*spec, (size_t)n_keys, (size_t)n_q, prompt_seed, o, default_threads(threads));
    });
}

int saap_train_head_partition(saap_ctx* ctx, const saap_head_spec* spec, uint64_t n_keys,
                              uint64_t n_buckets, uint64_t iters, uint64_t sink_count,
                              float* centroids, int threads) {
    return synth_guard([&] {
        if (!spec) throw std::invalid_argument("train_head_partition: null spec");
        const size_t d = (size_t)spec->dim;
        std::vector<float> kd(std::max<uint64_t>(n_keys, 1) * d);
        Outputs o{{kd.data(), 0, d}, {nullptr, 0, d}, {nullptr, 0, d}, {nullptr, 0, d},
                  {nullptr, 0, d}, nullptr};
        // experiments.cpp:288: only the keys matter (one query)
        generate(*spec, (size_t)n_keys, 1, kPartitionPromptSeed, o, default_threads(threads));
        if (n_keys <= sink_count)
            throw std::invalid_argument("train_head_partition: no keys beyond the sink span");
        const uint64_t n = n_keys - sink_count;
        if (n_buckets < 1) throw std::invalid_argument("kmeans_train: need at least 1 bucket");
        if (n < n_buckets)
            throw std::invalid_argument("kmeans_train: " + std::to_string(n) + " keys cannot seed " +
                                        std::to_string(n_buckets) + " buckets");
        // kmeans_train's seed draws (partition.cpp:80-82) from Rng(seed).child(kKmeansStream)
        Rng rng = Rng(spec->seed).child(kKmeansStream);
        std::vector<uint64_t> seeds = rng.sample_without_replacement(n, n_buckets);
        rng.shuffle(seeds);
        const int krc = saap_kmeans_train(ctx, kd.data() + sink_count * d, n, d, n_buckets, iters,
                                          seeds.data(), centroids, nullptr, nullptr, nullptr);
        if (krc != SAAP_OK) throw Passthrough{krc};
    });
}

}  // extern "C"
