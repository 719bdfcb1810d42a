// Drop-in check of include/saap_b200.hpp: the reference's own C++ types
// (saap::TensorBlock, saap::Partition, saap::SparseAttnConfig, ...) flow
// unchanged into saap_b200:: calls, and every result is compared with the
// reference's saap:: implementation (oracle/_ref, test infrastructure).
// Exit code = number of failed checks (0 = pass).  Needs an sm_100 GPU.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "saap/attention.hpp"
#include "saap/experiments.hpp"
#include "saap/partition.hpp"
#include "saap/synthdata.hpp"
#include "saap_b200.hpp"

static int g_fail = 0;
static void check(bool ok, const std::string& what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++g_fail;
}

static float bf16(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
}
static void round_block(saap::TensorBlock& t) {
    for (float& v : t.data) v = bf16(v);
}
static double max_rel(const saap::TensorBlock& a, const saap::TensorBlock& b) {
    double w = 0;
    for (size_t i = 0; i < a.data.size(); ++i)
        w = std::max(w, std::abs((double)a.data[i] - b.data[i]) / std::max(std::abs((double)b.data[i]), 1e-3));
    return w;
}
static saap::TensorBlock rows(const saap::TensorBlock& t, size_t lo, size_t hi) {
    saap::TensorBlock o(hi - lo, t.dim);
    std::memcpy(o.data.data(), t.row(lo), (hi - lo) * t.dim * 4);
    return o;
}

int main() {
    saap::HeadSpec spec;
    spec.dim = 128;
    spec.seed = 3;
    spec.drift_rate = 0.0;
    const size_t n = 8192, C = 256;
    saap::SyntheticPrompt p = saap::generate_prompt(spec, n, 8, 0);
    round_block(p.keys_roped);
    round_block(p.values);
    round_block(p.keys_deroped);
    round_block(p.queries_roped);
    round_block(p.queries_deroped);
    saap::Partition part = saap::train_head_partition(spec, 4096, C, 3, 1);

    // assign_keys / build_ivf
    saap::TensorBlock kd = rows(p.keys_deroped, 1, n);
    saap::KeyAssignment ra = saap::assign_keys(kd, part);
    auto ga = saap_b200::assign_keys(kd, part);
    check(ga.bucket_of == ra.bucket_of, "assign_keys bit-exact");
    saap::IVFIndex ri = saap::build_ivf(ra, C);
    auto gi = saap_b200::build_ivf(ra, C);
    check(gi.off == ri.off && gi.idx == ri.idx, "build_ivf bit-exact");

    // ContextStore (reference built field by field on the same pre-RoPE keys)
    saap::ContextStore ref;
    ref.keys = p.keys_roped;
    ref.values = p.values;
    ref.id_offset = 1;
    ref.partition = part;
    ref.assignment = ra;
    ref.index = ri;
    saap_b200::ContextStore ours(p.keys_roped, p.values, spec.rope_base, part, 1, &p.keys_deroped);
    check(ours.assignment().bucket_of == ra.bucket_of && ours.index().idx == ri.idx,
          "ContextStore index bit-exact");

    saap::CentroidRouter rr(part, true);
    saap_b200::CentroidRouter gr(part, true);
    saap::TensorBlock qr = rows(p.queries_roped, 0, 4), qd = rows(p.queries_deroped, 0, 4);
    check(gr.select(qr, qd, 16) == rr.select(qr, qd, 16), "CentroidRouter::select bit-exact");

    const size_t cfgs[][2] = {{16, 2047}, {32, 2047}, {0, 2047}, {8, 500}, {8, 3000}, {4, 100000}};
    for (auto& c : cfgs) {
        saap::SparseAttnConfig cfg;
        cfg.probes = c[0];
        cfg.dense = saap::DenseWindow{1, c[1]};
        saap::AttnResult r1 = saap::sparse_attention(qr, qd, ref, rr, cfg);
        saap_b200::AttnResult r2 = saap_b200::sparse_attention(qr, qd, ours, gr, cfg);
        saap::TensorBlock o2(r2.output.rows, r2.output.dim);
        o2.data = r2.output.data;
        const double e = max_rel(o2, r1.output);
        check(r1.keys_scored == r2.keys_scored && r1.max_visited_bucket == r2.max_visited_bucket &&
                      r1.empty_attention == r2.empty_attention && e <= 1e-3,
              "sparse_attention probes=" + std::to_string(c[0]) + " recent=" + std::to_string(c[1]) +
                      " max_rel=" + std::to_string(e));
    }
    saap::TensorBlock f1 = saap::full_attention(qr, p.keys_roped, p.values);
    saap_b200::TensorBlock f2 = saap_b200::full_attention(qr, p.keys_roped, p.values);
    saap::TensorBlock f2r(f2.rows, f2.dim);
    f2r.data = f2.data;
    check(max_rel(f2r, f1) <= 1e-3, "full_attention");
    try {
        saap::SparseAttnConfig bad;
        bad.probes = C + 1;
        saap_b200::sparse_attention(qr, qd, ours, gr, bad);
        check(false, "probes > C throws");
    } catch (const std::invalid_argument& e) {
        check(std::string(e.what()).rfind("sparse_attention: probes", 0) == 0, "probes > C throws invalid_argument");
    }
    // kmeans_train with the reference's own Rng and KMeansStats types
    {
        saap::TensorBlock tk = rows(p.keys_deroped, 1, 4097);
        saap::Rng r1 = saap::Rng(spec.seed).child(2ull << 32), r2 = r1;
        saap::KMeansStats s1, s2;
        saap::Partition k1 = saap::kmeans_train(tk, 64, 4, r1, &s1);
        auto k2 = saap_b200::kmeans_train(tk, 64, 4, r2, &s2);
        check(std::memcmp(k1.centroids.data.data(), k2.centroids.data.data(),
                          k1.centroids.data.size() * 4) == 0 &&
                      s1.objective_per_iter == s2.objective_per_iter &&
                      s1.empty_cluster_repairs == s2.empty_cluster_repairs &&
                      r1.next_u64() == r2.next_u64(),
              "kmeans_train bit-exact (saap::Rng, saap::KMeansStats)");
        try {
            saap::Rng r3(14);
            saap_b200::kmeans_train(rows(tk, 0, 3), 4, 10, r3);
            check(false, "kmeans_train throws with too few keys");
        } catch (const std::invalid_argument& e) {
            check(std::string(e.what()) == "kmeans_train: 3 keys cannot seed 4 buckets",
                  "kmeans_train too few keys message");
        }
    }
    // attention_over_ids: fp64 on the device, bit-exact with the reference
    {
        std::vector<std::uint64_t> ids;
        for (std::uint64_t i = 0; i < 700; ++i) ids.push_back((i * 7919) % n);
        bool e1 = false, e2 = false;
        saap::TensorBlock a1 = saap::attention_over_ids(qr, p.keys_roped, p.values, ids, &e1);
        saap_b200::TensorBlock a2 = saap_b200::attention_over_ids(qr, p.keys_roped, p.values, ids, &e2);
        check(e1 == e2 && std::memcmp(a1.data.data(), a2.data.data(), a1.data.size() * 4) == 0,
              "attention_over_ids bit-exact");
    }
    std::printf("%d failed\n", g_fail);
    return g_fail;
}
