// C ABI of libsaap_b200: host orchestration of the sm_100a kernels behind the
// reference's C++ API (see include/saap_b200.h for the interface map).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "api.cuh"
#include "args.cuh"

namespace saap_b200 {

// ---- kernels (decode.cu / pack.cu / route.cu / synth.cu)
void launch_route_plan(const PlanArgs& a, uint32_t n_groups, bool pdl, cudaStream_t st);
void launch_route_cluster(int D, const ClusterRouteArgs& a, uint32_t n_slots, cudaStream_t st);
bool route_cluster_supported(int D, uint32_t C);
void launch_route_approx(int D, const ApproxArgs& a, uint32_t n_slots, cudaStream_t st);
void launch_route_score(const RouteArgs& a, uint32_t n_groups, cudaStream_t st);
void launch_decode(int D, const DecodeMaps& m, const DecodeArgs& a, int grid, cudaStream_t st, bool tc);
void launch_combine(int D, const CombineArgs& ca, uint32_t n_qslots, cudaStream_t st);
void p2p_fill(saap_ctx* c, CombineArgs& ca);
void launch_qmodel_probs(const QModelArgs& a, uint32_t n_groups, cudaStream_t st, uint32_t n_slots = 0);
void launch_assign_exact(int D, bool bf16_keys, const TileDesc* tiles, uint32_t n_tiles,
                         const void* keys, const uint64_t* key_row0, const double* const* cent64,
                         uint32_t C, uint32_t* out, const uint64_t* out_base, cudaStream_t st,
                         uint32_t max_tile_count = 1u << 31);
void launch_append_off(const GroupMeta* meta, uint32_t n_groups, const uint32_t* assign, uint32_t k,
                       uint32_t C, uint32_t* off, cudaStream_t st);
void launch_pack(int D, const TileDesc* tiles, uint32_t n_tiles, const uint32_t* tile_first,
                 uint32_t n_groups, const GroupMeta* meta, const uint32_t* assign, uint32_t C,
                 uint32_t* hist, uint32_t* countA, uint32_t* off, uint32_t* offA, uint32_t* idx,
                 uint32_t* invA, uint32_t* posA, uint32_t* dst_row, uint64_t total_ns,
                 const uint16_t* Ksrc, const uint16_t* Vsrc, const uint64_t* src_row0,
                 uint16_t* Kdst, uint16_t* Vdst, cudaStream_t st);
void launch_coverage(const GroupMeta* meta, uint32_t n_groups, const uint16_t* K,
                     const uint32_t* posA, const uint32_t* assign, const float* q, uint32_t G,
                     uint32_t D, const uint32_t* sel, uint32_t l, uint32_t C, uint32_t recent,
                     double* out, cudaStream_t st);
void launch_f32_to_bf16(const float* in, uint16_t* out, uint64_t n, cudaStream_t st);
void launch_derope(const float* x, const double* cs, uint64_t rows, uint32_t D, float* out,
                   cudaStream_t st);
void launch_debug_exp(const double* x, uint64_t n, double* y, cudaStream_t st);
uint32_t km_dim_max(uint32_t D);
void launch_acc_init(double* out, double* sumexp, double* runmax, uint32_t H, uint32_t dv,
                     cudaStream_t st);
void launch_acc_absorb(const float* q, uint32_t H, uint32_t d, const float* K, const float* V,
                       uint32_t n, uint32_t dv, double scale, double* S, double* rescale,
                       double* out, double* sumexp, double* runmax, cudaStream_t st);
void launch_acc_merge(double* out, double* sumexp, double* runmax, const double* p_out,
                      const double* p_sumexp, const double* p_runmax, uint32_t H, uint32_t dv,
                      cudaStream_t st);
void launch_acc_finalize(const double* out_acc, const double* sumexp, uint32_t H, uint32_t dv,
                         float* out, int* any_empty, cudaStream_t st);
void launch_append_rows(int D, const GroupMeta* meta, uint32_t n_groups, uint32_t k,
                        const uint16_t* Ksrc, const uint16_t* Vsrc, uint16_t* Kdst, uint16_t* Vdst,
                        cudaStream_t st);
void qtrain_forward(saap_qtrainer* t, uint32_t n, cudaStream_t st);
void qtrain_update(saap_qtrainer* t, uint32_t n, cudaStream_t st);
void launch_attention_target(const float* q, uint32_t n, uint32_t d, const float* K,
                             uint32_t n_keys, const uint32_t* assign, uint32_t C, double* a,
                             double* out, cudaStream_t st);
void launch_km_assign(const float* keys, uint32_t n, uint32_t D, const float* cent, uint32_t C,
                      uint32_t* assign, double* score, unsigned long long* zero_keys,
                      cudaStream_t st);
void launch_km_iteration_tail(const float* keys, uint32_t n, uint32_t D, uint32_t* assign,
                              double* score, uint32_t* counts, uint32_t C,
                              unsigned long long* repairs, cudaStream_t st);
void launch_km_objective(const double* score, uint32_t n, double* out, cudaStream_t st);
void launch_km_seed(const float* keys, uint32_t D, const uint64_t* seed_rows, uint32_t C,
                    float* cent, cudaStream_t st);
void launch_km_update(const float* keys, uint32_t D, const uint32_t* off, const uint32_t* idx,
                      uint32_t C, float* cent, cudaStream_t st);
uint32_t tc_cpad(uint32_t C);
void launch_split_centroids(const float* cent, uint32_t C, uint32_t D, uint16_t* hi, uint16_t* mid,
                            cudaStream_t st);
void build_tc_tiles(const std::vector<GroupMeta>& meta, const std::vector<uint32_t>& part_slot,
                    std::vector<TcTile>& tiles, bool split);
void launch_assign_tc(const uint16_t* keys, uint64_t key_rows, const uint16_t* hi,
                      const uint16_t* mid, uint32_t n_parts, const TcAssignArgs& args,
                      uint32_t n_tiles, cudaStream_t st, const uint16_t* keys_lo);
void launch_refine(const uint32_t* list, const uint32_t* count, const void* keys,
                   const uint64_t* key_row0, const double* const* cent64, const uint64_t* out_base,
                   uint32_t C, uint32_t* out, uint32_t n_groups, int sm_count, cudaStream_t st,
                   bool f32_keys);
void launch_split_rows(const float* x, uint64_t n, uint16_t* hi, uint16_t* lo, cudaStream_t st);
void launch_synth(uint16_t* out, uint64_t rows, uint32_t D, uint64_t seed, int kind,
                  const float* centers, uint64_t n_centers, float center_scale, float noise,
                  cudaStream_t st);

}  // namespace saap_b200


using namespace saap_b200;

namespace {

template <typename T>
T* dmalloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    SAAP_CUDA(cudaMalloc(&p, count * sizeof(T)));
    return static_cast<T*>(p);
}
template <typename T>
void dfree(T*& p) {
    if (p) cudaFree((void*)p);
    p = nullptr;
}

void* ensure(saap_ctx* c, saap_scratch& s, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (bytes <= s.cap) return s.p;
    if (c->capturing)
        throw Failure{SAAP_ERR_INVALID_ARGUMENT,
                      "scratch grows during graph capture: run the call once uncaptured first"};
    if (s.p) {
        SAAP_CUDA(cudaStreamSynchronize(c->stream));
        cudaFree(s.p);
        s.p = nullptr;
        s.cap = 0;
    }
    const size_t cap = std::max<size_t>(bytes, 4096) * 5 / 4;
    SAAP_CUDA(cudaMalloc(&s.p, cap));
    s.cap = cap;
    c->scratch_gen++;
    return s.p;
}


// scratch whose contents must start at zero (per-slot step counters)
void* ensure_zero(saap_ctx* c, saap_scratch& s, size_t bytes) {
    if (bytes <= s.cap) return s.p;
    void* p = ensure(c, s, bytes);
    SAAP_CUDA(cudaMemset(p, 0, s.cap));
    return p;
}


// live contexts, so destroying a layer / router retires every cached host graph
// that references it
std::vector<saap_ctx*>& live_contexts() {
    static std::vector<saap_ctx*> v;
    return v;
}
void purge_host_graphs(saap_ctx* c, const void* layer, const void* router) {
    auto& hg = c->host_graphs;
    for (size_t i = 0; i < hg.size();) {
        bool hit = (layer && hg[i].layer == layer);
        for (const void* r : hg[i].routers) hit |= (router && r == router);
        if (hit) {
            if (hg[i].exec) cudaGraphExecDestroy(hg[i].exec);
            hg.erase(hg.begin() + i);
        } else {
            ++i;
        }
    }
}

void h2d(void* d, const void* h, size_t bytes, cudaStream_t st) {
    if (bytes) SAAP_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
}
void d2h(void* h, const void* d, size_t bytes, cudaStream_t st) {
    if (bytes) SAAP_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st));
}
void sync(saap_ctx* c) { SAAP_CUDA(cudaStreamSynchronize(c->stream)); }

uint32_t next_pow2(uint32_t x) {
    uint32_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

bool supported_dim(uint64_t d) { return d == 32 || d == 64 || d == 128; }

// glibc-exact RoPE removal table: (cos, sin) of (-1.0 * p) * theta_j with
// theta_j = pow(base, -2.0 * j * (1/dim))   rope.cpp:20-27, 29-41
std::vector<double> rope_table(const uint64_t* positions, uint64_t rows, uint64_t dim,
                               double base) {
    const double inv_dim = 1.0 / static_cast<double>(dim);
    std::vector<double> th(dim / 2);
    for (size_t j = 0; j < th.size(); ++j)
        th[j] = std::pow(base, -2.0 * static_cast<double>(j) * inv_dim);
    std::vector<double> cs(rows * dim);
    for (uint64_t i = 0; i < rows; ++i) {
        const double p = static_cast<double>(positions[i]);
        for (size_t j = 0; j < th.size(); ++j) {
            const double angle = -1.0 * p * th[j];
            cs[(i * (dim / 2) + j) * 2] = std::cos(angle);
            cs[(i * (dim / 2) + j) * 2 + 1] = std::sin(angle);
        }
    }
    return cs;
}

// Tiles of <= kPackTile local ids per group, in group order.
void build_tiles(const std::vector<GroupMeta>& meta, std::vector<TileDesc>& tiles,
                 std::vector<uint32_t>& first) {
    tiles.clear();
    first.assign(meta.size() + 1, 0);
    for (size_t g = 0; g < meta.size(); ++g) {
        first[g] = (uint32_t)tiles.size();
        const uint32_t ns = meta[g].n - meta[g].sink;
        for (uint32_t f = 0; f < ns; f += kPackTile)
            tiles.push_back(TileDesc{(uint32_t)g, f, std::min(kPackTile, ns - f), 0});
    }
    first[meta.size()] = (uint32_t)tiles.size();
}

// Route pointer tables: one centT / Q-model triple per group, cached on the layer.
void bind_routers(saap_layer* L, const saap_router* const* routers, int& mode, int& use_deroped) {
    std::vector<const saap_router*> rs(routers, routers + L->n_groups);
    for (auto* r : rs) need(r, "sparse_attention: router");
    const int kind = rs[0]->kind;
    use_deroped = rs[0]->use_deroped;
    for (auto* r : rs) {
        if (r->kind != kind) unsupported("sparse_attention: mixed router kinds in one call");
        if (kind == 0 && r->use_deroped != use_deroped)
            unsupported("sparse_attention: mixed roped/de-roped centroid routers in one call");
    }
    mode = kind == 0 ? 1 : 2;
    if (rs == L->cached_routers) return;
    if (L->ctx->capturing) invalid("router set changed during graph capture");
    if (kind == 0) {
        std::vector<const float*> p(L->n_groups), pr(L->n_groups);
        std::vector<float> cm(L->n_groups);
        for (size_t g = 0; g < p.size(); ++g) {
            p[g] = rs[g]->part->centT;
            pr[g] = rs[g]->part->cent;
            cm[g] = rs[g]->part->cmax;
        }
        if (!L->d_centT) L->d_centT = (const float**)(dmalloc<void*>(L->n_groups));
        if (!L->d_centR) L->d_centR = (const float**)(dmalloc<void*>(L->n_groups));
        if (!L->d_cmax) L->d_cmax = dmalloc<float>(L->n_groups);
        SAAP_CUDA(cudaMemcpy(L->d_centT, p.data(), p.size() * sizeof(void*), cudaMemcpyHostToDevice));
        SAAP_CUDA(cudaMemcpy(L->d_centR, pr.data(), pr.size() * sizeof(void*), cudaMemcpyHostToDevice));
        SAAP_CUDA(cudaMemcpy(L->d_cmax, cm.data(), cm.size() * 4, cudaMemcpyHostToDevice));
        // slots: groups sharing one partition share the approximate scoring loads
        std::vector<const saap_partition*> uniq;
        std::vector<std::vector<uint32_t>> members;
        for (size_t g = 0; g < rs.size(); ++g) {
            auto it = std::find(uniq.begin(), uniq.end(), rs[g]->part);
            if (it == uniq.end()) {
                uniq.push_back(rs[g]->part);
                members.emplace_back();
                it = uniq.end() - 1;
            }
            members[it - uniq.begin()].push_back((uint32_t)g);
        }
        std::vector<ApproxSlot> tab;
        for (size_t u = 0; u < uniq.size(); ++u)
            for (size_t k0 = 0; k0 < members[u].size(); k0 += kSlotGroups) {
                ApproxSlot sl{};
                sl.centT = uniq[u]->centT;
                sl.centB = uniq[u]->centB;
                sl.count = (uint32_t)std::min<size_t>(kSlotGroups, members[u].size() - k0);
                for (uint32_t k = 0; k < sl.count; ++k) sl.group[k] = members[u][k0 + k];
                tab.push_back(sl);
            }
        if (!L->d_route_slots) L->d_route_slots = dmalloc<ApproxSlot>(L->n_groups);  // <= one slot per group
        SAAP_CUDA(cudaMemcpy(L->d_route_slots, tab.data(), tab.size() * sizeof(ApproxSlot),
                             cudaMemcpyHostToDevice));
        L->n_route_slots = (uint32_t)tab.size();
        L->h_route_slots.assign((const uint8_t*)tab.data(), (const uint8_t*)(tab.data() + tab.size()));
    } else {
        std::vector<const double*> p(3 * L->n_groups);
        for (size_t g = 0; g < L->n_groups; ++g) {
            p[3 * g] = rs[g]->model->w1;
            p[3 * g + 1] = rs[g]->model->w2;
            p[3 * g + 2] = rs[g]->model->vec;
        }
        L->qm_w_finite = true;
        for (size_t g = 0; g < L->n_groups; ++g) L->qm_w_finite = L->qm_w_finite && rs[g]->model->w_finite;
        if (!L->d_qm) L->d_qm = (const double**)(dmalloc<void*>(3 * L->n_groups));
        SAAP_CUDA(cudaMemcpy(L->d_qm, p.data(), p.size() * sizeof(void*), cudaMemcpyHostToDevice));
        // slots: contexts routed by one Q-model share its W2 loads
        std::vector<const saap_qmodel*> uniq;
        std::vector<std::vector<uint32_t>> members;
        for (size_t g = 0; g < rs.size(); ++g) {
            auto it = std::find(uniq.begin(), uniq.end(), rs[g]->model);
            if (it == uniq.end()) {
                uniq.push_back(rs[g]->model);
                members.emplace_back();
                it = uniq.end() - 1;
            }
            members[it - uniq.begin()].push_back((uint32_t)g);
        }
        std::vector<uint32_t> tab;
        for (auto& m : members)
            for (size_t k0 = 0; k0 < m.size(); k0 += kQmSlot)
                for (size_t k = 0; k < (size_t)kQmSlot; ++k)
                    tab.push_back(k0 + k < m.size() ? m[k0 + k] : 0xFFFFFFFFu);
        if (!L->d_qm_slots) L->d_qm_slots = dmalloc<uint32_t>(L->n_groups * kQmSlot);
        SAAP_CUDA(cudaMemcpy(L->d_qm_slots, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice));
        L->n_qm_slots = (uint32_t)(tab.size() / kQmSlot);
    }
    L->cached_routers = rs;
}

void check_router_dims(const saap_router* r, uint64_t d, uint64_t C, uint64_t l) {
    if (r->kind == 0) {
        if (d != r->part->d)
            invalid("CentroidRouter: query dim " + std::to_string(d) + " vs centroid dim " +
                    std::to_string(r->part->d));
        if (l > r->part->C) invalid("CentroidRouter: l exceeds bucket count");
        if (C && r->part->C != C) invalid("sparse_attention: router bucket count differs from store");
    } else {
        if (d != r->model->d)
            invalid("qmodel: query dim " + std::to_string(d) + " does not match model dim " +
                    std::to_string(r->model->d));
        if (l < 1 || l > r->model->C)
            invalid("batched_bucket_select: l=" + std::to_string(l) + " outside [1, " +
                    std::to_string(r->model->C) + "]");
        if (C && r->model->C != C) invalid("sparse_attention: router bucket count differs from store");
    }
}

// Routing is split over ceil(C / slice) CTAs per context; each keeps its
// top-min(l, slice) candidates, which route_plan_kernel merges.
struct RouteGeo {
    uint32_t slice, n_slices, keep, n_cand, P2;
};
RouteGeo route_geo(uint64_t C, uint64_t probes, uint64_t n_groups, int sm_count) {
    RouteGeo r;
    r.slice = C <= kSliceMax ? (uint32_t)C : (uint32_t)kSliceMax;  // one thread per centroid
    // smaller slices until the launch covers the SMs, while the planner's
    // candidate merge (next_pow2(n_slices * keep) entries) stays <= 256
    while (r.slice > 128 && r.slice % 2 == 0 &&
           n_groups * ((C + r.slice - 1) / r.slice) < (uint64_t)sm_count) {
        const uint64_t half = r.slice / 2;
        const uint64_t nc = ((C + half - 1) / half) * std::min<uint64_t>(probes, half);
        if (next_pow2((uint32_t)std::max<uint64_t>(nc, 1)) > 256) break;
        r.slice = (uint32_t)half;
    }
    r.n_slices = (uint32_t)((C + r.slice - 1) / r.slice);
    r.keep = (uint32_t)std::min<uint64_t>(probes, r.slice);
    r.n_cand = r.n_slices * r.keep;
    r.P2 = next_pow2(std::max<uint32_t>(r.n_cand, 1));
    return r;
}

// stage-1 routing launch for n groups (mode 1 centroid / 2 Q-model scores).
// Centroid routing with C <= 1024 uses fp32 scores + exact re-scoring of the
// boundary candidates in the planner; otherwise every score is exact fp64.
void enqueue_route_score(saap_ctx* c, uint64_t n_groups, uint64_t D, uint64_t C, uint64_t G,
                         uint64_t probes, int mode, const float* const* centT,
                         const float* q_route, const double* probs, PlanArgs& pa,
                         const float* cmax = nullptr, const float* const* centR = nullptr,
                         const ApproxSlot* slots = nullptr, uint32_t n_slots = 0) {
    const RouteGeo geo = route_geo(C, probes, n_groups, c->sm_count);
    const bool approx = mode == 1 && C <= kPlanThreads && cmax != nullptr && centR != nullptr;
    double* cs = (double*)ensure(c, c->cand_s, n_groups * geo.n_cand * sizeof(double));
    uint32_t* ci = (uint32_t*)ensure(c, c->cand_i, n_groups * geo.n_cand * sizeof(uint32_t));
    RouteArgs ra{};
    ra.mode = mode;
    ra.centT = centT;
    ra.q_route = q_route;
    ra.scores = probs;
    ra.G = (uint32_t)G;
    ra.D = (uint32_t)D;
    ra.C = (uint32_t)C;
    ra.probes = (uint32_t)probes;
    ra.slice = geo.slice;
    ra.n_slices = geo.n_slices;
    ra.keep = geo.keep;
    ra.cand_s = cs;
    ra.cand_i = ci;
    if (approx) {
        // fp32 scores of every centroid; the planner re-scores the boundary exactly
        ApproxArgs aa{};
        aa.centT = centT;
        aa.q_route = q_route;
        aa.slots = slots;
        aa.G = (uint32_t)G;
        aa.C = (uint32_t)C;
        aa.approx = (float*)ensure(c, c->approx, n_groups * C * sizeof(float));
        aa.tl = c->tl;
        launch_route_approx((int)D, aa, slots ? n_slots : (uint32_t)n_groups, c->stream);
        pa.approx = aa.approx;
        pa.centT = centT;
        pa.centR = centR;
        pa.cmax = cmax;
    } else {
        launch_route_score(ra, (uint32_t)n_groups, c->stream);
    }
    c->launches++;
    pa.P2 = approx ? next_pow2((uint32_t)C) : geo.P2;
    pa.n_cand = geo.n_cand;
    pa.cand_s = cs;
    pa.cand_i = ci;
}

// Everything a decode step reads about its cache.
struct DecodeSrc {
    uint64_t n_groups = 0, D = 0, C = 1, max_n = 0, rows = 0;
    const GroupMeta* meta = nullptr;
    const uint32_t *off = nullptr, *offA = nullptr, *idx = nullptr, *assign = nullptr,
                   *invA = nullptr;
    const uint16_t *K = nullptr, *V = nullptr;
    uint16_t *gK = nullptr, *gV = nullptr;
    uint64_t gather_cap = 0;
    uint64_t recent_hint = ~0ull;  // packed-layout window (layers only)
    bool uniform_window = false;   // every routed context has recent_begin == T
    const DecodeMaps* maps = nullptr;
};

DecodeMaps* build_maps(const void* K, const void* V, uint64_t rows, uint32_t D, const void* gK,
                       const void* gV, uint64_t grows) {
    auto* m = new DecodeMaps;
    const void* a = gK ? gK : K;
    const void* b = gV ? gV : V;
    const uint64_t r = gK ? grows : rows;
    for (int i = 0; i < kBoxSizes; ++i) {
        m->map[0 * kBoxSizes + i] = make_group_map(K, rows, D, (uint32_t)i + 1);
        m->map[1 * kBoxSizes + i] = make_group_map(V, rows, D, (uint32_t)i + 1);
        m->map[2 * kBoxSizes + i] = make_group_map(a, r, D, (uint32_t)i + 1);
        m->map[3 * kBoxSizes + i] = make_group_map(b, r, D, (uint32_t)i + 1);
    }
    m->rows = rows;
    m->grows = r;
    return m;
}

// Static part of a decode work stream, planned on the host: per group the
// dense window (sink span [0, sink) and the recent tail [max(n - recent, T), n)
// of the packed layout), or every row when the window covers the context or
// for full attention (mode 0).  Segments take 8-aligned virtual rows and are
// cut into 128-row tiles (attention.cpp:342-347: the window is absorbed
// before any bucket).
// reuse: refresh that plan in place (stream-ordered uploads into its
// buffers when they are large enough) after the layout grew by an append
saap_static_plan* build_static_plan(const std::vector<GroupMeta>& meta, int mode, uint64_t recent,
                                    uint32_t nh, saap_static_plan* reuse = nullptr,
                                    cudaStream_t st = nullptr) {
    auto* sp = reuse ? reuse : new saap_static_plan;
    sp->max_slot_tiles = 0;
    sp->mode = mode;
    sp->recent = recent;
    sp->n_hchunks = nh;
    std::vector<TileRec> tiles;
    std::vector<uint32_t> cnt(meta.size() * nh, 0);
    for (size_t g = 0; g < meta.size(); ++g) {
        const GroupMeta& gm = meta[g];
        const uint64_t n = gm.n, sink = gm.sink, T = gm.T;
        std::vector<std::pair<uint64_t, uint64_t>> segs;  // (first row, rows)
        if (mode == 0 || n <= sink + recent) {
            segs.push_back({0, n});
        } else {
            const uint64_t rb = n - recent, tail0 = std::max(rb, T);
            if (sink) segs.push_back({0, sink});
            if (n > tail0) segs.push_back({tail0, n - tail0});
        }
        std::vector<uint64_t> v0(segs.size());
        uint64_t v = 0;
        for (size_t i = 0; i < segs.size(); ++i) {
            v0[i] = v;
            v += (segs[i].second + 7) & ~7ull;
        }
        const uint64_t ntiles = (v + kTileRows - 1) / kTileRows;
        std::vector<TileRec> gt(ntiles);
        for (auto& t : gt) std::memset(&t, 0, sizeof t);
        for (size_t i = 0; i < segs.size(); ++i) {
            const uint64_t s0 = v0[i], s8 = s0 + ((segs[i].second + 7) & ~7ull), send = s0 + segs[i].second;
            for (uint64_t t = s0 / kTileRows; t * kTileRows < s8; ++t) {
                const uint64_t a0 = std::max(s0, t * kTileRows), b0 = std::min(s8, (t + 1) * kTileRows);
                const uint64_t kend = std::min(b0, send);
                if (kend <= a0) continue;
                TileRec& tr = gt[t];
                PieceRec& pr = tr.p[tr.npieces++];
                pr.len = (uint32_t)(kend - a0);
                pr.srow = (uint32_t)(a0 - t * kTileRows);
                pr.row = gm.row_base + segs[i].first + (a0 - s0);
            }
        }
        for (uint32_t hc = 0; hc < nh; ++hc) {
            for (size_t i = 0; i < gt.size(); ++i) {
                TileRec t = gt[i];
                t.qslot = (uint32_t)(g * nh + hc);
                t.ready = 0;
                t.end = i + 1 == gt.size() ? 1u : 0u;
                tile_finish(t);
                tiles.push_back(t);
            }
            cnt[g * nh + hc] = (uint32_t)ntiles;
        }
        sp->max_slot_tiles = std::max<uint32_t>(sp->max_slot_tiles, (uint32_t)ntiles);
    }
    sp->n_tiles = (uint32_t)tiles.size();
    if (reuse && tiles.size() <= sp->cap_tiles) {
        h2d(sp->tiles, tiles.data(), tiles.size() * sizeof(TileRec), st);
        h2d(sp->cnt, cnt.data(), cnt.size() * 4, st);
        return sp;
    }
    if (reuse) {
        SAAP_CUDA(cudaStreamSynchronize(st));
        cudaFree(sp->tiles);
        cudaFree(sp->cnt);
    }
    sp->cap_tiles = std::max<size_t>(tiles.size(), 1) + (reuse ? tiles.size() / 8 : 0);
    sp->tiles = dmalloc<TileRec>(sp->cap_tiles);
    sp->cnt = dmalloc<uint32_t>(std::max<size_t>(cnt.size(), 1));
    if (!tiles.empty())
        SAAP_CUDA(cudaMemcpy(sp->tiles, tiles.data(), tiles.size() * sizeof(TileRec), cudaMemcpyHostToDevice));
    if (!cnt.empty())
        SAAP_CUDA(cudaMemcpy(sp->cnt, cnt.data(), cnt.size() * 4, cudaMemcpyHostToDevice));
    return sp;
}

void free_static_plan(saap_static_plan* sp) {
    if (!sp) return;
    if (sp->tiles) cudaFree(sp->tiles);
    if (sp->cnt) cudaFree(sp->cnt);
    delete sp;
}

// cached per handle: plans depend only on the (immutable) group layout
const saap_static_plan* static_plan(saap_ctx* c, std::vector<saap_static_plan*>& cache,
                                    const std::vector<GroupMeta>& meta, int mode, uint64_t recent,
                                    uint32_t nh) {
    const uint64_t rkey = mode == 0 ? 0 : recent;
    for (auto* p : cache)
        if (p->mode == mode && p->recent == rkey && p->n_hchunks == nh) {
            if (!p->stale) return p;
            if (c->capturing) invalid("decode plan refresh after an append during graph capture: run once uncaptured first");
            build_static_plan(meta, mode, rkey, nh, p, c->stream);
            p->stale = false;
            return p;
        }
    if (c->capturing) invalid("decode plan for a new window/head count during graph capture: run once uncaptured first");
    cache.push_back(build_static_plan(meta, mode, rkey, nh));
    return cache.back();
}

// Enqueue one decode step on the context stream: [Q-model] -> [routing] ->
// planner (dynamic tiles) -> decode (static + dynamic work stream) -> combine.
// mode: 0 dense/full (no planner), 1 centroid, 2 Q-model, 3 window only.
void enqueue_decode(saap_ctx* c, const DecodeSrc& src, const saap_static_plan* sp, int mode,
                    const float* const* centT, const double* const* qm, const float* q_attn,
                    const float* q_route, uint64_t G, uint64_t probes, uint64_t recent, float* out,
                    saap_attn_stats* stats, uint32_t* selected, uint32_t chunk,
                    uint32_t qm_hidden = 0, const float* cmax = nullptr,
                    const float* const* centR = nullptr, const ApproxSlot* slots = nullptr,
                    uint32_t n_slots = 0, const uint32_t* qm_slots = nullptr,
                    uint32_t n_qm_slots = 0, const uint32_t* given = nullptr,
                    const ApproxSlot* h_slots = nullptr, bool qm_finite = false) {
    const cudaStream_t st = c->stream;
    const uint64_t n_groups = src.n_groups, D = src.D, C = src.C;
    const uint64_t n_hchunks = (G + kHeadsPerSlot - 1) / kHeadsPerSlot;
    const uint64_t qslots = n_groups * n_hchunks;
    if (reinterpret_cast<uintptr_t>(q_attn) & 15) invalid("decode: queries must be 16-byte aligned");
    const bool plan = mode != 0;
    const uint64_t nseg = probes + 2;
    const uint64_t dyn_per_group = plan ? (src.max_n + 8 * nseg) / kTileRows + nseg + 2 : 0;
    // a run is >= 1 tile of one slot (the stream's tail goes out tile by tile)
    const uint64_t run_cap = sp->max_slot_tiles + dyn_per_group + 2;
    TileRec* dyn = plan ? (TileRec*)ensure_zero(c, c->tiles, n_groups * dyn_per_group * n_hchunks * sizeof(TileRec))
                        : nullptr;
    float* pO = (float*)ensure(c, c->part_O, qslots * run_cap * kHeadsPerSlot * D * sizeof(float));
    float* pml = (float*)ensure(c, c->part_ml, qslots * run_cap * 8 * sizeof(float));
    unsigned long long* rd = (unsigned long long*)ensure_zero(c, c->runs, qslots * 8);
    uint32_t* pflag = (uint32_t*)ensure_zero(c, c->part_flag, qslots * run_cap * 4);
    uint32_t* dcnt = plan ? (uint32_t*)ensure_zero(c, c->dyn_cnt, qslots * 4) : nullptr;
    if (plan && !stats) stats = (saap_attn_stats*)ensure(c, c->stats, n_groups * sizeof(saap_attn_stats));
    double* probs = nullptr;
    if (mode == 2) probs = (double*)ensure(c, c->probs, n_groups * G * (C + qm_hidden) * sizeof(double));

    cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;
    if (c->timing && !c->capturing) {
        for (cudaEvent_t* e : {&e0, &e1, &e2}) SAAP_CUDA(cudaEventCreate(e));
        SAAP_CUDA(cudaEventRecord(e0, st));
    }
    if (plan) {
        if (mode == 2) {
            QModelArgs qa{};
            qa.logits_variant = c->opt.qm_logits;
            qa.w_finite = qm_finite ? 1u : 0u;
            qa.q = q_route;
            qa.prm = qm;
            qa.G = (uint32_t)G;
            qa.d = (uint32_t)D;
            qa.h = qm_hidden;
            qa.C = (uint32_t)C;
            qa.probs = probs;
            qa.hid = probs + n_groups * G * C;
            qa.slot_g = qm_slots;
            launch_qmodel_probs(qa, (uint32_t)n_groups, st, n_qm_slots);
            c->launches++;
        }
        PlanArgs pa{};
        pa.meta = src.meta;
        pa.off = src.off;
        pa.offA = src.offA;
        pa.idx = src.idx;
        pa.assign = src.assign;
        pa.invA = src.invA;
        pa.C = (uint32_t)C;
        pa.mode = mode;
        pa.q_route = q_route;
        pa.scores = probs;
        pa.G = (uint32_t)G;
        pa.D = (uint32_t)D;
        pa.n_hchunks = (uint32_t)n_hchunks;
        pa.probes = (uint32_t)probes;
        pa.recent = (uint32_t)std::min<uint64_t>(recent, 0xFFFFFFFFull);
        pa.route_only = 0;
        pa.K = src.K;
        pa.V = src.V;
        pa.gK = src.gK;
        pa.gV = src.gV;
        pa.gather_cap = src.gather_cap;
        pa.dyn_tiles = dyn;
        pa.ctr = c->counters;
        pa.dyn_cnt = dcnt;
        pa.stats = stats;
        pa.selected = selected;
        pa.given = given;
        if (mode == 4) pa.P2 = next_pow2((uint32_t)std::max<uint64_t>(probes, 1));
        const bool routed = (mode == 1 || mode == 2) && probes > 0;
        const bool trace_on = c->opt.trace_plan != 0;
        const bool no_cluster = c->opt.cluster_route == 0;
        // fused cluster routing: centroid router, C a power of two <= 1024,
        // the packed layout's window (every routed context has rb == T)
        const bool fused = routed && mode == 1 && slots && cmax && centR && !no_cluster &&
                           route_cluster_supported((int)D, (uint32_t)C) && probes <= C &&
                           src.uniform_window;
        if (fused) {
            ClusterRouteArgs ra{};
            ra.slots = slots;
            if (h_slots && n_slots <= (uint32_t)kInlineSlots) {  // (one fewer round trip)
                std::copy(h_slots, h_slots + n_slots, ra.islots);
                ra.n_inline = n_slots;
            }
            ra.meta = src.meta;
            ra.off = src.off;
            ra.offA = src.offA;
            ra.q_route = q_route;
            ra.centR = centR;
            ra.cmax = cmax;
            ra.G = (uint32_t)G;
            ra.C = (uint32_t)C;
            ra.probes = (uint32_t)probes;
            ra.recent = (uint32_t)std::min<uint64_t>(recent, 0xFFFFFFFFull);
            ra.n_hchunks = (uint32_t)n_hchunks;
            ra.dyn_tiles = dyn;
            ra.ctr = c->counters;
            ra.dyn_cnt = dcnt;
            ra.stats = stats;
            ra.selected = selected;
            ra.tl = c->tl;
            if (trace_on) ra.trace = (unsigned long long*)ensure(c, c->trace, 128 + 48 * 1024);
            launch_route_cluster((int)D, ra, n_slots, st);
            c->launches++;
        } else {
            if (routed)
                enqueue_route_score(c, n_groups, D, C, G, probes, mode, centT, q_route, probs, pa, cmax,
                                    centR, slots, n_slots);
            pa.tl = c->tl;
            if (trace_on) pa.trace = (unsigned long long*)ensure(c, c->trace, 128 + 48 * 1024);
            launch_route_plan(pa, (uint32_t)n_groups, routed, st);
            c->launches++;
        }
    }
    if (e1) SAAP_CUDA(cudaEventRecord(e1, st));

    DecodeArgs da{};
    da.st_tiles = (const TileRec*)sp->tiles;
    da.dyn_tiles = dyn;
    da.n_static = sp->n_tiles;
    da.n_plan_groups = plan ? (uint32_t)n_groups : 0u;
    da.chunk = chunk;
    da.ctr = c->counters;
    da.q = q_attn;
    da.G = (uint32_t)G;
    da.n_hchunks = (uint32_t)n_hchunks;
    da.qscale = (float)(1.4426950408889634 / std::sqrt((double)D));
    da.part_O = pO;
    da.part_ml = pml;
    da.part_flag = pflag;
    da.run_cap = (uint32_t)run_cap;
    da.rd = rd;
    const uint64_t max_stream = sp->n_tiles + n_groups * dyn_per_group * n_hchunks;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)c->sm_count,
                                                                    (max_stream + chunk - 1) / chunk));
    da.tail = c->opt.tail_per_cta * (uint32_t)grid;
    da.poll_ns = c->opt.decode_poll_ns;
    da.tl = c->tl;
    da.wait_plan = plan && c->opt.decode_wait ? 1u : 0u;
    da.debug_skip = c->opt.debug_skip;
    da.min_chunk = c->opt.min_chunk;
    da.claim_lead = c->opt.claim_lead;
    da.fetch_lead = c->opt.fetch_lead;
    da.inflight = c->opt.inflight;
    // static tickets: enough to give every CTA a share of the window
    // pre-assigned first chunk per CTA (no atomic before its first loads): with
    // a planner running, CTAs on the SMs it holds start late, so they hold
    // only 2 tiles of reserved work; everything else is claimed from the counter
    const uint32_t cst = c->opt.chunk_st ? c->opt.chunk_st : 2u;  // pre-assigned window tiles per CTA
    da.chunk_st = plan ? std::max<uint32_t>(1u, std::min<uint32_t>(cst, sp->n_tiles / (uint32_t)grid)) : chunk;
    if (c->opt.trace_decode) {
        da.dtrace = (unsigned long long*)ensure(c, c->dtrace, (size_t)c->sm_count * (128 + kTraceTiles * 64));
        da.dtiles = da.dtrace + (size_t)c->sm_count * 16;
    }
    launch_decode((int)D, *src.maps, da, grid, st, c->opt.decode_tc != 0);
    CombineArgs ca{};
    ca.st_cnt = sp->cnt;
    ca.dyn_cnt = dcnt;
    ca.rd = rd;
    ca.part_O = pO;
    ca.part_ml = pml;
    ca.part_flag = pflag;
    ca.run_cap = (uint32_t)run_cap;
    ca.G = (uint32_t)G;
    ca.n_hchunks = (uint32_t)n_hchunks;
    ca.out = out;
    ca.tl = c->tl;
    ca.poll_ns = c->opt.combine_poll_ns;
    if (c->p2p) p2p_fill(c, ca);
    launch_combine((int)D, ca, (uint32_t)qslots, st);
    c->launches += 2;
    if (e2) {
        SAAP_CUDA(cudaEventRecord(e2, st));
        c->ev.insert(c->ev.end(), {e0, e1, e2});
    }
}

// Rows of a group between the packed layout's split T and this call's
// recent_begin (0 when the window matches the layout: the fast planner path).
// Appended keys (saap_layer_append) grow the position-ordered tail, so the
// skew is per group, not recent - recent_hint.
uint64_t window_skew(const GroupMeta& gm, uint64_t recent) {
    if (gm.n <= gm.sink + recent) return 0;
    const uint64_t rb = gm.n - recent;
    return rb > gm.T ? rb - gm.T : gm.T - rb;
}

// The layer's decode view (maps built once; gather buffer sized on demand).
DecodeSrc layer_src(saap_layer* L, uint64_t recent, bool need_gather) {
    if (need_gather) {
        uint64_t cap = 0;
        for (auto& gm : L->h_meta)
            cap = std::max<uint64_t>(cap, std::min<uint64_t>(gm.n - gm.sink, window_skew(gm, recent)));
        if (cap > L->gather_cap) {
            if (L->ctx->capturing) invalid("gather buffer grows during graph capture");
            SAAP_CUDA(cudaStreamSynchronize(L->ctx->stream));
            dfree(L->gK);
            dfree(L->gV);
            L->gK = dmalloc<uint16_t>(L->n_groups * cap * L->d);
            L->gV = dmalloc<uint16_t>(L->n_groups * cap * L->d);
            L->gather_cap = cap;
            delete (DecodeMaps*)L->maps;
            L->maps = nullptr;
            // saved step graphs hold the old gK/gV and maps as kernel arguments
            L->ctx->scratch_gen++;
        }
    }
    if (!L->maps)
        L->maps = build_maps(L->K, L->V, L->cap_rows, (uint32_t)L->d, L->gK, L->gV,
                             L->n_groups * L->gather_cap);
    DecodeSrc s;
    s.n_groups = L->n_groups;
    s.D = L->d;
    s.C = L->C;
    for (auto& gm : L->h_meta) s.max_n = std::max<uint64_t>(s.max_n, gm.n);
    s.rows = L->cap_rows;
    s.meta = L->meta;
    s.off = L->off;
    s.offA = L->offA;
    s.idx = L->idx;
    s.assign = L->assign;
    s.invA = L->invA;
    s.K = L->K;
    s.V = L->V;
    s.gK = L->gK;
    s.gV = L->gV;
    s.gather_cap = L->gather_cap;
    s.recent_hint = L->recent_hint;
    s.uniform_window = true;
    for (auto& gm : L->h_meta) s.uniform_window &= window_skew(gm, recent) == 0;
    s.maps = (const DecodeMaps*)L->maps;
    return s;
}

}  // namespace

namespace saap_b200 {
void set_error(const std::string& m) { g_err = m; }
[[noreturn]] void fail(int code, const std::string& msg) { throw Failure{code, msg}; }
void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Failure{SAAP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
    }
}
}  // namespace saap_b200

extern "C" {

const char* saap_last_error(void) { return g_err.c_str(); }
const char* saap_version(void) { return "saap_b200 0.1 (sm_100a)"; }

// ============================================================ context
int saap_ctx_create(int device, saap_ctx** out) {
    return guard([&] {
        need(out, "saap_ctx_create");
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            throw Failure{SAAP_ERR_NO_DEVICE, "no CUDA device visible: libsaap_b200 has no CPU path"};
        }
        if (device < 0 || device >= n) invalid("saap_ctx_create: device out of range");
        cudaDeviceProp prop;
        SAAP_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10)
            throw Failure{SAAP_ERR_NO_DEVICE,
                          std::string("libsaap_b200 needs an sm_100 (B200) device, found ") +
                                  prop.name};
        SAAP_CUDA(cudaSetDevice(device));
        auto* c = new saap_ctx;
        live_contexts().push_back(c);
        c->device = device;
        c->sm_count = prop.multiProcessorCount;
        SAAP_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
        c->counters = dmalloc<StepCounters>(1);
        SAAP_CUDA(cudaMemset(c->counters, 0, sizeof(StepCounters)));
        *out = c;
    });
}

int saap_ctx_destroy(saap_ctx* c) {
    return guard([&] {
        if (!c) return;
        cudaSetDevice(c->device);
        cudaStreamSynchronize(c->stream);
        for (saap_scratch* s : {&c->approx, &c->trace, &c->dtrace, &c->cand_s, &c->cand_i,
                                &c->tiles, &c->part_O, &c->part_ml, &c->probs, &c->stats, &c->sel,
                                &c->qr, &c->qd, &c->out, &c->misc, &c->zeros, &c->runs, &c->dyn_cnt, &c->part_flag})
            if (s->p) cudaFree(s->p);
        dfree(c->counters);
        dfree(c->tl);
        for (auto& g : c->host_graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        auto& lc = live_contexts();
        lc.erase(std::remove(lc.begin(), lc.end(), c), lc.end());
        if (c->side) cudaStreamDestroy(c->side);
        if (c->ev_fork) cudaEventDestroy(c->ev_fork);
        if (c->ev_join) cudaEventDestroy(c->ev_join);
        if (c->own_stream) cudaStreamDestroy(c->stream);
        delete c;
    });
}

int saap_ctx_set_stream(saap_ctx* c, void* stream) {
    return guard([&] {
        DeviceGuard dg(c);
        if (c->own_stream) {
            SAAP_CUDA(cudaStreamSynchronize(c->stream));
            cudaStreamDestroy(c->stream);
        }
        c->stream = (cudaStream_t)stream;
        c->own_stream = false;
    });
}

int saap_ctx_get_stream(saap_ctx* c, void** stream) {
    return guard([&] {
        need(c, "ctx");
        need(stream, "stream");
        *stream = (void*)c->stream;
    });
}

int saap_ctx_synchronize(saap_ctx* c) {
    return guard([&] {
        DeviceGuard dg(c);
        sync(c);
    });
}

int saap_ctx_sm_count(saap_ctx* c, int* out) {
    return guard([&] {
        need(c, "ctx");
        *out = c->sm_count;
    });
}

int saap_ctx_enable_timing(saap_ctx* c, int on) {
    return guard([&] {
        need(c, "ctx");
        c->timing = on != 0;
    });
}

int saap_ctx_timing(saap_ctx* c, double* plan_ms, double* attn_ms, uint64_t* steps) {
    return guard([&] {
        DeviceGuard dg(c);
        sync(c);
        double a = 0, b = 0;
        for (size_t i = 0; i + 2 < c->ev.size(); i += 3) {
            float x = 0, y = 0;
            SAAP_CUDA(cudaEventElapsedTime(&x, c->ev[i], c->ev[i + 1]));
            SAAP_CUDA(cudaEventElapsedTime(&y, c->ev[i + 1], c->ev[i + 2]));
            a += x;
            b += y;
        }
        if (plan_ms) *plan_ms = a;
        if (attn_ms) *attn_ms = b;
        if (steps) *steps = c->ev.size() / 3;
        for (auto e : c->ev) cudaEventDestroy(e);
        c->ev.clear();
    });
}

int saap_ctx_launch_count(saap_ctx* c, uint64_t* out) {
    return guard([&] {
        need(c, "ctx");
        *out = c->launches;
    });
}

// Tuning / diagnostic options (the round-1 environment knobs), per context.
int saap_ctx_set_option(saap_ctx* c, const char* name, int64_t value) {
    return guard([&] {
        DeviceGuard dg(c);
        need(name, "option name");
        const std::string n(name);
        auto& o = c->opt;
        auto clamp = [&](int64_t lo, int64_t hi) {
            if (value < lo || value > hi)
                invalid("saap_ctx_set_option: " + n + "=" + std::to_string(value) + " outside [" +
                        std::to_string(lo) + ", " + std::to_string(hi) + "]");
            return (uint32_t)value;
        };
        if (c->capturing) invalid("saap_ctx_set_option during graph capture");
        if (n == "chunk") o.chunk = clamp(1, 32);
        else if (n == "chunk_dense") o.chunk_dense = clamp(1, 32);
        else if (n == "tail_per_cta") o.tail_per_cta = clamp(0, 8);
        else if (n == "decode_poll_ns") o.decode_poll_ns = clamp(0, 100000);
        else if (n == "combine_poll_ns") o.combine_poll_ns = clamp(0, 100000);
        else if (n == "decode_wait") o.decode_wait = clamp(0, 1);
        else if (n == "cluster_route") o.cluster_route = clamp(0, 1);
        else if (n == "debug_skip") o.debug_skip = clamp(0, 2);
        else if (n == "min_chunk") o.min_chunk = clamp(1, 16);
        else if (n == "chunk_st") o.chunk_st = clamp(0, 16);
        else if (n == "claim_lead") o.claim_lead = clamp(0, 32);
        else if (n == "fetch_lead") o.fetch_lead = clamp(0, 32);
        else if (n == "inflight") o.inflight = clamp(0, 8);
        else if (n == "decode_tc") o.decode_tc = clamp(0, 1);
        else if (n == "qm_logits") o.qm_logits = clamp(0, 7);
        else if (n == "assign_f32_tc") o.assign_f32_tc = clamp(0, 1);
        else if (n == "host_graph") o.host_graph = clamp(0, 1);
        else if (n == "trace_decode") o.trace_decode = clamp(0, 1);
        else if (n == "trace_plan") o.trace_plan = clamp(0, 1);
        else if (n == "trace_step") {
            o.trace_step = clamp(0, 1);
            if (o.trace_step && !c->tl) {
                c->tl = dmalloc<unsigned long long>(16);
                SAAP_CUDA(cudaMemset(c->tl, 0, 128));
            } else if (!o.trace_step && c->tl) {
                sync(c);
                dfree(c->tl);
            }
        } else {
            invalid("saap_ctx_set_option: unknown option '" + n + "'");
        }
        // saved host-API step graphs hold the old launch parameters
        for (auto& g : c->host_graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        c->host_graphs.clear();
    });
}

// ============================================================ partitions / models / routers
int saap_partition_create(saap_ctx* c, const float* cent, uint64_t C, uint64_t d,
                          saap_partition** out) {
    return guard([&] {
        DeviceGuard dg(c);
        need(cent, "saap_partition_create");
        if (C == 0 || d == 0) invalid("Partition: empty centroid block");
        auto* p = new saap_partition;
        p->ctx = c;
        p->C = C;
        p->d = d;
        p->host.assign(cent, cent + C * d);
        std::vector<float> t(C * d);
        std::vector<double> d64(C * d);
        for (uint64_t i = 0; i < C; ++i)
            for (uint64_t j = 0; j < d; ++j) {
                t[j * C + i] = cent[i * d + j];
                d64[i * d + j] = (double)cent[i * d + j];
            }
        double cm = 0;
        for (uint64_t i = 0; i < C; ++i) {
            double n2 = 0;
            for (uint64_t j = 0; j < d; ++j) n2 += (double)cent[i * d + j] * cent[i * d + j];
            cm = std::max(cm, std::sqrt(n2));
        }
        p->cmax = (float)(cm * (1 + 1e-6));
        p->cent = dmalloc<float>(C * d);
        p->centT = dmalloc<float>(C * d);
        p->cent64 = dmalloc<double>(C * d);
        SAAP_CUDA(cudaMemcpy(p->cent, cent, C * d * 4, cudaMemcpyHostToDevice));
        SAAP_CUDA(cudaMemcpy(p->centT, t.data(), C * d * 4, cudaMemcpyHostToDevice));
        SAAP_CUDA(cudaMemcpy(p->cent64, d64.data(), C * d * 8, cudaMemcpyHostToDevice));
        if (C % kClusterCtas == 0) {  // the cluster router's slabs, contiguous per rank
            const uint64_t S = C / kClusterCtas;
            std::vector<float> b(C * d);
            for (uint64_t r = 0; r < (uint64_t)kClusterCtas; ++r)
                for (uint64_t j = 0; j < d; ++j)
                    for (uint64_t s2 = 0; s2 < S; ++s2) b[(r * d + j) * S + s2] = cent[(r * S + s2) * d + j];
            p->centB = dmalloc<float>(C * d);
            SAAP_CUDA(cudaMemcpy(p->centB, b.data(), C * d * 4, cudaMemcpyHostToDevice));
        }
        *out = p;
    });
}

int saap_partition_destroy(saap_partition* p) {
    return guard([&] {
        if (!p) return;
        cudaSetDevice(p->ctx->device);
        dfree(p->cent);
        dfree(p->centT);
        dfree(p->centB);
        dfree(p->cent64);
        delete p;
    });
}

int saap_qmodel_create(saap_ctx* c, uint64_t d, uint64_t h, uint64_t C, const double* w1,
                       const double* b1, const double* gamma, const double* beta,
                       const double* mean, const double* var, const double* w2, const double* b2,
                       saap_qmodel** out) {
    return guard([&] {
        DeviceGuard dg(c);
        if (d == 0 || h == 0 || C == 0) invalid("qmodel_init: zero dimension");
        for (auto* p : {w1, b1, gamma, beta, mean, var, w2, b2}) need(p, "saap_qmodel_create");
        const size_t smem = 4 * (d + h + C) * sizeof(double);
        if (smem > 227 * 1024) unsupported("Q-model router: d + h + C too large for one CTA");
        auto* m = new saap_qmodel;
        m->ctx = c;
        m->d = d;
        m->h = h;
        m->C = C;
        m->w1 = dmalloc<double>(d * h);
        m->w2 = dmalloc<double>(h * C);
        m->vec = dmalloc<double>(5 * h + C);
        SAAP_CUDA(cudaMemcpy(m->w1, w1, d * h * 8, cudaMemcpyHostToDevice));
        SAAP_CUDA(cudaMemcpy(m->w2, w2, h * C * 8, cudaMemcpyHostToDevice));
        const double* parts[5] = {b1, gamma, beta, mean, var};
        for (int i = 0; i < 5; ++i)
            SAAP_CUDA(cudaMemcpy(m->vec + i * h, parts[i], h * 8, cudaMemcpyHostToDevice));
        SAAP_CUDA(cudaMemcpy(m->vec + 5 * h, b2, C * 8, cudaMemcpyHostToDevice));
        m->w_finite = true;
        for (uint64_t i = 0; i < h * C && m->w_finite; ++i) m->w_finite = std::isfinite(w2[i]);
        for (uint64_t i = 0; i < d * h && m->w_finite; ++i) m->w_finite = std::isfinite(w1[i]);
        *out = m;
    });
}

int saap_qmodel_destroy(saap_qmodel* m) {
    return guard([&] {
        if (!m) return;
        cudaSetDevice(m->ctx->device);
        dfree(m->w1);
        dfree(m->w2);
        dfree(m->vec);
        delete m;
    });
}

int saap_router_create_centroid(saap_ctx* c, const saap_partition* p, int use_deroped,
                                saap_router** out) {
    return guard([&] {
        need(c, "ctx");
        need(p, "CentroidRouter: partition");
        auto* r = new saap_router;
        r->kind = 0;
        r->use_deroped = use_deroped ? 1 : 0;
        r->part = p;
        *out = r;
    });
}

int saap_router_create_qmodel(saap_ctx* c, const saap_qmodel* m, saap_router** out) {
    return guard([&] {
        need(c, "ctx");
        need(m, "QModelRouter: model");
        auto* r = new saap_router;
        r->kind = 1;
        r->model = m;
        *out = r;
    });
}

int saap_router_destroy(saap_router* r) {
    if (r)
        for (saap_ctx* c : live_contexts()) purge_host_graphs(c, nullptr, r);
    delete r;
    return SAAP_OK;
}

// Standalone routing runs the same route_plan kernel as a decode step, in
// route-only mode, for one query group.
static void route_once(saap_ctx* c, const saap_router* r, const float* q_route, uint64_t G,
                       uint64_t d, uint64_t l, uint32_t* out) {
    const uint64_t C = r->kind == 0 ? r->part->C : r->model->C;
    const cudaStream_t st = c->stream;
    float* dq = (float*)ensure(c, c->qd, G * d * 4);
    h2d(dq, q_route, G * d * 4, st);
    uint32_t* dsel = (uint32_t*)ensure(c, c->sel, l * 4);
    GroupMeta gm{0, 0, 2, 0, 0, 0};  // n > sink + recent so routing runs
    GroupMeta* dmeta = (GroupMeta*)ensure(c, c->misc, sizeof(GroupMeta) + sizeof(void*) * 4 + 16);
    void** dptr = reinterpret_cast<void**>(reinterpret_cast<char*>(dmeta) + sizeof(GroupMeta));
    float* dcmax = reinterpret_cast<float*>(dptr + 4);
    void* ptrs[4] = {nullptr, nullptr, nullptr, nullptr};
    int mode;
    double* probs = nullptr;
    if (r->kind == 0) {
        ptrs[0] = (void*)r->part->centT;
        ptrs[3] = (void*)r->part->cent;
        mode = 1;
    } else {
        ptrs[0] = (void*)r->model->w1;
        ptrs[1] = (void*)r->model->w2;
        ptrs[2] = (void*)r->model->vec;
        mode = 2;
        probs = (double*)ensure(c, c->probs, G * (C + r->model->h) * 8);
    }
    h2d(dmeta, &gm, sizeof gm, st);
    h2d(dptr, ptrs, sizeof(void*) * 4, st);
    if (r->kind == 0) h2d(dcmax, &r->part->cmax, 4, st);
    if (mode == 2) {
        QModelArgs qa{};
        qa.logits_variant = c->opt.qm_logits;
        qa.q = dq;
        qa.prm = (const double* const*)dptr;
        qa.G = (uint32_t)G;
        qa.d = (uint32_t)d;
        qa.h = (uint32_t)r->model->h;
        qa.C = (uint32_t)C;
        qa.probs = probs;
        qa.hid = probs + G * C;
        launch_qmodel_probs(qa, 1, st);
        c->launches++;
    }
    PlanArgs pa{};
    pa.meta = dmeta;
    pa.C = (uint32_t)C;
    pa.mode = mode;
    pa.q_route = dq;
    pa.scores = probs;
    pa.G = (uint32_t)G;
    pa.D = (uint32_t)d;
    pa.n_hchunks = 1;
    pa.probes = (uint32_t)l;
    pa.recent = 0;
    pa.route_only = 1;
    pa.selected = dsel;
    enqueue_route_score(c, 1, d, C, G, l, mode, (const float* const*)dptr, dq, probs, pa,
                        r->kind == 0 ? dcmax : nullptr,
                        r->kind == 0 ? (const float* const*)(dptr + 3) : nullptr);
    launch_route_plan(pa, 1, true, st);
    c->launches++;
    d2h(out, dsel, l * 4, st);
    sync(c);
}

int saap_router_select(saap_ctx* c, const saap_router* r, const float* q_roped,
                       const float* q_deroped, uint64_t G, uint64_t d, uint64_t l, uint32_t* out) {
    return guard([&] {
        DeviceGuard dg(c);
        need(r, "router");
        if (l == 0) return;  // attention.cpp:278-280, 311-313
        check_router_dims(r, d, 0, l);
        if (G == 0) {
            if (r->kind == 1) invalid("qmodel: empty query batch");
            // CentroidRouter: pooled = 0 scores every centroid 0, so the
            // (score desc, id asc) order gives ids 0..l-1 (attention.cpp:284-305)
            for (uint64_t i = 0; i < l; ++i) out[i] = (uint32_t)i;
            return;
        }
        const bool deroped = r->kind == 1 || r->use_deroped;
        const float* q = deroped ? q_deroped : q_roped;
        need(q, "router queries");
        route_once(c, r, q, G, d, l, out);
    });
}

int saap_batched_bucket_select(saap_ctx* c, const saap_qmodel* m, const float* q, uint64_t G,
                               uint64_t d, uint64_t l, uint32_t* out) {
    return guard([&] {
        DeviceGuard dg(c);
        need(m, "model");
        saap_router r;
        r.kind = 1;
        r.model = m;
        check_router_dims(&r, d, 0, l);
        if (G == 0) invalid("qmodel: empty query batch");
        route_once(c, &r, q, G, d, l, out);
    });
}

// qmodel_forward(model, queries_deroped) in eval mode (qmodel.cpp:375-377):
// row-softmax probabilities, fp64 on the device, narrowed to f32 like
// Mat::to_tensor.  Same kernels as the router (route.cu).
int saap_qmodel_forward(saap_ctx* c, const saap_qmodel* m, const float* q, uint64_t n, uint64_t d,
                        float* out) {
    return guard([&] {
        DeviceGuard dg(c);
        need(m, "model");
        if (d != m->d)
            invalid("qmodel: query dim " + std::to_string(d) + " does not match model dim " +
                    std::to_string(m->d));
        if (n == 0) invalid("qmodel: empty query batch");
        need(q, "qmodel_forward: queries");
        need(out, "qmodel_forward: out");
        const cudaStream_t st = c->stream;
        const uint64_t C = m->C;
        float* dq = (float*)ensure(c, c->qd, n * d * 4);
        double* probs = (double*)ensure(c, c->probs, n * (C + m->h) * 8);
        void** dptr = (void**)ensure(c, c->misc, 3 * sizeof(void*));
        const void* ptrs[3] = {m->w1, m->w2, m->vec};
        h2d(dq, q, n * d * 4, st);
        h2d(dptr, ptrs, sizeof ptrs, st);
        QModelArgs qa{};
        qa.logits_variant = c->opt.qm_logits;
        qa.q = dq;
        qa.prm = (const double* const*)dptr;
        qa.G = (uint32_t)n;
        qa.d = (uint32_t)d;
        qa.h = (uint32_t)m->h;
        qa.C = (uint32_t)C;
        qa.probs = probs;
        qa.hid = probs + n * C;
        launch_qmodel_probs(qa, 1, st);
        c->launches += 3;
        std::vector<double> p64(n * C);
        d2h(p64.data(), probs, n * C * 8, st);
        sync(c);
        for (uint64_t i = 0; i < n * C; ++i) out[i] = (float)p64[i];
    });
}

// ============================================================ assignment / IVF / rope
int saap_assign_keys(saap_ctx* c, const saap_partition* p, const float* keys, uint64_t n,
                     uint64_t d, uint32_t* out) {
    return guard([&] {
        DeviceGuard dg(c);
        need(p, "assign_keys: partition");
        if (d != p->d)
            invalid("assign_key: key dim " + std::to_string(d) + " does not match centroids " +
                    std::to_string(p->C) + "x" + std::to_string(p->d));
        if (!supported_dim(d) && km_dim_max((uint32_t)d) == 0)
            unsupported("assign_keys: unsupported key dim " + std::to_string(d));
        if (n == 0) return;
        const cudaStream_t st = c->stream;
        float* dk = (float*)ensure(c, c->qr, n * d * 4);
        h2d(dk, keys, n * d * 4, st);
        if (!supported_dim(d)) {  // other dims <= 128: the k-means scorer (same best_bucket)
            if (n >= 0xFFFFFFFFull) unsupported("assign_keys: more than 2^32-1 keys");
            char* b = (char*)ensure(c, c->misc, n * 12 + 256);
            uint32_t* dout = (uint32_t*)b;
            double* dsc = (double*)(b + ((n * 4 + 255) & ~size_t(255)));
            launch_km_assign(dk, (uint32_t)n, (uint32_t)d, p->cent, (uint32_t)p->C, dout, dsc,
                             nullptr, st);
            c->launches++;
            d2h(out, dout, n * 4, st);
            sync(c);
            return;
        }
        std::vector<GroupMeta> meta{GroupMeta{0, 0, (uint32_t)n, 0, 0, 0}};
        std::vector<TileDesc> tiles;
        std::vector<uint32_t> first;
        build_tiles(meta, tiles, first);
        char* base = (char*)ensure(c, c->misc, tiles.size() * sizeof(TileDesc) + 64 + n * 4);
        TileDesc* dt = (TileDesc*)base;
        uint64_t* zero64 = (uint64_t*)(base + tiles.size() * sizeof(TileDesc));
        const double** dc = (const double**)(zero64 + 1);
        uint32_t* dout = (uint32_t*)(base + tiles.size() * sizeof(TileDesc) + 64);
        const uint64_t z = 0;
        const double* cp = p->cent64;
        h2d(dt, tiles.data(), tiles.size() * sizeof(TileDesc), st);
        h2d(zero64, &z, 8, st);
        h2d(dc, &cp, sizeof cp, st);
        launch_assign_exact((int)d, false, dt, (uint32_t)tiles.size(), dk, zero64, dc,
                            (uint32_t)p->C, dout, zero64, st);
        c->launches++;
        d2h(out, dout, n * 4, st);
        sync(c);
    });
}

int saap_build_ivf(saap_ctx* c, const uint32_t* assignment, uint64_t n, uint64_t C, uint64_t* off,
                   uint64_t* idx) {
    return guard([&] {
        DeviceGuard dg(c);
        for (uint64_t i = 0; i < n; ++i)
            if (assignment[i] >= C)
                invalid("build_ivf: bucket id " + std::to_string(assignment[i]) +
                        " out of range for " + std::to_string(C) + " buckets");
        if (n >= 0xFFFFFFFFull) unsupported("build_ivf: more than 2^32-1 keys");
        const cudaStream_t st = c->stream;
        std::vector<GroupMeta> meta{GroupMeta{0, 0, (uint32_t)n, 0, 0, 0}};
        std::vector<TileDesc> tiles;
        std::vector<uint32_t> first;
        build_tiles(meta, tiles, first);
        const size_t nt = tiles.size();
        // one scratch block: meta | tiles | first | hist | countA | off | offA | assign | idx | invA
        size_t o = 0;
        auto take = [&](size_t bytes) {
            size_t r = o;
            o += (bytes + 255) & ~size_t(255);
            return r;
        };
        const size_t o_meta = take(sizeof(GroupMeta)), o_tiles = take(nt * sizeof(TileDesc)),
                     o_first = take(first.size() * 4), o_hist = take(nt * C * 4),
                     o_cA = take(2 * C * 4), o_off = take((C + 1) * 4), o_offA = take((C + 1) * 4),
                     o_as = take(n * 4), o_idx = take(n * 4), o_inv = take(n * 4);
        char* b = (char*)ensure(c, c->misc, o);
        h2d(b + o_meta, meta.data(), sizeof(GroupMeta), st);
        h2d(b + o_tiles, tiles.data(), nt * sizeof(TileDesc), st);
        h2d(b + o_first, first.data(), first.size() * 4, st);
        h2d(b + o_as, assignment, n * 4, st);
        launch_pack(32, (TileDesc*)(b + o_tiles), (uint32_t)nt, (uint32_t*)(b + o_first), 1,
                    (GroupMeta*)(b + o_meta), (uint32_t*)(b + o_as), (uint32_t)C,
                    (uint32_t*)(b + o_hist), (uint32_t*)(b + o_cA), (uint32_t*)(b + o_off),
                    (uint32_t*)(b + o_offA), (uint32_t*)(b + o_idx), (uint32_t*)(b + o_inv),
                    nullptr, nullptr, n, nullptr, nullptr, nullptr, nullptr, nullptr, st);
        c->launches += 4;
        std::vector<uint32_t> off32(C + 1), idx32(n);
        d2h(off32.data(), b + o_off, (C + 1) * 4, st);
        d2h(idx32.data(), b + o_idx, n * 4, st);
        sync(c);
        for (uint64_t i = 0; i <= C; ++i) off[i] = off32[i];
        for (uint64_t i = 0; i < n; ++i) idx[i] = idx32[i];
    });
}

// kmeans_train(keys, C, iters, rng, stats)   partition.cpp:52-179.  The
// caller's Rng draws the seed rows (sample_without_replacement then shuffle,
// :80-82); everything after that runs on the device (kmeans.cu).
int saap_kmeans_train(saap_ctx* c, const float* keys, uint64_t n, uint64_t d, uint64_t C,
                      uint64_t iters, const uint64_t* seed_rows, float* centroids,
                      double* objective_per_iter, uint64_t* zero_vector_keys,
                      uint64_t* empty_cluster_repairs) {
    return guard([&] {
        DeviceGuard dg(c);
        if (C < 1) invalid("kmeans_train: need at least 1 bucket");
        if (n < C)
            invalid("kmeans_train: " + std::to_string(n) + " keys cannot seed " +
                    std::to_string(C) + " buckets");
        if (iters < 1) invalid("kmeans_train: iters must be >= 1");
        need(keys, "kmeans_train: keys");
        need(seed_rows, "kmeans_train: seed rows");
        need(centroids, "kmeans_train: centroids");
        if (d == 0 || km_dim_max((uint32_t)d) == 0)
            unsupported("kmeans_train: unsupported key dim " + std::to_string(d));
        if (n >= 0xFFFFFFFFull) unsupported("kmeans_train: more than 2^32-1 keys");
        for (uint64_t i = 0; i < C; ++i)
            if (seed_rows[i] >= n) invalid("kmeans_train: seed row out of range");
        const cudaStream_t st = c->stream;
        std::vector<GroupMeta> meta{GroupMeta{0, 0, (uint32_t)n, 0, 0, 0}};
        std::vector<TileDesc> tiles;
        std::vector<uint32_t> first;
        build_tiles(meta, tiles, first);
        const size_t nt = tiles.size();
        size_t o = 0;
        auto take = [&](size_t bytes) {
            size_t r = o;
            o += (bytes + 255) & ~size_t(255);
            return r;
        };
        const size_t o_keys = take(n * d * 4), o_cent = take(C * d * 4), o_seed = take(C * 8),
                     o_as = take(n * 4), o_sc = take(n * 8), o_cnt = take(C * 4),
                     o_meta = take(sizeof(GroupMeta)), o_tiles = take(nt * sizeof(TileDesc)),
                     o_first = take(first.size() * 4), o_hist = take(nt * C * 4),
                     o_cA = take(2 * C * 4), o_off = take((C + 1) * 4), o_offA = take((C + 1) * 4),
                     o_idx = take(n * 4), o_inv = take(n * 4), o_obj = take(iters * 8),
                     o_ctr = take(16);
        char* b = nullptr;
        SAAP_CUDA(cudaMalloc(&b, o));
        std::unique_ptr<char, void (*)(char*)> hold(b, [](char* p) { cudaFree(p); });
        const float* dk = (const float*)(b + o_keys);
        float* dc = (float*)(b + o_cent);
        uint32_t* das = (uint32_t*)(b + o_as);
        double* dsc = (double*)(b + o_sc);
        uint32_t* dcnt = (uint32_t*)(b + o_cnt);
        double* dobj = (double*)(b + o_obj);
        unsigned long long* ctr = (unsigned long long*)(b + o_ctr);
        h2d(b + o_keys, keys, n * d * 4, st);
        h2d(b + o_seed, seed_rows, C * 8, st);
        h2d(b + o_meta, meta.data(), sizeof(GroupMeta), st);
        h2d(b + o_tiles, tiles.data(), nt * sizeof(TileDesc), st);
        h2d(b + o_first, first.data(), first.size() * 4, st);
        SAAP_CUDA(cudaMemsetAsync(ctr, 0, 16, st));
        const uint32_t N = (uint32_t)n, D = (uint32_t)d, CC = (uint32_t)C;
        launch_km_seed(dk, D, (const uint64_t*)(b + o_seed), CC, dc, st);
        c->launches++;
        for (uint64_t it = 0; it < iters; ++it) {
            launch_km_assign(dk, N, D, dc, CC, das, dsc, it == 0 ? ctr : nullptr, st);
            if (it > 0 && objective_per_iter) launch_km_objective(dsc, N, dobj + it - 1, st);
            launch_km_iteration_tail(dk, N, D, das, dsc, dcnt, CC, ctr + 1, st);
            launch_pack(32, (TileDesc*)(b + o_tiles), (uint32_t)nt, (uint32_t*)(b + o_first), 1,
                        (GroupMeta*)(b + o_meta), das, CC, (uint32_t*)(b + o_hist),
                        (uint32_t*)(b + o_cA), (uint32_t*)(b + o_off), (uint32_t*)(b + o_offA),
                        (uint32_t*)(b + o_idx), (uint32_t*)(b + o_inv), nullptr, nullptr, n,
                        nullptr, nullptr, nullptr, nullptr, nullptr, st);
            launch_km_update(dk, D, (const uint32_t*)(b + o_off), (const uint32_t*)(b + o_idx), CC,
                             dc, st);
            c->launches += 4 + 4 + (it > 0 && objective_per_iter ? 1 : 0);
        }
        if (objective_per_iter) {  // objective of the last update: one more scoring pass
            launch_km_assign(dk, N, D, dc, CC, das, dsc, nullptr, st);
            launch_km_objective(dsc, N, dobj + iters - 1, st);
            c->launches += 2;
        }
        unsigned long long hc[2];
        d2h(centroids, dc, C * d * 4, st);
        d2h(hc, ctr, 16, st);
        if (objective_per_iter) d2h(objective_per_iter, dobj, iters * 8, st);
        sync(c);
        if (zero_vector_keys) *zero_vector_keys = hc[0];
        if (empty_cluster_repairs) *empty_cluster_repairs = hc[1];
    });
}

// ---------------------------------------------------------------- Q-model training
// TrainerState + QModel on the device (qmodel.hpp:66-75, qtrain.cu).
int saap_qtrainer_create(saap_ctx* c, uint64_t d, uint64_t h, uint64_t C,
                         const double* const* params, const double* hyper, uint64_t step,
                         saap_qtrainer** out) {
    return guard([&] {
        DeviceGuard dg(c);
        need(out, "qtrainer: out");
        need(params, "qtrainer: params");
        if (d == 0 || h == 0 || C == 0) invalid("qmodel_init: zero dimension");
        auto* t = new saap_qtrainer();
        std::unique_ptr<saap_qtrainer> hold(t);
        t->ctx = c;
        t->d = d;
        t->h = h;
        t->C = C;
        if (hyper) {
            t->lr = hyper[0];
            t->beta1 = hyper[1];
            t->beta2 = hyper[2];
            t->eps = hyper[3];
            t->bn_momentum = hyper[4];
        }
        t->step = step;
        const uint64_t cnt[8] = {d * h, h, h, h, h, h, h * C, C};
        for (int k = 0; k < 8; ++k) {
            need(params[k], "qtrainer: parameter");
            t->p[k] = dmalloc<double>(cnt[k]);
            t->m[k] = dmalloc<double>(cnt[k]);
            t->v[k] = dmalloc<double>(cnt[k]);
            t->g[k] = dmalloc<double>(cnt[k]);
            SAAP_CUDA(cudaMemcpy(t->p[k], params[k], cnt[k] * 8, cudaMemcpyHostToDevice));
            SAAP_CUDA(cudaMemset(t->m[k], 0, cnt[k] * 8));
            SAAP_CUDA(cudaMemset(t->v[k], 0, cnt[k] * 8));
        }
        t->mean = dmalloc<double>(h);
        t->var = dmalloc<double>(h);
        t->w2T = dmalloc<double>(h * C);
        t->loss = dmalloc<double>(1);
        *out = hold.release();
    });
}

static void qtrainer_free_acts(saap_qtrainer* t) {
    for (double** a : {&t->x, &t->z, &t->xhat, &t->y, &t->r, &t->pr, &t->tgt, &t->dl, &t->dy,
                       &t->dz, &t->loss_rows})
        dfree(*a);
    dfree(t->q32);
    t->n_cap = 0;
}

int saap_qtrainer_destroy(saap_qtrainer* t) {
    return guard([&] {
        if (!t) return;
        cudaSetDevice(t->ctx->device);
        qtrainer_free_acts(t);
        for (int k = 0; k < 8; ++k) {
            dfree(t->p[k]);
            dfree(t->m[k]);
            dfree(t->v[k]);
            dfree(t->g[k]);
        }
        dfree(t->mean);
        dfree(t->var);
        dfree(t->w2T);
        dfree(t->loss);
        delete t;
    });
}

// train_step_on_target(model, state, queries_deroped, target)  qmodel.cpp:419-433
int saap_qtrainer_step(saap_ctx* c, saap_qtrainer* t, const float* q, uint64_t n, uint64_t d,
                       const double* target, double* loss) {
    return guard([&] {
        DeviceGuard dg(c);
        need(t, "qtrainer");
        if (d != t->d)
            invalid("qmodel: query dim " + std::to_string(d) + " does not match model dim " +
                    std::to_string(t->d));
        if (n == 0) invalid("qmodel: empty query batch");
        if (n < 2) invalid("qmodel: train-mode forward needs >= 2 rows for batch stats");
        need(q, "qtrainer: queries");
        need(target, "qtrainer: target");
        const cudaStream_t st = c->stream;
        if (n > t->n_cap) {
            SAAP_CUDA(cudaStreamSynchronize(st));
            qtrainer_free_acts(t);
            const uint64_t h = t->h, C = t->C;
            t->x = dmalloc<double>(n * t->d);
            for (double** a : {&t->z, &t->xhat, &t->y, &t->r, &t->dy, &t->dz}) *a = dmalloc<double>(n * h);
            for (double** a : {&t->pr, &t->tgt, &t->dl}) *a = dmalloc<double>(n * C);
            t->loss_rows = dmalloc<double>(n);
            t->q32 = dmalloc<float>(n * t->d);
            t->n_cap = n;
        }
        h2d(t->q32, q, n * d * 4, st);
        h2d(t->tgt, target, n * t->C * 8, st);
        qtrain_forward(t, (uint32_t)n, st);
        double l = 0;
        d2h(&l, t->loss, 8, st);
        sync(c);
        c->launches += 6;
        if (!std::isfinite(l))
            fail(SAAP_ERR_RUNTIME, "train_step: non-finite loss at step " + std::to_string(t->step + 1));
        qtrain_update(t, (uint32_t)n, st);
        c->launches += 14;
        if (loss) *loss = l;
        sync(c);
    });
}

int saap_qtrainer_read(saap_ctx* c, const saap_qtrainer* t, double* const* params, uint64_t* step) {
    return guard([&] {
        DeviceGuard dg(c);
        need(t, "qtrainer");
        const uint64_t d = t->d, h = t->h, C = t->C;
        const uint64_t cnt[8] = {d * h, h, h, h, h, h, h * C, C};
        if (params)
            for (int k = 0; k < 8; ++k)
                if (params[k]) d2h(params[k], t->p[k], cnt[k] * 8, c->stream);
        sync(c);
        if (step) *step = t->step;
    });
}

// attention_target_rows(q_roped, keys_roped, assignment, C)  qmodel.cpp:384-407
int saap_attention_target(saap_ctx* c, const float* q, uint64_t n, uint64_t d, const float* keys,
                          uint64_t n_keys, const uint32_t* assignment, uint64_t C, double* out) {
    return guard([&] {
        DeviceGuard dg(c);
        if (n_keys == 0) invalid("attention_target: empty key set");
        for (uint64_t k = 0; k < n_keys; ++k)
            if (assignment[k] >= C) invalid("attention_target: bucket id out of range");
        if (n == 0) return;
        if (C * 8 > 200 * 1024) unsupported("attention_target: more than 25600 buckets");
        const cudaStream_t st = c->stream;
        size_t o = 0;
        auto take = [&](size_t bytes) {
            size_t r = o;
            o += (bytes + 255) & ~size_t(255);
            return r;
        };
        const size_t o_q = take(n * d * 4), o_k = take(n_keys * d * 4), o_as = take(n_keys * 4),
                     o_a = take(n * n_keys * 8), o_out = take(n * C * 8);
        char* b = nullptr;
        SAAP_CUDA(cudaMalloc(&b, o));
        std::unique_ptr<char, void (*)(char*)> hold(b, [](char* p) { cudaFree(p); });
        h2d(b + o_q, q, n * d * 4, st);
        h2d(b + o_k, keys, n_keys * d * 4, st);
        h2d(b + o_as, assignment, n_keys * 4, st);
        launch_attention_target((const float*)(b + o_q), (uint32_t)n, (uint32_t)d,
                                (const float*)(b + o_k), (uint32_t)n_keys,
                                (const uint32_t*)(b + o_as), (uint32_t)C, (double*)(b + o_a),
                                (double*)(b + o_out), st);
        c->launches += 3;
        d2h(out, b + o_out, n * C * 8, st);
        sync(c);
    });
}

// ---------------------------------------------------------------- accumulators
// PartialAccumulator and its operations (attention.hpp:30-70, attention.cpp:
// 34-161, 197-203), fp64 on the device, bit-exact (accum.cu).
int saap_accum_create(saap_ctx* c, uint64_t heads, uint64_t value_dim, saap_accum** out) {
    return guard([&] {
        DeviceGuard dg(c);
        need(out, "accumulator: out");
        auto* a = new saap_accum();
        std::unique_ptr<saap_accum> hold(a);
        a->ctx = c;
        a->heads = heads;
        a->dv = value_dim;
        a->out = dmalloc<double>(std::max<uint64_t>(heads * value_dim, 1));
        a->sumexp = dmalloc<double>(std::max<uint64_t>(heads, 1));
        a->runmax = dmalloc<double>(std::max<uint64_t>(heads, 1));
        a->rescale = dmalloc<double>(std::max<uint64_t>(heads, 1));
        if (heads) launch_acc_init(a->out, a->sumexp, a->runmax, (uint32_t)heads, (uint32_t)value_dim, c->stream);
        sync(c);
        *out = hold.release();
    });
}

int saap_accum_destroy(saap_accum* a) {
    return guard([&] {
        if (!a) return;
        cudaSetDevice(a->ctx->device);
        dfree(a->out);
        dfree(a->sumexp);
        dfree(a->runmax);
        dfree(a->rescale);
        delete a;
    });
}

int saap_accum_read(saap_ctx* c, const saap_accum* a, double* out_acc, double* sumexp, double* runmax) {
    return guard([&] {
        DeviceGuard dg(c);
        need(a, "accumulator");
        if (out_acc) d2h(out_acc, a->out, a->heads * a->dv * 8, c->stream);
        if (sumexp) d2h(sumexp, a->sumexp, a->heads * 8, c->stream);
        if (runmax) d2h(runmax, a->runmax, a->heads * 8, c->stream);
        sync(c);
    });
}

int saap_accum_write(saap_ctx* c, saap_accum* a, const double* out_acc, const double* sumexp,
                     const double* runmax) {
    return guard([&] {
        DeviceGuard dg(c);
        need(a, "accumulator");
        if (out_acc) h2d(a->out, out_acc, a->heads * a->dv * 8, c->stream);
        if (sumexp) h2d(a->sumexp, sumexp, a->heads * 8, c->stream);
        if (runmax) h2d(a->runmax, runmax, a->heads * 8, c->stream);
        sync(c);
    });
}

// shared absorb: validation as absorb_impl (:38-48), rows staged by id order
static void absorb_rows(saap_ctx* c, saap_accum* a, const float* q, uint64_t G, uint64_t d,
                        const float* keys, const float* values, uint64_t n_rows, uint64_t kd,
                        uint64_t dv, const uint64_t* ids, uint64_t begin, uint64_t count) {
    need(a, "accumulator");
    if (a->heads != G || a->dv != dv)
        invalid("pattn_absorb: accumulator " + std::to_string(a->heads) + "x" +
                std::to_string(a->dv) + " does not fit group " + std::to_string(G) + "x" +
                std::to_string(dv));
    if (d != kd)  // absorb_impl :40-43, after check_kv / check_acc
        invalid("pattn_absorb: query dim " + std::to_string(d) + " vs key dim " + std::to_string(kd));
    if (count == 0 || G == 0) return;
    need(q, "pattn_absorb: queries");
    need(keys, "pattn_absorb: keys");
    need(values, "pattn_absorb: values");
    if (ids)
        for (uint64_t j = 0; j < count; ++j)
            if (ids[j] >= n_rows)
                invalid("pattn_absorb: key id " + std::to_string(ids[j]) + " out of range");
    if (count >= 0xFFFFFFFFull || d == 0) unsupported("pattn_absorb: shape");
    std::vector<float> Ks(count * d), Vs(count * dv);
    for (uint64_t j = 0; j < count; ++j) {
        const uint64_t r = ids ? ids[j] : begin + j;
        std::memcpy(&Ks[j * d], keys + r * d, d * 4);
        std::memcpy(&Vs[j * dv], values + r * dv, dv * 4);
    }
    const cudaStream_t st = c->stream;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t r = o;
        o += (bytes + 255) & ~size_t(255);
        return r;
    };
    const size_t o_q = take(G * d * 4), o_k = take(count * d * 4), o_v = take(count * dv * 4),
                 o_s = take(G * count * 8);
    char* b = (char*)ensure(c, c->misc, o);
    h2d(b + o_q, q, G * d * 4, st);
    h2d(b + o_k, Ks.data(), count * d * 4, st);
    h2d(b + o_v, Vs.data(), count * dv * 4, st);
    launch_acc_absorb((const float*)(b + o_q), (uint32_t)G, (uint32_t)d, (const float*)(b + o_k),
                      (const float*)(b + o_v), (uint32_t)count, (uint32_t)dv,
                      1.0 / std::sqrt((double)d), (double*)(b + o_s), a->rescale, a->out, a->sumexp,
                      a->runmax, st);
    c->launches += 3;
    sync(c);
}

int saap_pattn_absorb(saap_ctx* c, saap_accum* a, const float* q, uint64_t G, uint64_t d,
                      const float* keys, const float* values, uint64_t n_keys, uint64_t key_dim,
                      uint64_t n_values, uint64_t dv, const uint64_t* ids, uint64_t count) {
    return guard([&] {
        DeviceGuard dg(c);
        if (n_keys != n_values)
            invalid("attention: " + std::to_string(n_keys) + " keys vs " + std::to_string(n_values) +
                    " values");
        if (count) need(ids, "pattn_absorb: ids");
        absorb_rows(c, a, q, G, d, keys, values, n_keys, key_dim, dv, ids, 0, count);
    });
}

int saap_pattn_absorb_range(saap_ctx* c, saap_accum* a, const float* q, uint64_t G, uint64_t d,
                            const float* keys, const float* values, uint64_t n_keys,
                            uint64_t key_dim, uint64_t n_values, uint64_t dv, uint64_t begin,
                            uint64_t end) {
    return guard([&] {
        DeviceGuard dg(c);
        if (end > n_keys || begin > end)
            invalid("pattn_absorb_range: bad range [" + std::to_string(begin) + ", " +
                    std::to_string(end) + ")");
        if (n_keys != n_values)
            invalid("attention: " + std::to_string(n_keys) + " keys vs " + std::to_string(n_values) +
                    " values");
        absorb_rows(c, a, q, G, d, keys, values, n_keys, key_dim, dv, nullptr, begin, end - begin);
    });
}

int saap_merge_into(saap_ctx* c, saap_accum* a, const saap_accum* part) {
    return guard([&] {
        DeviceGuard dg(c);
        need(a, "merge_into: accumulator");
        need(part, "merge_into: part");
        if (a->heads != part->heads || a->dv != part->dv)
            invalid("merge_into: accumulator shapes differ");
        if (!a->heads) return;
        launch_acc_merge(a->out, a->sumexp, a->runmax, part->out, part->sumexp, part->runmax,
                         (uint32_t)a->heads, (uint32_t)a->dv, c->stream);
        c->launches++;
        sync(c);
    });
}

// merge_partials(parts): result = parts[0] merged with parts[1..] in order
int saap_merge_partials(saap_ctx* c, const saap_accum* const* parts, uint64_t n, saap_accum* out) {
    return guard([&] {
        DeviceGuard dg(c);
        if (n == 0) invalid("merge_partials: empty list");
        need(parts, "merge_partials: parts");
        need(out, "merge_partials: out");
        const saap_accum* p0 = parts[0];
        need(p0, "merge_partials: part");
        if (out->heads != p0->heads || out->dv != p0->dv) invalid("merge_into: accumulator shapes differ");
        const cudaStream_t st = c->stream;
        if (out != p0) {
            SAAP_CUDA(cudaMemcpyAsync(out->out, p0->out, p0->heads * p0->dv * 8, cudaMemcpyDeviceToDevice, st));
            SAAP_CUDA(cudaMemcpyAsync(out->sumexp, p0->sumexp, p0->heads * 8, cudaMemcpyDeviceToDevice, st));
            SAAP_CUDA(cudaMemcpyAsync(out->runmax, p0->runmax, p0->heads * 8, cudaMemcpyDeviceToDevice, st));
        }
        for (uint64_t i = 1; i < n; ++i) {
            need(parts[i], "merge_partials: part");
            if (parts[i]->heads != out->heads || parts[i]->dv != out->dv)
                invalid("merge_into: accumulator shapes differ");
            if (!out->heads) continue;
            launch_acc_merge(out->out, out->sumexp, out->runmax, parts[i]->out, parts[i]->sumexp,
                             parts[i]->runmax, (uint32_t)out->heads, (uint32_t)out->dv, st);
            c->launches++;
        }
        sync(c);
    });
}

int saap_pattn_finalize(saap_ctx* c, const saap_accum* a, float* out, int* any_empty) {
    return guard([&] {
        DeviceGuard dg(c);
        need(a, "pattn_finalize: accumulator");
        need(out, "pattn_finalize: out");
        const cudaStream_t st = c->stream;
        char* b = (char*)ensure(c, c->misc, a->heads * a->dv * 4 + 256);
        int* flag = (int*)b;
        float* dout = (float*)(b + 256);
        SAAP_CUDA(cudaMemsetAsync(flag, 0, 4, st));
        if (a->heads) {
            launch_acc_finalize(a->out, a->sumexp, (uint32_t)a->heads, (uint32_t)a->dv, dout, flag, st);
            c->launches++;
        }
        int fl = 0;
        d2h(out, dout, a->heads * a->dv * 4, st);
        d2h(&fl, flag, 4, st);
        sync(c);
        if (any_empty) *any_empty = fl;
    });
}

// attention_over_ids(q, keys, values, ids): one absorb into a fresh
// accumulator, then finalize (attention.cpp:197-203)
int saap_attention_over_ids(saap_ctx* c, const float* q, uint64_t G, uint64_t d, const float* keys,
                            const float* values, uint64_t n_keys, uint64_t key_dim,
                            uint64_t n_values, uint64_t dv, const uint64_t* ids, uint64_t count,
                            float* out, int* any_empty) {
    saap_accum* a = nullptr;
    int rc = saap_accum_create(c, G, dv, &a);
    if (rc != SAAP_OK) return rc;
    rc = saap_pattn_absorb(c, a, q, G, d, keys, values, n_keys, key_dim, n_values, dv, ids, count);
    if (rc == SAAP_OK) rc = saap_pattn_finalize(c, a, out, any_empty);
    if (rc != SAAP_OK) {
        const std::string keep = g_err;
        saap_accum_destroy(a);
        g_err = keep;
        return rc;
    }
    return saap_accum_destroy(a);
}

int saap_rope_remove(saap_ctx* c, const float* x, uint64_t rows, uint64_t d,
                     const uint64_t* positions, double base, float* out) {
    return guard([&] {
        DeviceGuard dg(c);
        if (d == 0 || d % 2)
            invalid("RopeConfig: dim must be even and positive, got " + std::to_string(d));
        if (!(base > 0.0)) invalid("RopeConfig: base_theta must be positive");
        if (rows == 0) return;
        const cudaStream_t st = c->stream;
        std::vector<double> cs = rope_table(positions, rows, d, base);
        float* dx = (float*)ensure(c, c->qr, rows * d * 4);
        float* dy = (float*)ensure(c, c->out, rows * d * 4);
        double* dcs = (double*)ensure(c, c->misc, cs.size() * 8);
        h2d(dx, x, rows * d * 4, st);
        h2d(dcs, cs.data(), cs.size() * 8, st);
        launch_derope(dx, dcs, rows, (uint32_t)d, dy, st);
        c->launches++;
        d2h(out, dy, rows * d * 4, st);
        sync(c);
    });
}

// ============================================================ layers (context stores)
int saap_layer_create(saap_ctx* c, uint64_t n_groups, uint64_t d, uint64_t C,
                      const uint64_t* n_keys, uint64_t sink, uint64_t recent_hint,
                      saap_layer** out) {
    return saap_layer_create_cap(c, n_groups, d, C, n_keys, nullptr, sink, recent_hint, out);
}

int saap_layer_create_cap(saap_ctx* c, uint64_t n_groups, uint64_t d, uint64_t C,
                          const uint64_t* n_keys, const uint64_t* n_cap, uint64_t sink,
                          uint64_t recent_hint, saap_layer** out) {
    return guard([&] {
        DeviceGuard dg(c);
        need(n_keys, "saap_layer_create: n_keys");
        if (n_groups == 0) invalid("saap_layer_create: no groups");
        if (!supported_dim(d)) unsupported("store: unsupported head dim " + std::to_string(d));
        if (C == 0) invalid("Partition: empty centroid block");
        if (C > 16384) unsupported("store: more than 16384 buckets per head");
        auto* L = new saap_layer;
        L->ctx = c;
        L->n_groups = n_groups;
        L->d = d;
        L->C = C;
        L->sink = sink;
        L->recent_hint = recent_hint;
        uint64_t rows = 0, ns = 0, src = 0, src_ns = 0;
        for (uint64_t g = 0; g < n_groups; ++g) {
            const uint64_t n = n_keys[g];
            const uint64_t cap = n_cap ? n_cap[g] : n;
            if (n <= sink) {
                delete L;
                invalid("build_context_store: no keys left to index after " + std::to_string(sink) +
                        " sink keys");
            }
            if (n >= (1ull << 30)) {
                delete L;
                unsupported("store: context longer than 2^30 keys");
            }
            if (cap < n || cap >= (1ull << 30)) {
                delete L;
                invalid("saap_layer_create: capacity " + std::to_string(cap) + " below " +
                        std::to_string(n) + " keys or above 2^30");
            }
            const uint64_t T = n > sink + recent_hint ? n - recent_hint : sink;
            L->h_meta.push_back(GroupMeta{rows, ns, (uint32_t)n, (uint32_t)sink, (uint32_t)T, 0});
            L->h_src0.push_back(src);
            L->h_cap.push_back(cap);
            rows += cap;
            ns += cap - sink;
            src += n;
            src_ns += n - sink;
        }
        L->total_rows = src;
        L->total_ns = src_ns;
        L->cap_rows = rows;
        L->cap_ns = ns;
        L->meta = dmalloc<GroupMeta>(n_groups);
        L->row_base = dmalloc<uint64_t>(n_groups);
        L->K = dmalloc<uint16_t>(rows * d);
        L->V = dmalloc<uint16_t>(rows * d);
        L->assign = dmalloc<uint32_t>(ns);
        L->idx = dmalloc<uint32_t>(ns);
        L->invA = dmalloc<uint32_t>(ns);
        L->posA = dmalloc<uint32_t>(ns);
        L->list = dmalloc<uint32_t>(ns);  // per-key destination row (pack scratch)
        L->off = dmalloc<uint32_t>(n_groups * (C + 1));
        L->offA = dmalloc<uint32_t>(n_groups * (C + 1));
        std::vector<TileDesc> tiles;
        std::vector<uint32_t> first;
        build_tiles(L->h_meta, tiles, first);
        L->n_tiles = (uint32_t)tiles.size();
        L->tiles = dmalloc<TileDesc>(tiles.size());
        L->tile_first = dmalloc<uint32_t>(first.size());
        L->hist = dmalloc<uint32_t>(tiles.size() * C);
        L->countA = dmalloc<uint32_t>(2 * n_groups * C);  // countA | per-bucket totals
        L->d_cent64 = (const double**)(dmalloc<void*>(n_groups));
        std::vector<uint64_t> rb(n_groups), kr0(n_groups), ib(n_groups);
        for (uint64_t g = 0; g < n_groups; ++g) {
            rb[g] = L->h_meta[g].row_base;
            kr0[g] = L->h_src0[g] + L->h_meta[g].sink;  // assignment keys: source rows
            ib[g] = L->h_meta[g].ivf_base;
        }
        L->key_row0 = dmalloc<uint64_t>(n_groups);
        L->ivf_base = dmalloc<uint64_t>(n_groups);
        SAAP_CUDA(cudaMemcpy(L->key_row0, kr0.data(), n_groups * 8, cudaMemcpyHostToDevice));
        SAAP_CUDA(cudaMemcpy(L->ivf_base, ib.data(), n_groups * 8, cudaMemcpyHostToDevice));
        SAAP_CUDA(cudaMemcpy(L->meta, L->h_meta.data(), n_groups * sizeof(GroupMeta),
                             cudaMemcpyHostToDevice));
        SAAP_CUDA(cudaMemcpy(L->row_base, rb.data(), n_groups * 8, cudaMemcpyHostToDevice));
        L->src_row0 = dmalloc<uint64_t>(n_groups);
        SAAP_CUDA(cudaMemcpy(L->src_row0, L->h_src0.data(), n_groups * 8, cudaMemcpyHostToDevice));
        SAAP_CUDA(cudaMemcpy(L->tiles, tiles.data(), tiles.size() * sizeof(TileDesc),
                             cudaMemcpyHostToDevice));
        SAAP_CUDA(cudaMemcpy(L->tile_first, first.data(), first.size() * 4, cudaMemcpyHostToDevice));
        *out = L;
    });
}

// Re-sorts idx (and re-derives the other index tables, unchanged for region
// A) from the assignments after appends: the build's counting sort, no rows move.
void ensure_index(saap_ctx* c, saap_layer* L) {
    if (!L->idx_stale) return;
    if (c->capturing) invalid("index re-sort after an append during graph capture: run once uncaptured first");
    const cudaStream_t st = c->stream;
    std::vector<TileDesc> tiles;
    std::vector<uint32_t> first;
    build_tiles(L->h_meta, tiles, first);
    if (tiles.size() > L->n_tiles) {
        SAAP_CUDA(cudaStreamSynchronize(st));
        dfree(L->tiles);
        dfree(L->hist);
        L->tiles = dmalloc<TileDesc>(tiles.size());
        L->hist = dmalloc<uint32_t>(tiles.size() * L->C);
    }
    L->n_tiles = (uint32_t)tiles.size();
    h2d(L->tiles, tiles.data(), tiles.size() * sizeof(TileDesc), st);
    h2d(L->tile_first, first.data(), first.size() * 4, st);
    launch_pack((int)L->d, L->tiles, L->n_tiles, L->tile_first, (uint32_t)L->n_groups, L->meta,
                L->assign, (uint32_t)L->C, L->hist, L->countA, L->off, L->offA, L->idx, L->invA,
                L->posA, L->list, L->cap_ns, nullptr, nullptr, nullptr, nullptr, nullptr, st);
    c->launches += 4;
    L->idx_stale = false;
}

// Incremental decode index: k new keys per context go
// to the position-ordered tail (rows [n, n + k)), are assigned on the device
// (exact, like the build), and the index (off / idx / region-A tables) is
// rebuilt from the assignments by the counting sort.  Region A and its rows
// never move: keys that slide out of the window stay in the tail and the
// planner filters them by bucket (the general-window path), so every later
// step equals build_context_store over the grown context (attention.cpp:
// 249-255, 317-376).  Captured graphs of this layer must be re-captured.
int saap_layer_append(saap_ctx* c, saap_layer* L, const void* keys_roped_bf16,
                      const void* values_bf16, const void* keys_assign_bf16, uint64_t k) {
    return guard([&] {
        DeviceGuard dg(c);
        need(L, "layer");
        if (!L->built) invalid("append: store not built");
        need(keys_roped_bf16, "append: keys");
        need(values_bf16, "append: values");
        need(keys_assign_bf16, "append: assignment keys");
        if (c->capturing) invalid("append: not capturable");
        if (k == 0) return;
        for (size_t g = 0; g < L->h_meta.size(); ++g)
            if (L->h_meta[g].n + k > L->h_cap[g])
                invalid("append: context " + std::to_string(g) + " would exceed its capacity " +
                        std::to_string(L->h_cap[g]) + " keys");
        const cudaStream_t st = c->stream;
        const uint32_t ng = (uint32_t)L->n_groups;
        // rows into place (meta still holds the old n)
        launch_append_rows((int)L->d, L->meta, ng, (uint32_t)k, (const uint16_t*)keys_roped_bf16,
                           (const uint16_t*)values_bf16, L->K, L->V, st);
        // exact assignment of the new keys: local ids [n - sink, n - sink + k)
        std::vector<GroupMeta> am;
        std::vector<uint64_t> kr0(ng);
        for (uint32_t g = 0; g < ng; ++g) {
            const GroupMeta& gm = L->h_meta[g];
            am.push_back(gm);
            kr0[g] = (uint64_t)g * k - (uint64_t)(gm.n - gm.sink);  // modular: row g*k for the first new id
        }
        std::vector<TileDesc> at;
        for (uint32_t g = 0; g < ng; ++g) {
            const uint32_t first = L->h_meta[g].n - L->h_meta[g].sink;
            for (uint64_t f = 0; f < k; f += kPackTile)
                at.push_back(TileDesc{g, first + (uint32_t)f, (uint32_t)std::min<uint64_t>(kPackTile, k - f), 0});
        }
        char* b = (char*)ensure(c, c->misc, at.size() * sizeof(TileDesc) + ng * 8 + 64);
        h2d(b, at.data(), at.size() * sizeof(TileDesc), st);
        h2d(b + at.size() * sizeof(TileDesc), kr0.data(), ng * 8, st);
        launch_assign_exact((int)L->d, true, (const TileDesc*)b, (uint32_t)at.size(), keys_assign_bf16,
                            (const uint64_t*)(b + at.size() * sizeof(TileDesc)), L->d_cent64,
                            (uint32_t)L->C, L->assign, L->ivf_base, st, (uint32_t)std::min<uint64_t>(k, kPackTile));
        // grow the contexts; source rows follow the new sizes
        uint64_t src = 0, src_ns = 0;
        for (uint32_t g = 0; g < ng; ++g) {
            L->h_meta[g].n += (uint32_t)k;
            L->h_src0[g] = src;
            src += L->h_meta[g].n;
            src_ns += L->h_meta[g].n - L->h_meta[g].sink;
        }
        L->total_rows = src;
        L->total_ns = src_ns;
        std::vector<uint64_t> skr0(ng);
        for (uint32_t g = 0; g < ng; ++g) skr0[g] = L->h_src0[g] + L->h_meta[g].sink;
        h2d(L->meta, L->h_meta.data(), ng * sizeof(GroupMeta), st);
        h2d(L->src_row0, L->h_src0.data(), ng * 8, st);
        h2d(L->key_row0, skr0.data(), ng * 8, st);
        // raw bucket sizes grow in place; idx (ids in bucket order) is only
        // read by read_index and by windows reaching into region A, so it is
        // re-sorted lazily (ensure_index)
        launch_append_off(L->meta, ng, L->assign, (uint32_t)k, (uint32_t)L->C, L->off, st);
        c->launches += 3;
        L->idx_stale = true;
        for (auto* p : L->plans) p->stale = true;  // refreshed in place at the next step
        L->tc_parts.clear();  // tcgen05 tiles follow the sizes at the next build
        L->appended = true;
        for (saap_ctx* cc : live_contexts()) purge_host_graphs(cc, L, nullptr);
    });
}

// Host f32 rows [n_groups x k x dim] each, rounded to the bf16 cache (RNE)
// on the device, then appended like saap_layer_append.
int saap_layer_append_host(saap_ctx* c, saap_layer* L, const float* keys_roped,
                           const float* values, const float* keys_assign, uint64_t k) {
    int rc = SAAP_OK;
    const int g = guard([&] {
        DeviceGuard dg(c);
        need(L, "layer");
        need(keys_roped, "append: keys");
        need(values, "append: values");
        need(keys_assign, "append: assignment keys");
        if (k == 0) return;
        const uint64_t elems = L->n_groups * k * L->d;
        float* f32 = dmalloc<float>(elems);
        uint16_t* b = dmalloc<uint16_t>(3 * elems);
        const cudaStream_t st = c->stream;
        try {
            const float* src[3] = {keys_roped, values, keys_assign};
            for (int i = 0; i < 3; ++i) {
                h2d(f32, src[i], elems * 4, st);
                launch_f32_to_bf16(f32, b + i * elems, elems, st);
                c->launches++;
            }
            sync(c);
            rc = saap_layer_append(c, L, b, b + elems, b + 2 * elems, k);
            sync(c);
        } catch (...) {
            cudaFree(f32);
            cudaFree(b);
            throw;
        }
        cudaFree(f32);
        cudaFree(b);
    });
    return g != SAAP_OK ? g : rc;
}

int saap_layer_destroy(saap_layer* L) {
    return guard([&] {
        if (!L) return;
        cudaSetDevice(L->ctx->device);
        cudaStreamSynchronize(L->ctx->stream);
        for (saap_ctx* c : live_contexts()) purge_host_graphs(c, L, nullptr);
        dfree(L->meta);
        dfree(L->src_row0);
        dfree(L->row_base);
        dfree(L->K);
        dfree(L->V);
        dfree(L->assign);
        dfree(L->idx);
        dfree(L->invA);
        dfree(L->posA);
        dfree(L->list);
        dfree(L->gK);
        dfree(L->gV);
        delete (DecodeMaps*)L->maps;
        for (auto* p : L->plans) free_static_plan(p);
        dfree(L->off);
        dfree(L->offA);
        dfree(L->tiles);
        dfree(L->tile_first);
        dfree(L->hist);
        dfree(L->countA);
        for (auto e : L->bev)
            if (e) cudaEventDestroy(e);
        dfree(L->d_cent64);
        dfree(L->key_row0);
        dfree(L->ivf_base);
        dfree(L->tc_hi);
        dfree(L->tc_mid);
        dfree(L->tc_cmax);
        dfree(L->tc_refine);
        dfree(L->tc_refine_count);
        if (L->tc_tiles) cudaFree(L->tc_tiles);
        dfree(L->d_centT);
        dfree(L->d_centR);
        dfree(L->d_cmax);
        dfree(L->d_route_slots);
        dfree(L->split_hi);
        dfree(L->split_lo);
        dfree(L->d_qm);
        dfree(L->d_qm_slots);
        delete L;
    });
}

static void bind_parts(saap_layer* L, const saap_partition* const* parts) {
    need(parts, "build_context_store: partitions");
    std::vector<const double*> p(L->n_groups);
    L->parts.assign(parts, parts + L->n_groups);
    for (uint64_t g = 0; g < L->n_groups; ++g) {
        need(parts[g], "build_context_store: partition");
        if (parts[g]->d != L->d)
            invalid("assign_key: key dim " + std::to_string(L->d) + " does not match centroids " +
                    std::to_string(parts[g]->C) + "x" + std::to_string(parts[g]->d));
        if (parts[g]->C != L->C)
            invalid("build_context_store: partition has " + std::to_string(parts[g]->C) +
                    " buckets, store expects " + std::to_string(L->C));
        p[g] = parts[g]->cent64;
    }
    SAAP_CUDA(cudaMemcpy(L->d_cent64, p.data(), p.size() * sizeof(void*), cudaMemcpyHostToDevice));
}

// assignment + pack from device bf16 sources laid out like the layer rows
// keys: bf16 assignment keys; or (split mode, f32 keys) keys = k_hi, keys_lo =
// k_lo and keys_f32 the f32 rows (norms and the exact re-scoring)
static void assign_tc_path(saap_layer* L, const uint16_t* keys, const uint16_t* keys_lo = nullptr,
                           const float* keys_f32 = nullptr) {
    saap_ctx* c = L->ctx;
    const cudaStream_t st = c->stream;
    const uint32_t Cpad = tc_cpad((uint32_t)L->C);
    const bool split = keys_f32 != nullptr;
    if (L->tc_parts != L->parts || L->tc_split != split) {
        // distinct partitions -> slots of the concatenated (hi, mid) split arrays
        std::vector<const saap_partition*> slots;
        std::vector<uint32_t> slot_of(L->n_groups);
        for (uint64_t g = 0; g < L->n_groups; ++g) {
            auto it = std::find(slots.begin(), slots.end(), L->parts[g]);
            slot_of[g] = (uint32_t)(it - slots.begin());
            if (it == slots.end()) slots.push_back(L->parts[g]);
        }
        const size_t elems = slots.size() * (size_t)Cpad * L->d;
        if (elems > L->tc_split_elems) {
            dfree(L->tc_hi);
            dfree(L->tc_mid);
            L->tc_hi = dmalloc<uint16_t>(elems);
            L->tc_mid = dmalloc<uint16_t>(elems);
            L->tc_split_elems = elems;
        }
        std::vector<float> cmax(slots.size());
        for (size_t i = 0; i < slots.size(); ++i) {
            launch_split_centroids(slots[i]->cent, (uint32_t)L->C, (uint32_t)L->d,
                                   L->tc_hi + i * (size_t)Cpad * L->d,
                                   L->tc_mid + i * (size_t)Cpad * L->d, st);
            c->launches++;
            double m = 0;
            for (uint64_t r = 0; r < L->C; ++r) {
                double n2 = 0;
                for (uint64_t j = 0; j < L->d; ++j) {
                    const double v = slots[i]->host[r * L->d + j];
                    n2 += v * v;
                }
                m = std::max(m, std::sqrt(n2));
            }
            cmax[i] = (float)(m * (1 + 1e-6));
        }
        std::vector<TcTile> tiles;
        build_tc_tiles(L->h_meta, slot_of, tiles, split);
        dfree(L->tc_cmax);
        L->tc_cmax = dmalloc<float>(slots.size());
        SAAP_CUDA(cudaMemcpy(L->tc_cmax, cmax.data(), cmax.size() * 4, cudaMemcpyHostToDevice));
        if (L->tc_n_tiles != tiles.size()) {
            if (L->tc_tiles) cudaFree(L->tc_tiles);
            L->tc_tiles = dmalloc<TcTile>(tiles.size());
            L->tc_n_tiles = (uint32_t)tiles.size();
        }
        SAAP_CUDA(cudaMemcpy(L->tc_tiles, tiles.data(), tiles.size() * sizeof(TcTile),
                             cudaMemcpyHostToDevice));
        L->tc_parts = L->parts;
        L->tc_split = split;
        L->tc_nslots = (uint32_t)slots.size();
    }
    if (!L->tc_refine) {
        L->tc_refine = dmalloc<uint32_t>(std::max<uint64_t>(L->cap_ns, 1));
        L->tc_refine_count = dmalloc<uint32_t>(L->n_groups);
    }
    SAAP_CUDA(cudaMemsetAsync(L->tc_refine_count, 0, L->n_groups * 4, st));
    TcAssignArgs args{};
    args.tiles = (const TcTile*)L->tc_tiles;
    args.key_row0 = L->key_row0;
    args.out_base = L->ivf_base;
    args.cmax = L->tc_cmax;
    args.C = (uint32_t)L->C;
    args.Cpad = Cpad;
    args.out = L->assign;
    args.refine = L->tc_refine;
    args.refine_count = L->tc_refine_count;
    args.keys = keys;
    args.keys_f32 = keys_f32;
    launch_assign_tc(keys, L->total_rows, L->tc_hi, L->tc_mid, L->tc_nslots, args, L->tc_n_tiles,
                     st, keys_lo);
    if (split)
        launch_refine(L->tc_refine, L->tc_refine_count, keys_f32, L->key_row0, L->d_cent64, L->ivf_base,
                      (uint32_t)L->C, L->assign, (uint32_t)L->n_groups, c->sm_count, st, true);
    else
        launch_refine(L->tc_refine, L->tc_refine_count, keys, L->key_row0, L->d_cent64, L->ivf_base,
                      (uint32_t)L->C, L->assign, (uint32_t)L->n_groups, c->sm_count, st, false);
    c->launches += 2;
    L->last_tc = true;
}

static void build_from_device(saap_layer* L, const uint16_t* Ksrc, const uint16_t* Vsrc,
                              const void* keys_assign, bool assign_bf16) {
    saap_ctx* c = L->ctx;
    const cudaStream_t st = c->stream;
    L->last_tc = false;
    const bool timed = c->timing && !c->capturing;
    if (timed) {
        for (auto& e : L->bev)
            if (!e) SAAP_CUDA(cudaEventCreate(&e));
        SAAP_CUDA(cudaEventRecord(L->bev[0], st));
    }
    if (assign_bf16 && L->d == 128 && c->assign_mode == 0) {
        assign_tc_path(L, (const uint16_t*)keys_assign);
    } else if (!assign_bf16 && L->d == 128 && c->assign_mode == 0 && c->opt.assign_f32_tc) {
        // f32 keys on the tensor cores: k = k_hi + k_lo (bf16 terms), the
        // bound widened for the split; ambiguous keys re-scored from the f32 rows
        const uint64_t elems = L->total_rows * L->d;
        if (elems > L->split_elems) {  // (kept with the layer: rebuilds reuse them)
            sync(c);
            dfree(L->split_hi);
            dfree(L->split_lo);
            L->split_hi = dmalloc<uint16_t>(elems);
            L->split_lo = dmalloc<uint16_t>(elems);
            L->split_elems = elems;
        }
        launch_split_rows((const float*)keys_assign, elems, L->split_hi, L->split_lo, st);
        assign_tc_path(L, L->split_hi, L->split_lo, (const float*)keys_assign);
        c->launches++;
    } else {
        launch_assign_exact((int)L->d, assign_bf16, L->tiles, L->n_tiles, keys_assign, L->key_row0,
                            L->d_cent64, (uint32_t)L->C, L->assign, L->ivf_base, st);
        c->launches++;
    }
    if (timed) SAAP_CUDA(cudaEventRecord(L->bev[1], st));
    launch_pack((int)L->d, L->tiles, L->n_tiles, L->tile_first, (uint32_t)L->n_groups, L->meta,
                L->assign, (uint32_t)L->C, L->hist, L->countA, L->off, L->offA, L->idx, L->invA,
                L->posA, L->list, L->cap_ns, Ksrc, Vsrc, L->src_row0, L->K, L->V, st);
    c->launches += 6;
    if (timed) SAAP_CUDA(cudaEventRecord(L->bev[2], st));
    L->built = true;
    L->idx_stale = false;
}

int saap_layer_build(saap_ctx* c, saap_layer* L, const saap_partition* const* parts,
                     const float* keys_roped, const float* values, const float* keys_assign,
                     double rope_base) {
    return guard([&] {
        DeviceGuard dg(c);
        need(L, "layer");
        need(keys_roped, "build_context_store: keys");
        need(values, "build_context_store: values");
        bind_parts(L, parts);
        const cudaStream_t st = c->stream;
        const uint64_t elems = L->total_rows * L->d;
        float* f32 = dmalloc<float>(elems);
        uint16_t* Ks = dmalloc<uint16_t>(elems);
        uint16_t* Vs = dmalloc<uint16_t>(elems);
        try {
            h2d(f32, keys_roped, elems * 4, st);
            launch_f32_to_bf16(f32, Ks, elems, st);
            h2d(f32, values, elems * 4, st);
            launch_f32_to_bf16(f32, Vs, elems, st);
            c->launches += 2;
            // assignment keys (f32): caller's pre-RoPE keys, or de-rope on device
            if (keys_assign) {
                h2d(f32, keys_assign, elems * 4, st);
            } else {
                if (!(rope_base > 0.0)) invalid("RopeConfig: base_theta must be positive");
                h2d(f32, keys_roped, elems * 4, st);
                std::vector<uint64_t> pos(L->total_rows);
                for (size_t g = 0; g < L->h_meta.size(); ++g)
                    for (uint32_t i = 0; i < L->h_meta[g].n; ++i) pos[L->h_src0[g] + i] = i;
                std::vector<double> cs = rope_table(pos.data(), L->total_rows, L->d, rope_base);
                double* dcs = dmalloc<double>(cs.size());
                float* der = dmalloc<float>(elems);
                h2d(dcs, cs.data(), cs.size() * 8, st);
                launch_derope(f32, dcs, L->total_rows, (uint32_t)L->d, der, st);
                c->launches++;
                sync(c);
                cudaFree(dcs);
                cudaFree(f32);
                f32 = der;
            }
            build_from_device(L, Ks, Vs, f32, false);
            sync(c);
        } catch (...) {
            cudaFree(f32);
            cudaFree(Ks);
            cudaFree(Vs);
            throw;
        }
        cudaFree(f32);
        cudaFree(Ks);
        cudaFree(Vs);
    });
}

int saap_layer_build_dev(saap_ctx* c, saap_layer* L, const saap_partition* const* parts,
                         const void* keys_roped_bf16, const void* values_bf16,
                         const void* keys_assign_bf16) {
    return guard([&] {
        DeviceGuard dg(c);
        need(L, "layer");
        need(keys_roped_bf16, "build: keys");
        need(values_bf16, "build: values");
        need(keys_assign_bf16, "build: assignment keys");
        bind_parts(L, parts);
        build_from_device(L, (const uint16_t*)keys_roped_bf16, (const uint16_t*)values_bf16,
                          keys_assign_bf16, true);
    });
}

// ContextStore{keys, values, id_offset, partition, assignment, index} built
// field by field (attention_test.cpp:418-432): pack under the caller's
// assignment instead of computing one.
int saap_layer_build_assigned(saap_ctx* c, saap_layer* L, const saap_partition* const* parts,
                              const float* keys_roped, const float* values,
                              const uint32_t* assignment) {
    return guard([&] {
        DeviceGuard dg(c);
        need(L, "layer");
        need(keys_roped, "build_context_store: keys");
        need(values, "build_context_store: values");
        bind_parts(L, parts);
        uint64_t ns_total = 0;
        for (auto& gm : L->h_meta) ns_total += gm.n - gm.sink;
        if (ns_total) need(assignment, "build_context_store: assignment");
        for (uint64_t i = 0; i < ns_total; ++i)
            if (assignment[i] >= L->C)
                invalid("build_ivf: bucket id " + std::to_string(assignment[i]) + " out of range " +
                        std::to_string(L->C));
        const cudaStream_t st = c->stream;
        const uint64_t elems = L->total_rows * L->d;
        float* f32 = dmalloc<float>(elems);
        uint16_t* Ks = dmalloc<uint16_t>(elems);
        uint16_t* Vs = dmalloc<uint16_t>(elems);
        try {
            h2d(f32, keys_roped, elems * 4, st);
            launch_f32_to_bf16(f32, Ks, elems, st);
            h2d(f32, values, elems * 4, st);
            launch_f32_to_bf16(f32, Vs, elems, st);
            c->launches += 2;
            uint64_t a0 = 0;
            for (auto& gm : L->h_meta) {
                const uint64_t ns = gm.n - gm.sink;
                if (ns) h2d(L->assign + gm.ivf_base, assignment + a0, ns * 4, st);
                a0 += ns;
            }
            L->last_tc = false;
            launch_pack((int)L->d, L->tiles, L->n_tiles, L->tile_first, (uint32_t)L->n_groups, L->meta,
                        L->assign, (uint32_t)L->C, L->hist, L->countA, L->off, L->offA, L->idx, L->invA,
                        L->posA, L->list, L->cap_ns, Ks, Vs, L->src_row0, L->K, L->V, st);
            c->launches += 6;
            L->built = true;
            L->idx_stale = false;
            sync(c);
        } catch (...) {
            cudaFree(f32);
            cudaFree(Ks);
            cudaFree(Vs);
            throw;
        }
        cudaFree(f32);
        cudaFree(Ks);
        cudaFree(Vs);
    });
}

int saap_ctx_set_assign_mode(saap_ctx* c, int mode) {
    return guard([&] {
        need(c, "ctx");
        if (mode != 0 && mode != 1) invalid("assign mode must be 0 (tensor cores) or 1 (exact fp64)");
        c->assign_mode = mode;
    });
}

int saap_layer_build_timing(saap_ctx* c, const saap_layer* L, double* assign_ms, double* pack_ms) {
    return guard([&] {
        DeviceGuard dg(c);
        need(L, "layer");
        if (!L->bev[2]) invalid("no timed build: enable timing before saap_layer_build_dev");
        sync(c);
        float a = 0, b = 0;
        SAAP_CUDA(cudaEventElapsedTime(&a, L->bev[0], L->bev[1]));
        SAAP_CUDA(cudaEventElapsedTime(&b, L->bev[1], L->bev[2]));
        if (assign_ms) *assign_ms = a;
        if (pack_ms) *pack_ms = b;
    });
}

int saap_layer_assign_info(saap_ctx* c, const saap_layer* L, int* used_tensor_cores,
                           uint64_t* refined_keys) {
    return guard([&] {
        DeviceGuard dg(c);
        need(L, "layer");
        uint64_t n = 0;
        if (L->last_tc) {
            std::vector<uint32_t> cnt(L->n_groups);
            SAAP_CUDA(cudaMemcpyAsync(cnt.data(), L->tc_refine_count, L->n_groups * 4,
                                      cudaMemcpyDeviceToHost, c->stream));
            sync(c);
            for (uint32_t x : cnt) n += x;
        }
        if (used_tensor_cores) *used_tensor_cores = L->last_tc ? 1 : 0;
        if (refined_keys) *refined_keys = n;
    });
}

int saap_layer_read_index(saap_ctx* c, const saap_layer* L, uint64_t g, uint32_t* assignment,
                          uint64_t* off, uint64_t* idx) {
    return guard([&] {
        DeviceGuard dg(c);
        need(L, "layer");
        if (!L->built) invalid("store not built");
        if (g >= L->n_groups) invalid("group out of range");
        ensure_index(c, const_cast<saap_layer*>(L));
        const GroupMeta& gm = L->h_meta[g];
        const uint64_t ns = gm.n - gm.sink;
        const cudaStream_t st = c->stream;
        std::vector<uint32_t> off32(L->C + 1), idx32(ns);
        if (assignment) d2h(assignment, L->assign + gm.ivf_base, ns * 4, st);
        d2h(off32.data(), L->off + g * (L->C + 1), (L->C + 1) * 4, st);
        d2h(idx32.data(), L->idx + gm.ivf_base, ns * 4, st);
        sync(c);
        if (off)
            for (uint64_t i = 0; i <= L->C; ++i) off[i] = off32[i];
        if (idx)
            for (uint64_t i = 0; i < ns; ++i) idx[i] = idx32[i];
    });
}

int saap_layer_packed_rows(const saap_layer* L, void** k, void** v, uint64_t* rows) {
    return guard([&] {
        need(L, "layer");
        if (k) *k = L->K;
        if (v) *v = L->V;
        if (rows) *rows = L->cap_rows;
    });
}

static void validate_cfg(const saap_layer* L, const saap_sparse_cfg* cfg) {
    need(cfg, "sparse_attention: cfg");
    if (cfg->probes > L->C)
        invalid("sparse_attention: probes " + std::to_string(cfg->probes) +
                " exceed bucket count " + std::to_string(L->C));
    if (cfg->block_size < 1) invalid("sparse_attention: block_size must be >= 1");
    if (cfg->sink_count != L->sink)
        invalid("sparse_attention: window sinks " + std::to_string(cfg->sink_count) +
                " keys but the store indexes from id " + std::to_string(L->sink));
}

static uint64_t max_keys(const saap_layer* L) {
    uint64_t m = 0;
    for (auto& gm : L->h_meta) m = std::max<uint64_t>(m, gm.n);
    return m;
}

// given != null: the bucket lists come from the caller's BucketRouter
// ([n_groups][l_given] ids < C, attention.cpp:351) instead of a library router.
static void sparse_dev(saap_ctx* c, const saap_layer* Lc, const saap_router* const* routers,
                       const float* qr, const float* qd, uint64_t G, const saap_sparse_cfg* cfg,
                       float* out, saap_attn_stats* stats, uint32_t* selected,
                       const uint32_t* given = nullptr, uint64_t l_given = 0) {
    saap_layer* L = const_cast<saap_layer*>(Lc);
    if (!L->built) invalid("store not built");
    validate_cfg(L, cfg);
    int mode = 3, use_deroped = 1;
    const uint64_t maxn = max_keys(L);
    // routers only run when some group's context exceeds the window (attention.cpp:336-351)
    bool any_route = false;
    for (auto& gm : L->h_meta) any_route |= gm.n > cfg->sink_count + cfg->recent_count;
    uint64_t probes = cfg->probes;
    if (given) {
        if (cfg->probes > 0 && any_route && l_given > 0) {
            mode = 4;
            probes = l_given;
        } else {
            probes = 0;
        }
    } else if (cfg->probes > 0 && any_route) {
        need(routers, "sparse_attention: routers");
        bind_routers(L, routers, mode, use_deroped);
        for (uint64_t g = 0; g < L->n_groups; ++g) check_router_dims(routers[g], L->d, L->C, cfg->probes);
    }
    const float* q_route = (mode == 2 || (mode == 1 && use_deroped)) ? qd : qr;
    if (mode != 3) need(q_route, "sparse_attention: routing queries");
    uint64_t hq = 0;
    if (mode == 2) hq = L->cached_routers[0]->model->h;
    // Q-model hidden width must be uniform (kernel reads it from args)
    if (mode == 2)
        for (auto* r : L->cached_routers)
            if (r->model->h != hq) unsupported("sparse_attention: Q-models with different widths");
    (void)maxn;
    bool need_gather = false, into_region_a = false;
    for (auto& gm : L->h_meta)
        if (window_skew(gm, cfg->recent_count)) {
            const bool below = gm.n - cfg->recent_count < gm.T;  // window reaches into region A
            into_region_a |= below;
            need_gather |= below || (mode != 3 && probes > 0);
        }
    if (into_region_a) ensure_index(c, L);
    const DecodeSrc src = layer_src(L, cfg->recent_count, need_gather);
    const uint32_t nh = (uint32_t)((G + kHeadsPerSlot - 1) / kHeadsPerSlot);
    const saap_static_plan* sp = static_plan(c, L->plans, L->h_meta, 1, cfg->recent_count, nh);
    enqueue_decode(c, src, sp, mode, L->d_centT, L->d_qm, qr, q_route, G, probes,
                   cfg->recent_count, out, stats, mode == 4 ? nullptr : selected, c->opt.chunk, (uint32_t)hq,
                   mode == 1 ? L->d_cmax : nullptr, mode == 1 ? L->d_centR : nullptr,
                   mode == 1 ? (const ApproxSlot*)L->d_route_slots : nullptr, mode == 1 ? L->n_route_slots : 0,
                   mode == 2 ? L->d_qm_slots : nullptr, mode == 2 ? L->n_qm_slots : 0,
                   mode == 4 ? given : nullptr,
                   mode == 1 && !L->h_route_slots.empty() ? (const ApproxSlot*)L->h_route_slots.data() : nullptr,
                   mode == 2 && L->qm_w_finite);
}

int saap_sparse_attention_dev(saap_ctx* c, const saap_layer* L, const saap_router* const* routers,
                              const float* qr, const float* qd, uint64_t G,
                              const saap_sparse_cfg* cfg, float* out, saap_attn_stats* stats,
                              uint32_t* selected) {
    return guard([&] {
        DeviceGuard dg(c);
        need(L, "layer");
        need(qr, "sparse_attention: queries");
        need(out, "sparse_attention: out");
        if (G == 0) return;
        sparse_dev(c, L, routers, qr, qd, G, cfg, out, stats, selected);
    });
}

static bool pinned(const void* p) {
    if (!p) return true;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}
int saap_sparse_attention(saap_ctx* c, const saap_layer* L, const saap_router* const* routers,
                          const float* q_roped, const float* q_deroped, uint64_t G,
                          const saap_sparse_cfg* cfg, float* out, saap_attn_stats* stats,
                          uint32_t* selected) {
    return guard([&] {
        DeviceGuard dg(c);
        need(L, "layer");
        need(q_roped, "sparse_attention: queries");
        need(out, "sparse_attention: out");
        if (G == 0) return;
        validate_cfg(L, cfg);
        const cudaStream_t st = c->stream;
        const uint64_t qn = L->n_groups * G * L->d;
        float* dqr = (float*)ensure(c, c->qr, qn * 4);
        float* dqd = nullptr;
        // one upload when the caller passes the same rows for both roles
        const int qmode = !q_deroped ? 0 : (q_deroped == q_roped ? 1 : 2);
        if (qmode == 2) dqd = (float*)ensure(c, c->qd, qn * 4);
        // (writing the results straight into mapped pinned host memory from the
        // kernels was measured slower than one download: 4-16 byte PCIe writes)
        float* dout = (float*)ensure(c, c->out, qn * 4);
        saap_attn_stats* dst = (saap_attn_stats*)ensure(c, c->stats, L->n_groups * sizeof(saap_attn_stats));
        uint32_t* dsel = selected ? (uint32_t*)ensure(c, c->sel, L->n_groups * std::max<uint64_t>(cfg->probes, 1) * 4) : nullptr;
        if (qmode == 1) dqd = dqr;
        auto upload = [&] {
            if (qmode == 2) {
                // the two query uploads run concurrently (the attention rows on
                // a side branch), joined before the step's first kernel
                if (!c->side) {
                    SAAP_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
                    SAAP_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
                    SAAP_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
                }
                SAAP_CUDA(cudaEventRecord(c->ev_fork, st));
                SAAP_CUDA(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
                h2d(dqr, q_roped, qn * 4, c->side);
                SAAP_CUDA(cudaEventRecord(c->ev_join, c->side));
                h2d(dqd, q_deroped, qn * 4, st);
                SAAP_CUDA(cudaStreamWaitEvent(st, c->ev_join, 0));
            } else {
                h2d(dqr, q_roped, qn * 4, st);
            }
        };
        auto download = [&] {
            d2h(out, dout, qn * 4, st);
            if (stats) d2h(stats, dst, L->n_groups * sizeof(saap_attn_stats), st);
            if (selected && cfg->probes) d2h(selected, dsel, L->n_groups * cfg->probes * 4, st);
        };
        // Repeated calls with the same (layer, routers, cfg, shapes) replay a
        // CUDA graph of the step captured on the second call (the first sizes
        // the scratch); with pinned caller buffers the graph also carries the
        // uploads and downloads, so a call is one graph launch and one
        // synchronize.  Timing and trace modes stay eager.
        const bool no_graph = !c->opt.host_graph || c->opt.trace_step || c->opt.trace_decode ||
                              c->opt.trace_plan;
        saap_ctx::HostGraph* hg = nullptr;
        if (!no_graph && !c->timing) {
            const uint64_t ck[4] = {cfg->probes, cfg->block_size, cfg->sink_count, cfg->recent_count};
            for (auto& e : c->host_graphs)
                if (e.layer == L && e.routers.size() == L->n_groups &&
                    std::equal(e.routers.begin(), e.routers.end(), (const void* const*)routers) &&
                    std::equal(ck, ck + 4, e.cfg) && e.G == G && e.qmode == qmode &&
                    e.sel == (selected != nullptr) &&
                    e.h_out == out && e.h_stats == stats &&  // (mapped results are baked in)
                    (!e.copies || (e.h_qr == q_roped && e.h_qd == q_deroped && e.h_sel == selected))) {
                    hg = &e;
                    break;
                }
            if (!hg) {
                c->host_graphs.emplace_back();
                hg = &c->host_graphs.back();
                hg->layer = L;
                hg->routers.assign(routers, routers + L->n_groups);
                std::copy(ck, ck + 4, hg->cfg);
                hg->G = G;
                hg->qmode = qmode;
                hg->sel = selected != nullptr;
                hg->copies = pinned(q_roped) && (qmode != 2 || pinned(q_deroped)) && pinned(out) &&
                             pinned(stats) && pinned(selected);
                hg->h_out = out;
                hg->h_stats = stats;
                if (hg->copies) {
                    hg->h_qr = q_roped;
                    hg->h_qd = q_deroped;
                    hg->h_sel = selected;
                }
            }
        }
        if (hg && hg->exec && hg->gen == c->scratch_gen) {
            // the graph reads the layer's router tables (centroid / Q-model
            // pointers, slots), which another router set may have rewritten
            if (!std::equal(L->cached_routers.begin(), L->cached_routers.end(), hg->routers.begin(),
                            hg->routers.end())) {
                int m = 0, u = 0;
                bind_routers(const_cast<saap_layer*>(L), routers, m, u);
            }
            if (!hg->copies) upload();
            SAAP_CUDA(cudaGraphLaunch(hg->exec, st));
            c->launches += hg->nlaunch;
            if (!hg->copies) download();
        } else {
            upload();
            sparse_dev(c, L, routers, dqr, dqd, G, cfg, dout, dst, dsel);
            download();
            if (hg && hg->seen++ > 0) {
                sync(c);
                if (hg->exec) cudaGraphExecDestroy(hg->exec);
                hg->exec = nullptr;
                const uint64_t gen = c->scratch_gen, launches = c->launches;
                SAAP_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
                c->capturing = true;
                cudaGraph_t graph = nullptr;
                try {
                    if (hg->copies) upload();
                    sparse_dev(c, L, routers, dqr, dqd, G, cfg, dout, dst, dsel);
                    if (hg->copies) download();
                } catch (...) {
                    c->capturing = false;
                    cudaStreamEndCapture(st, &graph);
                    if (graph) cudaGraphDestroy(graph);
                    throw;
                }
                c->capturing = false;
                hg->nlaunch = c->launches - launches;
                c->launches = launches;  // captured, not run
                SAAP_CUDA(cudaStreamEndCapture(st, &graph));
                const cudaError_t ie = cudaGraphInstantiate(&hg->exec, graph, 0);
                cudaGraphDestroy(graph);
                SAAP_CUDA(ie);
                hg->gen = gen;
            }
        }
        sync(c);
    });
}

// sparse_attention with the bucket lists of any BucketRouter (attention.hpp:
// 102-108): selected[g * l + b] is what router.select returned for group g.
static void check_selected(const saap_layer* L, const uint32_t* selected, uint64_t l) {
    if (l > (1u << 16)) unsupported("sparse_attention: more than 65536 selected buckets per group");
    if (l) need(selected, "sparse_attention: selected buckets");
    for (uint64_t i = 0; i < L->n_groups * l; ++i)
        if (selected[i] >= L->C)
            invalid("sparse_attention: router returned bucket " + std::to_string(selected[i]) +
                    " of " + std::to_string(L->C));
}

int saap_sparse_attention_selected(saap_ctx* c, const saap_layer* L, const float* q_roped,
                                   uint64_t G, const uint32_t* selected, uint64_t l,
                                   const saap_sparse_cfg* cfg, float* out, saap_attn_stats* stats) {
    return guard([&] {
        DeviceGuard dg(c);
        need(L, "layer");
        need(q_roped, "sparse_attention: queries");
        need(out, "sparse_attention: out");
        if (G == 0) return;
        validate_cfg(L, cfg);
        check_selected(L, selected, l);
        const cudaStream_t st = c->stream;
        const uint64_t qn = L->n_groups * G * L->d;
        float* dq = (float*)ensure(c, c->qr, qn * 4);
        float* dout = (float*)ensure(c, c->out, qn * 4);
        saap_attn_stats* dst = (saap_attn_stats*)ensure(c, c->stats, L->n_groups * sizeof(saap_attn_stats));
        uint32_t* dsel = (uint32_t*)ensure(c, c->sel, std::max<uint64_t>(L->n_groups * l, 1) * 4);
        h2d(dq, q_roped, qn * 4, st);
        if (l) h2d(dsel, selected, L->n_groups * l * 4, st);
        sparse_dev(c, L, nullptr, dq, nullptr, G, cfg, dout, dst, nullptr, dsel, l);
        d2h(out, dout, qn * 4, st);
        if (stats) d2h(stats, dst, L->n_groups * sizeof(saap_attn_stats), st);
        sync(c);
    });
}

int saap_sparse_attention_selected_dev(saap_ctx* c, const saap_layer* L, const float* q_roped_dev,
                                       uint64_t G, const uint32_t* selected_dev, uint64_t l,
                                       const saap_sparse_cfg* cfg, float* out_dev,
                                       saap_attn_stats* stats_dev) {
    return guard([&] {
        DeviceGuard dg(c);
        need(L, "layer");
        need(q_roped_dev, "sparse_attention: queries");
        need(out_dev, "sparse_attention: out");
        if (G == 0) return;
        if (l > (1u << 16)) unsupported("sparse_attention: more than 65536 selected buckets per group");
        if (l) need(selected_dev, "sparse_attention: selected buckets");
        sparse_dev(c, L, nullptr, q_roped_dev, nullptr, G, cfg, out_dev, stats_dev, nullptr,
                   selected_dev, l);
    });
}

// mse(approx, exact)   attention.cpp:385-399 (host arithmetic: the
// reference's sequential fp64 sum, bit-identical)
int saap_mse(const float* approx, uint64_t rows_a, uint64_t dim_a, const float* exact,
             uint64_t rows_e, uint64_t dim_e, double* out) {
    return guard([&] {
        need(out, "mse: out");
        if (rows_a != rows_e || dim_a != dim_e)
            invalid("mse: shapes " + std::to_string(rows_a) + "x" + std::to_string(dim_a) + " vs " +
                    std::to_string(rows_e) + "x" + std::to_string(dim_e));
        const uint64_t n = rows_a * dim_a;
        if (n == 0) invalid("mse: empty inputs");
        need(approx, "mse: approx");
        need(exact, "mse: exact");
        double total = 0.0;
        for (uint64_t i = 0; i < n; ++i) {
            const double d = (double)approx[i] - (double)exact[i];
            total += d * d;
        }
        *out = total / (double)n;
    });
}

int saap_attention_mass_coverage(saap_ctx* c, const saap_layer* L, const float* q_roped,
                                 uint64_t G, const uint32_t* selected, uint64_t l, uint64_t sink,
                                 uint64_t recent, double* out) {
    return guard([&] {
        DeviceGuard dg(c);
        need(L, "layer");
        if (!L->built) invalid("store not built");
        if (sink != L->sink)
            invalid("coverage: window sinks " + std::to_string(sink) +
                    " keys but the store indexes from id " + std::to_string(L->sink));
        for (uint64_t i = 0; i < L->n_groups * l; ++i)
            if (selected[i] >= L->C) invalid("coverage: bucket id out of range");
        if (G == 0) invalid("coverage: empty query group");
        const cudaStream_t st = c->stream;
        const uint64_t qn = L->n_groups * G * L->d;
        float* dq = (float*)ensure(c, c->qr, qn * 4);
        uint32_t* dsel = (uint32_t*)ensure(c, c->sel, std::max<uint64_t>(L->n_groups * l, 1) * 4);
        double* dout = (double*)ensure(c, c->out, L->n_groups * 8);
        h2d(dq, q_roped, qn * 4, st);
        h2d(dsel, selected, L->n_groups * l * 4, st);
        launch_coverage(L->meta, (uint32_t)L->n_groups, L->K, L->posA, L->assign, dq, (uint32_t)G,
                        (uint32_t)L->d, dsel, (uint32_t)l, (uint32_t)L->C,
                        (uint32_t)std::min<uint64_t>(recent, 0xFFFFFFFFull), dout, st);
        c->launches++;
        d2h(out, dout, L->n_groups * 8, st);
        sync(c);
    });
}

int saap_layer_full_attention(saap_ctx* c, const saap_layer* L, const float* q, uint64_t G,
                              float* out) {
    return guard([&] {
        DeviceGuard dg(c);
        need(L, "layer");
        if (!L->built) invalid("store not built");
        if (G == 0) return;
        const cudaStream_t st = c->stream;
        const uint64_t qn = L->n_groups * G * L->d;
        float* dq = (float*)ensure(c, c->qr, qn * 4);
        float* dout = (float*)ensure(c, c->out, qn * 4);
        h2d(dq, q, qn * 4, st);
        const DecodeSrc src = layer_src(const_cast<saap_layer*>(L), L->recent_hint, false);
        const uint32_t nh = (uint32_t)((G + kHeadsPerSlot - 1) / kHeadsPerSlot);
        const saap_static_plan* sp = static_plan(c, const_cast<saap_layer*>(L)->plans, L->h_meta, 0, 0, nh);
        enqueue_decode(c, src, sp, 0, nullptr, nullptr, dq, nullptr, G, 0, 0, dout, nullptr, nullptr,
                       c->opt.chunk_dense);
        d2h(out, dout, qn * 4, st);
        sync(c);
    });
}

int saap_full_attention(saap_ctx* c, const float* q, uint64_t G, const float* keys,
                        const float* values, uint64_t n, uint64_t d, float* out) {
    return guard([&] {
        DeviceGuard dg(c);
        if (n == 0) invalid("full_attention: empty key set");
        if (!supported_dim(d)) unsupported("full_attention: unsupported head dim " + std::to_string(d));
        if (n >= (1ull << 30)) unsupported("full_attention: more than 2^30 keys");
        if (G == 0) return;
        const cudaStream_t st = c->stream;
        float* f32 = dmalloc<float>(n * d);
        uint16_t* Kb = dmalloc<uint16_t>(n * d);
        uint16_t* Vb = dmalloc<uint16_t>(n * d);
        h2d(f32, keys, n * d * 4, st);
        launch_f32_to_bf16(f32, Kb, n * d, st);
        h2d(f32, values, n * d * 4, st);
        launch_f32_to_bf16(f32, Vb, n * d, st);
        c->launches += 2;
        GroupMeta gm{0, 0, (uint32_t)n, 0, 0, 0};
        char* b = (char*)ensure(c, c->misc, 256 + 64);
        GroupMeta* dm = (GroupMeta*)b;
        uint64_t* drb = (uint64_t*)(b + 256);
        const uint64_t z = 0;
        h2d(dm, &gm, sizeof gm, st);
        h2d(drb, &z, 8, st);
        float* dq = (float*)ensure(c, c->qr, G * d * 4);
        float* dout = (float*)ensure(c, c->out, G * d * 4);
        h2d(dq, q, G * d * 4, st);
        (void)drb;
        DecodeSrc src;
        src.n_groups = 1;
        src.D = d;
        src.max_n = n;
        src.rows = n;
        src.meta = dm;
        src.K = Kb;
        src.V = Vb;
        std::unique_ptr<DecodeMaps> maps(build_maps(Kb, Vb, n, (uint32_t)d, nullptr, nullptr, 0));
        src.maps = maps.get();
        const uint32_t nh = (uint32_t)((G + kHeadsPerSlot - 1) / kHeadsPerSlot);
        if (c->capturing) invalid("full_attention: not capturable (uploads its keys)");
        saap_static_plan* sp = build_static_plan({gm}, 0, 0, nh);
        enqueue_decode(c, src, sp, 0, nullptr, nullptr, dq, nullptr, G, 0, 0, dout, nullptr, nullptr,
                       c->opt.chunk_dense);
        d2h(out, dout, G * d * 4, st);
        sync(c);
        free_static_plan(sp);
        cudaFree(f32);
        cudaFree(Kb);
        cudaFree(Vb);
    });
}

// ============================================================ dense baseline cache
int saap_kvcache_create(saap_ctx* c, uint64_t n_groups, uint64_t d, const void* K, const void* V,
                        const uint64_t* row_base, const uint64_t* n_keys, saap_kvcache** out) {
    return guard([&] {
        DeviceGuard dg(c);
        if (!supported_dim(d)) unsupported("kvcache: unsupported head dim " + std::to_string(d));
        need(K, "kvcache: keys");
        need(V, "kvcache: values");
        auto* kc = new saap_kvcache;
        kc->ctx = c;
        kc->n_groups = n_groups;
        kc->d = d;
        kc->K = (const uint16_t*)K;
        kc->V = (const uint16_t*)V;
        std::vector<GroupMeta> m(n_groups);
        for (uint64_t g = 0; g < n_groups; ++g) {
            if (n_keys[g] == 0) {
                delete kc;
                invalid("full_attention: empty key set");
            }
            m[g] = GroupMeta{row_base[g], 0, (uint32_t)n_keys[g], 0, 0, 0};
            kc->max_n = std::max<uint64_t>(kc->max_n, n_keys[g]);
            kc->rows = std::max<uint64_t>(kc->rows, row_base[g] + n_keys[g]);
        }
        kc->h_meta = m;
        kc->maps = build_maps(K, V, kc->rows, (uint32_t)d, nullptr, nullptr, 0);
        kc->meta = dmalloc<GroupMeta>(n_groups);
        kc->row_base = dmalloc<uint64_t>(n_groups);
        SAAP_CUDA(cudaMemcpy(kc->meta, m.data(), n_groups * sizeof(GroupMeta), cudaMemcpyHostToDevice));
        SAAP_CUDA(cudaMemcpy(kc->row_base, row_base, n_groups * 8, cudaMemcpyHostToDevice));
        *out = kc;
    });
}

int saap_kvcache_destroy(saap_kvcache* kc) {
    return guard([&] {
        if (!kc) return;
        cudaSetDevice(kc->ctx->device);
        dfree(kc->meta);
        dfree(kc->row_base);
        for (auto* p : kc->plans) free_static_plan(p);
        delete (DecodeMaps*)kc->maps;
        delete kc;
    });
}

int saap_dense_attention_dev(saap_ctx* c, const saap_kvcache* kc, const float* q, uint64_t G,
                             float* out) {
    return guard([&] {
        DeviceGuard dg(c);
        need(kc, "kvcache");
        if (G == 0) return;
        DecodeSrc src;
        src.n_groups = kc->n_groups;
        src.D = kc->d;
        src.max_n = kc->max_n;
        src.rows = kc->rows;
        src.meta = kc->meta;
        src.K = kc->K;
        src.V = kc->V;
        src.maps = (const DecodeMaps*)kc->maps;
        const uint32_t nh = (uint32_t)((G + kHeadsPerSlot - 1) / kHeadsPerSlot);
        const saap_static_plan* sp =
                static_plan(c, const_cast<saap_kvcache*>(kc)->plans, kc->h_meta, 0, 0, nh);
        enqueue_decode(c, src, sp, 0, nullptr, nullptr, q, nullptr, G, 0, 0, out, nullptr, nullptr,
                       c->opt.chunk_dense);
    });
}

// ============================================================ graphs
int saap_graph_begin(saap_ctx* c) {
    return guard([&] {
        DeviceGuard dg(c);
        SAAP_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        c->capturing = true;
    });
}

int saap_graph_end(saap_ctx* c, saap_graph** out) {
    return guard([&] {
        DeviceGuard dg(c);
        c->capturing = false;
        auto* g = new saap_graph;
        SAAP_CUDA(cudaStreamEndCapture(c->stream, &g->graph));
        SAAP_CUDA(cudaGraphInstantiate(&g->exec, g->graph, 0));
        *out = g;
    });
}

int saap_graph_launch(saap_ctx* c, saap_graph* g) {
    return guard([&] {
        need(g, "graph");
        SAAP_CUDA(cudaGraphLaunch(g->exec, c->stream));
    });
}

int saap_graph_destroy(saap_graph* g) {
    return guard([&] {
        if (!g) return;
        if (g->exec) cudaGraphExecDestroy(g->exec);
        if (g->graph) cudaGraphDestroy(g->graph);
        delete g;
    });
}

// ============================================================ diagnostics
int saap_debug_exp(saap_ctx* c, const double* x, uint64_t n, double* out) {
    return guard([&] {
        DeviceGuard dg(c);
        if (!n) return;
        double* dx = (double*)ensure(c, c->misc, n * 16);
        h2d(dx, x, n * 8, c->stream);
        launch_debug_exp(dx, n, dx + n, c->stream);
        c->launches++;
        d2h(out, dx + n, n * 8, c->stream);
        sync(c);
    });
}

int saap_debug_plan_trace(saap_ctx* c, uint64_t* out) {
    return guard([&] {
        DeviceGuard dg(c);
        if (!c->trace.p) invalid("plan tracing off: set option trace_plan before the first decode");
        d2h(out, c->trace.p, 128 + 48 * 1024, c->stream);
        sync(c);
    });
}

// Between decode steps every per-step counter and flag must be back at zero
// (the last decode CTA, the combine and the producer re-arm them).  out[8]:
// {tickets, dyn reserved, planner groups, published, exited, nonzero run
// counters, nonzero done counters + dyn counts, nonzero part/ready flags}.
int saap_debug_step_state(saap_ctx* c, uint64_t* out) {
    return guard([&] {
        DeviceGuard dg(c);
        need(out, "out");
        sync(c);
        StepCounters h{};
        SAAP_CUDA(cudaMemcpy(&h, c->counters, sizeof h, cudaMemcpyDeviceToHost));
        out[0] = h.tickets;
        out[1] = (uint32_t)h.dynres;
        out[2] = (uint32_t)(h.dynres >> 32);
        out[3] = h.published;
        out[4] = h.exited;
        auto nonzero = [](const void* d, size_t bytes) {
            std::vector<uint32_t> v(bytes / 4);
            if (!v.empty()) SAAP_CUDA(cudaMemcpy(v.data(), d, v.size() * 4, cudaMemcpyDeviceToHost));
            uint64_t n = 0;
            for (uint32_t x : v) n += x != 0;
            return n;
        };
        out[5] = c->runs.p ? nonzero(c->runs.p, c->runs.cap) : 0;
        out[6] = c->dyn_cnt.p ? nonzero(c->dyn_cnt.p, c->dyn_cnt.cap) : 0;
        uint64_t flags = c->part_flag.p ? nonzero(c->part_flag.p, c->part_flag.cap) : 0;
        if (c->tiles.p) {
            std::vector<TileRec> t(c->tiles.cap / sizeof(TileRec));
            SAAP_CUDA(cudaMemcpy(t.data(), c->tiles.p, t.size() * sizeof(TileRec), cudaMemcpyDeviceToHost));
            for (auto& r : t) flags += r.ready != 0;
        }
        out[7] = flags;
    });
}

int saap_debug_step_trace(saap_ctx* c, uint64_t* out, int reset) {
    return guard([&] {
        DeviceGuard dg(c);
        if (!c->tl) invalid("step tracing off: saap_ctx_set_option(ctx, \"trace_step\", 1) first");
        if (reset) {
            uint64_t init[16];
            for (int k = 0; k < 8; ++k) {
                init[2 * k] = ~0ull;
                init[2 * k + 1] = 0;
            }
            h2d(c->tl, init, 128, c->stream);
        } else {
            d2h(out, c->tl, 128, c->stream);
        }
        sync(c);
    });
}

int saap_debug_decode_trace(saap_ctx* c, uint64_t* out, uint64_t n_ctas) {
    return guard([&] {
        DeviceGuard dg(c);
        if (!c->dtrace.p) invalid("decode tracing off: set option trace_decode before the first decode");
        if (n_ctas > (uint64_t)c->sm_count) invalid("decode trace: more CTAs than SMs");
        d2h(out, c->dtrace.p, n_ctas * 128, c->stream);
        sync(c);
    });
}

// With option trace_decode set: per attention CTA of the last decode step,
// kTraceTiles x {TMA issued | flags, data landed, consumed, producer phase stamps x5}.
int saap_debug_decode_tiles(saap_ctx* c, uint64_t* out, uint64_t n_ctas) {
    return guard([&] {
        DeviceGuard dg(c);
        if (!c->dtrace.p) invalid("decode tracing off: set option trace_decode before the first decode");
        if (n_ctas > (uint64_t)c->sm_count) invalid("debug_decode_tiles: n_ctas > SM count");
        d2h(out, (char*)c->dtrace.p + (size_t)c->sm_count * 128, n_ctas * kTraceTiles * 64, c->stream);
        sync(c);
    });
}

// ============================================================ synthetic data
int saap_synth_fill_dev(saap_ctx* c, void* out, uint64_t rows, uint64_t d, uint64_t seed, int kind,
                        const float* centers, uint64_t n_centers, float center_scale, float noise) {
    return guard([&] {
        DeviceGuard dg(c);
        need(out, "synth: out");
        if (kind == 1 && (!centers || n_centers == 0)) invalid("synth: clustered keys need centers");
        launch_synth((uint16_t*)out, rows, (uint32_t)d, seed, kind, centers, n_centers, center_scale,
                     noise, c->stream);
        c->launches++;
    });
}

}  // extern "C"
