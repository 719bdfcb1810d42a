// Shared device helpers and internal types of libsaap_b200 (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "saap_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libsaap_b200 is written for sm_100a (B200) only"
#endif

namespace saap_b200 {

// ---------------------------------------------------------------- errors
struct Error {
    int code;
    std::string msg;
};
void set_error(const std::string& m);
[[noreturn]] void fail(int code, const std::string& msg);
void check_cuda(cudaError_t e, const char* what);
#define SAAP_CUDA(x) ::saap_b200::check_cuda((x), #x)

// Launch with programmatic stream serialization (PDL): the kernel may be
// scheduled while the previous kernel on the stream drains; it must call
// pdl_wait() before touching that kernel's outputs.  Captured into graphs as
// programmatic edges.
template <typename... KArgs, typename... Args>
void launch_pdl(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    check_cuda(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx");
}

// ---------------------------------------------------------------- layout
// One (sequence, KV head) context of a layer.
struct GroupMeta {
    uint64_t row_base;  // first packed K/V row of this group
    uint64_t ivf_base;  // first entry of this group in assign/idx/invA (sum of N_s before)
    uint32_t n;         // keys incl. the sink span
    uint32_t sink;      // id_offset
    uint32_t T;         // rows [sink,T) bucket-packed, [T,n) position order
    uint32_t pad;
};

enum : uint32_t { KIND_ROWS = 0, KIND_INVA = 1, KIND_LIST = 2 };

constexpr uint32_t kPackTile = 2048;  // local ids per histogram / assignment tile

struct TileDesc {
    uint32_t group;
    uint32_t first;  // first local id (0-based, after the sink span)
    uint32_t count;
    uint32_t pad;
};

// Per-step device counters.  Zero at allocation; the last decode CTA of a
// step resets them for the next step (every reader has finished by then).
struct StepCounters {
    unsigned long long dynres;  // (planner CTAs that reserved << 32) | dynamic tiles reserved
    uint32_t published;         // planner CTAs whose tiles are all published
    uint32_t tickets;           // work-stream tickets handed out beyond the static first batch
    uint32_t exited;            // decode CTAs finished
    uint32_t pad[27];
};

constexpr int kHeadsPerSlot = 4;  // query heads processed together (GQA group)
constexpr int kTileKeys = 64;     // keys per smem stage
constexpr int kComputeWarps = 8;

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ float bf16lo(uint32_t x) { return __uint_as_float(x << 16); }
__device__ __forceinline__ float bf16hi(uint32_t x) { return __uint_as_float(x & 0xFFFF0000u); }

__device__ __forceinline__ uint16_t f32_to_bf16_rne(float f) {
    uint32_t u = __float_as_uint(f);
    uint32_t lsb = (u >> 16) & 1u;
    return (uint16_t)((u + 0x7FFFu + lsb) >> 16);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    return ok != 0;
}
// non-blocking test of a phase's completion
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
// 1-D bulk copy global -> shared (TMA engine), completes tx bytes on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(dst)),
            "l"(src), "r"(bytes), "r"(smem_u32(bar))
            : "memory");
}
// Programmatic dependent launch: a kernel launched with launch_pdl() may start
// while its predecessor drains; pdl_wait() blocks until the predecessor grid
// has completed and its writes are visible (no-op without the attribute).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long atom_acq_rel_add_u64(unsigned long long* p,
                                                                unsigned long long v) {
    unsigned long long old;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
    return old;
}
__device__ __forceinline__ uint32_t atom_acq_rel_add_u32(uint32_t* p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void red_release_add_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// debug step timeline: kernel k's first start / last end (globaltimer ns)
__device__ __forceinline__ void tl_mark(unsigned long long* tl, int k, bool start) {
    if (!tl) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    if (start) atomicMin(tl + 2 * k, t);
    else atomicMax(tl + 2 * k + 1, t);
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ---------------------------------------------------------------- host side
struct LaunchCounter {
    uint64_t n = 0;
};

}  // namespace saap_b200

// ---------------------------------------------------------------- handles
struct saap_scratch {
    void* p = nullptr;
    size_t cap = 0;
};

struct saap_p2p;
struct saap_ctx {
    int device = 0;
    int sm_count = 0;
    // attached fused output exchange (saap_p2p_attach)
    saap_p2p* p2p = nullptr;
    uint32_t p2p_hl = 0, p2p_h0 = 0, p2p_kvh = 0;
    cudaStream_t stream = nullptr;
    // host API: the two query uploads run on parallel branches
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool own_stream = false;
    uint64_t launches = 0;
    // growable device scratch (sized by uncaptured calls; graphs reuse it)
    saap_scratch approx, trace, dtrace, cand_s, cand_i, tiles, part_O, part_ml, probs, stats, sel, qr, qd, out, misc, zeros;
    saap_scratch runs, dyn_cnt, part_flag;  // zero between steps (the combine re-arms them)
    unsigned long long* tl = nullptr;  // debug step timeline (option trace_step)
    saap_b200::StepCounters* counters = nullptr;  // persistent, 128 B
    // host-API graph cache (saap_sparse_attention): graphs reference scratch,
    // so any scratch reallocation bumps scratch_gen and retires them
    uint64_t scratch_gen = 0;
    struct HostGraph {
        const void* layer = nullptr;
        std::vector<const void*> routers;
        uint64_t cfg[4] = {}, G = 0, gen = 0;
        int qmode = 0, sel = 0, seen = 0;
        // pinned caller buffers: the graph carries the copies too (H2D queries,
        // D2H outputs / counters / lists); null: copies outside the graph
        const void *h_qr = nullptr, *h_qd = nullptr;
        void *h_out = nullptr, *h_stats = nullptr, *h_sel = nullptr;
        bool copies = false;
        uint64_t nlaunch = 0;  // kernels in the captured step
        cudaGraphExec_t exec = nullptr;
    };
    std::vector<HostGraph> host_graphs;
    // capture state
    bool capturing = false;
    int assign_mode = 0;  // 0: tcgen05 path where applicable, 1: exact CUDA-core only
    // optional per-kernel timing (eager steps)
    bool timing = false;
    std::vector<cudaEvent_t> ev;  // triples: before plan, before attention, after
    // tuning / diagnostics, per context (saap_ctx_set_option; no environment reads)
    struct Options {
        uint32_t chunk = 8;             // work-stream tiles per decode ticket (sparse)
        uint32_t chunk_dense = 16;      // ... (dense / full attention)
        uint32_t tail_per_cta = 1;      // (unused since guided claims)
        uint32_t min_chunk = 4;         // smallest guided claim at the stream's end (tiles)
        uint32_t chunk_st = 0;          // pre-assigned window tiles per decode CTA (0: 2)
        uint32_t claim_lead = 3;        // decode producer: claim when <= this many tiles are left to issue
        uint32_t assign_f32_tc = 1;     // f32 assignment keys on tcgen05 (split keys); 0: fp64 kernel
        uint32_t qm_logits = 0;         // Q-model logits geometry (route.cu launch_qmodel_probs)
        uint32_t decode_tc = 0;         // 1: tcgen05 consumers (d = 128)
        uint32_t inflight = 0;          // ... 0: ring depth, else max tiles issued and unconsumed
        uint32_t fetch_lead = 2;        // ... fetch the next records when <= this many are left
        uint32_t decode_poll_ns = 100;  // producer back-off while waiting for the planner
        uint32_t combine_poll_ns = 1000;  // combine back-off while no run is published
        uint32_t decode_wait = 0;       // 1: decode waits for routing to finish (PDL grid wait)
        uint32_t debug_skip = 0;        // profiling only (wrong outputs): 1 skip consumer math, 2 skip K/V loads
        uint32_t cluster_route = 1;     // 0: force the general routing path
        uint32_t host_graph = 1;        // 0: saap_sparse_attention never replays graphs
        uint32_t trace_step = 0;        // step timeline (saap_debug_step_trace)
        uint32_t trace_decode = 0;      // per-CTA decode timeline (saap_debug_decode_trace)
        uint32_t trace_plan = 0;        // routing phases (saap_debug_plan_trace)
    } opt;
};

// Host-planned static part of a decode work stream (the dense window, or
// every row for full attention) for one (cache, mode, recent, head chunks).
struct saap_static_plan {
    int mode = 0;
    uint64_t recent = 0;
    uint32_t n_hchunks = 0;
    void* tiles = nullptr;      // TileRec[n_tiles] (device)
    uint32_t n_tiles = 0;
    uint32_t* cnt = nullptr;    // [qslots] static tiles per query slot (device)
    uint32_t max_slot_tiles = 0;
    size_t cap_tiles = 0;  // TileRec capacity of `tiles`
    bool stale = false;    // the layout grew (append): rebuild in place before use
};

struct saap_partition {
    saap_ctx* ctx = nullptr;
    uint64_t C = 0, d = 0;
    float* cent = nullptr;     // C x d f32 (device)
    double* cent64 = nullptr;  // C x d fp64 (device, exact assignment)
    float* centT = nullptr;    // d x C f32 (device, routing slabs; exact in fp64)
    float* centB = nullptr;    // [8][d][C/8] f32: centT blocked by cluster rank (one bulk copy per slab)
    float cmax = 0.f;          // max centroid L2 norm (routing error bound)
    std::vector<float> host;   // kept for validation / read-back
};

struct saap_qmodel {
    saap_ctx* ctx = nullptr;
    uint64_t d = 0, h = 0, C = 0;
    double* w1 = nullptr;  // d x h
    double* w2 = nullptr;  // h x C
    double* vec = nullptr; // b1, gamma, beta, mean, var (5 x h) then b2 (C)
    bool w_finite = false;   // every W1 / W2 weight finite: a zero input's term adds exactly +-0
};

// Q-model trainer (qtrain.cu): model + TrainerState resident on the device.
struct saap_qtrainer {
    saap_ctx* ctx = nullptr;
    uint64_t d = 0, h = 0, C = 0;
    double lr = 1e-5, beta1 = 0.9, beta2 = 0.999, eps = 1e-8, bn_momentum = 0.9;
    uint64_t step = 0;
    // params in checkpoint order: w1 [d x h], b1, gamma, beta, run_mean,
    // run_var [h], w2 [h x C], b2 [C]; Adam moments for the 6 trained ones
    double* p[8] = {};
    double* m[8] = {};
    double* v[8] = {};
    // activations / grads (capacity n_cap rows)
    uint64_t n_cap = 0;
    double *x = nullptr, *z = nullptr, *xhat = nullptr, *y = nullptr, *r = nullptr, *pr = nullptr,
           *tgt = nullptr, *dl = nullptr, *dy = nullptr, *dz = nullptr, *w2T = nullptr;
    double *mean = nullptr, *var = nullptr, *g[8] = {}, *loss_rows = nullptr, *loss = nullptr;
    float* q32 = nullptr;
};

// PartialAccumulator on the device (accum.cu): out_acc [heads x dv], sumexp,
// runmax (fp64), plus absorb scratch.
struct saap_accum {
    saap_ctx* ctx = nullptr;
    uint64_t heads = 0, dv = 0;
    double* out = nullptr;
    double* sumexp = nullptr;
    double* runmax = nullptr;
    double* rescale = nullptr;
};

struct saap_router {
    int kind = 0;  // 0 centroid, 1 qmodel
    int use_deroped = 1;
    const saap_partition* part = nullptr;
    const saap_qmodel* model = nullptr;
};

struct saap_layer {
    saap_ctx* ctx = nullptr;
    uint64_t n_groups = 0, d = 0, C = 0, sink = 0, recent_hint = 0;
    uint64_t total_rows = 0, total_ns = 0;  // source rows / keys (sum of n, n - sink)
    uint64_t cap_rows = 0, cap_ns = 0;       // layer extents (per-group capacity)
    std::vector<uint64_t> h_src0;            // per group: first source row (sum of n before)
    uint64_t* src_row0 = nullptr;            // device copy of h_src0
    std::vector<uint64_t> h_cap;             // per group: row capacity (>= n)
    bool appended = false;                   // keys were appended after the build
    bool idx_stale = false;                  // idx not yet re-sorted after an append
    std::vector<saap_b200::GroupMeta> h_meta;
    saap_b200::GroupMeta* meta = nullptr;
    uint64_t* row_base = nullptr;  // device copy of h_meta[].row_base
    uint16_t* K = nullptr;         // packed bf16 rows
    uint16_t* V = nullptr;
    uint32_t* assign = nullptr;  // total_ns
    uint32_t* idx = nullptr;     // total_ns (local ids, ascending within bucket)
    uint32_t* invA = nullptr;    // total_ns: position-sink -> packed row (region A)
    uint32_t* posA = nullptr;    // total_ns: packed row-sink -> position (region A)
    uint32_t* list = nullptr;    // total_ns: packing scratch (destination row per key)
    uint32_t* off = nullptr;     // n_groups x (C+1)
    uint32_t* offA = nullptr;    // n_groups x (C+1)
    bool built = false;
    // prefill work decomposition
    saap_b200::TileDesc* tiles = nullptr;
    uint32_t n_tiles = 0;
    uint32_t* tile_first = nullptr;  // n_groups + 1
    uint32_t* hist = nullptr;        // n_tiles x C
    uint32_t* countA = nullptr;      // n_groups x C
    const double** d_cent64 = nullptr;  // per group partition (exact assignment)
    std::vector<const saap_partition*> parts;
    // tcgen05 assignment resources
    void* tc_tiles = nullptr;
    uint32_t tc_n_tiles = 0;
    uint16_t* tc_hi = nullptr;
    uint16_t* tc_mid = nullptr;
    size_t tc_split_elems = 0;
    float* tc_cmax = nullptr;
    uint32_t* tc_refine = nullptr;   // total_ns: per-group lists of ambiguous keys
    uint32_t* tc_refine_count = nullptr;  // n_groups
    uint64_t* key_row0 = nullptr;    // per group: row_base + sink
    uint64_t* ivf_base = nullptr;    // per group
    uint64_t last_refined = 0;
    bool last_tc = false;
    std::vector<const saap_partition*> tc_parts;  // partitions the tc resources were built for
    bool tc_split = false;                         // tc tile list built for split (f32-key) mode
    uint16_t* split_hi = nullptr;                  // f32 assignment keys split into bf16 terms
    uint16_t* split_lo = nullptr;
    uint64_t split_elems = 0;
    uint32_t tc_nslots = 0;
    cudaEvent_t bev[3] = {nullptr, nullptr, nullptr};  // last build: start, after assign, after pack
    // routing parameter table cache (device arrays of per-group pointers)
    std::vector<const saap_router*> cached_routers;
    const float** d_centT = nullptr;   // per group centT
    const float** d_centR = nullptr;   // per group row-major centroids
    float* d_cmax = nullptr;           // per group partition cmax
    void* d_route_slots = nullptr;     // ApproxSlot[]: approximate-scoring slots (<= 8 contexts of one partition)
    uint32_t n_route_slots = 0;
    bool qm_w_finite = false;   // every bound Q-model's weights are finite
    std::vector<uint8_t> h_route_slots;  // host copy of the ApproxSlot table (inlined into the routing launch)
    const double** d_qm = nullptr;     // per group: w1, w2, vec (3 pointers)
    uint32_t* d_qm_slots = nullptr;    // [n_qm_slots][kQmSlot] contexts sharing a Q-model
    uint32_t n_qm_slots = 0;
    // decode: TMA maps over the packed cache (+ gather buffer), built lazily
    void* maps = nullptr;              // DecodeMaps (host copy)
    uint16_t* gK = nullptr;            // gather buffer for general windows
    uint16_t* gV = nullptr;
    uint64_t gather_cap = 0;           // rows per group
    std::vector<saap_static_plan*> plans;  // static work streams by (mode, recent, head chunks)
};

struct saap_kvcache {
    saap_ctx* ctx = nullptr;
    uint64_t n_groups = 0, d = 0, max_n = 0, rows = 0;
    const uint16_t* K = nullptr;  // borrowed
    const uint16_t* V = nullptr;
    saap_b200::GroupMeta* meta = nullptr;
    uint64_t* row_base = nullptr;
    void* maps = nullptr;  // DecodeMaps
    std::vector<saap_b200::GroupMeta> h_meta;
    std::vector<saap_static_plan*> plans;
};

struct saap_graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
};
