// Argument blocks of the decode-side kernels (shared by the .cu files).
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace saap_b200 {

constexpr int kTileRows = 128;   // smem rows per decode tile (8 warps x 16 keys)
constexpr int kMaxPieces = 16;   // contiguous row runs per tile (each >= 8 virtual rows)
constexpr int kSliceMax = 1024;  // centroids scored by one routing CTA
constexpr int kPlanThreads = 1024;

// A contiguous run of cache rows placed at smem row `srow` of a tile.
struct PieceRec {
    uint32_t len;    // rows (<= 128; loaded rounded up to 8) | 0x80000000 if gather buffer
    uint32_t srow;   // first smem row (multiple of 8)
    uint64_t row;    // first row in its tensor (layer cache or gather buffer)
};
// One 128-row tile of decode work for one query slot.  The decode work
// stream is [static tiles | dynamic tiles]: static tiles (the dense window:
// sink + recent tail, or every row for full attention) are planned on the host
// once per (cache, window, heads) and are ready when the step starts; dynamic
// tiles (selected buckets, general-window gathers) are appended by the
// planner and published through `ready` (the decode producer clears it).
struct alignas(16) TileRec {
    uint32_t npieces;
    uint32_t qslot;  // group * n_hchunks + head chunk
    uint32_t ready;  // dynamic tiles: 1 = published
    uint32_t end;    // 1: last tile of its slot's contiguous range (a run ends here)
    // derived from the pieces by the planner (tile_finish), so the decode's
    // TMA issuer reads them instead of reducing over the pieces per tile
    uint32_t rows8;     // sum of the pieces' 8-rounded rows (bytes = rows8 * 2 * row bytes)
    uint32_t pad[3];
    uint32_t valid[4];  // 128-bit mask of the tile's valid smem rows
    PieceRec p[kMaxPieces];
};
// rows8 and the validity mask of a tile whose pieces are set
__host__ __device__ inline void tile_finish(TileRec& t) {
    uint32_t r8 = 0, vm[4] = {0u, 0u, 0u, 0u};
    for (uint32_t i = 0; i < t.npieces; ++i) {
        const uint32_t len = t.p[i].len & 0x7FFFFFFFu, s0 = t.p[i].srow;
        r8 += (len + 7) & ~7u;
        for (uint32_t r = s0; r < s0 + len && r < 128; ++r) vm[r >> 5] |= 1u << (r & 31);
    }
    t.rows8 = r8;
    t.pad[0] = t.pad[1] = t.pad[2] = 0;
    for (int q = 0; q < 4; ++q) t.valid[q] = vm[q];
}
constexpr uint32_t kPieceGather = 0x80000000u;

// Routing, stage 1: one CTA scores a slice of <= kSliceMax centroids and
// keeps its top-min(l, slice) (score, id) pairs in reference order.
struct RouteArgs {
    int mode;                      // 1 centroid, 2 precomputed Q-model probabilities
    const float* const* centT;     // per group, d x C f32 (exact in fp64)
    const float* q_route;          // [groups][G][D]
    const double* scores;          // [groups][G][C]
    uint32_t G, D, C, probes;
    uint32_t slice, n_slices, keep;  // keep = min(probes, slice)
    double* cand_s;                // [groups][n_slices][keep]
    uint32_t* cand_i;
};
// Routing, approximate stage (centroid router, C <= kPlanThreads): fp32
// scores of every centroid for every context.  Contexts sharing one
// partition (same KV head, different sequences) form a slot and share each
// centroid load.
constexpr int kSlotGroups = 8;  // contexts per approximate-scoring slot
struct ApproxSlot {
    const float* centT;            // d x C f32 of the slot's partition
    const float* centB;            // [8][d][C/8] blocked copy (cluster routing; null if C % 8)
    uint32_t count;                // member contexts (<= kSlotGroups)
    uint32_t group[kSlotGroups];
    uint32_t pad;
};
struct ApproxArgs {
    const float* const* centT;     // per group, d x C f32 (slots == null: slot s = group s)
    const ApproxSlot* slots;       // one load gives the centroids and the members
    const float* q_route;          // [groups][G][D]
    uint32_t G, C;
    float* approx;                 // [groups][C]
    unsigned long long* tl;        // debug step timeline (null: off)
};
// Fused routing + planning for the centroid router (C <= 1024, power of two):
// one cluster of 8 CTAs per approximate-scoring slot.
constexpr int kInlineSlots = 16;  // slot table carried in the launch parameters
struct ClusterRouteArgs {
    ApproxSlot islots[kInlineSlots];  // slots [0, n_inline) (else read from `slots`)
    uint32_t n_inline;
    const ApproxSlot* slots;
    const GroupMeta* meta;
    const uint32_t* off;
    const uint32_t* offA;
    const float* q_route;        // [groups][G][D]
    const float* const* centR;   // per group C x d f32 centroids (exact re-scoring)
    const float* cmax;           // per group max centroid norm
    uint32_t G, C, probes, recent, n_hchunks;
    TileRec* dyn_tiles;
    StepCounters* ctr;
    uint32_t* dyn_cnt;
    saap_attn_stats* stats;
    uint32_t* selected;          // nullable [groups][probes]
    unsigned long long* trace;   // debug: clock64 per phase (slot 0, rank 0)
    unsigned long long* tl;      // debug step timeline (null: off)
};
constexpr int kClusterCtas = 8;
constexpr int kClusterThreads = 512;

struct PlanArgs {
    const GroupMeta* meta;
    const uint32_t* off;
    const uint32_t* offA;
    const uint32_t* idx;
    const uint32_t* assign;
    const uint32_t* invA;
    uint32_t C;
    int mode;                    // 0 dense, 1 centroid, 2 precomputed scores, 3 window only,
                                 // 4 caller-selected bucket lists (`given`)
    const float* q_route;        // [groups][G][D]
    const double* scores;        // [groups][G][C] per-row probabilities (mode 2)
    uint32_t G, D, n_hchunks;
    uint32_t probes, recent;
    uint32_t P2;                 // pow2 >= n_slices * keep (candidates to merge)
    uint32_t n_cand;             // n_slices * keep
    const double* cand_s;        // routing candidates from route_score_kernel
    const uint32_t* cand_i;
    const float* approx;         // centroid router, C <= 1024: fp32 scores [groups][C]
    const float* const* centT;   // per group d x C f32 centroids (exact re-scoring)
    const float* const* centR;   // per group C x d f32 centroids (row-major)
    const float* cmax;           // per group max centroid norm
    unsigned long long* trace;   // debug: clock64 per planning phase (CTA 0)
    unsigned long long* tl;      // debug step timeline (null: off)
    int route_only;              // BucketRouter::select: write `selected`, plan nothing
    // general-window rows are gathered into a contiguous buffer
    const uint16_t* K;
    const uint16_t* V;
    uint16_t* gK;
    uint16_t* gV;
    uint64_t gather_cap;         // rows per group in the gather buffer
    // outputs
    TileRec* dyn_tiles;          // dynamic part of the work stream
    StepCounters* ctr;           // dyn (tiles reserved), groups_done
    uint32_t* dyn_cnt;           // [qslots] dynamic tiles | kCntValid
    saap_attn_stats* stats;
    uint32_t* selected;          // nullable [groups][probes]
    const uint32_t* given;       // mode 4: [groups][probes] bucket ids from the caller's router
};
constexpr uint32_t kCntValid = 0x80000000u;
constexpr int kTraceTiles = 48;  // debug tile stamps per decode CTA

struct DecodeArgs {
    const TileRec* st_tiles;   // static part of the work stream [n_static]
    TileRec* dyn_tiles;        // dynamic part (ready flags cleared after use)
    uint32_t n_static;
    uint32_t n_plan_groups;    // planner CTAs that publish dynamic tiles (0: static only)
    uint32_t chunk;            // work-stream tiles per ticket (dynamic part)
    uint32_t chunk_st;         // tiles per ticket in the static part
    uint32_t tail;             // the stream's last `tail` tiles go out one per ticket
    uint32_t wait_plan;        // 1: wait for the planner grid before streaming
    uint32_t debug_skip;       // profiling only: 1 consumers skip the math, 2 producer skips TMA
    uint32_t min_chunk;        // smallest guided claim (tiles)
    uint32_t claim_lead;       // claim the next chunk when <= this many tiles of the current one are unissued
    uint32_t inflight;         // 0: ring depth; else at most this many tiles issued and unconsumed
    uint32_t fetch_lead;       // fetch the next unit's records at <= this many unissued tiles
    uint32_t poll_ns;          // producer's sleep between polls for planner tiles
    StepCounters* ctr;
    const float* q;            // [groups][G][D] attention queries (f32)
    uint32_t G;
    uint32_t n_hchunks;
    float qscale;  // log2(e)/sqrt(d): scores live in the exp2 domain
    float* part_O;   // [qslots][run_cap][4][D] unnormalised run partials
    float* part_ml;  // [qslots][run_cap][8]: m then l
    uint32_t* part_flag;  // [qslots][run_cap] run partial published
    uint32_t run_cap;
    unsigned long long* rd;  // [qslots] (runs reserved << 32) | tiles published
    unsigned long long* dtrace;  // debug: per CTA {start, first tile, end (globaltimer ns), tiles}
    unsigned long long* dtiles;  // debug: per CTA x 48 tiles {TMA issued, data landed, consumed}
    unsigned long long* tl;      // debug step timeline (null: off)
};

struct CombineArgs {
    const uint32_t* st_cnt;  // [qslots] static tiles
    uint32_t* dyn_cnt;       // [qslots] dynamic tiles | kCntValid (null: static only)
    unsigned long long* rd;  // [qslots] (runs reserved << 32) | tiles published
    const float* part_O;
    const float* part_ml;
    uint32_t* part_flag;
    uint32_t run_cap;
    uint32_t G, n_hchunks;
    uint32_t poll_ns;        // sleep between polls without progress
    float* out;
    unsigned long long* tl;  // debug step timeline (null: off)
    // fused output exchange (saap_p2p): every rank's full buffer and counter
    float* const* p2p_out;   // [p2p_n] (null: off)
    uint32_t* const* p2p_flag;
    uint32_t p2p_n, p2p_hl, p2p_h0, p2p_kvh;
};

// Decode tiles live in shared memory as 8-row groups [group][half][8 rows][HALF
// bytes] (HALF = min(row bytes, 128), TMA-swizzled).  One 4-D TMA request
// moves 8*G rows (G = 1..16) of both halves of K (or V) straight into that
// layout: dims {HALF elems, rows, halves, 16 groups} with strides {row, HALF,
// 8 rows} (the group dimension overlaps the row dimension on purpose, so a
// piece of any 8-row multiple is one request).  The 64 maps (K, V, gather K,
// gather V) x 16 heights live in device memory.
constexpr int kBoxSizes = 16;  // boxes of 8, 16, ..., 128 rows
// Passed by value as a __grid_constant__ kernel parameter (8 KB): descriptors
// in parameter space are per launch, never served stale from the TMA
// descriptor cache (device-memory maps at a reused address would be).
struct DecodeMaps {
    CUtensorMap map[4 * kBoxSizes];  // [K, V, gather K, gather V][height]
    uint64_t rows = 0, grows = 0;
};

struct QModelArgs {
    const float* q;            // [groups][G][d] de-roped queries
    const double* const* prm;  // per group: w1, w2, vec (3 pointers)
    uint32_t G, d, h, C;
    double* probs;             // [groups][G][C]
    double* hid;               // [groups][G][h] scratch: post-ReLU hidden rows
    const uint32_t* slot_g;    // optional [n_slots][kQmSlot] groups sharing one model (pad ~0u)
    uint32_t logits_variant;   // qm_logits geometry (rows per thread, CTA width); see launch_qmodel_probs
    uint32_t w_finite;         // 1: W1 and W2 finite, the zero-skip test of mm (qmodel.cpp:30-51) can go
};
#ifndef SAAP_QM_SLOT
#define SAAP_QM_SLOT 2
#endif
constexpr int kQmSlot = SAAP_QM_SLOT;  // contexts of one Q-model whose logits share the W2 loads

// host: TMA descriptor for a [rows x D] bf16 row-major tensor, boxes of
// (min(D,64) elements x box_rows rows) with the matching swizzle.
CUtensorMap make_row_map(const void* base, uint64_t rows, uint32_t D, uint32_t box_rows);
// host: the 4-D grouped view above, boxes of 8 * groups rows
CUtensorMap make_group_map(const void* base, uint64_t rows, uint32_t D, uint32_t groups);

// tcgen05 key assignment (assign_tc.cu): key tiles and kernel arguments
struct TcTile {
    uint32_t group;
    uint32_t lid0;   // first local id of the tile
    uint32_t count;  // valid keys (0 = padding tile)
    uint32_t part;   // partition slot (rows part*Cpad.. in the split arrays)
};

struct TcAssignArgs {
    const TcTile* tiles;
    const uint64_t* key_row0;  // per group: row of local id 0 in the key tensor map
    const uint64_t* out_base;  // per group: assignment base (ivf_base)
    const float* cmax;         // per partition slot: max centroid norm
    uint32_t C;                // buckets
    uint32_t Cpad;             // C rounded up to CN
    uint32_t* out;
    uint32_t* refine;          // per group (at out_base): local ids of ambiguous keys
    uint32_t* refine_count;    // per group
    const uint16_t* keys;      // same tensor the map covers (for |k|)
    // split mode (f32 keys): keys = k_hi, map_klo covers k_lo = bf16(k - k_hi);
    // each pair is one key tile whose second A slot holds k_lo, accumulated
    // into the first tile's columns; |k| from the f32 keys
    const float* keys_f32;     // non-null: split mode
};

}  // namespace saap_b200
