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
struct TileRec {
    uint32_t npieces;
    uint32_t pad[3];
    PieceRec p[kMaxPieces];
};
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
struct ApproxArgs {
    const float* const* centT;     // per group, d x C f32
    const float* q_route;          // [groups][G][D]
    const uint32_t* slot_off;      // [n_slots + 1] into slot_list; null: slot s = group s
    const uint32_t* slot_list;     // groups by slot
    uint32_t G, C;
    float* approx;                 // [groups][C]
};
struct ItemRec {
    uint32_t qslot;
    uint32_t tile_first;
    uint32_t ntiles;
    uint32_t pad;
};

struct PlanArgs {
    const GroupMeta* meta;
    const uint32_t* off;
    const uint32_t* offA;
    const uint32_t* idx;
    const uint32_t* assign;
    const uint32_t* invA;
    uint32_t C;
    int mode;                    // 0 dense, 1 centroid, 2 precomputed scores, 3 window only
    const float* q_route;        // [groups][G][D]
    const double* scores;        // [groups][G][C] per-row probabilities (mode 2)
    uint32_t G, D, n_hchunks;
    uint32_t probes, recent;
    uint32_t item_tiles;
    uint32_t P2;                 // pow2 >= n_slices * keep (candidates to merge)
    uint32_t n_cand;             // n_slices * keep
    const double* cand_s;        // routing candidates from route_score_kernel
    const uint32_t* cand_i;
    const float* approx;         // centroid router, C <= 1024: fp32 scores [groups][C]
    const float* const* centT;   // per group d x C f32 centroids (exact re-scoring)
    const float* const* centR;   // per group C x d f32 centroids (row-major)
    const float* cmax;           // per group max centroid norm
    unsigned long long* trace;   // debug: clock64 per planning phase (CTA 0)
    int route_only;              // BucketRouter::select: write `selected`, plan nothing
    // general-window rows are gathered into a contiguous buffer
    const uint16_t* K;
    const uint16_t* V;
    uint16_t* gK;
    uint16_t* gV;
    uint64_t gather_cap;         // rows per group in the gather buffer
    const float* q_attn;         // [groups][G][D] queries the attention uses (roped)
    uint16_t* qA;                // out: [qslots][16][D] bf16 A operand (3-term split, swizzled)
    // outputs
    TileRec* tiles;
    ItemRec* items;
    StepCounters* ctr;           // n_items, work, n_tiles (pad[0])
    QSlot* qslots;
    saap_attn_stats* stats;
    uint32_t* selected;          // nullable [groups][probes]
    float* out;                  // [groups][G][D]
};

struct DecodeArgs {
    const ItemRec* items;
    const TileRec* tiles;
    StepCounters* ctr;
    const uint16_t* qA;  // [qslots][16][D] prepared by route_plan_kernel
    uint32_t G;
    uint32_t n_hchunks;
    float qscale;  // log2(e)/sqrt(d): scores live in the exp2 domain
    float* part_O;
    float* part_ml;  // [items][2][4]: m then l
    const QSlot* qslots;
    uint32_t* done;
    float* out;
    unsigned long long* dtrace;  // debug: per CTA {start, first tile, end (globaltimer ns), tiles}
};

struct DecodeMaps {
    CUtensorMap k64, k8, v64, v8;    // layer (or dense) cache, boxes of 64 / 8 rows
    CUtensorMap gk64, gk8, gv64, gv8;  // gather buffer
};

struct QModelArgs {
    const float* q;            // [groups][G][d] de-roped queries
    const double* const* prm;  // per group: w1, w2, vec (3 pointers)
    uint32_t G, d, h, C;
    double* probs;             // [groups][G][C]
};

// host: TMA descriptor for a [rows x D] bf16 row-major tensor, boxes of
// (min(D,64) elements x box_rows rows) with the matching swizzle.
CUtensorMap make_row_map(const void* base, uint64_t rows, uint32_t D, uint32_t box_rows);

}  // namespace saap_b200
