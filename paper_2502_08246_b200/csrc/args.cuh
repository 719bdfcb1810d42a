// Argument blocks of the decode-side kernels (shared by the .cu files).
#pragma once
#include "common.cuh"

namespace saap_b200 {

struct PlanArgs {
    const GroupMeta* meta;
    const uint32_t* off;
    const uint32_t* offA;
    const uint32_t* idx;
    const uint32_t* assign;
    uint32_t* list;
    uint32_t C;
    int mode;                   // 0 dense, 1 centroid, 2 precomputed scores, 3 window only
    const float* const* centT;  // per group, d x C (mode 1)
    const float* q_route;       // [groups][G][D]
    const double* scores;       // [groups][G][C] per-row probabilities (mode 2)
    uint32_t G, D, n_hchunks;
    uint32_t probes, recent;
    uint32_t item_keys;
    uint32_t P2;  // pow2 >= C (mode 1/2)
    int route_only;  // BucketRouter::select: write `selected`, plan nothing
    Item* items;
    StepCounters* ctr;
    QSlot* qslots;
    saap_attn_stats* stats;
    uint32_t* selected;  // nullable [groups][probes]
    float* out;          // [groups][G][D]
};

struct DecodeArgs {
    const Item* items;
    StepCounters* ctr;
    const uint16_t* K;
    const uint16_t* V;
    const uint64_t* row_base;
    const uint32_t* invA;
    const uint32_t* list;
    const float* q;
    uint32_t G;
    uint32_t n_hchunks;
    float qscale;  // log2(e)/sqrt(d): scores live in the exp2 domain
    float* part_O;
    float* part_ml;  // [items][2][4]: m then l
    const QSlot* qslots;
    uint32_t* done;
    float* out;
};

struct QModelArgs {
    const float* q;            // [groups][G][d] de-roped queries
    const double* const* prm;  // per group: w1, w2, vec (3 pointers)
    uint32_t G, d, h, C;
    double* probs;             // [groups][G][C]
};

}  // namespace saap_b200
