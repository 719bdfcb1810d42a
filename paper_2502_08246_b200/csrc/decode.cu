// Decode step of SAAP: routing + work planning (one CTA per context) and the
// split-K sparse/dense attention kernel with a fused log-sum-exp combine.
//
// Reference semantics (all /root/reference/proj/core/src):
//   sparse_attention        attention.cpp:317-376  (visited set, counters)
//   absorb_impl / Alg. 1    attention.cpp:34-78    (online softmax partials)
//   merge_into / finalize   attention.cpp:102-161  (Alg. 2 LSE combine)
//   CentroidRouter::select  attention.cpp:275-306  (fp64 pooled scores)
//   top_l_ids               attention.cpp:259-271  (score desc, id asc)
//   full_attention          attention.cpp:163-195
#include <math.h>

#include "args.cuh"

namespace saap_b200 {

// ============================================================ route + plan


struct Seg {
    uint32_t kind;
    uint32_t len;
    uint64_t start;
};

__device__ __forceinline__ bool precedes(double sa, uint32_t ia, double sb, uint32_t ib) {
    return sa > sb || (sa == sb && ia < ib);
}

// Bitonic sort of (score, id) pairs in shared memory: the comparator is the
// reference's total order (attention.cpp:263-268), so the prefix equals the
// std::partial_sort result bit for bit.
__device__ void block_bitonic(double* ss, uint32_t* si, uint32_t n) {
    for (uint32_t k = 2; k <= n; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
                uint32_t ixj = i ^ j;
                if (ixj > i) {
                    bool asc = (i & k) == 0;  // "ascending" = precedes-order
                    double a = ss[i], b = ss[ixj];
                    uint32_t ia = si[i], ib = si[ixj];
                    bool swap = asc ? precedes(b, ib, a, ia) : precedes(a, ia, b, ib);
                    if (swap) {
                        ss[i] = b;
                        ss[ixj] = a;
                        si[i] = ib;
                        si[ixj] = ia;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(512) route_plan_kernel(PlanArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t g = blockIdx.x;
    const uint32_t tid = threadIdx.x;
    const GroupMeta gm = a.meta[g];
    const uint32_t n = gm.n, sink = gm.sink, T = gm.T;
    const uint32_t Cb = a.C;
    const bool fallback = (a.mode == 0) || (n <= sink + a.recent);
    const bool route = !fallback && a.probes > 0 && (a.mode == 1 || a.mode == 2);
    const uint32_t L = route ? a.probes : 0;

    // smem carve: [sort scores P2 f64][sort ids P2 u32][bitmap C/32][segs L+4][misc]
    double* ss = reinterpret_cast<double*>(smem);
    uint32_t* si = reinterpret_cast<uint32_t*>(ss + (route ? a.P2 : 0));
    uint32_t* bitmap = si + (route ? a.P2 : 0);
    const uint32_t bm_words = route ? (Cb + 31) / 32 : 0;
    Seg* segs = reinterpret_cast<Seg*>(
            (reinterpret_cast<uintptr_t>(bitmap + bm_words) + 15) & ~uintptr_t(15));
    __shared__ double pooled[128];
    __shared__ unsigned long long s_keys;
    __shared__ uint32_t s_maxv, s_nseg, s_base, s_total, s_wcnt[16], s_filtered;

    if (tid == 0) {
        s_keys = 0;
        s_maxv = 0;
        s_filtered = 0;
    }

    // ---------------- routing: scores -> (score desc, id asc) order
    if (route) {
        if (a.mode == 1) {
            // pooled_j = sum_i q_ij (fp64, rows in order)   attention.cpp:289-295
            const float* q = a.q_route + (size_t)g * a.G * a.D;
            for (uint32_t j = tid; j < a.D; j += blockDim.x) {
                double s = 0.0;
                for (uint32_t i = 0; i < a.G; ++i) s = __dadd_rn(s, (double)q[(size_t)i * a.D + j]);
                pooled[j] = s;
            }
            __syncthreads();
            // s_c = sum_j pooled_j * c_cj, mul rounded before add (no FMA)
            //                                              attention.cpp:296-304
            const float* cT = a.centT[g];
            for (uint32_t c = tid; c < a.P2; c += blockDim.x) {
                if (c < Cb) {
                    double s = 0.0;
#pragma unroll 8
                    for (uint32_t j = 0; j < a.D; ++j)
                        s = __dadd_rn(s, __dmul_rn(pooled[j], (double)cT[(size_t)j * Cb + c]));
                    ss[c] = s;
                    si[c] = c;
                } else {
                    ss[c] = -INFINITY;
                    si[c] = 0xFFFFFFFFu;
                }
            }
        } else {
            // Q-model: score_c = sum_i p_ic over the group rows in order
            //                                              qmodel.cpp:493-499
            const double* p = a.scores + (size_t)g * a.G * Cb;
            for (uint32_t c = tid; c < a.P2; c += blockDim.x) {
                if (c < Cb) {
                    double s = 0.0;
                    for (uint32_t i = 0; i < a.G; ++i) s = __dadd_rn(s, p[(size_t)i * Cb + c]);
                    ss[c] = s;
                    si[c] = c;
                } else {
                    ss[c] = -INFINITY;
                    si[c] = 0xFFFFFFFFu;
                }
            }
        }
        __syncthreads();
        block_bitonic(ss, si, a.P2);
        for (uint32_t w = tid; w < bm_words; w += blockDim.x) bitmap[w] = 0;
        __syncthreads();
        for (uint32_t b = tid; b < L; b += blockDim.x) {
            atomicOr(&bitmap[si[b] >> 5], 1u << (si[b] & 31));
            if (a.selected) a.selected[(size_t)g * a.probes + b] = si[b];
        }
        __syncthreads();
    }
    if (a.route_only) return;

    // ---------------- segments of the visited set      attention.cpp:342-372
    const uint32_t rb = fallback ? 0 : n - a.recent;  // recent_begin
    const uint32_t* offg = a.off + (size_t)g * (Cb + 1);
    const uint32_t* offAg = a.offA + (size_t)g * (Cb + 1);
    const uint32_t* idxg = a.idx + gm.ivf_base;
    uint32_t nfixed = 0;  // window segments live after the L bucket segments
    if (tid == 0) {
        Seg* w = segs + L;
        if (fallback) {
            w[nfixed++] = Seg{KIND_ROWS, n, 0};
        } else {
            if (sink) w[nfixed++] = Seg{KIND_ROWS, sink, 0};
            const uint32_t tail0 = rb > T ? rb : T;
            if (n > tail0) w[nfixed++] = Seg{KIND_ROWS, n - tail0, tail0};
            if (rb < T)  // region-A keys inside the recent window, via pos -> row map
                w[nfixed++] = Seg{KIND_INVA, T - rb, gm.ivf_base + (rb - sink)};
        }
        s_nseg = L + nfixed;
    }
    // bucket segments: region-A prefix of each selected bucket, cut at rb
    unsigned long long my_keys = 0;
    uint32_t my_max = 0;
    for (uint32_t b = tid; b < L; b += blockDim.x) {
        const uint32_t c = si[b];
        const uint32_t raw = offg[c + 1] - offg[c];
        uint32_t lenA = offAg[c + 1] - offAg[c];
        if (rb < T) {  // ids ascend inside a bucket: the in-window ids are a suffix
            uint32_t lo = 0, hi = lenA;
            const uint32_t lim = rb - sink;
            const uint32_t* seg = idxg + offg[c];
            while (lo < hi) {
                uint32_t mid = (lo + hi) >> 1;
                if (seg[mid] < lim) lo = mid + 1;
                else hi = mid;
            }
            lenA = lo;
        }
        segs[b] = Seg{KIND_ROWS, lenA, (uint64_t)sink + offAg[c]};
        my_keys += lenA;
        my_max = max(my_max, raw);
    }
    if (my_keys) atomicAdd(&s_keys, my_keys);
    if (my_max) atomicMax(&s_maxv, my_max);
    __syncthreads();

    // region-B keys (positions [T, rb)) of selected buckets: compact a row list
    if (route && rb > T) {
        uint32_t base = 0;
        const uint32_t warp = tid >> 5, lane = tid & 31;
        for (uint32_t p0 = T; p0 < rb; p0 += blockDim.x) {
            const uint32_t pos = p0 + tid;
            bool f = false;
            if (pos < rb) {
                const uint32_t c = a.assign[gm.ivf_base + (pos - sink)];
                f = (bitmap[c >> 5] >> (c & 31)) & 1u;
            }
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, f);
            if (lane == 0) s_wcnt[warp] = __popc(bal);
            __syncthreads();
            uint32_t wex = 0, tot = 0;
            for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
                if (w < warp) wex += s_wcnt[w];
                tot += s_wcnt[w];
            }
            if (f) a.list[gm.ivf_base + base + wex + __popc(bal & ((1u << lane) - 1))] = pos;
            base += tot;
            __syncthreads();
        }
        if (tid == 0 && base) {
            segs[L + nfixed] = Seg{KIND_LIST, base, gm.ivf_base};
            s_nseg = L + nfixed + 1;
            s_filtered = base;
        }
        __syncthreads();
    }

    // ---------------- items: segments cut into item_keys chunks
    if (tid == 0) {
        uint32_t total = 0;
        for (uint32_t s = 0; s < s_nseg; ++s) total += (segs[s].len + a.item_keys - 1) / a.item_keys;
        s_total = total;
        s_base = total ? atomicAdd(&a.ctr->n_items, total * a.n_hchunks) : 0;
        unsigned long long keys;
        if (fallback) keys = n;
        else keys = (unsigned long long)sink + (n - rb) + s_keys + s_filtered;
        saap_attn_stats st;
        st.keys_scored = keys;
        st.max_visited_bucket = fallback ? 0 : s_maxv;
        st.empty_attention = keys == 0 ? 1 : 0;
        st.reserved = 0;
        a.stats[g] = st;
        for (uint32_t hc = 0; hc < a.n_hchunks; ++hc)
            a.qslots[g * a.n_hchunks + hc] = QSlot{s_base + hc * total, total};
    }
    __syncthreads();
    const uint32_t total = s_total, base = s_base;
    if (total == 0) {  // nothing visited: zero rows, empty_attention (attention.cpp:147-152)
        for (uint32_t e = tid; e < a.G * a.D; e += blockDim.x) a.out[(size_t)g * a.G * a.D + e] = 0.f;
        return;
    }
    // chunk prefix per segment (serial over <= L+4 segments, then parallel write)
    __shared__ uint32_t s_pref[1];
    (void)s_pref;
    for (uint32_t s = tid; s < s_nseg; s += blockDim.x) {
        uint32_t before = 0;
        for (uint32_t t = 0; t < s; ++t) before += (segs[t].len + a.item_keys - 1) / a.item_keys;
        const Seg sg = segs[s];
        const uint32_t nch = (sg.len + a.item_keys - 1) / a.item_keys;
        for (uint32_t k = 0; k < nch; ++k) {
            const uint32_t len = min(a.item_keys, sg.len - k * a.item_keys);
            for (uint32_t hc = 0; hc < a.n_hchunks; ++hc) {
                Item it;
                it.qslot = g * a.n_hchunks + hc;
                it.n_kind = len | (sg.kind << 30);
                it.start = sg.start + (uint64_t)k * a.item_keys;
                a.items[base + hc * total + before + k] = it;
            }
        }
    }
}

// ============================================================ attention


template <int D, int NS>
struct DecodeSmem {
    uint16_t K[NS][kTileKeys][D];
    uint16_t V[NS][kTileKeys][D];
    float red[kComputeWarps][kHeadsPerSlot][D];
    float P[kTileKeys][kHeadsPerSlot];
    float wmax[kComputeWarps][kHeadsPerSlot];
    float wl[kComputeWarps][kHeadsPerSlot];
    uint64_t full[NS];
    uint64_t empty[NS];
    int4 meta[NS];  // item, tile, nt, last
    int flag;
};

template <int D>
__device__ __forceinline__ void load_v(const uint16_t* row, int lane, float* v) {
    constexpr int DPL = D / 32;
    if constexpr (DPL == 4) {
        uint2 x = *reinterpret_cast<const uint2*>(row + lane * 4);
        v[0] = bf16lo(x.x);
        v[1] = bf16hi(x.x);
        v[2] = bf16lo(x.y);
        v[3] = bf16hi(x.y);
    } else if constexpr (DPL == 2) {
        uint32_t x = *reinterpret_cast<const uint32_t*>(row + lane * 2);
        v[0] = bf16lo(x);
        v[1] = bf16hi(x);
    } else {
        v[0] = __uint_as_float(((uint32_t)row[lane]) << 16);
    }
}

// Warp roles: warps 0..7 compute, warp 8 produces (TMA bulk copies of 64-key
// K/V tiles into an NS-deep ring; contiguous bucket segments are one copy
// per tile, row lists one copy per row).  Items are fetched dynamically.
template <int D, int NS>
__global__ void __launch_bounds__((kComputeWarps + 1) * 32, 1) decode_kernel(DecodeArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    auto& s = *reinterpret_cast<DecodeSmem<D, NS>*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&s.full[i], 1);
            mbar_init(&s.empty[i], kComputeWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    const uint32_t n_items = *reinterpret_cast<volatile uint32_t*>(&a.ctr->n_items);

    if (warp == kComputeWarps) {
        // ------------------------------------------------ producer
        uint32_t stage = 0, phase = 0;
        for (;;) {
            uint32_t it = 0;
            if (lane == 0) it = atomicAdd(&a.ctr->work, 1u);
            it = __shfl_sync(0xFFFFFFFFu, it, 0);
            if (it >= n_items) {
                if (lane == 0) {
                    mbar_wait(&s.empty[stage], phase ^ 1);
                    s.meta[stage] = make_int4(-1, 0, 0, 0);
                    mbar_arrive(&s.full[stage]);
                }
                break;
            }
            const Item itm = a.items[it];
            const uint32_t n = itm.n_kind & 0x3FFFFFFFu, kind = itm.n_kind >> 30;
            const uint32_t g = itm.qslot / a.n_hchunks;
            const uint64_t rbase = a.row_base[g];
            const uint32_t ntiles = (n + kTileKeys - 1) / kTileKeys;
            for (uint32_t t = 0; t < ntiles; ++t) {
                const uint32_t nt = min((uint32_t)kTileKeys, n - t * kTileKeys);
                if (lane == 0) {
                    mbar_wait(&s.empty[stage], phase ^ 1);
                    s.meta[stage] = make_int4((int)it, (int)t, (int)nt, t + 1 == ntiles);
                    mbar_arrive_expect_tx(&s.full[stage], nt * D * 2 * 2);
                }
                __syncwarp();
                if (kind == KIND_ROWS) {
                    if (lane == 0) {
                        const uint64_t r0 = rbase + itm.start + (uint64_t)t * kTileKeys;
                        bulk_g2s(&s.K[stage][0][0], a.K + r0 * D, nt * D * 2, &s.full[stage]);
                        bulk_g2s(&s.V[stage][0][0], a.V + r0 * D, nt * D * 2, &s.full[stage]);
                    }
                } else {
                    const uint32_t* lst = kind == KIND_INVA ? a.invA : a.list;
                    for (uint32_t j = lane; j < nt; j += 32) {
                        const uint64_t r = rbase + lst[itm.start + (uint64_t)t * kTileKeys + j];
                        bulk_g2s(&s.K[stage][j][0], a.K + r * D, D * 2, &s.full[stage]);
                        bulk_g2s(&s.V[stage][j][0], a.V + r * D, D * 2, &s.full[stage]);
                    }
                }
                if (++stage == NS) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        return;
    }

    // ---------------------------------------------------- consumers
    constexpr int LPK = D / 8;    // lanes per key row in QK (8 dims each)
    constexpr int KPI = 32 / LPK; // keys per warp instruction
    constexpr int STEPS = 8 / KPI;
    constexpr int DPL = D / 32;   // dims per lane in PV
    const int tid = threadIdx.x;  // 0..255
    const int hl = lane & 3;      // head of the score this lane ends up holding
    const int idx = lane & (LPK - 1);
    const int key_local = (idx >> 2) * KPI + lane / LPK;

    float qr[4][8];
    float m_run[4];
    float acc[4][DPL];
    float l_lane = 0.f;
    uint32_t cur_qslot = 0, cur_item = 0;

    uint32_t stage = 0, phase = 0;
    for (;;) {
        mbar_wait(&s.full[stage], phase);
        const int4 mt = s.meta[stage];
        if (mt.x < 0) break;
        const int nt = mt.z;
        if (mt.y == 0) {  // item start: load the query slot's 4 heads, reset state
            cur_item = (uint32_t)mt.x;
            cur_qslot = a.items[cur_item].qslot;
            const uint32_t g = cur_qslot / a.n_hchunks, hc = cur_qslot % a.n_hchunks;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const uint32_t head = hc * 4 + h;
                if (head < a.G) {
                    const float4* qp = reinterpret_cast<const float4*>(
                            a.q + ((size_t)g * a.G + head) * D + (lane % LPK) * 8);
                    float4 x0 = qp[0], x1 = qp[1];
                    qr[h][0] = x0.x * a.qscale;
                    qr[h][1] = x0.y * a.qscale;
                    qr[h][2] = x0.z * a.qscale;
                    qr[h][3] = x0.w * a.qscale;
                    qr[h][4] = x1.x * a.qscale;
                    qr[h][5] = x1.y * a.qscale;
                    qr[h][6] = x1.z * a.qscale;
                    qr[h][7] = x1.w * a.qscale;
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) qr[h][j] = 0.f;
                }
                m_run[h] = -INFINITY;
#pragma unroll
                for (int j = 0; j < DPL; ++j) acc[h][j] = 0.f;
            }
            l_lane = 0.f;
        }

        // ---- S = q . k for this warp's 8 keys (lane owns 8 dims of a key)
        float part[LPK];
        const uint16_t* Ks = &s.K[stage][0][0];
#pragma unroll
        for (int st = 0; st < STEPS; ++st) {
            const int key = warp * 8 + st * KPI + lane / LPK;
            const uint4 kv = *reinterpret_cast<const uint4*>(Ks + key * D + (lane % LPK) * 8);
            const float k0 = bf16lo(kv.x), k1 = bf16hi(kv.x), k2 = bf16lo(kv.y), k3 = bf16hi(kv.y);
            const float k4 = bf16lo(kv.z), k5 = bf16hi(kv.z), k6 = bf16lo(kv.w), k7 = bf16hi(kv.w);
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                float x = qr[h][0] * k0;
                x = fmaf(qr[h][1], k1, x);
                x = fmaf(qr[h][2], k2, x);
                x = fmaf(qr[h][3], k3, x);
                x = fmaf(qr[h][4], k4, x);
                x = fmaf(qr[h][5], k5, x);
                x = fmaf(qr[h][6], k6, x);
                x = fmaf(qr[h][7], k7, x);
                part[st * 4 + h] = x;
            }
        }
        // transpose-reduce across the LPK lanes of each key: lane keeps value #idx
#pragma unroll
        for (int m = LPK / 2; m >= 1; m >>= 1) {
            const bool up = (lane & m) != 0;
#pragma unroll
            for (int i = 0; i < m; ++i) {
                const float send = up ? part[i] : part[i + m];
                const float keep = up ? part[i + m] : part[i];
                part[i] = keep + __shfl_xor_sync(0xFFFFFFFFu, send, m);
            }
        }
        const int key = warp * 8 + key_local;
        const bool valid = key < nt;
        const float sc = valid ? part[0] : -INFINITY;

        // ---- online softmax over the tile (Alg. 1)
        float v = sc;
        v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, 4));
        v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, 8));
        v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, 16));
        if (lane < 4) s.wmax[warp][lane] = v;
        named_bar_sync(1, kComputeWarps * 32);
        float alpha[4], mnew[4];
        {
            float4 t = *reinterpret_cast<const float4*>(s.wmax[0]);
#pragma unroll
            for (int w = 1; w < kComputeWarps; ++w) {
                const float4 u = *reinterpret_cast<const float4*>(s.wmax[w]);
                t.x = fmaxf(t.x, u.x);
                t.y = fmaxf(t.y, u.y);
                t.z = fmaxf(t.z, u.z);
                t.w = fmaxf(t.w, u.w);
            }
            mnew[0] = fmaxf(m_run[0], t.x);
            mnew[1] = fmaxf(m_run[1], t.y);
            mnew[2] = fmaxf(m_run[2], t.z);
            mnew[3] = fmaxf(m_run[3], t.w);
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                alpha[h] = fast_exp2(m_run[h] - mnew[h]);
                m_run[h] = mnew[h];
            }
        }
        const float m_h = hl == 0 ? mnew[0] : hl == 1 ? mnew[1] : hl == 2 ? mnew[2] : mnew[3];
        const float a_h = hl == 0 ? alpha[0] : hl == 1 ? alpha[1] : hl == 2 ? alpha[2] : alpha[3];
        const float p = valid ? fast_exp2(sc - m_h) : 0.f;
        l_lane = l_lane * a_h + p;
        s.P[key][hl] = p;
        named_bar_sync(1, kComputeWarps * 32);

        // ---- O += P V (lane owns DPL dims x 4 heads; warp owns keys w, w+8, ..)
#pragma unroll
        for (int h = 0; h < 4; ++h)
#pragma unroll
            for (int j = 0; j < DPL; ++j) acc[h][j] *= alpha[h];
        const uint16_t* Vs = &s.V[stage][0][0];
#pragma unroll 4
        for (int i = 0; i < 8; ++i) {
            const int k = warp + 8 * i;
            if (k < nt) {
                const float4 pk = *reinterpret_cast<const float4*>(s.P[k]);
                float vv[DPL];
                load_v<D>(Vs + k * D, lane, vv);
#pragma unroll
                for (int j = 0; j < DPL; ++j) {
                    acc[0][j] = fmaf(pk.x, vv[j], acc[0][j]);
                    acc[1][j] = fmaf(pk.y, vv[j], acc[1][j]);
                    acc[2][j] = fmaf(pk.z, vv[j], acc[2][j]);
                    acc[3][j] = fmaf(pk.w, vv[j], acc[3][j]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&s.empty[stage]);

        if (mt.w) {
            // ---- item done: reduce the 8 warps' partials (m is shared)
            float lw = l_lane;
            lw += __shfl_xor_sync(0xFFFFFFFFu, lw, 4);
            lw += __shfl_xor_sync(0xFFFFFFFFu, lw, 8);
            lw += __shfl_xor_sync(0xFFFFFFFFu, lw, 16);
            if (lane < 4) s.wl[warp][lane] = lw;
#pragma unroll
            for (int h = 0; h < 4; ++h)
#pragma unroll
                for (int j = 0; j < DPL; ++j) s.red[warp][h][lane * DPL + j] = acc[h][j];
            named_bar_sync(1, kComputeWarps * 32);

            const QSlot qs = a.qslots[cur_qslot];
            const uint32_t g = cur_qslot / a.n_hchunks, hc = cur_qslot % a.n_hchunks;
            constexpr int NOUT = 4 * D;
            constexpr int PER = (NOUT + kComputeWarps * 32 - 1) / (kComputeWarps * 32);
            if (qs.count == 1) {
#pragma unroll
                for (int e0 = 0; e0 < PER; ++e0) {
                    const int e = tid + e0 * kComputeWarps * 32;
                    if (e >= NOUT) break;
                    const int h = e / D, d = e % D;
                    float o = 0.f, lsum = 0.f;
#pragma unroll
                    for (int w = 0; w < kComputeWarps; ++w) {
                        o += s.red[w][h][d];
                        lsum += s.wl[w][h];
                    }
                    const uint32_t head = hc * 4 + h;
                    if (head < a.G) a.out[((size_t)g * a.G + head) * D + d] = o / lsum;
                }
            } else {
                float* pO = a.part_O + (size_t)cur_item * 4 * D;
#pragma unroll
                for (int e0 = 0; e0 < PER; ++e0) {
                    const int e = tid + e0 * kComputeWarps * 32;
                    if (e >= NOUT) break;
                    const int h = e / D, d = e % D;
                    float o = 0.f;
#pragma unroll
                    for (int w = 0; w < kComputeWarps; ++w) o += s.red[w][h][d];
                    pO[e] = o;
                }
                if (tid < 4) {
                    float lsum = 0.f;
#pragma unroll
                    for (int w = 0; w < kComputeWarps; ++w) lsum += s.wl[w][tid];
                    a.part_ml[(size_t)cur_item * 8 + tid] = m_run[tid];
                    a.part_ml[(size_t)cur_item * 8 + 4 + tid] = lsum;
                }
                __threadfence();
                named_bar_sync(1, kComputeWarps * 32);
                if (tid == 0) {
                    const uint32_t prev = atomicAdd(&a.done[cur_qslot], 1u);
                    s.flag = (prev + 1 == qs.count);
                }
                named_bar_sync(1, kComputeWarps * 32);
                if (s.flag) {
                    // last partial of this query slot: LSE combine (Alg. 2)
                    __threadfence();
#pragma unroll
                    for (int e0 = 0; e0 < PER; ++e0) {
                        const int e = tid + e0 * kComputeWarps * 32;
                        if (e >= NOUT) break;
                        const int h = e / D;
                        float M = -INFINITY;
                        for (uint32_t i = 0; i < qs.count; ++i)
                            M = fmaxf(M, __ldcg(a.part_ml + (size_t)(qs.base + i) * 8 + h));
                        float o = 0.f, lsum = 0.f;
                        for (uint32_t i = 0; i < qs.count; ++i) {
                            const size_t it = qs.base + i;
                            const float wgt = fast_exp2(__ldcg(a.part_ml + it * 8 + h) - M);
                            o = fmaf(__ldcg(a.part_O + it * 4 * D + e), wgt, o);
                            lsum = fmaf(__ldcg(a.part_ml + it * 8 + 4 + h), wgt, lsum);
                        }
                        const uint32_t head = hc * 4 + h;
                        if (head < a.G) a.out[((size_t)g * a.G + head) * D + (e % D)] = o / lsum;
                    }
                    if (tid == 0) a.done[cur_qslot] = 0;
                }
            }
            named_bar_sync(1, kComputeWarps * 32);
        }
        if (++stage == NS) {
            stage = 0;
            phase ^= 1;
        }
    }
}

// ============================================================ launchers
template <int D, int NS>
static void launch_decode_t(const DecodeArgs& a, int grid, cudaStream_t st) {
    const size_t smem = sizeof(DecodeSmem<D, NS>);
    static bool configured = false;
    if (!configured) {
        SAAP_CUDA(cudaFuncSetAttribute(decode_kernel<D, NS>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = true;
    }
    decode_kernel<D, NS><<<grid, (kComputeWarps + 1) * 32, smem, st>>>(a);
    SAAP_CUDA(cudaGetLastError());
}

void launch_decode(int D, const DecodeArgs& a, int grid, cudaStream_t st) {
    switch (D) {
        case 128: launch_decode_t<128, 4>(a, grid, st); break;
        case 64: launch_decode_t<64, 6>(a, grid, st); break;
        case 32: launch_decode_t<32, 8>(a, grid, st); break;
        default: fail(SAAP_ERR_UNSUPPORTED, "decode: unsupported head dim " + std::to_string(D));
    }
}

void launch_route_plan(const PlanArgs& a, uint32_t n_groups, cudaStream_t st) {
    const bool route = a.mode == 1 || a.mode == 2;
    size_t smem = 0;
    if (route) smem = (size_t)a.P2 * 12 + ((a.C + 31) / 32) * 4 + 16;
    smem += (size_t)(a.probes + 8) * sizeof(Seg);
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        SAAP_CUDA(cudaFuncSetAttribute(route_plan_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    route_plan_kernel<<<n_groups, 512, smem, st>>>(a);
    SAAP_CUDA(cudaGetLastError());
}

}  // namespace saap_b200
