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

// ============================================================ shared layout helpers
// Row-major bf16 tiles are kept in smem as [half][rows][HALF bytes] with the
// TMA swizzle (128-byte rows: chunk ^ (row & 7); 64-byte rows (d=32):
// chunk ^ ((row >> 1) & 3)), so ldmatrix row fetches are conflict-free.
__host__ __device__ __forceinline__ uint32_t swz_bytes(uint32_t D, uint32_t row, uint32_t chunk) {
    const uint32_t half = 2 * D >= 128 ? 128 : 2 * D;
    if (half == 128) return row * 128 + ((chunk ^ (row & 7)) << 4);
    return row * 64 + ((chunk ^ ((row >> 1) & 3)) << 4);
}
// byte offset of element (row, d) in a rows-tall swizzled bf16 tile
__host__ __device__ __forceinline__ uint32_t swz_elem(uint32_t D, uint32_t rows, uint32_t row, uint32_t d) {
    const uint32_t half = 2 * D >= 128 ? 128 : 2 * D;
    const uint32_t per_half = half / 2;  // elements per swizzle row
    const uint32_t h = d / per_half, dd = d % per_half;
    return h * rows * half + swz_bytes(D, row, dd / 8) + (dd % 8) * 2;
}
__device__ __forceinline__ uint32_t bf16x2_rn(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// ============================================================ route + plan
struct Seg {
    uint32_t kind;  // KIND_ROWS (layer rows) or KIND_LIST (gather buffer rows)
    uint32_t len;
    uint64_t start;  // ROWS: group-relative row; LIST: gather-buffer row
};

// Tile records of one group's dynamic tiles (attention.cpp:342-372 visited
// set, laid out as tiles): segment s occupies the 8-aligned virtual rows
// [vpre[s], vpre[s] + ceil8(len_s)), tile t the virtual rows [128t, 128t+128).
// One thread per tile (threads first, first + stride, ...): a binary search
// finds the segment holding the tile's first row, the overlapped segments
// become its pieces in order.  No counters, no second pass: every record
// (header with ready = 0, pieces) is written once; head chunks > 0 get copies.
__device__ __forceinline__ void emit_tiles(TileRec* base, uint32_t ntiles, uint32_t nh, uint32_t qslot0,
                                           const Seg* segs, const uint32_t* vpre, uint32_t ns,
                                           uint64_t row_base, uint32_t first, uint32_t stride) {
#pragma unroll 1
    for (uint32_t t = first; t < ntiles; t += stride) {
        const uint32_t v_lo = t * kTileRows, v_hi = v_lo + kTileRows;
        uint32_t lo = 0, hi = ns;  // last segment with vpre <= v_lo (vpre[0] == 0)
#pragma unroll 1
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (vpre[mid] <= v_lo) lo = mid;
            else hi = mid;
        }
        uint32_t np = 0, r8 = 0;
        uint32_t vm[4] = {0u, 0u, 0u, 0u};
#pragma unroll 1
        for (uint32_t b = lo; b < ns; ++b) {
            const uint32_t v0 = vpre[b];
            if (v0 >= v_hi) break;
            const Seg sg = segs[b];
            const uint32_t a0 = max(v0, v_lo), kend = min(v0 + sg.len, v_hi);
            if (kend <= a0) continue;
            const uint64_t row = (sg.kind == KIND_LIST ? 0 : row_base) + sg.start + (a0 - v0);
            const uint32_t len = kend - a0, s0 = a0 - v_lo;
            const uint4 pr = make_uint4(len | (sg.kind == KIND_LIST ? kPieceGather : 0u), s0,
                                        (uint32_t)row, (uint32_t)(row >> 32));
#pragma unroll 1
            for (uint32_t hc = 0; hc < nh; ++hc)
                *reinterpret_cast<uint4*>(&base[(size_t)hc * ntiles + t].p[np]) = pr;
            ++np;
            r8 += (len + 7) & ~7u;
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // rows [s0, s0 + len) of the tile's 128
                const uint32_t qlo = max(s0, (uint32_t)q * 32), qhi = min(s0 + len, (uint32_t)q * 32 + 32);
                if (qhi > qlo)
                    vm[q] |= (qhi - qlo == 32 ? 0xFFFFFFFFu : ((1u << (qhi - qlo)) - 1u)) << (qlo - q * 32);
            }
        }
#pragma unroll 1
        for (uint32_t hc = 0; hc < nh; ++hc) {
            TileRec& tr = base[(size_t)hc * ntiles + t];
            *reinterpret_cast<uint4*>(&tr.rows8) = make_uint4(r8, 0u, 0u, 0u);
            *reinterpret_cast<uint4*>(&tr.valid[0]) = make_uint4(vm[0], vm[1], vm[2], vm[3]);
            *reinterpret_cast<uint4*>(&tr) = make_uint4(np, qslot0 + hc, 0u, t + 1 == ntiles ? 1u : 0u);
        }
    }
}

// Warp-parallel emit_tiles (same records): warp w takes tiles w, w + nw, ...;
// the lanes take 32 consecutive segments at a time from the tile's first one,
// each builds its piece, and a ballot orders the non-empty pieces.
__device__ __forceinline__ void emit_tiles_warp(TileRec* base, uint32_t ntiles, uint32_t nh, uint32_t qslot0,
                                                const Seg* segs, const uint32_t* vpre, uint32_t ns,
                                                uint64_t row_base, uint32_t warp, uint32_t nw, uint32_t lane) {
#pragma unroll 1
    for (uint32_t t = warp; t < ntiles; t += nw) {
        const uint32_t v_lo = t * kTileRows, v_hi = v_lo + kTileRows;
        uint32_t lo = 0, hi = ns;  // last segment with vpre <= v_lo (vpre[0] == 0)
#pragma unroll 1
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (vpre[mid] <= v_lo) lo = mid;
            else hi = mid;
        }
        uint32_t np = 0, r8 = 0;
        uint32_t vm[4] = {0u, 0u, 0u, 0u};
#pragma unroll 1
        for (uint32_t b0 = lo; b0 < ns; b0 += 32) {
            const uint32_t b = b0 + lane;
            bool has = false, more = false;
            uint32_t len = 0, s0 = 0;
            uint4 pr = make_uint4(0u, 0u, 0u, 0u);
            if (b < ns) {
                const uint32_t v0 = vpre[b];
                more = v0 < v_hi;
                if (more) {
                    const Seg sg = segs[b];
                    const uint32_t a0 = max(v0, v_lo), kend = min(v0 + sg.len, v_hi);
                    if (kend > a0) {
                        has = true;
                        const uint64_t row = (sg.kind == KIND_LIST ? 0 : row_base) + sg.start + (a0 - v0);
                        len = kend - a0;
                        s0 = a0 - v_lo;
                        pr = make_uint4(len | (sg.kind == KIND_LIST ? kPieceGather : 0u), s0, (uint32_t)row,
                                        (uint32_t)(row >> 32));
                    }
                }
            }
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, has);
            if (has) {
                const uint32_t idx = np + __popc(bal & ((1u << lane) - 1));
                for (uint32_t hc = 0; hc < nh; ++hc)
                    *reinterpret_cast<uint4*>(&base[(size_t)hc * ntiles + t].p[idx]) = pr;
            }
            np += __popc(bal);
            r8 += __reduce_add_sync(0xFFFFFFFFu, has ? (len + 7) & ~7u : 0u);
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // rows [s0, s0 + len) of the tile's 128
                uint32_t m = 0;
                if (has) {
                    const uint32_t qlo = max(s0, (uint32_t)q * 32), qhi = min(s0 + len, (uint32_t)q * 32 + 32);
                    if (qhi > qlo) m = (qhi - qlo == 32 ? 0xFFFFFFFFu : ((1u << (qhi - qlo)) - 1u)) << (qlo - q * 32);
                }
                vm[q] |= __reduce_or_sync(0xFFFFFFFFu, m);
            }
            // segments past the tile end the scan (vpre ascends)
            if (__shfl_sync(0xFFFFFFFFu, (uint32_t)more, 31) == 0u) break;
        }
        for (uint32_t hc = lane; hc < nh; hc += 32) {
            TileRec& tr = base[(size_t)hc * ntiles + t];
            *reinterpret_cast<uint4*>(&tr.rows8) = make_uint4(r8, 0u, 0u, 0u);
            *reinterpret_cast<uint4*>(&tr.valid[0]) = make_uint4(vm[0], vm[1], vm[2], vm[3]);
            *reinterpret_cast<uint4*>(&tr) = make_uint4(np, qslot0 + hc, 0u, t + 1 == ntiles ? 1u : 0u);
        }
        __syncwarp();
    }
}

__device__ __forceinline__ bool precedes(double sa, uint32_t ia, double sb, uint32_t ib) {
    return sa > sb || (sa == sb && ia < ib);
}

// Bitonic sort of (score, id) pairs under the reference's total order
// (score desc, id asc; attention.cpp:263-268), so the prefix is exactly
// std::partial_sort's.  n <= blockDim.x: one element per thread in registers,
// distances < 32 through shuffles, larger ones through shared memory.
__device__ void bitonic_regs(double& s, uint32_t& id, uint32_t n, double* xs, uint32_t* xi) {
    const uint32_t t = threadIdx.x;
    for (uint32_t k = 2; k <= n; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            double ps = 0.0;
            uint32_t pi = 0;
            if (j >= 32) {
                if (t < n) {
                    xs[t] = s;
                    xi[t] = id;
                }
                __syncthreads();
                if (t < n) {
                    ps = xs[t ^ j];
                    pi = xi[t ^ j];
                }
                __syncthreads();
            } else {
                ps = __shfl_xor_sync(0xFFFFFFFFu, s, j);
                pi = __shfl_xor_sync(0xFFFFFFFFu, id, j);
            }
            if (t < n) {
                const bool dir = (t & k) == 0;    // this block sorts in "precedes" order
                const bool lower = (t & j) == 0;  // lower index of the pair
                const bool p_first = precedes(ps, pi, s, id);
                if ((lower == dir) ? p_first : !p_first) {
                    s = ps;
                    id = pi;
                }
            }
        }
    }
}

// fp32 variant (approximate scores; same total order)
__device__ void bitonic_regs_f(float& s, uint32_t& id, uint32_t n, float* xs, uint32_t* xi) {
    const uint32_t t = threadIdx.x;
    for (uint32_t k = 2; k <= n; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            float ps = 0.f;
            uint32_t pi = 0;
            if (j >= 32) {
                if (t < n) {
                    xs[t] = s;
                    xi[t] = id;
                }
                __syncthreads();
                if (t < n) {
                    ps = xs[t ^ j];
                    pi = xi[t ^ j];
                }
                __syncthreads();
            } else {
                ps = __shfl_xor_sync(0xFFFFFFFFu, s, j);
                pi = __shfl_xor_sync(0xFFFFFFFFu, id, j);
            }
            if (t < n) {
                const bool dir = (t & k) == 0;
                const bool lower = (t & j) == 0;
                const bool p_first = ps > s || (ps == s && pi < id);
                if ((lower == dir) ? p_first : !p_first) {
                    s = ps;
                    id = pi;
                }
            }
        }
    }
}

__device__ void bitonic_smem(double* ss, uint32_t* si, uint32_t n) {
    for (uint32_t k = 2; k <= n; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
                const uint32_t ixj = i ^ j;
                if (ixj > i) {
                    const bool asc = (i & k) == 0;
                    const double a = ss[i], b = ss[ixj];
                    const uint32_t ia = si[i], ib = si[ixj];
                    if (asc ? precedes(b, ib, a, ia) : precedes(a, ia, b, ib)) {
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

// pooled_j = sum_i q_ij in fp64, rows in order (attention.cpp:289-295); the
// row loads are issued 8 at a time so the chain waits on one round trip.
template <typename T>
__device__ __forceinline__ double pooled_sum(const T* q, uint32_t G, size_t stride) {
    double s = 0.0;
    for (uint32_t i0 = 0; i0 < G; i0 += 8) {
        T v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = i0 + u < G ? q[(size_t)(i0 + u) * stride] : (T)0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (i0 + u < G) s = __dadd_rn(s, (double)v[u]);
    }
    return s;
}

// Stage 1: score a slice of centroids (one thread per centroid) and keep the
// slice's top-`keep` in reference order.  Each thread reads its centroid's
// column of the transposed f32 centroids straight from global memory (a warp
// reads consecutive centroids: coalesced), eight loads ahead of the ordered
// fp64 chain, so a slice can hold kSliceMax centroids with no shared-memory
// slab.
__global__ void __launch_bounds__(kSliceMax) route_score_kernel(RouteArgs a) {
    __shared__ double pooled[128];
    __shared__ double xs[kSliceMax];
    __shared__ uint32_t xi[kSliceMax];
    pdl_trigger();
    const uint32_t g = blockIdx.x, sl = blockIdx.y, tid = threadIdx.x;
    const uint32_t c0 = sl * a.slice, nsl = min(a.slice, a.C - c0);
    if (a.mode == 1) {
        // pooled_j = sum_i q_ij (fp64, rows in order)   attention.cpp:289-295
        const float* q = a.q_route + (size_t)g * a.G * a.D;
        for (uint32_t j = tid; j < a.D; j += blockDim.x) pooled[j] = pooled_sum(q + j, a.G, a.D);
        __syncthreads();
    }
    double sc = -INFINITY;
    uint32_t id = 0xFFFFFFFFu;
    if (tid < nsl) {
        const uint32_t c = c0 + tid;
        double s = 0.0;
        if (a.mode == 1) {
            // s_c = sum_j pooled_j * c_cj, mul rounded before add  attention.cpp:296-304
            const float* col = a.centT[g] + c;
            for (uint32_t j = 0; j < a.D; j += 8) {  // D is a multiple of 8
                float v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = __ldg(col + (size_t)(j + u) * a.C);
#pragma unroll
                for (int u = 0; u < 8; ++u) s = __dadd_rn(s, __dmul_rn(pooled[j + u], (double)v[u]));
            }
        } else {
            // Q-model: score_c = sum_i p_ic over the group rows   qmodel.cpp:493-499
            s = pooled_sum(a.scores + (size_t)g * a.G * a.C + c, a.G, a.C);
        }
        sc = s;
        id = c;
    }
    bitonic_regs(sc, id, blockDim.x, xs, xi);
    if (tid < a.keep) {
        const size_t o = ((size_t)g * a.n_slices + sl) * a.keep + tid;
        a.cand_s[o] = sc;
        a.cand_i[o] = id;
    }
}

// Approximate routing scores.  CTA (slot, 32 centroids): warp w owns dims
// [w*D/8, (w+1)*D/8) and lane the centroid, so every centroid value is loaded
// once (coalesced rows of the transposed centroids) and reused by all the
// slot's contexts; the 8 warps' partial dot products are summed in shared
// memory.  pooled = fp64 row sum of the group's queries rounded to f32
// (route_plan_kernel bounds the resulting error).
constexpr uint32_t kStageOff = 2049;  // planner stages off/offA in shared memory up to C = 2048
constexpr int kPlanTileCnt = 1024;    // planner keeps per-tile piece counts in shared memory


template <int D>
__global__ void __launch_bounds__(256) route_approx_kernel(ApproxArgs a) {
    constexpr int DW = D / 8;
    __shared__ float pf[kSlotGroups][D];
    __shared__ float red[8][kSlotGroups][33];
    pdl_trigger();
    const uint32_t s = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) tl_mark(a.tl, 0, true);
    ApproxSlot sl;
    if (a.slots) {
        sl = a.slots[s];
    } else {
        sl.centT = a.centT[s];
        sl.count = 1;
        sl.group[0] = s;
    }
    const uint32_t ng = sl.count;
    const float* cT = sl.centT;
    const uint32_t c = blockIdx.y * 32 + lane;
    // centroid slice and member queries are loaded together (one round trip)
    float cv[DW];
#pragma unroll
    for (int jj = 0; jj < DW; ++jj) cv[jj] = c < a.C ? cT[(size_t)(warp * DW + jj) * a.C + c] : 0.f;
    for (uint32_t e = tid; e < ng * D; e += blockDim.x) {
        const uint32_t k = e / D, j = e % D;
        pf[k][j] = (float)pooled_sum(a.q_route + (size_t)sl.group[k] * a.G * D + j, a.G, D);
    }
    __syncthreads();
    for (uint32_t k = 0; k < ng; ++k) {
        float x = 0.f;
#pragma unroll
        for (int jj = 0; jj < DW; ++jj) x = fmaf(pf[k][warp * DW + jj], cv[jj], x);
        red[warp][k][lane] = x;
    }
    __syncthreads();
    for (uint32_t e = tid; e < ng * 32; e += blockDim.x) {
        const uint32_t k = e / 32, l = e % 32, cc = blockIdx.y * 32 + l;
        float x = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) x += red[w][k][l];
        if (cc < a.C) a.approx[(size_t)sl.group[k] * a.C + cc] = x;
    }
    if (tid == 0) tl_mark(a.tl, 0, false);
}

// Stage 2 (one CTA per context): merge the slices' candidates into the top-l
// list, build the visited set and cut it into tiles and work items.
__global__ void __launch_bounds__(kPlanThreads) route_plan_kernel(PlanArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    pdl_trigger();
    if (threadIdx.x == 0) tl_mark(a.tl, 1, true);
    pdl_wait();
    const uint32_t g = blockIdx.x;
    const uint32_t tid = threadIdx.x, nth = blockDim.x;
    const GroupMeta gm = a.meta[g];
    const uint32_t n = gm.n, sink = gm.sink, T = gm.T;
    const uint32_t Cb = a.C;
    const bool fallback = (a.mode == 0) || (n <= sink + a.recent);
    const bool route = !fallback && a.probes > 0 && (a.mode == 1 || a.mode == 2 || a.mode == 4);
    const uint32_t L = route ? a.probes : 0;

    // smem carve: [cand scores P2 f64][cand ids P2 u32][bitmap C/32][segs L+4][seg prefix]
    double* ss = reinterpret_cast<double*>(smem);
    uint32_t* si = reinterpret_cast<uint32_t*>(ss + (route ? a.P2 : 0));
    uint32_t* bitmap = si + (route ? a.P2 : 0);
    const uint32_t bm_words = route ? (Cb + 31) / 32 : 0;
    Seg* segs = reinterpret_cast<Seg*>(
            (reinterpret_cast<uintptr_t>(bitmap + bm_words) + 15) & ~uintptr_t(15));
    uint32_t* vpre = reinterpret_cast<uint32_t*>(segs + L + 4);  // virtual-row prefix per seg
    __shared__ unsigned long long s_keys;
    __shared__ uint32_t s_maxv, s_wcnt[32], s_filtered, s_gbase, s_nseg, s_vrows;
    __shared__ uint32_t s_tile0, s_ntiles, s_item0, s_nitems;

    if (tid == 0) {
        s_keys = 0;
        s_maxv = 0;
        s_filtered = 0;
        s_gbase = 0;
    }

    unsigned long long t0 = 0;
    auto trace = [&](int k) {
        if (a.trace && route && g == 0 && tid == 0) a.trace[k] = clock64() - t0;
    };
    if (a.trace && g == 0 && tid == 0) t0 = clock64();
    // the group's bucket offsets, staged while routing runs (C <= kStageOff)
    const bool stage_off = route && !a.route_only && Cb + 1 <= kStageOff;
    uint32_t* s_off = vpre + L + 4;
    uint32_t* s_offA = s_off + (stage_off ? Cb + 1 : 0);
    if (stage_off) {
        const uint32_t* og = a.off + (size_t)g * (Cb + 1);
        const uint32_t* oAg = a.offA + (size_t)g * (Cb + 1);
        for (uint32_t c = tid; c <= Cb; c += nth) {
            s_off[c] = og[c];
            s_offA[c] = oAg[c];
        }
    }
    // ---------------- routing: candidates -> top-L in reference order
    if (route && a.approx) {
        // centroid router, C <= blockDim: exact top-L from fp32 scores.  With
        // B = 2^-16 |pooled|_2 max|c|_2 >= |approx - exact| (pooled rounded to
        // f32: 2^-24 rel; fp32 accumulation of D products: D * 2^-24 rel), every
        // centroid whose approx score is below t_L - 2B (t_L = L-th largest
        // approx) ranks below L others exactly; the rest are re-scored with
        // the reference's fp64 chain (attention.cpp:296-304) and sorted exactly.
        __shared__ double pooled[128];
        __shared__ uint32_t hist[256];
        __shared__ uint32_t s_pref, s_need, s_ncand;
        __shared__ double s_n2[32];
        constexpr uint32_t kMaxCand = 64;
        __shared__ float crow[kMaxCand][129];  // candidate centroid rows (padded)
        __shared__ uint32_t cand_id[kMaxCand];
        const float* q = a.q_route + (size_t)g * a.G * a.D;
        double part = 0.0;
        for (uint32_t j = tid; j < a.D; j += nth) {
            const double sj = pooled_sum(q + j, a.G, a.D);
            pooled[j] = sj;
            part += sj * sj;
        }
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xFFFFFFFFu, part, o);
        if ((tid & 31) == 0) s_n2[tid >> 5] = part;
        const float av = tid < Cb ? a.approx[(size_t)g * Cb + tid] : -INFINITY;
        if (a.trace && g == 0) {
            __syncthreads();
            trace(8);
        }
        const uint32_t u = __float_as_uint(av);
        const uint32_t key = (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // order-preserving
        // radix select (MSB first, 8-bit digits): the L-th largest key
        if (tid == 0) {
            s_pref = 0;
            s_need = L;
        }
        for (int shift = 24; shift >= 0; shift -= 8) {
            if (tid < 256) hist[tid] = 0;
            __syncthreads();
            const uint32_t pref = s_pref;
            const uint32_t hmask = shift == 24 ? 0u : (0xFFFFFFFFu << (shift + 8));
            if (tid < Cb && (key & hmask) == (pref & hmask)) atomicAdd(&hist[(key >> shift) & 255u], 1u);
            __syncthreads();
            if (tid < 32) {
                // bins high -> low: lane owns bins 255-8*lane .. 248-8*lane
                uint32_t cnt[8], tot = 0;
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    cnt[b] = hist[255 - 8 * tid - b];
                    tot += cnt[b];
                }
                uint32_t incl = tot;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                    if (tid >= (uint32_t)o) incl += v;
                }
                const uint32_t need = s_need, before = incl - tot;
                if (before < need && incl >= need) {
                    uint32_t run = before;
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        if (run + cnt[b] >= need) {
                            s_pref = pref | ((uint32_t)(255 - 8 * tid - b) << shift);
                            s_need = need - run;
                            break;
                        }
                        run += cnt[b];
                    }
                }
            }
            __syncthreads();
        }
        trace(9);
        const uint32_t tk = s_pref;
        const float t_l = __uint_as_float((tk & 0x80000000u) ? (tk & 0x7FFFFFFFu) : ~tk);
        double n2 = 0.0;
        for (uint32_t w = 0; w < nth / 32; ++w) n2 += s_n2[w];
        const float B2 = (float)(2.0 * 0x1p-16 * sqrt(n2) * (double)a.cmax[g]) * 1.0001f;
        // candidates: approx >= t_L - 2B (a superset of the exact top-L)
        if (tid == 0) s_ncand = 0;
        __syncthreads();
        const bool cand = tid < Cb && av >= t_l - B2;
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, cand);
        uint32_t wbase = 0;
        if ((tid & 31) == 0 && bal) wbase = atomicAdd(&s_ncand, __popc(bal));
        wbase = __shfl_sync(0xFFFFFFFFu, wbase, 0);
        const uint32_t slot = wbase + __popc(bal & ((1u << (tid & 31)) - 1));
        if (cand && slot < kMaxCand) cand_id[slot] = tid;
        __syncthreads();
        const uint32_t nS = s_ncand;
        trace(1);
        // The candidates are a superset of the exact top-L; when there are
        // exactly L of them they ARE the exact set.  Attention does not depend
        // on the bucket order, so without a `selected` output no fp64 chain
        // is needed (the usual case: approx gaps >> 2B at the boundary).
        const bool set_only = a.selected == nullptr && nS == L && L <= kMaxCand;
        double ex = -INFINITY;
        uint32_t eid = 0xFFFFFFFFu;
        if (set_only) {
            if (tid < L) eid = cand_id[tid];
        } else if (nS <= kMaxCand) {
            // stage the candidates' centroid rows (coalesced) and run the chains from smem
            const float* cr = a.centR[g];
            for (uint32_t e = tid; e < nS * a.D; e += nth) {
                const uint32_t r = e / a.D, jj = e % a.D;
                crow[r][jj] = cr[(size_t)cand_id[r] * a.D + jj];
            }
            __syncthreads();
            trace(10);
            if (tid < nS) {
                double sx = 0.0;
#pragma unroll 8
                for (uint32_t j = 0; j < a.D; ++j) sx = __dadd_rn(sx, __dmul_rn(pooled[j], (double)crow[tid][j]));
                ex = sx;
                eid = cand_id[tid];
            }
        } else {
            // degenerate (many near-ties): exact chains for every candidate, rank by position
            if (cand) {
                const float* cT = a.centT[g];
                double sx = 0.0;
#pragma unroll 8
                for (uint32_t j = 0; j < a.D; ++j) sx = __dadd_rn(sx, __dmul_rn(pooled[j], (double)cT[(size_t)j * Cb + tid]));
                ex = sx;
                eid = tid;
            }
        }
        uint32_t p2s = 1;
        while (p2s < (nS <= kMaxCand ? nS : Cb)) p2s <<= 1;
        trace(2);
        if (!set_only) bitonic_regs(ex, eid, nS <= kMaxCand ? p2s : a.P2, ss, si);
        __syncthreads();
        if (tid < L) si[tid] = eid;
        for (uint32_t w = tid; w < bm_words; w += nth) bitmap[w] = 0;
        __syncthreads();
        for (uint32_t b = tid; b < L; b += nth) {
            atomicOr(&bitmap[si[b] >> 5], 1u << (si[b] & 31));
            if (a.selected) a.selected[(size_t)g * a.probes + b] = si[b];
        }
        __syncthreads();
        trace(3);
    } else if (route && a.mode == 4) {
        // a BucketRouter of the caller's: its list, in its order (attention.cpp:351-353);
        // a repeated id is absorbed once per occurrence, like the reference
        for (uint32_t w = tid; w < bm_words; w += nth) bitmap[w] = 0;
        __syncthreads();
        for (uint32_t b = tid; b < L; b += nth) {
            const uint32_t c = a.given[(size_t)g * a.probes + b];
            si[b] = c;
            atomicOr(&bitmap[c >> 5], 1u << (c & 31));
        }
        __syncthreads();
    } else if (route) {
        const double* cs = a.cand_s + (size_t)g * a.n_cand;
        const uint32_t* ci = a.cand_i + (size_t)g * a.n_cand;
        if (a.P2 <= nth) {
            double sc = -INFINITY;
            uint32_t id = 0xFFFFFFFFu;
            if (tid < a.n_cand) {
                sc = cs[tid];
                id = ci[tid];
            }
            bitonic_regs(sc, id, a.P2, ss, si);
            __syncthreads();
            if (tid < L) si[tid] = id;
        } else {
            for (uint32_t c = tid; c < a.P2; c += nth) {
                ss[c] = c < a.n_cand ? cs[c] : -INFINITY;
                si[c] = c < a.n_cand ? ci[c] : 0xFFFFFFFFu;
            }
            __syncthreads();
            bitonic_smem(ss, si, a.P2);
        }
        for (uint32_t w = tid; w < bm_words; w += nth) bitmap[w] = 0;
        __syncthreads();
        for (uint32_t b = tid; b < L; b += nth) {
            atomicOr(&bitmap[si[b] >> 5], 1u << (si[b] & 31));
            if (a.selected) a.selected[(size_t)g * a.probes + b] = si[b];
        }
        __syncthreads();
    }
    if (a.route_only) return;

    // ---------------- fast path (no general-window gathers): one warp plans
    // the bucket segments with shuffles only -- sizes, counters, one tile
    // reservation, pieces, publication                attention.cpp:342-372
    {
        const uint32_t rb0 = fallback ? 0 : n - a.recent;
        const bool fast = fallback || rb0 == T || (rb0 > T && !route);
        if (fast) {
            if (tid >= 32) return;
            const uint32_t lane = tid, nh = a.n_hchunks;
            const uint32_t* offg = stage_off ? s_off : a.off + (size_t)g * (Cb + 1);
            const uint32_t* offAg = stage_off ? s_offA : a.offA + (size_t)g * (Cb + 1);
            unsigned long long keys = 0;
            uint32_t mx = 0, vrows = 0;
            for (uint32_t b0 = 0; b0 < L; b0 += 32) {
                const uint32_t b = b0 + lane;
                uint32_t lenA = 0, st = 0;
                if (b < L) {
                    const uint32_t c = si[b];
                    mx = max(mx, offg[c + 1] - offg[c]);  // raw bucket size (attention.cpp:356)
                    lenA = offAg[c + 1] - offAg[c];        // rb >= T: no in-window ids in region A
                    st = sink + offAg[c];
                }
                keys += lenA;
                const uint32_t v8 = (lenA + 7) & ~7u;
                uint32_t incl = v8;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                    if (lane >= (uint32_t)o) incl += v;
                }
                if (b < L) {
                    segs[b] = Seg{KIND_ROWS, lenA, st};
                    vpre[b] = vrows + incl - v8;
                }
                vrows += __shfl_sync(0xFFFFFFFFu, incl, 31);
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                keys += __shfl_xor_sync(0xFFFFFFFFu, keys, o);
                mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
            }
            const uint32_t ntiles = (vrows + kTileRows - 1) / kTileRows;
            uint32_t tile0 = 0;
            if (lane == 0) {
                // one atomic reserves the tiles and reports this group
                tile0 = (uint32_t)atomicAdd(&a.ctr->dynres, (1ull << 32) | (unsigned long long)(ntiles * nh));
                for (uint32_t hc = 0; hc < nh; ++hc) a.dyn_cnt[g * nh + hc] = ntiles | kCntValid;
                saap_attn_stats stt;
                stt.keys_scored = fallback ? (unsigned long long)n : (unsigned long long)sink + (n - rb0) + keys;
                stt.max_visited_bucket = fallback ? 0 : mx;
                stt.empty_attention = stt.keys_scored == 0 ? 1 : 0;
                stt.reserved = 0;
                a.stats[g] = stt;
            }
            trace(5);
            if (ntiles == 0) {
                if (lane == 0) {
                    __threadfence();
                    atomicAdd(&a.ctr->published, 1u);
                }
                return;
            }
            tile0 = __shfl_sync(0xFFFFFFFFu, tile0, 0);
            emit_tiles(a.dyn_tiles + tile0, ntiles, nh, g * nh, segs, vpre, L, gm.row_base, lane, 32);
            // one fence per lane orders every record the warp wrote (the warp
            // barrier makes the other lanes' writes cumulative) before the flags
            __syncwarp();
            __threadfence();
            __syncwarp();
            for (uint32_t e = lane; e < ntiles * nh; e += 32)
                *reinterpret_cast<volatile uint32_t*>(&a.dyn_tiles[tile0 + e].ready) = 1u;
            __syncwarp();
            if (lane == 0) {
                __threadfence();
                atomicAdd(&a.ctr->published, 1u);
                tl_mark(a.tl, 1, false);
            }
            trace(7);
            return;
        }
    }

    // ---------------- segments of the visited set      attention.cpp:342-372
    // The dense window (sink span + recent tail) is static work planned on the
    // host; this CTA appends the routed bucket segments and, for general
    // windows, the gathered rows.
    const uint32_t rb = fallback ? 0 : n - a.recent;  // recent_begin
    const uint32_t* offg = stage_off ? s_off : a.off + (size_t)g * (Cb + 1);
    const uint32_t* offAg = stage_off ? s_offA : a.offA + (size_t)g * (Cb + 1);
    const uint32_t* idxg = a.idx + gm.ivf_base;
    const uint64_t gbuf = (uint64_t)g * a.gather_cap;  // this group's gather rows
    // bucket segments: region-A prefix of each selected bucket, cut at rb
    unsigned long long my_keys = 0;
    uint32_t my_max = 0;
    for (uint32_t b = tid; b < L; b += nth) {
        const uint32_t c = si[b];
        const uint32_t raw = offg[c + 1] - offg[c];
        uint32_t lenA = offAg[c + 1] - offAg[c];
        if (rb < T) {  // ids ascend inside a bucket: the in-window ids are a suffix
            uint32_t lo = 0, hi = lenA;
            const uint32_t lim = rb - sink;
            const uint32_t* seg = idxg + offg[c];
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
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
    trace(4);

    // general windows: materialise the out-of-order rows in the gather buffer
    //   recent > hint (rb < T): region-A rows with position in [rb, T) (pos -> row map)
    //   recent < hint (rb > T): region-B rows in [T, rb) of selected buckets
    auto gather_row = [&](uint32_t src_row, uint32_t dst) {
        const uint32_t chunks = a.D / 8;  // 16-byte chunks per row
        for (uint32_t e = 0; e < chunks; ++e) {
            const uint64_t so = (gm.row_base + src_row) * a.D + e * 8;
            const uint64_t d = (gbuf + dst) * a.D + e * 8;
            *reinterpret_cast<uint4*>(a.gK + d) = *reinterpret_cast<const uint4*>(a.K + so);
            *reinterpret_cast<uint4*>(a.gV + d) = *reinterpret_cast<const uint4*>(a.V + so);
        }
    };
    if (!fallback && rb < T) {
        for (uint32_t p = tid; p < T - rb; p += nth)
            gather_row(a.invA[gm.ivf_base + (rb + p - sink)], p);
        if (tid == 0) s_gbase = T - rb;
    }
    if (route && rb > T) {
        uint32_t base = 0;
        const uint32_t warp = tid >> 5, lane = tid & 31;
        for (uint32_t p0 = T; p0 < rb; p0 += nth) {
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
            for (uint32_t w = 0; w < nth / 32; ++w) {
                if (w < warp) wex += s_wcnt[w];
                tot += s_wcnt[w];
            }
            if (f) gather_row(pos, base + wex + __popc(bal & ((1u << lane) - 1)));
            base += tot;
            __syncthreads();
        }
        if (tid == 0) {
            s_filtered = base;
            s_gbase = base;
        }
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t nseg = L;
        if (!fallback && s_gbase) segs[nseg++] = Seg{KIND_LIST, s_gbase, gbuf};
        s_nseg = nseg;
    }
    __syncthreads();

    // ---------------- virtual row layout: segment s occupies 8-aligned rows
    // [vpre[s], vpre[s] + ceil8(len_s)); tile t = virtual rows [128t, 128t+128)
    const uint32_t nseg = s_nseg;
    {
        const uint32_t per = (nseg + nth - 1) / nth;
        const uint32_t lo = min(nseg, tid * per), hi = min(nseg, lo + per);
        uint32_t sum = 0;
        for (uint32_t s2 = lo; s2 < hi; ++s2) sum += (segs[s2].len + 7) & ~7u;
        const uint32_t lane = tid & 31, warp = tid >> 5;
        uint32_t incl = sum;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= (uint32_t)o) incl += v;
        }
        if (lane == 31) s_wcnt[warp] = incl;
        __syncthreads();
        uint32_t wbase = 0, tot = 0;
        for (uint32_t w = 0; w < nth / 32; ++w) {
            if (w < warp) wbase += s_wcnt[w];
            tot += s_wcnt[w];
        }
        uint32_t run = wbase + incl - sum;
        for (uint32_t s2 = lo; s2 < hi; ++s2) {
            vpre[s2] = run;
            run += (segs[s2].len + 7) & ~7u;
        }
        if (tid == 0) s_vrows = tot;
    }
    __syncthreads();
    const uint32_t nh = a.n_hchunks;
    if (tid == 0) {
        const uint32_t ntiles = (s_vrows + kTileRows - 1) / kTileRows;
        s_ntiles = ntiles;
        // reserve this group's dynamic tiles, then report the reservation:
        // decode producers treat the stream as final once every group has
        s_tile0 = (uint32_t)atomicAdd(&a.ctr->dynres, (1ull << 32) | (unsigned long long)(ntiles * nh));
        for (uint32_t hc = 0; hc < nh; ++hc) a.dyn_cnt[g * nh + hc] = ntiles | kCntValid;
        unsigned long long keys;
        if (fallback) keys = n;
        else keys = (unsigned long long)sink + (n - rb) + s_keys + s_filtered;
        saap_attn_stats st;
        st.keys_scored = keys;
        st.max_visited_bucket = fallback ? 0 : s_maxv;
        st.empty_attention = keys == 0 ? 1 : 0;
        st.reserved = 0;
        a.stats[g] = st;
    }
    __syncthreads();
    trace(5);
    const uint32_t ntiles = s_ntiles, tile0 = s_tile0;
    if (ntiles == 0) {
        if (tid == 0) {
            __threadfence();
            atomicAdd(&a.ctr->published, 1u);
        }
        return;
    }
    trace(6);
    emit_tiles(a.dyn_tiles + tile0, ntiles, nh, g * nh, segs, vpre, nseg, gm.row_base, tid, nth);
    __threadfence();  // records before the ready flags
    __syncthreads();
    for (uint32_t e = tid; e < ntiles * nh; e += nth)
        *reinterpret_cast<volatile uint32_t*>(&a.dyn_tiles[tile0 + e].ready) = 1u;
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        atomicAdd(&a.ctr->published, 1u);
    }
    trace(7);
}

// ============================================================ fused cluster routing
// Centroid router + planner in one launch (CentroidRouter::select
// attention.cpp:275-306, top_l_ids :259-271, visited set :342-372).  A cluster
// of 8 CTAs serves one slot (<= 8 contexts sharing a partition): CTA r scores
// centroids [r*C/8, (r+1)*C/8) for every context of the slot in fp32 (its
// centroid slice stays in registers) and stores context k's scores into CTA
// k's shared memory (distributed shared memory).  After one cluster barrier
// CTA k owns all C scores of context k and selects its top-l exactly: select
// of the l-th score, candidates within the error bound 2B of it; when more
// than l, an fp64 re-scoring of the candidates with its own (1e-9 x smaller)
// band, and exact fp64 chains (reference operation order) only when that is
// still ambiguous or the ordered list is requested.  Warp 0 then plans and
// publishes the context's bucket tiles.
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void dsmem_st_f32(float* local, uint32_t cta, float v) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(cta));
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(remote), "f"(v) : "memory");
}
__device__ __forceinline__ void dsmem_st_f64(double* local, uint32_t cta, double v) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(cta));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(remote), "d"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int D, int S>
__global__ void __launch_bounds__(kClusterThreads, 1) route_cluster_kernel(ClusterRouteArgs a) {
    constexpr uint32_t NT = kClusterThreads;
    constexpr uint32_t TPC = NT / S, DPT = D / TPC;  // threads per centroid, dims per thread
    static_assert(NT % S == 0 && D % TPC == 0 && DPT % 4 == 0, "slice geometry");
    constexpr uint32_t kMaxC = 1024;
    constexpr uint32_t kMaxCand = 64;
    __shared__ float sc_all[kMaxC];            // this CTA's context: every centroid's approximate (f32) score
    __shared__ double pd[D];                   // own context: pooled query in fp64
    __shared__ uint32_t s_off[kMaxC + 1], s_offA[kMaxC + 1];
    __shared__ uint32_t hist[256];
    __shared__ uint32_t cand_id[kMaxCand], sel[kMaxC];
    // phase-local buffers share one region: scoring | exact sort | planning
    union Phase {
        struct {
            float pf[kSlotGroups][D];     // pooled queries (f32-rounded) of the slot's contexts
        } score;
        struct {
            double xs[kMaxC];
            uint32_t xi[kMaxC];
        } sort;
        struct {
            Seg segs[kMaxC];
            uint32_t vpre[kMaxC];
        } plan;
    };
    __shared__ __align__(16) Phase ph;
    auto& pf = ph.score.pf;
    auto& xs = ph.sort.xs;
    auto& xi = ph.sort.xi;
    auto& segs = ph.plan.segs;
    auto& vpre = ph.plan.vpre;
    __shared__ uint32_t s_pref, s_need, s_ncand, s_nb, s_bsel, s_bcnt;
    __shared__ double s_mm[2][NT / 32], s_bnd[32], s_tl;
    __shared__ double s_n2[NT / 32];
    pdl_trigger();
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    const uint32_t rank = cluster_rank(), slot = blockIdx.x / kClusterCtas;
    if (tid == 0) tl_mark(a.tl, 1, true);
    auto gt = []() {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        return t;
    };
    if (a.trace && tid == 0) a.trace[16 + 6 * blockIdx.x] = gt();
    unsigned long long t0 = 0;
    const bool tr = a.trace && slot == 0 && rank == 0 && tid == 0;
    if (tr) t0 = clock64();
    auto trace = [&](int k) {
        if (tr) a.trace[k] = clock64() - t0;
    };
    extern __shared__ __align__(16) float dyn_smem[];
    float* slab = dyn_smem;                    // [D][S] this CTA's centroid slice (transposed)
    const ApproxSlot sl = slot < a.n_inline ? a.islots[slot] : a.slots[slot];
    const uint32_t ng = sl.count, C = a.C;  // C == 8 * S
    float* qs = slab + (size_t)D * S;          // [ng][G][D] member queries
    // partial dot products [8][NT] during scoring; the same bytes hold the
    // candidate rows of the re-scoring later
    float (*red)[NT] = reinterpret_cast<float (*)[NT]>(qs + (size_t)kSlotGroups * a.G * D);
    const bool own = rank < ng;
    const uint32_t g = own ? sl.group[rank] : 0u;
    // ---- loads, all in one round trip: the slice rows and the member query
    // rows by bulk copies (TMA engine) onto one barrier, own offsets by loads
    __shared__ __align__(8) uint64_t bar;
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint32_t qbytes = a.G * D * 4;
    if (tid == 0) mbar_arrive_expect_tx(&bar, D * S * 4 + ng * qbytes);
    __syncthreads();
    if (sl.centB) {  // the rank's slab is contiguous: one bulk copy
        if (tid == 0) bulk_g2s(slab, sl.centB + (size_t)rank * D * S, D * S * 4, &bar);
    } else {
        for (uint32_t j = tid; j < D; j += NT)
            bulk_g2s(slab + (size_t)j * S, sl.centT + (size_t)j * C + rank * S, S * 4, &bar);
    }
    for (uint32_t k = tid; k < ng; k += NT)
        bulk_g2s(qs + (size_t)k * a.G * D, a.q_route + (size_t)sl.group[k] * a.G * D, qbytes, &bar);
    GroupMeta gm{};
    if (own) {
        gm = a.meta[g];
        const uint32_t* og = a.off + (size_t)g * (C + 1);
        const uint32_t* oAg = a.offA + (size_t)g * (C + 1);
        for (uint32_t i = tid; i <= C; i += NT) {
            s_off[i] = og[i];
            s_offA[i] = oAg[i];
        }
    }
    mbar_wait(&bar, 0);
    // pooled_j = sum_i q_ij in fp64, rows in order   attention.cpp:289-295
    // (rows of absent members are zero: the scoring below runs every chain)
    for (uint32_t e = tid; e < kSlotGroups * D; e += NT) {
        const uint32_t k = e / D, j = e % D;
        const double ps = k < ng ? pooled_sum(qs + (size_t)k * a.G * D + j, a.G, D) : 0.0;
        pf[k][j] = (float)ps;
        if (k == rank) pd[j] = ps;
    }
    __syncthreads();
    trace(0);
    // ---- f32 scores of this CTA's slice for every member, to the owners
    // the slice column stays in registers; pooled rows are float4 broadcasts.
    // f32 FMA chains (4x the fp64 rate): the candidate band below holds more
    // than the l winners only when a score lies within ~1e-5 |p| cmax of the
    // boundary; those contexts are re-scored in fp64 (and exactly if needed)
    const uint32_t cl = tid % S, part = tid / S;
    float cv[DPT];
#pragma unroll
    for (int jj = 0; jj < (int)DPT; ++jj) cv[jj] = slab[(part * DPT + jj) * S + cl];
    // the slot's contexts are independent accumulation chains (ILP)
    float x[kSlotGroups];
#pragma unroll
    for (int k = 0; k < kSlotGroups; ++k) x[k] = 0.f;
#pragma unroll
    for (int j4 = 0; j4 < (int)DPT / 4; ++j4) {
        float4 p4[kSlotGroups];
#pragma unroll
        for (int k = 0; k < kSlotGroups; ++k) p4[k] = reinterpret_cast<const float4*>(&pf[k][part * DPT])[j4];
#pragma unroll
        for (int k = 0; k < kSlotGroups; ++k) {
            x[k] = fmaf(p4[k].x, cv[4 * j4], x[k]);
            x[k] = fmaf(p4[k].y, cv[4 * j4 + 1], x[k]);
            x[k] = fmaf(p4[k].z, cv[4 * j4 + 2], x[k]);
            x[k] = fmaf(p4[k].w, cv[4 * j4 + 3], x[k]);
        }
    }
#pragma unroll
    for (int k = 0; k < kSlotGroups; ++k)
        if ((uint32_t)k < ng) red[k][tid] = x[k];
    __syncthreads();
    trace(6);
    for (uint32_t e = tid; e < ng * S; e += NT) {
        const uint32_t k = e / S, cc = e % S;
        float x = 0.f;
        for (uint32_t p = 0; p < TPC; ++p) x += red[k][p * S + cc];
        dsmem_st_f32(&sc_all[rank * S + cc], k, x);
    }
    trace(7);
    // every owner now holds all C scores of its context; no distributed
    // shared memory is touched after this barrier, so each CTA leaves as soon
    // as it is done (its SM goes to a decode CTA)
    cluster_sync_all();
    trace(1);
    if (a.trace && tid == 0) a.trace[16 + 6 * blockIdx.x + 1] = gt();
    if (!own) {
        if (tid == 0) tl_mark(a.tl, 1, false);
        return;
    }
    const uint32_t n = gm.n, sink = gm.sink, T = gm.T;
    const bool fallback = n <= sink + a.recent;
    const bool route = !fallback && a.probes > 0;
    const uint32_t L = route ? a.probes : 0u;
    constexpr uint32_t PER = kMaxC / NT;  // scores per thread
    if (route) {
        // |pooled|_2 for the error bound
        double part2 = 0.0;
        for (uint32_t j = tid; j < D; j += NT) part2 += pd[j] * pd[j];
        for (int o = 16; o; o >>= 1) part2 += __shfl_xor_sync(0xFFFFFFFFu, part2, o);
        if (lane == 0) s_n2[tid >> 5] = part2;
        // radix select (8-bit digits, MSB first): the L-th largest score
        uint32_t key[PER];  // (radix fallback: order-preserving keys of the f32-rounded scores)
        double av[PER];
#pragma unroll
        for (uint32_t i = 0; i < PER; ++i) {
            const uint32_t cc = tid + i * NT;
            av[i] = cc < C ? sc_all[cc] : -INFINITY;
            const uint32_t u = __float_as_uint((float)av[i]);
            key[i] = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
        }
        // the L-th largest score.  Pass 1: 256 linear buckets over [min, max]
        // (monotone in the score), suffix counts find the boundary bucket;
        // pass 2: one warp ranks its (usually few) members.  Radix select
        // (8-bit digits, MSB first) when the boundary bucket holds > 32.
        {
            double lmn = INFINITY, lmx = -INFINITY;
#pragma unroll
            for (uint32_t i = 0; i < PER; ++i)
                if (tid + i * NT < C) {
                    lmn = fmin(lmn, av[i]);
                    lmx = fmax(lmx, av[i]);
                }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                lmn = fmin(lmn, __shfl_xor_sync(0xFFFFFFFFu, lmn, o));
                lmx = fmax(lmx, __shfl_xor_sync(0xFFFFFFFFu, lmx, o));
            }
            if (lane == 0) {
                s_mm[0][tid >> 5] = lmn;
                s_mm[1][tid >> 5] = lmx;
            }
            if (tid < 256) hist[tid] = 0;
            if (tid == 0) {
                s_nb = 0;
                s_bcnt = 0xFFFFFFFFu;
                s_ncand = 0;  // (the candidate scan below needs no barrier of its own)
            }
            __syncthreads();
            // every warp reduces the NT/32 warp extremes itself (one load per
            // lane and shuffles, no serial scan of shared memory)
            constexpr uint32_t NW = NT / 32;
            static_assert(NW <= 32 && (NW & (NW - 1)) == 0, "warp count");
            double vmn = s_mm[0][lane % NW], vmx = s_mm[1][lane % NW];
#pragma unroll
            for (uint32_t o = NW / 2; o; o >>= 1) {
                vmn = fmin(vmn, __shfl_xor_sync(0xFFFFFFFFu, vmn, o));
                vmx = fmax(vmx, __shfl_xor_sync(0xFFFFFFFFu, vmx, o));
            }
            const double span = vmx - vmn, scale = 256.0 / span;
            const bool lin = span > 0.0 && scale < INFINITY && vmx < INFINITY && vmn > -INFINITY;
            uint32_t bk[PER];
            if (lin) {
#pragma unroll
                for (uint32_t i = 0; i < PER; ++i) {
                    bk[i] = min(255u, (uint32_t)((av[i] - vmn) * scale));
                    if (tid + i * NT < C) atomicAdd(&hist[bk[i]], 1u);
                }
                __syncthreads();
                if (tid < 32) {
                    uint32_t cnt[8], tot = 0;
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        cnt[b] = hist[255 - 8 * tid - b];
                        tot += cnt[b];
                    }
                    uint32_t incl = tot;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                        if (tid >= (uint32_t)o) incl += v;
                    }
                    const uint32_t before = incl - tot;
                    if (before < L && incl >= L) {
                        uint32_t run = before;
#pragma unroll
                        for (int b = 0; b < 8; ++b) {
                            if (run + cnt[b] >= L) {
                                s_bsel = 255 - 8 * tid - b;
                                s_need = L - run;
                                s_bcnt = cnt[b];
                                break;
                            }
                            run += cnt[b];
                        }
                    }
                }
                __syncthreads();
            }
            if (lin && s_bcnt <= 32) {
                const uint32_t bsel = s_bsel;
#pragma unroll
                for (uint32_t i = 0; i < PER; ++i)
                    if (tid + i * NT < C && bk[i] == bsel) s_bnd[atomicAdd(&s_nb, 1u)] = av[i];
                __syncthreads();
                if (tid < 32) {
                    const uint32_t nb = s_nb;
                    const double v = tid < nb ? s_bnd[tid] : -INFINITY;
                    uint32_t rank = 0;
                    for (uint32_t k = 0; k < nb; ++k) {
                        const double u = s_bnd[k];
                        rank += (u > v || (u == v && k < tid)) ? 1u : 0u;
                    }
                    if (tid < nb && rank == s_need - 1) s_tl = v;  // the exact l-th largest
                }
                __syncthreads();
            } else {
            if (tid == 0) {
                s_pref = 0;
                s_need = L;
            }
            for (int shift = 24; shift >= 0; shift -= 8) {
                if (tid < 256) hist[tid] = 0;
                __syncthreads();
                const uint32_t pref = s_pref;
                const uint32_t hmask = shift == 24 ? 0u : (0xFFFFFFFFu << (shift + 8));
    #pragma unroll
                for (uint32_t i = 0; i < PER; ++i)
                    if (tid + i * NT < C && (key[i] & hmask) == (pref & hmask)) atomicAdd(&hist[(key[i] >> shift) & 255u], 1u);
                __syncthreads();
                if (tid < 32) {
                    uint32_t cnt[8], tot = 0;
    #pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        cnt[b] = hist[255 - 8 * tid - b];
                        tot += cnt[b];
                    }
                    uint32_t incl = tot;
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                        if (tid >= (uint32_t)o) incl += v;
                    }
                    const uint32_t need = s_need, before = incl - tot;
                    if (before < need && incl >= need) {
                        uint32_t run = before;
    #pragma unroll
                        for (int b = 0; b < 8; ++b) {
                            if (run + cnt[b] >= need) {
                                s_pref = pref | ((uint32_t)(255 - 8 * tid - b) << shift);
                                s_need = need - run;
                                break;
                            }
                            run += cnt[b];
                        }
                    }
                }
                __syncthreads();
            }
            // radix select ran on the f32-rounded scores: the l-th largest
            // f32 key, lowered by its rounding (<= 2^-24 relative) so the
            // band below stays a superset
            if (tid == 0) {
                const uint32_t tk = s_pref;
                const double t32 = (double)__uint_as_float((tk & 0x80000000u) ? (tk & 0x7FFFFFFFu) : ~tk);
                s_tl = t32 - fabs(t32) * 0x1p-23;
            }
            __syncthreads();
            }
        }
        trace(2);
        const double t_l = s_tl;
        double n2 = 0.0;
        {  // (any order: n2 only sizes the error bound, which carries a 1% margin)
            n2 = s_n2[lane % (NT / 32)];
#pragma unroll
            for (uint32_t o = (NT / 32) / 2; o; o >>= 1) n2 += __shfl_xor_sync(0xFFFFFFFFu, n2, o);
        }
        // |approx - exact| <= B: the approximate dot (f32 FMA chains of DPT
        // terms over the f32-rounded pooled query, TPC partial sums in f32)
        // and the reference's sequential fp64 chain of the fp64 pooled query
        // (D products, D sums) each lie within gamma_n sum|p_j c_j| of the
        // real dot product (u = 2^-24 and 2^-53), sum|p_j c_j| <= |p|_2
        // max|c|_2; the band is 2B, widened 2x
        const double pc = sqrt(n2) * (double)a.cmax[g];
        const double B2 = 2.0 * 2.0 * ((double)(DPT + TPC + 2) * 0x1p-24 + (double)(2 * D + 2) * 0x1p-53) * pc * 1.01;
#pragma unroll
        for (uint32_t i = 0; i < PER; ++i) {
            const uint32_t cc = tid + i * NT;
            const bool cand = cc < C && av[i] >= t_l - B2;
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, cand);
            uint32_t wbase = 0;
            if (lane == 0 && bal) wbase = atomicAdd(&s_ncand, __popc(bal));
            wbase = __shfl_sync(0xFFFFFFFFu, wbase, 0);
            const uint32_t slotc = wbase + __popc(bal & ((1u << lane) - 1));
            if (cand && slotc < kMaxCand) cand_id[slotc] = cc;
        }
        __syncthreads();
        const uint32_t nS = s_ncand;
        trace(3);
        // the candidates are a superset of the exact top-L: exactly L of them
        // are the exact set (attention does not depend on the order)
        if (a.selected == nullptr && nS == L && L <= kMaxCand) {
            if (tid < L) sel[tid] = cand_id[tid];
        } else if (nS <= kMaxCand) {
            // the candidates' centroid rows come from global memory (row-major,
            // L2-resident; one round trip with every load in flight).
            // First an fp64 FMA re-scoring (TPR threads per candidate): its
            // band (~1e-14 |p| cmax) almost always holds exactly the l winners
            const float* cR = a.centR[g];
            bool done = false;
            if (a.selected == nullptr) {
                constexpr uint32_t TPR = NT / kMaxCand, DPR = D / TPR;
                static_assert(NT % kMaxCand == 0 && D % (4 * TPR) == 0 && TPR <= 32, "re-scoring geometry");
                const uint32_t ci = tid / TPR, pr = tid % TPR;
                double sx = 0.0;
                if (ci < nS) {
                    const float4* row = reinterpret_cast<const float4*>(cR + (size_t)cand_id[ci] * D + pr * DPR);
                    float4 v[DPR / 4];
#pragma unroll
                    for (uint32_t i = 0; i < DPR / 4; ++i) v[i] = __ldg(row + i);
                    const double* pp = pd + pr * DPR;
#pragma unroll
                    for (uint32_t i = 0; i < DPR / 4; ++i) {
                        sx = fma(pp[4 * i], (double)v[i].x, sx);
                        sx = fma(pp[4 * i + 1], (double)v[i].y, sx);
                        sx = fma(pp[4 * i + 2], (double)v[i].z, sx);
                        sx = fma(pp[4 * i + 3], (double)v[i].w, sx);
                    }
                }
#pragma unroll
                for (uint32_t o = 1; o < TPR; o <<= 1) sx += __shfl_xor_sync(0xFFFFFFFFu, sx, o);
                if (pr == 0 && ci < nS) xs[ci] = sx;
                if (tid == 0) s_nb = 0;
                __syncthreads();
                if (a.trace && tid == 0) a.trace[16 + 6 * blockIdx.x + 5] = gt();
                if (tid < nS) {  // the l-th largest fp64 score, by rank
                    const double v = xs[tid];
                    uint32_t r = 0;
#pragma unroll 8
                    for (uint32_t k = 0; k < nS; ++k) {
                        const double u = xs[k];
                        r += (u > v || (u == v && k < tid)) ? 1u : 0u;
                    }
                    if (r == L - 1) s_tl = v;
                }
                __syncthreads();
                const double B64 = 2.0 * 2.0 * (double)(DPR + TPR + 2 * D + 2) * 0x1p-53 * pc * 1.01;
                if (tid < nS && xs[tid] >= s_tl - B64) xi[atomicAdd(&s_nb, 1u)] = cand_id[tid];
                __syncthreads();
                done = s_nb == L;
                if (done && tid < L) sel[tid] = xi[tid];
                __syncthreads();
            }
            if (!done) {
                // exact fp64 chains (attention.cpp:296-304: mul rounded before
                // add), ordered (score desc, id asc): attention.cpp:263-268
                double ex = -INFINITY;
                uint32_t eid = 0xFFFFFFFFu;
                if (tid < nS) {
                    const float* row = cR + (size_t)cand_id[tid] * D;
                    double sx = 0.0;
#pragma unroll 8
                    for (uint32_t j = 0; j < D; ++j) sx = __dadd_rn(sx, __dmul_rn(pd[j], (double)__ldg(row + j)));
                    ex = sx;
                    eid = cand_id[tid];
                }
                uint32_t p2s = 1;
                while (p2s < nS) p2s <<= 1;
                bitonic_regs(ex, eid, p2s, xs, xi);
                __syncthreads();
                if (tid < L) sel[tid] = eid;
            }
        } else {
            // degenerate (many near-ties): exact chains for every candidate
            uint32_t P2 = 1;
            while (P2 < C) P2 <<= 1;
            for (uint32_t cc = tid; cc < P2; cc += NT) {
                double ex = -INFINITY;
                uint32_t eid = 0xFFFFFFFFu;
                if (cc < C && sc_all[cc] >= t_l - B2) {
                    const float* row = a.centR[g] + (size_t)cc * D;
                    double sx = 0.0;
                    for (uint32_t j = 0; j < D; ++j) sx = __dadd_rn(sx, __dmul_rn(pd[j], (double)row[j]));
                    ex = sx;
                    eid = cc;
                }
                xs[cc] = ex;
                xi[cc] = eid;
            }
            __syncthreads();
            bitonic_smem(xs, xi, P2);
            if (tid < L) sel[tid] = xi[tid];
        }
        __syncthreads();
        if (a.selected)
            for (uint32_t b = tid; b < L; b += NT) a.selected[(size_t)g * a.probes + b] = sel[b];
        trace(4);
        if (a.trace && tid == 0) {
            a.trace[16 + 6 * blockIdx.x + 2] = gt();
            a.trace[16 + 6 * blockIdx.x + 4] = nS;
        }
    }
    // ---- plan: warp 0 lays the bucket segments out as 8-aligned virtual rows
    // and reserves the context's tiles; every thread then writes tile records
    const uint32_t nh = a.n_hchunks;
    const uint32_t rb0 = fallback ? 0 : n - a.recent;  // == T (recent == the layer's hint)
    __shared__ uint32_t s_tile0, s_ntiles;
    unsigned long long res = 0;  // warp 0 lane 0: the pending tile reservation
    if (tid < 32) {
        unsigned long long keys = 0;
        uint32_t mx = 0, vrows = 0;
        for (uint32_t b0 = 0; b0 < L; b0 += 32) {
            const uint32_t b = b0 + lane;
            uint32_t lenA = 0, st = 0;
            if (b < L) {
                const uint32_t cc = sel[b];
                mx = max(mx, s_off[cc + 1] - s_off[cc]);  // raw bucket size (attention.cpp:356)
                lenA = s_offA[cc + 1] - s_offA[cc];
                st = sink + s_offA[cc];
            }
            keys += lenA;
            const uint32_t v8 = (lenA + 7) & ~7u;
            uint32_t incl = v8;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= (uint32_t)o) incl += v;
            }
            if (b < L) {
                segs[b] = Seg{KIND_ROWS, lenA, st};
                vpre[b] = vrows + incl - v8;
            }
            vrows += __shfl_sync(0xFFFFFFFFu, incl, 31);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            keys += __shfl_xor_sync(0xFFFFFFFFu, keys, o);
            mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
        }
        const uint32_t ntiles = (vrows + kTileRows - 1) / kTileRows;
        if (lane == 0) {
            // the reservation travels while the records are built (its
            // result is read only after emit_tiles)
            res = atomicAdd(&a.ctr->dynres, (1ull << 32) | (unsigned long long)(ntiles * nh));
            s_ntiles = ntiles;
            for (uint32_t hc = 0; hc < nh; ++hc) a.dyn_cnt[g * nh + hc] = ntiles | kCntValid;
            saap_attn_stats stt;
            stt.keys_scored = fallback ? (unsigned long long)n : (unsigned long long)sink + (n - rb0) + keys;
            stt.max_visited_bucket = fallback ? 0 : mx;
            stt.empty_attention = stt.keys_scored == 0 ? 1 : 0;
            stt.reserved = 0;
            a.stats[g] = stt;
        }
    }
    (void)T;
    __syncthreads();
    const uint32_t ntiles = s_ntiles;
    // records are built in shared memory (the centroid slice is no longer
    // read) and copied out once the reservation is back
    TileRec* stage = reinterpret_cast<TileRec*>(slab);
    const bool staged = ntiles * nh <= (uint32_t)((size_t)D * S * 4 / sizeof(TileRec));
    // (a few tiles: a warp per tile builds its pieces in parallel; many tiles:
    // a thread per tile)
    if (ntiles && staged) {
        if (ntiles <= NT / 32) emit_tiles_warp(stage, ntiles, nh, g * nh, segs, vpre, L, gm.row_base, tid >> 5, NT / 32, lane);
        else emit_tiles(stage, ntiles, nh, g * nh, segs, vpre, L, gm.row_base, tid, NT);
    }
    if (tid == 0) s_tile0 = (uint32_t)res;
    __syncthreads();
    const uint32_t tile0 = s_tile0;
    trace(8);
    if (ntiles) {
        if (staged) {
            constexpr uint32_t W16 = sizeof(TileRec) / 16;
            const uint4* src = reinterpret_cast<const uint4*>(stage);
            uint4* dst = reinterpret_cast<uint4*>(a.dyn_tiles + tile0);
            for (uint32_t e = tid; e < ntiles * nh * W16; e += NT) dst[e] = src[e];
        } else {
            emit_tiles(a.dyn_tiles + tile0, ntiles, nh, g * nh, segs, vpre, L, gm.row_base, tid, NT);
        }
        // every thread orders its own records; the barrier makes them all
        // precede every ready flag
        __threadfence();
        __syncthreads();
        trace(9);
        for (uint32_t e = tid; e < ntiles * nh; e += NT)
            *reinterpret_cast<volatile uint32_t*>(&a.dyn_tiles[tile0 + e].ready) = 1u;
        trace(10);
    }
    __syncthreads();
    // the context is published by a thread with no unfenced store (the record
    // copies were fenced above): its release reduction does not wait
    if (tid == NT - 1) {
        asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(&a.ctr->published), "r"(1u) : "memory");
        tl_mark(a.tl, 1, false);
        if (a.trace) a.trace[16 + 6 * blockIdx.x + 3] = gt();
    }
    trace(5);
}

// ============================================================ attention
// One CTA per SM.  Warp 8 produces: TMA (cp.async.bulk.tensor, 128B/64B
// swizzle) loads of 128-row K and V tiles into an NS-deep ring; the 8
// compute warps each own 16 rows of a tile and run QK^T and PV on the tensor
// cores (mma.sync m16n8k16, fp32 accumulation):
//   S: A = [q1; q2; q3] (3-term bf16 split of q, fp32-exact), B = K rows
//   O: A = [p1; p2; p3] (3-term bf16 split of the fp32 softmax weights,
//      ~fp32-exact), B = V rows (ldmatrix.trans)
// with a per-warp online softmax (lazy rescaling), merged across warps at
// the end of an item and across items by the last CTA of a query slot.
template <int D>
struct DecodeCfg {
    static constexpr int RB = 2 * D;                   // bytes per row
    static constexpr int HALF = RB >= 128 ? 128 : RB;  // swizzle row bytes
    static constexpr int HALVES = RB / HALF;
    static constexpr int TILE_BYTES = kTileRows * RB;  // K (or V) bytes per tile
    static constexpr int NS = D == 128 ? 3 : (D == 64 ? 6 : 8);
    static constexpr int KSTEPS = D / 16;
    static constexpr int NT = D / 8;  // PV n-tiles
};

constexpr int kUnit = 8;  // work records per bulk copy (two units in flight)

template <int D>
struct DecodeSmem {
    using CF = DecodeCfg<D>;
    static constexpr bool kPostQ = false;
    uint8_t K[CF::NS][CF::TILE_BYTES];
    uint8_t V[CF::NS][CF::TILE_BYTES];
    // the run's A fragments (3-term bf16 split of its f32 queries), built once per run by
    // the 8 consumer warps together: per k-step 16 lanes x {t1, t3} x {lo, hi}
    // + 16 lanes x {t2} x {lo, hi}
    alignas(16) uint32_t qfrag[CF::KSTEPS * 96];
    float redO[kComputeWarps][kHeadsPerSlot][D];
    float redm[kComputeWarps][kHeadsPerSlot];
    float redl[kComputeWarps][kHeadsPerSlot];
    uint64_t full[CF::NS];
    uint64_t empty[CF::NS];
    int4 meta[CF::NS];    // qslot (-1: end), flags (1 first | 2 last | nq << 8), run index, run tiles
    uint4 valid[CF::NS];  // 128-bit row validity mask
    uint64_t st_full;     // the 8 consumer warps deposited a run's (m, l, O) states
    uint64_t st_empty;    // the merge warp has read them
    uint32_t st_slot, st_tiles, st_run;
    // producer's record units: up to kUnit consecutive work records per bulk
    // copy, two in flight
    alignas(16) TileRec urec[2][kUnit];
    uint64_t urec_bar[2];
};

// byte offset of (row, 16-byte chunk of the row) in a tile laid out as 8-row
// groups [group][half][8][HALF] with the TMA swizzle (128B: chunk ^ row;
// 64B: chunk ^ (row >> 1)); ldmatrix reads of 8 rows are conflict-free
template <int D>
__device__ __forceinline__ uint32_t toff(uint32_t row, uint32_t chunk) {
    using CF = DecodeCfg<D>;
    constexpr uint32_t CPH = CF::HALF / 16;  // chunks per half row
    const uint32_t g = row >> 3, r = row & 7, h = chunk / CPH, cc = chunk % CPH;
    const uint32_t base = g * 8 * CF::RB + h * 8 * CF::HALF;
    if constexpr (CF::HALF == 128) return base + r * 128 + ((cc ^ r) << 4);
    else return base + r * 64 + ((cc ^ ((r >> 1) & 3)) << 4);
}

// K/V rows are streamed once per step: loaded with an L2 evict_first policy so
// the step's small hot data (work records, offsets, partials) stays in L2.
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int x, int y,
                                      uint64_t* bar, uint64_t policy) {
    asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
            "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
            "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
            : "memory");
}
__device__ __forceinline__ void tma4d(void* dst, const CUtensorMap* map, int y, uint64_t* bar,
                                      uint64_t policy) {
    asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
            "[%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
            "l"(map), "r"(0), "r"(y), "r"(0), "r"(0), "r"(smem_u32(bar)), "l"(policy)
            : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, "
            "{%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};"
            : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    return (uint32_t)f32_to_bf16_rne(lo) | ((uint32_t)f32_to_bf16_rne(hi) << 16);
}
__device__ __forceinline__ float bf16_round(float x) {
    return __uint_as_float((uint32_t)f32_to_bf16_rne(x) << 16);
}

// The decode producer warp (shared by the mma.sync and tcgen05 decode
// kernels): claims work-stream chunks, fetches their records and issues the
// K/V tile loads into the stage ring of `s` (full/empty barriers, meta,
// valid, urec).
template <int D, class SM>
__device__ __forceinline__ void decode_producer(const DecodeArgs& a, const DecodeMaps& maps, SM& s,
                                                int lane) {
    using CF = DecodeCfg<D>;
    auto gtime = []() {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        return t;
    };
    // ------------------------------------------------ producer
    // Work stream: [static tiles | dynamic tiles].  Guided self-scheduling
    // over one tile counter: CTA b first takes static tiles
    // [b*CS, (b+1)*CS) without an atomic, then claims chunks from the
    // counter whose size shrinks with the remaining work once the stream
    // length is final (ceil(rem / 2P), capped at `chunk`), so no CTA holds
    // a large chunk when the others run dry.  A claim is issued one chunk
    // ahead (its atomic travels while the current chunk is issued).
    // A chunk's records arrive in units of up to kUnit consecutive records,
    // one bulk copy each, double-buffered.  Each record carries its byte
    // count and row mask (tile_finish), so issuing a tile is a stage wait,
    // one expect_tx and one TMA request per piece for K and V.
    asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.map[lane]) : "memory");
    const uint64_t pol = l2_evict_first_policy();
    const uint32_t W = a.n_static, CH = a.chunk;
    const uint32_t CS = a.chunk_st, P = gridDim.x;
    const uint32_t pre = min(W, P * CS);  // tiles of the pre-assigned first chunks
    uint32_t total = a.n_plan_groups ? 0xFFFFFFFFu : W;  // stream length once final
    uint32_t known = W;                                  // W + reserved dynamic tiles
    // (shared counters are read by lane 0 and broadcast: every lane must
    // see the same stream length and claim size, whatever their timing)
    auto refresh = [&]() {
        if (total != 0xFFFFFFFFu) return;
        unsigned long long dr = 0;
        if (lane == 0) dr = ld_acquire_u64(&a.ctr->dynres);
        dr = __shfl_sync(0xFFFFFFFFu, dr, 0);
        known = W + (uint32_t)dr;
        if ((uint32_t)(dr >> 32) >= a.n_plan_groups) total = known;
    };
    bool all_pub = a.n_plan_groups == 0;
    // dynamic records are published with release stores: once every
    // planner CTA reported (one acquire) no per-record check is needed;
    // before that every lane acquires one flag of the chunk, and the warp
    // barrier orders them before lane 0's (async-proxy) record copies
    auto dyn_ready = [&](uint32_t b0, uint32_t b1) -> bool {
        if (all_pub) return true;
        uint32_t pub = 0;
        if (lane == 0) pub = ld_acquire_u32(&a.ctr->published);
        if (__shfl_sync(0xFFFFFFFFu, pub, 0) >= a.n_plan_groups) {
            all_pub = true;
            __syncwarp();
            return true;
        }
        bool ok = true;
        const uint32_t i = max(b0, W) + lane;
        if (i < b1) ok = ld_acquire_u32(&a.dyn_tiles[i - W].ready) != 0;
        const bool all = __all_sync(0xFFFFFFFFu, ok);
        __syncwarp();
        return all;
    };
    // claims: [pre + returned, + size).  A claim is issued late -- when
    // claim_lead tiles of the current chunk are left to issue -- so a CTA
    // never holds more than about one chunk beyond its ring: at the
    // stream's end no CTA sits on tiles while the others run dry.  Its
    // atomic travels while those tiles are issued (the result register is
    // read only when the next chunk's records are fetched).
    uint32_t cl_ret = 0, cl_size = 0, hint = pre;
    bool cl_pend = false;
    // (false: no ticket now -- the planner has not reserved the tiles a claim
    // would cover yet; the caller polls)
    auto claim = [&]() -> bool {
        uint32_t sz = CH;
        if (total != 0xFFFFFFFFu) {
            // the counter has moved on by about one claim per CTA since
            // this CTA's last claim returned `hint`
            const uint32_t seen = hint + P * cl_size;
            const uint32_t rem = total > seen ? total - seen : 0u;
            // a dynamic part of at most a tile per CTA goes out a tile per claim
            const uint32_t lo = a.n_plan_groups && total - W <= P ? 1u : min(a.min_chunk, CH);
            sz = max(lo, min(CH, (rem + 2 * P - 1) / (2 * P)));
        } else if (W < P * a.min_chunk) {
            // small static part (short contexts, small batches): while the
            // dynamic part is being planned, no ticket past the reserved tiles
            // (a CTA must not sit on tiles it cannot fetch while the others,
            // idle, could take them once they are published)
            uint32_t tk = 0;
            if (lane == 0) tk = ld_acquire_u32(&a.ctr->tickets);
            tk = __shfl_sync(0xFFFFFFFFu, tk, 0);
            const uint32_t pos = pre + tk;
            if (pos >= known) return false;
            // static tiles in chunks; reserved dynamic tiles one at a time
            // until the stream length is final (they are spread over the
            // CTAs as the contexts' plans arrive)
            sz = pos < W ? min(CH, W - pos) : 1u;
        }
        if (lane == 0) cl_ret = atomicAdd(&a.ctr->tickets, sz);
        cl_size = sz;
        cl_pend = true;
        return true;
    };
    bool first = true;
    if (a.dtrace && lane == 0) a.dtrace[16 * blockIdx.x + 12] = gtime();
    uint32_t pc0 = 0, pc1 = 0;  // the current chunk's remaining tiles
    bool pend = false, feeding = true;
    // unit slots 0/1 in registers (selects, no local memory)
    uint32_t u_cnt0 = 0, u_cnt1 = 0, u_base0 = 0, u_base1 = 0;
    bool u_last0 = false, u_last1 = false;
    uint32_t u_ph = 0;  // phase bit per unit slot
    // next unit of records into `slot`: false when none can be fetched now
    // (planner behind, or end of stream: feeding = false)
    auto fetch_unit = [&](int slot) -> bool {
        if (!feeding) return false;
        if (!pend) {
            uint32_t b0 = 0, b1 = 0;
            if (first && blockIdx.x * CS < pre) {
                b0 = blockIdx.x * CS;
                b1 = min(pre, b0 + CS);
            } else {
                if (!cl_pend) {
                    refresh();
                    if (!claim()) return false;  // planner behind: poll
                }
                b0 = pre + __shfl_sync(0xFFFFFFFFu, cl_ret, 0);
                b1 = b0 + cl_size;
                refresh();
                if (total != 0xFFFFFFFFu) {
                    if (b0 >= total) {
                        feeding = false;
                        return false;
                    }
                    b1 = min(b1, total);
                } else if (b1 > known) {
                    return false;  // not reserved by the planner yet
                }
                if (b1 > W && !dyn_ready(b0, b1)) return false;
                hint = b1;
                cl_pend = false;
            }
            first = false;
            // acquired generic-proxy data (records, gathered rows) is read by
            // the bulk and tensor copies (async proxy)
            if (b1 > W) asm volatile("fence.proxy.async.global;" ::: "memory");
            pc0 = b0;
            pc1 = b1;
            pend = true;
        }
        // a unit stays in one record array (static | dynamic)
        const uint32_t n = min(min(pc1 - pc0, (uint32_t)kUnit), pc0 < W ? W - pc0 : 0xFFFFFFFFu);
        if (lane == 0) {
            if (a.dtrace && a.dtrace[16 * blockIdx.x + 13] == 0) a.dtrace[16 * blockIdx.x + 13] = gtime();
            const TileRec* src = pc0 < W ? a.st_tiles + pc0 : a.dyn_tiles + (pc0 - W);
            mbar_arrive_expect_tx(&s.urec_bar[slot], n * (uint32_t)sizeof(TileRec));
            bulk_g2s(&s.urec[slot][0], src, n * (uint32_t)sizeof(TileRec), &s.urec_bar[slot]);
        }
        __syncwarp();
        if (slot) {
            u_cnt1 = n;
            u_base1 = pc0;
            u_last1 = pc0 + n == pc1;
        } else {
            u_cnt0 = n;
            u_base0 = pc0;
            u_last0 = pc0 + n == pc1;
        }
        pc0 += n;
        if (pc0 == pc1) pend = false;
        return true;
    };
    uint32_t stage = 0, phase = 0;
    bool run_first = true;
    uint32_t run_tiles = 0;
    unsigned long long p_wait = 0, p_sleep = 0;
    const unsigned long long p_t0 = clock64();
    uint32_t p_tiles = 0;
    auto pstamp = [&](int k) {
        if (a.dtiles && lane == 0 && p_tiles < (uint32_t)kTraceTiles)
            a.dtiles[((size_t)blockIdx.x * kTraceTiles + p_tiles) * 8 + k] = gtime();
    };
    int cur = 0;
    while (!fetch_unit(cur) && feeding) {  // the first unit (the planner may be behind)
        const unsigned long long ts = clock64();
        __nanosleep(a.poll_ns);
        p_sleep += clock64() - ts;
    }
    while (cur ? u_cnt1 : u_cnt0) {
        const int nx = cur ^ 1;
        // the next unit's records are fetched (and the chunk after this
        // one claimed) while this unit's last tiles are issued
        bool have_next = false;
        mbar_wait(&s.urec_bar[cur], (u_ph >> cur) & 1u);
        u_ph ^= 1u << cur;
        if (a.dtrace && lane == 0 && a.dtrace[16 * blockIdx.x + 10] == 0) a.dtrace[16 * blockIdx.x + 10] = gtime();
        const uint32_t ucnt = cur ? u_cnt1 : u_cnt0, ubase = cur ? u_base1 : u_base0;
        const bool ulast = cur ? u_last1 : u_last0;
        // dynamic records are re-armed for the next step once copied
        if (ubase >= W && (uint32_t)lane < ucnt) a.dyn_tiles[ubase - W + lane].ready = 0;
        for (uint32_t i = 0; i < ucnt; ++i) {
            pstamp(3);
            const TileRec& R = s.urec[cur][i];
            const uint4 hdr = *reinterpret_cast<const uint4*>(&R);
            const uint32_t np = hdr.x, qslot = hdr.y;
            const bool last_in_chunk = ulast && i + 1 == ucnt;
            const bool last_of_run = last_in_chunk || hdr.w != 0;
            uint32_t len = 0, srow = 0, gat = 0;
            uint64_t row = 0;
            if ((uint32_t)lane < np) {
                const uint4 v = *reinterpret_cast<const uint4*>(&R.p[lane]);
                len = v.x & ~kPieceGather;
                gat = v.x & kPieceGather;
                srow = v.y;
                row = ((uint64_t)v.w << 32) | v.z;
            }
            ++run_tiles;
            if (lane == 0) {
                const unsigned long long tw = clock64();
                if (a.inflight && a.inflight < (uint32_t)CF::NS && p_tiles >= a.inflight) {
                    // at most `inflight` tiles loading or unconsumed: wait for tile
                    // p_tiles - inflight (its stage's (j / NS)-th completion)
                    const uint32_t j = p_tiles - a.inflight;
                    mbar_wait(&s.empty[j % CF::NS], (j / CF::NS) & 1u);
                }
                mbar_wait(&s.empty[stage], phase ^ 1);
                p_wait += clock64() - tw;
                pstamp(7);
                s.valid[stage] = *reinterpret_cast<const uint4*>(&R.valid[0]);
                const uint32_t g = qslot / a.n_hchunks, hc = qslot - g * a.n_hchunks;
                const uint32_t nq = min((uint32_t)kHeadsPerSlot, a.G - hc * kHeadsPerSlot);
                const uint32_t flags = (run_first ? 1u : 0u) | (last_of_run ? 2u : 0u) | (nq << 8);
                const uint32_t qoff = (uint32_t)(((size_t)g * a.G + hc * kHeadsPerSlot) * D);
                s.meta[stage] = make_int4((int)qslot, (int)flags, (int)qoff, (int)run_tiles);
                const uint32_t bytes = a.debug_skip == 2 ? 0u : R.rows8 * (uint32_t)CF::RB * 2u;
                mbar_arrive_expect_tx(&s.full[stage], bytes);
            }
            __syncwarp();
            if (run_first) {
                // the run's query rows (<= 2 KB) into this SM's L1 ahead of the
                // consumers' fragment build (no shared-memory staging)
                const uint32_t g = qslot / a.n_hchunks, hc = qslot - g * a.n_hchunks;
                const uint32_t nq = min((uint32_t)kHeadsPerSlot, a.G - hc * kHeadsPerSlot);
                const float* qb = a.q + ((size_t)g * a.G + hc * kHeadsPerSlot) * D;
                if ((uint32_t)lane * 32u < nq * D)
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(qb + lane * 32) : "memory");
                if constexpr (SM::kPostQ) {  // the Q warp builds the run's B operand now
                    if (lane == 0) {
                        const uint32_t r = s.n_qreq++, qbi = r & 1;
                        mbar_wait(&s.q_req_empty[qbi], ((r >> 1) & 1) ^ 1);
                        s.qreq_off[qbi] = (uint32_t)(((size_t)g * a.G + hc * kHeadsPerSlot) * D);
                        s.qreq_nq[qbi] = nq;
                        mbar_arrive(&s.q_req[qbi]);
                    }
                }
            }
            if (len && a.debug_skip != 2) {
                // one request per piece for K and one for V: a box of r8/8 groups
                // when the rounded-up rows exist; else the piece's whole groups
                // plus a bounds-checked 8-row box (zero fill past the end)
                const uint32_t r8 = (len + 7) & ~7u;
                const CUtensorMap* mk = &maps.map[(gat ? 2 : 0) * kBoxSizes];
                const CUtensorMap* mv = mk + kBoxSizes;
                const uint64_t lim = gat ? maps.grows : maps.rows;
                const uint32_t off = (srow >> 3) * 8 * CF::RB;
                if (row + r8 <= lim) {
                    tma4d(&s.K[stage][off], mk + (r8 / 8 - 1), (int)row, &s.full[stage], pol);
                    tma4d(&s.V[stage][off], mv + (r8 / 8 - 1), (int)row, &s.full[stage], pol);
                } else {
                    const uint32_t full = len & ~7u;
                    if (full) {
                        tma4d(&s.K[stage][off], mk + (full / 8 - 1), (int)row, &s.full[stage], pol);
                        tma4d(&s.V[stage][off], mv + (full / 8 - 1), (int)row, &s.full[stage], pol);
                    }
                    if (r8 > full) {
                        const uint32_t off2 = ((srow + full) >> 3) * 8 * CF::RB;
                        tma4d(&s.K[stage][off2], mk, (int)(row + full), &s.full[stage], pol);
                        tma4d(&s.V[stage][off2], mv, (int)(row + full), &s.full[stage], pol);
                    }
                }
            }
            __syncwarp();
            if (a.dtrace && lane == 0 && a.dtrace[16 * blockIdx.x + 11] == 0) a.dtrace[16 * blockIdx.x + 11] = gtime();
            if (a.dtiles && lane == 0 && p_tiles < (uint32_t)kTraceTiles)
                a.dtiles[((size_t)blockIdx.x * kTraceTiles + p_tiles) * 8] =
                        (gtime() & ~63ull) | np | (last_in_chunk ? 32u : 0u);  // stamp | pieces | chunk end
            ++p_tiles;
            if (++stage == CF::NS) {
                stage = 0;
                phase ^= 1;
            }
            run_first = last_of_run;
            if (last_of_run) run_tiles = 0;
            __syncwarp();
            if (!have_next && feeding) {
                const uint32_t left = ucnt - 1 - i;  // tiles of this unit still to issue
                // (pend: the chunk has units after this one -- no claim yet)
                if (!pend && !cl_pend && left <= a.claim_lead) {
                    refresh();
                    claim();
                }
                if (left <= a.fetch_lead) have_next = fetch_unit(nx);
            }
        }
        if (cur) u_cnt1 = 0;
        else u_cnt0 = 0;
        if (!have_next) {  // fetch now (poll while the planner is behind)
            while (!fetch_unit(nx) && feeding) {
                const unsigned long long ts = clock64();
                __nanosleep(a.poll_ns);
                p_sleep += clock64() - ts;
            }
        }
        cur = nx;
    }
    if (lane == 0) {
        if (a.dtrace) {
            a.dtrace[16 * blockIdx.x + 4] = p_wait;
            a.dtrace[16 * blockIdx.x + 5] = clock64() - p_t0;
            a.dtrace[16 * blockIdx.x + 14] = p_sleep;
        }
        mbar_wait(&s.empty[stage], phase ^ 1);
        if constexpr (SM::kPostQ) {  // stop the Q warp
            const uint32_t r = s.n_qreq++, qbi = r & 1;
            mbar_wait(&s.q_req_empty[qbi], ((r >> 1) & 1) ^ 1);
            s.qreq_nq[qbi] = 0xFFu;
            mbar_arrive(&s.q_req[qbi]);
        }
        s.meta[stage] = make_int4(-1, 0, 0, 0);
        mbar_arrive(&s.full[stage]);
        // the last CTA out re-arms the step counters (every reader is done)
        if (atomicAdd(&a.ctr->exited, 1u) == gridDim.x - 1) {
            a.ctr->tickets = 0;
            a.ctr->dynres = 0;
            a.ctr->published = 0;
            a.ctr->exited = 0;
            __threadfence();
        }
    }
}

template <int D>
__global__ void __maxnreg__(144)
        decode_kernel(const __grid_constant__ DecodeArgs a, const __grid_constant__ DecodeMaps maps) {
    using CF = DecodeCfg<D>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    auto& s = *reinterpret_cast<DecodeSmem<D>*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    auto gtime = []() {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        return t;
    };
    if (a.dtrace && threadIdx.x == 0) {
        a.dtrace[16 * blockIdx.x] = gtime();
        a.dtrace[16 * blockIdx.x + 10] = 0;
        a.dtrace[16 * blockIdx.x + 11] = 0;
        a.dtrace[16 * blockIdx.x + 13] = 0;
    }
    if (threadIdx.x == 0) tl_mark(a.tl, 2, true);
    if (threadIdx.x == 0) {
        for (int i = 0; i < CF::NS; ++i) {
            mbar_init(&s.full[i], 1);
            mbar_init(&s.empty[i], kComputeWarps);
        }
        mbar_init(&s.st_full, kComputeWarps);
        mbar_init(&s.st_empty, 1);
        for (int i = 0; i < 2; ++i) mbar_init(&s.urec_bar[i], 1);
        fence_mbar_init();
    }
    // (gap rows of a tile hold stale shared memory: their V fragments are
    // masked to zero before the PV MMA, their scores to -inf)
    __syncthreads();
    // No grid wait: static tiles are ready now, dynamic tiles are published
    // by the (resident) planner through ready flags.  The combine grid may
    // launch once every decode CTA is resident.
    pdl_trigger();
    if (a.wait_plan) pdl_wait();  // routing runs on an idle memory system first

    if (warp == kComputeWarps + 1) {
        // ------------------------------------------------ merge warp
        // LSE-merges the 8 consumer warps' states of a finished run into the
        // run's partial (Alg. 2, attention.cpp:102-128), publishes it at gpu
        // scope and counts its tiles for the combine -- off the consumers' path.
        constexpr int NOUT = kHeadsPerSlot * D;
        constexpr int PER = NOUT / 32;
        uint32_t ph = 0;
        for (;;) {
            mbar_wait(&s.st_full, ph);
            ph ^= 1;
            const uint32_t slot = s.st_slot, tiles = s.st_tiles;
            if (slot == 0xFFFFFFFFu) break;
            // the run's partial slot (reserved here, off the consumers' path;
            // before its tiles are counted, so a complete count implies every
            // run is reserved)
            unsigned long long run_raw = 0;
            if (lane == 0) run_raw = atomicAdd(&a.rd[slot], 1ull << 32);
            // lane = (warp w, head h): per-head max and scale of every warp state
            const int w = lane >> 2, h = lane & 3;
            const float mw = s.redm[w][h];
            float M = mw;
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) M = fmaxf(M, __shfl_xor_sync(0xFFFFFFFFu, M, o));
            const float sc = M == -INFINITY ? 0.f : fast_exp2(mw - M);
            float Lp = s.redl[w][h] * sc;
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) Lp += __shfl_xor_sync(0xFFFFFFFFu, Lp, o);
            float res[PER];
#pragma unroll
            for (int e0 = 0; e0 < PER; ++e0) {
                const int e = lane + 32 * e0, hh = e / D, d = e % D;
                float O = 0.f;
#pragma unroll
                for (int ww = 0; ww < kComputeWarps; ++ww)
                    O = fmaf(s.redO[ww][hh][d], __shfl_sync(0xFFFFFFFFu, sc, ww * 4 + hh), O);
                res[e0] = O;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.st_empty);  // state buffer free
            const uint32_t run = __shfl_sync(0xFFFFFFFFu, (uint32_t)(run_raw >> 32), 0);
            const size_t pidx = (size_t)slot * a.run_cap + run;
            float* pO = a.part_O + pidx * NOUT;
#pragma unroll
            for (int e0 = 0; e0 < PER; ++e0) pO[lane + 32 * e0] = res[e0];
            if (lane < 4) {
                a.part_ml[pidx * 8 + lane] = M;  // lanes 0-3: w = 0, h = lane
                a.part_ml[pidx * 8 + 4 + lane] = Lp;
            }
            // the release store by lane 0 is cumulative over the partial (the
            // warp barrier orders the other lanes' writes before it)
            __syncwarp();
            if (lane == 0) {
                st_release_u32(a.part_flag + pidx, 1u);  // the combine folds it in now
                // tiles published (low word), a release too: once the combine
                // reads every tile counted, every partial is visible
                red_release_add_u64(&a.rd[slot], (unsigned long long)tiles);
                tl_mark(a.tl, 4, false);  // last run published
            }
        }
        return;
    }

    if (warp == kComputeWarps) {
        decode_producer<D>(a, maps, s, lane);
        return;
    }

    // ---------------------------------------------------- consumers
    const int gid = lane >> 2, tig = lane & 3;
    const bool upper = lane >= 16;  // rows g+4: q2 / p2
    const int hq = gid & 3;         // head of this lane's score rows
    const int row0 = warp * 16;     // this warp's 16 rows of the tile
    const int mtx = lane >> 3, r8 = lane & 7;

    // A fragments of [q1; q2; q3; 0] live in s.qfrag for the whole run (the next
    // run's build starts only once every consumer warp reached it)
    const uint32_t qf_off = upper ? 64u + 2u * (uint32_t)(lane - 16) : 4u * (uint32_t)lane;
    float o[CF::NT][4];
    float m_run = -INFINITY, l_run = 0.f;
    uint32_t st_ph = 0;
    // named barrier of the 8 consumer warps (run starts share one fragment build)
    auto consumer_bar = []() { asm volatile("bar.sync 1, %0;" ::"n"(kComputeWarps * 32) : "memory"); };

    uint32_t stage = 0, phase = 0;
    uint32_t n_tiles_done = 0;
    unsigned long long c_wait = 0;
    for (;;) {
        if (a.dtrace && threadIdx.x == 0) {
            const unsigned long long t0 = clock64();
            mbar_wait(&s.full[stage], phase);
            c_wait += clock64() - t0;
        } else {
            mbar_wait(&s.full[stage], phase);
        }
        const int4 mt = s.meta[stage];
        if (a.dtiles && threadIdx.x == 0 && n_tiles_done < (uint32_t)kTraceTiles)
            a.dtiles[((size_t)blockIdx.x * kTraceTiles + n_tiles_done) * 8 + 1] = gtime();
        if (a.dtrace && threadIdx.x == 0) {
            if (n_tiles_done == 0) a.dtrace[16 * blockIdx.x + 1] = gtime();
            if (mt.x < 0) {
                a.dtrace[16 * blockIdx.x + 2] = gtime();
                a.dtrace[16 * blockIdx.x + 3] = n_tiles_done;
                a.dtrace[16 * blockIdx.x + 6] = c_wait;
            }
        }
        ++n_tiles_done;
        if (mt.x < 0) {
            if (threadIdx.x == 0) tl_mark(a.tl, 2, false);
            // stop the merge warp once it has drained the last run
            mbar_wait(&s.st_empty, st_ph ^ 1);
            if (threadIdx.x == 0) s.st_slot = 0xFFFFFFFFu;
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.st_full);
            break;
        }
        const uint32_t flags = (uint32_t)mt.y;
        if (flags & 1u) {
            // A operand [q1; q2; q3; 0]: 3-term bf16 split of the f32 queries
            // (~fp32-exact).  Rows g (lanes < 16: q1, else q2) and g + 8 (q3 / 0).
            // Warp w converts k-steps w, w + 8, ... for every lane position into
            // qfrag (each element converted once per CTA, not once per warp);
            // the consumer warps then load their fragments.
            const uint32_t nq = (flags >> 8) & 7u;
            const float* qh = a.q + (uint32_t)mt.z + hq * D;  // L1 (prefetched by the producer)
            const bool live = (uint32_t)hq < nq;
            consumer_bar();  // every warp has loaded the previous run's fragments
            for (int k = warp; k < CF::KSTEPS; k += kComputeWarps) {
                const float2 lo2 = live ? __ldg(reinterpret_cast<const float2*>(qh + 16 * k + 2 * tig)) : make_float2(0.f, 0.f);
                const float2 hi2 = live ? __ldg(reinterpret_cast<const float2*>(qh + 16 * k + 8 + 2 * tig)) : make_float2(0.f, 0.f);
                // x = t1 + t2 + t3 (bf16 terms, hardware RNE conversions)
                const uint32_t a1 = bf16x2_rn(lo2.x, lo2.y), b1 = bf16x2_rn(hi2.x, hi2.y);
                const float ra0 = lo2.x - bf16lo(a1), ra1 = lo2.y - bf16hi(a1);
                const float rb0 = hi2.x - bf16lo(b1), rb1 = hi2.y - bf16hi(b1);
                const uint32_t a2 = bf16x2_rn(ra0, ra1), b2 = bf16x2_rn(rb0, rb1);
                if (!upper)
                    *reinterpret_cast<uint4*>(&s.qfrag[k * 96 + 4 * lane]) =
                            make_uint4(a1, bf16x2_rn(ra0 - bf16lo(a2), ra1 - bf16hi(a2)), b1,
                                       bf16x2_rn(rb0 - bf16lo(b2), rb1 - bf16hi(b2)));
                else
                    *reinterpret_cast<uint2*>(&s.qfrag[k * 96 + 64 + 2 * (lane - 16)]) = make_uint2(a2, b2);
            }
            consumer_bar();  // fragments complete (read from qfrag by every tile of the run)
#pragma unroll
            for (int n = 0; n < CF::NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
            m_run = -INFINITY;
            l_run = 0.f;
        }
        if (a.dtiles && threadIdx.x == 0 && n_tiles_done - 1 < (uint32_t)kTraceTiles)
            a.dtiles[((size_t)blockIdx.x * kTraceTiles + n_tiles_done - 1) * 8 + 4] = gtime();
        const uint32_t vbits = ((&s.valid[stage].x)[warp >> 1] >> ((warp & 1) * 16)) & 0xFFFFu;
        if (vbits && a.debug_skip != 1) {
            // ---- S = [q1; q2; q3] K^T for this warp's 16 rows
            const uint32_t kbase = smem_u32(&s.K[stage][0]);
            float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f};
            const uint32_t krow = row0 + (mtx >> 1) * 8 + r8;
#pragma unroll
            for (int k = 0; k < CF::KSTEPS; ++k) {
                const uint32_t chunk = 2 * k + (mtx & 1);  // 16-byte chunk within the row
                uint32_t b0, b1, b2, b3;
                ldsm_x4(kbase + toff<D>(krow, chunk), b0, b1, b2, b3);
                uint32_t qa0, qa1, qa2, qa3;
                if (!upper) {
                    const uint4 v = *reinterpret_cast<const uint4*>(&s.qfrag[k * 96 + qf_off]);
                    qa0 = v.x;
                    qa1 = v.y;
                    qa2 = v.z;
                    qa3 = v.w;
                } else {
                    const uint2 v = *reinterpret_cast<const uint2*>(&s.qfrag[k * 96 + qf_off]);
                    qa0 = v.x;
                    qa1 = 0u;
                    qa2 = v.y;
                    qa3 = 0u;
                }
                mma16816(c0, qa0, qa1, qa2, qa3, b0, b1);
                mma16816(c1, qa0, qa1, qa2, qa3, b2, b3);
            }
            // scores for head hq; keys c0 -> row0 + 2*tig + {0,1}, c1 -> row0 + 8 + 2*tig + {0,1}
            // rows g + g+8 here, g+4 (+ zero row g+12) on lane ^ 16
            float sc[4] = {c0[0] + c0[2], c0[1] + c0[3], c1[0] + c1[2], c1[1] + c1[3]};
#pragma unroll
            for (int i = 0; i < 4; ++i) sc[i] = (sc[i] + __shfl_xor_sync(0xFFFFFFFFu, sc[i], 16)) * a.qscale;
            const uint32_t kb = 2 * tig;
            if (!((vbits >> kb) & 1)) sc[0] = -INFINITY;
            if (!((vbits >> (kb + 1)) & 1)) sc[1] = -INFINITY;
            if (!((vbits >> (kb + 8)) & 1)) sc[2] = -INFINITY;
            if (!((vbits >> (kb + 9)) & 1)) sc[3] = -INFINITY;
            float mx = fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3]));
            mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, 2));
            // lazy rescale: keep the running max unless this tile exceeds it by 2^8
            const bool grow = mx > m_run + 8.f;
            if (__any_sync(0xFFFFFFFFu, grow)) {
                const float mnew = grow ? mx : m_run;
                const float alpha = fast_exp2(m_run - mnew);
                m_run = mnew;
                l_run *= alpha;
#pragma unroll
                for (int n = 0; n < CF::NT; ++n) {
                    o[n][0] *= alpha;
                    o[n][1] *= alpha;
                    o[n][2] *= alpha;
                    o[n][3] *= alpha;
                }
            }
            float p[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) p[i] = fast_exp2(sc[i] - m_run);  // -inf -> 0
            if (!upper) l_run += (p[0] + p[1]) + (p[2] + p[3]);
            // 3-term bf16 split: lanes < 16 carry p1 (rows g) and p3 (rows g+8),
            // lanes >= 16 carry p2 (rows g+4) and zeros (rows g+12)
            uint32_t pa0, pa1, pa2, pa3;
            {
                const uint32_t h01 = bf16x2_rn(p[0], p[1]), h23 = bf16x2_rn(p[2], p[3]);
                const float r0 = p[0] - bf16lo(h01), r1 = p[1] - bf16hi(h01);
                const float r2 = p[2] - bf16lo(h23), r3 = p[3] - bf16hi(h23);
                const uint32_t m01 = bf16x2_rn(r0, r1), m23 = bf16x2_rn(r2, r3);
                if (!upper) {
                    pa0 = h01;
                    pa2 = h23;
                    pa1 = bf16x2_rn(r0 - bf16lo(m01), r1 - bf16hi(m01));
                    pa3 = bf16x2_rn(r2 - bf16lo(m23), r3 - bf16hi(m23));
                } else {
                    pa0 = m01;
                    pa2 = m23;
                    pa1 = 0u;
                    pa3 = 0u;
                }
            }
            if (a.dtiles && threadIdx.x == 0 && n_tiles_done - 1 < (uint32_t)kTraceTiles)
                a.dtiles[((size_t)blockIdx.x * kTraceTiles + n_tiles_done - 1) * 8 + 5] = gtime();
            // ---- O += P V   (B = V rows via ldmatrix.trans)
            const uint32_t vbase = smem_u32(&s.V[stage][0]);
            const uint32_t vrow = row0 + (mtx & 1) * 8 + r8;
            // this lane's B elements are rows 2tig, 2tig+1 (b0, b2) and 2tig+8,
            // 2tig+9 (b1, b3): zero the invalid ones (stale smem may be NaN)
            const uint32_t m_lo = (((vbits >> kb) & 1u) ? 0x0000FFFFu : 0u) | (((vbits >> (kb + 1)) & 1u) ? 0xFFFF0000u : 0u);
            const uint32_t m_hi = (((vbits >> (kb + 8)) & 1u) ? 0x0000FFFFu : 0u) | (((vbits >> (kb + 9)) & 1u) ? 0xFFFF0000u : 0u);
#pragma unroll
            for (int j = 0; j < CF::NT / 2; ++j) {
                const uint32_t chunk = 2 * j + (mtx >> 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(vbase + toff<D>(vrow, chunk), b0, b1, b2, b3);
                b0 &= m_lo;
                b1 &= m_hi;
                b2 &= m_lo;
                b3 &= m_hi;
                mma16816(o[2 * j], pa0, pa1, pa2, pa3, b0, b1);
                mma16816(o[2 * j + 1], pa0, pa1, pa2, pa3, b2, b3);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&s.empty[stage]);
        if (a.dtiles && threadIdx.x == 0 && n_tiles_done - 1 < (uint32_t)kTraceTiles)
            a.dtiles[((size_t)blockIdx.x * kTraceTiles + n_tiles_done - 1) * 8 + 2] = gtime();

        if (flags & 2u) {
            // ---- run done: deposit this warp's (m, l, O) state for the merge warp
            const uint32_t slot = (uint32_t)mt.x;
            float lw = l_run;
            lw += __shfl_xor_sync(0xFFFFFFFFu, lw, 1);
            lw += __shfl_xor_sync(0xFFFFFFFFu, lw, 2);
            float xo[CF::NT][2];
#pragma unroll
            for (int n = 0; n < CF::NT; ++n) {
                // lanes < 16 hold p1 (c[0..1]) + p3 (c[2..3]); lanes >= 16 hold p2
                float x0 = o[n][0] + (upper ? 0.f : o[n][2]);
                float x1 = o[n][1] + (upper ? 0.f : o[n][3]);
                xo[n][0] = x0 + __shfl_xor_sync(0xFFFFFFFFu, x0, 16);
                xo[n][1] = x1 + __shfl_xor_sync(0xFFFFFFFFu, x1, 16);
            }
            mbar_wait(&s.st_empty, st_ph ^ 1);  // previous run's states consumed
            if (!upper) {
#pragma unroll
                for (int n = 0; n < CF::NT; ++n)
                    *reinterpret_cast<float2*>(&s.redO[warp][hq][n * 8 + 2 * tig]) = make_float2(xo[n][0], xo[n][1]);
                if (tig == 0) {
                    s.redm[warp][hq] = m_run;
                    s.redl[warp][hq] = lw;
                }
            }
            if (threadIdx.x == 0) {
                s.st_slot = slot;
                s.st_tiles = (uint32_t)mt.w;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.st_full);
            st_ph ^= 1;
        }
        if (++stage == CF::NS) {
            stage = 0;
            phase ^= 1;
        }
    }
}

// ============================================================ tcgen05 decode (d = 128)
// Same work stream, producer and partials as decode_kernel; the consumers
// run on the 5th-gen tensor cores.  Per tile (128 keys):
//   S^T [128 keys x 16] = K [128 x d] . Q^T      (A = K tile, K-major SW128;
//                                                 B = [q1;q2;q3] x 4 heads + 4
//                                                 zero rows, built once per run)
//   O^T [d x 16]       += V^T [d x 128] . P^T    (A = V tile read MN-major;
//                                                 B = [p1;p2;p3] x 4 heads)
// with fp32 accumulation in TMEM (S double-buffered, O double-buffered per
// run).  One thread issues the MMAs (QK of tile t before PV of tile t-1, so
// the tensor core works while the softmax warps handle tile t-1); four
// softmax warps own TMEM lane quarters: thread = key row of S (scores, tile
// max across the warps, lazy rescale of O in TMEM when a head's max grows
// by 2^8, 3-term bf16 split of the weights into P) and thread = dimension
// of O at a run's end (the run partial, same layout as decode_kernel's).
namespace dtc {
constexpr int NSW = 4;                 // softmax warps (TMEM lane quarters)
constexpr int PRODUCER = NSW;          // warp 4
constexpr int MMA = NSW + 1;           // warp 5
constexpr int QW = NSW + 2;            // warp 6: builds each run's Q operand
constexpr int THREADS = (NSW + 3) * 32;
constexpr uint32_t NQ = 16;            // B rows: 3 terms x 4 heads + 4 zero rows
constexpr uint32_t TMEM_COLS = 64;     // S[2] x 16 | O[2] x 16
constexpr uint32_t S_COL = 0, O_COL = 32;
}  // namespace dtc

template <int D>
struct DecodeTcSmem {
    using CF = DecodeCfg<D>;
    static constexpr bool kPostQ = true;  // the producer posts each run's query rows to the Q warp
    uint8_t K[CF::NS][CF::TILE_BYTES];
    uint8_t V[CF::NS][CF::TILE_BYTES];
    // B operands, [n-group][64-column half][8 rows][128 B] with the 128B swizzle
    // (the K/V tiles' layout): Qb[run parity] rows n = 4 * term + head over d,
    // Pb[tile parity] rows n over the tile's 128 keys
    uint8_t Qb[2][dtc::NQ * D * 2];
    uint8_t Pb[2][dtc::NQ * kTileRows * 2];
    uint64_t full[CF::NS];
    uint64_t empty[CF::NS];
    uint64_t s_full[2], s_empty[2], p_full[2], p_empty[2];
    uint64_t q_full[2], q_empty[2], o_full[2], o_empty[2];
    uint64_t q_req[2], q_req_empty[2];
    uint32_t qreq_off[2], qreq_nq[2], n_qreq;
    int4 meta[CF::NS];
    uint4 valid[CF::NS];
    alignas(16) TileRec urec[2][kUnit];
    uint64_t urec_bar[2];
    uint4 pvinfo[CF::NS];  // MMA thread: per stage (flags, O buffer, run) of the tile awaiting PV
    float red[2][dtc::NSW][4];
    float lred[dtc::NSW][4];
    uint32_t run_slot;
    uint32_t tmem_base;
};

__device__ __forceinline__ uint64_t umma_sdesc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;  // SWIZZLE_128B
    return d;
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_arrive(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
            "%12, %13, %14, %15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
              "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
            "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
            "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
            "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
            "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
            "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
            "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
            "r"(__float_as_uint(v[15]))
            : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// byte offset of element (row n, column c) of a 16-row B operand laid out as
// [n >> 3][c >> 6][n & 7][128 B], 16-byte chunks XOR-swizzled by (n & 7)
__device__ __forceinline__ uint32_t boff16(uint32_t n, uint32_t c, uint32_t cols) {
    return (n >> 3) * (cols * 16) + (c >> 6) * 1024 + (n & 7) * 128 + ((((c & 63) >> 3) ^ (n & 7)) << 4) +
           (c & 7) * 2;
}

template <int D>
__global__ void __launch_bounds__(dtc::THREADS, 1)
        decode_tc_kernel(const __grid_constant__ DecodeArgs a, const __grid_constant__ DecodeMaps maps) {
    static_assert(D == 128, "tcgen05 decode: d = 128 (O^T has d TMEM lanes)");
    using CF = DecodeCfg<D>;
    using namespace dtc;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    auto& s = *reinterpret_cast<DecodeTcSmem<D>*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto gtime = []() {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        return t;
    };
    if (a.dtrace && threadIdx.x == 0) {
        a.dtrace[16 * blockIdx.x] = gtime();
        a.dtrace[16 * blockIdx.x + 10] = 0;
        a.dtrace[16 * blockIdx.x + 11] = 0;
        a.dtrace[16 * blockIdx.x + 13] = 0;
    }
    if (threadIdx.x == 0) tl_mark(a.tl, 2, true);
    if (threadIdx.x == 0) {
        for (int i = 0; i < CF::NS; ++i) {
            mbar_init(&s.full[i], 1);
            mbar_init(&s.empty[i], 1);  // the PV MMAs' commit
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s.s_full[i], 1);
            mbar_init(&s.s_empty[i], NSW);
            mbar_init(&s.p_full[i], NSW);
            mbar_init(&s.p_empty[i], 1);
            mbar_init(&s.q_full[i], 1);
            mbar_init(&s.q_empty[i], 1);
            mbar_init(&s.o_full[i], 1);
            mbar_init(&s.o_empty[i], NSW);
            mbar_init(&s.q_req[i], 1);
            mbar_init(&s.q_req_empty[i], 1);
            mbar_init(&s.urec_bar[i], 1);
        }
        s.n_qreq = 0;
        fence_mbar_init();
    }
    if (warp < NSW) {
        // the MMAs read every row of a tile: gap rows must hold finite values,
        // so the ring starts zeroed (later it only ever holds loaded rows);
        // the B operands' padding rows stay zero
        uint4* z = reinterpret_cast<uint4*>(&s.K[0][0]);
        constexpr uint32_t NZ = (2u * CF::NS * CF::TILE_BYTES + sizeof(s.Qb) + sizeof(s.Pb)) / 16;
        for (uint32_t i = threadIdx.x; i < NZ; i += NSW * 32) z[i] = make_uint4(0u, 0u, 0u, 0u);
        fence_async_smem();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(&s.tmem_base)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem_base;
    pdl_trigger();
    if (a.wait_plan) pdl_wait();

    if (warp == PRODUCER) {
        decode_producer<D>(a, maps, s, lane);
    } else if (warp == QW) {
        // ------------------------------------------------ Q warp: each run's B
        // operand [q1; q2; q3] x 4 heads (3-term bf16 split of the f32 queries)
        for (uint32_t r = 0;; ++r) {
            const uint32_t qbi = r & 1;
            mbar_wait(&s.q_req[qbi], (r >> 1) & 1);
            const uint32_t qoff = s.qreq_off[qbi], nq = s.qreq_nq[qbi];
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.q_req_empty[qbi]);
            if (nq == 0xFFu) break;
            mbar_wait(&s.q_empty[qbi], ((r >> 1) & 1) ^ 1);  // run r-2's QK MMAs are done
            const float* qh = a.q + qoff;
            uint8_t* qbuf = &s.Qb[qbi][0];
#pragma unroll
            for (uint32_t h = 0; h < 4; ++h)
#pragma unroll
                for (uint32_t j = 0; j < (uint32_t)D / 32; ++j) {
                    const uint32_t d = j * 32 + lane;
                    const float x = h < nq ? __ldg(qh + h * D + d) : 0.f;
                    const uint16_t t1 = f32_to_bf16_rne(x);
                    const float r1 = x - __uint_as_float((uint32_t)t1 << 16);
                    const uint16_t t2 = f32_to_bf16_rne(r1);
                    const uint16_t t3 = f32_to_bf16_rne(r1 - __uint_as_float((uint32_t)t2 << 16));
                    *reinterpret_cast<uint16_t*>(qbuf + boff16(h, d, D)) = t1;
                    *reinterpret_cast<uint16_t*>(qbuf + boff16(4 + h, d, D)) = t2;
                    *reinterpret_cast<uint16_t*>(qbuf + boff16(8 + h, d, D)) = t3;
                }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.q_full[qbi]);
        }
    } else if (warp == MMA) {
        // ------------------------------------------------ MMA issuer (one thread)
        // Two streams, each issued as soon as its inputs are ready (polling,
        // no blocking wait on either): QK of tile t once its K/V landed, its
        // run's Q is built and S[t & 1] is free; PV of tile t once its P is
        // written.  PV right after P frees the K/V stage early (the stage
        // ring, not the tensor core, bounds the tiles in flight).
        if (lane == 0) {
            constexpr uint32_t idesc_qk = (1u << 4) | (1u << 7) | (1u << 10) | ((NQ >> 3) << 17) |
                                          ((uint32_t)(kTileRows >> 4) << 24);
            constexpr uint32_t idesc_pv = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((NQ >> 3) << 17) |
                                          ((uint32_t)(D >> 4) << 24);
            uint32_t q_stage = 0, q_phase = 0, nqk = 0, npv = 0, ri = 0, qb = 0, ob = 0;
            bool ended = false;
            for (;;) {
                if (npv < nqk) {
                    const uint32_t pst = npv % CF::NS, pb = npv & 1;
                    const uint4 inf = s.pvinfo[pst];
                    bool ok = mbar_test_wait(&s.p_full[pb], (npv >> 1) & 1);
                    // a run's first PV overwrites O[ob]: run ri - 2's epilogue read it
                    if (ok && (inf.x & 1u) && inf.z >= 2) ok = mbar_test_wait(&s.o_empty[inf.y], ((inf.z >> 1) & 1) ^ 1);
                    if (ok) {
                        tc_fence_after();
                        if (a.dtiles && npv < (uint32_t)kTraceTiles)
                            a.dtiles[((size_t)blockIdx.x * kTraceTiles + npv) * 8 + 4] = gtime();
                        const uint32_t vb = smem_u32(&s.V[pst][0]), pbase = smem_u32(&s.Pb[pb][0]);
                        const uint32_t dcol = tmem + O_COL + inf.y * NQ;
#pragma unroll
                        for (uint32_t kk = 0; kk < kTileRows / 16; ++kk)
                            umma_f16(dcol, umma_sdesc_sw128(vb + kk * 4096, 1024, 2048),
                                     umma_sdesc_sw128(pbase + (kk >> 2) * 1024 + (kk & 3) * 32, 16, 2048),
                                     idesc_pv, ((inf.x & 1u) && kk == 0) ? 0u : 1u);
                        umma_arrive(&s.empty[pst]);  // K and V of the tile read
                        umma_arrive(&s.p_empty[pb]);
                        if (inf.x & 2u) umma_arrive(&s.o_full[inf.y]);
                        ++npv;
                    }
                }
                if (!ended && mbar_test_wait(&s.full[q_stage], q_phase)) {
                    const int4 mt = s.meta[q_stage];
                    if (mt.x < 0) {
                        ended = true;
                    } else {
                        const uint32_t flags = (uint32_t)mt.y;
                        bool ok = true;
                        if (flags & 1u) ok = mbar_test_wait(&s.q_full[ri & 1], (ri >> 1) & 1);
                        if (ok) ok = mbar_test_wait(&s.s_empty[nqk & 1], ((nqk >> 1) & 1) ^ 1);
                        if (ok) {
                            uint32_t this_ri = ri - 1;
                            if (flags & 1u) {
                                qb = ri & 1;
                                ob = ri & 1;
                                this_ri = ri++;
                            }
                            tc_fence_after();
                            const uint32_t sb = nqk & 1;
                            const uint32_t kb = smem_u32(&s.K[q_stage][0]), qbase = smem_u32(&s.Qb[qb][0]);
                            if (a.dtiles && nqk < (uint32_t)kTraceTiles)
                                a.dtiles[((size_t)blockIdx.x * kTraceTiles + nqk) * 8 + 3] = gtime();
#pragma unroll
                            for (uint32_t kk = 0; kk < (uint32_t)CF::KSTEPS; ++kk) {
                                const uint32_t off = (kk >> 2) * 1024 + (kk & 3) * 32;
                                umma_f16(tmem + S_COL + sb * NQ, umma_sdesc_sw128(kb + off, 16, 2048),
                                         umma_sdesc_sw128(qbase + off, 16, 2048), idesc_qk, kk ? 1u : 0u);
                            }
                            umma_arrive(&s.s_full[sb]);
                            if (flags & 2u) umma_arrive(&s.q_empty[qb]);
                            s.pvinfo[q_stage] = make_uint4(flags, ob, this_ri, 0u);
                            ++nqk;
                            if (++q_stage == CF::NS) {
                                q_stage = 0;
                                q_phase ^= 1;
                            }
                        }
                    }
                }
                if (ended && npv == nqk) break;
            }
        }
    } else {
        // ------------------------------------------------ softmax warps
        const uint32_t tid = threadIdx.x;  // key row of S / dimension of O
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
        auto named_bar = []() { asm volatile("bar.sync 1, %0;" ::"n"(NSW * 32) : "memory"); };
        uint32_t stage = 0, phase = 0, t = 0, ri = 0, ob = 0, cur_run = 0;
        float m_run[4], l_part[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            m_run[h] = -INFINITY;
            l_part[h] = 0.f;
        }
        unsigned long long run_raw = 0;
        // a finished run's partial is written after the next tile's weights
        // (its last PV runs meanwhile)
        bool epi = false;
        uint32_t e_ob = 0, e_slot = 0, e_tiles = 0, e_run = 0;
        unsigned long long e_raw = 0;
        float e_m[4], e_l[4];
        auto epilogue = [&]() {
            mbar_wait(&s.o_full[e_ob], (e_run >> 1) & 1);
            tc_fence_after();
            float ov[16];
            tmem_ld16(tmem + lane_base + O_COL + e_ob * NQ, ov);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.o_empty[e_ob]);
#pragma unroll
            for (int o = 16; o; o >>= 1)
#pragma unroll
                for (int h = 0; h < 4; ++h) e_l[h] += __shfl_xor_sync(0xFFFFFFFFu, e_l[h], o);
            if (lane < 4) s.lred[warp][lane] = lane == 0 ? e_l[0] : lane == 1 ? e_l[1] : lane == 2 ? e_l[2] : e_l[3];
            if (tid == 0) s.run_slot = (uint32_t)(e_raw >> 32);
            named_bar();
            const uint32_t run = s.run_slot;
            const size_t pidx = (size_t)e_slot * a.run_cap + run;
            float* pO = a.part_O + pidx * (kHeadsPerSlot * D);
#pragma unroll
            for (int h = 0; h < 4; ++h) pO[h * D + tid] = (ov[h] + ov[8 + h]) + ov[4 + h];
            if (tid < 4) {
                a.part_ml[pidx * 8 + tid] = tid == 0 ? e_m[0] : tid == 1 ? e_m[1] : tid == 2 ? e_m[2] : e_m[3];
                a.part_ml[pidx * 8 + 4 + tid] = (s.lred[0][tid] + s.lred[1][tid]) + (s.lred[2][tid] + s.lred[3][tid]);
            }
            named_bar();
            if (tid == 0) {
                st_release_u32(a.part_flag + pidx, 1u);  // the combine folds it in now
                red_release_add_u64(&a.rd[e_slot], (unsigned long long)e_tiles);
                tl_mark(a.tl, 4, false);
            }
            epi = false;
        };
        for (;;) {
            mbar_wait(&s.full[stage], phase);
            const int4 mt = s.meta[stage];
            if (a.dtrace && tid == 0 && t == 0) a.dtrace[16 * blockIdx.x + 1] = gtime();
            if (mt.x < 0) {
                if (epi) epilogue();
                if (a.dtrace && tid == 0) {
                    a.dtrace[16 * blockIdx.x + 2] = gtime();
                    a.dtrace[16 * blockIdx.x + 3] = t;
                }
                if (tid == 0) tl_mark(a.tl, 2, false);
                break;
            }
            const uint32_t flags = (uint32_t)mt.y, slot = (uint32_t)mt.x;
            const uint32_t vbits = (&s.valid[stage].x)[tid >> 5];
            if (flags & 1u) {
                // run start: reserve the run's partial slot (the atomic travels
                // during the run)
                if (tid == 0) run_raw = atomicAdd(&a.rd[slot], 1ull << 32);
                ob = ri & 1;
                cur_run = ri;
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    m_run[h] = -INFINITY;
                    l_part[h] = 0.f;
                }
                ++ri;
            }
            // ---- scores of this thread's key
            const uint32_t sb = t & 1;
            mbar_wait(&s.s_full[sb], (t >> 1) & 1);
            if (a.dtiles && tid == 0 && t < (uint32_t)kTraceTiles)
                a.dtiles[((size_t)blockIdx.x * kTraceTiles + t) * 8 + 5] = gtime();
            tc_fence_after();
            float sv[16];
            tmem_ld16(tmem + lane_base + S_COL + sb * NQ, sv);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.s_empty[sb]);
            if (a.dtiles && tid == 0 && t < (uint32_t)kTraceTiles)
                a.dtiles[((size_t)blockIdx.x * kTraceTiles + t) * 8 + 1] = gtime();
            const bool valid = (vbits >> lane) & 1u;
            float sc[4], mx[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                sc[h] = valid ? ((sv[h] + sv[8 + h]) + sv[4 + h]) * a.qscale : -INFINITY;
                mx[h] = sc[h];
            }
#pragma unroll
            for (int o = 16; o; o >>= 1)
#pragma unroll
                for (int h = 0; h < 4; ++h) mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xFFFFFFFFu, mx[h], o));
            if (lane < 4) s.red[t & 1][warp][lane] = lane == 0 ? mx[0] : lane == 1 ? mx[1] : lane == 2 ? mx[2] : mx[3];
            named_bar();
            if (a.dtiles && tid == 0 && t < (uint32_t)kTraceTiles)
                a.dtiles[((size_t)blockIdx.x * kTraceTiles + t) * 8 + 6] = gtime();
            bool grow = false;
            float M[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                M[h] = fmaxf(fmaxf(s.red[t & 1][0][h], s.red[t & 1][1][h]), fmaxf(s.red[t & 1][2][h], s.red[t & 1][3][h]));
                grow |= M[h] > m_run[h] + 8.f;
            }
            if (grow) {  // (uniform: every thread sees the same maxima)
                float alpha[4];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const bool g = M[h] > m_run[h] + 8.f;
                    alpha[h] = g ? fast_exp2(m_run[h] - M[h]) : 1.f;  // m_run = -inf -> 0
                    if (g) m_run[h] = M[h];
                    l_part[h] *= alpha[h];
                }
                if (!(flags & 1u)) {
                    // O holds this run's earlier tiles: wait for the last PV, rescale in TMEM
                    mbar_wait(&s.p_empty[(t - 1) & 1], ((t - 1) >> 1) & 1);
                    tc_fence_after();
                    float ov[16];
                    const uint32_t oaddr = tmem + lane_base + O_COL + ob * NQ;
                    tmem_ld16(oaddr, ov);
#pragma unroll
                    for (int i = 0; i < 12; ++i) ov[i] *= alpha[i & 3];
                    tmem_st16(oaddr, ov);
                    tc_fence_before();
                }
            }
            // ---- weights, 3-term split into P (row 4 * term + head, column = key)
            float p[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                p[h] = fast_exp2(sc[h] - (m_run[h] == -INFINITY ? 0.f : m_run[h]));  // -inf -> 0
                l_part[h] += p[h];
            }
            const uint32_t pb = t & 1;
            mbar_wait(&s.p_empty[pb], ((t >> 1) & 1) ^ 1);
            if (a.dtiles && tid == 0 && t < (uint32_t)kTraceTiles)
                a.dtiles[((size_t)blockIdx.x * kTraceTiles + t) * 8 + 7] = gtime();
            uint8_t* pbuf = &s.Pb[pb][0];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const uint16_t t1 = f32_to_bf16_rne(p[h]);
                const float r1 = p[h] - __uint_as_float((uint32_t)t1 << 16);
                const uint16_t t2 = f32_to_bf16_rne(r1);
                const uint16_t t3 = f32_to_bf16_rne(r1 - __uint_as_float((uint32_t)t2 << 16));
                *reinterpret_cast<uint16_t*>(pbuf + boff16(h, tid, kTileRows)) = t1;
                *reinterpret_cast<uint16_t*>(pbuf + boff16(4 + h, tid, kTileRows)) = t2;
                *reinterpret_cast<uint16_t*>(pbuf + boff16(8 + h, tid, kTileRows)) = t3;
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.p_full[pb]);
            if (a.dtiles && tid == 0 && t < (uint32_t)kTraceTiles)
                a.dtiles[((size_t)blockIdx.x * kTraceTiles + t) * 8 + 2] = gtime();
            if (epi) epilogue();  // the previous run's partial
            if (flags & 2u) {  // this run's partial after the next tile's weights
                epi = true;
                e_ob = ob;
                e_slot = slot;
                e_tiles = (uint32_t)mt.w;
                e_run = cur_run;
                e_raw = run_raw;
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    e_m[h] = m_run[h];
                    e_l[h] = l_part[h];
                }
            }
            ++t;
            if (++stage == CF::NS) {
                stage = 0;
                phase ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

// ============================================================ LSE combine (Alg. 2)
// One CTA per query slot: O = sum_r O_r 2^(m_r - M) / sum_r l_r 2^(m_r - M)
// over the slot's run partials (merge_into / pattn_finalize,
// attention.cpp:102-161; Alg. 2).  Launched (PDL) once every decode
// CTA is resident; its CTAs become resident as decode CTAs retire and combine
// a slot as soon as the slot's tiles are all published, so only the last
// slots' combines trail the decode.  A slot with no visited key gets zero
// rows (attention.cpp:147-152).
// D threads (one float4 of the slot's 4 x D outputs each): small enough to
// sit next to a decode CTA
template <int D>
__global__ void __maxnreg__(80) combine_kernel(CombineArgs a) {
    constexpr int NOUT = kHeadsPerSlot * D;
    constexpr int PER = 4;  // consecutive outputs per thread (one head)
    constexpr int U = 8;  // runs in flight
    const uint32_t qsi = blockIdx.x;
    __shared__ uint32_t s_nr, s_fin;
    const uint32_t e0 = threadIdx.x * PER, h = e0 / D;
    const uint32_t g = qsi / a.n_hchunks, hc = qsi % a.n_hchunks;
    const uint32_t head = hc * kHeadsPerSlot + h;
    float* out = a.out + ((size_t)g * a.G + head) * D + (e0 % D);
    const size_t base = (size_t)qsi * a.run_cap;
    if (threadIdx.x == 0) tl_mark(a.tl, 3, true);
    // Streaming fold: run partials are merged as the decode publishes them
    // (per-run release flags), so only the last ones trail the decode.
    float M = -INFINITY, O[PER], L = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) O[i] = 0.f;
    uint32_t total = 0, have_total = 0, folded = 0;
    __shared__ uint32_t s_res, s_first, s_dn;
    for (;;) {
        if (threadIdx.x == 0) {
            if (!have_total) {
                total = a.st_cnt[qsi];
                if (a.dyn_cnt) {
                    const uint32_t v = ld_acquire_u32(a.dyn_cnt + qsi);
                    if (v & kCntValid) {
                        total += v & ~kCntValid;
                        have_total = 1;
                    }
                } else {
                    have_total = 1;
                }
            }
            // one load: (runs reserved << 32) | tiles published; once every
            // tile is counted, every run is reserved (reserved, flagged, counted)
            const unsigned long long v = ld_acquire_u64(a.rd + qsi);
            s_dn = have_total && (uint32_t)v >= total;
            s_res = (uint32_t)(v >> 32);
            s_first = 0xFFFFFFFFu;
        }
        __syncthreads();
        // the published prefix of the reserved runs: every thread checks one
        // flag (once every tile is counted, every reserved run is published)
        const uint32_t res = s_res;
        if (!s_dn) {
            for (uint32_t r = folded + threadIdx.x; r < res; r += blockDim.x)
                if (!ld_acquire_u32(a.part_flag + base + r)) atomicMin(&s_first, r);
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const uint32_t nr = min(res, s_first);
            s_nr = nr;
            s_fin = s_dn && nr == res;
        }
        __syncthreads();
        const uint32_t nr = s_nr, fin = s_fin;
        __syncthreads();
        for (uint32_t i0 = folded; i0 < nr; i0 += U) {
            float4 v[U];
            float mu[U], lu[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool ok = i0 + u < nr;
                v[u] = ok ? __ldcg(reinterpret_cast<const float4*>(a.part_O + (base + i0 + u) * NOUT + e0))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
                mu[u] = ok ? __ldcg(a.part_ml + (base + i0 + u) * 8 + h) : -INFINITY;
                lu[u] = ok ? __ldcg(a.part_ml + (base + i0 + u) * 8 + 4 + h) : 0.f;
            }
            float Mn = M;
#pragma unroll
            for (int u = 0; u < U; ++u) Mn = fmaxf(Mn, mu[u]);
            if (Mn == -INFINITY) continue;
            const float sc = fast_exp2(M - Mn);  // M = -inf -> 0
#pragma unroll
            for (int i = 0; i < PER; ++i) O[i] *= sc;
            L *= sc;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const float wgt = fast_exp2(mu[u] - Mn);  // empty run -> 0
                O[0] = fmaf(v[u].x, wgt, O[0]);
                O[1] = fmaf(v[u].y, wgt, O[1]);
                O[2] = fmaf(v[u].z, wgt, O[2]);
                O[3] = fmaf(v[u].w, wgt, O[3]);
                L = fmaf(lu[u], wgt, L);
            }
            M = Mn;
        }
        const bool progress = nr > folded;
        folded = nr;
        if (fin) {
            if (threadIdx.x == 0) tl_mark(a.tl, 5, false);  // slot complete
            break;
        }
        if (threadIdx.x == 0 && !progress) __nanosleep(s_dn ? 32u : a.poll_ns);  // light polling next to the decode
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // re-arm the slot for the next step (this CTA is the only reader)
        for (uint32_t r = 0; r < folded; ++r) a.part_flag[base + r] = 0;
        if (a.dyn_cnt) a.dyn_cnt[qsi] = 0;
        a.rd[qsi] = 0;
    }
    float res[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) res[i] = L > 0.f ? O[i] / L : 0.f;
    if (head < a.G)
#pragma unroll
        for (int i = 0; i < PER; ++i) out[i] = res[i];
    if (a.p2p_out) {
        // fused exchange: the slot's rows into every rank's full buffer, then
        // one system-scope arrival per rank (release: fence, then the count)
        const uint32_t seq = g / a.p2p_hl, lh = g - seq * a.p2p_hl;
        const size_t fi = (((size_t)seq * a.p2p_kvh + a.p2p_h0 + lh) * a.G + head) * D + (e0 % D);
        if (head < a.G)
            for (uint32_t r = 0; r < a.p2p_n; ++r)
                *reinterpret_cast<float4*>(a.p2p_out[r] + fi) = make_float4(res[0], res[1], res[2], res[3]);
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0)
            for (uint32_t r = 0; r < a.p2p_n; ++r) atomicAdd_system(a.p2p_flag[r], 1u);
    }
    if (threadIdx.x == 0) tl_mark(a.tl, 3, false);
}

// ============================================================ launchers
void launch_combine(int D, const CombineArgs& ca, uint32_t n_qslots, cudaStream_t st) {
    // same shared-memory carveout as the decode kernel, so combine CTAs can sit
    // next to decode CTAs and combine each slot as soon as it completes
    static bool configured = false;
    if (!configured) {
        for (const void* f : {(const void*)combine_kernel<128>, (const void*)combine_kernel<64>,
                              (const void*)combine_kernel<32>})
            SAAP_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                           (int)cudaSharedmemCarveoutMaxShared));
        configured = true;
    }
#define SAAP_COMBINE(DD) \
    launch_pdl(true, combine_kernel<DD>, dim3(n_qslots), dim3(DD), 0, st, ca)
    switch (D) {
        case 128: SAAP_COMBINE(128); break;
        case 64: SAAP_COMBINE(64); break;
        case 32: SAAP_COMBINE(32); break;
        default: fail(SAAP_ERR_UNSUPPORTED, "combine: unsupported head dim");
    }
#undef SAAP_COMBINE
}

// a combine CTA (1 KB) must fit next to a decode CTA on one SM (228 KB, 1 KB
// reserved per CTA) so each slot is combined as soon as it completes
static_assert(sizeof(DecodeSmem<128>) + 1024 + 1024 + 2048 <= 228 * 1024, "decode smem leaves no room for combine CTAs");

template <int D>
static void launch_decode_t(const DecodeMaps& m, const DecodeArgs& a, int grid, cudaStream_t st) {
    const size_t smem = sizeof(DecodeSmem<D>) + 1024;
    static bool configured = false;
    if (!configured) {
        SAAP_CUDA(cudaFuncSetAttribute(decode_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        SAAP_CUDA(cudaFuncSetAttribute(decode_kernel<D>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       (int)cudaSharedmemCarveoutMaxShared));
        configured = true;
    }
    launch_pdl(true, decode_kernel<D>, dim3(grid), dim3((kComputeWarps + 2) * 32), smem, st, a, m);
}

static void launch_decode_tc(const DecodeMaps& m, const DecodeArgs& a, int grid, cudaStream_t st) {
    const size_t smem = sizeof(DecodeTcSmem<128>) + 1024;
    static bool configured = false;
    if (!configured) {
        SAAP_CUDA(cudaFuncSetAttribute(decode_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        SAAP_CUDA(cudaFuncSetAttribute(decode_tc_kernel<128>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       (int)cudaSharedmemCarveoutMaxShared));
        configured = true;
    }
    launch_pdl(true, decode_tc_kernel<128>, dim3(grid), dim3(dtc::THREADS), smem, st, a, m);
}

void launch_decode(int D, const DecodeMaps& m, const DecodeArgs& a, int grid, cudaStream_t st, bool tc) {
    if (tc && D == 128) {
        launch_decode_tc(m, a, grid, st);
        return;
    }
    switch (D) {
        case 128: launch_decode_t<128>(m, a, grid, st); break;
        case 64: launch_decode_t<64>(m, a, grid, st); break;
        case 32: launch_decode_t<32>(m, a, grid, st); break;
        default: fail(SAAP_ERR_UNSUPPORTED, "decode: unsupported head dim " + std::to_string(D));
    }
}

void launch_route_score(const RouteArgs& a, uint32_t n_groups, cudaStream_t st) {
    uint32_t threads = 32;
    while (threads < a.slice) threads <<= 1;
    route_score_kernel<<<dim3(n_groups, a.n_slices), threads, 0, st>>>(a);
    SAAP_CUDA(cudaGetLastError());
}

void launch_route_approx(int D, const ApproxArgs& a, uint32_t n_slots, cudaStream_t st) {
    const dim3 grid(n_slots, (a.C + 31) / 32);
    switch (D) {
        case 128: route_approx_kernel<128><<<grid, 256, 0, st>>>(a); break;
        case 64: route_approx_kernel<64><<<grid, 256, 0, st>>>(a); break;
        case 32: route_approx_kernel<32><<<grid, 256, 0, st>>>(a); break;
        default: fail(SAAP_ERR_UNSUPPORTED, "route: unsupported head dim " + std::to_string(D));
    }
    SAAP_CUDA(cudaGetLastError());
}

bool route_cluster_supported(int D, uint32_t C) {
    const uint32_t S = C / kClusterCtas;
    if (C % kClusterCtas) return false;
    return (D == 128 && (S == 128 || S == 64 || S == 32)) || (D == 64 && (S == 128 || S == 64)) ||
           (D == 32 && S == 128);
}

void launch_route_cluster(int D, const ClusterRouteArgs& a, uint32_t n_slots, cudaStream_t st) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(n_slots * kClusterCtas);
    cfg.blockDim = dim3(kClusterThreads);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kClusterCtas;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // dynamic smem: centroid slice [D][C/8] + member queries [8][G][D] (f32)
    // + partial dots [8][512] (f32; sized for f64)
    cfg.dynamicSmemBytes = ((size_t)D * (a.C / kClusterCtas) + (size_t)kSlotGroups * a.G * D) * 4 +
                           std::max<size_t>((size_t)64 * (D + 1) * 4, (size_t)kSlotGroups * kClusterThreads * 8);
    if (cfg.dynamicSmemBytes > 160 * 1024) fail(SAAP_ERR_UNSUPPORTED, "route: slice too large");
    static bool configured = false;
    if (!configured) {
        for (auto kern : {route_cluster_kernel<128, 128>, route_cluster_kernel<128, 64>,
                          route_cluster_kernel<128, 32>, route_cluster_kernel<64, 128>,
                          route_cluster_kernel<64, 64>, route_cluster_kernel<32, 128>})
            SAAP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        configured = true;
    }
    auto go = [&](void (*kern)(ClusterRouteArgs)) { SAAP_CUDA(cudaLaunchKernelEx(&cfg, kern, a)); };
    const uint32_t S = a.C / kClusterCtas;
    if (D == 128 && S == 128) go(route_cluster_kernel<128, 128>);
    else if (D == 128 && S == 64) go(route_cluster_kernel<128, 64>);
    else if (D == 128 && S == 32) go(route_cluster_kernel<128, 32>);
    else if (D == 64 && S == 128) go(route_cluster_kernel<64, 128>);
    else if (D == 64 && S == 64) go(route_cluster_kernel<64, 64>);
    else if (D == 32 && S == 128) go(route_cluster_kernel<32, 128>);
    else fail(SAAP_ERR_UNSUPPORTED, "route: no fused routing kernel for this geometry");
}

void launch_route_plan(const PlanArgs& a, uint32_t n_groups, bool pdl, cudaStream_t st) {
    const bool route = a.mode == 1 || a.mode == 2 || a.mode == 4;
    size_t smem = 0;
    if (route) smem = (size_t)std::max<uint32_t>(a.P2, kPlanThreads) * 12 + ((a.C + 31) / 32) * 4 + 16;
    smem += (size_t)(a.probes + 8) * (sizeof(Seg) + 4);
    if (route && a.C + 1 <= kStageOff) smem += (size_t)2 * (a.C + 1) * 4;  // staged off/offA
    static bool configured = false;  // static smem (~36 KB) + dynamic can exceed 48 KB
    if (!configured) {
        SAAP_CUDA(cudaFuncSetAttribute(route_plan_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024));
        configured = true;
    }
    if (smem > 180 * 1024) fail(SAAP_ERR_UNSUPPORTED, "route_plan: too many buckets/probes for one CTA");
    launch_pdl(pdl, route_plan_kernel, dim3(n_groups), dim3(kPlanThreads), smem, st, a);
}

}  // namespace saap_b200
