// Prefill side of SAAP: key assignment and the bucket-contiguous KV layout.
//
// Reference semantics (/root/reference/proj/core/src):
//   best_bucket / assign_keys  partition.cpp:38-48, 181-198
//   build_ivf                  partition.cpp:200-223  (stable counting sort)
//   derope_indexed             attention.cpp:207-222, rotate_with rope.cpp:29-41
#include <algorithm>

#include "common.cuh"

namespace saap_b200 {

// ------------------------------------------------------------ exact assignment
// argmax_c sum_j k_j c_cj with the sum in fp64 in index order; products of
// f32 (or bf16) by f32 are exact in fp64, so each DFMA equals the reference's
// mulsd+addsd pair.  Strict '>' in ascending c => lowest id
// wins ties; the all-zero key stays on bucket 0.
template <typename KT, int D>
__global__ void __launch_bounds__(128) assign_exact_kernel(
        const TileDesc* tiles, const KT* keys, const uint64_t* key_row0,
        const double* const* cent64, uint32_t C, uint32_t* out, const uint64_t* out_base,
        const uint32_t* sel_list, uint32_t sel_count) {
    constexpr int CB = 32;  // centroids per smem chunk
    __shared__ double sc[CB][D];
    uint32_t lid, g;
    bool active;
    if (sel_list) {  // refine mode: explicit (group, local id) list
        const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
        active = e < sel_count;
        const uint32_t v = active ? sel_list[e] : 0;
        g = tiles[0].group;  // refine lists are per single-group launch
        lid = v;
    } else {
        const TileDesc td = tiles[blockIdx.x];
        g = td.group;
        lid = td.first + blockIdx.y * blockDim.x + threadIdx.x;
        active = (blockIdx.y * blockDim.x + threadIdx.x) < td.count;
    }
    float k[D];
    if (active) {
        const KT* kp = keys + (key_row0[g] + lid) * D;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            if constexpr (sizeof(KT) == 2) k[j] = __uint_as_float(((uint32_t)kp[j]) << 16);
            else k[j] = kp[j];
        }
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j) k[j] = 0.f;
    }
    const double* cg = cent64[g];
    double best = -INFINITY;
    uint32_t best_id = 0;
    for (uint32_t c0 = 0; c0 < C; c0 += CB) {
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < CB * D; e += blockDim.x) {
            const uint32_t cc = c0 + e / D;
            sc[e / D][e % D] = cc < C ? cg[(size_t)cc * D + e % D] : 0.0;
        }
        __syncthreads();
#pragma unroll 1
        for (int cc = 0; cc < CB; cc += 8) {
            double s[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) s[u] = 0.0;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const double kd = (double)k[j];
#pragma unroll
                for (int u = 0; u < 8; ++u) s[u] = fma(kd, sc[cc + u][j], s[u]);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t c = c0 + cc + u;
                if (c < C && s[u] > best) {
                    best = s[u];
                    best_id = c;
                }
            }
        }
    }
    if (active) out[out_base[g] + lid] = best_id;
}

// ------------------------------------------------------------ histograms
// hist[tile][c] = #keys of bucket c in the tile; countA[g][c] += #keys of
// bucket c with position < T (region A).
__global__ void __launch_bounds__(512) hist_kernel(const TileDesc* tiles, const GroupMeta* meta,
                                                   const uint32_t* assign, uint32_t C,
                                                   uint32_t* hist, uint32_t* countA) {
    extern __shared__ uint32_t hs[];  // 2*C
    uint32_t* h = hs;
    uint32_t* hA = hs + C;
    const TileDesc td = tiles[blockIdx.x];
    const GroupMeta gm = meta[td.group];
    for (uint32_t c = threadIdx.x; c < 2 * C; c += blockDim.x) hs[c] = 0;
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < td.count; e += blockDim.x) {
        const uint32_t lid = td.first + e;
        const uint32_t c = assign[gm.ivf_base + lid];
        if (c >= C) continue;  // validated on the host for host inputs
        atomicAdd(&h[c], 1u);
        if (gm.sink + lid < gm.T) atomicAdd(&hA[c], 1u);
    }
    __syncthreads();
    uint32_t* ht = hist + (size_t)blockIdx.x * C;
    for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) {
        ht[c] = h[c];
        if (hA[c]) atomicAdd(&countA[(size_t)td.group * C + c], hA[c]);
    }
}

// Per group: tile bases within each bucket (exclusive over tiles), then the
// exclusive scans over buckets -> off (all keys) and offA (region A).
// Stage 1, CTA (group, 32 buckets): thread (chunk k, bucket b) sums a run of
// tiles with all loads in flight, the 32 chunk sums are scanned in shared
// memory, then each thread rewrites its run as exclusive prefixes.
constexpr int kScanChunks = 32;
__global__ void __launch_bounds__(1024) scan_tiles_kernel(const uint32_t* tile_first, uint32_t C,
                                                          uint32_t* hist, uint32_t* tot) {
    __shared__ uint32_t part[kScanChunks][33];
    const uint32_t g = blockIdx.x, b = threadIdx.x & 31, k = threadIdx.x >> 5;
    const uint32_t c = blockIdx.y * 32 + b;
    const uint32_t t0 = tile_first[g], nt = tile_first[g + 1] - t0;
    const uint32_t per = (nt + kScanChunks - 1) / kScanChunks;
    const uint32_t lo = t0 + min(nt, k * per), hi = t0 + min(nt, (k + 1) * per);
    constexpr int U = 16;
    uint32_t sum = 0;
    if (c < C) {
        for (uint32_t t = lo; t < hi; t += U) {
            uint32_t v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = t + u < hi ? hist[(size_t)(t + u) * C + c] : 0u;
#pragma unroll
            for (int u = 0; u < U; ++u) sum += v[u];
        }
    }
    part[k][b] = sum;
    __syncthreads();
    uint32_t run = 0;
    for (uint32_t j = 0; j < k; ++j) run += part[j][b];
    if (k == kScanChunks - 1 && c < C) tot[(size_t)g * C + c] = run + sum;
    if (c < C) {
        for (uint32_t t = lo; t < hi; t += U) {
            uint32_t v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = t + u < hi ? hist[(size_t)(t + u) * C + c] : 0u;
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (t + u < hi) {
                    hist[(size_t)(t + u) * C + c] = run;
                    run += v[u];
                }
        }
    }
}

// Stage 2, one CTA per group: exclusive scans of tot (all keys) and countA
// (region A) over buckets.
__global__ void __launch_bounds__(1024) scan_buckets_kernel(uint32_t C, const uint32_t* totg,
                                                            const uint32_t* countA, uint32_t* off,
                                                            uint32_t* offA) {
    __shared__ uint32_t wsum[2][32];
    const uint32_t g = blockIdx.x;
    const uint32_t* t_all = totg + (size_t)g * C;
    const uint32_t* t_A = countA + (size_t)g * C;
    // thread owns a chunk of buckets
    const uint32_t per = (C + blockDim.x - 1) / blockDim.x;
    const uint32_t lo = min(C, threadIdx.x * per), hi = min(C, lo + per);
    uint32_t s0 = 0, s1 = 0;
    for (uint32_t c = lo; c < hi; ++c) {
        s0 += t_all[c];
        s1 += t_A[c];
    }
    // warp inclusive scans
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t i0 = s0, i1 = s1;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t a0 = __shfl_up_sync(0xFFFFFFFFu, i0, o);
        const uint32_t a1 = __shfl_up_sync(0xFFFFFFFFu, i1, o);
        if (lane >= (uint32_t)o) {
            i0 += a0;
            i1 += a1;
        }
    }
    if (lane == 31) {
        wsum[0][warp] = i0;
        wsum[1][warp] = i1;
    }
    __syncthreads();
    if (warp == 0) {
        uint32_t w0 = lane < blockDim.x / 32 ? wsum[0][lane] : 0;
        uint32_t w1 = lane < blockDim.x / 32 ? wsum[1][lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t a0 = __shfl_up_sync(0xFFFFFFFFu, w0, o);
            const uint32_t a1 = __shfl_up_sync(0xFFFFFFFFu, w1, o);
            if (lane >= (uint32_t)o) {
                w0 += a0;
                w1 += a1;
            }
        }
        wsum[0][lane] = w0;
        wsum[1][lane] = w1;
    }
    __syncthreads();
    uint32_t e0 = i0 - s0 + (warp ? wsum[0][warp - 1] : 0);
    uint32_t e1 = i1 - s1 + (warp ? wsum[1][warp - 1] : 0);
    uint32_t* og = off + (size_t)g * (C + 1);
    uint32_t* oAg = offA + (size_t)g * (C + 1);
    for (uint32_t c = lo; c < hi; ++c) {
        og[c] = e0;
        oAg[c] = e1;
        e0 += t_all[c];
        e1 += t_A[c];
    }
    if (hi == C && lo < hi) {
        og[C] = e0;
        oAg[C] = e1;
    }
    if (C == 0 && threadIdx.x == 0) {
        og[0] = 0;
        oAg[0] = 0;
    }
}

// ------------------------------------------------------------ rank + scatter
// One warp per tile, 32 keys per step in id order: match_any groups equal
// buckets, the leader bumps the bucket's running position -> stable ranks, so
// idx ascends within each bucket exactly as the reference's forward scatter.
// The running positions (off + tile base) and the region-A shift (offA - off)
// live in shared memory, so the only global loads in the loop are the
// (prefetched) assignments.  Writes idx/invA/posA and each key's destination
// row for move_rows_kernel.
constexpr int kScatterWarps = 4;  // warps per tile (fewer when C is large): each ranks one sub-range
__global__ void __launch_bounds__(32 * kScatterWarps) scatter_kernel(
        const TileDesc* tiles, const GroupMeta* meta, const uint32_t* assign, uint32_t C,
        const uint32_t* hist, const uint32_t* off, const uint32_t* offA, uint32_t* idx,
        uint32_t* invA, uint32_t* posA, uint32_t* dst_row) {
    extern __shared__ uint32_t sm[];  // shiftA[C], run[W][C]
    uint32_t* shA = sm;
    uint32_t* runw = sm + C;
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
    const TileDesc td = tiles[blockIdx.x];
    const GroupMeta gm = meta[td.group];
    const uint32_t* ht = hist + (size_t)blockIdx.x * C;
    const uint32_t* og = off + (size_t)td.group * (C + 1);
    const uint32_t* oAg = offA + (size_t)td.group * (C + 1);
    for (uint32_t e = threadIdx.x; e < W * C; e += blockDim.x) runw[e] = 0;
    __syncthreads();
    // warp w ranks keys [e_lo, e_hi) of the tile (whole 32-key steps)
    const uint32_t sub = ((td.count + W - 1) / W + 31) & ~31u;
    const uint32_t e_lo = min(td.count, w * sub), e_hi = min(td.count, e_lo + sub);
    const uint32_t* as = assign + gm.ivf_base + td.first;
    for (uint32_t e = e_lo + lane; e < e_hi; e += 32) atomicAdd(&runw[w * C + as[e]], 1u);
    __syncthreads();
    // exclusive prefix over the warps, from the tile's running position
    for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) {
        const uint32_t o = og[c];
        uint32_t r = o + ht[c];
        for (uint32_t ww = 0; ww < W; ++ww) {
            const uint32_t t = runw[ww * C + c];
            runw[ww * C + c] = r;
            r += t;
        }
        shA[c] = oAg[c] - o;
    }
    __syncthreads();
    uint32_t* run = runw + w * C;
    uint32_t cn = e_lo + lane < e_hi ? as[e_lo + lane] : 0xFFFFFFFFu;
    for (uint32_t e0 = e_lo; e0 < e_hi; e0 += 32) {
        const uint32_t e = e0 + lane;
        const bool act = e < e_hi;
        const uint32_t c = cn;
        cn = e + 32 < e_hi ? as[e + 32] : 0xFFFFFFFFu;  // next step's bucket in flight
        const uint32_t lid = td.first + e;
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, c);
        const uint32_t leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (act && lane == leader) {
            base = run[c];
            run[c] = base + __popc(peers);
        }
        base = __shfl_sync(0xFFFFFFFFu, base, leader);
        if (act) {
            const uint32_t q = base + __popc(peers & ((1u << lane) - 1));  // position in group idx
            idx[gm.ivf_base + q] = lid;
            const uint32_t pos = gm.sink + lid;
            uint32_t row = pos;
            if (pos < gm.T) {
                row = gm.sink + q + shA[c];
                invA[gm.ivf_base + lid] = row;
                if (posA) posA[gm.ivf_base + (row - gm.sink)] = pos;
            }
            if (dst_row) dst_row[gm.ivf_base + lid] = row;
        }
        __syncwarp();
    }
}

// Streams K/V rows to their packed rows.  One warp moves one key per step:
// the K row and the V row as 16-byte chunks across the lanes (coalesced
// 2 x 256-byte reads and writes at d=128), U keys in flight per warp.  The
// key's context is found once per run of keys (contexts are contiguous in the
// key order); dst_row comes from scatter_kernel.
template <int D>
__global__ void __launch_bounds__(256) move_rows_kernel(const GroupMeta* meta, const uint32_t* n_tile_group,
                                                        uint32_t n_groups, uint64_t total_ns,
                                                        const uint32_t* dst_row, const uint16_t* Ksrc,
                                                        const uint16_t* Vsrc, const uint64_t* src_row0,
                                                        uint16_t* Kdst, uint16_t* Vdst) {
    constexpr uint32_t CH = D / 8;                 // 16-byte chunks per row
    constexpr uint32_t KPW = 32 / (2 * CH);        // keys per warp step (1 at d=128, 2 at 64, 4 at 32)
    constexpr int U = 1;                           // warp steps in flight
    const uint32_t lane = threadIdx.x & 31, sub = lane / (2 * CH), part = lane % (2 * CH);
    const bool isv = part >= CH;
    const uint32_t cc = isv ? part - CH : part;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t step = n_warps * KPW;
    uint64_t g_lo = 1, g_hi = 0;  // cached context key range [g_lo, g_hi)
    uint32_t g = 0;
    GroupMeta gm{};
    uint64_t srow0 = 0;
    auto locate = [&](uint64_t key) {
        if (key >= g_lo && key < g_hi) return;
        uint32_t lo = 0, hi = n_groups;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (meta[mid].ivf_base <= key) lo = mid;
            else hi = mid;
        }
        g = lo;
        gm = meta[lo];
        srow0 = src_row0[lo];
        g_lo = gm.ivf_base;
        g_hi = gm.ivf_base + (gm.n - gm.sink);
    };
    for (uint64_t k0 = warp * KPW + sub; k0 < total_ns; k0 += U * step) {
        uint4 v[U];
        uint16_t* dst[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t key = k0 + u * step;
            dst[u] = nullptr;
            if (key >= total_ns) continue;
            locate(key);
            const uint64_t lid = key - gm.ivf_base;
            if (lid >= gm.n - gm.sink) continue;  // capacity gap after the group's keys
            const uint16_t* src = (isv ? Vsrc : Ksrc) + (srow0 + gm.sink + lid) * D + cc * 8;
            v[u] = __ldcs(reinterpret_cast<const uint4*>(src));
            dst[u] = (isv ? Vdst : Kdst) + (gm.row_base + dst_row[key]) * D + cc * 8;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (dst[u]) __stcs(reinterpret_cast<uint4*>(dst[u]), v[u]);
    }
    (void)g;
    (void)n_tile_group;
}

// sink rows [0, sink) keep their position
template <int D>
__global__ void copy_sink_kernel(const GroupMeta* meta, uint32_t n_groups, const uint16_t* Ksrc,
                                 const uint16_t* Vsrc, const uint64_t* src_row0, uint16_t* Kdst,
                                 uint16_t* Vdst) {
    const uint32_t g = blockIdx.x;
    const GroupMeta gm = meta[g];
    constexpr int CH = D / 8;
    for (uint32_t e = threadIdx.x; e < gm.sink * CH; e += blockDim.x) {
        const uint32_t r = e / CH, cc = e % CH;
        const uint64_t s = (src_row0[g] + r) * D + cc * 8, d = (gm.row_base + r) * D + cc * 8;
        *reinterpret_cast<uint4*>(Kdst + d) = *reinterpret_cast<const uint4*>(Ksrc + s);
        *reinterpret_cast<uint4*>(Vdst + d) = *reinterpret_cast<const uint4*>(Vsrc + s);
    }
}

// Appended keys: rows [n, n + k) of every group (position order, after the
// window) from a [n_groups x k] staging block; meta still holds the old n.
template <int D>
__global__ void append_rows_kernel(const GroupMeta* meta, uint32_t k, const uint16_t* Ksrc,
                                   const uint16_t* Vsrc, uint16_t* Kdst, uint16_t* Vdst) {
    const uint32_t g = blockIdx.y;
    const GroupMeta gm = meta[g];
    constexpr int CH = D / 8;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < k * CH; e += gridDim.x * blockDim.x) {
        const uint32_t r = e / CH, cc = e % CH;
        const uint64_t s = ((uint64_t)g * k + r) * D + cc * 8, d = (gm.row_base + gm.n + r) * D + cc * 8;
        *reinterpret_cast<uint4*>(Kdst + d) = *reinterpret_cast<const uint4*>(Ksrc + s);
        *reinterpret_cast<uint4*>(Vdst + d) = *reinterpret_cast<const uint4*>(Vsrc + s);
    }
}

// ------------------------------------------------------------ dtype + rope
__global__ void f32_to_bf16_kernel(const float* in, uint16_t* out, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = f32_to_bf16_rne(in[i]);
}

// x' = (x0 c - x1 s, x0 s + x1 c) in fp64 with the products rounded before
// the add (rope.cpp:32-39); (c, s) come from a host table computed with the
// same libm calls as the reference, so the result is bit-identical.
__global__ void derope_kernel(const float* x, const double* cs, uint64_t rows, uint32_t D,
                              float* out) {
    const uint64_t half = D / 2;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < rows * half;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = e / half, j = e % half;
        const double c = cs[e * 2], s = cs[e * 2 + 1];
        const double x0 = x[i * D + 2 * j], x1 = x[i * D + 2 * j + 1];
        out[i * D + 2 * j] = (float)__dadd_rn(__dmul_rn(x0, c), -__dmul_rn(x1, s));
        out[i * D + 2 * j + 1] = (float)__dadd_rn(__dmul_rn(x0, s), __dmul_rn(x1, c));
    }
}

// ------------------------------------------------------------ coverage
// attention_mass_coverage (attention.cpp:427-462): per query row, the share of
// softmax(q k / sqrt(d)) mass over non-window keys [lo, hi) that falls in the
// selected buckets; mean over the rows.  One CTA per context walks its packed
// rows once (positions via posA / identity) with an online (max, denom, hit)
// per row, merged across threads in shared memory.
constexpr int kCovRows = 8;  // query rows per pass
__global__ void __launch_bounds__(256) coverage_kernel(const GroupMeta* meta, const uint16_t* K,
                                                       const uint32_t* posA, const uint32_t* assign,
                                                       const float* q, uint32_t G, uint32_t D,
                                                       const uint32_t* sel, uint32_t l, uint32_t C,
                                                       uint32_t recent, double* out) {
    extern __shared__ float csm[];  // q rows (kCovRows x D) then bitmap (C/32 words)
    __shared__ float red[3][kCovRows][8];
    const uint32_t g = blockIdx.x, tid = threadIdx.x;
    const GroupMeta gm = meta[g];
    const uint32_t lo = min(gm.sink, gm.n);
    uint32_t hi = gm.n > recent ? gm.n - recent : 0;
    if (hi < lo) hi = lo;
    if (lo == hi) {
        if (tid == 0) out[g] = 1.0;  // nothing outside the window
        return;
    }
    uint32_t* bitmap = reinterpret_cast<uint32_t*>(csm + kCovRows * D);
    for (uint32_t w = tid; w < (C + 31) / 32; w += blockDim.x) bitmap[w] = 0;
    __syncthreads();
    for (uint32_t b = tid; b < l; b += blockDim.x) {
        const uint32_t c = sel[(size_t)g * l + b];
        atomicOr(&bitmap[c >> 5], 1u << (c & 31));
    }
    const float scale = 1.4426950408889634f / sqrtf((float)D);  // exp2 domain
    double total = 0.0;
    for (uint32_t r0 = 0; r0 < G; r0 += kCovRows) {
        const uint32_t nr = min((uint32_t)kCovRows, G - r0);
        __syncthreads();
        for (uint32_t e = tid; e < nr * D; e += blockDim.x)
            csm[e] = q[((size_t)g * G + r0) * D + e] * scale;
        __syncthreads();
        float m[kCovRows], den[kCovRows], hit[kCovRows];
#pragma unroll
        for (int i = 0; i < kCovRows; ++i) {
            m[i] = -INFINITY;
            den[i] = 0.f;
            hit[i] = 0.f;
        }
        for (uint32_t r = gm.sink + tid; r < gm.n; r += blockDim.x) {
            const uint32_t pos = r < gm.T ? posA[gm.ivf_base + (r - gm.sink)] : r;
            if (pos < lo || pos >= hi) continue;
            const uint32_t c = assign[gm.ivf_base + (pos - gm.sink)];
            const bool picked = (bitmap[c >> 5] >> (c & 31)) & 1u;
            const uint16_t* kr = K + (gm.row_base + r) * D;
#pragma unroll
            for (int i = 0; i < kCovRows; ++i) {
                if ((uint32_t)i >= nr) break;
                float sc = 0.f;
                for (uint32_t j = 0; j < D; j += 2) {
                    const uint32_t kk = *reinterpret_cast<const uint32_t*>(kr + j);
                    sc = fmaf(csm[i * D + j], bf16lo(kk), sc);
                    sc = fmaf(csm[i * D + j + 1], bf16hi(kk), sc);
                }
                if (sc > m[i]) {
                    const float a = exp2f(m[i] - sc);
                    den[i] *= a;
                    hit[i] *= a;
                    m[i] = sc;
                }
                const float p = exp2f(sc - m[i]);
                den[i] += p;
                if (picked) hit[i] += p;
            }
        }
        // block merge of (m, den, hit) per row: warp shuffles then shared memory
        const uint32_t lane = tid & 31, warp = tid >> 5;
#pragma unroll
        for (int i = 0; i < kCovRows; ++i) {
            for (int o = 16; o; o >>= 1) {
                const float om = __shfl_xor_sync(0xFFFFFFFFu, m[i], o);
                const float od = __shfl_xor_sync(0xFFFFFFFFu, den[i], o);
                const float oh = __shfl_xor_sync(0xFFFFFFFFu, hit[i], o);
                const float M = fmaxf(m[i], om);
                const float a = M == -INFINITY ? 0.f : exp2f(m[i] - M), b = M == -INFINITY ? 0.f : exp2f(om - M);
                den[i] = den[i] * a + od * b;
                hit[i] = hit[i] * a + oh * b;
                m[i] = M;
            }
            if (lane == 0) {
                red[0][i][warp] = m[i];
                red[1][i][warp] = den[i];
                red[2][i][warp] = hit[i];
            }
        }
        __syncthreads();
        if (tid < nr) {
            float M = -INFINITY;
            for (uint32_t w = 0; w < blockDim.x / 32; ++w) M = fmaxf(M, red[0][tid][w]);
            double dn = 0.0, ht = 0.0;
            for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
                const double a = red[0][tid][w] == -INFINITY ? 0.0 : exp2((double)red[0][tid][w] - M);
                dn += red[1][tid][w] * a;
                ht += red[2][tid][w] * a;
            }
            red[0][tid][0] = (float)(ht / dn);
        }
        __syncthreads();
        if (tid == 0)
            for (uint32_t i = 0; i < nr; ++i) total += red[0][i][0];
    }
    if (tid == 0) out[g] = total / (double)G;
}

// ------------------------------------------------------------ launchers
void launch_assign_exact(int D, bool bf16_keys, const TileDesc* tiles, uint32_t n_tiles,
                         const void* keys, const uint64_t* key_row0, const double* const* cent64,
                         uint32_t C, uint32_t* out, const uint64_t* out_base, cudaStream_t st,
                         uint32_t max_tile_count) {
    // CTAs of 128 keys per tile: only as many as the largest tile needs
    dim3 grid(n_tiles, (std::min<uint32_t>(max_tile_count, kPackTile) + 127) / 128);
#define SAAP_ASSIGN(DD)                                                                       \
    if (bf16_keys)                                                                            \
        assign_exact_kernel<uint16_t, DD><<<grid, 128, 0, st>>>(                              \
                tiles, (const uint16_t*)keys, key_row0, cent64, C, out, out_base, nullptr, 0); \
    else                                                                                      \
        assign_exact_kernel<float, DD><<<grid, 128, 0, st>>>(                                 \
                tiles, (const float*)keys, key_row0, cent64, C, out, out_base, nullptr, 0);
    switch (D) {
        case 128: SAAP_ASSIGN(128); break;
        case 64: SAAP_ASSIGN(64); break;
        case 32: SAAP_ASSIGN(32); break;
        default: fail(SAAP_ERR_UNSUPPORTED, "assign_keys: unsupported key dim " + std::to_string(D));
    }
#undef SAAP_ASSIGN
    SAAP_CUDA(cudaGetLastError());
}

void launch_pack(int D, const TileDesc* tiles, uint32_t n_tiles, const uint32_t* tile_first,
                 uint32_t n_groups, const GroupMeta* meta, const uint32_t* assign, uint32_t C,
                 uint32_t* hist, uint32_t* countA, uint32_t* off, uint32_t* offA, uint32_t* idx,
                 uint32_t* invA, uint32_t* posA, uint32_t* dst_row, uint64_t total_ns,
                 const uint16_t* Ksrc, const uint16_t* Vsrc, const uint64_t* src_row0,
                 uint16_t* Kdst, uint16_t* Vdst, cudaStream_t st) {
    const size_t hsm = (size_t)2 * C * 4;
    static size_t cfg_h = 0, cfg_s = 0;
    if (hsm > 48 * 1024 && hsm > cfg_h) {
        SAAP_CUDA(cudaFuncSetAttribute(hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)hsm));
        cfg_h = hsm;
    }
    SAAP_CUDA(cudaMemsetAsync(countA, 0, (size_t)n_groups * C * 4, st));
    uint32_t* tot = countA + (size_t)n_groups * C;  // per-bucket totals (second half)
    if (n_tiles) hist_kernel<<<n_tiles, 512, hsm, st>>>(tiles, meta, assign, C, hist, countA);
    if (C) scan_tiles_kernel<<<dim3(n_groups, (C + 31) / 32), 1024, 0, st>>>(tile_first, C, hist, tot);
    scan_buckets_kernel<<<n_groups, 1024, 0, st>>>(C, tot, countA, off, offA);
    uint32_t sw = kScatterWarps;
    while (sw > 1 && (size_t)(1 + sw) * C * 4 > 200 * 1024) --sw;
    const size_t ssm = (size_t)(1 + sw) * C * 4;
    if (ssm > 227 * 1024) fail(SAAP_ERR_UNSUPPORTED, "pack: too many buckets for the scatter kernel");
    if (ssm > 48 * 1024 && ssm > cfg_s) {
        SAAP_CUDA(cudaFuncSetAttribute(scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)ssm));
        cfg_s = ssm;
    }
    if (n_tiles)
        scatter_kernel<<<n_tiles, 32 * sw, ssm, st>>>(tiles, meta, assign, C, hist, off, offA, idx, invA,
                                                 posA, Ksrc ? dst_row : nullptr);
#define SAAP_SCATTER(DD)                                                                         \
    if (total_ns)                                                                                \
        move_rows_kernel<DD><<<148 * 8, 256, 0, st>>>(meta, nullptr, n_groups, total_ns, dst_row,  \
                                                       Ksrc, Vsrc, src_row0, Kdst, Vdst);        \
    copy_sink_kernel<DD><<<n_groups, 128, 0, st>>>(meta, n_groups, Ksrc, Vsrc, src_row0, Kdst, Vdst);
    if (Ksrc) switch (D) {
        case 128: SAAP_SCATTER(128); break;
        case 64: SAAP_SCATTER(64); break;
        case 32: SAAP_SCATTER(32); break;
        default: fail(SAAP_ERR_UNSUPPORTED, "pack: unsupported head dim " + std::to_string(D));
    }
#undef SAAP_SCATTER
    SAAP_CUDA(cudaGetLastError());
}

void launch_append_rows(int D, const GroupMeta* meta, uint32_t n_groups, uint32_t k,
                        const uint16_t* Ksrc, const uint16_t* Vsrc, uint16_t* Kdst, uint16_t* Vdst,
                        cudaStream_t st) {
    const dim3 grid(std::max<uint32_t>(1, std::min<uint32_t>(64, (k * (D / 8) + 255) / 256)), n_groups);
    switch (D) {
        case 128: append_rows_kernel<128><<<grid, 256, 0, st>>>(meta, k, Ksrc, Vsrc, Kdst, Vdst); break;
        case 64: append_rows_kernel<64><<<grid, 256, 0, st>>>(meta, k, Ksrc, Vsrc, Kdst, Vdst); break;
        case 32: append_rows_kernel<32><<<grid, 256, 0, st>>>(meta, k, Ksrc, Vsrc, Kdst, Vdst); break;
        default: fail(SAAP_ERR_UNSUPPORTED, "append: unsupported head dim " + std::to_string(D));
    }
    SAAP_CUDA(cudaGetLastError());
}

// Incremental off update for appended keys: off[c] += #new keys of buckets < c
// (the raw per-bucket sizes of the grown context; attention.cpp:356).
__global__ void __launch_bounds__(1024) append_off_kernel(const GroupMeta* meta, const uint32_t* assign,
                                                          uint32_t k, uint32_t C, uint32_t* off) {
    extern __shared__ uint32_t hs[];  // C counters
    __shared__ uint32_t wsum[32];
    const uint32_t g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const GroupMeta gm = meta[g];  // n already grown
    for (uint32_t c = tid; c < C; c += blockDim.x) hs[c] = 0;
    __syncthreads();
    const uint32_t first = gm.n - gm.sink - k;
    for (uint32_t e = tid; e < k; e += blockDim.x) atomicAdd(&hs[assign[gm.ivf_base + first + e]], 1u);
    __syncthreads();
    // block exclusive scan over C (each thread a contiguous chunk)
    const uint32_t per = (C + blockDim.x - 1) / blockDim.x;
    const uint32_t lo = min(C, tid * per), hi = min(C, lo + per);
    uint32_t sum = 0;
    for (uint32_t c = lo; c < hi; ++c) sum += hs[c];
    uint32_t incl = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= (uint32_t)o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < blockDim.x / 32 ? wsum[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, w, o);
            if (lane >= (uint32_t)o) w += v;
        }
        wsum[lane] = w;
    }
    __syncthreads();
    uint32_t run = incl - sum + (warp ? wsum[warp - 1] : 0);
    uint32_t* og = off + (size_t)g * (C + 1);
    for (uint32_t c = lo; c < hi; ++c) {
        og[c] += run;
        run += hs[c];
    }
    if (tid == 0) og[C] += k;
}

void launch_append_off(const GroupMeta* meta, uint32_t n_groups, const uint32_t* assign, uint32_t k,
                       uint32_t C, uint32_t* off, cudaStream_t st) {
    const size_t smem = (size_t)C * 4;
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        SAAP_CUDA(cudaFuncSetAttribute(append_off_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        configured = smem;
    }
    append_off_kernel<<<n_groups, 1024, smem, st>>>(meta, assign, k, C, off);
    SAAP_CUDA(cudaGetLastError());
}

void launch_coverage(const GroupMeta* meta, uint32_t n_groups, const uint16_t* K,
                     const uint32_t* posA, const uint32_t* assign, const float* q, uint32_t G,
                     uint32_t D, const uint32_t* sel, uint32_t l, uint32_t C, uint32_t recent,
                     double* out, cudaStream_t st) {
    const size_t smem = (size_t)kCovRows * D * 4 + ((C + 31) / 32) * 4;
    coverage_kernel<<<n_groups, 256, smem, st>>>(meta, K, posA, assign, q, G, D, sel, l, C, recent, out);
    SAAP_CUDA(cudaGetLastError());
}

void launch_f32_to_bf16(const float* in, uint16_t* out, uint64_t n, cudaStream_t st) {
    if (!n) return;
    const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 65535);
    f32_to_bf16_kernel<<<(unsigned)blocks, 256, 0, st>>>(in, out, n);
    SAAP_CUDA(cudaGetLastError());
}

void launch_derope(const float* x, const double* cs, uint64_t rows, uint32_t D, float* out,
                   cudaStream_t st) {
    const uint64_t n = rows * (D / 2);
    if (!n) return;
    const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 65535);
    derope_kernel<<<(unsigned)blocks, 256, 0, st>>>(x, cs, rows, D, out);
    SAAP_CUDA(cudaGetLastError());
}

}  // namespace saap_b200
