// Key assignment on the 5th-gen tensor cores (tcgen05 + TMEM + TMA), exact.
//
// Reference: best_bucket / assign_keys, partition.cpp:38-48, 191-198:
//   argmax_c sum_j k_j c_cj (fp64, index order), strict '>' (lowest id wins).
//
// Scores S = K (C_hi + C_mid)^T with bf16 keys and a two-term bf16 split of
// the f32 centroids, fp32 accumulation in TMEM.  Per key the epilogue keeps
// the best and second-best approximate score.  With
//   B = 2^-14 * |k|_2 * max_c |c|_2
// bounding |approx - exact| (split residual <= 2^-18 |c| per element, fp32
// accumulation of 256 exact products <= 256 * 2^-23 * sum|k_j c_j|), a key
// whose margin best - second exceeds 2B has the reference's argmax; every
// other key (incl. exact ties and all-zero keys) is re-scored in fp64 with the
// reference's operation order by refine_kernel.  Result: bit-exact.
//
// CTA: 2 tiles of 128 keys (M=128 each) share every 128-centroid B chunk;
// warp 8 issues TMA, warp 9 issues tcgen05.mma (one thread), warps 0-7 drain
// TMEM (warp w: tile w/4, lanes 32*(w%4).., lane = key row) while the next
// chunk accumulates in the other half of TMEM (2 x 256 columns).
#include <cuda.h>

#include "args.cuh"

namespace saap_b200 {

namespace tc {
constexpr int TM = 128;       // keys per tile (UMMA M)
constexpr int NT = 2;         // key tiles per CTA
constexpr int CN = 128;       // centroids per chunk (UMMA N)
constexpr int KD = 128;       // key dim (UMMA K total per term)
constexpr int NSTAGE = 2;     // B ring depth
constexpr int BOX = 64;       // bf16 elements per 128-byte swizzle row
constexpr uint32_t A_TILE_BYTES = TM * KD * 2;         // 32 KB
constexpr uint32_t B_TERM_BYTES = CN * KD * 2;         // 32 KB
constexpr uint32_t B_STAGE_BYTES = 2 * B_TERM_BYTES;   // hi + mid
constexpr uint32_t TMEM_COLS = 512;
constexpr int EPI = 8;        // epilogue warps: (tile, TMEM lane quarter)
constexpr int THREADS = (EPI + 2) * 32;  // warps 0..EPI-1 epilogue, EPI TMA, EPI+1 MMA
}  // namespace tc

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;    // LBO (unused for swizzled K-major) = 1
    d |= (uint64_t)64 << 32;   // SBO = 1024 B between 8-row groups
    d |= (uint64_t)1 << 46;    // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;    // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
    asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
            "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
            : "memory");
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
            "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
            "%28, %29, %30, %31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
              "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
              "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
              "=r"(r[31])
            : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

struct __align__(1024) TcSmem {
    uint8_t A[tc::NT][tc::A_TILE_BYTES];          // [tile][box(2)][128 rows][128 B]
    uint8_t B[tc::NSTAGE][tc::B_STAGE_BYTES];     // [stage][term(2)][box(2)][CN rows][128 B]
    uint64_t a_full;
    uint64_t a_empty;  // the pair's last MMAs have read A (tcgen05.commit)
    uint64_t b_full[tc::NSTAGE];
    uint64_t b_empty[tc::NSTAGE];
    uint64_t t_full[2];
    uint64_t t_empty[2];
    uint32_t tmem_base;
    // column-half partial results of the epilogue: [tile][row] best, second, id
    float pb1[tc::NT][tc::TM], pb2[tc::NT][tc::TM];
    uint32_t pi1[tc::NT][tc::TM];
};

// Persistent: one CTA per SM walks key-tile pairs p = blockIdx.x, + gridDim.x,
// ...  TMEM is allocated and the barriers initialised once; the next pair's
// centroid chunks stream as soon as a B stage frees, and its key tiles load as
// soon as the last MMAs of the current pair have read A, so the fill of one
// pair overlaps the epilogue drain of the previous one.
__global__ void __launch_bounds__(tc::THREADS, 1)
        assign_tc_kernel(const __grid_constant__ CUtensorMap map_k,
                         const __grid_constant__ CUtensorMap map_hi,
                         const __grid_constant__ CUtensorMap map_mid, TcAssignArgs a,
                         uint32_t n_pairs, const __grid_constant__ CUtensorMap map_klo) {
    using namespace tc;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    TcSmem& s = *reinterpret_cast<TcSmem*>(
            (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nchunks = a.Cpad / CN;

    if (threadIdx.x == 0) {
        mbar_init(&s.a_full, 1);
        mbar_init(&s.a_empty, 1);
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(&s.b_full[i], 1);
            mbar_init(&s.b_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s.t_full[i], 1);
            mbar_init(&s.t_empty[i], EPI);  // one arrive per epilogue warp
        }
        fence_mbar_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(&s.tmem_base)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s.tmem_base;

    if (warp == EPI) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&map_k) : "memory");
            if (a.keys_f32) asm volatile("prefetch.tensormap [%0];" ::"l"(&map_klo) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&map_hi) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&map_mid) : "memory");
            uint32_t jg = 0, np = 0;  // chunks / pairs issued by this CTA
            for (uint32_t p = blockIdx.x; p < n_pairs; p += gridDim.x, ++np) {
                if (np) mbar_wait(&s.a_empty, (np - 1) & 1);  // previous pair's MMAs read A
                mbar_arrive_expect_tx(&s.a_full, NT * A_TILE_BYTES);
                for (int t = 0; t < NT; ++t) {
                    const bool lo = a.keys_f32 && t == 1;  // split mode: slot 1 = k_lo of tile 0
                    const TcTile tt = a.tiles[p * NT + (lo ? 0 : t)];
                    const int y = (int)(a.key_row0[tt.group] + tt.lid0);
                    for (int b = 0; b < 2; ++b)
                        tma_load_2d(&s.A[t][b * TM * 128], lo ? &map_klo : &map_k, b * BOX, y, &s.a_full);
                }
                const int ybase = (int)(a.tiles[p * NT].part * a.Cpad);
                for (uint32_t j = 0; j < nchunks; ++j, ++jg) {
                    const uint32_t st = jg % NSTAGE, ph = (jg / NSTAGE) & 1;
                    mbar_wait(&s.b_empty[st], ph ^ 1);
                    mbar_arrive_expect_tx(&s.b_full[st], B_STAGE_BYTES);
                    for (int term = 0; term < 2; ++term)
                        for (int b = 0; b < 2; ++b)
                            tma_load_2d(&s.B[st][term * B_TERM_BYTES + b * CN * 128],
                                        term ? &map_mid : &map_hi, b * BOX, ybase + (int)(j * CN),
                                        &s.b_full[st]);
                }
            }
        }
    } else if (warp == EPI + 1) {
        // ------------------------------------------------ MMA issuer (one thread)
        if (lane == 0) {
            constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) |
                                       ((uint32_t)(CN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
            uint32_t jg = 0, np = 0;
            for (uint32_t p = blockIdx.x; p < n_pairs; p += gridDim.x, ++np) {
                mbar_wait(&s.a_full, np & 1);
                for (uint32_t j = 0; j < nchunks; ++j, ++jg) {
                    const uint32_t st = jg % NSTAGE, ph = (jg / NSTAGE) & 1;
                    const uint32_t buf = jg & 1, bph = (jg >> 1) & 1;
                    mbar_wait(&s.b_full[st], ph);
                    mbar_wait(&s.t_empty[buf], bph ^ 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    for (int t = 0; t < NT; ++t) {
                        // split mode: k_lo accumulates into tile 0's columns
                        const bool lo = a.keys_f32 && t == 1;
                        const uint32_t dcol = tmem + buf * (NT * CN) + (lo ? 0 : t) * CN;
                        for (int term = 0; term < 2; ++term) {
#pragma unroll
                            for (int kk = 0; kk < KD / 16; ++kk) {
                                const uint32_t aoff = (kk >> 2) * TM * 128 + (kk & 3) * 32;
                                const uint32_t boff = term * B_TERM_BYTES + (kk >> 2) * CN * 128 + (kk & 3) * 32;
                                umma_bf16(dcol, umma_desc_sw128(smem_u32(&s.A[t][0]) + aoff),
                                          umma_desc_sw128(smem_u32(&s.B[st][0]) + boff), idesc,
                                          (lo || term || kk) ? 1u : 0u);
                            }
                        }
                    }
                    umma_commit(&s.b_empty[st]);
                    umma_commit(&s.t_full[buf]);
                }
                umma_commit(&s.a_empty);  // A free for the next pair
            }
        }
    } else {
        // ------------------------------------------------ epilogue: warp w drains
        // tile w/4, TMEM lanes 32*(w%4).. (lane = key row); branchless top-2
        // (EPI = 16 would split each chunk's columns into halves merged per
        // pair: measured slower, the extra warps contend for TMEM reads)
        const int t = (warp >> 2) & 1, q4 = warp & 3, half = EPI == 16 ? warp >> 3 : 0;
        const int row = q4 * 32 + lane;
        uint32_t jg = 0;
        for (uint32_t p = blockIdx.x; p < n_pairs; p += gridDim.x) {
            const bool idle = a.keys_f32 && t == 1;  // split mode: tile 1's columns are unused
            const TcTile tt = a.tiles[p * NT + t];
            float b1 = -INFINITY, b2 = -INFINITY;
            uint32_t i1 = 0;
            float n2 = 0.f;
            if (!idle && half == 0 && (uint32_t)row < tt.count) {
                if (a.keys_f32) {
                    const float4* kp = reinterpret_cast<const float4*>(a.keys_f32 + (a.key_row0[tt.group] + tt.lid0 + row) * KD);
#pragma unroll
                    for (int q = 0; q < KD / 4; ++q) {
                        const float4 u = kp[q];
                        n2 = fmaf(u.x, u.x, fmaf(u.y, u.y, fmaf(u.z, u.z, fmaf(u.w, u.w, n2))));
                    }
                } else {
                    const uint4* kp = reinterpret_cast<const uint4*>(a.keys + (a.key_row0[tt.group] + tt.lid0 + row) * KD);
#pragma unroll
                    for (int q = 0; q < KD / 8; ++q) {
                        const uint4 u = kp[q];
                        const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float lo = bf16lo(w4[e]), hi = bf16hi(w4[e]);
                            n2 = fmaf(lo, lo, fmaf(hi, hi, n2));
                        }
                    }
                }
            }
            // split mode: 512 fp32-accumulated products (2^-14) and the key
            // split residual |k - k_hi - k_lo| <= 2^-18 |k| on top of the
            // centroid split: 2^-13 covers both
            const float bound = (a.keys_f32 ? 0x1p-13f : 0x1p-14f) * 1.0001f * sqrtf(n2) * a.cmax[tt.part];
            const uint32_t taddr0 = tmem + ((uint32_t)(q4 * 32) << 16) + t * CN;
            for (uint32_t j = 0; j < nchunks; ++j, ++jg) {
                const uint32_t buf = jg & 1, bph = (jg >> 1) & 1;
                mbar_wait(&s.t_full[buf], bph);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t lim = (j + 1) * CN > a.C ? a.C - j * CN : CN;  // valid columns
#pragma unroll 1
                for (int q = half * (CN / 32) / (EPI / 8); !idle && q < (half + 1) * (CN / 32) / (EPI / 8); ++q) {
                    float v[32];
                    tmem_ld32(taddr0 + buf * (NT * CN) + q * 32, v);
                    const uint32_t c0 = j * CN + q * 32;
                    if ((uint32_t)(q * 32 + 32) > lim) {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if ((uint32_t)(q * 32 + i) >= lim) v[i] = -INFINITY;
                    }
                    // running best (value, lowest id) and second-best value
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const float x = v[i];
                        b2 = fmaxf(b2, fminf(x, b1));
                        const bool g1 = x > b1;
                        b1 = g1 ? x : b1;
                        i1 = g1 ? c0 + i : i1;
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.t_empty[buf]);
            }
            // merge the column halves: half 1 hands its (best, second, id) over
            if (EPI == 16 && half == 1) {
                s.pb1[t][row] = b1;
                s.pb2[t][row] = b2;
                s.pi1[t][row] = i1;
            }
            if (EPI == 16) asm volatile("bar.sync 1, %0;" ::"n"(EPI * 32) : "memory");
            if (EPI == 16 && half == 0) {
                const float ob1 = s.pb1[t][row], ob2 = s.pb2[t][row];
                const uint32_t oi1 = s.pi1[t][row];
                // equal bests: the lower id wins (each half scanned its ids in order)
                b2 = fmaxf(fmaxf(b2, ob2), fminf(b1, ob1));
                if (ob1 > b1 || (ob1 == b1 && oi1 < i1)) {
                    b1 = ob1;
                    i1 = oi1;
                }
            }
            if (EPI == 16) asm volatile("bar.sync 1, %0;" ::"n"(EPI * 32) : "memory");
            if (!idle && half == 0 && (uint32_t)row < tt.count) {
                const uint32_t lid = tt.lid0 + row;
                if (b1 - b2 > 2.f * bound) {
                    a.out[a.out_base[tt.group] + lid] = i1;
                } else {  // ambiguous (near tie, exact tie, zero key): fp64 re-scan
                    const uint32_t slot = atomicAdd(&a.refine_count[tt.group], 1u);
                    a.refine[a.out_base[tt.group] + slot] = lid;
                }
            }
        }
    }
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(TMEM_COLS));
    }
}

// fp64 re-score of ambiguous keys in the reference's exact operation order
// (sequential over d; products of bf16 keys and f32 centroids are exact, so
// DFMA == mulsd+addsd), batched per group so each centroid chunk staged in
// shared memory serves RB keys.  CTA (y, g) takes batches y, y+Y, ... of
// group g's list; lane = key (bf16 pairs in shared memory), warp w scores
// centroids w + 8i of each chunk reading (j, j+1) centroid pairs as one
// 16-byte broadcast, then a (score desc, id asc) reduction over warps.
namespace rf {
constexpr int RB = 32;    // keys per batch (one per lane)
constexpr int RC = 64;    // centroids per staged chunk
constexpr int THREADS = 256;
constexpr int NW = THREADS / 32;
constexpr int PER = RC / NW;  // chains per thread
}  // namespace rf

// (F32: the keys are f32 rows -- the split-mode assignment of f32 keys; the
// products stay exact in fp64, so the DFMA chain is the reference's)
template <int D, bool F32 = false>
__global__ void __launch_bounds__(rf::THREADS) refine_kernel(const uint32_t* list,
                                                             const uint32_t* count,
                                                             const void* keys_any,
                                                             const uint64_t* key_row0,
                                                             const double* const* cent64,
                                                             const uint64_t* out_base, uint32_t C,
                                                             uint32_t* out) {
    using namespace rf;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    double* cs = reinterpret_cast<double*>(smem_raw);  // [RC][D]
    constexpr int KW = F32 ? D + 1 : D / 2 + 1;         // words per staged key row (padded)
    __shared__ uint32_t ks[RB * KW];                    // keys as bf16 pairs, or f32
    __shared__ double red_s[NW][RB];
    __shared__ uint32_t red_i[NW][RB];
    const uint32_t g = blockIdx.y;
    const uint32_t n = count[g];
    const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const double* cg = cent64[g];
    const uint32_t* lg = list + out_base[g];
    for (uint32_t b0 = blockIdx.x * RB; b0 < n; b0 += gridDim.x * RB) {
        const uint32_t nb = min((uint32_t)RB, n - b0);
        __syncthreads();
        constexpr uint32_t WPR = F32 ? D : D / 2;  // words per key row
        for (uint32_t e = tid; e < (uint32_t)RB * WPR; e += THREADS) {
            const uint32_t r = e / WPR, j2 = e % WPR;
            const size_t row = key_row0[g] + lg[b0 + min(r, nb - 1)];
            ks[r * KW + j2] = F32 ? reinterpret_cast<const uint32_t*>(reinterpret_cast<const float*>(keys_any) + row * D)[j2]
                                  : reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint16_t*>(keys_any) + row * D)[j2];
        }
        const uint32_t* kw = ks + lane * KW;
        double best = -INFINITY;
        uint32_t bid = 0xFFFFFFFFu;
        for (uint32_t c0 = 0; c0 < C; c0 += RC) {
            const uint32_t nc = min((uint32_t)RC, C - c0);
            __syncthreads();
            for (uint32_t e = tid; e < (uint32_t)RC * D / 2; e += THREADS)
                reinterpret_cast<double2*>(cs)[e] = 2 * e < nc * D
                        ? reinterpret_cast<const double2*>(cg + (size_t)c0 * D)[e]
                        : make_double2(0.0, 0.0);
            __syncthreads();
#pragma unroll 1
            for (int i0 = 0; i0 < PER; i0 += 4) {
                double acc[4] = {0.0, 0.0, 0.0, 0.0};
                const double* cw = cs + (w + NW * i0) * D;
#pragma unroll 8
                for (int j2 = 0; j2 < D / 2; ++j2) {
                    const double k0 = F32 ? (double)__uint_as_float(kw[2 * j2]) : (double)__uint_as_float(kw[j2] << 16);
                    const double k1 = F32 ? (double)__uint_as_float(kw[2 * j2 + 1])
                                          : (double)__uint_as_float(kw[j2] & 0xFFFF0000u);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const double2 cv = reinterpret_cast<const double2*>(cw + NW * i * D)[j2];
                        acc[i] = fma(k0, cv.x, acc[i]);
                        acc[i] = fma(k1, cv.y, acc[i]);
                    }
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {  // ascending centroid ids: strict > keeps the lowest
                    const uint32_t c = w + NW * (i0 + i);
                    if (c < nc && acc[i] > best) {
                        best = acc[i];
                        bid = c0 + c;
                    }
                }
            }
        }
        red_s[w][lane] = best;
        red_i[w][lane] = bid;
        __syncthreads();
        if (tid < nb) {
            double bs = red_s[0][tid];
            uint32_t bi = red_i[0][tid];
            for (int v = 1; v < NW; ++v) {
                const double o = red_s[v][tid];
                const uint32_t oi = red_i[v][tid];
                if (o > bs || (o == bs && oi < bi)) {
                    bs = o;
                    bi = oi;
                }
            }
            out[out_base[g] + lg[b0 + tid]] = bi == 0xFFFFFFFFu ? 0u : bi;
        }
    }
}

// f32 centroids -> (hi, mid) bf16 terms, rows padded to Cpad with zeros.
__global__ void split_centroids_kernel(const float* cent, uint32_t C, uint32_t Cpad, uint32_t D,
                                       uint16_t* hi, uint16_t* mid) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < Cpad * D; e += gridDim.x * blockDim.x) {
        const uint32_t c = e / D;
        float x = c < C ? cent[e] : 0.f;
        const uint16_t h = f32_to_bf16_rne(x);
        const float r = x - __uint_as_float((uint32_t)h << 16);
        hi[e] = h;
        mid[e] = f32_to_bf16_rne(r);
    }
}

// f32 rows -> (hi, lo) bf16 split (the split-mode assignment's keys)
__global__ void split_rows_kernel(const float* x, uint64_t n, uint16_t* hi, uint16_t* lo) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x) {
        const float v = x[e];
        const uint16_t h = f32_to_bf16_rne(v);
        hi[e] = h;
        lo[e] = f32_to_bf16_rne(v - __uint_as_float((uint32_t)h << 16));
    }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        SAAP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p)
            fail(SAAP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = (EncodeTiledFn)p;
    }
    return fn;
}

static CUtensorMap make_map(const void* base, uint64_t rows, uint32_t box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)tc::KD, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)tc::KD * 2};
    const cuuint32_t box[2] = {(cuuint32_t)tc::BOX, box_rows};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                             strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(SAAP_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

// [rows x D] bf16 row-major tensor, boxes of min(D,64) elements x box_rows;
// 128-byte swizzle for D >= 64 (per 64-element half), 64-byte for D = 32.
CUtensorMap make_row_map(const void* base, uint64_t rows, uint32_t D, uint32_t box_rows) {
    CUtensorMap m;
    const uint32_t inner = D >= 64 ? 64 : D;
    const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)(rows ? rows : 1)};
    const cuuint64_t strides[1] = {(cuuint64_t)D * 2};
    const cuuint32_t box[2] = {inner, box_rows};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                             strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             inner == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        fail(SAAP_ERR_CUDA, "cuTensorMapEncodeTiled (rows) failed: " + std::to_string((int)r));
    return m;
}

CUtensorMap make_group_map(const void* base, uint64_t rows, uint32_t D, uint32_t groups) {
    CUtensorMap m;
    const uint32_t inner = D >= 64 ? 64 : D;   // elements per swizzle row (128 or 64 bytes)
    const uint32_t halves = D / inner;
    const cuuint64_t dims[4] = {(cuuint64_t)inner, (cuuint64_t)(rows ? rows : 1), (cuuint64_t)halves, 16};
    const cuuint64_t strides[3] = {(cuuint64_t)D * 2, (cuuint64_t)inner * 2, (cuuint64_t)D * 2 * 8};
    const cuuint32_t box[4] = {inner, 8, halves, groups};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims,
                             strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             inner == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        fail(SAAP_ERR_CUDA, "cuTensorMapEncodeTiled (grouped rows) failed: " + std::to_string((int)r));
    return m;
}

uint32_t tc_cpad(uint32_t C) { return (C + tc::CN - 1) / tc::CN * tc::CN; }

void launch_split_rows(const float* x, uint64_t n, uint16_t* hi, uint16_t* lo, cudaStream_t st) {
    if (!n) return;
    split_rows_kernel<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 32), 256, 0, st>>>(x, n, hi, lo);
    SAAP_CUDA(cudaGetLastError());
}

void launch_split_centroids(const float* cent, uint32_t C, uint32_t D, uint16_t* hi, uint16_t* mid,
                            cudaStream_t st) {
    const uint32_t Cpad = tc_cpad(C);
    split_centroids_kernel<<<(Cpad * D + 255) / 256, 256, 0, st>>>(cent, C, Cpad, D, hi, mid);
    SAAP_CUDA(cudaGetLastError());
}

// Host tile list: per group, 128-key tiles padded to an even count so the
// two tiles of a CTA share one partition.
void build_tc_tiles(const std::vector<GroupMeta>& meta, const std::vector<uint32_t>& part_slot,
                    std::vector<TcTile>& tiles, bool split) {
    tiles.clear();
    for (size_t g = 0; g < meta.size(); ++g) {
        const uint32_t ns = meta[g].n - meta[g].sink;
        const size_t first = tiles.size();
        for (uint32_t f = 0; f < ns; f += tc::TM) {
            tiles.push_back(TcTile{(uint32_t)g, f, std::min<uint32_t>(tc::TM, ns - f), part_slot[g]});
            if (split) tiles.push_back(TcTile{(uint32_t)g, f, 0, part_slot[g]});  // its k_lo slot
        }
        if ((tiles.size() - first) % tc::NT) tiles.push_back(TcTile{(uint32_t)g, 0, 0, part_slot[g]});
    }
}

void launch_assign_tc(const uint16_t* keys, uint64_t key_rows, const uint16_t* hi,
                      const uint16_t* mid, uint32_t n_parts, const TcAssignArgs& args,
                      uint32_t n_tiles, cudaStream_t st, const uint16_t* keys_lo) {
    const CUtensorMap mk = make_map(keys, key_rows, tc::TM);
    const CUtensorMap mlo = make_map(keys_lo ? keys_lo : keys, key_rows, tc::TM);
    const CUtensorMap mh = make_map(hi, (uint64_t)n_parts * args.Cpad, tc::CN);
    const CUtensorMap mm = make_map(mid, (uint64_t)n_parts * args.Cpad, tc::CN);
    const size_t smem = sizeof(TcSmem) + 1024;
    static bool configured = false;
    if (!configured) {
        SAAP_CUDA(cudaFuncSetAttribute(assign_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        configured = true;
    }
    const uint32_t n_pairs = n_tiles / tc::NT;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t grid = std::max<uint32_t>(1u, std::min<uint32_t>(n_pairs, (uint32_t)sms));
    assign_tc_kernel<<<grid, tc::THREADS, smem, st>>>(mk, mh, mm, args, n_pairs, mlo);
    SAAP_CUDA(cudaGetLastError());
}

void launch_refine(const uint32_t* list, const uint32_t* count, const void* keys,
                   const uint64_t* key_row0, const double* const* cent64, const uint64_t* out_base,
                   uint32_t C, uint32_t* out, uint32_t n_groups, int sm_count, cudaStream_t st,
                   bool f32_keys) {
    using namespace rf;
    const size_t smem = (size_t)RC * tc::KD * sizeof(double);
    static bool configured = false;
    if (!configured) {
        SAAP_CUDA(cudaFuncSetAttribute(refine_kernel<tc::KD>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        SAAP_CUDA(cudaFuncSetAttribute(refine_kernel<tc::KD, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = true;
    }
    const uint32_t y = std::max<uint32_t>(1, (uint32_t)(2 * sm_count) / std::max<uint32_t>(n_groups, 1));
    if (f32_keys)
        refine_kernel<tc::KD, true><<<dim3(y, n_groups), THREADS, smem, st>>>(list, count, keys, key_row0, cent64,
                                                                           out_base, C, out);
    else
        refine_kernel<tc::KD><<<dim3(y, n_groups), THREADS, smem, st>>>(list, count, keys, key_row0, cent64,
                                                                     out_base, C, out);
    SAAP_CUDA(cudaGetLastError());
}

}  // namespace saap_b200
