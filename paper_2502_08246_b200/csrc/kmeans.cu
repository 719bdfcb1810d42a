// Device spherical k-means: the partition trainer the
// 1M-token sweep needs, bit-exact with the reference's kmeans_train.
//
// Reference semantics (/root/reference/proj/core/src/partition.cpp):
//   seeding            :79-90   C seed rows (caller's Rng), copy + normalize_row,
//                               zero row -> e_{c mod d}
//   assignment step    :95-110  norm==0 -> (0, 0.0); else best_bucket (:38-48)
//   empty-cluster fix  :117-139 ascending empty c: steal the lowest-score key of
//                               a cluster with >= 2 members (first index on ties),
//                               its score becomes its own norm
//   update step        :142-161 f32 member sums in key order, normalize_row
//                               (:19-31); cancelled sums -> e_{c mod d}
//   objective          :163-167 sum_i best_bucket(k_i).score in key order (fp64)
//
// Every rounding point is reproduced: fp64 dot products in index order (the
// f32 x f32 products are exact in fp64, so a DFMA equals mulsd+addsd), f32
// member sums added sequentially in ascending key order (the bucket order of
// the stable counting sort, pack.cu), sqrt / 1.0/n in IEEE fp64, f32 scaling.
// The objective of iteration t is the score sum of iteration t+1's assignment
// pass (same centroids, same best_bucket), so no extra pass is needed except
// after the last update.
#include "common.cuh"

namespace saap_b200 {

namespace {

constexpr int kAssignThreads = 128;
constexpr int kCentChunk = 32;  // centroids per shared-memory chunk

// One key per thread, keys in registers (zero padded to DM: trailing +0
// products leave an fp64 sum unchanged); centroid chunks staged in shared
// memory as fp64 and broadcast.  Strict '>' over ascending c keeps the lowest
// id on ties, exactly like best_bucket.
template <int DM>
__global__ void __launch_bounds__(kAssignThreads) km_assign_kernel(
        const float* __restrict__ keys, uint32_t n, uint32_t D, const float* __restrict__ cent,
        uint32_t C, uint32_t* __restrict__ assign, double* __restrict__ score,
        unsigned long long* zero_keys) {
    __shared__ double sc[kCentChunk][DM];
    const uint32_t i = blockIdx.x * kAssignThreads + threadIdx.x;
    const bool active = i < n;
    float k[DM];
    bool nz = false;
#pragma unroll
    for (int j = 0; j < DM; ++j) {
        k[j] = (active && (uint32_t)j < D) ? keys[(size_t)i * D + j] : 0.f;
        nz |= k[j] != 0.f;
    }
    double best = -INFINITY;
    uint32_t best_id = 0;
    for (uint32_t c0 = 0; c0 < C; c0 += kCentChunk) {
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < kCentChunk * DM; e += kAssignThreads) {
            const uint32_t cc = c0 + e / DM, j = e % DM;
            sc[e / DM][j] = (cc < C && j < D) ? (double)cent[(size_t)cc * D + j] : 0.0;
        }
        __syncthreads();
#pragma unroll 1
        for (int cc = 0; cc < kCentChunk; cc += 8) {
            double s[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) s[u] = 0.0;
#pragma unroll
            for (int j = 0; j < DM; ++j) {
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
    if (!active) return;
    if (!nz) {  // norm_f == 0 exactly iff every component is +-0
        best = 0.0;
        best_id = 0;
        if (zero_keys) atomicAdd(zero_keys, 1ull);
    }
    assign[i] = best_id;
    score[i] = best;
}

__global__ void km_count_kernel(const uint32_t* assign, uint32_t n, uint32_t* counts) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        atomicAdd(&counts[assign[i]], 1u);
}

// sqrt(sum_j x_j^2) with the sum in fp64 in index order (norm_f, partition.cpp:15-17)
__device__ double row_norm(const float* x, uint32_t D) {
    double s = 0.0;
    for (uint32_t j = 0; j < D; ++j) s = fma((double)x[j], (double)x[j], s);
    return sqrt(s);
}

// Sequential fp64 sum of score[0..n) in index order (the reference's
// objective loop).  Warps 1.. stage the next chunk while warp 0's lane 0 adds
// the current one.
constexpr int kSumChunk = 2048;
__global__ void __launch_bounds__(256) km_objective_kernel(const double* score, uint32_t n,
                                                           double* out) {
    __shared__ double buf[2][kSumChunk];
    double acc = 0.0;
    const uint32_t n_chunks = (n + kSumChunk - 1) / kSumChunk;
    for (uint32_t e = threadIdx.x; e < kSumChunk; e += blockDim.x)
        buf[0][e] = e < n ? score[e] : 0.0;
    __syncthreads();
    for (uint32_t ch = 0; ch < n_chunks; ++ch) {
        const uint32_t nxt = (ch + 1) * kSumChunk;
        if (threadIdx.x >= 32 && ch + 1 < n_chunks)
            for (uint32_t e = threadIdx.x - 32; e < kSumChunk; e += blockDim.x - 32)
                buf[(ch + 1) & 1][e] = nxt + e < n ? score[nxt + e] : 0.0;
        if (threadIdx.x == 0) {
            const uint32_t m = min((uint32_t)kSumChunk, n - ch * kSumChunk);
            const double* b = buf[ch & 1];
            for (uint32_t e = 0; e < m; ++e) acc += b[e];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = acc;
}

// Empty-cluster repair, one CTA (partition.cpp:117-139).  A repair never
// empties a cluster (the victim's cluster keeps >= 1 member), so the empty
// set is fixed up front and processed in ascending order; each repair is one
// block-wide argmin over (score, index) among keys whose cluster has >= 2.
constexpr int kRepairThreads = 1024;
__global__ void __launch_bounds__(kRepairThreads) km_repair_kernel(
        const float* keys, uint32_t n, uint32_t D, uint32_t* assign, double* score,
        uint32_t* counts, uint32_t C, unsigned long long* repairs) {
    __shared__ double red_s[kRepairThreads / 32];
    __shared__ uint32_t red_i[kRepairThreads / 32];
    __shared__ uint32_t victim_sh;
    __shared__ int any_sh;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t c0 = 0; c0 < C; c0 += kRepairThreads) {
        if (threadIdx.x == 0) any_sh = 0;
        __syncthreads();
        const uint32_t cm = c0 + threadIdx.x;
        if (cm < C && counts[cm] == 0) any_sh = 1;
        __syncthreads();
        if (!any_sh) continue;
        const uint32_t cend = min(C, c0 + kRepairThreads);
        for (uint32_t c = c0; c < cend; ++c) {
            if (counts[c] != 0) continue;  // uniform: counts[c] only changes below, after a sync
            double bs = INFINITY;
            uint32_t bi = n;
            for (uint32_t i = threadIdx.x; i < n; i += kRepairThreads) {
                if (counts[assign[i]] < 2) continue;
                const double s = score[i];
                if (s < bs) {  // ascending i per thread: first minimum kept
                    bs = s;
                    bi = i;
                }
            }
            for (int o = 16; o; o >>= 1) {
                const double os = __shfl_xor_sync(0xFFFFFFFFu, bs, o);
                const uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, bi, o);
                if (os < bs || (os == bs && oi < bi)) {
                    bs = os;
                    bi = oi;
                }
            }
            if (lane == 0) {
                red_s[warp] = bs;
                red_i[warp] = bi;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                double s = red_s[0];
                uint32_t v = red_i[0];
                for (int w = 1; w < kRepairThreads / 32; ++w)
                    if (red_s[w] < s || (red_s[w] == s && red_i[w] < v)) {
                        s = red_s[w];
                        v = red_i[w];
                    }
                // a victim exists iff some key sits in a cluster of >= 2; an
                // infinite score never occurs for finite keys and centroids
                if (v < n) {
                    counts[assign[v]]--;
                    assign[v] = c;
                    score[v] = row_norm(keys + (size_t)v * D, D);
                    counts[c] = 1;
                    if (repairs) atomicAdd(repairs, 1ull);
                }
                victim_sh = v;
            }
            __syncthreads();
            if (victim_sh >= n) break;  // no cluster can spare a member: later empties stay empty too
        }
    }
}

// normalize_row on a shared-memory row (partition.cpp:19-31); returns false
// (row untouched) for a zero row.  Thread 0 computes the norm sequentially.
__device__ bool normalize_row_smem(float* row, uint32_t D, float* inv_sh, int* ok_sh) {
    if (threadIdx.x == 0) {
        const double nrm = row_norm(row, D);
        *ok_sh = nrm != 0.0;
        *inv_sh = nrm != 0.0 ? (float)(1.0 / nrm) : 0.f;
    }
    __syncthreads();
    const bool ok = *ok_sh;
    if (ok)
        for (uint32_t j = threadIdx.x; j < D; j += blockDim.x) row[j] *= *inv_sh;
    __syncthreads();
    return ok;
}

// Seeding: centroid c = normalize(keys[seed[c]]); a zero seed keeps its
// (signed) zeros and gets 1.0 at c mod d (partition.cpp:84-89).
__global__ void km_seed_kernel(const float* keys, uint32_t D, const uint64_t* seed_rows,
                               float* cent) {
    extern __shared__ float row[];
    __shared__ float inv;
    __shared__ int ok;
    const uint32_t c = blockIdx.x;
    const float* src = keys + seed_rows[c] * D;
    for (uint32_t j = threadIdx.x; j < D; j += blockDim.x) row[j] = src[j];
    __syncthreads();
    if (!normalize_row_smem(row, D, &inv, &ok) && threadIdx.x == 0) row[c % D] = 1.0f;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < D; j += blockDim.x) cent[(size_t)c * D + j] = row[j];
}

// Update: one CTA per cluster; thread j sums component j over the members in
// ascending key order (idx from the stable counting sort), all f32 adds in the
// reference's order; then normalize_row, with the cancelled-sum fallback.
// Clusters left empty keep their centroid.
__global__ void km_update_kernel(const float* keys, uint32_t D, const uint32_t* off,
                                 const uint32_t* idx, float* cent) {
    extern __shared__ float row[];
    __shared__ float inv;
    __shared__ int ok;
    const uint32_t c = blockIdx.x;
    const uint32_t b = off[c], e = off[c + 1];
    if (b == e) return;
    for (uint32_t j = threadIdx.x; j < D; j += blockDim.x) {
        float s = 0.f;
        uint32_t m = b;
        constexpr int U = 8;
        for (; m + U <= e; m += U) {
            float v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = __ldg(keys + (size_t)idx[m + u] * D + j);
#pragma unroll
            for (int u = 0; u < U; ++u) s = __fadd_rn(s, v[u]);
        }
        for (; m < e; ++m) s = __fadd_rn(s, __ldg(keys + (size_t)idx[m] * D + j));
        row[j] = s;
    }
    __syncthreads();
    if (!normalize_row_smem(row, D, &inv, &ok)) {
        // members cancelled: the (zero) sums with 1.0 at c mod d, normalized
        if (threadIdx.x == 0) row[c % D] = 1.0f;
        __syncthreads();
        normalize_row_smem(row, D, &inv, &ok);
    }
    for (uint32_t j = threadIdx.x; j < D; j += blockDim.x) cent[(size_t)c * D + j] = row[j];
}

}  // namespace

uint32_t km_dim_max(uint32_t D) { return D <= 8 ? 8 : D <= 32 ? 32 : D <= 64 ? 64 : D <= 128 ? 128 : 0; }

void launch_km_assign(const float* keys, uint32_t n, uint32_t D, const float* cent, uint32_t C,
                      uint32_t* assign, double* score, unsigned long long* zero_keys,
                      cudaStream_t st) {
    const uint32_t grid = (n + kAssignThreads - 1) / kAssignThreads;
    if (!grid) return;
    switch (km_dim_max(D)) {
        case 8: km_assign_kernel<8><<<grid, kAssignThreads, 0, st>>>(keys, n, D, cent, C, assign, score, zero_keys); break;
        case 32: km_assign_kernel<32><<<grid, kAssignThreads, 0, st>>>(keys, n, D, cent, C, assign, score, zero_keys); break;
        case 64: km_assign_kernel<64><<<grid, kAssignThreads, 0, st>>>(keys, n, D, cent, C, assign, score, zero_keys); break;
        case 128: km_assign_kernel<128><<<grid, kAssignThreads, 0, st>>>(keys, n, D, cent, C, assign, score, zero_keys); break;
        default: fail(SAAP_ERR_UNSUPPORTED, "kmeans_train: unsupported key dim " + std::to_string(D));
    }
    SAAP_CUDA(cudaGetLastError());
}

void launch_km_iteration_tail(const float* keys, uint32_t n, uint32_t D, uint32_t* assign,
                              double* score, uint32_t* counts, uint32_t C,
                              unsigned long long* repairs, cudaStream_t st) {
    SAAP_CUDA(cudaMemsetAsync(counts, 0, (size_t)C * 4, st));
    km_count_kernel<<<148 * 4, 256, 0, st>>>(assign, n, counts);
    km_repair_kernel<<<1, kRepairThreads, 0, st>>>(keys, n, D, assign, score, counts, C, repairs);
    SAAP_CUDA(cudaGetLastError());
}

void launch_km_objective(const double* score, uint32_t n, double* out, cudaStream_t st) {
    km_objective_kernel<<<1, 256, 0, st>>>(score, n, out);
    SAAP_CUDA(cudaGetLastError());
}

static uint32_t row_threads(uint32_t D) { return std::min<uint32_t>(256, (D + 31) / 32 * 32); }

void launch_km_seed(const float* keys, uint32_t D, const uint64_t* seed_rows, uint32_t C,
                    float* cent, cudaStream_t st) {
    km_seed_kernel<<<C, row_threads(D), D * 4, st>>>(keys, D, seed_rows, cent);
    SAAP_CUDA(cudaGetLastError());
}

void launch_km_update(const float* keys, uint32_t D, const uint32_t* off, const uint32_t* idx,
                      uint32_t C, float* cent, cudaStream_t st) {
    km_update_kernel<<<C, row_threads(D), D * 4, st>>>(keys, D, off, idx, cent);
    SAAP_CUDA(cudaGetLastError());
}

}  // namespace saap_b200
