// Device Q-model training, bit-exact with the
// reference's fp64 manual backprop.  Compiled with -fmad=false: every fp64
// `a * b + c` below is a separately rounded multiply and add, exactly the
// reference's mulsd/addsd (it is built without FMA contraction).
//
// Reference (/root/reference/proj/core/src/qmodel.cpp):
//   mm / mm_at_b / mm_a_bt / col_sums   :30-106  (loop orders, zero skips)
//   softmax_rows_inplace                :108-125 (glibc exp, sequential total)
//   forward_pass (train)                :147-225 (batch mean / biased var)
//   update_running_stats                :227-235
//   kl_from_cache                       :237-257 (loss: CUDA log, not glibc)
//   backward_pass                       :260-305
//   adam_step                           :307-333 (bias corrections from host pow)
//   train_step_on_target                :419-433
//   attention_target_rows               :384-407
//
// Parallel shape: one thread per output element, the reduction index walked
// sequentially in the reference's order, so every sum rounds identically.
// The work per step is small (batch 64, hidden 1024, C <= 1024: ~0.2 GFLOP
// fp64); the kernels are latency-bound and the trainer keeps parameters,
// Adam moments and activations resident on the device between steps.
#include <cmath>
#include <string>
#include <vector>

#include "common.cuh"
#include "exp_glibc.cuh"


namespace saap_b200 {
namespace {

constexpr double kBnEps = 1e-5;
constexpr double kLogFloor = 1e-12;
constexpr int kT = 128;
constexpr int kU = 8;  // loads issued ahead of each sequential add chain
constexpr int kP = 16;  // weights per pipeline stage (two stages in flight)

// z[i][j] = (sum_k x[i][k] w1[k][j], k ascending, zero x skipped) + b1[j]
__global__ void qt_linear1(const float* q, uint32_t n, uint32_t d, uint32_t h, const double* w1,
                           const double* b1, double* x, double* z) {
    const uint32_t j = blockIdx.x * kT + threadIdx.x, i = blockIdx.y;
    if (blockIdx.x == 0)
        for (uint32_t k = threadIdx.x; k < d; k += kT) x[(size_t)i * d + k] = (double)q[(size_t)i * d + k];
    if (j >= h) return;
    // operands of 8 steps loaded ahead; the adds stay in k order
    double s = 0.0;
    uint32_t k = 0;
    for (; k + kU <= d; k += kU) {
        double a[kU], w[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            a[u] = (double)q[(size_t)i * d + k + u];
            w[u] = w1[(size_t)(k + u) * h + j];
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (a[u] != 0.0) s += a[u] * w[u];
    }
    for (; k < d; ++k) {
        const double a = (double)q[(size_t)i * d + k];
        if (a == 0.0) continue;
        s += a * w1[(size_t)k * h + j];
    }
    z[(size_t)i * h + j] = s + b1[j];
}

// batch mean / biased variance per hidden unit (rows in order), then the
// normalized activations
__global__ void qt_bn(const double* z, uint32_t n, uint32_t h, const double* gamma,
                      const double* beta, double* mean, double* var, double* xhat, double* y,
                      double* r) {
    const uint32_t j = blockIdx.x * kT + threadIdx.x;
    if (j >= h) return;
    double mu = 0.0;
    for (uint32_t i = 0; i < n; ++i) mu += z[(size_t)i * h + j];
    mu /= (double)n;
    double vr = 0.0;
    for (uint32_t i = 0; i < n; ++i) {
        const double dd = z[(size_t)i * h + j] - mu;
        vr += dd * dd;
    }
    vr /= (double)n;
    mean[j] = mu;
    var[j] = vr;
    const double inv_std = 1.0 / sqrt(vr + kBnEps);
    for (uint32_t i = 0; i < n; ++i) {
        const size_t o = (size_t)i * h + j;
        const double xh = (z[o] - mu) * inv_std;
        const double yy = gamma[j] * xh + beta[j];
        xhat[o] = xh;
        y[o] = yy;
        r[o] = yy > 0.0 ? yy : 0.0;
    }
}

// logits[i][c] = (sum_k r[i][k] w2[k][c], zero r skipped) + b2[c]
__global__ void qt_linear2(const double* r, uint32_t n, uint32_t h, uint32_t C, const double* w2,
                           const double* b2, double* out) {
    const uint32_t c = blockIdx.x * kT + threadIdx.x, i = blockIdx.y;
    if (c >= C) return;
    double s = 0.0;
    const double* rr = r + (size_t)i * h;
    // two stages of kP weights in flight ahead of the ordered chain
    const uint32_t kfull = h / kP * kP;
    double wa[kP], wb[kP];
    if (kfull) {
#pragma unroll
        for (int u = 0; u < kP; ++u) wa[u] = w2[(size_t)u * C + c];
    }
    uint32_t k = 0;
    for (; k < kfull; k += kP) {
        const bool more = k + kP < kfull;
#pragma unroll
        for (int u = 0; u < kP; ++u) wb[u] = more ? w2[(size_t)(k + kP + u) * C + c] : 0.0;
#pragma unroll
        for (int u = 0; u < kP; ++u) {
            const double a = rr[k + u];
            if (a != 0.0) s += a * wa[u];
        }
#pragma unroll
        for (int u = 0; u < kP; ++u) wa[u] = wb[u];
    }
    for (; k < h; ++k) {
        const double a = rr[k];
        if (a == 0.0) continue;
        s += a * w2[(size_t)k * C + c];
    }
    out[(size_t)i * C + c] = s + b2[c];
}

// softmax_rows_inplace on one row per CTA: max (order-free), glibc exp,
// sequential total by one thread, 1/total scaling
__global__ void qt_softmax_rows(double* a, uint32_t cols) {
    __shared__ double red[kT];
    __shared__ double s_tot;
    double* row = a + (size_t)blockIdx.x * cols;
    double mx = -INFINITY;
    for (uint32_t j = threadIdx.x; j < cols; j += kT) mx = fmax(mx, row[j]);
    red[threadIdx.x] = mx;
    __syncthreads();
    for (int o = kT / 2; o; o >>= 1) {
        if ((int)threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
        __syncthreads();
    }
    mx = red[0];
    for (uint32_t j = threadIdx.x; j < cols; j += kT) row[j] = exp_glibc(row[j] - mx);
    __syncthreads();
    if (threadIdx.x == 0) {  // loads run ahead of the ordered chain
        double t = 0.0;
        uint32_t j = 0;
        for (; j + kU <= cols; j += kU) {
            double v[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) v[u] = row[j + u];
#pragma unroll
            for (int u = 0; u < kU; ++u) t += v[u];
        }
        for (; j < cols; ++j) t += row[j];
        s_tot = 1.0 / t;
    }
    __syncthreads();
    const double inv = s_tot;
    for (uint32_t j = threadIdx.x; j < cols; j += kT) row[j] *= inv;
}

// KL(target || p) per row (CUDA log; the loss is reported, not differentiated)
__global__ void qt_kl_rows(const double* p, const double* t, uint32_t C, double* rows) {
    __shared__ double red[kT];
    const size_t o = (size_t)blockIdx.x * C;
    double s = 0.0;
    for (uint32_t j = threadIdx.x; j < C; j += kT) {
        const double tv = t[o + j];
        if (tv > 0.0) s += tv * (log(tv) - log(fmax(p[o + j], kLogFloor)));
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int k = kT / 2; k; k >>= 1) {
        if ((int)threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0) rows[blockIdx.x] = red[0];
}

__global__ void qt_kl_total(const double* rows, uint32_t n, double* out) {
    double s = 0.0;
    for (uint32_t i = 0; i < n; ++i) s += rows[i];
    *out = s / (double)n;
}

// dlogits = (p - t) / n; col sums -> g.b2 (rows in order)
__global__ void qt_dlogits(const double* p, const double* t, uint32_t n, uint32_t C, double* dl,
                           double* gb2) {
    const uint32_t c = blockIdx.x * kT + threadIdx.x;
    if (c >= C) return;
    const double inv_n = 1.0 / (double)n;
    double s = 0.0;
    for (uint32_t i = 0; i < n; ++i) {
        const size_t o = (size_t)i * C + c;
        const double v = (p[o] - t[o]) * inv_n;
        dl[o] = v;
        s += v;
    }
    gb2[c] = s;
}

// out[k][j] = sum_i a[i][k] b[i][j] (mm_at_b: i ascending, zero a skipped)
__global__ void qt_at_b(const double* a, const double* b, uint32_t n, uint32_t K, uint32_t M,
                        double* out) {
    const uint32_t j = blockIdx.x * kT + threadIdx.x, k = blockIdx.y;
    if (j >= M) return;
    double s = 0.0;
    uint32_t i = 0;
    for (; i + kU <= n; i += kU) {
        double av[kU], bv[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            av[u] = a[(size_t)(i + u) * K + k];
            bv[u] = b[(size_t)(i + u) * M + j];
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (av[u] != 0.0) s += av[u] * bv[u];
    }
    for (; i < n; ++i) {
        const double av = a[(size_t)i * K + k];
        if (av == 0.0) continue;
        s += av * b[(size_t)i * M + j];
    }
    out[(size_t)k * M + j] = s;
}

// w2T[c][j] = w2[j][c] (coalesced reads for mm_a_bt)
__global__ void qt_transpose(const double* w2, uint32_t h, uint32_t C, double* w2T) {
    __shared__ double t[32][33];
    const uint32_t c0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
    for (uint32_t y = threadIdx.y; y < 32; y += blockDim.y)
        if (j0 + y < h && c0 + threadIdx.x < C) t[y][threadIdx.x] = w2[(size_t)(j0 + y) * C + c0 + threadIdx.x];
    __syncthreads();
    for (uint32_t y = threadIdx.y; y < 32; y += blockDim.y)
        if (c0 + y < C && j0 + threadIdx.x < h) w2T[(size_t)(c0 + y) * h + j0 + threadIdx.x] = t[threadIdx.x][y];
}

// dy[i][j] = sum_c dl[i][c] w2[j][c] (mm_a_bt: s = 0, c ascending, no skip),
// masked where y <= 0
__global__ void qt_dy(const double* dl, const double* w2T, const double* y, uint32_t h, uint32_t C,
                      double* dy) {
    const uint32_t j = blockIdx.x * kT + threadIdx.x, i = blockIdx.y;
    if (j >= h) return;
    const double* dr = dl + (size_t)i * C;
    double s = 0.0;
    const uint32_t cfull = C / kP * kP;
    double wa[kP], wb[kP];
    if (cfull) {
#pragma unroll
        for (int u = 0; u < kP; ++u) wa[u] = w2T[(size_t)u * h + j];
    }
    uint32_t c = 0;
    for (; c < cfull; c += kP) {
        const bool more = c + kP < cfull;
#pragma unroll
        for (int u = 0; u < kP; ++u) wb[u] = more ? w2T[(size_t)(c + kP + u) * h + j] : 0.0;
#pragma unroll
        for (int u = 0; u < kP; ++u) s += dr[c + u] * wa[u];
#pragma unroll
        for (int u = 0; u < kP; ++u) wa[u] = wb[u];
    }
    for (; c < C; ++c) s += dr[c] * w2T[(size_t)c * h + j];
    const size_t o = (size_t)i * h + j;
    dy[o] = y[o] <= 0.0 ? 0.0 : s;
}

// g.gamma, g.beta (rows in order), then dz
__global__ void qt_bn_back(const double* dy, const double* xhat, const double* gamma,
                           const double* var, uint32_t n, uint32_t h, double* ggamma, double* gbeta,
                           double* dz) {
    const uint32_t j = blockIdx.x * kT + threadIdx.x;
    if (j >= h) return;
    double sg = 0.0, sb = 0.0;
    for (uint32_t i = 0; i < n; ++i) {
        const size_t o = (size_t)i * h + j;
        sg += dy[o] * xhat[o];
        sb += dy[o];
    }
    ggamma[j] = sg;
    gbeta[j] = sb;
    const double inv_n = 1.0 / (double)n;
    const double scale = gamma[j] / sqrt(var[j] + kBnEps);
    const double mean_dy = sb * inv_n, mean_dy_xhat = sg * inv_n;
    for (uint32_t i = 0; i < n; ++i) {
        const size_t o = (size_t)i * h + j;
        dz[o] = scale * (dy[o] - mean_dy - xhat[o] * mean_dy_xhat);
    }
}

__global__ void qt_col_sums(const double* a, uint32_t n, uint32_t M, double* out) {
    const uint32_t j = blockIdx.x * kT + threadIdx.x;
    if (j >= M) return;
    double s = 0.0;
    for (uint32_t i = 0; i < n; ++i) s += a[(size_t)i * M + j];
    out[j] = s;
}

__global__ void qt_running(double* rmean, double* rvar, const double* mean, const double* var,
                           uint32_t h, double mom) {
    const uint32_t j = blockIdx.x * kT + threadIdx.x;
    if (j >= h) return;
    rmean[j] = mom * rmean[j] + (1.0 - mom) * mean[j];
    rvar[j] = mom * rvar[j] + (1.0 - mom) * var[j];
}

__global__ void qt_adam(double* p, double* m, double* v, const double* g, uint64_t cnt, double b1,
                        double b2, double bc1, double bc2, double lr, double eps) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double gi = g[i];
        const double mi = b1 * m[i] + (1.0 - b1) * gi;
        const double vi = b2 * v[i] + (1.0 - b2) * gi * gi;
        m[i] = mi;
        v[i] = vi;
        const double mhat = mi / bc1, vhat = vi / bc2;
        p[i] -= lr * mhat / (sqrt(vhat) + eps);
    }
}

// attention_target_rows: a[i][k] = scale * dot_f(q_i, k_k); row softmax;
// target[i][b] += a[i][k] over k ascending.  One CTA per query row; the
// scatter-add is walked by one thread in key order (target row in smem).
__global__ void qt_target_logits(const float* q, const float* K, uint32_t n_keys, uint32_t d,
                                 double scale, double* a) {
    const uint32_t k = blockIdx.x * kT + threadIdx.x, i = blockIdx.y;
    if (k >= n_keys) return;
    double s = 0.0;
    for (uint32_t j = 0; j < d; ++j) s += (double)q[(size_t)i * d + j] * (double)K[(size_t)k * d + j];
    a[(size_t)i * n_keys + k] = scale * s;
}

__global__ void qt_target_scatter(const double* a, uint32_t n_keys, const uint32_t* assign,
                                  uint32_t C, double* out) {
    extern __shared__ double trow[];
    for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) trow[c] = 0.0;
    __syncthreads();
    const double* ar = a + (size_t)blockIdx.x * n_keys;
    if (threadIdx.x == 0)
        for (uint32_t k = 0; k < n_keys; ++k) trow[assign[k]] += ar[k];
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) out[(size_t)blockIdx.x * C + c] = trow[c];
}

inline dim3 g1(uint64_t n) { return dim3((uint32_t)((n + kT - 1) / kT)); }

}  // namespace

// train_step_on_target, part 1: train-mode forward and the loss.
void qtrain_forward(saap_qtrainer* t, uint32_t n, cudaStream_t st) {
    const uint32_t d = (uint32_t)t->d, h = (uint32_t)t->h, C = (uint32_t)t->C;
    qt_linear1<<<dim3(g1(h).x, n), kT, 0, st>>>(t->q32, n, d, h, t->p[0], t->p[1], t->x, t->z);
    qt_bn<<<g1(h), kT, 0, st>>>(t->z, n, h, t->p[2], t->p[3], t->mean, t->var, t->xhat, t->y, t->r);
    qt_linear2<<<dim3(g1(C).x, n), kT, 0, st>>>(t->r, n, h, C, t->p[6], t->p[7], t->pr);
    qt_softmax_rows<<<n, kT, 0, st>>>(t->pr, C);
    qt_kl_rows<<<n, kT, 0, st>>>(t->pr, t->tgt, C, t->loss_rows);
    qt_kl_total<<<1, 1, 0, st>>>(t->loss_rows, n, t->loss);
    SAAP_CUDA(cudaGetLastError());
}

// Part 2 (after the loss was found finite): backward, running stats, Adam.
void qtrain_update(saap_qtrainer* t, uint32_t n, cudaStream_t st) {
    const uint32_t d = (uint32_t)t->d, h = (uint32_t)t->h, C = (uint32_t)t->C;
    double *gam = t->p[2], *rm = t->p[4], *rv = t->p[5], *w2 = t->p[6];
    // grads in param_refs order: w1, b1, gamma, beta, w2, b2 (g[0..1], g[2..3], g[6..7])
    qt_dlogits<<<g1(C), kT, 0, st>>>(t->pr, t->tgt, n, C, t->dl, t->g[7]);
    qt_at_b<<<dim3(g1(C).x, h), kT, 0, st>>>(t->r, t->dl, n, h, C, t->g[6]);
    qt_transpose<<<dim3((C + 31) / 32, (h + 31) / 32), dim3(32, 8), 0, st>>>(w2, h, C, t->w2T);
    qt_dy<<<dim3(g1(h).x, n), kT, 0, st>>>(t->dl, t->w2T, t->y, h, C, t->dy);
    qt_bn_back<<<g1(h), kT, 0, st>>>(t->dy, t->xhat, gam, t->var, n, h, t->g[2], t->g[3], t->dz);
    qt_at_b<<<dim3(g1(h).x, d), kT, 0, st>>>(t->x, t->dz, n, d, h, t->g[0]);
    qt_col_sums<<<g1(h), kT, 0, st>>>(t->dz, n, h, t->g[1]);
    qt_running<<<g1(h), kT, 0, st>>>(rm, rv, t->mean, t->var, h, t->bn_momentum);
    t->step++;
    const double bc1 = 1.0 - std::pow(t->beta1, (double)t->step);
    const double bc2 = 1.0 - std::pow(t->beta2, (double)t->step);
    const uint64_t cnt[8] = {(uint64_t)d * h, h, h, h, 0, 0, (uint64_t)h * C, C};
    for (int k : {0, 1, 2, 3, 6, 7})
        qt_adam<<<(uint32_t)std::min<uint64_t>(148 * 8, (cnt[k] + 255) / 256), 256, 0, st>>>(
                t->p[k], t->m[k], t->v[k], t->g[k], cnt[k], t->beta1, t->beta2, bc1, bc2, t->lr,
                t->eps);
    SAAP_CUDA(cudaGetLastError());
}

void launch_attention_target(const float* q, uint32_t n, uint32_t d, const float* K,
                             uint32_t n_keys, const uint32_t* assign, uint32_t C, double* a,
                             double* out, cudaStream_t st) {
    const double scale = 1.0 / std::sqrt((double)d);
    qt_target_logits<<<dim3(g1(n_keys).x, n), kT, 0, st>>>(q, K, n_keys, d, scale, a);
    qt_softmax_rows<<<n, kT, 0, st>>>(a, n_keys);
    const size_t smem = (size_t)C * 8;
    if (smem > 48 * 1024)
        SAAP_CUDA(cudaFuncSetAttribute(qt_target_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    qt_target_scatter<<<n, kT, smem, st>>>(a, n_keys, assign, C, out);
    SAAP_CUDA(cudaGetLastError());
}

}  // namespace saap_b200
