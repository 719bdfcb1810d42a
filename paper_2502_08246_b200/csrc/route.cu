// Q-model router (SAAP's learned query->bucket classifier), eval mode, fp64.
//
// Reference: forward_pass (eval) qmodel.cpp:147-225, mm qmodel.cpp:30-51,
// softmax_rows_inplace qmodel.cpp:108-125, batched_bucket_select
// qmodel.cpp:485-511.  Every output is a sequential fp64 chain in the
// reference's index order with multiplies rounded before adds (__dmul_rn /
// __dadd_rn: nvcc would otherwise contract to DFMA), BN uses IEEE sqrt and
// division, and the softmax denominator is one sequential sum.  The
// per-row probabilities go to global memory; route_plan_kernel sums them over
// the group rows in order and selects the top-l.
#include "args.cuh"
#include "exp_glibc.cuh"

namespace saap_b200 {



constexpr int kQmRows = 4;  // group rows per pass (one W2 sweep per 4 rows)
constexpr int kQmU = 8;     // weight loads issued ahead of the ordered chains

__global__ void __launch_bounds__(1024) qmodel_probs_kernel(QModelArgs a) {
    extern __shared__ __align__(16) double qsm[];
    const uint32_t g = blockIdx.x;
    const double* w1 = a.prm[3 * g + 0];
    const double* w2 = a.prm[3 * g + 1];
    const double* vec = a.prm[3 * g + 2];
    const double* b1 = vec;
    const double* gamma = vec + a.h;
    const double* beta = vec + 2 * a.h;
    const double* mean = vec + 3 * a.h;
    const double* var = vec + 4 * a.h;
    const double* b2 = vec + 5 * a.h;
    double* x = qsm;                      // kQmRows x d
    double* r = x + kQmRows * a.d;        // kQmRows x h
    double* lg = r + kQmRows * a.h;       // kQmRows x C
    __shared__ double red[32][kQmRows];
    __shared__ double s_tot[kQmRows], s_max[kQmRows];

    for (uint32_t i0 = 0; i0 < a.G; i0 += kQmRows) {
        const uint32_t nr = min((uint32_t)kQmRows, a.G - i0);
        for (uint32_t e = threadIdx.x; e < nr * a.d; e += blockDim.x)
            x[e] = (double)a.q[((size_t)g * a.G + i0) * a.d + e];
        __syncthreads();
        // hidden layer: z = x W1 (+ b1), BN(running stats), ReLU
        for (uint32_t j = threadIdx.x; j < a.h; j += blockDim.x) {
            double z[kQmRows];
#pragma unroll
            for (int i = 0; i < kQmRows; ++i) z[i] = 0.0;
            // weights of kQmU steps in flight; the chains still add in k order
            uint32_t k = 0;
            for (; k + kQmU <= a.d; k += kQmU) {
                double w[kQmU];
#pragma unroll
                for (int u = 0; u < kQmU; ++u) w[u] = w1[(size_t)(k + u) * a.h + j];
#pragma unroll
                for (int u = 0; u < kQmU; ++u)
#pragma unroll
                    for (int i = 0; i < kQmRows; ++i) {
                        const double av = x[i * a.d + k + u];
                        if ((uint32_t)i < nr && av != 0.0) z[i] = __dadd_rn(z[i], __dmul_rn(av, w[u]));
                    }
            }
            for (; k < a.d; ++k) {
                const double w = w1[(size_t)k * a.h + j];
#pragma unroll
                for (int i = 0; i < kQmRows; ++i) {
                    const double av = x[i * a.d + k];
                    if ((uint32_t)i < nr && av != 0.0) z[i] = __dadd_rn(z[i], __dmul_rn(av, w));
                }
            }
            const double inv_std = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(var[j], 1e-5)));
#pragma unroll
            for (int i = 0; i < kQmRows; ++i) {
                if ((uint32_t)i >= nr) continue;
                const double zz = __dadd_rn(z[i], b1[j]);
                const double xh = __dmul_rn(__dadd_rn(zz, -mean[j]), inv_std);
                const double y = __dadd_rn(__dmul_rn(gamma[j], xh), beta[j]);
                r[i * a.h + j] = y > 0.0 ? y : 0.0;
            }
        }
        __syncthreads();
        // logits = r W2 (+ b2)
        double mx[kQmRows];
#pragma unroll
        for (int i = 0; i < kQmRows; ++i) mx[i] = -INFINITY;
        for (uint32_t c = threadIdx.x; c < a.C; c += blockDim.x) {
            double s[kQmRows];
#pragma unroll
            for (int i = 0; i < kQmRows; ++i) s[i] = 0.0;
            uint32_t k = 0;
            for (; k + kQmU <= a.h; k += kQmU) {
                double w[kQmU];
#pragma unroll
                for (int u = 0; u < kQmU; ++u) w[u] = w2[(size_t)(k + u) * a.C + c];
#pragma unroll
                for (int u = 0; u < kQmU; ++u)
#pragma unroll
                    for (int i = 0; i < kQmRows; ++i) {
                        const double av = r[i * a.h + k + u];
                        if ((uint32_t)i < nr && av != 0.0) s[i] = __dadd_rn(s[i], __dmul_rn(av, w[u]));
                    }
            }
            for (; k < a.h; ++k) {
                const double w = w2[(size_t)k * a.C + c];
#pragma unroll
                for (int i = 0; i < kQmRows; ++i) {
                    const double av = r[i * a.h + k];
                    if ((uint32_t)i < nr && av != 0.0) s[i] = __dadd_rn(s[i], __dmul_rn(av, w));
                }
            }
#pragma unroll
            for (int i = 0; i < kQmRows; ++i) {
                s[i] = __dadd_rn(s[i], b2[c]);
                lg[i * a.C + c] = s[i];
                mx[i] = fmax(mx[i], s[i]);
            }
        }
        // row max (order-free)
        const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
        for (int i = 0; i < kQmRows; ++i) {
            double v = mx[i];
            for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
            if (lane == 0) red[warp][i] = v;
        }
        __syncthreads();
        if (threadIdx.x < kQmRows) {
            double v = -INFINITY;
            for (uint32_t w = 0; w < blockDim.x / 32; ++w) v = fmax(v, red[w][threadIdx.x]);
            s_max[threadIdx.x] = v;
        }
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < nr * a.C; e += blockDim.x) {
            const uint32_t i = e / a.C;
            lg[e] = exp_glibc(__dadd_rn(lg[e], -s_max[i]));
        }
        __syncthreads();
        // denominator: one sequential chain per row (qmodel.cpp:116-119)
        if (threadIdx.x < nr) {
            double t = 0.0;
            const double* row = lg + threadIdx.x * a.C;
            for (uint32_t c = 0; c < a.C; ++c) t = __dadd_rn(t, row[c]);
            s_tot[threadIdx.x] = __ddiv_rn(1.0, t);
        }
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < nr * a.C; e += blockDim.x) {
            const uint32_t i = e / a.C;
            a.probs[((size_t)g * a.G + i0 + i) * a.C + (e % a.C)] = __dmul_rn(lg[e], s_tot[i]);
        }
        __syncthreads();
    }
}

__global__ void debug_exp_kernel(const double* x, uint64_t n, double* y) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        y[i] = exp_glibc(x[i]);
}

void launch_debug_exp(const double* x, uint64_t n, double* y, cudaStream_t st) {
    if (!n) return;
    debug_exp_kernel<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 4096), 256, 0, st>>>(x, n, y);
    SAAP_CUDA(cudaGetLastError());
}

void launch_qmodel_probs(const QModelArgs& a, uint32_t n_groups, cudaStream_t st) {
    const size_t smem = (size_t)kQmRows * (a.d + a.h + a.C) * sizeof(double);
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        SAAP_CUDA(cudaFuncSetAttribute(qmodel_probs_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    qmodel_probs_kernel<<<n_groups, 1024, smem, st>>>(a);
    SAAP_CUDA(cudaGetLastError());
}

}  // namespace saap_b200
