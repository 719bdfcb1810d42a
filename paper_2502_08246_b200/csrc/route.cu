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
constexpr int kQmP = 16;    // logits: weights per pipeline stage (two stages in flight)

// The forward pass runs as three grids so a step's 64 (context) rows of work
// spread over the SMs: hidden units (one thread per (row block, unit)),
// logits (one thread per (row block, bucket)), then one CTA per row for the
// softmax.  Every chain keeps the reference's order; loads run ahead of it.
constexpr int kQmT = 128;

template <bool SKIP0>
__global__ void __launch_bounds__(kQmT) qm_hidden_kernel(QModelArgs a) {
    extern __shared__ __align__(16) double xs[];  // kQmRows x d
    const uint32_t g = blockIdx.x, j = blockIdx.y * kQmT + threadIdx.x;
    const double* w1 = a.prm[3 * g + 0];
    const double* vec = a.prm[3 * g + 2];
    const double *b1 = vec, *gamma = vec + a.h, *beta = vec + 2 * a.h, *mean = vec + 3 * a.h,
                 *var = vec + 4 * a.h;
    for (uint32_t i0 = 0; i0 < a.G; i0 += kQmRows) {
        const uint32_t nr = min((uint32_t)kQmRows, a.G - i0);
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < nr * a.d; e += kQmT)
            xs[e] = (double)a.q[((size_t)g * a.G + i0) * a.d + e];
        __syncthreads();
        if (j >= a.h) continue;
        double z[kQmRows];
#pragma unroll
        for (int i = 0; i < kQmRows; ++i) z[i] = 0.0;
        constexpr int P = kQmP;  // two stages of W1 loads in flight
        const uint32_t kfull = a.d / P * P;
        double wa[P], wb[P];
        if (kfull) {
#pragma unroll
            for (int u = 0; u < P; ++u) wa[u] = w1[(size_t)u * a.h + j];
        }
        uint32_t k = 0;
        for (; k < kfull; k += P) {
            const bool more = k + P < kfull;
#pragma unroll
            for (int u = 0; u < P; ++u) wb[u] = more ? w1[(size_t)(k + P + u) * a.h + j] : 0.0;
#pragma unroll
            for (int u = 0; u < P; ++u)
#pragma unroll
                for (int i = 0; i < kQmRows; ++i) {
                    const double av = xs[i * a.d + k + u];
                    if (SKIP0) {
                        if ((uint32_t)i < nr && av != 0.0) z[i] = __dadd_rn(z[i], __dmul_rn(av, wa[u]));
                    } else {
                        z[i] = __dadd_rn(z[i], __dmul_rn(av, wa[u]));
                    }
                }
#pragma unroll
            for (int u = 0; u < P; ++u) wa[u] = wb[u];
        }
        for (; k < a.d; ++k) {
            const double w = w1[(size_t)k * a.h + j];
#pragma unroll
            for (int i = 0; i < kQmRows; ++i) {
                const double av = xs[i * a.d + k];
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
            a.hid[((size_t)g * a.G + i0 + i) * a.h + j] = y > 0.0 ? y : 0.0;
        }
    }
}

// logits = r W2 + b2.  CTA (slot, bucket block, row block): ROWS query rows
// of the slot (contexts sharing the model) x TL buckets; each W2 load feeds
// ROWS ordered chains, and the next P weights load while these are used.
template <int ROWS, int P, int TL, bool SKIP0>
__global__ void __launch_bounds__(TL) qm_logits_kernel(QModelArgs a) {
    extern __shared__ __align__(16) double rs[];  // ROWS x h
    const uint32_t slot = blockIdx.x, c = blockIdx.y * TL + threadIdx.x;
    const uint32_t* sg = a.slot_g ? a.slot_g + (size_t)slot * kQmSlot : nullptr;
    uint32_t ng = 1;
    if (sg)
        while (ng < kQmSlot && sg[ng] != 0xFFFFFFFFu) ++ng;
    const uint32_t g0 = sg ? sg[0] : slot;
    const double* w2 = a.prm[3 * g0 + 1];
    const double* b2 = a.prm[3 * g0 + 2] + 5 * a.h;
    const uint32_t R = ng * a.G;
    auto row_of = [&](uint32_t r) -> size_t {  // slot row -> (context, query row)
        const uint32_t g = sg ? sg[r / a.G] : slot;
        return (size_t)g * a.G + r % a.G;
    };
    for (uint32_t r0 = blockIdx.z * ROWS; r0 < R; r0 += gridDim.z * ROWS) {
        const uint32_t nr = min((uint32_t)ROWS, R - r0);
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < nr * a.h; e += TL)
            rs[e] = a.hid[row_of(r0 + e / a.h) * a.h + e % a.h];
        __syncthreads();
        if (c >= a.C) continue;
        double s[ROWS];
#pragma unroll
        for (int i = 0; i < ROWS; ++i) s[i] = 0.0;
        const uint32_t kfull = a.h / P * P;
        double wa[P], wb[P];
        if (kfull) {
#pragma unroll
            for (int u = 0; u < P; ++u) wa[u] = w2[(size_t)u * a.C + c];
        }
        uint32_t k = 0;
        for (; k < kfull; k += P) {
            const bool more = k + P < kfull;
#pragma unroll
            for (int u = 0; u < P; ++u) wb[u] = more ? w2[(size_t)(k + P + u) * a.C + c] : 0.0;
#pragma unroll
            for (int u = 0; u < P; ++u)
#pragma unroll
                for (int i = 0; i < ROWS; ++i) {
                    const double av = rs[i * a.h + k + u];
                    if (SKIP0) {
                        if ((uint32_t)i < nr && av != 0.0) s[i] = __dadd_rn(s[i], __dmul_rn(av, wa[u]));
                    } else {
                        s[i] = __dadd_rn(s[i], __dmul_rn(av, wa[u]));
                    }
                }
#pragma unroll
            for (int u = 0; u < P; ++u) wa[u] = wb[u];
        }
        for (; k < a.h; ++k) {
            const double w = w2[(size_t)k * a.C + c];
#pragma unroll
            for (int i = 0; i < ROWS; ++i) {
                const double av = rs[i * a.h + k];
                if ((uint32_t)i < nr && av != 0.0) s[i] = __dadd_rn(s[i], __dmul_rn(av, w));
            }
        }
#pragma unroll
        for (int i = 0; i < ROWS; ++i)
            if ((uint32_t)i < nr) a.probs[row_of(r0 + i) * a.C + c] = __dadd_rn(s[i], b2[c]);
    }
}

template <int ROWS, int P, int TL, bool SKIP0 = true>
static void launch_qm_logits(const QModelArgs& a, uint32_t n_slots, cudaStream_t st) {
    const size_t sm = (size_t)ROWS * a.h * sizeof(double);
    static size_t cfg = 0;
    if (sm > 48 * 1024 && sm > cfg) {
        SAAP_CUDA(cudaFuncSetAttribute(qm_logits_kernel<ROWS, P, TL, SKIP0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sm));
        cfg = sm;
    }
    const uint32_t rows = (a.slot_g ? kQmSlot : 1u) * a.G;
    qm_logits_kernel<ROWS, P, TL, SKIP0><<<dim3(n_slots, (a.C + TL - 1) / TL, (rows + ROWS - 1) / ROWS), TL, sm, st>>>(a);
}

// softmax_rows_inplace on one (context, row): max (order-free), glibc exp,
// one sequential denominator (qmodel.cpp:108-125)
__global__ void __launch_bounds__(256) qm_softmax_kernel(QModelArgs a) {
    __shared__ double red[8];
    __shared__ double s_inv;
    extern __shared__ double ex[];  // the row's exps: the ordered sum reads shared memory
    double* row = a.probs + (size_t)blockIdx.x * a.C;
    double mx = -INFINITY;
    for (uint32_t c = threadIdx.x; c < a.C; c += blockDim.x) mx = fmax(mx, row[c]);
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = red[0];
    for (int w = 1; w < 8; ++w) mx = fmax(mx, red[w]);
    for (uint32_t c = threadIdx.x; c < a.C; c += blockDim.x) ex[c] = exp_glibc(__dadd_rn(row[c], -mx));
    __syncthreads();
    if (threadIdx.x == 0) {  // loads run ahead of the ordered chain
        double t = 0.0;
        uint32_t c = 0;
        for (; c + 8 <= a.C; c += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = ex[c + u];
#pragma unroll
            for (int u = 0; u < 8; ++u) t = __dadd_rn(t, v[u]);
        }
        for (; c < a.C; ++c) t = __dadd_rn(t, ex[c]);
        s_inv = __ddiv_rn(1.0, t);
    }
    __syncthreads();
    const double inv = s_inv;
    for (uint32_t c = threadIdx.x; c < a.C; c += blockDim.x) row[c] = __dmul_rn(ex[c], inv);
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

void launch_qmodel_probs(const QModelArgs& a, uint32_t n_groups, cudaStream_t st, uint32_t n_slots) {
    const size_t sm1 = (size_t)kQmRows * a.d * sizeof(double);
    static size_t cfg1 = 0;
    if (sm1 > 48 * 1024 && sm1 > cfg1) {
        SAAP_CUDA(cudaFuncSetAttribute(qm_hidden_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
        SAAP_CUDA(cudaFuncSetAttribute(qm_hidden_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
        cfg1 = sm1;
    }
    if (a.w_finite) qm_hidden_kernel<false><<<dim3(n_groups, (a.h + kQmT - 1) / kQmT), kQmT, sm1, st>>>(a);
    else qm_hidden_kernel<true><<<dim3(n_groups, (a.h + kQmT - 1) / kQmT), kQmT, sm1, st>>>(a);
    // logits geometry (a.logits_variant): rows per thread x CTA width
    const uint32_t ns = a.slot_g ? n_slots : n_groups;
    switch (a.logits_variant) {
        case 0:  // default: without the zero-skip test when the weights are finite (same sums)
            if (a.w_finite) launch_qm_logits<4, 16, 256, false>(a, ns, st);
            else launch_qm_logits<8, 16, 256>(a, ns, st);
            break;
        case 1: launch_qm_logits<2, 16, 256, false>(a, ns, st); break;
        case 2: launch_qm_logits<4, 8, 256, false>(a, ns, st); break;
        case 3: launch_qm_logits<4, 16, 128, false>(a, ns, st); break;
        case 4: launch_qm_logits<8, 16, 128, false>(a, ns, st); break;
        case 5: launch_qm_logits<4, 32, 256, false>(a, ns, st); break;
        case 6: launch_qm_logits<8, 16, 256, false>(a, ns, st); break;
        case 7: launch_qm_logits<4, 16, 256, false>(a, ns, st); break;
        default: launch_qm_logits<8, 16, 256>(a, ns, st); break;
    }
    const size_t sm3 = (size_t)a.C * sizeof(double);
    static size_t cfg3 = 0;
    if (sm3 > 48 * 1024 && sm3 > cfg3) {
        SAAP_CUDA(cudaFuncSetAttribute(qm_softmax_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3));
        cfg3 = sm3;
    }
    qm_softmax_kernel<<<n_groups * a.G, 256, sm3, st>>>(a);
    SAAP_CUDA(cudaGetLastError());
}

}  // namespace saap_b200
