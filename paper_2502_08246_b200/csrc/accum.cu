// Partial-attention accumulators: the reference's
// online-softmax state and its absorb / merge / finalize operations, on the
// device in fp64 and bit-exact with the reference (glibc-exact exp port,
// reference loop orders, unfused multiplies and adds).
//
// Reference (/root/reference/proj/core/src/attention.cpp):
//   PartialAccumulator          attention.hpp:30-39, ctor :82-83
//   absorb_impl                 :34-78   (scores, rescale, ordered sums)
//   pattn_absorb / _range       :85-100
//   merge_into / merge_partials :102-139
//   pattn_finalize              :141-161
//   attention_over_ids          :197-203
#include "common.cuh"
#include "exp_glibc.cuh"

namespace saap_b200 {
namespace {

constexpr int kAT = 256;

// std::max(a, b): b only if a < b (keeps a on ties and signed zeros)
__device__ __forceinline__ double std_max(double a, double b) { return a < b ? b : a; }

// s[h][j] = dot_f(q_h, k_j) * scale: fp64 chain over d in index order (f32 x
// f32 products are exact in fp64), then one multiply
__global__ void __launch_bounds__(kAT) acc_scores_kernel(const float* q, const float* K, uint32_t n,
                                                         uint32_t d, double scale, double* S) {
    const uint32_t j = blockIdx.x * kAT + threadIdx.x, h = blockIdx.y;
    if (j >= n) return;
    const float* qh = q + (size_t)h * d;
    const float* kj = K + (size_t)j * d;
    double s = 0.0;
    for (uint32_t t = 0; t < d; ++t) s = __dadd_rn(s, __dmul_rn((double)qh[t], (double)kj[t]));
    S[(size_t)h * n + j] = __dmul_rn(s, scale);
}

// Per head: row max, new running max, rescale factor, weights w_j and the
// ordered denominator; the running state's scalars are updated here.
__global__ void __launch_bounds__(kAT) acc_weights_kernel(double* S, uint32_t n, double* sumexp,
                                                          double* runmax, double* rescale) {
    __shared__ double red[kAT / 32];
    __shared__ double s_m;
    const uint32_t h = blockIdx.x;
    double* sh = S + (size_t)h * n;
    double mx = -INFINITY;
    for (uint32_t j = threadIdx.x; j < n; j += kAT) mx = fmax(mx, sh[j]);
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = red[0];
        for (int w = 1; w < kAT / 32; ++w) m = fmax(m, red[w]);
        s_m = std_max(runmax[h], m);  // std::max(acc.runmax, rowmax)
    }
    __syncthreads();
    const double m_new = s_m;
    for (uint32_t j = threadIdx.x; j < n; j += kAT) sh[j] = exp_glibc(__dadd_rn(sh[j], -m_new));
    __syncthreads();
    if (threadIdx.x == 0) {
        const double r = exp_glibc(__dadd_rn(runmax[h], -m_new));  // 0 for a fresh head
        double se = __dmul_rn(sumexp[h], r);
        for (uint32_t j = 0; j < n; ++j) se = __dadd_rn(se, sh[j]);
        sumexp[h] = se;
        runmax[h] = m_new;
        rescale[h] = r;
    }
}

// out[h][t] = out[h][t] * rescale, then + w_j * v_j[t] for j in order
__global__ void __launch_bounds__(kAT) acc_values_kernel(const double* W, const float* V, uint32_t n,
                                                         uint32_t dv, const double* rescale, double* out) {
    const uint32_t t = blockIdx.x * kAT + threadIdx.x, h = blockIdx.y;
    if (t >= dv) return;
    const double* wh = W + (size_t)h * n;
    double o = __dmul_rn(out[(size_t)h * dv + t], rescale[h]);
    for (uint32_t j = 0; j < n; ++j) o = __dadd_rn(o, __dmul_rn(wh[j], (double)V[(size_t)j * dv + t]));
    out[(size_t)h * dv + t] = o;
}

// merge_into, one CTA per head: empty part = identity, empty acc = copy,
// else rescale both to the larger running max and add
__global__ void __launch_bounds__(kAT) acc_merge_kernel(double* out, double* sumexp, double* runmax,
                                                        const double* p_out, const double* p_sumexp,
                                                        const double* p_runmax, uint32_t dv) {
    const uint32_t h = blockIdx.x;
    const double se = sumexp[h], ps = p_sumexp[h], rm = runmax[h], pm = p_runmax[h];
    __syncthreads();
    if (ps == 0.0) return;
    double* dst = out + (size_t)h * dv;
    const double* src = p_out + (size_t)h * dv;
    if (se == 0.0) {
        for (uint32_t t = threadIdx.x; t < dv; t += kAT) dst[t] = src[t];
        if (threadIdx.x == 0) {
            sumexp[h] = ps;
            runmax[h] = pm;
        }
        return;
    }
    const double m = std_max(rm, pm);
    const double a_acc = exp_glibc(__dadd_rn(rm, -m)), a_part = exp_glibc(__dadd_rn(pm, -m));
    for (uint32_t t = threadIdx.x; t < dv; t += kAT)
        dst[t] = __dadd_rn(__dmul_rn(dst[t], a_acc), __dmul_rn(src[t], a_part));
    if (threadIdx.x == 0) {
        sumexp[h] = __dadd_rn(__dmul_rn(se, a_acc), __dmul_rn(ps, a_part));
        runmax[h] = m;
    }
}

// pattn_finalize: out = (float)(out_acc * (1 / sumexp)); sumexp = 0 -> zero row
__global__ void __launch_bounds__(kAT) acc_finalize_kernel(const double* out_acc, const double* sumexp,
                                                           uint32_t dv, float* out, int* any_empty) {
    const uint32_t h = blockIdx.x;
    const double se = sumexp[h];
    if (se == 0.0) {
        for (uint32_t t = threadIdx.x; t < dv; t += kAT) out[(size_t)h * dv + t] = 0.f;
        if (threadIdx.x == 0) atomicOr(any_empty, 1);
        return;
    }
    const double inv = __ddiv_rn(1.0, se);
    for (uint32_t t = threadIdx.x; t < dv; t += kAT)
        out[(size_t)h * dv + t] = (float)__dmul_rn(out_acc[(size_t)h * dv + t], inv);
}

__global__ void acc_init_kernel(double* out, double* sumexp, double* runmax, uint32_t H, uint32_t dv) {
    // value_dim 0 still has H (sumexp, runmax) pairs (attention.cpp:82-83)
    const uint32_t n = max(H * dv, H);
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        if (e < H * dv) out[e] = 0.0;
        if (e < H) {
            sumexp[e] = 0.0;
            runmax[e] = -INFINITY;
        }
    }
}

}  // namespace

void launch_acc_init(double* out, double* sumexp, double* runmax, uint32_t H, uint32_t dv,
                     cudaStream_t st) {
    acc_init_kernel<<<std::max<uint32_t>(1, std::min<uint32_t>(1024, (std::max(H * dv, H) + 255) / 256)), 256, 0, st>>>(
            out, sumexp, runmax, H, dv);
    SAAP_CUDA(cudaGetLastError());
}

// One absorb of n staged rows into (out, sumexp, runmax); S is [H x n] scratch.
void launch_acc_absorb(const float* q, uint32_t H, uint32_t d, const float* K, const float* V,
                       uint32_t n, uint32_t dv, double scale, double* S, double* rescale,
                       double* out, double* sumexp, double* runmax, cudaStream_t st) {
    acc_scores_kernel<<<dim3((n + kAT - 1) / kAT, H), kAT, 0, st>>>(q, K, n, d, scale, S);
    acc_weights_kernel<<<H, kAT, 0, st>>>(S, n, sumexp, runmax, rescale);
    acc_values_kernel<<<dim3((dv + kAT - 1) / kAT, H), kAT, 0, st>>>(S, V, n, dv, rescale, out);
    SAAP_CUDA(cudaGetLastError());
}

void launch_acc_merge(double* out, double* sumexp, double* runmax, const double* p_out,
                      const double* p_sumexp, const double* p_runmax, uint32_t H, uint32_t dv,
                      cudaStream_t st) {
    acc_merge_kernel<<<H, kAT, 0, st>>>(out, sumexp, runmax, p_out, p_sumexp, p_runmax, dv);
    SAAP_CUDA(cudaGetLastError());
}

void launch_acc_finalize(const double* out_acc, const double* sumexp, uint32_t H, uint32_t dv,
                         float* out, int* any_empty, cudaStream_t st) {
    acc_finalize_kernel<<<H, kAT, 0, st>>>(out_acc, sumexp, dv, out, any_empty);
    SAAP_CUDA(cudaGetLastError());
}

}  // namespace saap_b200
