// Measures B200 CUDA-core fp64 rates: throughput (many independent DFMA
// chains) and latency (one dependent chain), vs fp32 FFMA.  Diagnostic only.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void thr(T* out, int iters) {
    T a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const T m = (T)1.0000001, c = (T)1e-7;
    for (int i = 0; i < iters; ++i) {
        a0 = a0 * m + c; a1 = a1 * m + c; a2 = a2 * m + c; a3 = a3 * m + c;
        a4 = a4 * m + c; a5 = a5 * m + c; a6 = a6 * m + c; a7 = a7 * m + c;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void lat(double* out, int iters, long long* cyc) {
    double a = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) a = __dadd_rn(__dmul_rn(a, 1.0000001), 1e-7);
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double* d; float* f; long long* cyc;
    cudaMalloc(&d, 1 << 24); cudaMalloc(&f, 1 << 24); cudaMalloc(&cyc, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 4096, blocks = 148 * 8, threads = 256;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0); thr<double><<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * iters * (double)blocks * threads;
        if (rep) printf("fp64 FMA throughput: %.2f TFLOPS\n", flops / ms / 1e9);
        cudaEventRecord(e0); thr<float><<<blocks, threads>>>(f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("fp32 FMA throughput: %.2f TFLOPS\n", flops / ms / 1e9);
    }
    lat<<<1, 32>>>(d, 1024, cyc); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("fp64 dependent mul+add latency: %.1f cycles per pair\n", c / 1024.0);
    return 0;
}
