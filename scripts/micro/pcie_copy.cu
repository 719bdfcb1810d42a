// Small host<->device transfers on this box: copy-engine memcpy vs zero-copy kernels
// (profiling aid for the host API's step graph)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void up(const float4* __restrict__ h, float4* __restrict__ d, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) d[i] = h[i];
}
__global__ void down(const float4* __restrict__ d, float4* __restrict__ h, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) h[i] = d[i];
}
int main() {
    const size_t up_b = 262144, dn_b = 132608;
    float *h_up, *h_dn, *d_up, *d_dn, *hu_dev, *hd_dev;
    cudaHostAlloc(&h_up, up_b, cudaHostAllocMapped);
    cudaHostAlloc(&h_dn, dn_b, cudaHostAllocMapped);
    cudaHostGetDevicePointer(&hu_dev, h_up, 0);
    cudaHostGetDevicePointer(&hd_dev, h_dn, 0);
    cudaMalloc(&d_up, up_b); cudaMalloc(&d_dn, dn_b);
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto t = [&](auto fn, const char* name) {
        for (int i = 0; i < 20; ++i) fn();
        cudaStreamSynchronize(s);
        float best = 1e9;
        for (int r = 0; r < 50; ++r) {
            cudaEventRecord(e0, s); fn(); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        printf("%-40s %7.1f us\n", name, best * 1e3);
    };
    t([&] { cudaMemcpyAsync(d_up, h_up, up_b, cudaMemcpyHostToDevice, s); }, "memcpy H2D 256KB");
    t([&] { cudaMemcpyAsync(d_up, h_up, up_b / 2, cudaMemcpyHostToDevice, s); }, "memcpy H2D 128KB");
    t([&] { cudaMemcpyAsync(h_dn, d_dn, dn_b, cudaMemcpyDeviceToHost, s); }, "memcpy D2H 130KB");
    for (int blocks : {16, 64, 148, 296}) {
        char nm[64];
        snprintf(nm, 64, "kernel H2D 256KB (%d CTAs)", blocks);
        t([&] { up<<<blocks, 256, 0, s>>>((const float4*)hu_dev, (float4*)d_up, up_b / 16); }, nm);
        snprintf(nm, 64, "kernel D2H 130KB (%d CTAs)", blocks);
        t([&] { down<<<blocks, 256, 0, s>>>((const float4*)d_dn, (float4*)hd_dev, dn_b / 16); }, nm);
    }
    t([&] { cudaMemcpyAsync(d_up, h_up, up_b, cudaMemcpyHostToDevice, s);
            cudaMemcpyAsync(h_dn, d_dn, dn_b, cudaMemcpyDeviceToHost, s); }, "memcpy H2D + D2H");
    t([&] { up<<<148, 256, 0, s>>>((const float4*)hu_dev, (float4*)d_up, up_b / 16);
            down<<<148, 256, 0, s>>>((const float4*)d_dn, (float4*)hd_dev, dn_b / 16); }, "kernel H2D + D2H (148 CTAs)");
    return 0;
}
