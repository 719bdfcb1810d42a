// mma.sync m16n8k16 bf16 throughput on this GPU (profiling aid)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(float* out, int iters) {
    float c[4][4] = {};
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int j = 0; j < 4; ++j) for (int e = 0; e < 4; ++e) s += c[j][e];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* o; cudaMalloc(&o, 148 * 1024 * 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int warps : {4, 8, 16, 32}) {
        const int iters = 4096;
        k<<<sms, warps * 32>>>(o, 16);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<sms, warps * 32>>>(o, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double mmas = (double)sms * warps * iters * 4;
        double tflops = mmas * 4096 * 2 / (ms * 1e-3) / 1e12;
        printf("warps/SM %d: %.1f TFLOP/s  (%.2f mma/clk/SM at 1.9GHz, %.1f ns per mma per SMSP)\n", warps, tflops,
               mmas / sms / (ms * 1e-3) / 1.9e9, ms * 1e6 / (mmas / sms / 4));
    }
    return 0;
}
