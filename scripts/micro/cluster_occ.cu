// Max co-resident clusters of 1-CTA-per-SM kernels (~200 KB smem) for cluster
// sizes 1..16 on this GPU (profiling aid: can a whole persistent grid be clustered?)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { extern __shared__ int s[]; if (threadIdx.x == 0 && p) p[0] = s[0]; }
int main() {
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cs * 64); cfg.blockDim = dim3(320); cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        int n = 0; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k, &cfg);
        printf("cluster %2d: max active clusters %3d -> %3d SMs of %d (%s)\n", cs, n, n * cs, sms, cudaGetErrorString(e));
    }
}
