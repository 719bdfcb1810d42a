// Counter-based synthetic KV/query generator for the bench (not on the hot
// path).  Element (row, j) is a pure function of (seed, row, j), so any
// sub-range is reproducible on the CPU by bench.py's numpy restatement.
#include "common.cuh"

namespace saap_b200 {

__host__ __device__ __forceinline__ uint64_t splitmix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ float gauss(uint64_t h) {
    const float u1 = ((h >> 40) + 1) * (1.0f / 16777217.0f);  // (0, 1]
    const float u2 = ((h >> 16) & 0xFFFFFF) * (1.0f / 16777216.0f);
    return sqrtf(-2.0f * __logf(u1)) * __cosf(6.283185307f * u2);
}

// kind 0: noise * N(0,1); kind 1: centers[h(row) % n] * scale + noise * N(0,1)
__global__ void synth_kernel(uint16_t* out, uint64_t rows, uint32_t D, uint64_t seed, int kind,
                             const float* centers, uint64_t n_centers, float scale, float noise) {
    const uint64_t n = rows * D;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = e / D, j = e % D;
        float x = noise * gauss(splitmix(seed ^ splitmix(e)));
        if (kind == 1) {
            const uint64_t c = splitmix(seed * 0x2545F4914F6CDD1Dull + r) % n_centers;
            x += scale * centers[c * D + j];
        }
        out[e] = f32_to_bf16_rne(x);
    }
}

void launch_synth(uint16_t* out, uint64_t rows, uint32_t D, uint64_t seed, int kind,
                  const float* centers, uint64_t n_centers, float scale, float noise,
                  cudaStream_t st) {
    const uint64_t n = rows * D;
    if (!n) return;
    synth_kernel<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 64), 256, 0, st>>>(
            out, rows, D, seed, kind, centers, n_centers, scale, noise);
    SAAP_CUDA(cudaGetLastError());
}

}  // namespace saap_b200
