// Micro-benchmark: random 32-bit atomicAdd over a window of W words (W from 256K to 64M words),
// 100M atomics; prints ms and G atomics/s.  Is a few-MB window of random atomics L2-resident?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_atom(uint32_t* a, int64_t m, uint32_t wmask, uint32_t seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u ^ seed;
        h ^= h >> 15; h *= 0x2c1b3c6du; h ^= h >> 12;
        atomicAdd(a + (h & wmask), 1u);
    }
}
// windowed: the atomic's index = a sliding window over a big array (like buckets in order)
__global__ void k_atom_slide(uint32_t* a, int64_t m, uint32_t wmask, int64_t total, uint32_t seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u ^ seed;
        h ^= h >> 15; h *= 0x2c1b3c6du; h ^= h >> 12;
        const int64_t base = (i * (total - wmask - 1)) / m;
        atomicAdd(a + base + (h & wmask), 1u);
    }
}
int main() {
    const int64_t total = int64_t(1) << 27;  // 512 MB
    uint32_t* a; cudaMalloc(&a, total * 4); cudaMemset(a, 0, total * 4);
    const int64_t m = 100000000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int lw = 16; lw <= 27; lw += 1) {
        const uint32_t wmask = (uint32_t)((int64_t(1) << lw) - 1);
        for (int mode = 0; mode < 2; ++mode) {
            if (mode == 1 && lw >= 27) continue;
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (mode == 0) k_atom<<<148 * 8, 256>>>(a, m, wmask, rep);
                else k_atom_slide<<<148 * 8, 256>>>(a, m, wmask, total, rep);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                if (rep) printf("%s window %6.1f MB: %.3f ms  %.1f G atomics/s\n", mode ? "slide" : "fixed",
                                (double)(wmask + 1) * 4 / 1e6, ms, m / ms / 1e6);
            }
        }
    }
    return 0;
}
