// Microbenchmark: read bandwidth of an AoS float3 array (12 B/point) with three access
// patterns, to decide how the point-streaming kernels should load.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void strided(const float4* q, long nq, float* out) {  // thread reads quad i: q[3i..3i+2]
    float acc = 0;
    long stride = (long)gridDim.x * blockDim.x;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < nq; i += stride) {
        float4 a = __ldg(q + 3 * i), b = __ldg(q + 3 * i + 1), c = __ldg(q + 3 * i + 2);
        acc += a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w + c.x + c.y + c.z + c.w;
    }
    if (acc == 1234.5f) out[0] = acc;
}
__global__ void strided2(const float4* q, long nq, float* out) {  // two quads in flight
    float acc = 0;
    long stride = (long)gridDim.x * blockDim.x;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < nq; i += 2 * stride) {
        long j = i + stride < nq ? i + stride : i;
        float4 a = __ldg(q + 3 * i), b = __ldg(q + 3 * i + 1), c = __ldg(q + 3 * i + 2);
        float4 d = __ldg(q + 3 * j), e = __ldg(q + 3 * j + 1), f = __ldg(q + 3 * j + 2);
        acc += a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w + c.x + c.y + c.z + c.w;
        acc += d.x + d.y + d.z + d.w + e.x + e.y + e.z + e.w + f.x + f.y + f.z + f.w;
    }
    if (acc == 1234.5f) out[0] = acc;
}
__global__ void coalesced(const float4* q, long nf4, float* out) {  // warp reads 3x512 B contiguous
    float acc = 0;
    long stride = (long)gridDim.x * blockDim.x;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < nf4; i += stride) {
        float4 a = __ldg(q + i);
        acc += a.x + a.y + a.z + a.w;
    }
    if (acc == 1234.5f) out[0] = acc;
}
__global__ void coalesced3(const float4* q, long nq, float* out) {  // per warp 96 float4 chunk, 3 loads
    float acc = 0;
    const int lane = threadIdx.x & 31;
    long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    long nw = ((long)gridDim.x * blockDim.x) >> 5;
    for (long c = warp; c * 32 < nq; c += nw) {
        const float4* b = q + c * 96;
        float4 x = __ldg(b + lane), y = __ldg(b + 32 + lane), z = __ldg(b + 64 + lane);
        acc += x.x + x.y + x.z + x.w + y.x + y.y + y.z + y.w + z.x + z.y + z.z + z.w;
    }
    if (acc == 1234.5f) out[0] = acc;
}
int main() {
    long n = 27417973L & ~127L;
    long nq = n / 4;
    float4* q;
    float* out;
    cudaMalloc(&q, n * 12);
    cudaMalloc(&out, 4);
    cudaMemset(q, 0, n * 12);
    float* flush;
    cudaMalloc(&flush, 256 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 148;
    for (int variant = 0; variant < 4; ++variant)
        for (int bps : {4, 8, 16, 32}) {
            int blocks = sms * bps;
            float best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                cudaMemsetAsync(flush, rep, 256 << 20);
                cudaEventRecord(e0);
                if (variant == 0) strided<<<blocks, 256>>>(q, nq, out);
                if (variant == 1) strided2<<<blocks, 256>>>(q, nq, out);
                if (variant == 2) coalesced<<<blocks, 256>>>(q, nq * 3, out);
                if (variant == 3) coalesced3<<<blocks, 256>>>(q, nq, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            printf("variant %d blocks/SM %2d: %.1f us  %.0f GB/s\n", variant, bps, best * 1e3, n * 12 / best / 1e6);
        }
    return 0;
}
