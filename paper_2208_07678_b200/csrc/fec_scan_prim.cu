// Device-wide exclusive scan (reduce-then-scan over 2048-element tiles, host recursion).
// Used for radix-sort digit offsets and for group/cell head flags.
#include "fec_internal.cuh"

namespace fec {

constexpr int SC_THREADS = 256;
constexpr int SC_ITEMS = 8;
constexpr int SC_TILE = SC_THREADS * SC_ITEMS;

// `ndev` (optional): the length is min(n, *ndev), read on the device (tiles past it only
// publish a zero tile sum), so a scan can be sized by a count a previous kernel produced.
template <typename T>
__global__ void __launch_bounds__(SC_THREADS) k_scan_tile(const T* __restrict__ in, T* __restrict__ out,
                                                         int64_t n, T* __restrict__ sums, const int* ndev) {
    __shared__ T s[SC_TILE];
    __shared__ T wsum[SC_THREADS / kWarp];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t base = (int64_t)blockIdx.x * SC_TILE;
    if (ndev) n = min(n, (int64_t)*ndev);
    if (base >= n) {
        if (tid == 0) sums[blockIdx.x] = T(0);
        return;
    }
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        int64_t i = base + k * SC_THREADS + tid;
        s[k * SC_THREADS + tid] = i < n ? in[i] : T(0);
    }
    __syncthreads();
    T loc[SC_ITEMS];
    T run = 0;
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        T v = s[tid * SC_ITEMS + k];
        loc[k] = run;
        run += v;
    }
    // warp inclusive scan of per-thread totals
    T x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        T v = lane < SC_THREADS / kWarp ? wsum[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        if (lane < SC_THREADS / kWarp) wsum[lane] = v;  // inclusive warp totals
    }
    __syncthreads();
    T prefix = (x - run) + (w > 0 ? wsum[w - 1] : T(0));
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) s[tid * SC_ITEMS + k] = prefix + loc[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        int64_t i = base + k * SC_THREADS + tid;
        if (i < n) out[i] = s[k * SC_THREADS + tid];
    }
    if (tid == 0) sums[blockIdx.x] = wsum[SC_THREADS / kWarp - 1];
}

template <typename T>
__global__ void __launch_bounds__(SC_THREADS) k_scan_add(T* __restrict__ out, int64_t n, const T* __restrict__ sums,
                                                        const int* ndev) {
    if (ndev) n = min(n, (int64_t)*ndev);
    const int64_t base = (int64_t)blockIdx.x * SC_TILE;
    if (base >= n) return;
    const T add = sums[blockIdx.x];
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        int64_t i = base + k * SC_THREADS + threadIdx.x;
        if (i < n) out[i] += add;
    }
}

size_t scan_scratch_elems(int64_t n) {
    size_t total = 0;
    int64_t m = n;
    while (m > 1) {
        int64_t nb = (m + SC_TILE - 1) / SC_TILE;
        total += (size_t)nb + 128;
        m = nb;
    }
    return total + 64;
}

template <typename T>
int exclusive_scan_dn(const T* in, T* out, int64_t n, const int* ndev, T* scratch, cudaStream_t st) {
    if (n <= 0) return 0;
    int launches = 1;
    int64_t nb = (n + SC_TILE - 1) / SC_TILE;
    k_scan_tile<T><<<(unsigned)nb, SC_THREADS, 0, st>>>(in, out, n, scratch, ndev);
    if (nb > 1) {
        T* next = scratch + ((nb + 63) / 64) * 64 + 64;
        launches += exclusive_scan_dn<T>(scratch, scratch, nb, nullptr, next, st);
        k_scan_add<T><<<(unsigned)nb, SC_THREADS, 0, st>>>(out, n, scratch, ndev);
        ++launches;
    }
    return launches;
}

template <typename T>
int exclusive_scan(const T* in, T* out, int64_t n, T* scratch, cudaStream_t st) {
    return exclusive_scan_dn<T>(in, out, n, nullptr, scratch, st);
}

template int exclusive_scan_dn<uint32_t>(const uint32_t*, uint32_t*, int64_t, const int*, uint32_t*, cudaStream_t);
template int exclusive_scan<uint32_t>(const uint32_t*, uint32_t*, int64_t, uint32_t*, cudaStream_t);
template int exclusive_scan<unsigned long long>(const unsigned long long*, unsigned long long*, int64_t,
                                                unsigned long long*, cudaStream_t);

}  // namespace fec
