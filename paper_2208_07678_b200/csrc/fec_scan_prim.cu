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
    pdl_prologue();
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
    pdl_prologue();
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

// Single-pass exclusive scan with decoupled look-back (uint32 data): tiles are taken in
// order from an atomic counter; each publishes its aggregate, then walks back over the
// published states of earlier tiles until an inclusive prefix is found.  One launch (+ one
// small memset) instead of the reduce-then-scan recursion's three or more.
__global__ void __launch_bounds__(SC_THREADS) k_scan_lb(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                       int64_t n, const int* ndev,
                                                       unsigned long long* __restrict__ state,
                                                       unsigned int* __restrict__ counter, const int* skip0,
                                                       const int* skip1) {
    pdl_prologue();
    if ((skip0 && *skip0) || (skip1 && *skip1)) return;  // device-side choice: this scan is not needed
    __shared__ uint32_t s[SC_TILE];
    __shared__ uint32_t wsum[SC_THREADS / kWarp];
    __shared__ unsigned int tile_sh;
    __shared__ uint32_t prefix_sh;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (ndev) n = min(n, (int64_t)*ndev);
    // persistent blocks take tiles in order from the counter until past the end (every
    // later tile is past the end too, so nobody looks back at those)
    while (true) {
    __syncthreads();
    if (tid == 0) tile_sh = atomicAdd(counter, 1u);
    __syncthreads();
    const unsigned tile = tile_sh;
    const int64_t base = (int64_t)tile * SC_TILE;
    if (base >= n) return;
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        int64_t i = base + k * SC_THREADS + tid;
        s[k * SC_THREADS + tid] = i < n ? in[i] : 0u;
    }
    __syncthreads();
    uint32_t loc[SC_ITEMS];
    uint32_t run = 0;
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        uint32_t v = s[tid * SC_ITEMS + k];
        loc[k] = run;
        run += v;
    }
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t v = lane < SC_THREADS / kWarp ? wsum[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        if (lane < SC_THREADS / kWarp) wsum[lane] = v;
        // publish this tile's aggregate, then look back 32 tiles at a time (warp 0)
        const unsigned long long agg = __shfl_sync(0xffffffffu, v, SC_THREADS / kWarp - 1);
        constexpr unsigned long long A = 1ull << 62, P = 2ull << 62, VAL = (1ull << 62) - 1;
        unsigned long long prefix = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(state, P | agg);
        } else {
            if (lane == 0) atomicExch(state + tile, A | agg);
            int j = (int)tile - 1;  // lane k examines tile j - k
            while (true) {
                const int idx = j - lane;
                unsigned long long sv = idx >= 0 ? *reinterpret_cast<volatile unsigned long long*>(state + idx) : P;
                const unsigned pmask = __ballot_sync(0xffffffffu, (sv & ~VAL) == P);
                // lanes up to the nearest inclusive prefix must all have published
                const int upto = pmask ? __ffs(pmask) - 1 : 31;
                if (!__all_sync(0xffffffffu, lane > upto || (sv & ~VAL) != 0)) continue;
                unsigned long long val = lane <= upto ? (sv & VAL) : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                prefix += val;
                if (pmask) break;
                j -= 32;
            }
            if (lane == 0) atomicExch(state + tile, P | (prefix + agg));
        }
        if (lane == 0) prefix_sh = (uint32_t)prefix;
    }
    __syncthreads();
    const uint32_t pre = prefix_sh + (x - run) + (w > 0 ? wsum[w - 1] : 0u);
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) s[tid * SC_ITEMS + k] = pre + loc[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        int64_t i = base + k * SC_THREADS + tid;
        if (i < n) out[i] = s[k * SC_THREADS + tid];
    }
    }  // tiles
}

size_t scan_scratch_elems(int64_t n) {
    size_t total = 0;
    int64_t m = n;
    while (m > 1) {
        int64_t nb = (m + SC_TILE - 1) / SC_TILE;
        total += (size_t)nb + 128;
        m = nb;
    }
    // the single-pass scan needs one 64-bit state per tile plus a counter
    const size_t lb = 2 * (size_t)((n + SC_TILE - 1) / SC_TILE) + 64;
    return (total > lb ? total : lb) + 64;
}

template <typename T>
int exclusive_scan_dn(const T* in, T* out, int64_t n, const int* ndev, T* scratch, cudaStream_t st) {
    if (n <= 0) return 0;
    int launches = 1;
    int64_t nb = (n + SC_TILE - 1) / SC_TILE;
    pdl(k_scan_tile<T>, (unsigned)nb, SC_THREADS, 0, st)(in, out, n, scratch, ndev);
    if (nb > 1) {
        T* next = scratch + ((nb + 63) / 64) * 64 + 64;
        launches += exclusive_scan_dn<T>(scratch, scratch, nb, nullptr, next, st);
        pdl(k_scan_add<T>, (unsigned)nb, SC_THREADS, 0, st)(out, n, scratch, ndev);
        ++launches;
    }
    return launches;
}

template <typename T>
int exclusive_scan(const T* in, T* out, int64_t n, T* scratch, cudaStream_t st) {
    return exclusive_scan_dn<T>(in, out, n, nullptr, scratch, st);
}

// uint32: the single-pass look-back scan for up to kLbTiles tiles and for device-sized
// scans (measured faster there); other large arrays keep the reduce-then-scan recursion
constexpr int64_t kLbTiles = 512;
template <typename T>
int scan_recursive(const T* in, T* out, int64_t n, const int* ndev, T* scratch, cudaStream_t st) {
    if (n <= 0) return 0;
    int launches = 1;
    int64_t nb = (n + SC_TILE - 1) / SC_TILE;
    pdl(k_scan_tile<T>, (unsigned)nb, SC_THREADS, 0, st)(in, out, n, scratch, ndev);
    if (nb > 1) {
        T* next = scratch + ((nb + 63) / 64) * 64 + 64;
        launches += scan_recursive<T>(scratch, scratch, nb, nullptr, next, st);
        pdl(k_scan_add<T>, (unsigned)nb, SC_THREADS, 0, st)(out, n, scratch, ndev);
        ++launches;
    }
    return launches;
}

template <>
int exclusive_scan_dn<uint32_t>(const uint32_t* in, uint32_t* out, int64_t n, const int* ndev, uint32_t* scratch,
                                cudaStream_t st) {
    if (n <= 0) return 0;
    const int64_t nb = (n + SC_TILE - 1) / SC_TILE;
    // device-sized scans (ndev) are mostly tiles past the end, which the look-back scan skips
    if (nb > kLbTiles && !ndev) return scan_recursive<uint32_t>(in, out, n, ndev, scratch, st);
    // scratch: [counter (8 B, padded to 256)] [state: nb x 8 B]
    unsigned int* counter = reinterpret_cast<unsigned int*>(scratch);
    unsigned long long* state = reinterpret_cast<unsigned long long*>(scratch + 64);
    cudaMemsetAsync(scratch, 0, 256 + (size_t)nb * 8, st);
    pdl(k_scan_lb, (unsigned)nb, SC_THREADS, 0, st)(in, out, n, ndev, state, counter, nullptr, nullptr);
    return 2;
}
// Single-pass scan whose look-back state (nb x 8 B) and counter were zeroed earlier in the call
// (k_zero): no memset node; a persistent grid of at most `max_blocks` blocks.
// skip0 / skip1 (optional device ints): the scan does nothing when either is nonzero.
int exclusive_scan_lb(const uint32_t* in, uint32_t* out, int64_t n, const int* ndev, unsigned long long* state,
                      unsigned int* counter, int max_blocks, const int* skip0, const int* skip1, cudaStream_t st) {
    if (n <= 0) return 0;
    const int64_t nb = (n + SC_TILE - 1) / SC_TILE;
    const unsigned blocks = (unsigned)(nb < max_blocks ? nb : max_blocks);
    pdl(k_scan_lb, blocks, SC_THREADS, 0, st)(in, out, n, ndev, state, counter, skip0, skip1);
    return 1;
}
int64_t scan_lb_tiles(int64_t n) { return (n + SC_TILE - 1) / SC_TILE; }

template <>
int exclusive_scan<uint32_t>(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* scratch, cudaStream_t st) {
    return exclusive_scan_dn<uint32_t>(in, out, n, nullptr, scratch, st);
}
template int exclusive_scan<unsigned long long>(const unsigned long long*, unsigned long long*, int64_t,
                                                unsigned long long*, cudaStream_t);

}  // namespace fec
