// Dense-grid path (the default whenever the bbox holds <= 32n + 2^26 grid cells).
//
// Binning: an occupancy bitmap over the linear grid cells gives every occupied cell a
// compact id; points are counting-sorted by compact cell id (a3).  Cells holding more than
// SPARSE_MAX points are "dense": each keeps a 64-bit occupancy mask of its 4x4x4 fine
// sub-cells (fec_subcell.cuh), split into at most 8 certain-connected components that
// become union-find nodes of their own (ids n + 8*record + k).  Then
//   * sparse cells: every point pair with a sparse forward neighbour is tested directly;
//   * dense cells: components of adjacent cells are united without any distance test when
//     a certain sub-cell pair joins them, and the rare pairs that are only "uncertain" go
//     to a queue of point tests (early exit at the first pred-true pair).
// DESIGN.md §4 describes why every edge of the graph of Eq. 1 is covered exactly.
#include "fec_internal.cuh"
#include "fec_kernels.cuh"
#include "fec_pairs.cuh"
#include "fec_subcell.cuh"

namespace fec {

__device__ SubcellTables d_sc;  // filled once per device (fec_capi.cu)

// Batched clouds (fec_cluster_batch_ws): the cloud holding input index i (binary search over
// the cloud offsets, a small L1-resident array).
__device__ __forceinline__ int cloud_of(const Grid& g, int64_t i) {
    int lo = 0, hi = g.nclouds;  // boff[lo] <= i < boff[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(g.boff + mid) <= i) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Fine sub-cell coordinates f = floor((x - lo) * inv_q) (inv_q = 4/c exactly twice inv_h,
// so cell = f >> 2 equals the coarse computation floor((x - lo) * inv_h) >> 1).  In batch
// mode each cloud uses its own origin and is shifted by a whole number of cells along z,
// with an empty cell layer between clouds, so no cell neighbourhood spans two clouds.
// `i` is the point's input index.
__device__ __forceinline__ void dense_cell_of(float x, float y, float z, int64_t i, const Grid& g, uint32_t& lin,
                                              int& q) {
    double l0 = g.lo[0], l1 = g.lo[1], l2 = g.lo[2];
    uint32_t zoff = 0;
    if (g.batch) {
        const int c = cloud_of(g, i);
        l0 = __ldg(g.blo + 3 * c);
        l1 = __ldg(g.blo + 3 * c + 1);
        l2 = __ldg(g.blo + 3 * c + 2);
        zoff = 4u * (uint32_t)__ldg(g.bz + c);
    }
    const uint32_t fx = sub_coord(x, l0, g.inv_q);
    const uint32_t fy = sub_coord(y, l1, g.inv_q);
    const uint32_t fz = sub_coord(z, l2, g.inv_q) + zoff;
    q = (int)((fx & 3u) | ((fy & 3u) << 2) | ((fz & 3u) << 4));
    lin = (fx >> 2) * g.stride[0] + (fy >> 2) * g.stride[1] + (fz >> 2) * g.stride[2];
}

__device__ __forceinline__ void dense_decode(uint32_t lin, const Grid& g, int c[3]) {
    // slow axis = perm[2] (stride sdiv[0]), middle = perm[1] (stride sdiv[1]), fast = perm[0]
    const uint32_t q2 = lin / g.sdiv[0];
    lin -= q2 * g.sdiv[0];
    const uint32_t q1 = lin / g.sdiv[1];
    const uint32_t q0 = lin - q1 * g.sdiv[1];
    c[0] = (int)(g.perm[2] == 0 ? q2 : (g.perm[1] == 0 ? q1 : q0));
    c[1] = (int)(g.perm[2] == 1 ? q2 : (g.perm[1] == 1 ? q1 : q0));
    c[2] = (int)(g.perm[2] == 2 ? q2 : (g.perm[1] == 2 ? q1 : q0));
}

__device__ __forceinline__ bool dense_neighbor(const Grid& g, const int c[3], int dx, int dy, int dz, uint32_t& lin) {
    const int x = c[0] + dx, y = c[1] + dy, z = c[2] + dz;
    if (x < 0 || y < 0 || z < 0 || x >= g.dims[0] || y >= g.dims[1] || z >= g.dims[2]) return false;
    lin = (uint32_t)x * g.stride[0] + (uint32_t)y * g.stride[1] + (uint32_t)z * g.stride[2];
    return true;
}

// Four consecutive input points per thread: three 16-byte loads when `points` is 16-byte
// aligned (more bytes in flight per thread than one scalar load per coordinate).
struct Pts4 {
    float x[4], y[4], z[4];
};
__device__ __forceinline__ void load_pts4(const float* __restrict__ p, int64_t n, int64_t base, bool vec, Pts4& P) {
    if (vec && base + 4 <= n) {
        const float4* q = reinterpret_cast<const float4*>(p + 3 * base);
        const float4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
        P.x[0] = a.x; P.y[0] = a.y; P.z[0] = a.z;
        P.x[1] = a.w; P.y[1] = b.x; P.z[1] = b.y;
        P.x[2] = b.z; P.y[2] = b.w; P.z[2] = c.x;
        P.x[3] = c.y; P.y[3] = c.z; P.z[3] = c.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t i = base + j;
            P.x[j] = i < n ? __ldg(p + 3 * i) : 0.f;
            P.y[j] = i < n ? __ldg(p + 3 * i + 1) : 0.f;
            P.z[j] = i < n ? __ldg(p + 3 * i + 2) : 0.f;
        }
    }
}

// One gathered point (random index): the 16-byte aligned word(s) covering its 12 bytes,
// so each point costs one (rarely two) memory transactions instead of three loads.
__device__ __forceinline__ void load_point(const float* __restrict__ p, int64_t i, float& x, float& y, float& z) {
    const int64_t f = 3 * i;  // first float
    if ((reinterpret_cast<uintptr_t>(p) & 15u) == 0) {
        const float4* q = reinterpret_cast<const float4*>(p) + (f >> 2);
        const float4 a = __ldg(q);
        switch (f & 3) {
            case 0: x = a.x; y = a.y; z = a.z; return;
            case 1: x = a.y; y = a.z; z = a.w; return;
            case 2: { const float4 b = __ldg(q + 1); x = a.z; y = a.w; z = b.x; return; }
            default: { const float4 b = __ldg(q + 1); x = a.w; y = b.x; z = b.y; return; }
        }
    }
    x = __ldg(p + f);
    y = __ldg(p + f + 1);
    z = __ldg(p + f + 2);
}

// ---- compact cell ids ---------------------------------------------------------------------
// Only occupied cells get storage: an occupancy bitmap over the linear cell ids, each 32-bit
// word paired with the number of occupied cells before it (uint2 {bits, base}), gives the
// compact id of an occupied cell with one 8-byte load and a popcount.  The bitmap is 1/32 B
// per grid cell (C4: 89M grid cells, 358k occupied -> 11 MB, L2-resident), so per-cell tables
// (counts / starts, dense records) are sized by the occupied cells, not the bounding box.
__device__ __forceinline__ uint32_t cid_of(const uint2* __restrict__ cw, uint32_t lin) {
    const uint2 v = __ldg(cw + (lin >> 5));
    return v.y + (uint32_t)__popc(v.x & ((1u << (lin & 31u)) - 1u));
}
__device__ __forceinline__ int cid_lookup(const uint2* __restrict__ cw, uint32_t lin) {
    const uint2 v = __ldg(cw + (lin >> 5));
    const uint32_t b = 1u << (lin & 31u);
    return (v.x & b) ? (int)(v.y + (uint32_t)__popc(v.x & (b - 1u))) : -1;
}

// ---- a2: occupancy bitmap ------------------------------------------------------------------
// Binning kernels aggregate per block through a small shared-memory hash table (keys = bitmap
// word or compact cell id): one global atomic per distinct key per tile of kBinTile points.
constexpr int kBinThreads = 256;
constexpr int kBinIpt = 4;
constexpr int kBinTile = kBinThreads * kBinIpt;
constexpr int kBinSlots = 2 * kBinTile;

// Insert `key`; a thread that claims a new slot appends it to `used` (so the flush visits only
// occupied slots).
__device__ __forceinline__ int bin_slot(int* keys, uint32_t key, int* used, int* nused) {
    uint32_t h = (key * 2654435761u) & (kBinSlots - 1);
    while (true) {
        const int cur = keys[h];
        if (cur == (int)key) return (int)h;
        if (cur == -1) {
            const int old = atomicCAS(keys + h, -1, (int)key);
            if (old == -1) {
                used[atomicAdd(nused, 1)] = (int)h;
                return (int)h;
            }
            if (old == (int)key) return (int)h;
        }
        h = (h + 1) & (kBinSlots - 1);
    }
}

__global__ void __launch_bounds__(kBinThreads) k_cmark(const float* __restrict__ p, int64_t n, Grid g,
                                                       uint2* __restrict__ cw) {
    pdl_prologue();
    __shared__ int keys[kBinSlots];
    __shared__ uint32_t bits[kBinSlots];
    __shared__ int used[kBinTile];
    __shared__ int nused;
    const bool vec = (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
    for (int k = threadIdx.x; k < kBinSlots; k += kBinThreads) { keys[k] = -1; bits[k] = 0u; }
    if (threadIdx.x == 0) nused = 0;
    __syncthreads();
    for (int64_t t0 = (int64_t)blockIdx.x * kBinTile; t0 < n; t0 += (int64_t)gridDim.x * kBinTile) {
        const int64_t b4 = t0 + kBinIpt * threadIdx.x;
        Pts4 P;
        load_pts4(p, n, b4, vec, P);
        // runs of this thread's points in the same bitmap word take one table update
        uint32_t word = 0xffffffffu, wbits = 0u;
#pragma unroll
        for (int j = 0; j < kBinIpt; ++j) {
            if (b4 + j < n) {
                uint32_t lin;
                int q;
                dense_cell_of(P.x[j], P.y[j], P.z[j], b4 + j, g, lin, q);
                if ((lin >> 5) != word) {
                    if (wbits) atomicOr(bits + bin_slot(keys, word, used, &nused), wbits);
                    word = lin >> 5;
                    wbits = 0u;
                }
                wbits |= 1u << (lin & 31u);
            }
        }
        if (wbits) atomicOr(bits + bin_slot(keys, word, used, &nused), wbits);
        __syncthreads();
        const int nu = nused;
        for (int e = threadIdx.x; e < nu; e += kBinThreads) {
            const int k = used[e];
            atomicOr(reinterpret_cast<unsigned int*>(cw + keys[k]), bits[k]);
            keys[k] = -1;
            bits[k] = 0u;
        }
        __syncthreads();
        if (threadIdx.x == 0) nused = 0;
        __syncthreads();
    }
}

// Fused word bases + cell list: a single-pass scan with decoupled look-back over the popcounts
// of the occupancy words (tiles of 2048 words, taken in order from an atomic counter), the
// exclusive prefix stored next to each word's bits, then the tile's occupied cells emitted:
// lane per cell of each nonzero word, so consecutive occupied cells are written by consecutive
// lanes.  One pass over the bitmap, one launch (+ the state memset).
constexpr int CS_THREADS = 256, CS_ITEMS = 8, CS_TILE = CS_THREADS * CS_ITEMS;

__global__ void __launch_bounds__(CS_THREADS) k_cscan(uint2* __restrict__ cw, int64_t words,
                                                     uint32_t* __restrict__ clin, uint32_t* __restrict__ count,
                                                     u64* __restrict__ cocc, u64* __restrict__ ccoord, Grid g,
                                                     Meta* __restrict__ meta, unsigned long long* __restrict__ state,
                                                     unsigned int* __restrict__ counter) {
    pdl_prologue();
    __shared__ uint32_t s[CS_TILE];
    __shared__ uint32_t sbits[CS_TILE];  // the tile's words, for the emission (no reload)
    __shared__ uint32_t wsum[CS_THREADS / kWarp];
    __shared__ unsigned int tile_sh;
    __shared__ uint32_t prefix_sh;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) tile_sh = atomicAdd(counter, 1u);
    __syncthreads();
    const unsigned tile = tile_sh;
    const int64_t n = words + 1;  // the extra element yields U = the total
    const int64_t base = (int64_t)tile * CS_TILE;
    if (base >= n) return;
#pragma unroll
    for (int k = 0; k < CS_ITEMS; ++k) {
        const int64_t i = base + k * CS_THREADS + tid;
        const uint32_t b = i < words ? cw[i].x : 0u;
        sbits[k * CS_THREADS + tid] = b;
        s[k * CS_THREADS + tid] = (uint32_t)__popc(b);
    }
    __syncthreads();
    uint32_t loc[CS_ITEMS];
    uint32_t run = 0;
#pragma unroll
    for (int k = 0; k < CS_ITEMS; ++k) {
        const uint32_t v = s[tid * CS_ITEMS + k];
        loc[k] = run;
        run += v;
    }
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t v = lane < CS_THREADS / kWarp ? wsum[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        if (lane < CS_THREADS / kWarp) wsum[lane] = v;
        const unsigned long long agg = __shfl_sync(0xffffffffu, v, CS_THREADS / kWarp - 1);
        constexpr unsigned long long A = 1ull << 62, P = 2ull << 62, VAL = (1ull << 62) - 1;
        unsigned long long prefix = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(state, P | agg);
        } else {
            if (lane == 0) atomicExch(state + tile, A | agg);
            int j = (int)tile - 1;
            while (true) {
                const int idx = j - lane;
                const unsigned long long sv = idx >= 0 ? *reinterpret_cast<volatile unsigned long long*>(state + idx) : P;
                const unsigned pmask = __ballot_sync(0xffffffffu, (sv & ~VAL) == P);
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
    for (int k = 0; k < CS_ITEMS; ++k) s[tid * CS_ITEMS + k] = pre + loc[k];
    __syncthreads();
    // word bases next to the bits; then warp w emits the cells of words [w*256, w*256 + 256)
#pragma unroll
    for (int k = 0; k < CS_ITEMS; ++k) {
        const int64_t i = base + k * CS_THREADS + tid;
        if (i < words) {
            cw[i].y = s[k * CS_THREADS + tid];
        } else if (i == words) {
            const uint32_t U = s[k * CS_THREADS + tid];
            meta->cells = (int)U;
            meta->cells1 = (int)U + 1;
            count[U] = 0u;
        }
    }
    for (int c = 0; c < CS_ITEMS; ++c) {
        const int li = w * (CS_ITEMS * kWarp) + c * kWarp + lane;
        const uint32_t bits = sbits[li];
        unsigned m = __ballot_sync(0xffffffffu, bits != 0u);
        while (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1;
            const uint32_t b = __shfl_sync(0xffffffffu, bits, j);
            const uint32_t r0 = s[w * (CS_ITEMS * kWarp) + c * kWarp + j];
            if ((b >> lane) & 1u) {
                const uint32_t r = r0 + (uint32_t)__popc(b & ((1u << lane) - 1u));
                const uint32_t lin = (uint32_t)((base + w * (CS_ITEMS * kWarp) + c * kWarp + j) * 32 + lane);
                int cc[3];
                dense_decode(lin, g, cc);
                clin[r] = lin;
                ccoord[r] = (u64)cc[0] | ((u64)cc[1] << 21) | ((u64)cc[2] << 42);
                count[r] = 0u;
                cocc[r] = 0ull;
            }
        }
    }
}

// ---- a2: per-cell counts, slot[i] = rank of point i inside its cell, fine occupancy ------
// Warp per tile of 128 consecutive points (4 per lane), aggregated through a per-warp
// shared-memory table: one global atomicAdd (+ atomicOr) per distinct cell per tile and only
// warp-level synchronisation (the input order is spatially coherent on this path).
constexpr int kWTile = 128;
constexpr int kWSlots = 256;

__device__ __forceinline__ int wbin_slot(int* keys, uint32_t key, int* used, int* nused) {
    uint32_t h = (key * 2654435761u) & (kWSlots - 1);
    while (true) {  // a tile has at most 128 distinct cells: the 256-slot table never fills
        const int cur = keys[h];
        if (cur == (int)key) return (int)h;
        if (cur == -1) {
            const int old = atomicCAS(keys + h, -1, (int)key);
            if (old == -1) {
                used[atomicAdd(nused, 1)] = (int)h;
                return (int)h;
            }
            if (old == (int)key) return (int)h;
        }
        h = (h + 1) & (kWSlots - 1);
    }
}

// Counting without return values: per warp-tile cell counts and fine-occupancy bits are added
// to the cell's counters fire-and-forget (no dependent round trip); slots are assigned later
// by k_dscatter2 against per-cell cursors.
__global__ void __launch_bounds__(256) k_dcount2(const float* __restrict__ p, int64_t n, Grid g,
                                                const uint2* __restrict__ cw, uint32_t* __restrict__ count,
                                                u64* __restrict__ cocc) {
    pdl_prologue();
    __shared__ int keys_all[256 / kWarp][kWSlots];
    __shared__ uint32_t cnt_all[256 / kWarp][kWSlots], olo_all[256 / kWarp][kWSlots], ohi_all[256 / kWarp][kWSlots];
    __shared__ int used_all[256 / kWarp][kWTile];
    __shared__ int nused_all[256 / kWarp];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int* keys = keys_all[wid];
    uint32_t *cnt = cnt_all[wid], *olo = olo_all[wid], *ohi = ohi_all[wid];
    int* used = used_all[wid];
    int* nused = nused_all + wid;
    for (int k = lane; k < kWSlots; k += 32) { keys[k] = -1; cnt[k] = 0u; olo[k] = 0u; ohi[k] = 0u; }
    if (lane == 0) *nused = 0;
    __syncwarp();
    const bool vec = (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kWTile; t0 < n; t0 += nw * kWTile) {
        const int64_t b4 = t0 + 4 * lane;
        Pts4 P;
        load_pts4(p, n, b4, vec, P);
        // runs of this thread's points in one cell take one table update
        uint32_t rc = 0xffffffffu, rn = 0u;
        u64 rb = 0ull;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (b4 + j < n) {
                uint32_t lin;
                int q;
                dense_cell_of(P.x[j], P.y[j], P.z[j], b4 + j, g, lin, q);
                const uint32_t cid = cid_of(cw, lin);
                if (cid != rc) {
                    if (rn) {
                        const int h = wbin_slot(keys, rc, used, nused);
                        atomicAdd(cnt + h, rn);
                        if ((uint32_t)rb) atomicOr(olo + h, (uint32_t)rb);
                        if ((uint32_t)(rb >> 32)) atomicOr(ohi + h, (uint32_t)(rb >> 32));
                    }
                    rc = cid;
                    rn = 0u;
                    rb = 0ull;
                }
                ++rn;
                rb |= 1ull << q;
            }
        }
        if (rn) {
            const int h = wbin_slot(keys, rc, used, nused);
            atomicAdd(cnt + h, rn);
            if ((uint32_t)rb) atomicOr(olo + h, (uint32_t)rb);
            if ((uint32_t)(rb >> 32)) atomicOr(ohi + h, (uint32_t)(rb >> 32));
        }
        __syncwarp();
        const int nu = *nused;
        for (int e = lane; e < nu; e += 32) {
            const int k = used[e];
            const int cid = keys[k];
            atomicAdd(count + cid, cnt[k]);
            atomicOr(cocc + cid, ((u64)ohi[k] << 32) | (u64)olo[k]);
            keys[k] = -1;
            cnt[k] = 0u;
            olo[k] = 0u;
            ohi[k] = 0u;
        }
        __syncwarp();
        if (lane == 0) *nused = 0;
        __syncwarp();
    }
}

// Scatter into cell order: per warp-tile, one atomicAdd on the cell's cursor (initialised to
// the cell start) per distinct cell gives the tile's base; ranks inside the tile come from
// the warp's shared-memory table.
__global__ void __launch_bounds__(256) k_dscatter2(const float* __restrict__ p, int64_t n, Grid g,
                                                  const uint2* __restrict__ cw, uint32_t* __restrict__ cursor,
                                                  float4* __restrict__ spts) {
    pdl_prologue();
    __shared__ int keys_all[256 / kWarp][kWSlots];
    __shared__ uint32_t cnt_all[256 / kWarp][kWSlots];
    __shared__ int used_all[256 / kWarp][kWTile];
    __shared__ int nused_all[256 / kWarp];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int* keys = keys_all[wid];
    uint32_t* cnt = cnt_all[wid];
    int* used = used_all[wid];
    int* nused = nused_all + wid;
    for (int k = lane; k < kWSlots; k += 32) { keys[k] = -1; cnt[k] = 0u; }
    if (lane == 0) *nused = 0;
    __syncwarp();
    const bool vec = (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kWTile; t0 < n; t0 += nw * kWTile) {
        const int64_t b4 = t0 + 4 * lane;
        Pts4 P;
        load_pts4(p, n, b4, vec, P);
        int hs[4];
        uint32_t rk[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            hs[j] = -1;
            rk[j] = 0u;
            if (b4 + j < n) {
                uint32_t lin;
                int q;
                dense_cell_of(P.x[j], P.y[j], P.z[j], b4 + j, g, lin, q);
                const int h = wbin_slot(keys, cid_of(cw, lin), used, nused);
                hs[j] = h;
                rk[j] = atomicAdd(cnt + h, 1u);
            }
        }
        __syncwarp();
        const int nu = *nused;
        for (int e = lane; e < nu; e += 32) {
            const int k = used[e];
            cnt[k] = atomicAdd(cursor + keys[k], cnt[k]);  // the tile's base inside the cell
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (hs[j] >= 0) spts[cnt[hs[j]] + rk[j]] = make_float4(P.x[j], P.y[j], P.z[j], __int_as_float((int)(b4 + j)));
        __syncwarp();
        for (int e = lane; e < nu; e += 32) {
            const int k = used[e];
            keys[k] = -1;
            cnt[k] = 0u;
        }
        if (lane == 0) *nused = 0;
        __syncwarp();
    }
}

// Dense bits of the occupied cells from the cell starts; also the scatter cursors.
__global__ void __launch_bounds__(256) k_ccount(const uint32_t* __restrict__ cstart, uint32_t* __restrict__ dbits,
                                               uint32_t* __restrict__ cursor, const Meta* __restrict__ meta) {
    pdl_prologue();
    const int64_t U = meta->cells;
    const int64_t ur = (U + 31) & ~int64_t(31);
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < ur; u += (int64_t)gridDim.x * blockDim.x) {
        bool dense = false;
        if (u < U) {
            const uint32_t c0 = __ldg(cstart + u);
            dense = __ldg(cstart + u + 1) - c0 > (uint32_t)SPARSE_MAX;
            cursor[u] = c0;
        }
        const unsigned m = __ballot_sync(0xffffffffu, dense);
        if ((threadIdx.x & 31) == 0) dbits[u >> 5] = m;
    }
}

// ---- a2/a3, sort path (shuffled inputs) ----------------------------------------------------
// For inputs without spatial coherence (C1, C5) the counting sort's per-point atomics and
// scatter hit random DRAM sectors; instead the linear cell ids are radix-sorted (coalesced
// digit passes), cells are the runs of equal keys, and points are gathered into cell order.
__global__ void __launch_bounds__(256) k_lkey(const float* __restrict__ p, int64_t n, Grid g, uint32_t* __restrict__ key,
                                             int* __restrict__ val) {
    pdl_prologue();
    const bool vec = (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
    const int64_t groups = (n + 3) / 4;
    for (int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < groups; gi += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b4 = 4 * gi;
        Pts4 P;
        load_pts4(p, n, b4, vec, P);
        uint32_t k[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int q;
            if (b4 + j < n) dense_cell_of(P.x[j], P.y[j], P.z[j], b4 + j, g, k[j], q);
        }
        if (b4 + 4 <= n) {
            *reinterpret_cast<uint4*>(key + b4) = make_uint4(k[0], k[1], k[2], k[3]);
            *reinterpret_cast<int4*>(val + b4) = make_int4((int)b4, (int)b4 + 1, (int)b4 + 2, (int)b4 + 3);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (b4 + j < n) {
                    key[b4 + j] = k[j];
                    val[b4 + j] = (int)(b4 + j);
                }
        }
    }
}

// Occupancy bits of the sorted keys' distinct values (heads only; a warp's heads share words).
__global__ void __launch_bounds__(256) k_smark(const uint32_t* __restrict__ key, int64_t n, uint2* __restrict__ cw) {
    pdl_prologue();
    const int64_t nr = (n + 31) & ~int64_t(31);
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nr; s += (int64_t)gridDim.x * blockDim.x) {
        const bool ok = s < n;
        const uint32_t k = ok ? __ldg(key + s) : 0u;
        const bool head = ok && (s == 0 || __ldg(key + s - 1) != k);
        const uint32_t w = head ? (k >> 5) : 0xffffffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, w);
        const uint32_t bits = __reduce_or_sync(peers, head ? (1u << (k & 31u)) : 0u);
        if (head && (threadIdx.x & 31) == __ffs(peers) - 1) atomicOr(reinterpret_cast<unsigned int*>(cw + w), bits);
    }
}

// Points into cell order (random 12-byte gathers, coalesced float4 stores), cell starts at
// the run heads, fine occupancy OR-ed per run (segmented within the warp, one atomic per run
// piece).
__global__ void __launch_bounds__(256) k_sgather(const float* __restrict__ p, const uint32_t* __restrict__ key,
                                                const int* __restrict__ val, int64_t n, Grid g,
                                                const uint2* __restrict__ cw, float4* __restrict__ spts,
                                                uint32_t* __restrict__ cstart, u64* __restrict__ cocc,
                                                int* __restrict__ parent, int* __restrict__ sidx,
                                                int* __restrict__ size, int* __restrict__ minidx,
                                                const Meta* __restrict__ meta) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    if (blockIdx.x == 0 && threadIdx.x == 0) cstart[meta->cells] = (uint32_t)n;
    // round j: positions s0 + j*256 + threadIdx.x (a warp holds 32 consecutive positions, so
    // the run reduction below works per round); the 4 rounds' gathers are issued together
    const int64_t per = 4 * (int64_t)blockDim.x;
    for (int64_t s0 = (int64_t)blockIdx.x * per; s0 < n; s0 += (int64_t)gridDim.x * per) {
        uint32_t k[4];
        int vi[4];
        float x[4], y[4], z[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t s = s0 + j * (int64_t)blockDim.x + threadIdx.x;
            k[j] = s < n ? __ldg(key + s) : 0xffffffffu;
            vi[j] = s < n ? __ldg(val + s) : 0;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            x[j] = y[j] = z[j] = 0.f;
            if (k[j] != 0xffffffffu) load_point(p, vi[j], x[j], y[j], z[j]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t s = s0 + j * (int64_t)blockDim.x + threadIdx.x;
            const bool ok = s < n;
            uint32_t cid = 0xffffffffu;
            u64 bit = 0;
            const uint32_t prev = __shfl_up_sync(0xffffffffu, k[j], 1);  // all lanes take part
            if (ok) {
                uint32_t lin;
                int q;
                dense_cell_of(x[j], y[j], z[j], vi[j], g, lin, q);
                cid = cid_of(cw, k[j]);
                bit = 1ull << q;
                spts[s] = make_float4(x[j], y[j], z[j], __int_as_float(vi[j]));
                sidx[s] = vi[j];
                parent[s] = (int)s;  // points of dense cells are re-parented by k_dparent
                size[s] = 0;
                minidx[s] = 0x7fffffff;
                const bool head = s == 0 || (lane > 0 ? prev != k[j] : __ldg(key + s - 1) != k[j]);
                if (head) cstart[cid] = (uint32_t)s;
            }
            // equal cids are contiguous: the last lane of each run publishes the run's OR
            const unsigned peers = __match_any_sync(0xffffffffu, cid);
            const uint32_t lo = __reduce_or_sync(peers, (uint32_t)bit);
            const uint32_t hi = __reduce_or_sync(peers, (uint32_t)(bit >> 32));
            if (ok && lane == 31 - __clz(peers)) atomicOr(cocc + cid, ((u64)hi << 32) | lo);
        }
    }
}

// Dense bits of the occupied cells from the run lengths (lanes = consecutive compact ids,
// so a warp fills one bitmap word with a plain store).
__global__ void __launch_bounds__(256) k_scount(const uint32_t* __restrict__ cstart, uint32_t* __restrict__ dbits,
                                               const Meta* __restrict__ meta) {
    pdl_prologue();
    const int64_t U = meta->cells;
    const int64_t ur = (U + 31) & ~int64_t(31);
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < ur; u += (int64_t)gridDim.x * blockDim.x) {
        const bool dense = u < U && __ldg(cstart + u + 1) - __ldg(cstart + u) > (uint32_t)SPARSE_MAX;
        const unsigned m = __ballot_sync(0xffffffffu, dense);
        if ((threadIdx.x & 31) == 0) dbits[u >> 5] = m;
    }
}

// ---- dense records: compact ids of the dense cells in ascending order -----------------------
__global__ void __launch_bounds__(256) k_dbits_popc(const uint32_t* __restrict__ dbits, int64_t words,
                                                   uint32_t* __restrict__ wcount) {
    pdl_prologue();
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w <= words; w += (int64_t)gridDim.x * blockDim.x)
        wcount[w] = w < words ? (uint32_t)__popc(__ldg(dbits + w)) : 0u;
}

__global__ void __launch_bounds__(256) k_dbits_list(const uint32_t* __restrict__ dbits, int64_t words,
                                                   const uint32_t* __restrict__ wpos, int* __restrict__ dlist,
                                                   int* __restrict__ crec, Meta* __restrict__ meta) {
    pdl_prologue();
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w <= words; w += (int64_t)gridDim.x * blockDim.x) {
        if (w == words) { meta->ndense = (int)wpos[words]; continue; }
        uint32_t bits = __ldg(dbits + w);
        int r = (int)__ldg(wpos + w);
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int cell = (int)(w * 32 + b);
            dlist[r] = cell;
            crec[cell] = r;
            ++r;
        }
    }
}

// ---- uncertain component pairs: queued, or tested in place when the queue is full ----------
// item = (P record, P component, Q record or point, Q component or -1 for a point)

__device__ __forceinline__ int cell_slot_of(const Grid& g, uint32_t lin_p, uint32_t lin_q) {
    int a[3], b[3];
    dense_decode(lin_p, g, a);
    dense_decode(lin_q, g, b);
    return sc_slot(b[0] - a[0], b[1] - a[1], b[2] - a[2]);
}

__device__ __forceinline__ u64 reach_of(const u64 m, int slot) {
    u64 r = 0;
    u64 b = m & d_sc.F[slot];
    while (b) {
        const int a = __ffsll((long long)b) - 1;
        b &= b - 1;
        r |= d_sc.U[slot][a];
    }
    return r;
}

// One thread tests an uncertain item by itself (queue overflow path; slow but rare).
__device__ __noinline__ void test_item_serial(const DenseCtx& C, const Grid& g, int4 it) {
    const float t2 = g.t2;
    const int cp = __ldg(C.dlist + it.x);
    const uint32_t lp = __ldg(C.clin + cp);
    const u64 ma = C.cmask[8 * it.x + it.y];
    const int na = C.nbase + 8 * it.x + it.y;
    int nb, b0, b1;
    u64 mb;
    int slot;
    if (it.w >= 0) {
        const int cq = __ldg(C.dlist + it.z);
        mb = C.cmask[8 * it.z + it.w];
        nb = C.nbase + 8 * it.z + it.w;
        b0 = (int)__ldg(C.cstart + cq);
        b1 = (int)__ldg(C.cstart + cq + 1);
        slot = cell_slot_of(g, lp, __ldg(C.clin + cq));
    } else {
        mb = ~0ull;
        nb = it.z;
        b0 = it.z;
        b1 = it.z + 1;
        uint32_t lq;
        int qq;
        const float4 v = C.spts[it.z];
        dense_cell_of(v.x, v.y, v.z, __float_as_int(v.w), g, lq, qq);
        slot = cell_slot_of(g, lp, lq);
    }
    const int a0 = (int)__ldg(C.cstart + cp), a1 = (int)__ldg(C.cstart + cp + 1);
    for (int i = a0; i < a1; ++i) {
        const float4 pa = C.spts[i];
        uint32_t l;
        int qa;
        dense_cell_of(pa.x, pa.y, pa.z, __float_as_int(pa.w), g, l, qa);
        if (!((ma >> qa) & 1ull)) continue;
        const u64 reach = d_sc.U[slot][qa];
        for (int j = b0; j < b1; ++j) {
            const float4 pb = C.spts[j];
            int qb;
            dense_cell_of(pb.x, pb.y, pb.z, __float_as_int(pb.w), g, l, qb);
            if (it.w >= 0 && !(((mb & reach) >> qb) & 1ull)) continue;
            if (pred(pa, pb, t2)) {
                uf_unite(C.parent, na, nb);
                return;
            }
        }
    }
}

// Queue a pair of nodes that may need point tests.  The lanes that push together share one
// atomicAdd.  Returns false when the queue is full (the caller marks the slot for
// k_dense_overflow, which tests such pairs in place).
__device__ __forceinline__ bool queue_item(const DenseCtx& C, int4 it) {
    const unsigned m = __activemask();
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(&C.meta->nitems, __popc(m));
    base = __shfl_sync(m, base, leader);
    const int k = base + __popc(m & ((1u << lane) - 1u));
    if (k >= C.item_cap) return false;
    C.items[k] = it;
    return true;
}

// ---- dense records: components of the fine occupancy, node init, in-cell uncertain pairs --
__global__ void __launch_bounds__(256) k_dcomps(Grid g, const u64* __restrict__ cocc, const u64* __restrict__ ccoord,
                                               int* __restrict__ ncomp,
                                               int* __restrict__ size, int* __restrict__ minidx,
                                               u64* __restrict__ dcoord, uint32_t* __restrict__ oflags, DenseCtx C) {
    pdl_prologue();
    const int nd = C.meta->ndense;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nd; r += gridDim.x * blockDim.x) {
        const int cid = __ldg(C.dlist + r);
        const u64 occ = __ldg(cocc + cid);
        dcoord[r] = __ldg(ccoord + cid);
        oflags[r] = 0u;
        u64 comp[kMaxComp];
        u64 rest;
        const int k = sc_components(occ, comp, rest);
        if (rest) atomicOr(&C.meta->internal_error, 1);  // impossible by the 8-component bound
        ncomp[r] = k;
#pragma unroll
        for (int j = 0; j < kMaxComp; ++j) {
            const int node = C.nbase + 8 * r + j;
            C.parent[node] = node;
            size[node] = 0;
            minidx[node] = 0x7fffffff;
            C.cmask[8 * r + j] = j < k ? comp[j] : 0ull;
        }
    }
}

// Node-level statistics (single-GPU tail of clouds with few sparse cells):
// points of dense cells add their count and minimum input index to their component node's own
// accumulators while parents are assigned; k_node_stats later moves each node's totals to its
// root, so the tail never walks the dense points.  Warp-aggregated: one atomic per distinct
// node among the warp's points of this round (key < 0 = not a dense point).
__device__ __forceinline__ void node_accumulate(int key, int si, int* __restrict__ size, int* __restrict__ minidx) {
    const int lane = threadIdx.x & 31;
    const bool ok = key >= 0;
    unsigned todo = __ballot_sync(0xffffffffu, ok);
    while (todo) {
        const int leader = __ffs(todo) - 1;
        const int k = __shfl_sync(0xffffffffu, key, leader);
        const bool mem = ok && key == k;
        const unsigned peers = __ballot_sync(0xffffffffu, mem);
        const int mn = __reduce_min_sync(0xffffffffu, mem ? si : 0x7fffffff);
        if (lane == leader) {
            atomicAdd(size + k, __popc(peers));
            atomicMin(minidx + k, mn);
        }
        todo &= ~peers;
    }
}

// Sorted-order initialisation (coalesced): points of sparse cells are their own parents,
// points of dense cells hang under their component's node; accumulators; input index.
__global__ void __launch_bounds__(256) k_dinit(const float4* __restrict__ spts, int64_t n, Grid g,
                                              const uint2* __restrict__ cw, const uint32_t* __restrict__ cstart,
                                              const int* __restrict__ crec, const int* __restrict__ ncomp,
                                              const u64* __restrict__ cmask, int nbase, int* __restrict__ parent,
                                              int* __restrict__ size, int* __restrict__ minidx,
                                              int* __restrict__ sidx, const Meta* __restrict__ meta, int node_stats) {
    pdl_prologue();
    const int64_t groups = (n + 3) / 4;
    const bool nstats = node_stats && 4 * (int64_t)meta->cells <= n;  // warp-uniform
    for (int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < groups; gi += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b4 = 4 * gi;
        float4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = b4 + j < n ? __ldg(spts + b4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        int par[4], si[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            par[j] = (int)(b4 + j);
            si[j] = __float_as_int(v[j].w);
            if (b4 + j >= n) continue;
            uint32_t lin;
            int q;
            dense_cell_of(v[j].x, v[j].y, v[j].z, __float_as_int(v[j].w), g, lin, q);
            const uint32_t cid = cid_of(cw, lin);
            if (__ldg(cstart + cid + 1) - __ldg(cstart + cid) > (uint32_t)SPARSE_MAX) {
                const int r = __ldg(crec + cid);
                const int k = __ldg(ncomp + r);
                int c = 0;
                if (k > 1)
                    while (c < k - 1 && !((__ldg(cmask + 8 * r + c) >> q) & 1ull)) ++c;
                par[j] = nbase + 8 * r + c;
            }
        }
        // accumulators of the possible root points (points of sparse cells); points of dense
        // cells hang under component nodes and never become roots
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (b4 + j < n && par[j] == (int)(b4 + j)) {
                size[b4 + j] = 0;
                minidx[b4 + j] = 0x7fffffff;
            }
        if (nstats) {
            // the thread's 4 consecutive positions mostly share one node: runs first, then the
            // first run of every lane aggregated over the warp by a labelled partition
            int key0 = -1, cnt0 = 0, min0 = 0x7fffffff;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int key = b4 + j < n && par[j] >= nbase ? par[j] : -1;
                if (key < 0) continue;
                if (key0 < 0 || key == key0) {
                    key0 = key;
                    ++cnt0;
                    min0 = min(min0, si[j]);
                } else {  // a second node inside the thread's 4 points (cell or component edge)
                    atomicAdd(size + key, 1);
                    atomicMin(minidx + key, si[j]);
                }
            }
            // lanes past the end left the grid-stride loop: aggregate over the ones still here
            const unsigned peers = __match_any_sync(__activemask(), key0);
            const int tot = __reduce_add_sync(peers, cnt0);
            const int mn = __reduce_min_sync(peers, min0);
            if (key0 >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) {
                atomicAdd(size + key0, tot);
                atomicMin(minidx + key0, mn);
            }
        }
        if (b4 + 4 <= n) {
            *reinterpret_cast<int4*>(parent + b4) = make_int4(par[0], par[1], par[2], par[3]);
            *reinterpret_cast<int4*>(sidx + b4) = make_int4(si[0], si[1], si[2], si[3]);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (b4 + j < n) {
                    parent[b4 + j] = par[j];
                    sidx[b4 + j] = si[j];
                }
        }
    }
}

// Key-sort path: points of dense cells hang under their component nodes (warp per dense
// record; the cell's points are contiguous).  k_sgather made every point its own parent.
__global__ void __launch_bounds__(256) k_dparent(const float4* __restrict__ spts, const uint32_t* __restrict__ cstart,
                                                const int* __restrict__ dlist, const int* __restrict__ ncomp,
                                                const u64* __restrict__ cmask, Grid g, int nbase,
                                                int* __restrict__ parent, const Meta* __restrict__ meta,
                                                const int* __restrict__ sidx, int* __restrict__ size,
                                                int* __restrict__ minidx, int node_stats, int64_t n) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    const int nd = meta->ndense;
    const bool nstats = node_stats && 4 * (int64_t)meta->cells <= n;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nd; r += warps) {
        const int cid = __ldg(dlist + r);
        const int k = __ldg(ncomp + r);
        const int a0 = (int)__ldg(cstart + cid), a1 = (int)__ldg(cstart + cid + 1);
        for (int s0 = a0; s0 < a1; s0 += 32) {  // warp-uniform trip count
            const int s = s0 + lane;
            int key = -1;
            if (s < a1) {
                int cc = 0;
                if (k > 1) {
                    const float4 v = __ldg(spts + s);
                    uint32_t lin;
                    int q;
                    dense_cell_of(v.x, v.y, v.z, __float_as_int(v.w), g, lin, q);
                    while (cc < k - 1 && !((__ldg(cmask + 8 * r + cc) >> q) & 1ull)) ++cc;
                }
                key = nbase + 8 * r + cc;
                parent[s] = key;
            }
            if (nstats) node_accumulate(key, s < a1 ? __ldg(sidx + s) : 0x7fffffff, size, minidx);
        }
    }
}


// ---- a6+a7: dense cells — certain unions across cells, uncertain pairs queued -------------
// Thread per dense record P, looping over the 26 neighbour slots in the same order in every
// thread (warp-uniform slot -> broadcast table reads): forward dense neighbours give
// component pairs, sparse neighbours (both directions) give their points against P's
// components; slot 26 stands for the pairs of P's own components.  Each unordered pair of
// adjacent cells is therefore handled once.  Pass 0 makes the certain
// unions and records, per record, the slots that still hold a non-certain pair within
// reach; pass 1 (after all certain unions) queues those pairs whose nodes are still apart.

// One (dense record r, slot k) item: certain component pairs are united at once; pairs that
// are not certain but may be within reach and whose nodes are (so far) apart are queued
// (k_dense_filter re-checks them after every certain union, k_dense_items tests the rest).
// `serial` (overflow path): such pairs are tested in place by this thread instead.
// Slot order: 0-2 forward faces, 3-12 forward edges and corners, 13-25 backward, 26 = P's own
// components.
__constant__ signed char c_slot[26][3] = {
    {1, 0, 0},   {0, 1, 0},   {0, 0, 1},                                         // forward faces
    {-1, 1, 0},  {1, 1, 0},   {0, -1, 1}, {-1, 0, 1}, {1, 0, 1}, {0, 1, 1},      // forward edges
    {-1, -1, 1}, {1, -1, 1},  {-1, 1, 1}, {1, 1, 1},                             // forward corners
    {-1, 0, 0},  {0, -1, 0},  {0, 0, -1},                                        // backward ...
    {1, -1, 0},  {-1, -1, 0}, {0, 1, -1}, {1, 0, -1}, {-1, 0, -1}, {0, -1, -1},
    {1, 1, -1},  {-1, 1, -1}, {1, -1, -1}, {-1, -1, -1}};

template <bool serial>
__device__ __forceinline__ void dense_link_item(int r, int k, const Grid& g, const uint2* __restrict__ cw,
                                                const int* __restrict__ crec, const int* __restrict__ ncomp,
                                                const u64* __restrict__ dcoord, uint32_t* __restrict__ oflags,
                                                const DenseCtx& C) {
    const int kp = __ldg(ncomp + r);
    const u64* mp = C.cmask + 8 * r;
    bool overflow = false;
    if (k == 26) {
        // P's own components (never certain-adjacent to each other)
        for (int i = 0; i + 1 < kp; ++i)
            for (int j = i + 1; j < kp; ++j) {
                const int na = C.nbase + 8 * r + i, nb = C.nbase + 8 * r + j;
                if (uf_find(C.parent, na) == uf_find(C.parent, nb)) continue;
                if constexpr (serial) test_item_serial(C, g, make_int4(r, i, r, j));
                else overflow |= !queue_item(C, make_int4(r, i, r, j));
            }
    } else {
        const u64 pc = __ldg(dcoord + r);
        const int c[3] = {(int)(pc & 0x1fffff), (int)((pc >> 21) & 0x1fffff), (int)(pc >> 42)};
        const int ox = c_slot[k][0], oy = c_slot[k][1], oz = c_slot[k][2];
        uint32_t lq;
        const int cq = dense_neighbor(g, c, ox, oy, oz, lq) ? cid_lookup(cw, lq) : -1;
        if (cq < 0) return;
        const int q0 = (int)__ldg(C.cstart + cq), q1 = (int)__ldg(C.cstart + cq + 1);
        const int slot = sc_slot(ox, oy, oz);
        if (q1 - q0 > SPARSE_MAX) {
            if (k >= 13) return;  // backward dense pairs belong to the other cell
            const int rq = __ldg(crec + cq);
            const int kq = __ldg(ncomp + rq);
            for (int x = 0; x < kp; ++x) {
                const u64 mx = mp[x];
                const u64 dc = sc_certain_across(d_sc, mx, slot);
                const bool near_p = (mx & d_sc.F[slot]) != 0;
                const int na = C.nbase + 8 * r + x;
                for (int y = 0; y < kq; ++y) {
                    const u64 my = C.cmask[8 * rq + y];
                    const int nb = C.nbase + 8 * rq + y;
                    if (dc & my) {
                        if constexpr (!serial) uf_unite(C.parent, na, nb);
                    } else if (near_p && (my & d_sc.F[26 - slot]) &&
                               uf_find(C.parent, na) != uf_find(C.parent, nb)) {
                        if constexpr (serial) test_item_serial(C, g, make_int4(r, x, rq, y));
                        else overflow |= !queue_item(C, make_int4(r, x, rq, y));
                    }
                }
            }
        } else {
            const int opp = 26 - slot;
            for (int t = q0; t < q1; ++t) {
                const float4 v = C.spts[t];
                uint32_t l;
                int qb;
                dense_cell_of(v.x, v.y, v.z, __float_as_int(v.w), g, l, qb);
                const u64 tc = d_sc.T[opp][qb], tu = d_sc.U[opp][qb];
                for (int x = 0; x < kp; ++x) {
                    const u64 mx = mp[x];
                    const int na = C.nbase + 8 * r + x;
                    if (tc & mx) {
                        if constexpr (!serial) uf_unite(C.parent, t, na);
                    } else if ((tu & mx) && uf_find(C.parent, na) != uf_find(C.parent, t)) {
                        if constexpr (serial) test_item_serial(C, g, make_int4(r, x, t, -1));
                        else overflow |= !queue_item(C, make_int4(r, x, t, -1));
                    }
                }
            }
        }
    }
    if (overflow) atomicOr(oflags + r, 1u << k);
}

// Slots [k0, k0 + gridDim.y) of every record (blockIdx.y = slot: a warp shares its slot).
// Launched for the face slots first, then the rest: by then most non-certain pairs of
// edge/corner neighbours are already connected through faces and are not queued.
__global__ void __launch_bounds__(256) k_dense_link(Grid g, const uint2* __restrict__ cw, const int* __restrict__ crec,
                                                   const int* __restrict__ ncomp, const u64* __restrict__ dcoord,
                                                   uint32_t* __restrict__ oflags, DenseCtx C, int k0) {
    pdl_prologue();
    const int nd = C.meta->ndense;
    const int k = k0 + blockIdx.y;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nd; r += gridDim.x * blockDim.x)
        dense_link_item<false>(r, k, g, cw, crec, ncomp, dcoord, oflags, C);
}

// Queue overflow: the marked slots' pairs are tested in place (one thread per record).
__global__ void __launch_bounds__(256) k_dense_overflow(Grid g, const uint2* __restrict__ cw,
                                                       const int* __restrict__ crec, const int* __restrict__ ncomp,
                                                       const u64* __restrict__ dcoord, uint32_t* __restrict__ oflags,
                                                       DenseCtx C) {
    pdl_prologue();
    const int nd = C.meta->ndense;
    if (C.meta->nitems <= C.item_cap) return;  // nothing overflowed
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nd; r += gridDim.x * blockDim.x) {
        uint32_t f = oflags[r];
        while (f) {
            const int k = __ffs(f) - 1;
            f &= f - 1;
            dense_link_item<true>(r, k, g, cw, crec, ncomp, dcoord, oflags, C);
        }
    }
}

// Queued pairs whose nodes are already connected (after all certain unions) are dropped;
// the others are compacted into items2 for k_dense_items.
// Heavy pairs (two big cells) are split over several warps along B's range: sub-item
// (k, K) tests B's k-th of K slices, and a per-pair flag stops the others at the first hit.
constexpr int kSliceWork = 4096;   // cell-size product per slice
constexpr int kMaxSlices = 128;

__global__ void __launch_bounds__(256) k_dense_filter(Grid g, DenseCtx C, int4* __restrict__ items2,
                                                     int4* __restrict__ slices2, int* __restrict__ idone) {
    pdl_prologue();
    const int ni = min(C.meta->nitems, C.item_cap);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ni; e += gridDim.x * blockDim.x) {
        const int4 it = C.items[e];  // queued before every certain union was done: re-check
        const int na = C.nbase + 8 * it.x + it.y;
        const int nb = it.w >= 0 ? C.nbase + 8 * it.z + it.w : it.z;
        if (uf_find(C.parent, na) == uf_find(C.parent, nb)) continue;
        const int cp = __ldg(C.dlist + it.x);
        const int wa = (int)(__ldg(C.cstart + cp + 1) - __ldg(C.cstart + cp));
        int wb = 1;
        if (it.w >= 0) {
            const int cq = __ldg(C.dlist + it.z);
            wb = (int)(__ldg(C.cstart + cq + 1) - __ldg(C.cstart + cq));
        }
        const long long work = (long long)wa * wb;
        int K = (int)min((long long)kMaxSlices, max(1ll, work / kSliceWork));
        K = min(K, wb);
        // items2 holds item_cap pairs plus item_cap extra slices: a pair whose extra slices
        // would not fit runs as one slice (there are at most item_cap surviving pairs)
        if (K > 1 && atomicAdd(&C.meta->nslices_extra, K - 1) + (K - 1) > C.item_cap) K = 1;
        idone[e] = 0;
        const int base = atomicAdd(&C.meta->nitems2, K);
        for (int k = 0; k < K; ++k) {
            items2[base + k] = it;
            slices2[base + k] = make_int4(k, K, e, 0);
        }
    }
}

// Component nodes -> their roots (shortens the finds of the uncertain pass).
__global__ void __launch_bounds__(256) k_flatten_nodes(int* __restrict__ parent, int nbase, const Meta* __restrict__ meta) {
    pdl_prologue();
    const int64_t nn = 8 * (int64_t)meta->ndense;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nn; t += (int64_t)gridDim.x * blockDim.x) {
        const int s = nbase + (int)t;
        int curr = ld_parent(parent, s), next;
        if (curr == s) continue;
        while (curr < (next = ld_parent(parent, curr))) curr = next;
        st_parent(parent, s, curr);
    }
}

// ---- a6+a7: queued uncertain pairs, warp per item, early exit ------------------------------
// A's points in sub-cells within reach of B are staged per lane (up to kAPer each, in
// batches); B's points stream through the warp 32 at a time and are broadcast by shuffle.
constexpr int kAPer = 4;

__global__ void __launch_bounds__(256) k_dense_items(Grid g, DenseCtx C, const int4* __restrict__ items2,
                                                    const int4* __restrict__ slices2, int* __restrict__ idone) {
    pdl_prologue();
    __shared__ float4 abuf_all[256 / kWarp][32 * kAPer];
    const int lane = threadIdx.x & 31;
    float4* abuf = abuf_all[threadIdx.x >> 5];
    const float t2 = g.t2;
    const int ni = C.meta->nitems2;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    unsigned long long n_tests = 0;
    for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < ni; w += warps) {
        const int4 it = items2[w];
        const int4 sl = slices2[w];
        volatile int* done = idone + sl.z;
        const int na = C.nbase + 8 * it.x + it.y;
        const int nb = it.w >= 0 ? C.nbase + 8 * it.z + it.w : it.z;
        int same = 0;
        if (lane == 0) same = *done || uf_find(C.parent, na) == uf_find(C.parent, nb);
        if (__shfl_sync(0xffffffffu, same, 0)) continue;
        const int cp = __ldg(C.dlist + it.x);
        const uint32_t lp = __ldg(C.clin + cp);
        const u64 ma = C.cmask[8 * it.x + it.y];
        int b0, b1, slot;
        u64 fa, fb;  // sub-cells of A within reach of B, and of B within reach of A
        if (it.w >= 0) {
            const int cq = __ldg(C.dlist + it.z);
            const u64 mb = C.cmask[8 * it.z + it.w];
            b0 = (int)__ldg(C.cstart + cq);
            b1 = (int)__ldg(C.cstart + cq + 1);
            slot = cell_slot_of(g, lp, __ldg(C.clin + cq));
            fb = reach_of(ma, slot) & mb;
            fa = reach_of(mb, 26 - slot) & ma;
            // this sub-item's slice of B
            const int len = b1 - b0;
            const int s0 = b0 + (int)(((long long)len * sl.x) / sl.y), s1 = b0 + (int)(((long long)len * (sl.x + 1)) / sl.y);
            b0 = s0;
            b1 = s1;
        } else {
            b0 = it.z;
            b1 = it.z + 1;
            const float4 v = C.spts[it.z];
            uint32_t lq;
            int qb;
            dense_cell_of(v.x, v.y, v.z, __float_as_int(v.w), g, lq, qb);
            slot = cell_slot_of(g, lp, lq);
            fb = ~0ull;
            fa = d_sc.U[26 - slot][qb] & ma;
        }
        const int a0 = (int)__ldg(C.cstart + cp), a1 = (int)__ldg(C.cstart + cp + 1);
        bool found = false;
        int ai = a0;
        while (ai < a1 && !found) {
            if (__shfl_sync(0xffffffffu, lane == 0 ? *done : 0, 0)) break;  // another slice found it
            // stage the next batch of A points (via shared memory): batch position k ends up in
            // lane k % 32, entry k / 32
            float4 pa[kAPer];
#pragma unroll
            for (int e = 0; e < kAPer; ++e) pa[e] = make_float4(0.f, 0.f, 0.f, 0.f);
            int total = 0;
            while (ai < a1) {
                const int i = ai + lane;
                bool v = false;
                float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
                if (i < a1) {
                    p = C.spts[i];
                    uint32_t l;
                    int qa;
                    dense_cell_of(p.x, p.y, p.z, __float_as_int(p.w), g, l, qa);
                    v = (fa >> qa) & 1ull;
                }
                const unsigned m = __ballot_sync(0xffffffffu, v);
                const int cnt = __popc(m);
                if (total + cnt > 32 * kAPer) break;  // this chunk starts the next batch
                if (v) abuf[total + __popc(m & ((1u << lane) - 1u))] = p;
                total += cnt;
                ai += 32;
            }
            __syncwarp();
            if (total == 0) continue;
            int na_l = (total - lane + 31) / 32;  // entries this lane holds
            na_l = na_l > kAPer ? kAPer : (na_l < 0 ? 0 : na_l);
#pragma unroll
            for (int e = 0; e < kAPer; ++e)
                if (e < na_l) pa[e] = abuf[e * 32 + lane];
            __syncwarp();
            for (int j0 = b0; j0 < b1 && !found; j0 += 32) {
                const int j = j0 + lane;
                float4 pb = make_float4(0.f, 0.f, 0.f, 0.f);
                bool vb = false;
                if (j < b1) {
                    pb = C.spts[j];
                    uint32_t l;
                    int qb;
                    dense_cell_of(pb.x, pb.y, pb.z, __float_as_int(pb.w), g, l, qb);
                    vb = (fb >> qb) & 1ull;
                }
                unsigned mb = __ballot_sync(0xffffffffu, vb);
                while (mb && !found) {
                    const int src = __ffs(mb) - 1;
                    mb &= mb - 1;
                    float4 q;
                    q.x = __shfl_sync(0xffffffffu, pb.x, src);
                    q.y = __shfl_sync(0xffffffffu, pb.y, src);
                    q.z = __shfl_sync(0xffffffffu, pb.z, src);
                    bool hit = false;
#pragma unroll
                    for (int e = 0; e < kAPer; ++e)
                        if (e < na_l) hit |= pred(pa[e], q, t2);
                    n_tests += (unsigned long long)na_l;
                    found = __any_sync(0xffffffffu, hit);
                }
            }
        }
        if (found && lane == 0) {
            *done = 1;
            uf_unite(C.parent, na, nb);
        }
        __syncwarp();
    }
    if (C.meta->instrument) {
        for (int o = 16; o > 0; o >>= 1) n_tests += __shfl_xor_sync(0xffffffffu, n_tests, o);
        if (lane == 0 && n_tests) atomicAdd(&C.meta->dense_tests, n_tests);
    }
}

// Instrumentation: dense-mode roots that are component nodes (points count themselves in
// k_stats) and the number of dense points.
__global__ void __launch_bounds__(256) k_dense_count(const int* __restrict__ ncomp, const int* __restrict__ dlist,
                                                    const uint32_t* __restrict__ cstart, DenseCtx C) {
    pdl_prologue();
    const int nd = C.meta->ndense;
    unsigned long long roots = 0, pts = 0;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nd; r += gridDim.x * blockDim.x) {
        const int k = ncomp[r];
        for (int j = 0; j < k; ++j) roots += C.parent[C.nbase + 8 * r + j] == C.nbase + 8 * r + j;
        const int cid = dlist[r];
        pts += cstart[cid + 1] - cstart[cid];
    }
    for (int o = 16; o > 0; o >>= 1) {
        roots += __shfl_xor_sync(0xffffffffu, roots, o);
        pts += __shfl_xor_sync(0xffffffffu, pts, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (roots) atomicAdd(&C.meta->components, roots);
        if (pts) atomicAdd(&C.meta->dense_points, pts);
    }
}

// Sparse cells.  The grid is one resident wave; each warp grid-strides over chunks of
// SP_CHUNK consecutive cells (so the wave sweeps the sorted order upwards), compacts the
// chunk's nonempty sparse cells into a per-warp list and gives every lane a real cell.
// Loops are warp-uniform with a reconvergence point per neighbour (SIMT efficiency).
constexpr int SP_CHUNK = 32;

// Sparse-dominated clouds (occupied cells > n/4, ~1-2 points per cell): lane per sparse
// cell, its own pairs and every sparse forward neighbour's points (dense neighbours are
// handled by k_dense_link).  Clouds with few sparse cells use k_union_sparse_local instead;
// both are launched and the one not chosen returns at once.
__device__ __forceinline__ void union_sparse_body(const float4* __restrict__ spts, const uint2* __restrict__ cw,
                                                  const u64* __restrict__ ccoord, const uint32_t* __restrict__ cstart,
                                                  const Grid& g, int* __restrict__ parent, Meta* __restrict__ meta,
                                                  int64_t n) {
    if (4 * (int64_t)meta->cells <= n) return;
    const uint32_t cells = (uint32_t)meta->cells;  // occupied cells (compact ids)
    __shared__ uint32_t lists[256 / kWarp][SP_CHUNK];
    unsigned long long n_tests = 0;
    const float t2 = g.t2;
    const int lane = threadIdx.x & 31;
    uint32_t* list = lists[threadIdx.x >> 5];
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t base = warp * SP_CHUNK; base < cells; base += nwarps * SP_CHUNK) {
        int total = 0;
#pragma unroll
        for (int j = 0; j < SP_CHUNK / 32; ++j) {
            const uint32_t P = base + j * 32 + lane;
            bool act = false;
            if (P < cells) {
                const int cnt = (int)__ldg(cstart + P + 1) - (int)__ldg(cstart + P);
                act = cnt > 0 && cnt <= SPARSE_MAX;
            }
            const unsigned m = __ballot_sync(0xffffffffu, act);
            if (act) list[total + __popc(m & ((1u << lane) - 1u))] = P;
            total += __popc(m);
        }
        __syncwarp();
        for (int e0 = 0; e0 < total; e0 += 32) {
            const int e = e0 + lane;
            const bool v = e < total;
            const uint32_t P = v ? list[e] : 0u;
            const int ps = v ? (int)__ldg(cstart + P) : 0;
            const int pe = v ? (int)__ldg(cstart + P + 1) : 0;
            for (int s = ps; s < pe; ++s) {
                const float4 a = __ldg(spts + s);
                for (int t = s + 1; t < pe; ++t) {
                    ++n_tests;
                    if (pred(a, __ldg(spts + t), t2)) uf_unite(parent, s, t);
                }
            }
            __syncwarp();
            const u64 pc = v ? __ldg(ccoord + P) : 0ull;
            const int c[3] = {(int)(pc & 0x1fffff), (int)((pc >> 21) & 0x1fffff), (int)(pc >> 42)};
#pragma unroll 1
            for (int k = 0; k < 13; ++k) {
                uint32_t Q;
                int qs = 0, qe = 0, qc = -1;
                if (v && dense_neighbor(g, c, c_fwd[k][0], c_fwd[k][1], c_fwd[k][2], Q)) qc = cid_lookup(cw, Q);
                if (qc >= 0) {
                    qs = (int)__ldg(cstart + qc);
                    qe = (int)__ldg(cstart + qc + 1);
                    if (qe - qs > SPARSE_MAX) qe = qs;  // dense neighbours are handled by k_dense_link
                }
                for (int s = ps; s < pe && qe > qs; ++s) {
                    const float4 a = __ldg(spts + s);
                    for (int t = qs; t < qe; ++t) {
                        ++n_tests;
                        if (pred(a, __ldg(spts + t), t2)) uf_unite(parent, s, t);
                    }
                }
                __syncwarp();
            }
        }
        __syncwarp();
    }
    if (meta->instrument) {
        for (int o = 16; o > 0; o >>= 1) n_tests += __shfl_xor_sync(0xffffffffu, n_tests, o);
        if (lane == 0 && n_tests) atomicAdd(&meta->pair_tests, n_tests);
    }
}

// LOCAL clouds: the sparse cells in one compact list, so every lane of the union kernel owns a
// real sparse cell and all of them run in one wave.
__global__ void __launch_bounds__(256) k_slist(const uint32_t* __restrict__ cstart, int* __restrict__ slist,
                                              Meta* __restrict__ meta, int64_t n) {
    pdl_prologue();
    if (4 * (int64_t)meta->cells > n) return;  // sparse-dominated: k_union_sparse walks the cells itself
    const int64_t U = meta->cells;
    const int64_t ur = (U + 31) & ~int64_t(31);
    const int lane = threadIdx.x & 31;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < ur; u += (int64_t)gridDim.x * blockDim.x) {
        bool sp = false;
        if (u < U) {
            const uint32_t c = __ldg(cstart + u + 1) - __ldg(cstart + u);
            sp = c > 0 && c <= (uint32_t)SPARSE_MAX;
        }
        const unsigned m = __ballot_sync(0xffffffffu, sp);
        if (!m) continue;
        int base = 0;
        if (lane == 0) base = atomicAdd(&meta->nsparse, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (sp) slist[base + __popc(m & ((1u << lane) - 1u))] = (int)u;
    }
}

__global__ void __launch_bounds__(256) k_union_sparse(const float4* __restrict__ spts, const uint2* __restrict__ cw,
                                                     const u64* __restrict__ ccoord,
                                                     const uint32_t* __restrict__ cstart, Grid g,
                                                     int* __restrict__ parent, Meta* __restrict__ meta, int64_t n) {
    pdl_prologue();
    union_sparse_body(spts, cw, ccoord, cstart, g, parent, meta, n);
}
// Node-level tail (see node_accumulate): every used component node finds its root, is
// flattened onto it, and adds its own totals to the root's; then the points of sparse cells
// (the compact list of k_slist) find their roots, are flattened and counted one by one.
// Only for dense-grid clouds with few sparse cells; the others run k_flat_stats / k_stats.




// LOCAL clouds have few sparse cells (C4: 73k of 358k cells, 0.8% of the points), so the
// kernel is a few short waves whose time is the dependent-load chain per cell.  16 lanes per
// sparse cell P (<= 6 points): lane l tests P's own pair l (15 pairs), the ballot gives P's
// local components (3-bit labels = min local index) and lanes 1..5 unite each point with its
// label; then lane k < 13 takes forward neighbour k and unites a neighbour point once per
// local component of P it touches.
__constant__ unsigned char c_pair_s[16] = {0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 3, 3, 4, 7};
__constant__ unsigned char c_pair_t[16] = {1, 2, 3, 4, 5, 2, 3, 4, 5, 3, 4, 5, 4, 5, 5, 7};
static_assert(SPARSE_MAX <= 6, "16-lane sparse kernel covers <= 15 own pairs");
__global__ void __launch_bounds__(256) k_union_sparse_local(const float4* __restrict__ spts,
                                                           const uint2* __restrict__ cw,
                                                           const u64* __restrict__ ccoord,
                                                           const uint32_t* __restrict__ cstart,
                                                           const int* __restrict__ slist, Grid g,
                                                           int* __restrict__ parent, Meta* __restrict__ meta,
                                                           int64_t n) {
    pdl_prologue();
    if (4 * (int64_t)meta->cells > n) return;
    const uint32_t nitems = (uint32_t)meta->nsparse;
    const int lane = threadIdx.x & 31, sub = lane & 15, half = lane >> 4;
    const float t2 = g.t2;
    unsigned long long n_tests = 0;
    const uint32_t stride = (gridDim.x * blockDim.x) >> 4;
    const uint32_t warp0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 2;
    for (uint32_t base = warp0; base < nitems; base += stride) {  // warp-uniform trip count
        const uint32_t it = base + half;
        const bool valid = it < nitems;
        int ps = 0, np = 0;
        uint32_t P = 0;
        if (valid) {
            P = (uint32_t)__ldg(slist + it);
            ps = (int)__ldg(cstart + P);
            np = (int)__ldg(cstart + P + 1) - ps;
        }
        // own pairs, one per lane
        const int ls = c_pair_s[sub], lt = c_pair_t[sub];
        bool e = false;
        if (valid && lt < np) {
            ++n_tests;
            e = pred(__ldg(spts + ps + ls), __ldg(spts + ps + lt), t2);
        }
        const unsigned em = (__ballot_sync(0xffffffffu, e) >> (16 * half)) & 0x7fffu;
        // closure over <= 6 nodes: reach[i] as 6-bit masks
        uint32_t r[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) r[i] = 1u << i;
#pragma unroll
        for (int p = 0; p < 15; ++p)
            if ((em >> p) & 1u) {
                const int a = (p < 5) ? 0 : (p < 9) ? 1 : (p < 12) ? 2 : (p < 14) ? 3 : 4;
                const int b = (p < 5) ? p + 1 : (p < 9) ? p - 3 : (p < 12) ? p - 6 : (p < 14) ? p - 8 : 5;
                r[a] |= 1u << b;
                r[b] |= 1u << a;
            }
#pragma unroll
        for (int round = 0; round < 3; ++round)
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                uint32_t acc = r[i];
#pragma unroll
                for (int j = 0; j < 6; ++j)
                    if ((r[i] >> j) & 1u) acc |= r[j];
                r[i] = acc;
            }
        uint32_t lab = 0;  // 3-bit label (min local index of the component) per local point
#pragma unroll
        for (int i = 0; i < 6; ++i) lab |= (uint32_t)(__ffs(r[i]) - 1) << (3 * i);
        if (valid && sub >= 1 && sub < np) {
            const int l = (int)((lab >> (3 * sub)) & 7u);
            if (l != sub) uf_unite(parent, ps + sub, ps + l);
        }
        // forward neighbour `sub`
        if (!valid || sub >= 13) continue;
        const u64 pc = __ldg(ccoord + P);
        const int c[3] = {(int)(pc & 0x1fffff), (int)((pc >> 21) & 0x1fffff), (int)(pc >> 42)};
        uint32_t Q;
        if (!dense_neighbor(g, c, c_fwd[sub][0], c_fwd[sub][1], c_fwd[sub][2], Q)) continue;
        const int qc = cid_lookup(cw, Q);
        if (qc < 0) continue;
        const int qs = (int)__ldg(cstart + qc), qe = (int)__ldg(cstart + qc + 1);
        if (qe - qs > SPARSE_MAX) continue;  // dense neighbours are handled by k_dense_link
        for (int t = qs; t < qe; ++t) {
            const float4 b = __ldg(spts + t);
            uint32_t touched = 0;  // local components of P within d of t
            for (int s2 = 0; s2 < np; ++s2) {
                ++n_tests;
                if (pred(__ldg(spts + ps + s2), b, t2)) touched |= 1u << ((lab >> (3 * s2)) & 7u);
            }
            while (touched) {
                const int l = __ffs(touched) - 1;
                touched &= touched - 1;
                uf_unite(parent, ps + l, t);
            }
        }
    }
    if (meta->instrument && n_tests) atomicAdd(&meta->pair_tests, n_tests);
}

}  // namespace fec

// ---- host: sub-cell tables, uploaded once per device -------------------------------------
#include <mutex>

namespace fec {

cudaError_t ensure_subcell_tables() {
    static std::mutex mu;
    static bool done[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    if (done[dev & 63]) return cudaSuccess;
    static SubcellTables t;
    sc_build_tables(t);
    // the bit-operation dilation used by the flood fill must equal the table's certain
    // relation inside a cell (slot 13); checked once on the host
    for (int a = 0; a < 64; ++a)
        if ((sc_dilate(1ull << a) | (1ull << a)) != (t.T[13][a] | (1ull << a))) return cudaErrorInvalidValue;
    // so must the whole-mask shift lists across the 26 neighbour slots
    for (int sl = 0; sl < 27; ++sl) {
        if (sl == 13) continue;
        if (t.nsh[sl] < 0) return cudaErrorInvalidValue;
        for (int a = 0; a < 64; ++a)
            if (sc_certain_across(t, 1ull << a, sl) != t.T[sl][a]) return cudaErrorInvalidValue;
    }
    e = cudaMemcpyToSymbol(d_sc, &t, sizeof(t));
    if (e == cudaSuccess) done[dev & 63] = true;
    return e;
}

}  // namespace fec

// ---- host-side diagnostics of the sub-cell relations (C ABI: fec_debug_subcell_*) -------------
extern "C" int32_t fec_debug_subcell_tables(unsigned long long* certain, unsigned long long* reach) {
    static fec::SubcellTables t;
    fec::sc_build_tables(t);
    for (int s = 0; s < 27; ++s)
        for (int a = 0; a < 64; ++a) {
            certain[64 * s + a] = t.T[s][a];
            reach[64 * s + a] = t.U[s][a];
        }
    return 0;
}

extern "C" unsigned long long fec_debug_subcell_dilate(unsigned long long m) { return fec::sc_dilate(m) | m; }

extern "C" int32_t fec_debug_subcell_components(unsigned long long occ, unsigned long long* comps) {
    fec::u64s c[fec::kMaxComp], rest;
    const int k = fec::sc_components(occ, c, rest);
    for (int i = 0; i < k; ++i) comps[i] = c[i];
    return rest ? -1 : k;
}
