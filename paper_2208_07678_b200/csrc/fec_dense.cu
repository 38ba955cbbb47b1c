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
#include "fec_subcell.cuh"

namespace fec {

__device__ SubcellTables d_sc = sc_make_tables();  // compile-time constant (fec_subcell.cuh)

// The 13 forward neighbour offsets: (dz>0) or (dz==0 and dy>0) or (dz==0, dy==0, dx>0).
// With same-cell pairs, every unordered pair of adjacent cells is visited exactly once.
__constant__ signed char c_fwd[13][3] = {
    {1, 0, 0},  {-1, 1, 0}, {0, 1, 0},  {1, 1, 0},  {-1, -1, 1}, {0, -1, 1}, {1, -1, 1},
    {-1, 0, 1}, {0, 0, 1},  {1, 0, 1},  {-1, 1, 1}, {0, 1, 1},   {1, 1, 1}};

// Neighbour slots of the dense-cell kernels: 0-2 forward faces, 3-12 forward edges and corners,
// 13-25 backward; slot 26 (not in the table) = a record's own component pairs.
__constant__ signed char c_slot[26][3] = {
    {1, 0, 0},   {0, 1, 0},   {0, 0, 1},                                         // forward faces
    {-1, 1, 0},  {1, 1, 0},   {0, -1, 1}, {-1, 0, 1}, {1, 0, 1}, {0, 1, 1},      // forward edges
    {-1, -1, 1}, {1, -1, 1},  {-1, 1, 1}, {1, 1, 1},                             // forward corners
    {-1, 0, 0},  {0, -1, 0},  {0, 0, -1},                                        // backward ...
    {1, -1, 0},  {-1, -1, 0}, {0, 1, -1}, {1, 0, -1}, {-1, 0, -1}, {0, -1, -1},
    {1, 1, -1},  {-1, 1, -1}, {1, -1, -1}, {-1, -1, -1}};


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
__device__ __forceinline__ void fine_of(float x, float y, float z, int64_t i, const Grid& g, uint32_t f[3]) {
    double l0 = g.lo[0], l1 = g.lo[1], l2 = g.lo[2];
    uint32_t zoff = 0;
    if (g.batch) {
        const int c = cloud_of(g, i);
        l0 = __ldg(g.blo + 3 * c);
        l1 = __ldg(g.blo + 3 * c + 1);
        l2 = __ldg(g.blo + 3 * c + 2);
        zoff = 4u * (uint32_t)__ldg(g.bz + c);
    }
    f[0] = sub_coord(x, l0, g.inv_q);
    f[1] = sub_coord(y, l1, g.inv_q);
    f[2] = sub_coord(z, l2, g.inv_q) + zoff;
}
__device__ __forceinline__ int fine_index(const uint32_t f[3]) {
    return (int)((f[0] & 3u) | ((f[1] & 3u) << 2) | ((f[2] & 3u) << 4));
}
// Fine sub-cell index (bit of the cell's 4x4x4 mask) of a point.
__device__ __forceinline__ int q_of(float x, float y, float z, int64_t i, const Grid& g) {
    uint32_t f[3];
    fine_of(x, y, z, i, g, f);
    return fine_index(f);
}

// ---- cell handles ---------------------------------------------------------------------------
// Bitmap mode (the grid holds <= 32n + 2^26 cells): handle = linear cell id, an index into an
// occupancy bitmap over the whole grid.  Hash mode (sparse, huge bounding boxes): handle = the
// slot of the cell's packed coordinates in an open-addressing table (linear probing, >= 2n
// slots), filled by k_cmark; the occupancy bitmap then runs over the table's slots.  Either
// way the compact id of an occupied cell is the rank of its handle's bit (cid_of), so every
// kernel after binning is the same for both.
__device__ __forceinline__ uint32_t hash_find(const Grid& g, u64 pc) {  // ~0u: absent
    uint32_t h = (uint32_t)hash_cell(pc) & g.hmask;
    while (true) {
        const u64 k = __ldg(g.hkey + h);  // read-only after k_cmark
        if (k == pc) return h;
        if (k == ~0ull) return 0xffffffffu;
        h = (h + 1) & g.hmask;
    }
}
// k_cmark (hash mode): slot of pc, inserting it if absent.
__device__ __forceinline__ uint32_t hash_insert(const Grid& g, u64 pc) {
    uint32_t h = (uint32_t)hash_cell(pc) & g.hmask;
    while (true) {
        u64 k = *reinterpret_cast<volatile u64*>(g.hkey + h);
        if (k == ~0ull) k = atomicCAS(g.hkey + h, ~0ull, pc);
        if (k == ~0ull || k == pc) return h;
        h = (h + 1) & g.hmask;
    }
}
__device__ __forceinline__ uint32_t cell_handle(const Grid& g, uint32_t cx, uint32_t cy, uint32_t cz) {
    if (g.hashed) return hash_find(g, pack_cell(cx, cy, cz));
    return cx * g.stride[0] + cy * g.stride[1] + cz * g.stride[2];
}
__device__ __forceinline__ void dense_cell_of(float x, float y, float z, int64_t i, const Grid& g, uint32_t& lin,
                                              int& q) {
    uint32_t f[3];
    fine_of(x, y, z, i, g, f);
    q = fine_index(f);
    lin = cell_handle(g, f[0] >> 2, f[1] >> 2, f[2] >> 2);
}

__device__ __forceinline__ void dense_decode(uint32_t lin, const Grid& g, int c[3]) {
    if (g.hashed) {
        const u64 pc = __ldg(g.hkey + lin);
        c[0] = (int)(pc & 0x1fffff);
        c[1] = (int)((pc >> 21) & 0x1fffff);
        c[2] = (int)(pc >> 42);
        return;
    }
    // slow axis = perm[2] (stride sdiv[0]), middle = perm[1] (stride sdiv[1]), fast = perm[0]
    const uint32_t q2 = lin / g.sdiv[0];
    lin -= q2 * g.sdiv[0];
    const uint32_t q1 = lin / g.sdiv[1];
    const uint32_t q0 = lin - q1 * g.sdiv[1];
    c[0] = (int)(g.perm[2] == 0 ? q2 : (g.perm[1] == 0 ? q1 : q0));
    c[1] = (int)(g.perm[2] == 1 ? q2 : (g.perm[1] == 1 ? q1 : q0));
    c[2] = (int)(g.perm[2] == 2 ? q2 : (g.perm[1] == 2 ? q1 : q0));
}

// Handle of the cell at c + (dx, dy, dz); false if it is outside the grid or (hash mode) empty.
__device__ __forceinline__ bool dense_neighbor(const Grid& g, const int c[3], int dx, int dy, int dz, uint32_t& lin) {
    const int x = c[0] + dx, y = c[1] + dy, z = c[2] + dz;
    if (x < 0 || y < 0 || z < 0 || x >= g.dims[0] || y >= g.dims[1] || z >= g.dims[2]) return false;
    lin = cell_handle(g, (uint32_t)x, (uint32_t)y, (uint32_t)z);
    return lin != 0xffffffffu;
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

// ---- scratch initialisation (device-sized) -------------------------------------------------
// The occupancy words (their count is planned on the device), the hash table (hash mode: all
// slots empty) and the host-sized arena of look-back states, counters and dense-cell bits.
__global__ void __launch_bounds__(256) k_zero(const Grid* __restrict__ gp, uint2* __restrict__ cw,
                                             u64* __restrict__ hkey, int64_t slots, uint32_t* __restrict__ arena,
                                             int64_t arena_words) {
    pdl_prologue();
    FEC_LOAD_GRID(gp);  // (right after k_bbox: the Grid is only safe after the wait)
    if (g.status) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nw2 = (g.words + 2) / 2;  // words + 1 uint2 entries, as uint4 pairs (256-B aligned)
    uint4* c4 = reinterpret_cast<uint4*>(cw);
    for (int64_t i = t0; i < nw2; i += stride) c4[i] = make_uint4(0u, 0u, 0u, 0u);
    if (g.hashed) {
        ulonglong2* h2 = reinterpret_cast<ulonglong2*>(hkey);
        for (int64_t i = t0; i < slots / 2; i += stride) h2[i] = make_ulonglong2(~0ull, ~0ull);
    }
    for (int64_t i = t0; i < arena_words; i += stride) arena[i] = 0u;
}

// ---- a2: occupancy bitmap ------------------------------------------------------------------
// Warp-synchronous aggregation (no shared-memory table): a thread's 4 consecutive points are
// merged into runs of one bitmap word; each thread's first run then meets the warp's other
// first runs in one __match_any_sync round, and one lane per distinct word ORs the combined
// bits into the bitmap (a reduction at L2, nothing waited on).  Later runs of a thread (a word
// boundary inside its 4 points) go straight to the bitmap.  Spatially coherent input (the
// counting path) makes the runs long and the distinct words per warp few.
__global__ void __launch_bounds__(256) k_cmark(const float* __restrict__ p, int64_t n, const Grid* __restrict__ gp,
                                              uint2* __restrict__ cw) {
    FEC_PROLOGUE_GRID(gp);
    if (g.status || g.key_sort) return;
    const bool vec = (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 128; t0 < n; t0 += nw * 128) {
        const int64_t b4 = t0 + 4 * lane;
        Pts4 P;
        load_pts4(p, n, b4, vec, P);
        uint32_t w0 = 0xffffffffu, bits0 = 0u;  // the thread's first run
        uint32_t w = 0xffffffffu, bits = 0u;     // the current (later) run
        u64 prev_pc = ~0ull;
        uint32_t lin = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (b4 + j >= n) continue;
            uint32_t f[3];
            fine_of(P.x[j], P.y[j], P.z[j], b4 + j, g, f);
            if (g.hashed) {  // insert the cell (consecutive points of one cell: one probe)
                const u64 pc = pack_cell(f[0] >> 2, f[1] >> 2, f[2] >> 2);
                if (pc != prev_pc) lin = hash_insert(g, pc);
                prev_pc = pc;
            } else {
                lin = (f[0] >> 2) * g.stride[0] + (f[1] >> 2) * g.stride[1] + (f[2] >> 2) * g.stride[2];
            }
            const uint32_t wd = lin >> 5, bit = 1u << (lin & 31u);
            if (w0 == 0xffffffffu || (wd == w0 && w == 0xffffffffu)) {
                w0 = wd;
                bits0 |= bit;
            } else if (wd == w) {
                bits |= bit;
            } else {
                if (w != 0xffffffffu) atomicOr(reinterpret_cast<unsigned int*>(cw + w), bits);
                w = wd;
                bits = bit;
            }
        }
        if (w != 0xffffffffu) atomicOr(reinterpret_cast<unsigned int*>(cw + w), bits);
        const unsigned peers = __match_any_sync(0xffffffffu, w0);
        const uint32_t all = __reduce_or_sync(peers, bits0);
        if (w0 != 0xffffffffu && lane == __ffs(peers) - 1) atomicOr(reinterpret_cast<unsigned int*>(cw + w0), all);
    }
}

// Word bases + cell list in three launches, no look-back chain: k_cpop sums the popcounts of
// each tile of 2048 occupancy words (every tile in parallel), k_tscan (one block) turns the
// tile sums into exclusive tile prefixes and the total U, and k_cscan stores each word's base
// next to its bits and emits the cells: each warp the cells of its 256 words, lane per cell
// (a binary search over the warp's word bases in shared memory), which keeps sparse (C4: 0.4%
// of the grid) and dense (C5: half) occupancy balanced and the stores coalesced.  (Measured
// alternatives: a look-back scan emitting word by word per warp, ~58 us on C4 -- the densest
// tiles serialised; a thread per cell with two global binary searches, 1.6 ms on C5; a
// thread per word, 3.9 ms on C5 -- uncoalesced stores, 6.9 GB of DRAM traffic for 2 GB.)
constexpr int CS_THREADS = 256, CS_ITEMS = 8, CS_TILE = CS_THREADS * CS_ITEMS;

__device__ __forceinline__ uint32_t block_sum_256(uint32_t v, uint32_t* red) {  // all threads get the sum
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    uint32_t t = 0;
#pragma unroll
    for (int k = 0; k < CS_THREADS / kWarp; ++k) t += red[k];
    return t;
}

__global__ void __launch_bounds__(CS_THREADS) k_cpop(const uint2* __restrict__ cw, uint32_t* __restrict__ tsum,
                                                    const Grid* __restrict__ gp) {
    FEC_PROLOGUE_GRID(gp);
    if (g.status) return;
    __shared__ uint32_t red[CS_THREADS / kWarp];
    const int64_t words = g.words;
    const int64_t tiles = (words + 1 + CS_TILE - 1) / CS_TILE;
    const uint4* c4 = reinterpret_cast<const uint4*>(cw);  // two words {bits, base} per uint4
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        uint32_t c = 0;
#pragma unroll
        for (int k = 0; k < CS_ITEMS / 2; ++k) {
            const int64_t i2 = t * (CS_TILE / 2) + k * CS_THREADS + threadIdx.x;  // word pair
            if (2 * i2 < words) {
                const uint4 v = __ldg(c4 + i2);
                c += __popc(v.x) + (2 * i2 + 1 < words ? __popc(v.z) : 0);
            }
        }
        c = block_sum_256(c, red);
        if (threadIdx.x == 0) tsum[t] = c;
    }
}

// One block: exclusive prefix of the tile sums in place, the total U -> meta.
__global__ void __launch_bounds__(1024) k_tscan(uint32_t* __restrict__ tsum, const Grid* __restrict__ gp,
                                               Meta* __restrict__ meta, uint32_t* __restrict__ count) {
    pdl_prologue();
    if (gp->status) return;
    __shared__ uint32_t wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t tiles = (gp->words + 1 + CS_TILE - 1) / CS_TILE;
    const int64_t per = (tiles + 1023) / 1024;  // contiguous chunk per thread
    const int64_t b = tid * per, e = min(tiles, b + per);
    uint32_t run = 0;
    for (int64_t t = b; t < e; ++t) run += tsum[t];
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t v = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        wsum[lane] = v;
    }
    __syncthreads();
    uint32_t pre = (x - run) + (w > 0 ? wsum[w - 1] : 0u);
    for (int64_t t = b; t < e; ++t) {
        const uint32_t v = tsum[t];
        tsum[t] = pre;
        pre += v;
    }
    if (tid == 1023) {
        const uint32_t U = wsum[31];
        meta->cells = (int)U;
        meta->cells1 = (int)U + 1;
        meta->dwords1 = (int)((U + 31) / 32) + 1;
        count[U] = 0u;
    }
}

// Shared-memory index with one pad word per 8: the thread-serial scan reads 8 consecutive
// entries per thread (stride 8 words: an 8-way bank conflict unpadded, none padded).
__device__ __forceinline__ int pad8(int j) { return j + (j >> 3); }

__global__ void __launch_bounds__(CS_THREADS) k_cscan(uint2* __restrict__ cw, const Grid* __restrict__ gp,
                                                     const uint32_t* __restrict__ tpre, uint32_t* __restrict__ clin,
                                                     uint32_t* __restrict__ count, u64* __restrict__ cocc,
                                                     int* __restrict__ cmin, u64* __restrict__ ccoord) {
    FEC_PROLOGUE_GRID(gp);
    if (g.status) return;
    __shared__ uint32_t s[CS_TILE + CS_TILE / 8 + 1];      // word bases (padded), + the tile's end
    __shared__ uint32_t sbits[CS_TILE + CS_TILE / 8 + 1];  // the words (padded)
    __shared__ uint32_t wsum[CS_THREADS / kWarp];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t words = g.words;
    const int64_t tiles = (words + 1 + CS_TILE - 1) / CS_TILE;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t base = tile * CS_TILE;
    __syncthreads();  // (the previous tile's emission read s / sbits)
#pragma unroll
    for (int k = 0; k < CS_ITEMS; ++k) {
        const int64_t i = base + k * CS_THREADS + tid;
        const uint32_t b = i < words ? cw[i].x : 0u;
        sbits[pad8(k * CS_THREADS + tid)] = b;
        s[pad8(k * CS_THREADS + tid)] = (uint32_t)__popc(b);
    }
    __syncthreads();
    uint32_t loc[CS_ITEMS];
    uint32_t run = 0;
#pragma unroll
    for (int k = 0; k < CS_ITEMS; ++k) {
        const uint32_t v = s[pad8(tid * CS_ITEMS + k)];
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
    }
    __syncthreads();
    const uint32_t t0 = __ldg(tpre + tile);
    const uint32_t pre = t0 + (x - run) + (w > 0 ? wsum[w - 1] : 0u);
#pragma unroll
    for (int k = 0; k < CS_ITEMS; ++k) s[pad8(tid * CS_ITEMS + k)] = pre + loc[k];
    if (tid == 0) s[pad8(CS_TILE)] = t0 + wsum[CS_THREADS / kWarp - 1];  // the tile's end
    __syncthreads();
    // word bases next to the bits
#pragma unroll
    for (int k = 0; k < CS_ITEMS; ++k) {
        const int64_t i = base + k * CS_THREADS + tid;
        if (i < words) cw[i].y = s[pad8(k * CS_THREADS + tid)];
    }
    // cells: warp w owns words [256w, 256w + 256); its cells [r0, r1) go 32 at a time, lane per
    // cell (coalesced stores), the word found by a binary search over the warp's word bases
    const int j0 = w * 256;
    const uint32_t r0 = s[pad8(j0)], r1 = s[pad8(j0 + 256)];
    for (uint32_t c = r0 + lane; c < r1; c += 32) {
        int lo = j0, hi = j0 + 256;  // the last word whose base is <= c
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s[pad8(mid)] <= c) lo = mid;
            else hi = mid;
        }
        const uint32_t bw = sbits[pad8(lo)];
        const uint32_t lin = (uint32_t)((base + lo) * 32) + (uint32_t)__fns(bw, 0u, (int)(c - s[pad8(lo)]) + 1);
        int cc[3];
        dense_decode(lin, g, cc);
        clin[c] = lin;
        ccoord[c] = (u64)cc[0] | ((u64)cc[1] << 21) | ((u64)cc[2] << 42);
        count[c] = 0u;
        cocc[c] = 0ull;
        cmin[c] = 0x7fffffff;
    }
    }  // tiles
}

// ---- a2: per-cell counts, slot[i] = rank of point i inside its cell, fine occupancy ------
// Warp per tile of 128 consecutive points (4 per lane), aggregated through a per-warp
// shared-memory table: one global atomicAdd (+ atomicOr) per distinct cell per tile and only
// warp-level synchronisation (the input order is spatially coherent on this path).
//
// (Measured alternatives: group reductions with __reduce_*_sync over __match_any_sync peer
// masks serialise per distinct mask -- 3x slower on C4; a segmented shuffle scan instead of the
// table, 1.3x slower.)
//
// A lane's 4 points fall into at most 4 runs of one compact cell id (k_dscatter's rounds).
struct PointRuns {
    uint32_t cid[4];  // compact cell id of each point (~0u past the end)
    int ri[4];        // run index of each point (runs of equal cid among the lane's 4 points)
    int off[4];       // position of the point inside its run
    int q[4];         // fine sub-cell of the point
};
__device__ __forceinline__ void point_runs(const Pts4& P, int64_t b4, int64_t n, const Grid& g,
                                           const uint2* __restrict__ cw, PointRuns& R) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        R.cid[j] = 0xffffffffu;
        R.q[j] = 0;
        if (b4 + j < n) {
            uint32_t lin;
            dense_cell_of(P.x[j], P.y[j], P.z[j], b4 + j, g, lin, R.q[j]);
            R.cid[j] = cid_of(cw, lin);
        }
        const bool fresh = j == 0 || R.cid[j] != R.cid[j > 0 ? j - 1 : 0];
        R.ri[j] = j == 0 ? 0 : R.ri[j > 0 ? j - 1 : 0] + (fresh ? 1 : 0);
        R.off[j] = fresh ? 0 : R.off[j > 0 ? j - 1 : 0] + 1;
    }
}

// 4 consecutive u32 of a per-point array (one 16-byte store when aligned and complete).
__device__ __forceinline__ void store4(uint32_t* __restrict__ a, int64_t b4, int64_t n, const uint32_t v[4]) {
    if (b4 + 4 <= n && (reinterpret_cast<uintptr_t>(a + b4) & 15u) == 0) {
        *reinterpret_cast<uint4*>(a + b4) = make_uint4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (b4 + j < n) a[b4 + j] = v[j];
    }
}
__device__ __forceinline__ void load4(const uint32_t* __restrict__ a, int64_t b4, int64_t n, uint32_t v[4]) {
    if (b4 + 4 <= n && (reinterpret_cast<uintptr_t>(a + b4) & 15u) == 0) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(a + b4));
        v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = b4 + j < n ? __ldg(a + b4 + j) : 0u;
    }
}
// The same for a read-once stream (k_dscatter's code loop): no L1 allocation, so the stream
// does not evict the small per-cell bitmaps that every code is looked up in.
__device__ __forceinline__ uint4 ldg_stream16(const uint4* a) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a));
    return v;
}
__device__ __forceinline__ void load4_stream(const uint32_t* __restrict__ a, int64_t b4, int64_t n, uint32_t v[4]) {
    if (b4 + 4 <= n && (reinterpret_cast<uintptr_t>(a + b4) & 15u) == 0) {
        const uint4 u = ldg_stream16(reinterpret_cast<const uint4*>(a + b4));
        v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = b4 + j < n ? __ldg(a + b4 + j) : 0u;
    }
}
// PointRuns from the codes k_dcount2 wrote (no coordinates needed).
__device__ __forceinline__ void point_runs_code(const uint32_t code[4], int64_t b4, int64_t n, PointRuns& R) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        R.cid[j] = b4 + j < n ? code[j] >> 6 : 0xffffffffu;
        R.q[j] = (int)(code[j] & 63u);
        const bool fresh = j == 0 || R.cid[j] != R.cid[j > 0 ? j - 1 : 0];
        R.ri[j] = j == 0 ? 0 : R.ri[j > 0 ? j - 1 : 0] + (fresh ? 1 : 0);
        R.off[j] = fresh ? 0 : R.off[j > 0 ? j - 1 : 0] + 1;
    }
}

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
// by k_dscatter against per-cell cursors.
__global__ void __launch_bounds__(256) k_dcount2(const float* __restrict__ p, int64_t n, const Grid* __restrict__ gp,
                                                const uint2* __restrict__ cw, uint32_t* __restrict__ count,
                                                u64* __restrict__ cocc, int* __restrict__ cmin,
                                                uint32_t* __restrict__ pcode, const Meta* __restrict__ meta) {
    FEC_PROLOGUE_GRID(gp);
    if (g.status || g.key_sort) return;
    const bool wcode = meta->cells <= kCodeCells;
    __shared__ int keys_all[256 / kWarp][kWSlots];
    __shared__ uint32_t cnt_all[256 / kWarp][kWSlots], olo_all[256 / kWarp][kWSlots], ohi_all[256 / kWarp][kWSlots];
    __shared__ int mn_all[256 / kWarp][kWSlots];
    __shared__ int used_all[256 / kWarp][kWTile];
    __shared__ int nused_all[256 / kWarp];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int* keys = keys_all[wid];
    uint32_t *cnt = cnt_all[wid], *olo = olo_all[wid], *ohi = ohi_all[wid];
    int* mn = mn_all[wid];
    int* used = used_all[wid];
    int* nused = nused_all + wid;
    for (int k = lane; k < kWSlots; k += 32) { keys[k] = -1; cnt[k] = 0u; olo[k] = 0u; ohi[k] = 0u; mn[k] = 0x7fffffff; }
    if (lane == 0) *nused = 0;
    __syncwarp();
    const bool vec = (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kWTile; t0 < n; t0 += nw * kWTile) {
        const int64_t b4 = t0 + 4 * lane;
        Pts4 P;
        load_pts4(p, n, b4, vec, P);
        // runs of this thread's points in one cell take one table update
        // (a run's first point has its smallest input index)
        uint32_t code[4] = {0u, 0u, 0u, 0u};
        uint32_t rc = 0xffffffffu, rn = 0u;
        int rfirst = 0;
        u64 rb = 0ull;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (b4 + j < n) {
                uint32_t lin;
                int q;
                dense_cell_of(P.x[j], P.y[j], P.z[j], b4 + j, g, lin, q);
                const uint32_t cid = cid_of(cw, lin);
                code[j] = (cid << 6) | (uint32_t)q;
                if (cid != rc) {
                    if (rn) {
                        const int h = wbin_slot(keys, rc, used, nused);
                        atomicAdd(cnt + h, rn);
                        atomicMin(mn + h, rfirst);
                        if ((uint32_t)rb) atomicOr(olo + h, (uint32_t)rb);
                        if ((uint32_t)(rb >> 32)) atomicOr(ohi + h, (uint32_t)(rb >> 32));
                    }
                    rc = cid;
                    rn = 0u;
                    rb = 0ull;
                    rfirst = (int)(b4 + j);
                }
                ++rn;
                rb |= 1ull << q;
            }
        }
        if (rn) {
            const int h = wbin_slot(keys, rc, used, nused);
            atomicAdd(cnt + h, rn);
            atomicMin(mn + h, rfirst);
            if ((uint32_t)rb) atomicOr(olo + h, (uint32_t)rb);
            if ((uint32_t)(rb >> 32)) atomicOr(ohi + h, (uint32_t)(rb >> 32));
        }
        if (wcode) store4(pcode, b4, n, code);
        __syncwarp();
        const int nu = *nused;
        for (int e = lane; e < nu; e += 32) {
            const int k = used[e];
            const int cid = keys[k];
            atomicAdd(count + cid, cnt[k]);
            atomicOr(cocc + cid, ((u64)ohi[k] << 32) | (u64)olo[k]);
            atomicMin(cmin + cid, mn[k]);
            keys[k] = -1;
            cnt[k] = 0u;
            olo[k] = 0u;
            ohi[k] = 0u;
            mn[k] = 0x7fffffff;
        }
        __syncwarp();
        if (lane == 0) *nused = 0;
        __syncwarp();
    }
}

// Counting path, a3: scatter into cell order, no shared memory.  Round r of a tile takes every
// lane's r-th run and groups the lanes holding the same cell with one __match_any_sync
// (coherent input: usually one or two rounds).  Per round, a group's base inside the cell is
// one atomicAdd on the cell's cursor (initialised to the cell start) by the group's lowest
// lane, issued for every round before any result is used; a lane's offset inside the group
// is the run lengths of the group's lower lanes (three ballots: lengths are 1-4).  A cell's
// points of one warp tile land contiguously.  Only the float4 (x, y, z, idx) is written here:
// the scattered store is the expensive part, and k_dinit derives everything else from the
// sorted float4s with coalesced accesses.
__global__ void __launch_bounds__(256) k_dscatter(const float* __restrict__ p, int64_t n,
                                                 const Grid* __restrict__ gp, const uint2* __restrict__ cw,
                                                 uint32_t* __restrict__ cursor, float4* __restrict__ spts,
                                                 const uint32_t* __restrict__ pcode, const Meta* __restrict__ meta,
                                                 const uint32_t* __restrict__ cneed0,
                                                 const uint32_t* __restrict__ cneed1, int phase, int node_stats,
                                                 int item_cap) {
    FEC_PROLOGUE_GRID(gp);
    if (g.status || g.key_sort) return;
    const bool rcode = meta->cells <= kCodeCells;
    // partial scatter (node-tail clouds of the single-GPU path): phase 0 writes the points of
    // sparse and multi-component cells, phase 1 those of single-component dense records that
    // a surviving queued item references (k_dense_filter marks them) -- every remaining one
    // if the item queue overflowed (k_dense_overflow then tests pairs in place)
    const bool partial = node_stats && 4 * (int64_t)meta->cells <= n;
    if (phase == 1 && !partial) return;
    const bool all1 = phase == 1 && meta->nitems > item_cap;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const bool vec = (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (rcode && partial) {  // the usual case: a lean loop over the codes
        const int64_t nt = (n + 127) / 128;
        for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < nt; t += nw) {
            const int64_t b4 = t * 128 + 4 * lane;
            uint32_t code[4];
            if (phase == 1) load4_stream(pcode, b4, n, code);  // (measured: phase 0 is faster with L1 allocation)
            else load4(pcode, b4, n, code);
            uint32_t cid[4];
            bool any = false;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t c = code[j] >> 6;
                bool keep = false;
                if (b4 + j < n) {  // (small bitmaps: L1 hits)
                    if (phase == 0 || all1) {
                        const bool in0 = (__ldg(cneed0 + (c >> 5)) >> (c & 31)) & 1u;
                        keep = phase == 0 ? in0 : !in0;
                    } else {  // cneed1 marks single-component records only (k_dense_filter)
                        keep = (__ldg(cneed1 + (c >> 5)) >> (c & 31)) & 1u;
                    }
                }
                cid[j] = keep ? c : 0xffffffffu;
                any |= keep;
            }
            if (!__any_sync(0xffffffffu, any)) continue;
            PointRuns R;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                R.cid[j] = cid[j];
                const bool fresh = j == 0 || cid[j] != cid[j > 0 ? j - 1 : 0];
                R.ri[j] = j == 0 ? 0 : R.ri[j > 0 ? j - 1 : 0] + (fresh ? 1 : 0);
                R.off[j] = fresh ? 0 : R.off[j > 0 ? j - 1 : 0] + 1;
            }
            Pts4 P;
            if (any) load_pts4(p, n, b4, vec, P);
            const int rounds = __reduce_max_sync(0xffffffffu, R.ri[3] + 1);
            uint32_t base[4] = {0u, 0u, 0u, 0u}, pre[4] = {0u, 0u, 0u, 0u};
            int lead[4] = {0, 0, 0, 0};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                if (r >= rounds) continue;  // (warp-uniform)
                uint32_t key = 0xffffffffu, len = 0u;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (R.ri[j] == r && R.cid[j] != 0xffffffffu) {
                        key = R.cid[j];
                        ++len;
                    }
                const unsigned peers = __match_any_sync(0xffffffffu, key);
                const unsigned b0 = __ballot_sync(0xffffffffu, len & 1u), b1 = __ballot_sync(0xffffffffu, len & 2u),
                               b2 = __ballot_sync(0xffffffffu, len & 4u);
                pre[r] = __popc(peers & lt & b0) + 2 * __popc(peers & lt & b1) + 4 * __popc(peers & lt & b2);
                lead[r] = __ffs(peers) - 1;
                if (key != 0xffffffffu && lane == lead[r])
                    base[r] = atomicAdd(cursor + key, __popc(peers & b0) + 2 * __popc(peers & b1) + 4 * __popc(peers & b2));
            }
            uint32_t pos[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                if (r >= rounds) continue;
                const uint32_t b = __shfl_sync(0xffffffffu, base[r], lead[r]) + pre[r];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (R.ri[j] == r) pos[j] = b + (uint32_t)R.off[j];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (R.cid[j] != 0xffffffffu)
                    spts[pos[j]] = make_float4(P.x[j], P.y[j], P.z[j], __int_as_float((int)(b4 + j)));
        }
        return;
    }
    for (int64_t t0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 128; t0 < n; t0 += nw * 128) {
        const int64_t b4 = t0 + 4 * lane;
        Pts4 P;
        PointRuns R;
        if (rcode) {
            uint32_t code[4];
            load4(pcode, b4, n, code);
            point_runs_code(code, b4, n, R);
        } else {
            load_pts4(p, n, b4, vec, P);
            point_runs(P, b4, n, g, cw, R);
        }
        if (partial) {  // drop the points this phase does not write (their runs stay split)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (R.cid[j] == 0xffffffffu) continue;
                const uint32_t c = R.cid[j];
                const bool in0 = (__ldg(cneed0 + (c >> 5)) >> (c & 31)) & 1u;  // small bitmaps: L1 hits
                const bool keep = phase == 0 ? in0 : (!in0 && (all1 || ((__ldg(cneed1 + (c >> 5)) >> (c & 31)) & 1u)));
                if (!keep) R.cid[j] = 0xffffffffu;
            }
        }
        if (rcode && (R.cid[0] & R.cid[1] & R.cid[2] & R.cid[3]) != 0xffffffffu) load_pts4(p, n, b4, vec, P);
        if (partial && !__any_sync(0xffffffffu, (R.cid[0] & R.cid[1] & R.cid[2] & R.cid[3]) != 0xffffffffu)) continue;
        const int rounds = __reduce_max_sync(0xffffffffu, R.ri[3] + 1);
        uint32_t base[4] = {0u, 0u, 0u, 0u}, pre[4] = {0u, 0u, 0u, 0u};
        int lead[4] = {0, 0, 0, 0};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (r >= rounds) continue;  // (warp-uniform)
            uint32_t key = 0xffffffffu, len = 0u;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (R.ri[j] == r && R.cid[j] != 0xffffffffu) {
                    key = R.cid[j];
                    ++len;
                }
            const unsigned peers = __match_any_sync(0xffffffffu, key);
            const unsigned b0 = __ballot_sync(0xffffffffu, len & 1u), b1 = __ballot_sync(0xffffffffu, len & 2u),
                           b2 = __ballot_sync(0xffffffffu, len & 4u);
            pre[r] = __popc(peers & lt & b0) + 2 * __popc(peers & lt & b1) + 4 * __popc(peers & lt & b2);
            lead[r] = __ffs(peers) - 1;
            if (key != 0xffffffffu && lane == lead[r])
                base[r] = atomicAdd(cursor + key, __popc(peers & b0) + 2 * __popc(peers & b1) + 4 * __popc(peers & b2));
        }
        uint32_t pos[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (r >= rounds) continue;
            const uint32_t b = __shfl_sync(0xffffffffu, base[r], lead[r]) + pre[r];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (R.ri[j] == r) pos[j] = b + (uint32_t)R.off[j];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (R.cid[j] != 0xffffffffu)
                spts[pos[j]] = make_float4(P.x[j], P.y[j], P.z[j], __int_as_float((int)(b4 + j)));
    }
}


// Counting path, a4: sorted-order initialisation (coalesced, 4 positions per thread): the
// point's cell from its coordinates, the cell's record word (crec: -1 for a sparse cell) gives
// the parent -- itself for a point of a sparse cell (accumulators reset), else its certain-
// connected component's node -- and the input index goes to sidx.  (Node statistics come from
// k_dcomps / k_dparent: no atomics here.)
__global__ void __launch_bounds__(256) k_dinit(const float4* __restrict__ spts, int64_t n, const Grid* __restrict__ gp,
                                              const uint2* __restrict__ cw, const int* __restrict__ crec,
                                              const u64* __restrict__ cmask, int nbase, int* __restrict__ parent,
                                              int* __restrict__ size, int* __restrict__ minidx,
                                              int* __restrict__ sidx, const Meta* __restrict__ meta,
                                              int all_parents) {
    FEC_PROLOGUE_GRID(gp);
    if (g.status || g.key_sort) return;
    // node-tail clouds of the single-GPU path read no sorted-order array of the dense points
    // (node statistics, k_relabel_in): k_cellscan initialises the points of sparse cells instead
    if (!all_parents && 4 * (int64_t)meta->cells <= n) return;
    const int64_t groups = (n + 3) / 4;
    for (int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < groups; gi += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b4 = 4 * gi;
        float4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = b4 + j < n ? __ldg(spts + b4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        int par[4], si[4], rv[4], q[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            par[j] = (int)(b4 + j);
            si[j] = __float_as_int(v[j].w);
            rv[j] = -1;
            q[j] = 0;
            if (b4 + j >= n) continue;
            uint32_t lin;
            dense_cell_of(v[j].x, v[j].y, v[j].z, si[j], g, lin, q[j]);
            rv[j] = __ldg(crec + cid_of(cw, lin));  // -1 sparse, else record << 3 | (components - 1)
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (b4 + j >= n) continue;
            if (rv[j] < 0) {  // a point of a sparse cell: a possible root
                size[b4 + j] = 0;
                minidx[b4 + j] = 0x7fffffff;
            } else {
                const int r = rv[j] >> 3, kc = (rv[j] & 7) + 1;
                int c = 0;
                if (kc > 1)
                    while (c < kc - 1 && !((__ldg(cmask + 8 * r + c) >> q[j]) & 1ull)) ++c;
                par[j] = node_of(nbase, g.rmask, r, c);
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

// Cell starts, scatter cursors and the dense record numbering in one reduce-then-scan over the
// occupied cells of the pair (points in the cell, cell is dense) packed in 64 bits -- point
// count low, dense flag high (< 2^32 points, so the low half never carries): k_cellred sums
// each tile of 2048 cells (every tile in parallel), k_celltscan (one block) scans the tile
// sums, k_cellscan scans each tile again from its prefix and writes, per cell, the start and
// the cursor (counting path: the counts are replaced in place; key path: the starts exist
// already and only the dense rank is scanned), dlist / crec (record, or -1 for a sparse cell)
// and the partial-scatter phase-0 bits of the sparse cells.  Replaces a counts scan, a
// dense-flag pass, a popcount pass, a second scan and a list pass.  (A single-pass
// decoupled look-back version took 0.7 ms on C5's 73M cells: the look-back chain.)
constexpr int CL_THREADS = 256, CL_ITEMS = 8, CL_TILE = CL_THREADS * CL_ITEMS;
__device__ __forceinline__ unsigned long long cell_pair(const uint32_t* __restrict__ cstart, int64_t i, int64_t U,
                                                        bool ks) {
    if (i >= U) return 0ull;
    const uint32_t c = ks ? __ldg(cstart + i + 1) - __ldg(cstart + i) : cstart[i];
    return (ks ? 0ull : (unsigned long long)c) | ((unsigned long long)(c > (uint32_t)SPARSE_MAX) << 32);
}
__global__ void __launch_bounds__(CL_THREADS) k_cellred(const uint32_t* __restrict__ cstart,
                                                      const Meta* __restrict__ meta, const Grid* __restrict__ gp,
                                                      unsigned long long* __restrict__ tsum) {
    pdl_prologue();
    if (gp->status) return;
    __shared__ unsigned long long red[CL_THREADS / kWarp];
    const int64_t U = meta->cells;
    const bool ks = gp->key_sort;
    const int64_t tiles = (U + 1 + CL_TILE - 1) / CL_TILE;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        unsigned long long v = 0ull;
#pragma unroll
        for (int k = 0; k < CL_ITEMS; ++k) v += cell_pair(cstart, t * CL_TILE + k * CL_THREADS + threadIdx.x, U, ks);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        __syncthreads();
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long tot = 0ull;
#pragma unroll
            for (int k = 0; k < CL_THREADS / kWarp; ++k) tot += red[k];
            tsum[t] = tot;
        }
    }
}
// One block: exclusive prefix of the tile sums in place; the totals -> ndense, cstart[U].
__global__ void __launch_bounds__(1024) k_celltscan(unsigned long long* __restrict__ tsum, Meta* __restrict__ meta,
                                                  const Grid* __restrict__ gp, uint32_t* __restrict__ cstart) {
    pdl_prologue();
    if (gp->status) return;
    __shared__ unsigned long long wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t U = meta->cells;
    const int64_t tiles = (U + 1 + CL_TILE - 1) / CL_TILE;
    const int64_t per = (tiles + 1023) / 1024;
    const int64_t b = tid * per, e = min(tiles, b + per);
    unsigned long long run = 0ull;
    for (int64_t t = b; t < e; ++t) run += tsum[t];
    unsigned long long x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        unsigned long long v = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        wsum[lane] = v;
    }
    __syncthreads();
    unsigned long long pre = (x - run) + (w > 0 ? wsum[w - 1] : 0ull);
    for (int64_t t = b; t < e; ++t) {
        const unsigned long long v = tsum[t];
        tsum[t] = pre;
        pre += v;
    }
    if (tid == 1023) {
        const unsigned long long tot = wsum[31];
        meta->ndense = (int)(tot >> 32);
        if (!gp->key_sort) cstart[U] = (uint32_t)tot;  // = n
    }
}
__global__ void __launch_bounds__(CL_THREADS) k_cellscan(uint32_t* __restrict__ cstart, uint32_t* __restrict__ cursor,
                                                       int* __restrict__ dlist, int* __restrict__ crec,
                                                       uint32_t* __restrict__ cneed0, Meta* __restrict__ meta,
                                                       const Grid* __restrict__ gp,
                                                       const unsigned long long* __restrict__ tpre,
                                                       int* __restrict__ slist, int64_t n, int local_only,
                                                       int all_parents, int* __restrict__ parent,
                                                       int* __restrict__ size, int* __restrict__ minidx) {
    pdl_prologue();
    if (gp->status) return;
    __shared__ unsigned long long sv[CL_TILE + CL_TILE / 8];  // padded (pad8)
    __shared__ unsigned long long wsum[CL_THREADS / kWarp];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t U = meta->cells;
    const bool ks = gp->key_sort;
    const int64_t tiles = (U + 1 + CL_TILE - 1) / CL_TILE;
    // the compact list of the sparse cells (LOCAL clouds and small clouds: k_union_sparse_local
    // and the node tail walk it) and, on the counting path of node-tail clouds, the union-find
    // init of their points (k_dinit does not run there)
    const bool node_tail = 4 * U <= n;
    const bool list = local_only || node_tail;
    const bool init = list && !ks && !all_parents && node_tail;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t base = tile * CL_TILE;
    __syncthreads();  // (the previous tile's writes read sv)
#pragma unroll
    for (int k = 0; k < CL_ITEMS; ++k) sv[pad8(k * CL_THREADS + tid)] = cell_pair(cstart, base + k * CL_THREADS + tid, U, ks);
    __syncthreads();
    // thread-serial over 8 consecutive elements, then warp and block scans
    unsigned long long loc[CL_ITEMS];
    unsigned long long run = 0ull;
#pragma unroll
    for (int k = 0; k < CL_ITEMS; ++k) {
        loc[k] = run;
        run += sv[pad8(tid * CL_ITEMS + k)];
    }
    unsigned long long x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        unsigned long long v = lane < CL_THREADS / kWarp ? wsum[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        if (lane < CL_THREADS / kWarp) wsum[lane] = v;
    }
    __syncthreads();
    const unsigned long long pre = __ldg(tpre + tile) + (x - run) + (w > 0 ? wsum[w - 1] : 0ull);
    // exclusive prefix of each element, keeping its own dense flag in bit 63 (free: < 2^62)
#pragma unroll
    for (int k = 0; k < CL_ITEMS; ++k) {
        const unsigned long long own = sv[pad8(tid * CL_ITEMS + k)];
        sv[pad8(tid * CL_ITEMS + k)] = (pre + loc[k]) | ((own >> 32) << 63);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < CL_ITEMS; ++k) {
        const int64_t i = base + k * CL_THREADS + tid;  // a warp: 32 consecutive cells
        const unsigned long long e = sv[pad8(k * CL_THREADS + tid)];
        const bool dense = (e >> 63) != 0;
        if (i < U) {
            if (!ks) {
                cstart[i] = (uint32_t)e;
                cursor[i] = (uint32_t)e;
            }
            if (dense) {
                const int r = (int)((e >> 32) & 0x3fffffffull);
                dlist[r] = (int)i;
                crec[i] = r;  // (k_dcomps replaces it by the record word)
            } else {
                crec[i] = -1;
            }
        }
        const unsigned sp = __ballot_sync(0xffffffffu, i < U && !dense);
        if (lane == 0 && i < ((U + 31) & ~int64_t(31))) cneed0[i >> 5] = sp;  // (k_dcomps adds multi-component cells)
        if (list && sp) {
            int lbase = 0;
            if (lane == 0) lbase = atomicAdd(&meta->nsparse, __popc(sp));
            lbase = __shfl_sync(0xffffffffu, lbase, 0);
            const bool mine = (sp >> lane) & 1u;
            if (mine) slist[lbase + __popc(sp & ((1u << lane) - 1u))] = (int)i;
            if (init && mine) {  // the cell's points: [its start, the next cell's start)
                const bool last = k == CL_ITEMS - 1 && tid == CL_THREADS - 1;
                const uint32_t s0 = (uint32_t)e;
                const uint32_t s1 = last ? (uint32_t)(__ldg(tpre + tile) + wsum[CL_THREADS / kWarp - 1])
                                         : (uint32_t)sv[pad8(k * CL_THREADS + tid + 1)];
                for (uint32_t t = s0; t < s1; ++t) {
                    parent[t] = (int)t;
                    size[t] = 0;
                    minidx[t] = 0x7fffffff;
                }
            }
        }
    }
    }  // tiles
}

// ---- a2/a3, sort path (shuffled inputs) ----------------------------------------------------
// For inputs without spatial coherence (C1, C5) the counting sort's per-point atomics and
// scatter hit random DRAM sectors; instead the linear cell ids are radix-sorted (coalesced
// digit passes), cells are the runs of equal keys, and points are gathered into cell order.
// Also the onesweep sort's digit histograms of all passes (ghist[pass][digit], block-
// aggregated in shared memory) and the zeroed look-back state of its first pass.
__global__ void __launch_bounds__(256) k_lkey(const float* __restrict__ p, int64_t n, const Grid* __restrict__ gp,
                                             uint32_t* __restrict__ key, int* __restrict__ val,
                                             uint32_t* __restrict__ ghist, uint32_t* __restrict__ state0,
                                             int64_t state_words) {
    FEC_PROLOGUE_GRID(gp);
    if (g.status || !g.key_sort) return;
    __shared__ uint32_t h[4][256];
    for (int k = threadIdx.x; k < 4 * 256; k += blockDim.x) (&h[0][0])[k] = 0u;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < state_words; k += (int64_t)gridDim.x * blockDim.x)
        state0[k] = 0u;
    __syncthreads();
    const int passes = g.passes;
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
            if (b4 + j < n) {
                dense_cell_of(P.x[j], P.y[j], P.z[j], b4 + j, g, k[j], q);
                for (int ps = 0; ps < passes; ++ps) atomicAdd(&h[ps][(k[j] >> (8 * ps)) & 255u], 1u);
            }
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
    __syncthreads();
    for (int k = threadIdx.x; k < passes * 256; k += blockDim.x) {
        const uint32_t c = (&h[0][0])[k];
        if (c) atomicAdd(ghist + k, c);
    }
}

// Occupancy bits of the sorted keys' distinct values (heads only; a warp's heads share words).
__global__ void __launch_bounds__(256) k_smark(const uint32_t* __restrict__ key0, const uint32_t* __restrict__ key1,
                                              int64_t n, uint2* __restrict__ cw, const Grid* __restrict__ gp) {
    pdl_prologue();
    if (gp->status || !gp->key_sort) return;
    const uint32_t* __restrict__ key = (gp->passes & 1) ? key1 : key0;  // the sort's output buffer
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
__global__ void __launch_bounds__(256) k_sgather(const float* __restrict__ p, const uint32_t* __restrict__ key0,
                                                const int* __restrict__ val0, const uint32_t* __restrict__ key1,
                                                const int* __restrict__ val1, int64_t n,
                                                const Grid* __restrict__ gp, const uint2* __restrict__ cw,
                                                float4* __restrict__ spts, uint32_t* __restrict__ cstart,
                                                u64* __restrict__ cocc, int* __restrict__ parent,
                                                int* __restrict__ sidx, int* __restrict__ size,
                                                int* __restrict__ minidx, const Meta* __restrict__ meta) {
    FEC_PROLOGUE_GRID(gp);
    if (g.status || !g.key_sort) return;
    const uint32_t* __restrict__ key = (g.passes & 1) ? key1 : key0;  // the sort's output buffers
    const int* __restrict__ val = (g.passes & 1) ? val1 : val0;
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
                const int q = q_of(x[j], y[j], z[j], vi[j], g);
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


// ---- uncertain component pairs: queued, or tested in place when the queue is full ----------
// item = (P record, P component, Q record or point, Q component or -1 for a point)

__device__ __forceinline__ int cell_slot_of(const Grid& g, uint32_t lin_p, uint32_t lin_q) {
    int a[3], b[3];
    dense_decode(lin_p, g, a);
    dense_decode(lin_q, g, b);
    return sc_slot(b[0] - a[0], b[1] - a[1], b[2] - a[2]);
}
// Neighbour slot of the cell holding point v relative to cell lin_p, and v's fine index.
__device__ __forceinline__ int point_slot_of(const Grid& g, uint32_t lin_p, float4 v, int& qv) {
    int a[3];
    dense_decode(lin_p, g, a);
    uint32_t f[3];
    fine_of(v.x, v.y, v.z, __float_as_int(v.w), g, f);
    qv = fine_index(f);
    return sc_slot((int)(f[0] >> 2) - a[0], (int)(f[1] >> 2) - a[1], (int)(f[2] >> 2) - a[2]);
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
    const int na = node_of(C.nbase, C.rmask, it.x, it.y);
    int nb, b0, b1;
    u64 mb;
    int slot;
    if (it.w >= 0) {
        const int cq = __ldg(C.dlist + it.z);
        mb = C.cmask[8 * it.z + it.w];
        nb = node_of(C.nbase, C.rmask, it.z, it.w);
        b0 = (int)__ldg(C.cstart + cq);
        b1 = (int)__ldg(C.cstart + cq + 1);
        slot = cell_slot_of(g, lp, __ldg(C.clin + cq));
    } else {
        mb = ~0ull;
        nb = it.z;
        b0 = it.z;
        b1 = it.z + 1;
        int qq;
        slot = point_slot_of(g, lp, C.spts[it.z], qq);
    }
    const int a0 = (int)__ldg(C.cstart + cp), a1 = (int)__ldg(C.cstart + cp + 1);
    for (int i = a0; i < a1; ++i) {
        const float4 pa = C.spts[i];
        const int qa = q_of(pa.x, pa.y, pa.z, __float_as_int(pa.w), g);
        if (!((ma >> qa) & 1ull)) continue;
        const u64 reach = d_sc.U[slot][qa];
        for (int j = b0; j < b1; ++j) {
            const float4 pb = C.spts[j];
            const int qb = q_of(pb.x, pb.y, pb.z, __float_as_int(pb.w), g);
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

// ---- dense records: components of the fine occupancy, node init, and the link items --------
// Thread per dense record: its certain-connected components (at most 8 union-find nodes), then
// its 26 neighbour cells (13 bitmap lookups in flight at a time) give the record's items for
// k_dense_link: every forward dense neighbour ("DD" list) and every sparse neighbour in either
// direction, plus slot 26 = its own component pairs when it has several ("DS" list).  Absent
// and backward-dense neighbours produce nothing, so the link kernel's threads all have work.
// Items are warp-aggregated (one atomic per list per warp) into two halves of `litems`; if a
// half overflows, meta->list_overflow makes k_dense_link (main stream) redo every (record, slot).
__global__ void __launch_bounds__(256) k_dcomps(const Grid* __restrict__ gp, const uint2* __restrict__ cw,
                                               int* __restrict__ crec,
                                               const u64* __restrict__ cocc, const u64* __restrict__ ccoord,
                                               int* __restrict__ ncomp, int* __restrict__ size,
                                               int* __restrict__ minidx, u64* __restrict__ dcoord,
                                               uint32_t* __restrict__ oflags, DenseCtx C, uint4* __restrict__ litems,
                                               int lhalf, const int* __restrict__ cmin, const int* __restrict__ sidx,
                                               int node_stats) {
    FEC_PROLOGUE_GRID(gp);
    if (g.status) return;
    // node-level statistics of single-component records come from their cell: the count is
    // the cell's size and the minimum input index was taken while counting (counting path;
    // the key path's stable sort puts it first in the cell)
    const bool nstats = node_stats && 4 * (int64_t)C.meta->cells <= (int64_t)C.nbase;
    __shared__ signed char soff[26][3];
    if (threadIdx.x < 26 * 3) (&soff[0][0])[threadIdx.x] = (&c_slot[0][0])[threadIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int nd = C.meta->ndense;
    for (int r0 = blockIdx.x * blockDim.x; r0 < nd; r0 += gridDim.x * blockDim.x) {  // block-uniform
        const int r = r0 + threadIdx.x;
        const bool v = r < nd;
        int kp = 0, cid = 0;
        int c[3] = {0, 0, 0};
        if (v) {
            cid = __ldg(C.dlist + r);
            const u64 occ = __ldg(cocc + cid);
            const u64 pc = __ldg(ccoord + cid);
            dcoord[r] = pc;
            c[0] = (int)(pc & 0x1fffff);
            c[1] = (int)((pc >> 21) & 0x1fffff);
            c[2] = (int)(pc >> 42);
            oflags[r] = 0u;
            u64 comp[kMaxComp];
            u64 rest;
            kp = sc_components(occ, comp, rest);
            if (rest) atomicOr(&C.meta->internal_error, 1);  // impossible by the 8-component bound
            ncomp[r] = kp;
            crec[cid] = (r << 3) | (kp - 1);  // the cell's record word (k_dense_link, k_relabel_in)
            if (kp > 1 && C.cneed0) atomicOr(C.cneed0 + (cid >> 5), 1u << (cid & 31));  // (k_dparent reads its points)
#pragma unroll
            for (int j = 0; j < kMaxComp; ++j) {
                const int node = node_of(C.nbase, C.rmask, r, j);
                C.parent[node] = node;
                size[node] = 0;
                minidx[node] = 0x7fffffff;
                C.cmask[8 * r + j] = j < kp ? comp[j] : 0ull;
            }
            if (kp == 1 && nstats) {
                const int a0 = (int)__ldg(C.cstart + cid);
                const int node0 = node_of(C.nbase, C.rmask, r, 0);
                size[node0] = (int)__ldg(C.cstart + cid + 1) - a0;
                minidx[node0] = g.key_sort ? __ldg(sidx + a0) : __ldg(cmin + cid);
            }
        }
        // neighbour slots that need work
        uint32_t mdd = 0u, mds = 0u;
#pragma unroll 1
        for (int k0 = 0; k0 < 26; k0 += 13) {
            int cq[13];
#pragma unroll
            for (int j = 0; j < 13; ++j) {
                uint32_t lq;
                cq[j] = (v && dense_neighbor(g, c, soff[k0 + j][0], soff[k0 + j][1], soff[k0 + j][2], lq))
                            ? cid_lookup(cw, lq) : -1;
            }
#pragma unroll
            for (int j = 0; j < 13; ++j) {
                if (cq[j] < 0) continue;
                const uint32_t cnt = __ldg(C.cstart + cq[j] + 1) - __ldg(C.cstart + cq[j]);
                if (cnt <= (uint32_t)SPARSE_MAX) mds |= 1u << (k0 + j);
                else if (k0 + j < 13) mdd |= 1u << (k0 + j);
            }
        }
        if (v && kp > 1) mds |= 1u << 26;
        // block-aggregated reservation in the two lists
        const int cdd = __popc(mdd), cds = __popc(mds);
        int xdd = cdd, xds = cds;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int ydd = __shfl_up_sync(0xffffffffu, xdd, o), yds = __shfl_up_sync(0xffffffffu, xds, o);
            if (lane >= o) {
                xdd += ydd;
                xds += yds;
            }
        }
        // warp-aggregated reservation (no block barrier waits on the atomics' round trip)
        int bdd = 0, bds = 0;
        if (lane == 31) {
            bdd = xdd ? atomicAdd(&C.meta->ndd, xdd) : 0;
            bds = xds ? atomicAdd(&C.meta->nds, xds) : 0;
            if ((xdd && bdd + xdd > lhalf) || (xds && bds + xds > lhalf)) atomicOr(&C.meta->list_overflow, 1);
        }
        bdd = __shfl_sync(0xffffffffu, bdd, 31);
        bds = __shfl_sync(0xffffffffu, bds, 31);
        int pdd = bdd + xdd - cdd, pds = bds + xds - cds;
        if (pdd + cdd <= lhalf && pds + cds <= lhalf) {
            uint32_t m = mdd;
            while (m) {
                const int k = __ffs(m) - 1;
                m &= m - 1;
                uint32_t lq;
                dense_neighbor(g, c, soff[k][0], soff[k][1], soff[k][2], lq);
                litems[pdd++] = make_uint4((uint32_t)r, (uint32_t)k, (uint32_t)cid_of(cw, lq), 0u);
            }
            m = mds;
            while (m) {
                const int k = __ffs(m) - 1;
                m &= m - 1;
                uint32_t cq = 0u;
                if (k < 26) {
                    uint32_t lq;
                    dense_neighbor(g, c, soff[k][0], soff[k][1], soff[k][2], lq);
                    cq = cid_of(cw, lq);
                }
                litems[lhalf + pds++] = make_uint4((uint32_t)r, (uint32_t)k, cq, 0u);
            }
        }
    }
}

// Warp per dense record (the cell's points are contiguous in sorted order).  Key path: every
// point of the cell hangs under its component's node (coalesced parent writes; k_sgather made
// every point its own parent).  Both paths: records with several components get their nodes'
// counts and minimum input indices (reduced in registers and stored once: the warp owns the
// record's nodes); single-component records got theirs in k_dcomps, and on the counting path
// k_dscatter already wrote the parents.
__global__ void __launch_bounds__(256) k_dparent(const float4* __restrict__ spts, const uint32_t* __restrict__ cstart,
                                                const int* __restrict__ dlist, const int* __restrict__ ncomp,
                                                const u64* __restrict__ cmask, const Grid* __restrict__ gp,
                                                int nbase, int* __restrict__ parent, const Meta* __restrict__ meta,
                                                const int* __restrict__ sidx, int* __restrict__ size,
                                                int* __restrict__ minidx, int node_stats, int64_t n) {
    FEC_PROLOGUE_GRID(gp);
    if (g.status) return;
    const int lane = threadIdx.x & 31;
    const int nd = meta->ndense;
    const bool nstats = node_stats && 4 * (int64_t)meta->cells <= n;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    // 32 records per warp iteration: the lanes read their records' component counts and the warp
    // then walks only the records with work (counting path: those with several components)
    for (int rb = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; rb < nd; rb += warps * 32) {
    const int kl = rb + lane < nd ? __ldg(ncomp + rb + lane) : 0;
    unsigned todo = __ballot_sync(0xffffffffu, kl > 1 || (kl > 0 && g.key_sort));
    while (todo) {
        const int j = __ffs(todo) - 1;
        todo &= todo - 1;
        const int r = rb + j;
        const int k = __shfl_sync(0xffffffffu, kl, j);
        const int cid = __ldg(dlist + r);
        const int a0 = (int)__ldg(cstart + cid), a1 = (int)__ldg(cstart + cid + 1);
        const int node0 = node_of(nbase, g.rmask, r, 0);
        if (k == 1) {  // key path, one component: every point under node 0 (stats: k_dcomps)
            for (int s = a0 + lane; s < a1; s += 32) parent[s] = node0;
            continue;
        }
        // several components: each point's component from its fine sub-cell; the warp owns the
        // record's nodes, so their totals are reduced in registers and stored once (no atomics)
        int accn[kMaxComp], accm[kMaxComp];
#pragma unroll
        for (int c = 0; c < kMaxComp; ++c) {
            accn[c] = 0;
            accm[c] = 0x7fffffff;
        }
        for (int s0 = a0; s0 < a1; s0 += 32) {  // warp-uniform trip count
            const int s = s0 + lane;
            int cc = -1, v = 0x7fffffff;
            if (s < a1) {
                const float4 pt = __ldg(spts + s);
                const int q = q_of(pt.x, pt.y, pt.z, __float_as_int(pt.w), g);
                cc = 0;
                while (cc < k - 1 && !((__ldg(cmask + 8 * r + cc) >> q) & 1ull)) ++cc;
                if (g.key_sort) parent[s] = node0 + cc;  // (counting path: k_dscatter wrote it)
                v = __float_as_int(pt.w);
            }
            if (nstats) {
#pragma unroll
                for (int c = 0; c < kMaxComp; ++c) {
                    if (c >= k) break;
                    const bool m = cc == c;
                    accn[c] += __popc(__ballot_sync(0xffffffffu, m));
                    accm[c] = min(accm[c], __reduce_min_sync(0xffffffffu, m ? v : 0x7fffffff));
                }
            }
        }
        if (nstats && lane == 0) {
#pragma unroll
            for (int c = 0; c < kMaxComp; ++c) {
                if (c >= k) break;
                size[node0 + c] = accn[c];
                minidx[node0 + c] = accm[c];
            }
        }
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

// The work of one (dense record r, neighbour slot k) item whose neighbour cell cq (compact id,
// occupied) is already known; k == 26 is the record's own component pairs (cq unused).
template <bool serial>
__device__ __forceinline__ void dense_link_pair(int r, int k, int ox, int oy, int oz, int cq, const Grid& g,
                                                const int* __restrict__ crec, const int* __restrict__ ncomp,
                                                uint32_t* __restrict__ oflags, const DenseCtx& C) {
    const int kp = __ldg(ncomp + r);
    const u64* mp = C.cmask + 8 * r;
    bool overflow = false;
    if (k == 26) {
        // P's own components (never certain-adjacent to each other)
        for (int i = 0; i + 1 < kp; ++i)
            for (int j = i + 1; j < kp; ++j) {
                const int na = node_of(C.nbase, C.rmask, r, i), nb = node_of(C.nbase, C.rmask, r, j);
                if (uf_find(C.parent, na) == uf_find(C.parent, nb)) continue;
                if constexpr (serial) test_item_serial(C, g, make_int4(r, i, r, j));
                else overflow |= !queue_item(C, make_int4(r, i, r, j));
            }
    } else {
        const int q0 = (int)__ldg(C.cstart + cq), q1 = (int)__ldg(C.cstart + cq + 1);
        const int slot = sc_slot(ox, oy, oz);
        if (q1 - q0 > SPARSE_MAX) {
            if (k >= 13) return;  // backward dense pairs belong to the other cell
            const int cw_q = __ldg(crec + cq);  // record << 3 | (components - 1)
            const int rq = cw_q >> 3, kq = (cw_q & 7) + 1;
            for (int x = 0; x < kp; ++x) {
                const u64 mx = mp[x];
                const u64 dc = sc_certain_across(d_sc, mx, slot);
                const bool near_p = (mx & d_sc.F[slot]) != 0;
                const int na = node_of(C.nbase, C.rmask, r, x);
                for (int y = 0; y < kq; ++y) {
                    const u64 my = C.cmask[8 * rq + y];
                    const int nb = node_of(C.nbase, C.rmask, rq, y);
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
                const int qb = q_of(v.x, v.y, v.z, __float_as_int(v.w), g);
                const u64 tc = d_sc.T[opp][qb], tu = d_sc.U[opp][qb];
                for (int x = 0; x < kp; ++x) {
                    const u64 mx = mp[x];
                    const int na = node_of(C.nbase, C.rmask, r, x);
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

// Overflow path: the same item with the neighbour looked up here.
__device__ __forceinline__ void dense_link_serial(int r, int k, const Grid& g, const uint2* __restrict__ cw,
                                                  const int* __restrict__ crec, const int* __restrict__ ncomp,
                                                  const u64* __restrict__ dcoord, uint32_t* __restrict__ oflags,
                                                  const DenseCtx& C) {
    int ox = 0, oy = 0, oz = 0, cq = 0;
    if (k != 26) {
        const u64 pc = __ldg(dcoord + r);
        const int c[3] = {(int)(pc & 0x1fffff), (int)((pc >> 21) & 0x1fffff), (int)(pc >> 42)};
        ox = c_slot[k][0];
        oy = c_slot[k][1];
        oz = c_slot[k][2];
        uint32_t lq;
        cq = dense_neighbor(g, c, ox, oy, oz, lq) ? cid_lookup(cw, lq) : -1;
        if (cq < 0) return;
    }
    dense_link_pair<true>(r, k, ox, oy, oz, cq, g, crec, ncomp, oflags, C);
}

// Fallback when the item lists overflowed (never on the configs measured): every (record,
// slot) is processed by its own thread, looking its neighbour up itself.  Unions are
// idempotent and queued duplicates are filtered, so items already handled do no harm.
__device__ __forceinline__ void dense_link_all_body(const Grid& g, const uint2* __restrict__ cw,
                                                    const int* __restrict__ crec, const int* __restrict__ ncomp,
                                                    const u64* __restrict__ dcoord, uint32_t* __restrict__ oflags,
                                                    const DenseCtx& C) {
    const int64_t total = 27 * (int64_t)C.meta->ndense;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(t / 27), k = (int)(t % 27);
        int ox = 0, oy = 0, oz = 0, cq = 0;
        if (k != 26) {
            const u64 pc = __ldg(dcoord + r);
            const int c[3] = {(int)(pc & 0x1fffff), (int)((pc >> 21) & 0x1fffff), (int)(pc >> 42)};
            ox = c_slot[k][0];
            oy = c_slot[k][1];
            oz = c_slot[k][2];
            uint32_t lq;
            cq = dense_neighbor(g, c, ox, oy, oz, lq) ? cid_lookup(cw, lq) : -1;
            if (cq < 0) continue;
        }
        dense_link_pair<false>(r, k, ox, oy, oz, cq, g, crec, ncomp, oflags, C);
    }
}

// a6+a7 for dense cells: one thread per listed item (k_dcomps), the forward dense pairs first,
// then the sparse neighbours and own pairs.  Certain component pairs are united at once;
// non-certain pairs within reach whose nodes are still apart are queued (k_dense_filter
// re-checks them after every certain union).
// `which`: 1 = the forward dense pairs only (they touch no point: this launch may run on a side
// stream concurrently with the scatter of the points), 2 = the sparse neighbours and own pairs
// only, 3 = both lists.  If an item list overflowed, the launch with the sparse neighbours
// (which & 2) runs the fallback over every (record, slot) instead (concurrent unions with a
// side-stream launch are harmless: they commute) and the other returns at once.
__global__ void __launch_bounds__(256, 4) k_dense_link(const Grid* __restrict__ gp, const int* __restrict__ crec,
                                                   const int* __restrict__ ncomp, uint32_t* __restrict__ oflags,
                                                   DenseCtx C, const uint4* __restrict__ litems, int lhalf, int which,
                                                   const uint2* __restrict__ cw, const u64* __restrict__ dcoord) {
    FEC_PROLOGUE_GRID(gp);
    if (g.status) return;
    if (C.meta->list_overflow) {
        if (which & 2) dense_link_all_body(g, cw, crec, ncomp, dcoord, oflags, C);
        return;
    }
    __shared__ signed char soff[26][3];
    if (threadIdx.x < 26 * 3) (&soff[0][0])[threadIdx.x] = (&c_slot[0][0])[threadIdx.x];
    __syncthreads();
    const int ndd = (which & 1) ? min(C.meta->ndd, lhalf) : 0, nds = (which & 2) ? min(C.meta->nds, lhalf) : 0;
    const int tot = ndd + nds;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += gridDim.x * blockDim.x) {
        const uint4 it = __ldg(litems + (i < ndd ? i : lhalf + (i - ndd)));
        const int k = (int)it.y;
        const int ox = k < 26 ? soff[k][0] : 0, oy = k < 26 ? soff[k][1] : 0, oz = k < 26 ? soff[k][2] : 0;
        dense_link_pair<false>((int)it.x, k, ox, oy, oz, (int)it.z, g, crec, ncomp, oflags, C);
    }
}

// Queue overflow: the marked slots' pairs are tested in place (one thread per record).
// (A separate launch: folded into k_dense_items it raised that kernel's registers 64 -> 80.)
__global__ void __launch_bounds__(256) k_dense_overflow(const Grid* __restrict__ gp, const uint2* __restrict__ cw,
                                                       const int* __restrict__ crec, const int* __restrict__ ncomp,
                                                       const u64* __restrict__ dcoord, uint32_t* __restrict__ oflags,
                                                       DenseCtx C) {
    FEC_PROLOGUE_GRID(gp);
    if (g.status) return;
    const int nd = C.meta->ndense;
    if (C.meta->nitems <= C.item_cap) return;  // nothing overflowed
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nd; r += gridDim.x * blockDim.x) {
        uint32_t f = oflags[r];
        while (f) {
            const int k = __ffs(f) - 1;
            f &= f - 1;
            dense_link_serial(r, k, g, cw, crec, ncomp, dcoord, oflags, C);
        }
    }
}

// Queued pairs whose nodes are already connected (after all certain unions) are dropped;
// the others are compacted into items2 for k_dense_items.
// Heavy pairs (two big cells) are split over several warps along B's range: sub-item
// (k, K) tests B's k-th of K slices, and a per-pair flag stops the others at the first hit.
constexpr int kSliceWork = 4096;   // cell-size product per slice
constexpr int kMaxSlices = 128;

// Also (first) component nodes -> their roots, which shortens the finds here and in
// k_dense_items (one launch: concurrent finds and flattening only ever move parents up).
__global__ void __launch_bounds__(256) k_dense_filter(DenseCtx C, int4* __restrict__ items2,
                                                     int4* __restrict__ slices2, int* __restrict__ idone) {
    pdl_prologue();
    if (C.meta->status) return;
    const int64_t nn = 8 * (int64_t)C.meta->ndense;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nn; t += (int64_t)gridDim.x * blockDim.x) {
        const int s = node_of(C.nbase, C.rmask, (int)(t >> 3), (int)(t & 7));
        int curr = ld_parent(C.parent, s), next;
        if (curr == s) continue;
        while (uf_above(next = ld_parent(C.parent, curr), curr)) curr = next;
        st_parent(C.parent, s, curr);
    }
    const int ni = min(C.meta->nitems, C.item_cap);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ni; e += gridDim.x * blockDim.x) {
        const int4 it = C.items[e];  // queued before every certain union was done: re-check
        const int na = node_of(C.nbase, C.rmask, it.x, it.y);
        const int nb = it.w >= 0 ? node_of(C.nbase, C.rmask, it.z, it.w) : it.z;
        if (uf_find(C.parent, na) == uf_find(C.parent, nb)) continue;
        // the records whose points k_dense_items reads (partial scatter, phase 1; an item
        // naming a sparse point references a sorted position written in phase 0)
        // (only single-component records: the cells of the others are in cneed0, written in
        // phase 0, so phase 1 tests one bitmap)
        const int cp = __ldg(C.dlist + it.x);
        if (C.cmask[8 * it.x + 1] == 0ull) atomicOr(C.cneed1 + (cp >> 5), 1u << (cp & 31));
        if (it.w >= 0) {
            const int cq = __ldg(C.dlist + it.z);
            if (C.cmask[8 * it.z + 1] == 0ull) atomicOr(C.cneed1 + (cq >> 5), 1u << (cq & 31));
        }
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

// ---- a6+a7: queued uncertain pairs, warp per item, early exit ------------------------------
// A's points in sub-cells within reach of B are staged per lane (up to kAPer each, in
// batches); B's points stream through the warp 32 at a time and are broadcast by shuffle.
constexpr int kAPer = 4;

__global__ void __launch_bounds__(256) k_dense_items(const Grid* __restrict__ gp, DenseCtx C,
                                                    const int4* __restrict__ items2,
                                                    const int4* __restrict__ slices2, int* __restrict__ idone) {
    FEC_PROLOGUE_GRID(gp);
    if (g.status) return;
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
        const int na = node_of(C.nbase, C.rmask, it.x, it.y);
        const int nb = it.w >= 0 ? node_of(C.nbase, C.rmask, it.z, it.w) : it.z;
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
            int qb;
            slot = point_slot_of(g, lp, C.spts[it.z], qb);
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
                    const int qa = q_of(p.x, p.y, p.z, __float_as_int(p.w), g);
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
                    const int qb = q_of(pb.x, pb.y, pb.z, __float_as_int(pb.w), g);
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
// the stats kernels) and the number of dense points.
__global__ void __launch_bounds__(256) k_dense_count(const int* __restrict__ ncomp, const int* __restrict__ dlist,
                                                    const uint32_t* __restrict__ cstart, DenseCtx C) {
    pdl_prologue();
    if (C.meta->status) return;
    const int nd = C.meta->ndense;
    unsigned long long roots = 0, pts = 0;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nd; r += gridDim.x * blockDim.x) {
        const int k = ncomp[r];
        for (int j = 0; j < k; ++j) roots += C.parent[node_of(C.nbase, C.rmask, r, j)] == node_of(C.nbase, C.rmask, r, j);
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

// The pair tests of a warp, dealt out evenly: lane l brings m_l pairs -- the rectangle
// [ps, ps+np) x [qs, qs+nq) of its cell and a neighbour, or (nq < 0) the triangle of its own
// cell's pairs -- the warp numbers all of them by a scan and takes them 32 at a time (a lane
// finds its pair's owner by a binary search over the scan), so it runs ceil(sum m / 32)
// rounds instead of max np x max nq lock-step iterations (C5: ~1 pair per lane and neighbour,
// 10% SIMT efficiency in the nested form).  Returns this lane's tests.
__device__ __forceinline__ int warp_pairs(const float4* __restrict__ spts, int* __restrict__ parent, float t2,
                                          int lane, int ps, int np, int qs, int nq) {
    const int m = nq >= 0 ? np * nq : np * (np - 1) / 2;
    int incl = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int tests = 0;
    for (int b0 = 0; b0 < total; b0 += 32) {
        const int idx = b0 + lane;
        int lo = 0;  // owner = number of lanes whose inclusive count is <= idx
#pragma unroll
        for (int step = 16; step > 0; step >>= 1)
            if (__shfl_sync(0xffffffffu, incl, lo + step - 1) <= idx) lo += step;
        const int ex = __shfl_sync(0xffffffffu, incl - m, lo);
        const int ops = __shfl_sync(0xffffffffu, ps, lo);
        const int oqs = __shfl_sync(0xffffffffu, qs, lo);
        const int onq = __shfl_sync(0xffffffffu, nq, lo);
        const int onp = __shfl_sync(0xffffffffu, np, lo);
        if (idx < total) {
            int k = idx - ex, s, t;
            if (onq > 0) {  // k < 36: k / onq = (k * ceil(256 / onq)) >> 8 (exact for k < 37)
                const int mg = (int)((0x5634201590100ull >> (9 * (onq - 1))) & 511u);
                const int q = (k * mg) >> 8;
                s = ops + q;
                t = oqs + (k - q * onq);
            } else {
                int i = 0;
                while (k >= onp - 1 - i) {
                    k -= onp - 1 - i;
                    ++i;
                }
                s = ops + i;
                t = s + 1 + k;
            }
            ++tests;
            if (pred(__ldg(spts + s), __ldg(spts + t), t2)) uf_unite(parent, s, t);
        }
    }
    return tests;
}

// Sparse-dominated clouds (occupied cells > n/4, ~1-2 points per cell): lane per sparse
// cell, its own pairs and every sparse forward neighbour's points (dense neighbours are
// handled by k_dense_link).  Clouds with few sparse cells use k_union_sparse_local instead;
// both are launched and the one not chosen returns at once.
__device__ __forceinline__ void union_sparse_body(const float4* __restrict__ spts, const uint2* __restrict__ cw,
                                                  const u64* __restrict__ ccoord, const uint32_t* __restrict__ cstart,
                                                  const Grid& g, int* __restrict__ parent, Meta* __restrict__ meta,
                                                  int64_t n, int local_only) {
    if (g.status || local_only || 4 * (int64_t)meta->cells <= n) return;
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
            const int np = v ? (int)__ldg(cstart + P + 1) - ps : 0;
            n_tests += warp_pairs(spts, parent, t2, lane, ps, np, 0, -1);  // own pairs
            const u64 pc = v ? __ldg(ccoord + P) : 0ull;
            const int c[3] = {(int)(pc & 0x1fffff), (int)((pc >> 21) & 0x1fffff), (int)(pc >> 42)};
#pragma unroll 1
            for (int k = 0; k < 13; ++k) {
                uint32_t Q;
                int qs = 0, nq = 0, qc = -1;
                if (v && dense_neighbor(g, c, c_fwd[k][0], c_fwd[k][1], c_fwd[k][2], Q)) qc = cid_lookup(cw, Q);
                if (qc >= 0) {
                    qs = (int)__ldg(cstart + qc);
                    nq = (int)__ldg(cstart + qc + 1) - qs;
                    if (nq > SPARSE_MAX) nq = 0;  // dense neighbours are handled by k_dense_link
                }
                n_tests += warp_pairs(spts, parent, t2, lane, ps, np, qs, nq);
            }
        }
        __syncwarp();
    }
    if (meta->instrument) {
        for (int o = 16; o > 0; o >>= 1) n_tests += __shfl_xor_sync(0xffffffffu, n_tests, o);
        if (lane == 0 && n_tests) atomicAdd(&meta->pair_tests, n_tests);
    }
}

__global__ void __launch_bounds__(256, 8) k_union_sparse(const float4* __restrict__ spts, const uint2* __restrict__ cw,
                                                     const u64* __restrict__ ccoord,
                                                     const uint32_t* __restrict__ cstart, const Grid* __restrict__ gp,
                                                     int* __restrict__ parent, Meta* __restrict__ meta, int64_t n,
                                                     int local_only) {
    FEC_PROLOGUE_GRID(gp);
    union_sparse_body(spts, cw, ccoord, cstart, g, parent, meta, n, local_only);
}
// Node-level tail (see node_accumulate): every used component node finds its root, is
// flattened onto it, and adds its own totals to the root's; then the points of sparse cells
// (the compact list of k_cellscan) find their roots, are flattened and counted one by one.
// Only for dense-grid clouds with few sparse cells; the others run k_flatten_if + k_tail_stats.




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
                                                           const int* __restrict__ slist,
                                                           const Grid* __restrict__ gp,
                                                           int* __restrict__ parent, Meta* __restrict__ meta,
                                                           int64_t n, int local_only) {
    FEC_PROLOGUE_GRID(gp);
    if (g.status || (!local_only && 4 * (int64_t)meta->cells > n)) return;
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

// a10, second half, clouds with few sparse cells (the node tail): walk the INPUT order, so the
// labels are written coalesced and no sorted-order array is read.  A point's cell (from its
// coordinates, the same arithmetic as binning) gives its record word: a point of a dense cell
// takes the folded label of its component's node (its fine sub-cell picks the component); a point
// of a sparse cell is found among the cell's <= 6 sorted points (by its index) and takes its
// root's folded label.  (The sorted-order pass below serves sparse-dominated clouds.)
__global__ void __launch_bounds__(256) k_relabel_in(const float* __restrict__ p, int64_t n,
                                                   const Grid* __restrict__ gp, const uint2* __restrict__ cw,
                                                   const int* __restrict__ crec, const u64* __restrict__ cmask,
                                                   const uint32_t* __restrict__ cstart,
                                                   const float4* __restrict__ spts, const int* __restrict__ parent,
                                                   const int* __restrict__ minidx, int* __restrict__ labels,
                                                   const Meta* __restrict__ meta, const uint32_t* __restrict__ pcode) {
    FEC_PROLOGUE_GRID(gp);
    if (g.status || 4 * (int64_t)meta->cells > n) return;  // (sparse-dominated: from the sorted order)
    const bool vec = (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
    // (codes exist on the counting path when cells <= kCodeCells; node-tail clouds have
    // cells <= n/4 and the key-sort path writes none)
    const bool rcode = !g.key_sort && meta->cells <= kCodeCells;
    const int64_t groups = (n + 3) / 4;
    for (int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < groups; gi += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b4 = 4 * gi;
        int rv[4], q[4];
        uint32_t cid[4];
        if (rcode) {
            load4_stream(pcode, b4, n, cid);  // (read once: no L1 allocation, the L1 keeps crec)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                q[j] = (int)(cid[j] & 63u);
                cid[j] >>= 6;
            }
        } else {
            Pts4 P;
            load_pts4(p, n, b4, vec, P);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                q[j] = 0;
                cid[j] = 0;
                if (b4 + j >= n) continue;
                uint32_t lin;
                dense_cell_of(P.x[j], P.y[j], P.z[j], b4 + j, g, lin, q[j]);
                cid[j] = cid_of(cw, lin);
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            rv[j] = 0;
            if (b4 + j >= n) continue;
            // -1 sparse cell; <= -2 single-component dense cell: -(label + 3) (k_rootlab);
            // >= 0 several components: record << 3 | (components - 1)
            rv[j] = __ldg(crec + cid[j]);
        }
        int lab[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            lab[j] = -1;
            if (b4 + j >= n) continue;
            if (rv[j] <= -2) {
                lab[j] = -rv[j] - 3;
            } else if (rv[j] >= 0) {
                const int r = rv[j] >> 3, kc = (rv[j] & 7) + 1;
                int c = 0;
                if (kc > 1)
                    while (c < kc - 1 && !((__ldg(cmask + 8 * r + c) >> q[j]) & 1ull)) ++c;
                lab[j] = __ldg(minidx + node_of((int)n, g.rmask, r, c));
            } else {
                const int s0 = (int)__ldg(cstart + cid[j]), s1 = (int)__ldg(cstart + cid[j] + 1);
                for (int t = s0; t < s1; ++t)
                    if (__float_as_int(__ldg(spts + t).w) == (int)(b4 + j)) {
                        lab[j] = __ldg(minidx + __ldg(parent + t));
                        break;
                    }
            }
            if (g.batch && lab[j] >= 0) lab[j] -= (int)__ldg(g.boff + cloud_of(g, b4 + j));
        }
        if (b4 + 4 <= n && (reinterpret_cast<uintptr_t>(labels) & 15u) == 0) {
            *reinterpret_cast<int4*>(labels + b4) = make_int4(lab[0], lab[1], lab[2], lab[3]);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (b4 + j < n) labels[b4 + j] = lab[j];
        }
    }
}

}  // namespace fec

// ---- host: sub-cell tables, uploaded once per device -------------------------------------
#include <mutex>

namespace fec {

// The device tables are a compile-time constant; this checks once, on the host, that the
// bit-operation dilation used by the flood fill and the whole-mask shift lists agree with
// the tables' certain relation (a failed check would be a build defect).
cudaError_t ensure_subcell_tables() {
    static const bool ok = [] {
        constexpr SubcellTables t = sc_make_tables();
        for (int a = 0; a < 64; ++a)
            if ((sc_dilate(1ull << a) | (1ull << a)) != (t.T[13][a] | (1ull << a))) return false;
        for (int sl = 0; sl < 27; ++sl) {
            if (sl == 13) continue;
            if (t.nsh[sl] < 0) return false;
            for (int a = 0; a < 64; ++a)
                if (sc_certain_across(t, 1ull << a, sl) != t.T[sl][a]) return false;
        }
        return true;
    }();
    return ok ? cudaSuccess : cudaErrorInvalidValue;
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
