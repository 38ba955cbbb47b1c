// FEC hot-path kernels for sm_100a.  Step numbering follows SURVEY.md §8(a) / DESIGN.md §4:
//   a1 K0 bbox+validate | a2 K1 keys | a3 K2 radix sort | a4 K3 gather | a5 K4 group/cell
//   tables | a6+a7 K5 neighbour scan + union | a8 K6 flatten | a9 K7 stats | a10 K8 relabel
#include <float.h>

#include "fec_internal.cuh"
#include "fec_kernels.cuh"
#include "fec_pairs.cuh"

namespace fec {

// =====================================================================================
// a1  K0: validation + bounding box (isfinite over all 3n floats; per-axis min/max)
// =====================================================================================
__device__ __forceinline__ void bb_acc(float v, float& mn, float& mx, int& bad) {
    bad |= !isfinite(v);
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
}

// Also counts consecutive input pairs (i, i+1) within `near` on every axis (spatial coherence
// of the input order: decides between the counting sort and the key sort).
__global__ void __launch_bounds__(256) k_bbox_partial(const float* __restrict__ p, int64_t n, int vec4,
                                                     float* __restrict__ part, int* __restrict__ nonfinite,
                                                     float near, unsigned long long* __restrict__ near_pairs) {
    pdl_prologue();
    float mn[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    int bad = 0;
    unsigned nearc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t tail_start = 0;
    if (vec4) {
        // 4 points = 12 floats = 3 float4 per quad; the pointer is 16-byte aligned
        const float4* q = reinterpret_cast<const float4*>(p);
        const int64_t nq = n >> 2;
        for (int64_t i = t0; i < nq; i += stride) {
            float4 a = __ldg(q + 3 * i), b = __ldg(q + 3 * i + 1), c = __ldg(q + 3 * i + 2);
            float v[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
#pragma unroll
            for (int k = 0; k < 12; ++k) bb_acc(v[k], mn[k % 3], mx[k % 3], bad);
#pragma unroll
            for (int j = 0; j < 3; ++j)
                nearc += fabsf(v[3 * j + 3] - v[3 * j]) <= near && fabsf(v[3 * j + 4] - v[3 * j + 1]) <= near &&
                         fabsf(v[3 * j + 5] - v[3 * j + 2]) <= near;
        }
        tail_start = nq << 2;
    }
    for (int64_t i = tail_start + t0; i < n; i += stride) {
#pragma unroll
        for (int k = 0; k < 3; ++k) bb_acc(__ldg(p + 3 * i + k), mn[k], mx[k], bad);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[k] = fminf(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], o));
            mx[k] = fmaxf(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], o));
        }
    }
    bad = __any_sync(0xffffffffu, bad);
    for (int o = 16; o > 0; o >>= 1) nearc += __shfl_xor_sync(0xffffffffu, nearc, o);
    if ((threadIdx.x & 31) == 0 && nearc) atomicAdd(near_pairs, (unsigned long long)nearc);
    __shared__ float s[8][6];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) { s[w][k] = mn[k]; s[w][3 + k] = mx[k]; }
        if (bad) atomicOr(nonfinite, 1);
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        float v = s[0][threadIdx.x];
        for (int ww = 1; ww < (int)(blockDim.x >> 5); ++ww)
            v = threadIdx.x < 3 ? fminf(v, s[ww][threadIdx.x]) : fmaxf(v, s[ww][threadIdx.x]);
        part[blockIdx.x * 6 + threadIdx.x] = v;
    }
}

__global__ void __launch_bounds__(256) k_bbox_final(const float* __restrict__ part, int nblocks,
                                                   Meta* __restrict__ meta, HostBBox* hb, int seq) {
    pdl_prologue();
    float mn[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            mn[k] = fminf(mn[k], part[b * 6 + k]);
            mx[k] = fmaxf(mx[k], part[b * 6 + 3 + k]);
        }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[k] = fminf(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], o));
            mx[k] = fmaxf(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], o));
        }
    }
    __shared__ float s[8][6];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) { s[w][k] = mn[k]; s[w][3 + k] = mx[k]; }
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        float v = s[0][threadIdx.x];
        for (int ww = 1; ww < (int)(blockDim.x >> 5); ++ww)
            v = threadIdx.x < 3 ? fminf(v, s[ww][threadIdx.x]) : fmaxf(v, s[ww][threadIdx.x]);
        meta->bbox[threadIdx.x] = v;
        if (hb) hb->bbox[threadIdx.x] = v;
    }
    if (hb) {
        __syncthreads();
        if (threadIdx.x == 0) {
            hb->nonfinite = meta->nonfinite;
            hb->near_pairs = meta->near_pairs;
            __threadfence_system();
            *reinterpret_cast<volatile int*>(&hb->seq) = seq;
        }
    }
}

// Batch mode: one block per cloud [off[c], off[c+1]): its bbox (6 floats at bb[6c]), the
// non-finite flag and the near-pair count (consecutive pairs inside the cloud).
__global__ void __launch_bounds__(256) k_bbox_clouds(const float* __restrict__ p, const int64_t* __restrict__ off,
                                                    float* __restrict__ bb, int* __restrict__ nonfinite, float near,
                                                    unsigned long long* __restrict__ near_pairs) {
    pdl_prologue();
    const int c = blockIdx.x;
    const int64_t a = off[c], b = off[c + 1];
    float mn[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    int bad = 0;
    unsigned nearc = 0;
    for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) {
        float v[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            v[k] = __ldg(p + 3 * i + k);
            bb_acc(v[k], mn[k], mx[k], bad);
        }
        if (i + 1 < b)
            nearc += fabsf(__ldg(p + 3 * i + 3) - v[0]) <= near && fabsf(__ldg(p + 3 * i + 4) - v[1]) <= near &&
                     fabsf(__ldg(p + 3 * i + 5) - v[2]) <= near;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[k] = fminf(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], o));
            mx[k] = fmaxf(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], o));
        }
    }
    bad = __any_sync(0xffffffffu, bad);
    for (int o = 16; o > 0; o >>= 1) nearc += __shfl_xor_sync(0xffffffffu, nearc, o);
    __shared__ float s[8][6];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) { s[w][k] = mn[k]; s[w][3 + k] = mx[k]; }
        if (bad) atomicOr(nonfinite, 1);
        if (nearc) atomicAdd(near_pairs, (unsigned long long)nearc);
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        float v = s[0][threadIdx.x];
        for (int ww = 1; ww < (int)(blockDim.x >> 5); ++ww)
            v = threadIdx.x < 3 ? fminf(v, s[ww][threadIdx.x]) : fmaxf(v, s[ww][threadIdx.x]);
        bb[6 * c + threadIdx.x] = v;
    }
}

// =====================================================================================
// a2  K1: sub-cell Morton keys; idx = iota
// =====================================================================================
__global__ void __launch_bounds__(256) k_keys(const float* __restrict__ p, int64_t n, Grid g,
                                             u64* __restrict__ key, int* __restrict__ val) {
    pdl_prologue();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t sx = sub_coord(__ldg(p + 3 * i), g.lo[0], g.inv_h);
        uint32_t sy = sub_coord(__ldg(p + 3 * i + 1), g.lo[1], g.inv_h);
        uint32_t sz = sub_coord(__ldg(p + 3 * i + 2), g.lo[2], g.inv_h);
        key[i] = subcell_key(sx, sy, sz, g);
        val[i] = (int)i;
    }
}

// =====================================================================================
// a3  K2: LSD radix sort, 8-bit digits, stable (reduce-then-scan per pass)
// =====================================================================================
template <typename K>
__device__ __forceinline__ void radix_hist(const K* __restrict__ key, int64_t n, int shift, uint32_t* __restrict__ counts,
                                           int num_tiles) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll 4
    for (int k = 0; k < RS_ITEMS; ++k) {
        int64_t i = base + k * RS_THREADS + threadIdx.x;
        if (i < n) atomicAdd(&h[(unsigned)(key[i] >> shift) & 255u], 1u);
    }
    __syncthreads();
    counts[(int64_t)threadIdx.x * num_tiles + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter.  Warp w of a tile owns the contiguous keys [w*512, w*512+512); iteration
// `it` covers 32 consecutive keys, so (warp, it, lane) order equals input order.  Ranks:
// (digit offset of this tile) + (same-digit keys in earlier warps) + (in earlier
// iterations of this warp) + (in lower lanes of this iteration).
template <typename K>
__device__ __forceinline__ void radix_scatter(const K* __restrict__ kin, const int* __restrict__ vin,
                                              K* __restrict__ kout, int* __restrict__ vout, int64_t n, int shift,
                                              const uint32_t* __restrict__ offs, int num_tiles) {
    __shared__ uint32_t wcnt[RS_THREADS / kWarp][256];
    __shared__ uint32_t goff[256];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int d = threadIdx.x; d < (RS_THREADS / kWarp) * 256; d += RS_THREADS) (&wcnt[0][0])[d] = 0;
    goff[threadIdx.x] = offs[(int64_t)threadIdx.x * num_tiles + blockIdx.x];
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE + (int64_t)w * (RS_ITEMS * kWarp);
    const unsigned lt = (1u << lane) - 1u;
    K k[RS_ITEMS];
    int v[RS_ITEMS];
    uint32_t rank[RS_ITEMS];
    int dig[RS_ITEMS];
#pragma unroll
    for (int it = 0; it < RS_ITEMS; ++it) {
        int64_t i = base + it * kWarp + lane;
        bool ok = i < n;
        k[it] = ok ? kin[i] : K(0);
        v[it] = ok ? vin[i] : 0;
        dig[it] = ok ? (int)((unsigned)(k[it] >> shift) & 255u) : 256;
    }
#pragma unroll
    for (int it = 0; it < RS_ITEMS; ++it) {
        const int d = dig[it];
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t c = d < 256 ? wcnt[w][d] : 0u;
        __syncwarp();
        rank[it] = c + __popc(peers & lt);
        if (d < 256 && (peers & lt) == 0u) wcnt[w][d] = c + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {
        const int d = threadIdx.x;
        uint32_t run = 0;
#pragma unroll
        for (int ww = 0; ww < RS_THREADS / kWarp; ++ww) {
            uint32_t t = wcnt[ww][d];
            wcnt[ww][d] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < RS_ITEMS; ++it) {
        const int d = dig[it];
        if (d < 256) {
            uint32_t pos = goff[d] + wcnt[w][d] + rank[it];
            kout[pos] = k[it];
            vout[pos] = v[it];
        }
    }
}

__global__ void __launch_bounds__(RS_THREADS) k_radix_hist(const u64* __restrict__ key, int64_t n, int shift,
                                                          uint32_t* __restrict__ counts, int num_tiles) {
    pdl_prologue();
    radix_hist<u64>(key, n, shift, counts, num_tiles);
}
__global__ void __launch_bounds__(RS_THREADS) k_radix_scatter(const u64* __restrict__ kin, const int* __restrict__ vin,
                                                             u64* __restrict__ kout, int* __restrict__ vout,
                                                             int64_t n, int shift, const uint32_t* __restrict__ offs,
                                                             int num_tiles) {
    pdl_prologue();
    radix_scatter<u64>(kin, vin, kout, vout, n, shift, offs, num_tiles);
}
// 32-bit keys (linear cell ids of the dense grid's key-sort path).  The scatter first sorts
// the tile by digit in shared memory, then writes each digit's run with consecutive threads
// (coalesced stores instead of one scattered 4-byte store per key and value).
__global__ void __launch_bounds__(RS_THREADS) k_radix_scatter32l(const uint32_t* __restrict__ kin,
                                                                const int* __restrict__ vin,
                                                                uint32_t* __restrict__ kout, int* __restrict__ vout,
                                                                int64_t n, int shift, const uint32_t* __restrict__ offs,
                                                                int num_tiles) {
    pdl_prologue();
    __shared__ uint32_t wcnt[RS_THREADS / kWarp][256];
    __shared__ uint32_t goff[256], tstart[256];
    __shared__ uint32_t sk[RS_TILE];
    __shared__ int sv[RS_TILE];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int d = threadIdx.x; d < (RS_THREADS / kWarp) * 256; d += RS_THREADS) (&wcnt[0][0])[d] = 0;
    goff[threadIdx.x] = offs[(int64_t)threadIdx.x * num_tiles + blockIdx.x];
    __syncthreads();
    const int64_t tbase = (int64_t)blockIdx.x * RS_TILE;
    const int64_t base = tbase + (int64_t)w * (RS_ITEMS * kWarp);
    const unsigned lt = (1u << lane) - 1u;
    uint32_t k[RS_ITEMS];
    int v[RS_ITEMS];
    uint32_t rank[RS_ITEMS];
    int dig[RS_ITEMS];
#pragma unroll
    for (int it = 0; it < RS_ITEMS; ++it) {
        int64_t i = base + it * kWarp + lane;
        bool ok = i < n;
        k[it] = ok ? kin[i] : 0u;
        v[it] = ok ? vin[i] : 0;
        dig[it] = ok ? (int)((k[it] >> shift) & 255u) : 256;
    }
#pragma unroll
    for (int it = 0; it < RS_ITEMS; ++it) {
        const int d = dig[it];
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t c = d < 256 ? wcnt[w][d] : 0u;
        __syncwarp();
        rank[it] = c + __popc(peers & lt);
        if (d < 256 && (peers & lt) == 0u) wcnt[w][d] = c + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {
        // per digit: exclusive offsets of the warps, and the tile's digit total
        const int d = threadIdx.x;
        uint32_t run = 0;
#pragma unroll
        for (int ww = 0; ww < RS_THREADS / kWarp; ++ww) {
            uint32_t t = wcnt[ww][d];
            wcnt[ww][d] = run;
            run += t;
        }
        tstart[d] = run;  // digit total for now
    }
    __syncthreads();
    // exclusive scan of the 256 digit totals (one warp)
    if (w == 0) {
        uint32_t a[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) { a[j] = tstart[8 * lane + j]; sum += a[j]; }
        uint32_t x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        uint32_t run = x - sum;
#pragma unroll
        for (int j = 0; j < 8; ++j) { tstart[8 * lane + j] = run; run += a[j]; }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < RS_ITEMS; ++it) {
        const int d = dig[it];
        if (d < 256) {
            const uint32_t lp = tstart[d] + wcnt[w][d] + rank[it];
            sk[lp] = k[it];
            sv[lp] = v[it];
        }
    }
    __syncthreads();
    const int cnt = (int)min((int64_t)RS_TILE, n - tbase);
    for (int lp = threadIdx.x; lp < cnt; lp += RS_THREADS) {
        const uint32_t key = sk[lp];
        const int d = (int)((key >> shift) & 255u);
        const uint32_t pos = goff[d] + ((uint32_t)lp - tstart[d]);
        kout[pos] = key;
        vout[pos] = sv[lp];
    }
}

__global__ void __launch_bounds__(RS_THREADS) k_radix_hist32(const uint32_t* __restrict__ key, int64_t n, int shift,
                                                            uint32_t* __restrict__ counts, int num_tiles) {
    pdl_prologue();
    radix_hist<uint32_t>(key, n, shift, counts, num_tiles);
}
__global__ void __launch_bounds__(RS_THREADS) k_radix_scatter32(const uint32_t* __restrict__ kin,
                                                               const int* __restrict__ vin, uint32_t* __restrict__ kout,
                                                               int* __restrict__ vout, int64_t n, int shift,
                                                               const uint32_t* __restrict__ offs, int num_tiles) {
    pdl_prologue();
    radix_scatter<uint32_t>(kin, vin, kout, vout, n, shift, offs, num_tiles);
}

// =====================================================================================
// a4  K3: gather points into sorted order as float4 (x, y, z, idx)
// =====================================================================================
__global__ void __launch_bounds__(256) k_gather(const float* __restrict__ p, const int* __restrict__ val, int64_t n,
                                               float4* __restrict__ spts) {
    pdl_prologue();
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        int i = val[s];
        spts[s] = make_float4(__ldg(p + 3 * (int64_t)i), __ldg(p + 3 * (int64_t)i + 1), __ldg(p + 3 * (int64_t)i + 2),
                              __int_as_float(i));
    }
}

// =====================================================================================
// a5  K4: group (sub-cell) and cell tables
// =====================================================================================
// flags[s] = groupHead | cellHead << 32 ; flags[n] = 0 (so the exclusive scan yields totals)
__global__ void __launch_bounds__(256) k_heads(const u64* __restrict__ key, int64_t n, u64* __restrict__ flags) {
    pdl_prologue();
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s <= n; s += (int64_t)gridDim.x * blockDim.x) {
        u64 f = 0;
        if (s < n) {
            u64 k = key[s];
            if (s == 0) {
                f = 1ull | (1ull << 32);
            } else {
                u64 kp = key[s - 1];
                f = (u64)(k != kp) | ((u64)((k >> 3) != (kp >> 3)) << 32);
            }
        }
        flags[s] = f;
    }
}

__device__ __forceinline__ void decode_cell(u64 key, const Grid& g, uint32_t& cx, uint32_t& cy, uint32_t& cz) {
    uint32_t c[3] = {0u, 0u, 0u};
    int pos = 3;
    int maxb = max(g.bits[0], max(g.bits[1], g.bits[2]));
    for (int l = 0; l < maxb; ++l) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (l < g.bits[a]) {
                c[a] |= (uint32_t)((key >> pos) & 1ull) << l;
                ++pos;
            }
        }
    }
    cx = c[0]; cy = c[1]; cz = c[2];
}

__global__ void __launch_bounds__(256) k_fill_tables(const u64* __restrict__ key, const u64* __restrict__ ex, int64_t n,
                                                    Grid g, Tables T, Meta* __restrict__ meta) {
    pdl_prologue();
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const u64 e0 = ex[s], e1 = ex[s + 1];
        const u64 d = e1 - e0;
        const int gidx = (int)(uint32_t)e0;
        const int cidx = (int)(e0 >> 32);
        if (d & 1ull) {  // group head
            const u64 k = key[s];
            T.gstart[gidx] = (int)s;
            T.goct[gidx] = (uint8_t)(k & 7ull);
            if (d >> 32) {  // cell head
                T.cell_gstart[cidx] = gidx;
                uint32_t cx, cy, cz;
                decode_cell(k, g, cx, cy, cz);
                const u64 pc = pack_cell(cx, cy, cz);
                T.cell_pc[cidx] = pc;
                if (g.dense) {
                    T.dense[((int64_t)cz * g.dims[1] + cy) * g.dims[0] + cx] = cidx;
                } else {
                    u64 slot = hash_cell(pc) & g.hash_mask;
                    while (true) {
                        u64 prev = atomicCAS(T.hkey + slot, ~0ull, pc);
                        if (prev == ~0ull) { T.hval[slot] = cidx; break; }
                        slot = (slot + 1) & g.hash_mask;
                    }
                }
            }
        }
        if (s == n - 1) {
            const u64 tot = ex[n];
            const int G = (int)(uint32_t)tot, U = (int)(tot >> 32);
            T.gstart[G] = (int)n;
            T.cell_gstart[U] = G;
            meta->groups = G;
            meta->cells = U;
        }
    }
}

// parent[s] = last point of s's sub-cell (sub-cells are cliques under pred: DESIGN.md §4.5);
// size/minidx accumulators initialised here too.
__global__ void __launch_bounds__(256) k_init_uf(const u64* __restrict__ ex, const int* __restrict__ gstart, int64_t n,
                                                int* __restrict__ parent, int* __restrict__ size,
                                                int* __restrict__ minidx) {
    pdl_prologue();
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const int gidx = (int)(uint32_t)ex[s + 1] - 1;
        parent[s] = gstart[gidx + 1] - 1;
        size[s] = 0;
        minidx[s] = 0x7fffffff;
    }
}

// =====================================================================================
// a6+a7  K5: neighbour scan fused with union (warp per cell; sub-cell group pairs)
// =====================================================================================
__device__ __forceinline__ int cell_lookup(const Grid& g, const Tables& T, int cx, int cy, int cz) {
    if (cx < 0 || cy < 0 || cz < 0 || cx >= g.dims[0] || cy >= g.dims[1] || cz >= g.dims[2]) return -1;
    const u64 pc = pack_cell((uint32_t)cx, (uint32_t)cy, (uint32_t)cz);
    u64 slot = hash_cell(pc) & g.hash_mask;
    while (true) {
        const u64 k = __ldg(T.hkey + slot);
        if (k == pc) return __ldg(T.hval + slot);
        if (k == ~0ull) return -1;
        slot = (slot + 1) & g.hash_mask;
    }
}

constexpr int kCellChunk = 8;  // cells taken per atomic on the dynamic work counter

// Hash mode (sparse, huge bounding boxes): warp per nonempty cell, cells visited in Morton
// order, groups = octants of the cell.
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_union(const float4* __restrict__ spts, Grid g, Tables T,
                                                           int* __restrict__ parent, Meta* __restrict__ meta) {
    pdl_prologue();
    __shared__ PairSmem sm[SCAN_THREADS / kWarp];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    PairSmem& S = sm[w];
    const int U = meta->cells;
    const float t2 = g.t2;
    unsigned long long n_tests = 0, n_pairs = 0;

    while (true) {
        int c0 = 0;
        if (lane == 0) c0 = atomicAdd(&meta->work, kCellChunk);
        c0 = __shfl_sync(0xffffffffu, c0, 0);
        if (c0 >= U) break;
        const int c1 = min(U, c0 + kCellChunk);
        for (int c = c0; c < c1; ++c) {
            const int gs = __ldg(T.cell_gstart + c), ge = __ldg(T.cell_gstart + c + 1);
            const int np = ge - gs;
            if (lane <= np) S.ps[lane] = __ldg(T.gstart + gs + lane);
            if (lane < np) S.po[lane] = __ldg(T.goct + gs + lane);
            const u64 pc = __ldg(T.cell_pc + c);
            const int cx = (int)(pc & 0x1fffff), cy = (int)((pc >> 21) & 0x1fffff), cz = (int)(pc >> 42);
            int qcell = -1;
            if (lane < 13) qcell = cell_lookup(g, T, cx + c_fwd[lane][0], cy + c_fwd[lane][1], cz + c_fwd[lane][2]);
            __syncwarp();
            for (int k = -1; k < 13; ++k) {
                const int q = k < 0 ? c : __shfl_sync(0xffffffffu, qcell, k);
                if (q < 0) continue;
                int nq;
                if (k < 0) {
                    nq = np;
                    if (lane <= np) S.qs[lane] = S.ps[lane];
                    if (lane < np) S.qo[lane] = S.po[lane];
                } else {
                    const int qgs = __ldg(T.cell_gstart + q), qge = __ldg(T.cell_gstart + q + 1);
                    nq = qge - qgs;
                    if (lane <= nq) S.qs[lane] = __ldg(T.gstart + qgs + lane);
                    if (lane < nq) S.qo[lane] = __ldg(T.goct + qgs + lane);
                }
                __syncwarp();
                load_roots(S, np, nq, parent, lane);
                const int2 nqueue = k < 0 ? build_queue(S, np, nq, true, 0, 0, 0, lane)
                                          : build_queue(S, np, nq, false, c_fwd[k][0], c_fwd[k][1], c_fwd[k][2], lane);
                n_pairs += (lane == 0) ? (unsigned long long)(nqueue.x + nqueue.y) : 0ull;
                process_queue(S, nqueue, spts, parent, t2, lane, n_tests);
            }
        }
    }
    if (meta->instrument) {
        for (int o = 16; o > 0; o >>= 1) {
            n_tests += __shfl_xor_sync(0xffffffffu, n_tests, o);
            n_pairs += __shfl_xor_sync(0xffffffffu, n_pairs, o);
        }
        if (lane == 0) {
            atomicAdd(&meta->pair_tests, n_tests);
            atomicAdd(&meta->group_pairs, n_pairs);
        }
    }
}

// =====================================================================================
// a8  K6: flatten   a9  K7: component stats   a10  K8: filter + relabel + scatter
// =====================================================================================
// Read-only root walk, then one store per element.  (A compressing find here would let a
// thread's late path-halving store overwrite another thread's final root with a stale
// intermediate; each parent[s] must be written only by its own thread.)
// Also initialises the accumulators of root points (component nodes get theirs in k_dcomps).
__global__ void __launch_bounds__(256) k_flatten(int* __restrict__ parent, int64_t n, int* __restrict__ size,
                                                int* __restrict__ minidx) {
    pdl_prologue();
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        int curr = ld_parent(parent, (int)s), next;
        if (curr == (int)s) {
            size[s] = 0;
            minidx[s] = 0x7fffffff;
            continue;
        }
        while (curr < (next = ld_parent(parent, curr))) curr = next;
        st_parent(parent, (int)s, curr);
    }
}

// Component size and minimum input index per root.  Atomics are aggregated per warp (one
// per distinct root in the warp) and then per block through a small shared-memory table,
// so a giant component (C5: ~40% of all points) costs one global atomic per block instead
// of one per warp.  Blocks own contiguous ranges (the sorted order is spatial).
constexpr int HH_SLOTS = 256;
// `only_sparse`: run only for sparse-dominated clouds (occupied cells > n/4; the forest was
// flattened by k_flatten_if), where per-lane aggregation of this form is the faster one.
__device__ __forceinline__ void stats_body(const int* __restrict__ parent, const int* __restrict__ val, int64_t n,
                                              int* __restrict__ size, int* __restrict__ minidx,
                                              Meta* __restrict__ meta, int only_sparse, int bid, int nblk) {
    if (only_sparse && 4 * (int64_t)meta->cells <= n) return;
    __shared__ int hkey[HH_SLOTS], hcnt[HH_SLOTS], hmin[HH_SLOTS];
    for (int k = threadIdx.x; k < HH_SLOTS; k += blockDim.x) { hkey[k] = -1; hcnt[k] = 0; hmin[k] = 0x7fffffff; }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned long long roots = 0;
    const int64_t chunk = ((n + nblk - 1) / nblk + 255) / 256 * 256;
    const int64_t b0 = (int64_t)bid * chunk, b1 = min(n, b0 + chunk);
    for (int64_t s0 = b0; s0 < b1; s0 += blockDim.x) {
        const int64_t s = s0 + threadIdx.x;
        const bool ok = s < b1;
        const int r = ok ? __ldg(parent + s) : -1;
        const int v = ok ? __ldg(val + s) : 0x7fffffff;
        roots += (ok && r == (int)s) ? 1ull : 0ull;
        unsigned todo = __ballot_sync(0xffffffffu, ok);
        while (todo) {
            const int leader = __ffs(todo) - 1;
            const int key = __shfl_sync(0xffffffffu, r, leader);
            const bool mem = ok && r == key;
            const unsigned peers = __ballot_sync(0xffffffffu, mem);
            const int mn = __reduce_min_sync(0xffffffffu, mem ? v : 0x7fffffff);
            if (lane == leader) {
                const int cnt = __popc(peers);
                unsigned h = ((unsigned)key * 2654435761u) >> 24;  // 256 slots
                bool done = false;
                for (int probe = 0; probe < 4 && !done; ++probe, h = (h + 1) & (HH_SLOTS - 1)) {
                    int cur = hkey[h];
                    if (cur == -1) cur = atomicCAS(&hkey[h], -1, key);
                    if (cur == -1 || cur == key) {
                        atomicAdd(&hcnt[h], cnt);
                        atomicMin(&hmin[h], mn);
                        done = true;
                    }
                }
                if (!done) {
                    atomicAdd(size + key, cnt);
                    atomicMin(minidx + key, mn);
                }
            }
            todo &= ~peers;
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < HH_SLOTS; k += blockDim.x) {
        if (hkey[k] >= 0) {
            atomicAdd(size + hkey[k], hcnt[k]);
            atomicMin(minidx + hkey[k], hmin[k]);
        }
    }
    if (meta->instrument) {
        for (int o = 16; o > 0; o >>= 1) roots += __shfl_xor_sync(0xffffffffu, roots, o);
        if (lane == 0 && roots) atomicAdd(&meta->components, roots);
    }
}
__global__ void __launch_bounds__(256) k_stats(const int* __restrict__ parent, const int* __restrict__ val, int64_t n,
                                              int* __restrict__ size, int* __restrict__ minidx,
                                              Meta* __restrict__ meta, int only_sparse) {
    pdl_prologue();
    stats_body(parent, val, n, size, minidx, meta, only_sparse, blockIdx.x, gridDim.x);
}

// Sparse-dominated clouds (many small components, deep forests: occupied cells > n/4)
// flatten in a separate pass first; k_flat_stats's walks are then one load each.
__global__ void __launch_bounds__(256) k_flatten_if(int* __restrict__ parent, int64_t n, const Meta* __restrict__ meta) {
    pdl_prologue();
    if (4 * (int64_t)meta->cells <= n) return;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        int curr = ld_parent(parent, (int)s), next;
        if (curr == (int)s) continue;
        while (curr < (next = ld_parent(parent, curr))) curr = next;
        st_parent(parent, (int)s, curr);
    }
}

// Single-GPU tail, a8+a9 fused: every point's root (read-only walk; the root is written back,
// which flattens the forest for k_relabel) and the component size + minimum input index,
// aggregated per warp and per block as in k_stats.  Roots' accumulators were initialised
// earlier (points of sparse cells in k_dinit / k_sgather, component nodes in k_dcomps, hashed
// mode in k_init_uf).
__device__ __forceinline__ void flat_stats_body(int* __restrict__ parent, const int* __restrict__ val, int64_t n,
                                                   int* __restrict__ size, int* __restrict__ minidx,
                                                   Meta* __restrict__ meta, int node_tail, int bid, int nblk) {
    if (4 * (int64_t)meta->cells > n) return;  // sparse-dominated: k_flatten_if + k_stats
    if (node_tail) return;                     // dense grid: k_node_stats + k_sparse_stats
    __shared__ int hkey[HH_SLOTS], hcnt[HH_SLOTS], hmin[HH_SLOTS];
    for (int k = threadIdx.x; k < HH_SLOTS; k += blockDim.x) { hkey[k] = -1; hcnt[k] = 0; hmin[k] = 0x7fffffff; }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned long long roots = 0;
    const int64_t per = 4 * (int64_t)blockDim.x;
    const int64_t chunk = ((n + nblk - 1) / nblk + per - 1) / per * per;
    const int64_t b0 = (int64_t)bid * chunk, b1 = min(n, b0 + chunk);
    for (int64_t s0 = b0; s0 < b1; s0 += per) {
        // round j covers positions s0 + j*blockDim + threadIdx.x: a warp holds 32 consecutive
        // positions per round (equal roots meet in one aggregation step); the 4 rounds' loads
        // are issued together
        int r[4], v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t s = s0 + j * (int64_t)blockDim.x + threadIdx.x;
            r[j] = s < b1 ? ld_parent(parent, (int)s) : -1;
            v[j] = s < b1 ? __ldg(val + s) : 0x7fffffff;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (r[j] < 0) continue;
            const int s = (int)(s0 + j * (int64_t)blockDim.x + threadIdx.x);
            if (r[j] == s) {
                ++roots;
                continue;
            }
            int curr = r[j], next;
            while (curr < (next = ld_parent(parent, curr))) curr = next;
            if (curr != r[j]) st_parent(parent, s, curr);
            r[j] = curr;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool ok = r[j] >= 0;
            unsigned todo = __ballot_sync(0xffffffffu, ok);
            while (todo) {
                const int leader = __ffs(todo) - 1;
                const int key = __shfl_sync(0xffffffffu, r[j], leader);
                const bool mem = ok && r[j] == key;
                const unsigned peers = __ballot_sync(0xffffffffu, mem);
                const int mn = __reduce_min_sync(0xffffffffu, mem ? v[j] : 0x7fffffff);
                if (lane == leader) {
                    const int cnt = __popc(peers);
                    unsigned h = ((unsigned)key * 2654435761u) >> 24;
                    bool done = false;
                    for (int probe = 0; probe < 4 && !done; ++probe, h = (h + 1) & (HH_SLOTS - 1)) {
                        int cur = hkey[h];
                        if (cur == -1) cur = atomicCAS(&hkey[h], -1, key);
                        if (cur == -1 || cur == key) {
                            atomicAdd(&hcnt[h], cnt);
                            atomicMin(&hmin[h], mn);
                            done = true;
                        }
                    }
                    if (!done) {
                        atomicAdd(size + key, cnt);
                        atomicMin(minidx + key, mn);
                    }
                }
                todo &= ~peers;
            }
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < HH_SLOTS; k += blockDim.x) {
        if (hkey[k] >= 0) {
            atomicAdd(size + hkey[k], hcnt[k]);
            atomicMin(minidx + hkey[k], hmin[k]);
        }
    }
    if (meta->instrument) {
        for (int o = 16; o > 0; o >>= 1) roots += __shfl_xor_sync(0xffffffffu, roots, o);
        if (lane == 0 && roots) atomicAdd(&meta->components, roots);
    }
}
__global__ void __launch_bounds__(256) k_flat_stats(int* __restrict__ parent, const int* __restrict__ val, int64_t n,
                                                   int* __restrict__ size, int* __restrict__ minidx,
                                                   Meta* __restrict__ meta, int node_tail) {
    pdl_prologue();
    flat_stats_body(parent, val, n, size, minidx, meta, node_tail, blockIdx.x, gridDim.x);
}


// ---- single-GPU tail, one launch for the stats of every mode ----------------------------
__device__ __forceinline__ void node_stats_body(int* __restrict__ parent, const int* __restrict__ ncomp,
                                                   int* __restrict__ size, int* __restrict__ minidx, int nbase,
                                                   Meta* __restrict__ meta, int64_t n, int bid, int nblk) {
    if (4 * (int64_t)meta->cells > n) return;
    const int64_t nn = 8 * (int64_t)meta->ndense;
    const int64_t nr = (nn + 31) & ~int64_t(31);  // whole warps stay in the loop
    const int lane = threadIdx.x & 31;
    for (int64_t t = (int64_t)bid * blockDim.x + threadIdx.x; t < nr; t += (int64_t)nblk * blockDim.x) {
        int root = -1, c = 0, m = 0x7fffffff;
        if (t < nn && (int)(t & 7) < __ldg(ncomp + (t >> 3))) {  // a used component slot
            const int node = nbase + (int)t;
            int curr = ld_parent(parent, node), next;
            if (curr == node) {  // a root keeps its own totals
                if (meta->instrument) atomicAdd(&meta->components, 1ull);
            } else {
                while (curr < (next = ld_parent(parent, curr))) curr = next;
                st_parent(parent, node, curr);
                c = size[node];
                if (c) {
                    root = curr;
                    m = minidx[node];
                }
            }
        }
        // nodes of one big component share a root: one atomic per distinct root per warp
        const unsigned peers = __match_any_sync(0xffffffffu, root);
        const int tot = __reduce_add_sync(peers, c);
        const int mn = __reduce_min_sync(peers, m);
        if (root >= 0 && lane == __ffs(peers) - 1) {
            atomicAdd(size + root, tot);
            atomicMin(minidx + root, mn);
        }
    }
}

__device__ __forceinline__ void sparse_stats_body(int* __restrict__ parent, const uint32_t* __restrict__ cstart,
                                                     const int* __restrict__ slist, const int* __restrict__ sidx,
                                                     int* __restrict__ size, int* __restrict__ minidx,
                                                     Meta* __restrict__ meta, int64_t n, int bid, int nblk) {
    if (4 * (int64_t)meta->cells > n) return;
    const int ns = meta->nsparse;
    const int lane = threadIdx.x & 31;
    // lane per sparse cell, the cells' points in lock-step rounds (<= SPARSE_MAX), and the
    // counts aggregated per distinct root over the warp (hot roots: one atomic per warp)
    const int nr = (ns + 31) & ~31;
    for (int e = bid * blockDim.x + threadIdx.x; e < nr; e += nblk * blockDim.x) {
        int a0 = 0, a1 = 0;
        if (e < ns) {
            const int P = __ldg(slist + e);
            a0 = (int)__ldg(cstart + P);
            a1 = (int)__ldg(cstart + P + 1);
        }
        for (int j = 0; j < SPARSE_MAX; ++j) {
            const int s = a0 + j;
            int curr = -1, v = 0x7fffffff;
            if (s < a1) {
                curr = ld_parent(parent, s);
                int next;
                if (curr != s) {
                    while (curr < (next = ld_parent(parent, curr))) curr = next;
                    st_parent(parent, s, curr);
                } else if (meta->instrument) {
                    atomicAdd(&meta->components, 1ull);
                }
                v = __ldg(sidx + s);
            }
            const unsigned peers = __match_any_sync(0xffffffffu, curr);
            const int cnt = __popc(peers);
            const int mn = __reduce_min_sync(peers, v);
            if (curr >= 0 && lane == __ffs(peers) - 1) {
                atomicAdd(size + curr, cnt);
                atomicMin(minidx + curr, mn);
            }
            if (!__any_sync(0xffffffffu, a0 + j + 1 < a1)) break;
        }
    }
}

__global__ void __launch_bounds__(256) k_node_stats(int* __restrict__ parent, const int* __restrict__ ncomp,
                                                   int* __restrict__ size, int* __restrict__ minidx, int nbase,
                                                   Meta* __restrict__ meta, int64_t n) {
    pdl_prologue();
    node_stats_body(parent, ncomp, size, minidx, nbase, meta, n, blockIdx.x, gridDim.x);
}

__global__ void __launch_bounds__(256) k_sparse_stats(int* __restrict__ parent, const uint32_t* __restrict__ cstart,
                                                     const int* __restrict__ slist, const int* __restrict__ sidx,
                                                     int* __restrict__ size, int* __restrict__ minidx,
                                                     Meta* __restrict__ meta, int64_t n) {
    pdl_prologue();
    sparse_stats_body(parent, cstart, slist, sidx, size, minidx, meta, n, blockIdx.x, gridDim.x);
}

// The component statistics of the single-GPU tail in one launch (the variant is a device-side
// choice): sparse-dominated clouds -> k_stats's body; dense grid with few sparse cells -> the
// node tail (first half of the blocks: component nodes, second half: points of sparse cells;
// independent: they only add into roots); otherwise (hashed mode) -> k_flat_stats's body.
__global__ void __launch_bounds__(256) k_tail_stats(int* __restrict__ parent, const int* __restrict__ val, int64_t n,
                                                   int* __restrict__ size, int* __restrict__ minidx,
                                                   Meta* __restrict__ meta, int dense, const int* __restrict__ ncomp,
                                                   const uint32_t* __restrict__ cstart, const int* __restrict__ slist) {
    pdl_prologue();
    if (4 * (int64_t)meta->cells > n) {
        stats_body(parent, val, n, size, minidx, meta, 1, blockIdx.x, gridDim.x);
    } else if (dense) {
        const int half = (int)(gridDim.x >> 1);  // >= 1: the host launches >= 2 blocks
        if ((int)blockIdx.x < half)
            node_stats_body(parent, ncomp, size, minidx, (int)n, meta, n, blockIdx.x, half);
        else
            sparse_stats_body(parent, cstart, slist, val, size, minidx, meta, n, blockIdx.x - half, gridDim.x - half);
    } else {
        flat_stats_body(parent, val, n, size, minidx, meta, 0, blockIdx.x, gridDim.x);
    }
}

// Sparse-dominated clouds (many components, roots scattered): fold the filter into the roots
// (minidx[r] = final label) so k_relabel reads one root word per point instead of two.
__global__ void __launch_bounds__(256) k_rootlab(const int* __restrict__ parent, const int* __restrict__ size,
                                                int* __restrict__ minidx, int64_t n, long long min_size,
                                                long long max_size, const Meta* __restrict__ meta) {
    pdl_prologue();
    if (4 * (int64_t)meta->cells <= n) return;
    const int64_t nodes = n + 8 * (int64_t)meta->ndense;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nodes; r += (int64_t)gridDim.x * blockDim.x) {
        if (__ldg(parent + r) != (int)r) continue;
        const long long sz = __ldg(size + r);
        if (!(sz >= min_size && sz <= max_size)) minidx[r] = -1;
    }
}

__global__ void __launch_bounds__(256) k_relabel(const int* __restrict__ parent, const int* __restrict__ val,
                                                const int* __restrict__ size, const int* __restrict__ minidx,
                                                int64_t n, long long min_size, long long max_size,
                                                int* __restrict__ labels, const Meta* __restrict__ meta,
                                                const int64_t* __restrict__ boff, int nclouds) {
    pdl_prologue();
    const bool folded = 4 * (int64_t)meta->cells > n;  // k_rootlab ran
    const int64_t groups = (n + 3) / 4;
    for (int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < groups; gi += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sb = 4 * gi;
        int r[4], v[4];
        if (sb + 4 <= n) {
            const int4 pr = __ldg(reinterpret_cast<const int4*>(parent + sb));
            const int4 vv = __ldg(reinterpret_cast<const int4*>(val + sb));
            r[0] = pr.x; r[1] = pr.y; r[2] = pr.z; r[3] = pr.w;
            v[0] = vv.x; v[1] = vv.y; v[2] = vv.z; v[3] = vv.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                r[j] = sb + j < n ? __ldg(parent + sb + j) : -1;
                v[j] = sb + j < n ? __ldg(val + sb + j) : -1;
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (r[j] < 0) continue;
            // a point of a dense cell points at its component node, which k_node_stats (or
            // the flattening walks) pointed at the root; roots point at themselves
            if (r[j] >= n) r[j] = __ldg(parent + r[j]);
            int lab;
            if (folded) {
                lab = __ldg(minidx + r[j]);
            } else {
                const long long sz = __ldg(size + r[j]);
                lab = (sz >= min_size && sz <= max_size) ? __ldg(minidx + r[j]) : -1;
            }
            if (boff && lab >= 0) {
                // batch mode: index inside the point's own cloud (the component never spans two)
                int lo = 0, hi = nclouds;
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (__ldg(boff + mid) <= (int64_t)v[j]) lo = mid;
                    else hi = mid;
                }
                lab -= (int)__ldg(boff + lo);
            }
            labels[v[j]] = lab;
        }
    }
}

// =====================================================================================
// diagnostic: the device predicate on m pairs (tests the fp32 order / no-FMA contract)
// =====================================================================================
__global__ void k_debug_pred(const float* __restrict__ a, const float* __restrict__ b, int64_t m, float t2,
                             uint8_t* __restrict__ out, float* __restrict__ d2out) {
    pdl_prologue();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        float4 pa = make_float4(a[3 * i], a[3 * i + 1], a[3 * i + 2], 0.f);
        float4 pb = make_float4(b[3 * i], b[3 * i + 1], b[3 * i + 2], 0.f);
        const float d2 = d2_rn(pa, pb);
        out[i] = d2 <= t2;
        if (d2out) d2out[i] = d2;
    }
}

}  // namespace fec
