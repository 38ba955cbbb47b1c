// FEC hot-path kernels for sm_100a.  Step numbering follows SURVEY.md §8(a) / DESIGN.md §4:
//   a1 K0 bbox+validate | a2 K1 keys | a3 K2 radix sort | a4 K3 gather | a5 K4 group/cell
//   tables | a6+a7 K5 neighbour scan + union | a8 K6 flatten | a9 K7 stats | a10 K8 relabel
#include <float.h>

#include "fec_internal.cuh"
#include "fec_kernels.cuh"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace fec {

// =====================================================================================
// a1  K0: validation + bounding box (isfinite over all 3n floats; per-axis min/max)
// =====================================================================================
__device__ __forceinline__ void bb_acc(float v, float& mn, float& mx, int& bad) {
    bad |= !isfinite(v);
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
}

// Device-side plan (reading A6 / A14), run by the last block of k_bbox:
// grid origin and dims from the bbox, bitmap vs hashed cell index, counting vs key sort, the
// number of key-sort passes, and the status (non-finite input, grid range).  The same double
// operations as sub_coord(); the host takes no part, so the whole call can be enqueued (and
// captured in a CUDA graph) without a round trip.
__device__ __forceinline__ int ceil_log2_dev(long long v) { return v <= 1 ? 0 : 64 - __clzll(v - 1); }

__device__ void plan_grid(const PlanArgs& a, const float bb[6], int nonfinite, unsigned long long near_pairs,
                          Meta* __restrict__ meta, Grid* __restrict__ gout) {
    Grid g = a.g0;
    int status = 0;
    long long cells = 1;
    for (int k = 0; k < 3; ++k) {
        g.lo[k] = (double)bb[k];
        const double smax = floor(__dmul_rn(__dadd_rn((double)bb[3 + k], -g.lo[k]), g.inv_h));
        if (!(smax < 2097152.0)) {  // >= 2^20 cells on this axis (or NaN extent)
            status = -3;             // FEC_ERR_GRID_RANGE
            g.dims[k] = 1;
        } else {
            g.dims[k] = (int32_t)(((long long)smax >> 1) + 1);
        }
        cells *= g.dims[k];
    }
    if (nonfinite) status = -2;  // FEC_ERR_NONFINITE
    g.status = status;
    g.cells_total = cells;
    g.hashed = (a.grid_mode == 1 || cells > a.dense_cap || cells >= 0xfffffff0ll) ? 1 : 0;
    if (!g.hashed) {
        // smallest dimension fastest in the linear cell id (L2 locality of the slow axis)
        int perm[3] = {0, 1, 2};
        for (int i = 0; i < 3; ++i)
            for (int j = i + 1; j < 3; ++j)
                if (g.dims[perm[j]] < g.dims[perm[i]]) { const int t = perm[i]; perm[i] = perm[j]; perm[j] = t; }
        for (int i = 0; i < 3; ++i) g.perm[i] = perm[i];
        g.stride[perm[0]] = 1;
        g.stride[perm[1]] = (uint32_t)g.dims[perm[0]];
        g.stride[perm[2]] = (uint32_t)g.dims[perm[0]] * (uint32_t)g.dims[perm[1]];
        g.sdiv[0] = g.stride[perm[2]];
        g.sdiv[1] = g.stride[perm[1]];
        g.words = (cells + 31) / 32;
        g.key_bits = max(1, ceil_log2_dev(cells));
        g.passes = (g.key_bits + 7) / 8;
    } else {
        g.words = ((long long)g.hmask + 1) / 32;
        g.key_bits = 0;
        g.passes = 0;
    }
    // input order: spatially coherent (LiDAR scan order) -> counting sort; shuffled -> key sort
    const double pairs = 3.0 * (double)(a.n / 4);
    const bool coherent = a.vec4 && (double)near_pairs >= 0.5 * pairs;
    g.key_sort = (!g.hashed && a.key_path && (a.grid_mode == 2 || (a.grid_mode != 3 && !coherent))) ? 1 : 0;
    if (!g.key_sort) g.passes = 0;
    *gout = g;
    for (int k = 0; k < 6; ++k) meta->bbox[k] = bb[k];
    meta->status = status;
    meta->instrument = a.instrument;
    if (a.status_dev) *a.status_dev = status;
}

// a1: isfinite over all 3n floats, per-axis min/max, and the number of consecutive input
// pairs (i, i+1) within `near` on every axis (spatial coherence of the input order: decides
// between the counting sort and the key sort).  Each block writes its
// partial bbox; the last block to finish (atomic ticket) reduces them and plans the grid.
__global__ void __launch_bounds__(256) k_bbox(const float* __restrict__ p, PlanArgs a, float* __restrict__ part,
                                             Meta* __restrict__ meta, Grid* __restrict__ gout) {
    pdl_prologue();
    const int64_t n = a.n;
    float mn[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    int bad = 0;
    unsigned nearc = 0;
    const float near = a.near;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t tail_start = 0;
    if (a.vec4) {
        // 4 points = 12 floats = 3 float4 per quad; the pointer is 16-byte aligned
        const float4* q = reinterpret_cast<const float4*>(p);
        const int64_t nq = n >> 2;
        // two quads (96 bytes) in flight per thread and iteration
        for (int64_t i = t0; i < nq; i += 2 * stride) {
            const bool two = i + stride < nq;
            float4 u[2], v4[2], w4[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t ii = h ? (two ? i + stride : i) : i;
                u[h] = __ldg(q + 3 * ii);
                v4[h] = __ldg(q + 3 * ii + 1);
                w4[h] = __ldg(q + 3 * ii + 2);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (h && !two) break;
                float v[12] = {u[h].x, u[h].y, u[h].z, u[h].w, v4[h].x, v4[h].y, v4[h].z, v4[h].w,
                               w4[h].x, w4[h].y, w4[h].z, w4[h].w};
#pragma unroll
                for (int k = 0; k < 12; ++k) bb_acc(v[k], mn[k % 3], mx[k % 3], bad);
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    nearc += fabsf(v[3 * j + 3] - v[3 * j]) <= near && fabsf(v[3 * j + 4] - v[3 * j + 1]) <= near &&
                             fabsf(v[3 * j + 5] - v[3 * j + 2]) <= near;
            }
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
    if ((threadIdx.x & 31) == 0 && nearc) atomicAdd(&meta->near_pairs, (unsigned long long)nearc);
    __shared__ float s[8][6];
    __shared__ int last;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) { s[w][k] = mn[k]; s[w][3 + k] = mx[k]; }
        if (bad) atomicOr(&meta->nonfinite, 1);
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        float v = s[0][threadIdx.x];
        for (int ww = 1; ww < (int)(blockDim.x >> 5); ++ww)
            v = threadIdx.x < 3 ? fminf(v, s[ww][threadIdx.x]) : fmaxf(v, s[ww][threadIdx.x]);
        part[blockIdx.x * 6 + threadIdx.x] = v;
    }
    // every thread's partial writes and atomics are ordered before the block's ticket
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&meta->ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // last block: reduce the partials (L2 reads: written by other blocks of this kernel)
    for (int k = 0; k < 3; ++k) { mn[k] = FLT_MAX; mx[k] = -FLT_MAX; }
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            mn[k] = fminf(mn[k], __ldcg(part + b * 6 + k));
            mx[k] = fmaxf(mx[k], __ldcg(part + b * 6 + 3 + k));
        }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[k] = fminf(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], o));
            mx[k] = fmaxf(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], o));
        }
    }
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) { s[w][k] = mn[k]; s[w][3 + k] = mx[k]; }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float bb[6];
        for (int k = 0; k < 6; ++k) {
            float v = s[0][k];
            for (int ww = 1; ww < (int)(blockDim.x >> 5); ++ww) v = k < 3 ? fminf(v, s[ww][k]) : fmaxf(v, s[ww][k]);
            bb[k] = v;
        }
        const int nf = *reinterpret_cast<volatile int*>(&meta->nonfinite);
        const unsigned long long np = *reinterpret_cast<volatile unsigned long long*>(&meta->near_pairs);
        plan_grid(a, bb, nf, np, meta, gout);
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
// =====================================================================================
// a8  K6: flatten   a9  K7: component stats   a10  K8: filter + relabel + scatter
// =====================================================================================
// Read-only root walk, then one store per element.  (A compressing find here would let a
// thread's late path-halving store overwrite another thread's final root with a stale
// intermediate; each parent[s] must be written only by its own thread.)
// Also initialises the accumulators of root points (component nodes get theirs in k_dcomps).
__global__ void __launch_bounds__(256) k_flatten(int* __restrict__ parent, int64_t n, int* __restrict__ size,
                                                int* __restrict__ minidx, const Meta* __restrict__ meta) {
    pdl_prologue();
    if (meta->status) return;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        int curr = ld_parent(parent, (int)s), next;
        if (curr == (int)s) {
            size[s] = 0;
            minidx[s] = 0x7fffffff;
            continue;
        }
        while (uf_above(next = ld_parent(parent, curr), curr)) curr = next;
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
                                              Meta* __restrict__ meta, int only_sparse, int bid, int nblk,
                                              bool count_sizes) {
    if (only_sparse && 4 * (int64_t)meta->cells <= n) return;
    __shared__ int hkey[HH_SLOTS], hcnt[HH_SLOTS], hmin[HH_SLOTS];
    for (int k = threadIdx.x; k < HH_SLOTS; k += blockDim.x) { hkey[k] = -1; hcnt[k] = 0; hmin[k] = 0x7fffffff; }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned long long roots = 0;
    // each thread takes 4 consecutive positions per round (int4 loads: 4 loads in flight); the
    // lanes of one distinct root meet in one __match_any_sync per position slot, and their
    // leader adds the group's count and minimum once: into the block's table if the root owns
    // its slot (the giant component claims one early), else straight to the root
    const int64_t chunk = ((n + nblk - 1) / nblk + 1023) / 1024 * 1024;
    const int64_t b0 = (int64_t)bid * chunk, b1 = min(n, b0 + chunk);
    const bool vec = ((reinterpret_cast<uintptr_t>(parent) | reinterpret_cast<uintptr_t>(val)) & 15u) == 0;
    for (int64_t s0 = b0; s0 < b1; s0 += 4 * (int64_t)blockDim.x) {
        const int64_t sb = s0 + 4 * (int64_t)threadIdx.x;
        int r[4], v[4];
        if (vec && sb + 4 <= b1) {
            const int4 pr = __ldg(reinterpret_cast<const int4*>(parent + sb));
            const int4 vv = __ldg(reinterpret_cast<const int4*>(val + sb));
            r[0] = pr.x; r[1] = pr.y; r[2] = pr.z; r[3] = pr.w;
            v[0] = vv.x; v[1] = vv.y; v[2] = vv.z; v[3] = vv.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                r[j] = sb + j < b1 ? __ldg(parent + sb + j) : -1;
                v[j] = sb + j < b1 ? __ldg(val + sb + j) : 0x7fffffff;
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int key = r[j];
            roots += (key >= 0 && key == (int)(sb + j)) ? 1ull : 0ull;
            const unsigned peers = __match_any_sync(0xffffffffu, key);
            const int mn = __reduce_min_sync(peers, v[j]);
            if (key >= 0 && lane == __ffs(peers) - 1) {
                const int cnt = __popc(peers);
                const unsigned h = ((unsigned)key * 2654435761u) >> 24;  // 256 slots
                int cur = hkey[h];
                if (cur == -1) cur = atomicCAS(&hkey[h], -1, key);
                if (cur == -1 || cur == key) {
                    if (count_sizes) atomicAdd(&hcnt[h], cnt);
                    atomicMin(&hmin[h], mn);
                } else {
                    if (count_sizes) atomicAdd(size + key, cnt);
                    atomicMin(minidx + key, mn);
                }
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
// Sparse-dominated clouds (many small components, deep forests: occupied cells > n/4)
// flatten in a separate pass first; k_tail_stats's walks are then one load each.
__global__ void __launch_bounds__(256) k_flatten_if(int* __restrict__ parent, int64_t n, const Meta* __restrict__ meta) {
    pdl_prologue();
    if (meta->status || 4 * (int64_t)meta->cells <= n) return;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        int curr = ld_parent(parent, (int)s), next;
        if (curr == (int)s) continue;
        while (uf_above(next = ld_parent(parent, curr), curr)) curr = next;
        st_parent(parent, (int)s, curr);
    }
}

// ---- single-GPU tail, one launch for the stats of every mode ----------------------------
__device__ __forceinline__ void node_stats_body(int* __restrict__ parent, const int* __restrict__ ncomp,
                                                   int* __restrict__ size, int* __restrict__ minidx, int nbase,
                                                   Meta* __restrict__ meta, int64_t n, int bid, int nblk,
                                                   uint32_t rmask) {
    if (4 * (int64_t)meta->cells > n) return;
    const int64_t nn = 8 * (int64_t)meta->ndense;
    const int64_t nr = (nn + 31) & ~int64_t(31);  // whole warps stay in the loop
    const int lane = threadIdx.x & 31;
    for (int64_t t = (int64_t)bid * blockDim.x + threadIdx.x; t < nr; t += (int64_t)nblk * blockDim.x) {
        int root = -1, c = 0, m = 0x7fffffff;
        if (t < nn && (int)(t & 7) < __ldg(ncomp + (t >> 3))) {  // a used component slot
            const int node = node_of(nbase, rmask, (int)(t >> 3), (int)(t & 7));
            int curr = ld_parent(parent, node), next;
            if (curr == node) {  // a root keeps its own totals
                if (meta->instrument) atomicAdd(&meta->components, 1ull);
            } else {
                while (uf_above(next = ld_parent(parent, curr), curr)) curr = next;
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
                                                     const int* __restrict__ slist, const float4* __restrict__ spts,
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
                    while (uf_above(next = ld_parent(parent, curr), curr)) curr = next;
                    st_parent(parent, s, curr);
                } else if (meta->instrument) {
                    atomicAdd(&meta->components, 1ull);
                }
                v = __float_as_int(__ldg(spts + s).w);
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

// The component statistics of the single-GPU tail in one launch (the variant is a device-side
// choice): sparse-dominated clouds (occupied cells > n/4) -> stats_body over the flattened
// forest; otherwise the node tail (first half of the blocks: component nodes, second half:
// points of sparse cells; independent: they only add into roots).
__global__ void __launch_bounds__(256) k_tail_stats(int* __restrict__ parent, const int* __restrict__ val, int64_t n,
                                                   int* __restrict__ size, int* __restrict__ minidx,
                                                   Meta* __restrict__ meta, const int* __restrict__ ncomp,
                                                   const uint32_t* __restrict__ cstart, const int* __restrict__ slist,
                                                   uint32_t rmask, const float4* __restrict__ spts, int count_sizes) {
    pdl_prologue();
    if (meta->status) return;
    if (4 * (int64_t)meta->cells > n) {
        // (count_sizes == 0: the size filter keeps every size -- min <= 1, max >= n -- and the
        // bucketed relabel reads no size, so only the minimum index is reduced)
        stats_body(parent, val, n, size, minidx, meta, 1, blockIdx.x, gridDim.x, count_sizes != 0);
    } else {
        const int half = (int)(gridDim.x >> 1);  // >= 1: the host launches >= 2 blocks
        if ((int)blockIdx.x < half)
            node_stats_body(parent, ncomp, size, minidx, (int)n, meta, n, blockIdx.x, half, rmask);
        else
            sparse_stats_body(parent, cstart, slist, spts, size, minidx, meta, n, blockIdx.x - half, gridDim.x - half);
    }
}

// a10 for large sparse-dominated clouds, in two passes.  k_relabel's label stores go to random
// input positions (shuffled input): each 4-byte store dirties a whole 32-byte sector and the
// sectors leave L2 long before their neighbours arrive (C5: 3.4 GB written for 0.44 GB of
// labels), and the store stream evicts the roots' labels the loads need.  Pass 1 computes the
// labels in sorted order (coalesced reads, roots nearby) and writes (input index, label) pairs
// bucket-major into a temporary: bucket b = input index >> RL_SHIFT owns the temporary's range
// [b << RL_SHIFT, ...) -- the sorted positions are a permutation of the input indices, so a
// bucket holds exactly as many pairs as its index range -- and a block reserves one run per
// bucket and tile (one global atomic each).  Pass 2 streams the temporary in order: the blocks
// in flight write into one or two buckets' 1 MB label ranges, which stay in L2 until their
// sectors are complete.
// (A separate launch, enqueued only for clouds of >= 2^22 points: folded into k_rootlab its
// shared tables and registers slowed that kernel on node-tail clouds, C4 25 -> 42 us.)
__global__ void __launch_bounds__(256) k_relabel_b1(const int* __restrict__ parent, const int* __restrict__ val,
                                                   const int* __restrict__ size, const int* __restrict__ minidx,
                                                   int64_t n, long long min_size, long long max_size,
                                                   uint2* __restrict__ tmp, unsigned int* __restrict__ cursor,
                                                   const Meta* __restrict__ meta, const Grid* __restrict__ gp) {
    pdl_prologue();
    if (meta->status || 4 * (int64_t)meta->cells <= n) return;
    const int64_t* __restrict__ boff = gp->batch ? gp->boff : nullptr;
    const int nclouds = gp->nclouds;
    constexpr int sh = RL_SHIFT;
    // block k owns the tiles k, k + G, ... (G = the grid, one resident wave: the tiles in
    // flight are a narrow window of the sorted order, so the roots' labels stay in L2).  Pass A
    // counts the block's pairs per bucket and reserves one run per bucket (G atomics per
    // cursor; tile-wise reservations serialised ~50k on each cursor's L2 slice), pass B
    // re-reads the tiles and writes the pairs.
    __shared__ unsigned int base[RL_MAX_BUCKETS], cnt[RL_MAX_BUCKETS];
    const int nb = (int)((n + (int64_t(1) << sh) - 1) >> sh);
    const int64_t stride = (int64_t)gridDim.x * RL_TILE;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) cnt[b] = 0u;
    __syncthreads();
    constexpr int PER = RL_TILE / 256;
    for (int64_t t0 = (int64_t)blockIdx.x * RL_TILE; t0 < n; t0 += stride) {
        int v[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {  // all loads in flight before the counts
            const int64_t s = t0 + j * 256 + threadIdx.x;
            v[j] = s < n ? __ldg(val + s) : -1;
        }
#pragma unroll
        for (int j = 0; j < PER; ++j)
            if (v[j] >= 0) atomicAdd(&cnt[v[j] >> sh], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        const unsigned int c = cnt[b];
        base[b] = c ? ((unsigned)b << sh) + atomicAdd(cursor + b * RL_CUR_STRIDE, c) : 0u;
    }
    // the size filter applied here (k_rootlab returns at once for these clouds); a filter that keeps every
    // size (min <= 1, max >= n) reads no size
    const bool filt = min_size > 1 || max_size < n;
    for (int64_t t0 = (int64_t)blockIdx.x * RL_TILE; t0 < n; t0 += stride) {
        for (int b = threadIdx.x; b < nb; b += blockDim.x) cnt[b] = 0u;
        __syncthreads();
        int v[PER], lab[PER];
        unsigned int rank[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int64_t s = t0 + j * 256 + threadIdx.x;
            v[j] = -1;
            if (s < n) {
                v[j] = __ldg(val + s);
                const int r = __ldg(parent + s);  // the root (flattened by k_flatten_if)
                int l = __ldg(minidx + r);
                if (filt) {
                    const long long sz = __ldg(size + r);
                    if (sz < min_size || sz > max_size) l = -1;
                }
                if (boff && l >= 0) {  // batch mode: index inside the point's own cloud
                    int lo = 0, hi = nclouds;
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (__ldg(boff + mid) <= (int64_t)v[j]) lo = mid;
                        else hi = mid;
                    }
                    l -= (int)__ldg(boff + lo);
                }
                lab[j] = l;
                rank[j] = atomicAdd(&cnt[v[j] >> sh], 1u);
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < PER; ++j)
            if (v[j] >= 0) tmp[base[v[j] >> sh] + rank[j]] = make_uint2((unsigned)v[j], (unsigned)lab[j]);
        __syncthreads();
        for (int b = threadIdx.x; b < nb; b += blockDim.x) base[b] += cnt[b];
    }
}

// a10, first half: the size filter folded into the union-find nodes, so k_relabel reads one
// word per point.  Every root (parent[x] == x) gets minidx[x] = its component's final label
// (the minimum input index, or -1 outside [min_size, max_size]); every component node that is
// not a root gets its root's final label (its own partial minimum is no longer needed: the
// statistics are complete).  The nodes visited: all points and node slots of sparse-dominated
// clouds; otherwise the node slots and the points of sparse cells (the compact list), since a
// point of a dense cell hangs under a component node.  A node that reads its root while the
// root's own thread folds it sees either the minimum or the folded label, which agree unless
// the size is filtered -- and then both sides write -1.
// Node-tail clouds: a single-component dense cell's record word (crec, >= 0) is replaced by its
// final label encoded as -(label + 3) (<= -2; -1 stays "sparse cell"), so k_relabel_in needs one
// lookup per point of such a cell.
__global__ void __launch_bounds__(256) k_rootlab(const int* __restrict__ parent, const int* __restrict__ size,
                                                int* __restrict__ minidx, int64_t n, long long min_size,
                                                long long max_size, const Meta* __restrict__ meta, uint32_t rmask,
                                                const uint32_t* __restrict__ cstart, const int* __restrict__ slist,
                                                const int* __restrict__ ncomp, const int* __restrict__ dlist,
                                                int* __restrict__ crec, int bucketed) {
    pdl_prologue();
    if (meta->status) return;
    const bool sparse_dom = 4 * (int64_t)meta->cells > n;
    if (sparse_dom && bucketed) return;  // (large sparse-dominated clouds: k_relabel_b1)
    const int64_t nslot = 8 * (int64_t)meta->ndense;
    const int64_t npts = sparse_dom ? n : (int64_t)meta->nsparse * SPARSE_MAX;  // points, or sparse-cell slots
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < npts + nslot;
         u += (int64_t)gridDim.x * blockDim.x) {
        int64_t x;
        if (u < npts) {
            if (sparse_dom) {
                x = u;
            } else {  // slot j of sparse cell e
                const int e = (int)(u / SPARSE_MAX), j = (int)(u % SPARSE_MAX);
                const int P = __ldg(slist + e);
                const int s0 = (int)__ldg(cstart + P);
                if (s0 + j >= (int)__ldg(cstart + P + 1)) continue;
                x = s0 + j;
            }
        } else {
            x = node_of((int)n, rmask, (int)((u - npts) >> 3), (int)((u - npts) & 7));
        }
        const int p = __ldg(parent + x);
        int lab = 0;
        if (p == (int)x) {
            const long long sz = __ldg(size + x);
            lab = (sz >= min_size && sz <= max_size) ? minidx[x] : -1;
            if (lab < 0) minidx[x] = -1;
        } else if (x >= n) {  // a component node under another root (flattened by the tail)
            const long long sz = __ldg(size + p);
            lab = (sz >= min_size && sz <= max_size) ? minidx[p] : -1;
            minidx[x] = lab;
        }
        if (!sparse_dom && u >= npts && ((u - npts) & 7) == 0) {  // component 0 of record r
            const int r = (int)((u - npts) >> 3);
            if (__ldg(ncomp + r) == 1) crec[__ldg(dlist + r)] = -(lab + 3);
        }
    }
}

// a10, second half: labels[input index] = the folded label of the point's parent (its root, or
// for a point of a dense cell its component node), scattered back to input order.
__global__ void __launch_bounds__(256) k_relabel(const int* __restrict__ parent, const int* __restrict__ val,
                                                const int* __restrict__ minidx, int64_t n,
                                                int* __restrict__ labels, const Meta* __restrict__ meta,
                                                const int64_t* __restrict__ boff, int nclouds) {
    pdl_prologue();
    // (a1 rejected the input: labels_out is left untouched; node-tail clouds: k_relabel_in)
    if (meta->status || 4 * (int64_t)meta->cells <= n) return;
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
        int lab[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) lab[j] = r[j] >= 0 ? __ldg(minidx + r[j]) : -1;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (r[j] < 0) continue;
            int l = lab[j];
            if (boff && l >= 0) {
                // batch mode: index inside the point's own cloud (the component never spans two)
                int lo = 0, hi = nclouds;
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (__ldg(boff + mid) <= (int64_t)v[j]) lo = mid;
                    else hi = mid;
                }
                l -= (int)__ldg(boff + lo);
            }
            labels[v[j]] = l;
        }
    }
}

// Staged form: a cluster of RL_CLUSTER CTAs per bucket holds the bucket's 1 MB label range in
// its distributed shared memory (CTA r: labels [r * 2^15, (r + 1) * 2^15) of the bucket); every
// CTA streams an eighth of the bucket's pairs and stores each label into the owning CTA's
// shared memory, then each CTA writes its 128 KB slice out coalesced -- no partial sector ever
// reaches L2.  (Every index of a bucket occurs exactly once: the sorted positions are a
// permutation of the input indices.)
__global__ void __cluster_dims__(RL_CLUSTER, 1, 1) __launch_bounds__(1024)
    k_relabel_b2c(const uint2* __restrict__ tmp, int64_t n, int* __restrict__ labels, const Meta* __restrict__ meta) {
    pdl_prologue();
    if (meta->status || 4 * (int64_t)meta->cells <= n) return;  // (uniform over the cluster)
    extern __shared__ int stage[];
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    constexpr int B = 1 << RL_SHIFT, S = 1 << RL_CTA_SHIFT;
    const int64_t nb = (n + B - 1) / B;
    const int64_t ncl = gridDim.x / RL_CLUSTER;
    for (int64_t b = blockIdx.x / RL_CLUSTER; b < nb; b += ncl) {
        const int64_t e0 = b * B;
        const int cnt = (int)min((int64_t)B, n - e0);
        const int per = (cnt + RL_CLUSTER - 1) / RL_CLUSTER;
        const int i0 = min(cnt, rank * per), i1 = min(cnt, i0 + per);
        // 8 pairs in flight per thread (the remote stores are fire-and-forget)
        constexpr int U = 8;
        for (int i = i0 + threadIdx.x; i < i1; i += U * blockDim.x) {
            uint2 e[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = i + u * blockDim.x;
                e[u] = k < i1 ? __ldcs(tmp + e0 + k) : make_uint2(0xffffffffu, 0u);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (e[u].x == 0xffffffffu) continue;
                const int loc = (int)(e[u].x - (unsigned)e0);
                int* dst = cluster.map_shared_rank(stage, loc >> RL_CTA_SHIFT);
                dst[loc & (S - 1)] = (int)e[u].y;
            }
        }
        cluster.sync();
        const int o0 = rank * S, oc = max(0, min(S, cnt - o0));
        if ((reinterpret_cast<uintptr_t>(labels) & 15u) == 0) {
            int4* out4 = reinterpret_cast<int4*>(labels + e0 + o0);  // (e0 + o0: a multiple of 4)
            for (int i = threadIdx.x; i < oc / 4; i += blockDim.x)
                out4[i] = make_int4(stage[4 * i], stage[4 * i + 1], stage[4 * i + 2], stage[4 * i + 3]);
            for (int i = (oc / 4) * 4 + threadIdx.x; i < oc; i += blockDim.x) labels[e0 + o0 + i] = stage[i];
        } else {
            for (int i = threadIdx.x; i < oc; i += blockDim.x) labels[e0 + o0 + i] = stage[i];
        }
        cluster.sync();  // (the next bucket's stores into this CTA wait for its slice to be out)
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
