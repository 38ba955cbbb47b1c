// Dense-grid path (the default whenever the bbox holds <= 4n + 2^22 cells): the points are
// counting-sorted by cell into a dense row-major cell table, cells holding more than
// SPARSE_MAX points are re-ordered by octant (sub-cell cliques), then
//   * sparse cells: one thread per point tests every candidate directly,
//   * dense cells:  one warp per cell evaluates sub-cell group pairs (fec_pairs.cuh).
// DESIGN.md §4 describes the responsibilities that make every adjacent cell pair examined
// exactly once.
#include "fec_internal.cuh"
#include "fec_kernels.cuh"
#include "fec_pairs.cuh"

namespace fec {

__device__ __forceinline__ void dense_cell_of(float x, float y, float z, const Grid& g, uint32_t& lin, int& oct) {
    const uint32_t sx = sub_coord(x, g.lo[0], g.inv_h);
    const uint32_t sy = sub_coord(y, g.lo[1], g.inv_h);
    const uint32_t sz = sub_coord(z, g.lo[2], g.inv_h);
    oct = (int)((sx & 1u) | ((sy & 1u) << 1) | ((sz & 1u) << 2));
    lin = (sx >> 1) * g.stride[0] + (sy >> 1) * g.stride[1] + (sz >> 1) * g.stride[2];
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

// ---- a2: per-cell counts; slot[i] = rank of point i inside its cell -----------------------
__global__ void __launch_bounds__(256) k_dcount(const float* __restrict__ p, int64_t n, Grid g,
                                               uint32_t* __restrict__ count, uint32_t* __restrict__ slot,
                                               int* __restrict__ dlist, Meta* __restrict__ meta) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
        const int64_t i = i0 + threadIdx.x;
        const bool ok = i < n;
        uint32_t lin = 0xffffffffu;
        int oct;
        if (ok) dense_cell_of(__ldg(p + 3 * i), __ldg(p + 3 * i + 1), __ldg(p + 3 * i + 2), g, lin, oct);
        // warp-aggregated atomics: one atomicAdd per distinct cell in the warp
        const unsigned peers = __match_any_sync(0xffffffffu, lin);
        const int leader = __ffs(peers) - 1;
        const uint32_t cnt = __popc(peers);
        uint32_t old = 0;
        if (ok && lane == leader) {
            old = atomicAdd(count + lin, cnt);
            if (old <= (uint32_t)SPARSE_MAX && old + cnt > (uint32_t)SPARSE_MAX)
                dlist[atomicAdd(&meta->ndense, 1)] = (int)lin;
            if (old == 0 && meta->instrument) atomicAdd(&meta->cells, 1);
        }
        old = __shfl_sync(0xffffffffu, old, leader);
        if (ok) slot[i] = old + __popc(peers & lt);
    }
}

// ---- a3: scatter into cell order (after the exclusive scan of count -> cstart) ------------
// Only the float4 (x, y, z, idx) is scattered: for shuffled inputs every scattered array
// costs a DRAM read-modify-write per point, so everything else is derived in sorted order.
__global__ void __launch_bounds__(256) k_dscatter(const float* __restrict__ p, int64_t n, Grid g,
                                                 const uint32_t* __restrict__ cstart, const uint32_t* __restrict__ slot,
                                                 float4* __restrict__ spts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float x = __ldg(p + 3 * i), y = __ldg(p + 3 * i + 1), z = __ldg(p + 3 * i + 2);
        uint32_t lin;
        int oct;
        dense_cell_of(x, y, z, g, lin, oct);
        const uint32_t pos = __ldg(cstart + lin) + __ldg(slot + i);
        spts[pos] = make_float4(x, y, z, __int_as_float((int)i));
    }
}

// Sorted-order initialisation (coalesced): singleton sets, accumulators, input index.
__global__ void __launch_bounds__(256) k_dinit(const float4* __restrict__ spts, int64_t n, int* __restrict__ parent,
                                              int* __restrict__ size, int* __restrict__ minidx,
                                              int* __restrict__ sidx) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        parent[s] = (int)s;
        size[s] = 0;
        minidx[s] = 0x7fffffff;
        sidx[s] = __float_as_int(__ldg(&spts[s].w));
    }
}

// ---- a4: dense cells -> octant order, group records, group-leader parents ------------------
constexpr int FIX_THREADS = 256;
constexpr int FIX_CAP = 2048;  // points staged in shared memory (40 KB); larger cells stage in global

__global__ void __launch_bounds__(FIX_THREADS) k_dfixup(const uint32_t* __restrict__ cstart,
                                                       const int* __restrict__ dlist, Meta* __restrict__ meta, Grid g,
                                                       float4* __restrict__ spts, int* __restrict__ sidx,
                                                       int* __restrict__ parent, DenseRec* __restrict__ drec,
                                                       int* __restrict__ crec, float4* __restrict__ tmp_pts) {
    __shared__ float4 sp[FIX_CAP];
    __shared__ int cnt[8], off[9], cur[8];
    const int nd = meta->ndense;
    for (int r = blockIdx.x; r < nd; r += gridDim.x) {
        const int cell = dlist[r];
        const int start = (int)cstart[cell], end = (int)cstart[cell + 1];
        const int m = end - start;
        if (threadIdx.x < 8) cnt[threadIdx.x] = 0;
        __syncthreads();
        const bool in_smem = m <= FIX_CAP;
        // octants from the coordinates (same arithmetic as the binning kernels)
        for (int q = threadIdx.x; q < m; q += FIX_THREADS) {
            const float4 v = spts[start + q];
            uint32_t lin;
            int o;
            dense_cell_of(v.x, v.y, v.z, g, lin, o);
            atomicAdd(&cnt[o], 1);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int run = 0;
            for (int k = 0; k < 8; ++k) { off[k] = run; cur[k] = run; run += cnt[k]; }
            off[8] = run;
            DenseRec R;
            R.cell = cell;
            for (int k = 0; k < 9; ++k) R.off[k] = start + off[k];
            drec[r] = R;
            crec[cell] = r;
            atomicAdd(&meta->dense_points, (unsigned long long)m);
        }
        __syncthreads();
        for (int q = threadIdx.x; q < m; q += FIX_THREADS) {
            const float4 v = spts[start + q];
            uint32_t lin;
            int o;
            dense_cell_of(v.x, v.y, v.z, g, lin, o);
            const int d = atomicAdd(&cur[o], 1);
            if (in_smem) sp[d] = v;
            else tmp_pts[start + d] = v;
        }
        __syncthreads();
        for (int q = threadIdx.x; q < m; q += FIX_THREADS) {
            int k = 0;
            while (q >= off[k + 1]) ++k;
            const float4 v = in_smem ? sp[q] : tmp_pts[start + q];
            spts[start + q] = v;
            sidx[start + q] = __float_as_int(v.w);
            parent[start + q] = start + off[k + 1] - 1;   // leader = last point of the octant group
        }
        __syncthreads();
    }
}

// ---- a6+a7: one fused sweep over the grid cells ------------------------------------------
// Thread per linear cell; a warp covers 32 consecutive cells, so the cell-table reads of a
// neighbour offset are coalesced, and blocks run in launch order, sweeping the sorted order
// upwards (roots of the union-find sit near the sweep front).
//   sparse cell P (1..SPARSE_MAX points): its lane tests every pair (s, t) with t in P
//       (t > s) or in a SPARSE forward neighbour Q;
//   dense cell P: the whole warp evaluates sub-cell group pairs of P with itself, with every
//       forward neighbour (dense: octant groups; sparse: single points) and with every
//       SPARSE backward neighbour.
// So each unordered pair of adjacent cells is examined exactly once.
__device__ __forceinline__ void dense_cell_work(int r, PairSmem& S, const float4* __restrict__ spts,
                                                const uint32_t* __restrict__ cstart,
                                                const DenseRec* __restrict__ drec, const int* __restrict__ crec,
                                                const Grid& g, int* __restrict__ parent, int lane,
                                                unsigned long long& n_tests, unsigned long long& n_pairs) {
    const float t2 = g.t2;
    const DenseRec* R = drec + r;
    int np = 0;
    {
        const int k = lane < 8 ? lane : 7;
        const int o0 = __ldg(&R->off[k]), o1 = __ldg(&R->off[k + 1]);
        const bool ne = lane < 8 && o1 > o0;
        const unsigned m = __ballot_sync(0xffffffffu, ne);
        if (ne) {
            const int j = __popc(m & ((1u << lane) - 1u));
            S.ps[j] = o0;
            S.po[j] = (uint8_t)k;
        }
        np = __popc(m);
        if (lane == 0) S.ps[np] = __ldg(&R->off[8]);
    }
    int c[3];
    dense_decode((uint32_t)__ldg(&R->cell), g, c);
    // neighbour table: lanes 0..12 forward, 13..25 backward
    int qstart = 0, qend = 0;
    if (lane < 26) {
        const int k = lane < 13 ? lane : lane - 13;
        const int sg = lane < 13 ? 1 : -1;
        uint32_t Q;
        if (dense_neighbor(g, c, sg * c_fwd[k][0], sg * c_fwd[k][1], sg * c_fwd[k][2], Q)) {
            qstart = (int)__ldg(cstart + Q);
            qend = (int)__ldg(cstart + Q + 1);
            if (qend - qstart > SPARSE_MAX) {
                if (lane >= 13) qend = qstart;       // dense backward: handled by that cell
                else qstart = -1 - __ldg(crec + Q);  // dense forward: encode record id
            }
        }
    }
    __syncwarp();
    for (int k = -1; k < 26; ++k) {
        int nq;
        const bool same = k < 0;
        if (same) {
            nq = np;
            if (lane <= np) S.qs[lane] = S.ps[lane];
            if (lane < np) S.qo[lane] = S.po[lane];
        } else {
            const int qs = __shfl_sync(0xffffffffu, qstart, k);
            const int qe = __shfl_sync(0xffffffffu, qend, k);
            if (qs >= 0 && qe <= qs) continue;
            if (qs < 0) {  // dense forward neighbour: its octant groups
                const DenseRec* RQ = drec + (-1 - qs);
                const int kk = lane < 8 ? lane : 7;
                const int o0 = __ldg(&RQ->off[kk]), o1 = __ldg(&RQ->off[kk + 1]);
                const bool ne = lane < 8 && o1 > o0;
                const unsigned m = __ballot_sync(0xffffffffu, ne);
                if (ne) {
                    const int j = __popc(m & ((1u << lane) - 1u));
                    S.qs[j] = o0;
                    S.qo[j] = (uint8_t)kk;
                }
                nq = __popc(m);
                if (lane == 0) S.qs[nq] = __ldg(&RQ->off[8]);
            } else {       // sparse neighbour: every point is its own group
                nq = qe - qs;
                if (lane <= nq) S.qs[lane] = qs + lane;
                if (lane < nq) S.qo[lane] = 0xFF;
            }
        }
        __syncwarp();
        const int kk = k < 13 ? k : k - 13;
        const int sg = k < 13 ? 1 : -1;
        const int nqueue = same ? build_queue(S, np, nq, true, 0, 0, 0, lane)
                                : build_queue(S, np, nq, false, sg * c_fwd[kk][0], sg * c_fwd[kk][1],
                                              sg * c_fwd[kk][2], lane);
        n_pairs += (lane == 0) ? (unsigned long long)nqueue : 0ull;
        load_roots(S, np, nq, parent, lane);
        process_queue(S, nqueue, spts, parent, t2, lane, n_tests);
    }
}

__global__ void __launch_bounds__(256) k_union_sparse(const float4* __restrict__ spts,
                                                     const uint32_t* __restrict__ cstart, uint32_t cells, Grid g,
                                                     int* __restrict__ parent, Meta* __restrict__ meta) {
    const int lane = threadIdx.x & 31;
    unsigned long long n_tests = 0, n_pairs = 0;
    const float t2 = g.t2;
    const uint32_t P = blockIdx.x * blockDim.x + threadIdx.x;
    const bool ok = P < cells;
    int ps = 0, pe = 0;
    if (ok) {
        ps = (int)__ldg(cstart + P);
        pe = (int)__ldg(cstart + P + 1);
    }
    const bool sparse = ok && pe > ps && pe - ps <= SPARSE_MAX;
    if (sparse) {
        for (int s = ps; s < pe; ++s) {
            const float4 a = __ldg(spts + s);
            for (int t = s + 1; t < pe; ++t) {
                ++n_tests;
                if (pred(a, __ldg(spts + t), t2)) uf_unite(parent, s, t);
            }
        }
        int c[3];
        dense_decode(P, g, c);
#pragma unroll 1
        for (int k = 0; k < 13; ++k) {
            uint32_t Q;
            if (!dense_neighbor(g, c, c_fwd[k][0], c_fwd[k][1], c_fwd[k][2], Q)) continue;
            const int qs = (int)__ldg(cstart + Q), qe = (int)__ldg(cstart + Q + 1);
            if (qe == qs || qe - qs > SPARSE_MAX) continue;
            for (int s = ps; s < pe; ++s) {
                const float4 a = __ldg(spts + s);
                for (int t = qs; t < qe; ++t) {
                    ++n_tests;
                    if (pred(a, __ldg(spts + t), t2)) uf_unite(parent, s, t);
                }
            }
        }
    }
    if (meta->instrument) {
        for (int o = 16; o > 0; o >>= 1) {
            n_tests += __shfl_xor_sync(0xffffffffu, n_tests, o);
            n_pairs += __shfl_xor_sync(0xffffffffu, n_pairs, o);
        }
        if (lane == 0 && (n_tests || n_pairs)) {
            atomicAdd(&meta->pair_tests, n_tests);
            atomicAdd(&meta->group_pairs, n_pairs);
        }
    }
}

// Dense cells: warp per cell, dynamic scheduling over the dense records (load balance:
// a few cells hold thousands of points).
__global__ void __launch_bounds__(SCAN_THREADS) k_union_dense(const float4* __restrict__ spts,
                                                            const uint32_t* __restrict__ cstart,
                                                            const DenseRec* __restrict__ drec,
                                                            const int* __restrict__ crec, Grid g,
                                                            int* __restrict__ parent, Meta* __restrict__ meta) {
    __shared__ PairSmem sm[SCAN_THREADS / kWarp];
    const int lane = threadIdx.x & 31;
    PairSmem& S = sm[threadIdx.x >> 5];
    const int nd = meta->ndense;
    unsigned long long n_tests = 0, n_pairs = 0;
    while (true) {
        int r = 0;
        if (lane == 0) r = atomicAdd(&meta->work, 1);
        r = __shfl_sync(0xffffffffu, r, 0);
        if (r >= nd) break;
        dense_cell_work(r, S, spts, cstart, drec, crec, g, parent, lane, n_tests, n_pairs);
    }
    if (meta->instrument) {
        for (int o = 16; o > 0; o >>= 1) {
            n_tests += __shfl_xor_sync(0xffffffffu, n_tests, o);
            n_pairs += __shfl_xor_sync(0xffffffffu, n_pairs, o);
        }
        if (lane == 0 && (n_tests || n_pairs)) {
            atomicAdd(&meta->dense_tests, n_tests);
            atomicAdd(&meta->group_pairs, n_pairs);
        }
    }
}

}  // namespace fec
