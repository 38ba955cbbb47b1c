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
                                               uint32_t* __restrict__ dbits, Meta* __restrict__ meta) {
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
                atomicOr(dbits + (lin >> 5), 1u << (lin & 31u));   // the cell just became dense
            if (old == 0 && meta->instrument) atomicAdd(&meta->cells, 1);
        }
        old = __shfl_sync(0xffffffffu, old, leader);
        if (ok) slot[i] = old + __popc(peers & lt);
    }
}

// ---- a2b: dense cells get records (in ascending cell order); their points get
// octant-ordered slots.  A cell with more than SPARSE_MAX points is laid out octant by
// octant (octant k = the sub-cell (sx&1, sy&1, sz&1)), so each octant is a contiguous
// clique group.
__global__ void __launch_bounds__(256) k_dbits_popc(const uint32_t* __restrict__ dbits, int64_t words,
                                                   uint32_t* __restrict__ wcount) {
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w <= words; w += (int64_t)gridDim.x * blockDim.x)
        wcount[w] = w < words ? (uint32_t)__popc(__ldg(dbits + w)) : 0u;
}

__global__ void __launch_bounds__(256) k_dbits_list(const uint32_t* __restrict__ dbits, int64_t words,
                                                   const uint32_t* __restrict__ wpos, int* __restrict__ dlist,
                                                   int* __restrict__ crec, uint32_t* __restrict__ ocnt,
                                                   Meta* __restrict__ meta) {
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
#pragma unroll
            for (int k = 0; k < 8; ++k) ocnt[8 * r + k] = 0u;
            ++r;
        }
    }
}

__global__ void __launch_bounds__(256) k_dcount_oct(const float* __restrict__ p, int64_t n, Grid g,
                                                   const uint32_t* __restrict__ count, const int* __restrict__ crec,
                                                   uint32_t* __restrict__ ocnt, uint32_t* __restrict__ slot) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
        const int64_t i = i0 + threadIdx.x;
        uint32_t key = 0xffffffffu;
        if (i < n) {
            uint32_t lin;
            int oct;
            dense_cell_of(__ldg(p + 3 * i), __ldg(p + 3 * i + 1), __ldg(p + 3 * i + 2), g, lin, oct);
            if (__ldg(count + lin) > (uint32_t)SPARSE_MAX) key = 8u * (uint32_t)__ldg(crec + lin) + (uint32_t)oct;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (key != 0xffffffffu && lane == leader) old = atomicAdd(ocnt + key, (uint32_t)__popc(peers));
        old = __shfl_sync(0xffffffffu, old, leader);
        if (key != 0xffffffffu) slot[i] = old + __popc(peers & lt);
    }
}

// After the scan: octant offsets of every dense record.
__global__ void __launch_bounds__(256) k_drec_fin(const int* __restrict__ dlist, Meta* __restrict__ meta,
                                                 const uint32_t* __restrict__ cstart,
                                                 const uint32_t* __restrict__ ocnt, DenseRec* __restrict__ drec) {
    const int nd = meta->ndense;
    unsigned long long pts = 0;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nd; r += gridDim.x * blockDim.x) {
        const int cell = __ldg(dlist + r);
        const int start = (int)__ldg(cstart + cell), m = (int)__ldg(cstart + cell + 1) - start;
        DenseRec R;
        R.cell = cell;
        int run = start;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            R.off[k] = run;
            run += (int)__ldg(ocnt + 8 * r + k);
        }
        R.off[8] = run;
        drec[r] = R;
        pts += (unsigned long long)m;
    }
    for (int o = 16; o > 0; o >>= 1) pts += __shfl_xor_sync(0xffffffffu, pts, o);
    if ((threadIdx.x & 31) == 0 && pts) atomicAdd(&meta->dense_points, pts);
}

// ---- a3: scatter into cell order (after the exclusive scan of count -> cstart) ------------
// Only the float4 (x, y, z, idx) is scattered: for shuffled inputs every scattered array
// costs a DRAM read-modify-write per point, so everything else is derived in sorted order.
__global__ void __launch_bounds__(256) k_dscatter(const float* __restrict__ p, int64_t n, Grid g,
                                                 const uint32_t* __restrict__ cstart, const uint32_t* __restrict__ slot,
                                                 const int* __restrict__ crec, const DenseRec* __restrict__ drec,
                                                 float4* __restrict__ spts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float x = __ldg(p + 3 * i), y = __ldg(p + 3 * i + 1), z = __ldg(p + 3 * i + 2);
        uint32_t lin;
        int oct;
        dense_cell_of(x, y, z, g, lin, oct);
        const uint32_t c0 = __ldg(cstart + lin), c1 = __ldg(cstart + lin + 1);
        uint32_t base = c0;
        if (c1 - c0 > (uint32_t)SPARSE_MAX) base = (uint32_t)__ldg(&drec[__ldg(crec + lin)].off[oct]);
        spts[base + __ldg(slot + i)] = make_float4(x, y, z, __int_as_float((int)i));
    }
}

// Sorted-order initialisation (coalesced): parent = self for points of sparse cells, the
// last point of the octant group for points of dense cells (groups are cliques, DESIGN.md
// §4.5); accumulators; input index.
__global__ void __launch_bounds__(256) k_dinit(const float4* __restrict__ spts, int64_t n, Grid g,
                                              const uint32_t* __restrict__ cstart, const int* __restrict__ crec,
                                              const DenseRec* __restrict__ drec, int* __restrict__ parent,
                                              int* __restrict__ size, int* __restrict__ minidx,
                                              int* __restrict__ sidx) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const float4 v = __ldg(spts + s);
        uint32_t lin;
        int oct;
        dense_cell_of(v.x, v.y, v.z, g, lin, oct);
        const uint32_t c0 = __ldg(cstart + lin), c1 = __ldg(cstart + lin + 1);
        int par = (int)s;
        if (c1 - c0 > (uint32_t)SPARSE_MAX) par = __ldg(&drec[__ldg(crec + lin)].off[oct + 1]) - 1;
        parent[s] = par;
        size[s] = 0;
        minidx[s] = 0x7fffffff;
        sidx[s] = __float_as_int(v.w);
    }
}

// ---- a6+a7: neighbour scan + union --------------------------------------------------------
// Responsibilities (each unordered pair of adjacent cells is examined exactly once,
// DESIGN.md §4.6):
//   sparse cell P (1..SPARSE_MAX points): one lane tests every pair (s, t) with t in P
//       (t > s) or in a SPARSE forward neighbour Q                       -> k_union_sparse
//   dense cell P: one warp evaluates sub-cell group pairs of P with itself, with every
//       forward neighbour (dense: octant groups; sparse: single points) and with every
//       SPARSE backward neighbour                                         -> k_union_dense

constexpr int QG_CAP = 13 * 8 + 13 * SPARSE_MAX;  // Q groups of one dense cell (all neighbours)
constexpr int PQ_CAP = 256;                        // pair queue capacity

struct DenseSmem {
    int ps[9];                 // P octant groups: [ps[a], ps[a+1])
    uint8_t po[8];
    int proot[8];
    int qs[QG_CAP], qe[QG_CAP];  // Q groups: [qs[b], qe[b])
    uint8_t qo[QG_CAP];        // octant, or 0xFF for a single point (no octant filter)
    uint8_t qk[QG_CAP];        // neighbour slot (0..12 forward, 13..25 backward, 26 own)
    int qroot[QG_CAP];
    uint16_t small[PQ_CAP], big[PQ_CAP];  // (a << 8) | b
    int slot_q[26], slot_rec[26], slot_cnt[26], slot_off[27];
};

__device__ __forceinline__ void slot_offset(int k, int& ox, int& oy, int& oz) {
    const int kk = k < 13 ? k : k - 13;
    const int sg = k < 13 ? 1 : -1;
    ox = sg * c_fwd[kk][0];
    oy = sg * c_fwd[kk][1];
    oz = sg * c_fwd[kk][2];
}

// Small pairs one lane each, big pairs the whole warp; both stop at the first pred-true pair.
__device__ __forceinline__ void run_pairs(DenseSmem& S, int nsmall, int nbig, int nq_total,
                                          const float4* __restrict__ spts, int* parent, float t2, int lane,
                                          unsigned long long& n_tests) {
    for (int e0 = 0; e0 < nsmall; e0 += 32) {
        const int e = e0 + lane;
        if (e < nsmall) {
            const int a = S.small[e] >> 8, b = S.small[e] & 255;
            const int sa = S.ps[a], ea = S.ps[a + 1], sb = S.qs[b], eb = S.qe[b];
            bool hit = false;
            for (int i = sa; i < ea && !hit; ++i) {
                const float4 pi = __ldg(spts + i);
                for (int j = sb; j < eb; ++j) {
                    ++n_tests;
                    if (pred(pi, __ldg(spts + j), t2)) { hit = true; break; }
                }
            }
            if (hit) uf_unite(parent, sa, sb);
        }
        __syncwarp();
    }
    for (int e = 0; e < nbig; ++e) {
        const int a = S.big[e] >> 8, b = S.big[e] & 255;
        if (S.proot[a] == S.qroot[b]) continue;  // joined by an earlier big pair
        int sa = S.ps[a], ea = S.ps[a + 1], sb = S.qs[b], eb = S.qe[b];
        if (eb - sb > ea - sa) { int t = sa; sa = sb; sb = t; t = ea; ea = eb; eb = t; }
        bool found = false;
        for (int i0 = sa; i0 < ea && !found; i0 += 32) {
            const int i = i0 + lane;
            const bool vi = i < ea;
            const float4 pi = vi ? __ldg(spts + i) : make_float4(0.f, 0.f, 0.f, 0.f);
            for (int j = sb; j < eb; ++j) {
                const float4 pj = __ldg(spts + j);
                n_tests += vi ? 1ull : 0ull;
                if (__any_sync(0xffffffffu, vi && pred(pi, pj, t2))) { found = true; break; }
            }
        }
        if (found) {
            const int ra = S.proot[a], rb = S.qroot[b];
            int rn = 0;
            if (lane == 0) {
                uf_unite(parent, S.ps[a], S.qs[b]);
                rn = uf_find(parent, S.ps[a]);
            }
            rn = __shfl_sync(0xffffffffu, rn, 0);
            __syncwarp();
            // every cached root equal to either old root now maps to the merged root
            if (lane < 8 && (S.proot[lane] == ra || S.proot[lane] == rb)) S.proot[lane] = rn;
            for (int q = lane; q < nq_total; q += 32)
                if (S.qroot[q] == ra || S.qroot[q] == rb) S.qroot[q] = rn;
            __syncwarp();
        }
    }
}

// Enumerate (a, b) for a < np and b in [b0, b1), keep those whose cached roots differ and
// whose sub-cell offset can hold a pred-true pair, and run them through run_pairs in
// batches of at most PQ_CAP.  `own`: the Q groups are P's own groups (only b > a).
__device__ __forceinline__ void pair_sweep(DenseSmem& S, int np, int b0, int b1, bool own,
                                           const float4* __restrict__ spts, int* parent, float t2, int lane,
                                           unsigned long long& n_tests, unsigned long long& n_pairs) {
    const int nb = b1 - b0;
    const int total = np * nb;
    int nsmall = 0, nbig = 0;
    for (int base = 0; base < total; base += 32) {
        const int pid = base + lane;
        bool ok = pid < total;
        int a = 0, b = 0;
        bool big = false;
        if (ok) {
            b = b0 + pid / np;
            a = pid - (b - b0) * np;
            if (own) {
                ok = b > a;
            } else if (S.qo[b] != 0xFF) {
                int ox, oy, oz;
                slot_offset(S.qk[b], ox, oy, oz);
                const int oa = S.po[a], ob = S.qo[b];
                const int dx = 2 * ox + (ob & 1) - (oa & 1);
                const int dy = 2 * oy + ((ob >> 1) & 1) - ((oa >> 1) & 1);
                const int dz = 2 * oz + ((ob >> 2) & 1) - ((oa >> 2) & 1);
                ok = dx <= 2 && dx >= -2 && dy <= 2 && dy >= -2 && dz <= 2 && dz >= -2;
            }
            ok = ok && S.proot[a] != S.qroot[b];
            big = (S.ps[a + 1] - S.ps[a]) * (S.qe[b] - S.qs[b]) > SMALL_PAIR;
        }
        const unsigned ms = __ballot_sync(0xffffffffu, ok && !big);
        const unsigned mb = __ballot_sync(0xffffffffu, ok && big);
        const unsigned lt = (1u << lane) - 1u;
        if (ok && !big) S.small[nsmall + __popc(ms & lt)] = (uint16_t)((a << 8) | b);
        if (ok && big) S.big[nbig + __popc(mb & lt)] = (uint16_t)((a << 8) | b);
        nsmall += __popc(ms);
        nbig += __popc(mb);
        __syncwarp();
        if (nsmall > PQ_CAP - 32 || nbig > PQ_CAP - 32 || base + 32 >= total) {
            n_pairs += lane == 0 ? (unsigned long long)(nsmall + nbig) : 0ull;
            run_pairs(S, nsmall, nbig, b1, spts, parent, t2, lane, n_tests);
            nsmall = nbig = 0;
            __syncwarp();
        }
    }
}

// phase 0: the cell's own octant-group pairs; phase 1: its neighbour pairs.  Running all
// cells' phase 0 first means phase 1 sees every dense cell's groups joined already, so
// after the first contact between two cells all their group pairs skip on cached roots.
__device__ void dense_cell_work(int r, int phase, DenseSmem& S, const float4* __restrict__ spts,
                                const uint32_t* __restrict__ cstart, const DenseRec* __restrict__ drec,
                                const int* __restrict__ crec, const Grid& g, int* __restrict__ parent, int lane,
                                unsigned long long& n_tests, unsigned long long& n_pairs) {
    const float t2 = g.t2;
    const DenseRec* R = drec + r;
    // P: nonempty octant groups
    int np;
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
    __syncwarp();
    // own-cell group pairs
    if (phase == 0) {
        if (np < 2) return;
        if (lane < np) {
            S.proot[lane] = uf_find(parent, S.ps[lane]);
            S.qs[lane] = S.ps[lane];
            S.qe[lane] = S.ps[lane + 1];
            S.qo[lane] = S.po[lane];
            S.qk[lane] = 26;
        }
        __syncwarp();
        if (lane < np) S.qroot[lane] = S.proot[lane];
        __syncwarp();
        pair_sweep(S, np, 0, np, true, spts, parent, t2, lane, n_tests, n_pairs);
        return;
    }
    // neighbour slots: lanes 0..25 (0..12 forward, 13..25 backward)
    int cnt = 0;
    if (lane < 26) {
        int c[3];
        dense_decode((uint32_t)__ldg(&R->cell), g, c);
        int ox, oy, oz;
        slot_offset(lane, ox, oy, oz);
        uint32_t Q;
        int rec = -1, qs = 0, qe = 0;
        if (dense_neighbor(g, c, ox, oy, oz, Q)) {
            qs = (int)__ldg(cstart + Q);
            qe = (int)__ldg(cstart + Q + 1);
            if (qe - qs > SPARSE_MAX) {
                if (lane < 13) {
                    rec = __ldg(crec + Q);
                    const DenseRec* RQ = drec + rec;
                    for (int k = 0; k < 8; ++k) cnt += __ldg(&RQ->off[k + 1]) > __ldg(&RQ->off[k]);
                }
            } else {
                cnt = qe - qs;
            }
        }
        S.slot_q[lane] = qs;
        S.slot_rec[lane] = rec;
        S.slot_cnt[lane] = cnt;
    }
    // exclusive scan of the group counts over the 26 slots
    int x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    const int nq = __shfl_sync(0xffffffffu, x, 25);
    if (lane < 26) S.slot_off[lane] = x - cnt;
    __syncwarp();
    if (nq == 0) return;
    if (lane < 26 && cnt > 0) {
        int o = x - cnt;
        const int rec = S.slot_rec[lane];
        if (rec >= 0) {
            const DenseRec* RQ = drec + rec;
            for (int k = 0; k < 8; ++k) {
                const int a0 = __ldg(&RQ->off[k]), a1 = __ldg(&RQ->off[k + 1]);
                if (a1 > a0) {
                    S.qs[o] = a0; S.qe[o] = a1; S.qo[o] = (uint8_t)k; S.qk[o] = (uint8_t)lane;
                    ++o;
                }
            }
        } else {
            const int qs = S.slot_q[lane];
            for (int k = 0; k < cnt; ++k) {
                S.qs[o] = qs + k; S.qe[o] = qs + k + 1; S.qo[o] = 0xFF; S.qk[o] = (uint8_t)lane;
                ++o;
            }
        }
    }
    __syncwarp();
    // current roots (P's own groups were joined in phase 0)
    if (lane < np) S.proot[lane] = uf_find(parent, S.ps[lane]);
    for (int b = lane; b < nq; b += 32) S.qroot[b] = uf_find(parent, S.qs[b]);
    __syncwarp();
    // keep only Q groups that can still need a test: when all P groups share one root R
    // (the usual case), a Q group already rooted at R is skipped as a whole
    const int R0 = S.proot[0];
    const bool allsame = __all_sync(0xffffffffu, lane >= np || S.proot[lane] == R0);
    int live_n = 0;
    for (int b0 = 0; b0 < nq; b0 += 32) {
        const int b = b0 + lane;
        const bool live = b < nq && (!allsame || S.qroot[b] != R0);
        int qs_ = 0, qe_ = 0, qr_ = 0;
        uint8_t qo_ = 0, qk_ = 0;
        if (live) { qs_ = S.qs[b]; qe_ = S.qe[b]; qr_ = S.qroot[b]; qo_ = S.qo[b]; qk_ = S.qk[b]; }
        const unsigned m = __ballot_sync(0xffffffffu, live);
        __syncwarp();
        if (live) {
            const int d = live_n + __popc(m & ((1u << lane) - 1u));
            S.qs[d] = qs_; S.qe[d] = qe_; S.qroot[d] = qr_; S.qo[d] = qo_; S.qk[d] = qk_;
        }
        live_n += __popc(m);
        __syncwarp();
    }
    if (live_n == 0) return;
    pair_sweep(S, np, 0, live_n, false, spts, parent, t2, lane, n_tests, n_pairs);
}

__global__ void __launch_bounds__(SCAN_THREADS) k_union_dense(const float4* __restrict__ spts,
                                                            const uint32_t* __restrict__ cstart,
                                                            const DenseRec* __restrict__ drec,
                                                            const int* __restrict__ crec,
                                                            int phase, Grid g,
                                                            int* __restrict__ parent, Meta* __restrict__ meta) {
    __shared__ DenseSmem sm[SCAN_THREADS / kWarp];
    const int lane = threadIdx.x & 31;
    DenseSmem& S = sm[threadIdx.x >> 5];
    const int nd = meta->ndense;
    unsigned long long n_tests = 0, n_pairs = 0;
    while (true) {
        int it = 0;
        if (lane == 0) it = atomicAdd(phase == 0 ? &meta->work : &meta->work2, 1);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= nd) break;
        // phase 1 visits the cells in a scattered order (a multiplicative permutation):
        // cells processed at the same time are then rarely neighbours, so each cell sees
        // the unions its neighbours already made and most group pairs skip on roots
        // (a sweep in cell order processes ~7k adjacent cells at once and tests 3x more).
        const int r = phase == 0 ? it : (int)(((unsigned long long)it * 2654435761ull) % (unsigned long long)nd);
        dense_cell_work(r, phase, S, spts, cstart, drec, crec, g, parent, lane, n_tests, n_pairs);
        __syncwarp();
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

// Sparse cells.  The grid is one resident wave; each warp grid-strides over chunks of
// 128 consecutive cells (so the wave sweeps the sorted order upwards), compacts the
// chunk's nonempty sparse cells into a per-warp list and gives every lane a real cell.
// Loops are warp-uniform with a reconvergence point per neighbour (SIMT efficiency).
constexpr int SP_CHUNK = 128;

__global__ void __launch_bounds__(256) k_union_sparse(const float4* __restrict__ spts,
                                                     const uint32_t* __restrict__ cstart, uint32_t cells, Grid g,
                                                     int* __restrict__ parent, Meta* __restrict__ meta) {
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
            int c[3];
            dense_decode(P, g, c);
#pragma unroll 1
            for (int k = 0; k < 13; ++k) {
                uint32_t Q;
                int qs = 0, qe = 0;
                if (v && dense_neighbor(g, c, c_fwd[k][0], c_fwd[k][1], c_fwd[k][2], Q)) {
                    qs = (int)__ldg(cstart + Q);
                    qe = (int)__ldg(cstart + Q + 1);
                    if (qe - qs > SPARSE_MAX) qe = qs;
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

}  // namespace fec
