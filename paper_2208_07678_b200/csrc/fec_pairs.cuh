// Group-pair evaluation shared by the neighbour-scan kernels (internal).
//
// A "group" is a run of sorted points that is known to be a clique under pred (one
// sub-cell of edge h = c/2), or a single point.  For two groups A and B it
// suffices to find ONE pred-true pair (a, b) and unite their leaders; if A and B already
// share a root the pair is skipped without any test.  Every unordered pair of groups that
// can hold a pred-true pair is examined by exactly one warp.
#pragma once
#include "fec_internal.cuh"
#include "fec_kernels.cuh"

namespace fec {

constexpr int QMAX = SPARSE_MAX > 8 ? SPARSE_MAX : 8;  // max groups on the Q side
constexpr int SMALL_PAIR = 16;  // |A|*|B| at or below which one lane handles the pair alone

struct PairSmem {
    int ps[9];                 // P group starts (+ end)
    int qs[QMAX + 1];          // Q group starts (+ end)
    uint8_t po[8];             // P octants
    uint8_t qo[QMAX];          // Q octants (0xFF: single point, no octant filter)
    uint16_t queue[8 * QMAX];  // small candidate group pairs (a << 8 | b), one lane each
    uint16_t bigq[8 * QMAX];   // big candidate group pairs, whole warp each
    int proot[8];              // cached roots of the P groups (may be stale: see below)
    int qroot[QMAX];           // cached roots of the Q groups
};

// Cache the current roots of all P and Q groups (one find per group instead of two per
// pair).  A stale cached root only causes redundant tests; equal cached roots always mean
// the groups are already connected (ancestry is monotone), so skipping on them is sound.
__device__ __forceinline__ void load_roots(PairSmem& S, int np, int nq, int* parent, int lane) {
    if (lane < np) S.proot[lane] = uf_find(parent, S.ps[lane]);
    else if (lane < np + nq) S.qroot[lane - np] = uf_find(parent, S.qs[lane - np]);
    __syncwarp();
}

// The 13 forward neighbour offsets: (dz>0) or (dz==0 and dy>0) or (dz==0, dy==0, dx>0).
// With same-cell pairs, every unordered pair of adjacent cells is visited exactly once.
__constant__ signed char c_fwd[13][3] = {
    {1, 0, 0},  {-1, 1, 0}, {0, 1, 0},  {1, 1, 0},  {-1, -1, 1}, {0, -1, 1}, {1, -1, 1},
    {-1, 0, 1}, {0, 0, 1},  {1, 0, 1},  {-1, 1, 1}, {0, 1, 1},   {1, 1, 1}};

// Enumerate candidate pairs (a in P groups, b in Q groups) that still need a test: their
// cached roots differ, and (unless a Q group is a single point, qo == 0xFF) their sub-cell
// offset is at most 2 on every axis (larger offsets are > c > d apart).  `same_cell`: only
// b > a.  (ox, oy, oz) is the cell offset Q - P.  Small pairs (|A|*|B| <= SMALL_PAIR) go to
// S.queue, big ones to S.bigq.  Call after load_roots().  Returns both lengths.
__device__ __forceinline__ int2 build_queue(PairSmem& S, int np, int nq, bool same_cell, int ox, int oy, int oz,
                                            int lane) {
    int nsmall = 0, nbig = 0;
    const int npairs = np * nq;
    for (int base = 0; base < npairs; base += 32) {
        const int pid = base + lane;
        bool ok = pid < npairs;
        int a = 0, b = 0;
        bool big = false;
        if (ok) {
            a = pid / nq;
            b = pid - a * nq;
            if (same_cell) {
                ok = b > a;
            } else if (S.qo[b] != 0xFF) {
                const int oa = S.po[a], ob = S.qo[b];
                const int dx = 2 * ox + (ob & 1) - (oa & 1);
                const int dy = 2 * oy + ((ob >> 1) & 1) - ((oa >> 1) & 1);
                const int dz = 2 * oz + ((ob >> 2) & 1) - ((oa >> 2) & 1);
                ok = dx <= 2 && dx >= -2 && dy <= 2 && dy >= -2 && dz <= 2 && dz >= -2;
            }
            ok = ok && S.proot[a] != S.qroot[b];
            big = (S.ps[a + 1] - S.ps[a]) * (S.qs[b + 1] - S.qs[b]) > SMALL_PAIR;
        }
        const unsigned ms = __ballot_sync(0xffffffffu, ok && !big);
        const unsigned mb = __ballot_sync(0xffffffffu, ok && big);
        const unsigned lt = (1u << lane) - 1u;
        if (ok && !big) S.queue[nsmall + __popc(ms & lt)] = (uint16_t)((a << 8) | b);
        if (ok && big) S.bigq[nbig + __popc(mb & lt)] = (uint16_t)((a << 8) | b);
        nsmall += __popc(ms);
        nbig += __popc(mb);
    }
    __syncwarp();
    return make_int2(nsmall, nbig);
}

// Evaluate the queued group pairs: small ones one lane each, big ones by the whole warp,
// both with an early exit at the first pred-true pair.
__device__ __forceinline__ void process_queue(PairSmem& S, int2 nq2, const float4* __restrict__ spts,
                                              int* parent, float t2, int lane, unsigned long long& n_tests) {
    for (int e = lane; e < nq2.x; e += 32) {
        const int a = S.queue[e] >> 8, b = S.queue[e] & 255;
        const int sa = S.ps[a], ea = S.ps[a + 1], sb = S.qs[b], eb = S.qs[b + 1];
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
    for (int e = 0; e < nq2.y; ++e) {
        const int a = S.bigq[e] >> 8, b = S.bigq[e] & 255;
        if (S.proot[a] == S.qroot[b]) continue;   // joined by an earlier big pair of this queue
        int sa = S.ps[a], ea = S.ps[a + 1], sb = S.qs[b], eb = S.qs[b + 1];
        // lanes stride over the larger group, the smaller one is broadcast
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
            if (lane == 0) {
                uf_unite(parent, sa, sb);
                const int r = uf_find(parent, sa);
                S.proot[a] = r;
                S.qroot[b] = r;
            }
            __syncwarp();
        }
    }
    __syncwarp();
}

}  // namespace fec
