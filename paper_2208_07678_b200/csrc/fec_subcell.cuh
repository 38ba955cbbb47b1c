// Fine sub-cells of the dense-grid path (internal).
//
// A grid cell (edge c = d(1+2^-16), reading A6) is split into 4x4x4 fine sub-cells of edge
// q = c/4; bit  x + 4y + 16z  of a 64-bit mask names sub-cell (x, y, z) of a cell.  For two
// sub-cells at integer offset o (in sub-cell units):
//   * every pair of points in them is within d when  sum (|o_i|+1)^2 <= 14   ("certain":
//     the largest distance between the two boxes is q*sqrt(sum) <= 0.9355 d; the fp32
//     predicate's rounding (< 2^-21 relative) cannot flip it).  This includes o = 0: a
//     fine sub-cell is a clique.
//   * no pair of points in them can be within d when  sum max(|o_i|-1, 0)^2 >= 16  (the
//     smallest box distance is >= 4q = c > d(1+3*2^-24), beyond any pred-true pair).
// Everything in between is "uncertain" and needs point tests.  Connected groups of occupied
// sub-cells under the certain relation ("components", at most 8 per cell: the largest set
// of pairwise non-certain sub-cells of a 4x4x4 block has 8 elements) are unions of cliques
// joined by all-pairs edges, hence connected in the graph of Eq. 1.
#pragma once
#include <stdint.h>

namespace fec {

using u64s = unsigned long long;
constexpr int kMaxComp = 8;

// In-cell dilation by the certain stencil (the 56 offsets with sum (|o|+1)^2 <= 14).
__host__ __device__ __forceinline__ u64s sc_xp(u64s m) { return (m << 1) & ~0x1111111111111111ull; }
__host__ __device__ __forceinline__ u64s sc_xm(u64s m) { return (m >> 1) & ~0x8888888888888888ull; }
__host__ __device__ __forceinline__ u64s sc_yp(u64s m) { return (m << 4) & ~0x000F000F000F000Full; }
__host__ __device__ __forceinline__ u64s sc_ym(u64s m) { return (m >> 4) & ~0xF000F000F000F000ull; }
__host__ __device__ __forceinline__ u64s sc_zp(u64s m) { return m << 16; }
__host__ __device__ __forceinline__ u64s sc_zm(u64s m) { return m >> 16; }

__host__ __device__ __forceinline__ u64s sc_dilate(u64s m) {
    u64s b = m | sc_xp(m) | sc_xm(m);
    b |= sc_yp(b) | sc_ym(b);
    b |= sc_zp(b) | sc_zm(b);                               // |o_i| <= 1 on every axis
    const u64s pyz = m | sc_yp(m) | sc_ym(m) | sc_zp(m) | sc_zm(m);
    const u64s pxz = m | sc_xp(m) | sc_xm(m) | sc_zp(m) | sc_zm(m);
    const u64s pxy = m | sc_xp(m) | sc_xm(m) | sc_yp(m) | sc_ym(m);
    b |= sc_xp(sc_xp(pyz)) | sc_xm(sc_xm(pyz));            // (+-2, <=1 on one other axis)
    b |= sc_yp(sc_yp(pxz)) | sc_ym(sc_ym(pxz));
    b |= sc_zp(sc_zp(pxy)) | sc_zm(sc_zm(pxy));
    return b;
}

// Split an occupancy mask into its certain-connected components (<= kMaxComp).  Returns
// the number of components; `rest` gets any bits left over (never, by the bound above).
__host__ __device__ __forceinline__ int sc_components(u64s occ, u64s comp[kMaxComp], u64s& rest) {
    int k = 0;
    while (occ && k < kMaxComp) {
        u64s c = occ & (~occ + 1ull);
        while (true) {
            const u64s nc = sc_dilate(c) & occ;
            if (nc == c) break;
            c = nc;
        }
        comp[k++] = c;
        occ &= ~c;
    }
    rest = occ;
    return k;
}

// Neighbour-cell slot index of a cell offset (ox, oy, oz) in {-1,0,1}^3: 0..26, centre 13;
// the opposite offset has index 26 - idx.
__host__ __device__ __forceinline__ int sc_slot(int ox, int oy, int oz) { return (ox + 1) + 3 * (oy + 1) + 9 * (oz + 1); }

// Tables (device copies filled once per device by the host, fec_capi.cu):
//   T[s][a]: Q-frame sub-cells certain-adjacent to sub-cell a of P, Q = P + offset(s)
//   U[s][a]: Q-frame sub-cells within reach of a (certain or uncertain)
//   F[s]   : sub-cells a of P with U[s][a] != 0
//   sh[s][i], shm[s][i] (i < nsh[s]): the certain relation across slot s as whole-mask
//       shifts: Q-frame mask certain-adjacent to X = OR_i shift(X, sh) & shm
constexpr int kMaxShift = 18;
struct SubcellTables {
    u64s T[27][64];
    u64s U[27][64];
    u64s F[27];
    int nsh[27];
    int sh[27][kMaxShift];     // shift amount dx + 4dy + 16dz (may be negative)
    u64s shm[27][kMaxShift];   // target bits whose source lies inside the block
};

__host__ __device__ __forceinline__ u64s sc_shift(u64s m, int s) { return s >= 0 ? (m << s) : (m >> -s); }

// Q-frame sub-cells certain-adjacent to the P-frame mask x across slot s (s != 13).
__host__ __device__ __forceinline__ u64s sc_certain_across(const SubcellTables& t, u64s x, int s) {
    u64s r = 0;
    for (int i = 0; i < t.nsh[s]; ++i) r |= sc_shift(x, t.sh[s][i]) & t.shm[s][i];
    return r;
}

// Construction from the arithmetic definition above (constexpr: the device copy is a
// compile-time constant, so no upload is needed and the first call may be graph-captured).
constexpr void sc_build_tables(SubcellTables& t) {
    for (int s = 0; s < 27; ++s) {
        const int ox = s % 3 - 1, oy = (s / 3) % 3 - 1, oz = s / 9 - 1;
        t.F[s] = 0;
        for (int a = 0; a < 64; ++a) {
            const int ax = a & 3, ay = (a >> 2) & 3, az = a >> 4;
            u64s tc = 0, tu = 0;
            for (int b = 0; b < 64; ++b) {
                const int bx = b & 3, by = (b >> 2) & 3, bz = b >> 4;
                const int o[3] = {4 * ox + bx - ax, 4 * oy + by - ay, 4 * oz + bz - az};
                int smax = 0, smin = 0;
                for (int i = 0; i < 3; ++i) {
                    const int v = o[i] < 0 ? -o[i] : o[i];
                    smax += (v + 1) * (v + 1);
                    const int w = v > 1 ? v - 1 : 0;
                    smin += w * w;
                }
                if (smax <= 14) tc |= 1ull << b;
                if (smin < 16) tu |= 1ull << b;
            }
            t.T[s][a] = tc;
            t.U[s][a] = tu;
            if (tu) t.F[s] |= 1ull << a;
        }
        // shift list: every certain offset o (sum (|o_i|+1)^2 <= 14, |o_i| <= 2) whose image
        // d = o - 4*off still lands inside the block for some source sub-cell
        t.nsh[s] = 0;
        if (s == 13) continue;  // in-cell relations use sc_dilate
        for (int pz = -2; pz <= 2; ++pz)
            for (int py = -2; py <= 2; ++py)
                for (int px = -2; px <= 2; ++px) {
                    const int o[3] = {px, py, pz};
                    int smax = 0;
                    for (int i = 0; i < 3; ++i) {
                        const int v = o[i] < 0 ? -o[i] : o[i];
                        smax += (v + 1) * (v + 1);
                    }
                    if (smax > 14) continue;
                    const int d[3] = {px - 4 * ox, py - 4 * oy, pz - 4 * oz};
                    u64s m = 0;
                    for (int b = 0; b < 64; ++b) {
                        const int sx = (b & 3) - d[0], sy = ((b >> 2) & 3) - d[1], sz = (b >> 4) - d[2];
                        if (sx >= 0 && sx < 4 && sy >= 0 && sy < 4 && sz >= 0 && sz < 4) m |= 1ull << b;
                    }
                    if (!m) continue;
                    if (t.nsh[s] >= kMaxShift) { t.nsh[s] = -1; return; }  // cannot happen (max 18)
                    const int k = t.nsh[s]++;
                    t.sh[s][k] = d[0] + 4 * d[1] + 16 * d[2];
                    t.shm[s][k] = m;
                }
    }
}

constexpr SubcellTables sc_make_tables() {
    SubcellTables t{};
    sc_build_tables(t);
    return t;
}

}  // namespace fec
