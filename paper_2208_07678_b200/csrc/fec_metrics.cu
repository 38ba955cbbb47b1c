// AP metric (include/fec_metrics.h; Eq. 2; SPEC.md
// L392-408; readings M1-M4 in DESIGN.md §8e).
//
//   k_ap_keys    key = (pred+1) << B | gt for gt != 0 (else all ones), cluster sizes |P|, |G|
//   radix sort   LSD, 8-bit digits, over the 2B significant bits (the clustering path's kernels)
//   k_ap_heads   run heads of equal (P, G) keys  -> scan -> k_ap_runs: the pair histogram rows
//   k_ap_pkeys   first row of every predicted cluster -> sort key (n - |P|) << B | P
//   radix sort   -> predicted clusters by descending size, ascending label
//   k_ap_prefs   every predicted cluster's preferred gt cluster in parallel; TP/FP directly
//                when no gt cluster is preferred twice (then greedy order cannot matter)
//   k_ap_greedy  otherwise one warp replays the greedy matching (M3) in order
#include <math.h>

#include <algorithm>

#include "fec.h"
#include "fec_internal.cuh"
#include "fec_kernels.cuh"
#include "fec_metrics.h"

namespace fec {
namespace {

struct ApWs {
    u64 *keyA, *keyB;
    int *valA, *valB;
    uint32_t* sizeP;   // [n + 1] by pred + 1
    uint32_t* sizeG;   // [n + 1] by gt
    uint32_t* flag;    // [n + 1]
    uint32_t* pos;     // [n + 1]
    uint32_t* scratch;
    uint32_t* counts;  // radix digit counts
    uint32_t* scan32;
    u64* rkey;         // [n] run keys
    uint32_t* rstart;  // [n + 1] run starts (+ end sentinel)
    uint8_t* matched;  // [n + 1]
    uint32_t* claims;  // [n + 1] predicted clusters preferring each gt cluster
    int* meta;         // [0] valid keys, [1] runs, [2] error, [3] contested, [4..7] n_pred, tp, fp, n_gt
    int num_tiles;
    size_t total;
};

int ap_bits(int64_t n) {
    int b = 1;
    while ((int64_t(1) << b) <= n + 1) ++b;
    return b;
}

ApWs ap_carve(char* base, int64_t n) {
    Carver c{base};
    ApWs w;
    const int64_t m = n + 1;
    w.num_tiles = (int)((m + RS_TILE - 1) / RS_TILE);
    w.keyA = c.take<u64>(m);
    w.keyB = c.take<u64>(m);
    w.valA = c.take<int>(m);
    w.valB = c.take<int>(m);
    w.sizeP = c.take<uint32_t>(m + 1);
    w.sizeG = c.take<uint32_t>(m + 1);
    w.flag = c.take<uint32_t>(m + 1);
    w.pos = c.take<uint32_t>(m + 1);
    w.scratch = c.take<uint32_t>(scan_scratch_elems(m + 1));
    w.counts = c.take<uint32_t>((size_t)256 * w.num_tiles + 1);
    w.scan32 = c.take<uint32_t>(scan_scratch_elems((int64_t)256 * w.num_tiles + 1));
    w.rkey = c.take<u64>(m);
    w.rstart = c.take<uint32_t>(m + 1);
    w.matched = c.take<uint8_t>(m + 1);
    w.claims = c.take<uint32_t>(m + 1);
    w.meta = c.take<int>(8);
    w.total = c.off + 256;
    return w;
}

__global__ void k_ap_clear(ApWs w, int64_t n) {
    pdl_prologue();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
        w.sizeP[i] = 0u;
        w.sizeG[i] = 0u;
        w.matched[i] = 0;
        w.claims[i] = 0u;
    }
    if (blockIdx.x == 0 && threadIdx.x < 8) w.meta[threadIdx.x] = 0;
}

__global__ void k_ap_keys(const int32_t* __restrict__ pred, const int32_t* __restrict__ gt, int64_t n, int B,
                          ApWs w) {
    pdl_prologue();
    int valid = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n + 1; i += (int64_t)gridDim.x * blockDim.x) {
        u64 key = ~0ull;
        if (i < n) {
            const int32_t p = pred[i], g = gt[i];
            if (p < -1 || p >= n || g < 0 || g > n) {
                atomicOr(w.meta + 2, 1);
            } else if (g != 0) {
                key = ((u64)(p + 1) << B) | (u64)g;
                atomicAdd(w.sizeG + g, 1u);
                if (p >= 0) atomicAdd(w.sizeP + p + 1, 1u);
                ++valid;
            }
        }
        w.keyA[i] = key;
        w.valA[i] = (int)i;
    }
    for (int o = 16; o > 0; o >>= 1) valid += __shfl_xor_sync(0xffffffffu, valid, o);
    if ((threadIdx.x & 31) == 0 && valid) atomicAdd(w.meta + 0, valid);
}

// run heads over the sorted keys (invalid keys sort last and start no run)
__global__ void k_ap_heads(const u64* __restrict__ key, int64_t m, uint32_t* __restrict__ flag) {
    pdl_prologue();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= m; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t f = 0u;
        if (i < m) {
            const u64 k = key[i];
            f = (k != ~0ull && (i == 0 || key[i - 1] != k)) ? 1u : 0u;
        }
        flag[i] = f;
    }
}

__global__ void k_ap_runs(const u64* __restrict__ key, int64_t m, const uint32_t* __restrict__ flag,
                          const uint32_t* __restrict__ pos, ApWs w) {
    pdl_prologue();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        if (flag[i]) {
            w.rkey[pos[i]] = key[i];
            w.rstart[pos[i]] = (uint32_t)i;
        }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const int runs = (int)pos[m];
        w.meta[1] = runs;
        w.rstart[runs] = (uint32_t)w.meta[0];  // end sentinel: the number of valid keys
    }
}

// one entry per predicted cluster (its first row), sort key (n - |P|) << B | P; the rest ~0
__global__ void k_ap_pkeys(int64_t n, int B, ApWs w, u64* __restrict__ pk, int* __restrict__ pv) {
    pdl_prologue();
    const int runs = w.meta[1];
    const u64 gmask = (1ull << B) - 1ull;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n + 1; r += (int64_t)gridDim.x * blockDim.x) {
        u64 key = ~0ull;
        if (r < runs) {
            const u64 pp = w.rkey[r] >> B;  // pred + 1
            const bool first = r == 0 || (w.rkey[r - 1] >> B) != pp;
            if (pp >= 1 && first) {
                const uint32_t sz = w.sizeP[pp];
                key = ((u64)((uint32_t)n - sz) << B) | (pp - 1);
            }
        }
        (void)gmask;
        pk[r] = key;
        pv[r] = (int)r;
    }
}

// Fast path: every predicted cluster's preferred gt cluster (largest IoU over all its rows,
// ties by smaller gt label).  If no gt cluster is preferred by two predicted clusters, the
// greedy matching of M3 takes exactly these (nothing a cluster prefers is consumed before
// its turn), so TP/FP follow in parallel; otherwise k_ap_greedy replays M3 in order.
__global__ void k_ap_prefs(int64_t n, int B, double thr, ApWs w) {
    pdl_prologue();
    const int runs = w.meta[1];
    const u64 gmask = (1ull << B) - 1ull;
    int np = 0, tp = 0, fp = 0, ng = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n + 1; r += (int64_t)gridDim.x * blockDim.x) {
        if (r >= 1 && w.sizeG[r] != 0u) ++ng;  // distinct gt labels (r doubles as a gt label)
        if (r >= runs) continue;
        const u64 pp = w.rkey[r] >> B;
        if (pp < 1 || (r > 0 && (w.rkey[r - 1] >> B) == pp)) continue;
        const int64_t sp = w.sizeP[pp];
        int64_t best = -1, bc = 0, bu = 1;
        for (int64_t q = r; q < runs && (w.rkey[q] >> B) == pp; ++q) {
            const int64_t g = (int64_t)(w.rkey[q] & gmask);
            const int64_t c = (int64_t)w.rstart[q + 1] - (int64_t)w.rstart[q];
            const int64_t u = sp + (int64_t)w.sizeG[g] - c;
            if (best < 0 || c * bu > bc * u) {
                best = g;
                bc = c;
                bu = u;
            }
        }
        ++np;
        if ((double)bc >= thr * (double)bu) ++tp;
        else ++fp;
        if (atomicAdd(w.claims + best, 1u) != 0u) w.meta[3] = 1;  // contested: replay M3
    }
    for (int o = 16; o > 0; o >>= 1) {
        np += __shfl_xor_sync(0xffffffffu, np, o);
        tp += __shfl_xor_sync(0xffffffffu, tp, o);
        fp += __shfl_xor_sync(0xffffffffu, fp, o);
        ng += __shfl_xor_sync(0xffffffffu, ng, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (np) atomicAdd(w.meta + 4, np);
        if (tp) atomicAdd(w.meta + 5, tp);
        if (fp) atomicAdd(w.meta + 6, fp);
        if (ng) atomicAdd(w.meta + 7, ng);
    }
}

// M3 in order (only when a gt cluster is contested): one warp, predicted clusters by the
// sorted keys, the lanes scan a cluster's rows and a warp argmax picks the unmatched best.
__global__ void k_ap_greedy(int64_t n, int B, double thr, const u64* __restrict__ pk, const int* __restrict__ pv,
                            ApWs w, fec_ap_result_t* __restrict__ res) {
    pdl_prologue();
    if (blockIdx.x != 0) return;
    const int lane = threadIdx.x & 31;
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    if (w.meta[2]) {
        if (lane == 0) {
            res->tp = res->fp = -1;
            res->n_pred = res->n_gt = 0;
            res->ap = qnan;
            res->status = -1;
            res->pad = 0;
        }
        return;
    }
    int64_t tp = w.meta[5], fp = w.meta[6];
    const int64_t npred = w.meta[4], ngt = w.meta[7];
    if (w.meta[3]) {
        const int runs = w.meta[1];
        const u64 gmask = (1ull << B) - 1ull;
        tp = fp = 0;
        for (int64_t e = 0; e < npred; ++e) {
            const int r0 = pv[e];
            const u64 pp = w.rkey[r0] >> B;
            const int64_t sp = w.sizeP[pp];
            int64_t best = -1, bc = 0, bu = 1;
            for (int64_t base = r0; base < runs; base += 32) {
                const int64_t q = base + lane;
                bool in = q < runs && (w.rkey[q] >> B) == pp;
                int64_t g = -1, c = 0, u = 1;
                if (in) {
                    g = (int64_t)(w.rkey[q] & gmask);
                    if (w.matched[g]) {
                        g = -1;
                    } else {
                        c = (int64_t)w.rstart[q + 1] - (int64_t)w.rstart[q];
                        u = sp + (int64_t)w.sizeG[g] - c;
                    }
                }
                // warp argmax of c/u (ties: smaller g)
                for (int o = 16; o > 0; o >>= 1) {
                    const int64_t g2 = __shfl_xor_sync(0xffffffffu, g, o);
                    const int64_t c2 = __shfl_xor_sync(0xffffffffu, c, o);
                    const int64_t u2 = __shfl_xor_sync(0xffffffffu, u, o);
                    const bool take = g2 >= 0 && (g < 0 || c2 * u > c * u2 || (c2 * u == c * u2 && g2 < g));
                    if (take) { g = g2; c = c2; u = u2; }
                }
                if (g >= 0 && (best < 0 || c * bu > bc * u || (c * bu == bc * u && g < best))) {
                    best = g;
                    bc = c;
                    bu = u;
                }
                if (!__all_sync(0xffffffffu, in)) break;  // the cluster's rows ended in this chunk
            }
            if (best < 0) {
                ++fp;
                continue;
            }
            if (lane == 0) w.matched[best] = 1;
            __syncwarp();
            if ((double)bc >= thr * (double)bu) ++tp;
            else ++fp;
        }
    }
    if (lane == 0) {
        res->tp = tp;
        res->fp = fp;
        res->n_pred = npred;
        res->n_gt = ngt;
        res->ap = (tp + fp) == 0 ? (ngt == 0 ? 1.0 : 0.0) : (double)tp / (double)(tp + fp);
        res->status = 0;
        res->pad = 0;
    }
}

int ap_sort(u64*& kin, u64*& kout, int*& vin, int*& vout, int64_t m, int bits, const ApWs& w, cudaStream_t st) {
    int launches = 0;
    const int passes = (bits + 7) / 8;
    for (int p = 0; p < passes; ++p) {
        const int shift = 8 * p;
        pdl(k_radix_hist, w.num_tiles, RS_THREADS, 0, st)(kin, m, shift, w.counts, w.num_tiles);
        launches += exclusive_scan<uint32_t>(w.counts, w.counts, (int64_t)256 * w.num_tiles, w.scan32, st);
        pdl(k_radix_scatter, w.num_tiles, RS_THREADS, 0, st)(kin, vin, kout, vout, m, shift, w.counts, w.num_tiles);
        launches += 2;
        std::swap(kin, kout);
        std::swap(vin, vout);
    }
    return launches;
}

}  // namespace
}  // namespace fec

using namespace fec;

extern "C" {

size_t fec_ap_workspace_bytes(int64_t n) {
    if (n < 0 || n > INT32_MAX - 1) return 0;
    return ap_carve(nullptr, n).total;
}

fec_status_t fec_average_precision(const int32_t* pred, const int32_t* gt, int64_t n, double threshold,
                                   fec_ap_result_t* result, void* workspace, size_t workspace_bytes,
                                   void* stream) {
    if (n < 0 || n > INT32_MAX - 1) { set_last_error("n out of range"); return FEC_ERR_INVALID_ARGUMENT; }
    if (!(threshold > 0.0 && threshold <= 1.0)) { set_last_error("threshold must be in (0, 1]"); return FEC_ERR_INVALID_ARGUMENT; }
    if (!result || !workspace || (n > 0 && (!pred || !gt))) { set_last_error("null pointer"); return FEC_ERR_INVALID_ARGUMENT; }
    if (((uintptr_t)workspace & 255) != 0) { set_last_error("workspace must be 256-B aligned"); return FEC_ERR_INVALID_ARGUMENT; }
    if (workspace_bytes < fec_ap_workspace_bytes(n)) { set_last_error("workspace too small (see fec_ap_workspace_bytes)"); return FEC_ERR_INVALID_ARGUMENT; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ApWs w = ap_carve(static_cast<char*>(workspace), n);
    const int B = ap_bits(n);
    const int64_t m = n + 1;  // one extra (invalid) key keeps every buffer non-empty
    const unsigned g = (unsigned)std::min<int64_t>((m + 255) / 256, 148 * 16);
    pdl(k_ap_clear, g, 256, 0, st)(w, n);
    pdl(k_ap_keys, g, 256, 0, st)(pred, gt, n, B, w);
    u64 *kin = w.keyA, *kout = w.keyB;
    int *vin = w.valA, *vout = w.valB;
    ap_sort(kin, kout, vin, vout, m, 2 * B, w, st);
    pdl(k_ap_heads, g, 256, 0, st)(kin, m, w.flag);
    exclusive_scan<uint32_t>(w.flag, w.pos, m + 1, w.scratch, st);
    pdl(k_ap_runs, g, 256, 0, st)(kin, m, w.flag, w.pos, w);
    // predicted clusters: keys into the buffers the pair sort no longer needs
    u64* pk = kout;
    int* pv = vout;
    pdl(k_ap_pkeys, g, 256, 0, st)(n, B, w, pk, pv);
    u64* pk2 = kin;
    int* pv2 = vin;
    ap_sort(pk, pk2, pv, pv2, m, 2 * B, w, st);
    pdl(k_ap_prefs, g, 256, 0, st)(n, B, threshold, w);
    pdl(k_ap_greedy, 1, 32, 0, st)(n, B, threshold, pk, pv, w, result);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_last_error(std::string("fec_average_precision launch: ") + cudaGetErrorString(e));
        return FEC_ERR_CUDA;
    }
    return FEC_OK;
}

}  // extern "C"
