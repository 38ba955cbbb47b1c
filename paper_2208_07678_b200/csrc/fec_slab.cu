// Multi-GPU slab path: owned-only component statistics,
// boundary-record packing, the replicated boundary union-find and the owned relabel.
//
// A rank holds its slab (owned points) plus a one-cell halo (the first cell layer of the
// next slab) and has already run a1..a8 on owned ∪ halo (run_core).  Local input order is
//   [0, n_first)         owned points in the slab's first cell layer (the previous rank's halo)
//   [n_first, n_owned)   the other owned points
//   [n_owned, n_local)   halo points (owned by the next rank)
// so "boundary" points (local index < n_first or >= n_owned) are exactly the points that
// two ranks see.  Every edge of the global fixed-radius graph lies inside some rank's
// owned ∪ halo (cut planes are cell boundaries of a grid with edge > d_th), so the global
// components are the local components joined through shared boundary points.
//
// Records (int32 words; layout in fec_slab_record_words()):
//   header  [0] = nP, [1] = nC, [2] = [3] = 0
//   P[k]    (gidx of a boundary point, key of its local component)           2 words
//           (rec_cap rounded up to even entries, so the C region is 16-byte aligned)
//   C[k]    (key, owned size, owned min gidx, local root)                     4 words
// key(K) = the largest gidx among K's boundary points: a member of K, so two keys from
// different ranks can only coincide when the components share that point (and then they
// belong to one global component anyway).
#include "fec_kernels.cuh"
#include "fec_slab.cuh"

namespace fec {

constexpr int SL_SLOTS = 256;

// Per local root r (a sorted position): size[r] = owned members, minidx[r] = min gidx of
// owned members, ckey[r] = max gidx of boundary members (-1: none).  size/minidx arrive
// initialised to 0 / INT_MAX by a4; ckey to -1.  Warp- then block-aggregated like k_tail_stats.
__global__ void __launch_bounds__(256) k_slab_stats(const int* __restrict__ parent, const int* __restrict__ val,
                                                   const int* __restrict__ gidx, int64_t n, int n_owned,
                                                   int n_first, int* __restrict__ size,
                                                   int* __restrict__ minidx, int* __restrict__ ckey,
                                                   Meta* __restrict__ meta) {
    pdl_prologue();
    if (meta->status) return;  // a1 rejected the input
    __shared__ int hkey[SL_SLOTS], hcnt[SL_SLOTS], hmin[SL_SLOTS], hbk[SL_SLOTS];
    for (int k = threadIdx.x; k < SL_SLOTS; k += blockDim.x) {
        hkey[k] = -1;
        hcnt[k] = 0;
        hmin[k] = 0x7fffffff;
        hbk[k] = -1;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned long long roots = 0;
    const int64_t chunk = ((n + gridDim.x - 1) / gridDim.x + 255) / 256 * 256;
    const int64_t b0 = (int64_t)blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    for (int64_t s0 = b0; s0 < b1; s0 += blockDim.x) {
        const int64_t s = s0 + threadIdx.x;
        const bool ok = s < b1;
        const int r = ok ? __ldg(parent + s) : -1;
        const int i = ok ? __ldg(val + s) : 0;
        const int gv = ok ? __ldg(gidx + i) : 0;
        const bool owned = ok && i < n_owned;
        const bool bnd = ok && (i < n_first || i >= n_owned);
        roots += (ok && r == (int)s) ? 1ull : 0ull;
        // the lanes of one root meet in one __match_any_sync; the group's leader adds once (into
        // the block's table if the root owns its slot -- a big component -- else to the root)
        const int key = ok ? r : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        const int cnt = __popc(peers & __ballot_sync(0xffffffffu, owned));
        const int mn = __reduce_min_sync(peers, owned ? gv : 0x7fffffff);
        const int bk = __reduce_max_sync(peers, bnd ? gv : -1);
        if (key >= 0 && lane == __ffs(peers) - 1) {
            const unsigned h = ((unsigned)key * 2654435761u) >> 24;
            int cur = hkey[h];
            if (cur == -1) cur = atomicCAS(&hkey[h], -1, key);
            if (cur == -1 || cur == key) {
                if (cnt) atomicAdd(&hcnt[h], cnt);
                if (mn != 0x7fffffff) atomicMin(&hmin[h], mn);
                if (bk >= 0) atomicMax(&hbk[h], bk);
            } else {
                if (cnt) atomicAdd(size + key, cnt);
                if (mn != 0x7fffffff) atomicMin(minidx + key, mn);
                if (bk >= 0) atomicMax(ckey + key, bk);
            }
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < SL_SLOTS; k += blockDim.x) {
        const int key = hkey[k];
        if (key >= 0) {
            if (hcnt[k]) atomicAdd(size + key, hcnt[k]);
            if (hmin[k] != 0x7fffffff) atomicMin(minidx + key, hmin[k]);
            if (hbk[k] >= 0) atomicMax(ckey + key, hbk[k]);
        }
    }
    if (meta->instrument) {
        for (int o = 16; o > 0; o >>= 1) roots += __shfl_xor_sync(0xffffffffu, roots, o);
        if (lane == 0 && roots) atomicAdd(&meta->components, roots);
    }
}

// Warp-aggregated append: returns this lane's slot (valid where `want`).
__device__ __forceinline__ int warp_append(int* counter, bool want) {
    const unsigned m = __ballot_sync(0xffffffffu, want);
    if (!m) return -1;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(counter, __popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    return base + __popc(m & ((1u << lane) - 1u));
}

// P records for every boundary point, C records for every boundary-touching local root.
// Roots are points or component nodes node_of(n, rmask, r, k), so the loop runs over the n
// points and the 8 node slots of every dense record.
__global__ void __launch_bounds__(256) k_slab_pack(const int* __restrict__ parent, const int* __restrict__ val,
                                                  const int* __restrict__ gidx, int64_t n, int n_owned,
                                                  int n_first, const int* __restrict__ size,
                                                  const int* __restrict__ minidx, const int* __restrict__ ckey,
                                                  int* __restrict__ rec, int rec_cap, const Meta* __restrict__ meta,
                                                  uint32_t rmask) {
    pdl_prologue();
    if (meta->status) return;  // header stays zero: no records
    int* P = rec + SLAB_HDR;
    int* Cr = rec + slab_c_off(rec_cap);
    const int64_t nodes = n + 8 * (int64_t)meta->ndense;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t nr = (nodes + 31) & ~int64_t(31);  // whole warps stay in the loop
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nr; u += stride) {
        const bool ok = u < nodes;
        const bool pt = u < n;
        const int64_t s = (pt || !ok) ? u : node_of((int)n, rmask, (int)((u - n) >> 3), (int)((u - n) & 7));
        const int r = ok ? __ldg(parent + s) : 0;
        const int i = pt ? __ldg(val + s) : 0;
        const bool bnd = pt && (i < n_first || i >= n_owned);
        const bool is_root = ok && r == (int)s;
        const int k = (bnd || is_root) ? __ldg(ckey + r) : -1;
        const int ps = warp_append(rec + 0, bnd);
        if (bnd) {
            P[2 * (int64_t)ps] = __ldg(gidx + i);
            P[2 * (int64_t)ps + 1] = k;
        }
        const bool emitc = is_root && k >= 0;
        const int cs = warp_append(rec + 1, emitc);
        if (emitc) {
            int4 c = make_int4(k, __ldg(size + r), __ldg(minidx + r), r);
            reinterpret_cast<int4*>(Cr)[cs] = c;
        }
    }
}

// ---- replicated boundary merge (every rank runs the same thing on the gathered records) --
__device__ __forceinline__ int mh_insert(int* hkey, unsigned mask, int key) {
    unsigned h = ((unsigned)key * 2654435761u) & mask;
    while (true) {
        int cur = hkey[h];
        if (cur == key) return (int)h;
        if (cur == -1) {
            cur = atomicCAS(hkey + h, -1, key);
            if (cur == -1 || cur == key) return (int)h;
        }
        h = (h + 1) & mask;
    }
}
__device__ __forceinline__ int mh_lookup(const int* hkey, unsigned mask, int key) {
    unsigned h = ((unsigned)key * 2654435761u) & mask;
    while (true) {
        const int cur = hkey[h];
        if (cur == key) return (int)h;
        if (cur == -1) return -1;
        h = (h + 1) & mask;
    }
}

__global__ void __launch_bounds__(256) k_merge_init(int* __restrict__ hkey, int* __restrict__ hpar,
                                                   int* __restrict__ gsize, int* __restrict__ gmin, int64_t hc) {
    pdl_prologue();
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < hc; k += (int64_t)gridDim.x * blockDim.x) {
        hkey[k] = -1;
        hpar[k] = (int)k;
        gsize[k] = 0;
        gmin[k] = 0x7fffffff;
    }
}

// Union the two nodes (boundary point gidx, component key) of every P record of every rank.
__global__ void __launch_bounds__(256) k_merge_link(const int* __restrict__ all, int world, int64_t words,
                                                   int rec_cap, int* __restrict__ hkey, unsigned mask,
                                                   int* __restrict__ hpar) {
    pdl_prologue();
    const int64_t total = (int64_t)world * rec_cap;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int rk = (int)(t / rec_cap), j = (int)(t % rec_cap);
        const int* rec = all + rk * words;
        if (j >= __ldg(rec + 0)) continue;
        const int q = __ldg(rec + SLAB_HDR + 2 * j), key = __ldg(rec + SLAB_HDR + 2 * j + 1);
        const int a = mh_insert(hkey, mask, q);
        const int b = (key == q) ? a : mh_insert(hkey, mask, key);
        if (a != b) uf_unite(hpar, a, b);
    }
}

// Sum owned sizes and take the min owned gidx of every C record at its global root.
__global__ void __launch_bounds__(256) k_merge_stats(const int* __restrict__ all, int world, int64_t words,
                                                    int rec_cap, const int* __restrict__ hkey, unsigned mask,
                                                    int* __restrict__ hpar, int* __restrict__ gsize,
                                                    int* __restrict__ gmin) {
    pdl_prologue();
    const int64_t total = (int64_t)world * rec_cap;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int rk = (int)(t / rec_cap), j = (int)(t % rec_cap);
        const int* rec = all + rk * words;
        if (j >= __ldg(rec + 1)) continue;
        const int4 c = reinterpret_cast<const int4*>(rec + slab_c_off(rec_cap))[j];
        const int root = uf_find(hpar, mh_lookup(hkey, mask, c.x));
        if (c.y) atomicAdd(gsize + root, c.y);
        if (c.z != 0x7fffffff) atomicMin(gmin + root, c.z);
    }
}

// Own C records: overwrite the local root's owned stats with the global component's.
__global__ void __launch_bounds__(256) k_merge_resolve(const int* __restrict__ own, int rec_cap,
                                                      const int* __restrict__ hkey, unsigned mask,
                                                      int* __restrict__ hpar, const int* __restrict__ gsize,
                                                      const int* __restrict__ gmin, int* __restrict__ size,
                                                      int* __restrict__ minidx) {
    pdl_prologue();
    const int nc = __ldg(own + 1);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nc; j += gridDim.x * blockDim.x) {
        const int4 c = reinterpret_cast<const int4*>(own + slab_c_off(rec_cap))[j];
        const int root = uf_find(hpar, mh_lookup(hkey, mask, c.x));
        size[c.w] = gsize[root];
        minidx[c.w] = gmin[root];
    }
}

// labels_owned[i] for owned local indices i: global min gidx of the component, or -1.
__global__ void __launch_bounds__(256) k_slab_relabel(const int* __restrict__ parent, const int* __restrict__ val,
                                                     const int* __restrict__ size, const int* __restrict__ minidx,
                                                     int64_t n, int n_owned, long long min_size,
                                                     long long max_size, int* __restrict__ labels,
                                                     const Meta* __restrict__ meta) {
    pdl_prologue();
    if (meta->status) return;  // the local step failed: labels_owned is left untouched
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const int i = __ldg(val + s);
        if (i >= n_owned) continue;
        const int r = __ldg(parent + s);
        const long long sz = __ldg(size + r);
        labels[i] = (sz >= min_size && sz <= max_size) ? __ldg(minidx + r) : -1;
    }
}

}  // namespace fec
