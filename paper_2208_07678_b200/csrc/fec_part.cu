// Multi-GPU Mode B: index-sharded input -> spatial slabs on the device.
//
// Every rank holds an arbitrary shard of the cloud (e.g. an index range) with the points'
// global input indices.  The slab decomposition of Mode A (include/fec.h "Multi-GPU slab
// path"; dist.plan_slabs on the host) is computed here from device data only:
//   bbox of the shard -> (caller: all-reduce min/max) -> cut axis = longest extent (ties ->
//   lowest axis), cell layers along it (edge c = d(1+2^-16), reading A6), histogram of the
//   shard's layers -> (caller: all-reduce sum) -> count-balanced cuts on layer boundaries, the
//   same rule as plan_slabs -> each point's destinations (its owner, and the previous rank
//   when it lies in its owner's first layer: the one-cell halo) packed by destination ->
//   (caller: all-to-all) -> the received points in the slab path's local order.
// Layer of x: floor((x - lo) * (1/(c/2))) >> 1 in fp64 -- exactly floor((x - lo) * (1/c)), the
// host planner's arithmetic, since both scale the same correctly rounded quotient by 2.
#include <float.h>

#include "fec_kernels.cuh"
#include "fec_part.cuh"

namespace fec {

__device__ __forceinline__ unsigned f2ord(float f) {  // order-preserving float -> uint
    const unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// state: [0..2] min xyz (ordered uint), [3..5] max xyz (ordered uint), [6] non-finite flag;
// hist[0 .. kPartMaxLayers) zeroed.
__global__ void __launch_bounds__(256) k_part_init(unsigned* __restrict__ state, int* __restrict__ hist) {
    pdl_prologue();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < 3) state[t] = f2ord(__int_as_float(0x7f800000));        // +inf: an empty shard's min
    else if (t < 6) state[t] = f2ord(__int_as_float(0xff800000));   // -inf: an empty shard's max
    else if (t < 8) state[t] = 0u;
    for (int i = t; i < kPartMaxLayers; i += gridDim.x * blockDim.x) hist[i] = 0;
}

// The shard's bbox and non-finite flag (ordered-uint atomics, block-reduced first).
__global__ void __launch_bounds__(256) k_part_bbox(const float* __restrict__ p, int64_t m, unsigned* __restrict__ state) {
    pdl_prologue();
    float mn[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float v = __ldg(p + 3 * i + k);
            bad |= !isfinite(v);
            mn[k] = fminf(mn[k], v);
            mx[k] = fmaxf(mx[k], v);
        }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k)
        for (int o = 16; o > 0; o >>= 1) {
            mn[k] = fminf(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], o));
            mx[k] = fmaxf(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], o));
        }
    bad = __any_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            atomicMin(state + k, f2ord(mn[k]));
            atomicMax(state + 3 + k, f2ord(mx[k]));
        }
        if (bad) atomicOr(state + 6, 1u);
    }
}

// bbox -> float[8] {min xyz, -max xyz, -nonfinite, 0}: one all-reduce MIN over the ranks gives
// the global bbox and whether any rank saw a NaN / inf.
__global__ void k_part_bbox_out(const unsigned* __restrict__ state, float* __restrict__ out) {
    pdl_prologue();
    if (threadIdx.x < 3) {
        out[threadIdx.x] = ord2f(state[threadIdx.x]);
        out[3 + threadIdx.x] = -ord2f(state[3 + threadIdx.x]);
    }
    if (threadIdx.x == 0) {
        out[6] = state[6] ? -1.0f : 0.0f;
        out[7] = 0.0f;
    }
}

// Cut axis, origin and layer count from the global bbox (gbb: {min xyz, -max xyz}).
struct PartAxis {
    int axis, nl, status;
    double lo, inv_h;
};
__device__ __forceinline__ PartAxis part_axis(const float* __restrict__ gbb, double inv_h) {
    PartAxis a;
    double best = -1.0;
    a.axis = 0;
    for (int k = 0; k < 3; ++k) {
        const double e = (double)(-gbb[3 + k]) - (double)gbb[k];
        if (e > best) {
            best = e;
            a.axis = k;
        }
    }
    a.lo = (double)gbb[a.axis];
    a.inv_h = inv_h;
    const double s = floor(__dmul_rn(__dadd_rn((double)(-gbb[3 + a.axis]), -a.lo), inv_h));
    a.status = (s < 2.0 * kPartMaxLayers && s >= 0.0) ? 0 : -3;  // FEC_ERR_GRID_RANGE
    if (gbb[6] < 0.0f) a.status = -2;                            // FEC_ERR_NONFINITE
    a.nl = a.status ? 1 : ((int)(long long)s >> 1) + 1;
    return a;
}
__device__ __forceinline__ int part_layer(float x, const PartAxis& a) {
    return (int)((long long)floor(__dmul_rn(__dadd_rn((double)x, -a.lo), a.inv_h)) >> 1);
}

// Histogram of the shard's layers along the cut axis; info = {axis, nlayers, status}.
__global__ void __launch_bounds__(256) k_part_hist(const float* __restrict__ p, int64_t m,
                                                  const float* __restrict__ gbb, double inv_h,
                                                  int* __restrict__ hist, int* __restrict__ info) {
    pdl_prologue();
    const PartAxis a = part_axis(gbb, inv_h);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        info[0] = a.axis;
        info[1] = a.nl;
        info[2] = a.status;
    }
    if (a.status) return;
    const int64_t mr = (m + 31) & ~int64_t(31);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < mr; i += (int64_t)gridDim.x * blockDim.x) {
        const int L = i < m ? part_layer(__ldg(p + 3 * i + a.axis), a) : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, L);
        if (L >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(hist + L, __popc(peers));
    }
}

// Count-balanced cuts on layer boundaries (one block; the rule of dist.plan_slabs): cum[k] =
// points in layers < k; cut r = the first k with cum[k] >= n*r/world, at least one layer past
// the previous cut, at most nlayers.  plan = {cuts[world+1], owned[world], first[world],
// halo[world], rec_cap} (int64).  cum: scratch of kPartMaxLayers + 1 int64.
__global__ void __launch_bounds__(1024) k_part_plan(const int* __restrict__ hist, const int* __restrict__ info,
                                                   int world, long long* __restrict__ cum,
                                                   long long* __restrict__ plan) {
    pdl_prologue();
    __shared__ long long wsum[32];
    __shared__ long long carry;
    const int nl = info[1];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (info[2]) {  // the cloud cannot be cut: a deterministic empty plan (k_part_status adds why)
        for (int i = tid; i < 4 * world + 2; i += blockDim.x) plan[i] = 0;
        return;
    }
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int b = 0; b < nl; b += 1024) {  // block scan in chunks: cum[k] = sum hist[< k]
        const int k = b + tid;
        long long v = k < nl ? hist[k] : 0;
        long long x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        if (w == 0) {
            long long s = wsum[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            wsum[lane] = s;
        }
        __syncthreads();
        const long long incl = carry + x + (w ? wsum[w - 1] : 0);
        if (k < nl) cum[k + 1] = incl;
        __syncthreads();
        if (tid == 1023) carry = incl;
        __syncthreads();
    }
    if (tid == 0) {
        cum[0] = 0;
        const long long n = cum[nl];
        long long* cuts = plan;
        long long* owned = plan + world + 1;
        long long* first = owned + world;
        long long* halo = first + world;
        cuts[0] = 0;
        cuts[world] = nl;
        for (int r = 1; r < world; ++r) {
            const long long target = (n * r) / world;
            int lo = 0, hi = nl;  // first k in [0, nl] with cum[k] >= target
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (cum[mid] >= target) hi = mid;
                else lo = mid + 1;
            }
            long long b = lo;
            if (b < cuts[r - 1] + 1) b = cuts[r - 1] + 1;
            cuts[r] = b < nl ? b : nl;
        }
        long long rc = 0;
        for (int r = 0; r < world; ++r) {
            owned[r] = cum[cuts[r + 1]] - cum[cuts[r]];
            first[r] = (r > 0 && cuts[r] < nl) ? hist[cuts[r]] : 0;
            halo[r] = (cuts[r + 1] < nl && cuts[r + 1] > cuts[r]) ? hist[cuts[r + 1]] : 0;
            if (owned[r] == 0) first[r] = halo[r] = 0;
        }
        if (world > 1)
            for (int r = 0; r < world; ++r) rc = max(rc, first[r] + halo[r]);
        plan[4 * world + 1] = rc;
    }
}

// plan[4*world + 2] = the partition status (0, or a device-found error).
__global__ void k_part_status(const int* __restrict__ info, long long* __restrict__ plan, int world) {
    pdl_prologue();
    if (threadIdx.x == 0) plan[4 * world + 2] = info[2];
}

// Owner rank of layer L (the last r with cuts[r] <= L; empty slabs own nothing).
__device__ __forceinline__ int part_owner(int L, const long long* __restrict__ cuts, int world) {
    int r = 0;
    while (r + 1 < world && cuts[r + 1] <= L) ++r;
    return r;
}

// mode 0: count per destination; mode 1: scatter into the destinations' segments (cursor[r]
// starts at the segment offset).  A point goes to its owner, and to the previous rank as halo
// when it lies in its owner's first layer and the previous rank owns points.
__global__ void __launch_bounds__(256) k_part_pack(const float* __restrict__ p, const int* __restrict__ gidx, int64_t m,
                                                  const float* __restrict__ gbb, double inv_h,
                                                  const int* __restrict__ info, const long long* __restrict__ plan,
                                                  int world, int mode, unsigned long long* __restrict__ cursor,
                                                  float* __restrict__ send_pts, int* __restrict__ send_gidx) {
    pdl_prologue();
    if (info[2]) return;
    const PartAxis a = part_axis(gbb, inv_h);
    const long long* cuts = plan;
    const long long* owned = plan + world + 1;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const float x = __ldg(p + 3 * i), y = __ldg(p + 3 * i + 1), z = __ldg(p + 3 * i + 2);
        const int L = part_layer(a.axis == 0 ? x : (a.axis == 1 ? y : z), a);
        const int r = part_owner(L, cuts, world);
        const bool halo = r > 0 && L == cuts[r] && owned[r - 1] > 0;
        for (int k = 0; k < (halo ? 2 : 1); ++k) {
            const int dst = k == 0 ? r : r - 1;
            const unsigned long long pos = atomicAdd(cursor + dst, 1ull);
            if (mode == 1) {
                send_pts[3 * pos] = x;
                send_pts[3 * pos + 1] = y;
                send_pts[3 * pos + 2] = z;
                send_gidx[pos] = __ldg(gidx + i);
            }
        }
    }
}

// Receiver: local order first-layer owned | other owned | halo.  mode 0 counts the three
// categories into cnt[0..2]; mode 1 scatters (cursor[c] = the category's start).
__global__ void __launch_bounds__(256) k_part_order(const float* __restrict__ rp, const int* __restrict__ rg, int64_t k,
                                                   const float* __restrict__ gbb, double inv_h,
                                                   const int* __restrict__ info, const long long* __restrict__ plan,
                                                   int world, int rank, int mode,
                                                   unsigned long long* __restrict__ cursor,
                                                   float* __restrict__ out_pts, int* __restrict__ out_gidx) {
    pdl_prologue();
    if (info[2]) return;
    const PartAxis a = part_axis(gbb, inv_h);
    const long long* cuts = plan;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        const float x = __ldg(rp + 3 * i), y = __ldg(rp + 3 * i + 1), z = __ldg(rp + 3 * i + 2);
        const int L = part_layer(a.axis == 0 ? x : (a.axis == 1 ? y : z), a);
        const int c = L >= cuts[rank + 1] ? 2 : ((rank > 0 && L == cuts[rank]) ? 0 : 1);
        const unsigned long long pos = atomicAdd(cursor + c, 1ull);
        if (mode == 1) {
            out_pts[3 * pos] = x;
            out_pts[3 * pos + 1] = y;
            out_pts[3 * pos + 2] = z;
            out_gidx[pos] = __ldg(rg + i);
        }
    }
}

// cursor[i] = sum_{j < i} counts[j] (i < n): the start of each destination / category segment.
__global__ void k_part_offsets(const unsigned long long* __restrict__ counts, int n, unsigned long long* __restrict__ cursor) {
    pdl_prologue();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int i = 0; i < n; ++i) {
            cursor[i] = s;
            s += counts[i];
        }
    }
}

}  // namespace fec
