// RANSAC plane-fit ground removal (include/fec_ground.h; PAPER.md L179-184,
// SPEC.md L307-310; readings G1-G7 in DESIGN.md §8c).
//
// Pipeline (one stream, no host synchronisation):
//   k_g_planes   one thread per hypothesis: binary64 plane from the three points, tilt flag
//   k_g_count    every point against every plane: planes in shared memory, 16 points per
//                thread as coordinate pairs, per plane a REDUX over the warp, shared then
//                global atomics.  Per test 1.5 FFMA2 + FSETP + predicated IADD.
//   k_g_best     argmax (count, then lowest h) over the tilt-valid planes; the result record
//   k_g_flags    per 2048-point tile: survivors, binary64 partial sums of the inliers
//                (relative to the hypothesis' first point) for the least-squares refit
//   scan         exclusive scan of the per-tile survivor counts
//   k_g_compact  stable compaction of the survivors (points + input indices)
//   k_g_refine   fixed-order reduction of the partial sums, 3x3 Jacobi eigen-solve
#include <math.h>

#include <algorithm>
#include <mutex>

#include "fec.h"
#include "fec_ground.h"
#include "fec_internal.cuh"

namespace fec {
namespace {

constexpr int kGTile = 2048;   // points per tile of the flags / compact kernels (256 x 8)
constexpr int kCountPts = 12;  // points per thread in k_g_count (pairs for FFMA2)

struct GroundWs {
    float4* planes;     // [H]
    int* valid;         // [H] 0 none, 1 plane outside the tilt bound, 2 valid
    unsigned* cnt;      // [H]
    uint32_t* tcount;   // [tiles] survivors per tile
    uint32_t* tscan;    // [tiles] exclusive scan
    uint32_t* scratch;  // scan scratch
    double* part;       // [tiles][9] inlier sums relative to r0
    size_t total;
};

int64_t g_tiles(int64_t n) { return (n + kGTile - 1) / kGTile; }

GroundWs g_carve(char* base, int64_t n, int32_t H) {
    Carver c{base};
    GroundWs w;
    const int64_t T = g_tiles(n) + 1;
    w.planes = c.take<float4>(H + 1);
    w.valid = c.take<int>(H + 1);
    w.cnt = c.take<unsigned>(H + 1);
    w.tcount = c.take<uint32_t>(T);
    w.tscan = c.take<uint32_t>(T);
    w.scratch = c.take<uint32_t>(scan_scratch_elems(T));
    w.part = c.take<double>(9 * T);
    w.total = c.off + 256;
    return w;
}

__global__ void k_g_planes(const float* __restrict__ p, int64_t n, const int32_t* __restrict__ tri, int H,
                           double cos_tilt, float4* __restrict__ planes, int* __restrict__ valid,
                           unsigned* __restrict__ cnt) {
    pdl_prologue();
    const int h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= H) return;
    cnt[h] = 0u;
    const float qnan = __int_as_float(0x7fc00000);
    float4 out = make_float4(qnan, qnan, qnan, qnan);  // no plane: every test is false
    int v = 0;
    const int a = tri[3 * h], b = tri[3 * h + 1], c = tri[3 * h + 2];
    if (a >= 0 && b >= 0 && c >= 0 && a < n && b < n && c < n && a != b && a != c && b != c) {
        const double p0x = p[3 * (int64_t)a], p0y = p[3 * (int64_t)a + 1], p0z = p[3 * (int64_t)a + 2];
        const double ux = __dsub_rn(p[3 * (int64_t)b], p0x), uy = __dsub_rn(p[3 * (int64_t)b + 1], p0y),
                     uz = __dsub_rn(p[3 * (int64_t)b + 2], p0z);
        const double vx = __dsub_rn(p[3 * (int64_t)c], p0x), vy = __dsub_rn(p[3 * (int64_t)c + 1], p0y),
                     vz = __dsub_rn(p[3 * (int64_t)c + 2], p0z);
        const double mx = __dsub_rn(__dmul_rn(uy, vz), __dmul_rn(uz, vy));
        const double my = __dsub_rn(__dmul_rn(uz, vx), __dmul_rn(ux, vz));
        const double mz = __dsub_rn(__dmul_rn(ux, vy), __dmul_rn(uy, vx));
        const double s = __dadd_rn(__dadd_rn(__dmul_rn(mx, mx), __dmul_rn(my, my)), __dmul_rn(mz, mz));
        const double L = __dsqrt_rn(s);
        if (L > 0.0 && isfinite(L)) {
            double nx = __ddiv_rn(mx, L), ny = __ddiv_rn(my, L), nz = __ddiv_rn(mz, L);
            if (nz < 0.0) { nx = -nx; ny = -ny; nz = -nz; }
            const double off = -__dadd_rn(__dadd_rn(__dmul_rn(nx, p0x), __dmul_rn(ny, p0y)), __dmul_rn(nz, p0z));
            out = make_float4(__double2float_rn(nx), __double2float_rn(ny), __double2float_rn(nz),
                              __double2float_rn(off));
            v = nz >= cos_tilt ? 2 : 1;
        }
    }
    planes[h] = out;
    valid[h] = v;
}

// reading G3: three single-rounded fused multiply-adds (explicit __fmaf_rn)
__device__ __forceinline__ bool g_inlier(float4 pl, float x, float y, float z, float t) {
    const float r = __fmaf_rn(pl.z, z, __fmaf_rn(pl.y, y, __fmaf_rn(pl.x, x, pl.w)));
    return fabsf(r) <= t;
}

// Two residuals at once: fma.rn.f32x2 (FFMA2) is two independent binary32 fused multiply-
// adds, each rounded once -- exactly reading G3's fmaf chain, two points per instruction.
__device__ __forceinline__ u64 g_fma2(u64 a, u64 b, u64 c) {
    u64 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ u64 g_pack(float lo, float hi) {
    return (u64)__float_as_uint(lo) | ((u64)__float_as_uint(hi) << 32);
}
// v += (|r| <= t): FSETP + predicated IADD
__device__ __forceinline__ void g_count_le(unsigned& v, float r, float t) {
    asm("{\n\t.reg .pred p;\n\t.reg .f32 a;\n\tabs.f32 a, %1;\n\tsetp.le.f32 p, a, %2;\n\t@p add.u32 %0, %0, 1;\n\t}"
        : "+r"(v) : "f"(r), "f"(t));
}

// Every point against every plane.  A warp holds 32 x kCountPts points (lane-contiguous
// rows, NaN padding past n: a NaN residual is never an inlier) as coordinate pairs; per
// plane (duplicated coefficients in shared memory) each lane evaluates its points two at a
// time (3 FFMA2 per pair, FSETP + predicated IADD per point), one REDUX sums the warp, lane 0
// adds it to the block's shared counter.
__global__ void __launch_bounds__(256, 4) k_g_count(const float* __restrict__ p, int64_t n,
                                                 const float4* __restrict__ planes, int H, float t,
                                                 unsigned* __restrict__ cnt) {
    pdl_prologue();
    extern __shared__ float4 g_smem[];
    ulonglong2* sp = reinterpret_cast<ulonglong2*>(g_smem);  // [H][2]: (nx,nx | ny,ny), (nz,nz | off,off)
    unsigned* sc = reinterpret_cast<unsigned*>(g_smem + 2 * H);
    for (int h = threadIdx.x; h < H; h += blockDim.x) {
        const float4 pl = planes[h];
        sp[2 * h] = make_ulonglong2(g_pack(pl.x, pl.x), g_pack(pl.y, pl.y));
        sp[2 * h + 1] = make_ulonglong2(g_pack(pl.z, pl.z), g_pack(pl.w, pl.w));
        sc[h] = 0u;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const float qnan = __int_as_float(0x7fc00000);
    const int64_t per_block = (int64_t)blockDim.x * kCountPts;
    constexpr int kPairs = kCountPts / 2;
    for (int64_t base = (int64_t)blockIdx.x * per_block; base < n; base += (int64_t)gridDim.x * per_block) {
        u64 X[kPairs], Y[kPairs], Z[kPairs];
#pragma unroll
        for (int k = 0; k < kPairs; ++k) {
            const int64_t i0 = base + (2 * k) * blockDim.x + threadIdx.x;
            const int64_t i1 = i0 + blockDim.x;
            const bool ok0 = i0 < n, ok1 = i1 < n;
            X[k] = g_pack(ok0 ? __ldg(p + 3 * i0) : qnan, ok1 ? __ldg(p + 3 * i1) : qnan);
            Y[k] = g_pack(ok0 ? __ldg(p + 3 * i0 + 1) : qnan, ok1 ? __ldg(p + 3 * i1 + 1) : qnan);
            Z[k] = g_pack(ok0 ? __ldg(p + 3 * i0 + 2) : qnan, ok1 ? __ldg(p + 3 * i1 + 2) : qnan);
        }
        for (int h0 = 0; h0 < H; h0 += 32) {
            // lane l collects the warp's count of plane h0 + l; one shared atomic per lane
            unsigned mine = 0u;
            const int hn = min(32, H - h0);
#pragma unroll 2
            for (int j = 0; j < hn; ++j) {
                const ulonglong2 a = sp[2 * (h0 + j)], b = sp[2 * (h0 + j) + 1];
                unsigned v0 = 0u, v1 = 0u;  // two chains of predicated increments
#pragma unroll
                for (int k = 0; k < kPairs; ++k) {
                    const u64 r = g_fma2(b.x, Z[k], g_fma2(a.y, Y[k], g_fma2(a.x, X[k], b.y)));
                    g_count_le(v0, __uint_as_float((unsigned)r), t);
                    g_count_le(v1, __uint_as_float((unsigned)(r >> 32)), t);
                }
                const unsigned c = __reduce_add_sync(0xffffffffu, v0 + v1);
                mine = lane == j ? c : mine;
            }
            if (lane < hn && mine) atomicAdd(sc + h0 + lane, mine);
        }
    }
    __syncthreads();
    for (int h = threadIdx.x; h < H; h += blockDim.x)
        if (sc[h]) atomicAdd(cnt + h, sc[h]);
}

__global__ void __launch_bounds__(1024) k_g_best(const float4* __restrict__ planes, const int* __restrict__ valid,
                                                 const unsigned* __restrict__ cnt, int H, int64_t n,
                                                 int64_t min_inliers, int64_t* __restrict__ counts,
                                                 fec_ground_result_t* __restrict__ res) {
    pdl_prologue();
    __shared__ u64 sbest[32];
    __shared__ int snv[32];
    u64 best = 0;
    int nv = 0;
    for (int h = threadIdx.x; h < H; h += blockDim.x) {
        if (counts) counts[h] = (int64_t)cnt[h];
        if (valid[h] == 2) {
            ++nv;
            const u64 key = ((u64)cnt[h] << 32) | (u64)(0xffffffffu - (unsigned)h);
            best = key > best ? key : best;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const u64 b2 = __shfl_xor_sync(0xffffffffu, best, o);
        best = b2 > best ? b2 : best;
        nv += __shfl_xor_sync(0xffffffffu, nv, o);
    }
    if ((threadIdx.x & 31) == 0) {
        sbest[threadIdx.x >> 5] = best;
        snv[threadIdx.x >> 5] = nv;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 b = 0;
        int tnv = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            b = sbest[w] > b ? sbest[w] : b;
            tnv += snv[w];
        }
        int hb = -1;
        int64_t c = 0;
        if (b != 0) {
            hb = (int)(0xffffffffu - (unsigned)(b & 0xffffffffu));
            c = (int64_t)(b >> 32);
            if (c < min_inliers) hb = -1;
        }
        const float qf = __int_as_float(0x7fc00000);
        const double qd = __longlong_as_double(0x7ff8000000000000ll);
        res->best = hb;
        res->n_valid = tnv;
        res->n_inliers = hb >= 0 ? c : 0;
        res->n_keep = n - (hb >= 0 ? c : 0);
        const float4 pl = hb >= 0 ? planes[hb] : make_float4(qf, qf, qf, qf);
        res->plane[0] = pl.x;
        res->plane[1] = pl.y;
        res->plane[2] = pl.z;
        res->plane[3] = pl.w;
        for (int k = 0; k < 4; ++k) res->refined[k] = qd;
    }
}

__device__ __forceinline__ bool g_is_ground(const fec_ground_result_t* res, float4 pl, float x, float y, float z,
                                            float t) {
    return res->best >= 0 && g_inlier(pl, x, y, z, t);
}

template <typename T>
__device__ __forceinline__ T block_sum_256(T v, T* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    T s = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < 8; ++w) s += sh[w];  // fixed order
    return s;
}

// per tile: survivors, and the inliers' binary64 sums relative to r0 (the best
// hypothesis' first point): S1 (3) and the upper triangle of S2 (6)
__global__ void __launch_bounds__(256) k_g_flags(const float* __restrict__ p, int64_t n,
                                                 const int32_t* __restrict__ tri,
                                                 const fec_ground_result_t* __restrict__ res, float t,
                                                 uint32_t* __restrict__ tcount, double* __restrict__ part) {
    pdl_prologue();
    __shared__ double shd[8];
    __shared__ uint32_t shu[8];
    const int best = res->best;
    const float4 pl = make_float4(res->plane[0], res->plane[1], res->plane[2], res->plane[3]);
    double r0x = 0, r0y = 0, r0z = 0;
    if (best >= 0) {
        const int64_t a = tri[3 * best];
        r0x = p[3 * a];
        r0y = p[3 * a + 1];
        r0z = p[3 * a + 2];
    }
    double s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t keep = 0;
    const int64_t base = (int64_t)blockIdx.x * kGTile;
    for (int k = 0; k < kGTile / 256; ++k) {
        const int64_t i = base + k * 256 + threadIdx.x;
        if (i >= n) break;
        const float x = __ldg(p + 3 * i), y = __ldg(p + 3 * i + 1), z = __ldg(p + 3 * i + 2);
        if (g_is_ground(res, pl, x, y, z, t)) {
            const double dx = __dsub_rn(x, r0x), dy = __dsub_rn(y, r0y), dz = __dsub_rn(z, r0z);
            s[0] += dx; s[1] += dy; s[2] += dz;
            s[3] += dx * dx; s[4] += dx * dy; s[5] += dx * dz;
            s[6] += dy * dy; s[7] += dy * dz; s[8] += dz * dz;
        } else {
            ++keep;
        }
    }
    const uint32_t kt = block_sum_256<uint32_t>(keep, shu);
    if (threadIdx.x == 0) tcount[blockIdx.x] = kt;
    if (best < 0) return;
    for (int q = 0; q < 9; ++q) {
        const double v = block_sum_256<double>(s[q], shd);
        if (threadIdx.x == 0) part[9 * (int64_t)blockIdx.x + q] = v;
    }
}

__global__ void __launch_bounds__(256) k_g_compact(const float* __restrict__ p, int64_t n,
                                                   const fec_ground_result_t* __restrict__ res, float t,
                                                   const uint32_t* __restrict__ tscan, float* __restrict__ kp,
                                                   int32_t* __restrict__ kidx) {
    pdl_prologue();
    __shared__ uint32_t wsum[8];
    const float4 pl = make_float4(res->plane[0], res->plane[1], res->plane[2], res->plane[3]);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t out = tscan[blockIdx.x];
    const int64_t base = (int64_t)blockIdx.x * kGTile;
    for (int k = 0; k < kGTile / 256; ++k) {
        const int64_t i = base + k * 256 + threadIdx.x;  // block-uniform rounds keep input order
        bool s = false;
        float x = 0.f, y = 0.f, z = 0.f;
        if (i < n) {
            x = __ldg(p + 3 * i);
            y = __ldg(p + 3 * i + 1);
            z = __ldg(p + 3 * i + 2);
            s = !g_is_ground(res, pl, x, y, z, t);
        }
        const unsigned m = __ballot_sync(0xffffffffu, s);
        if (lane == 0) wsum[warp] = __popc(m);
        __syncthreads();
        uint32_t before = 0, total = 0;
        for (int w = 0; w < 8; ++w) {
            before += w < warp ? wsum[w] : 0u;
            total += wsum[w];
        }
        if (s) {
            const uint32_t o = out + before + __popc(m & ((1u << lane) - 1u));
            kp[3 * (int64_t)o] = x;
            kp[3 * (int64_t)o + 1] = y;
            kp[3 * (int64_t)o + 2] = z;
            kidx[o] = (int32_t)i;
        }
        out += total;
        __syncthreads();
    }
}

// symmetric 3x3 eigen-solve by cyclic Jacobi rotations (binary64)
__device__ void jacobi3(double A[3][3], double V[3][3]) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) V[i][j] = i == j ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 50; ++sweep) {
        const double off = fabs(A[0][1]) + fabs(A[0][2]) + fabs(A[1][2]);
        const double diag = fabs(A[0][0]) + fabs(A[1][1]) + fabs(A[2][2]);
        if (off <= 1e-300 || off <= 1e-17 * diag) break;
        for (int pp = 0; pp < 2; ++pp)
            for (int q = pp + 1; q < 3; ++q) {
                if (A[pp][q] == 0.0) continue;
                const double theta = (A[q][q] - A[pp][pp]) / (2.0 * A[pp][q]);
                const double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(tt * tt + 1.0), s = tt * c;
                for (int k = 0; k < 3; ++k) {  // A <- J^T A J
                    const double akp = A[k][pp], akq = A[k][q];
                    A[k][pp] = c * akp - s * akq;
                    A[k][q] = s * akp + c * akq;
                }
                for (int k = 0; k < 3; ++k) {
                    const double apk = A[pp][k], aqk = A[q][k];
                    A[pp][k] = c * apk - s * aqk;
                    A[q][k] = s * apk + c * aqk;
                }
                for (int k = 0; k < 3; ++k) {
                    const double vkp = V[k][pp], vkq = V[k][q];
                    V[k][pp] = c * vkp - s * vkq;
                    V[k][q] = s * vkp + c * vkq;
                }
            }
    }
}

__global__ void __launch_bounds__(256) k_g_refine(const float* __restrict__ p, const int32_t* __restrict__ tri,
                                                  const double* __restrict__ part, int64_t tiles,
                                                  fec_ground_result_t* __restrict__ res) {
    pdl_prologue();
    __shared__ double sh[256][9];
    __shared__ double S[9];
    const int best = res->best;
    if (best < 0) return;
    // fixed-order reduction: thread t sums tiles t, t+256, ...; thread 0 sums the 256 partials
    double v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t b = threadIdx.x; b < tiles; b += blockDim.x)
#pragma unroll
        for (int q = 0; q < 9; ++q) v[q] += part[9 * b + q];
#pragma unroll
    for (int q = 0; q < 9; ++q) sh[threadIdx.x][q] = v[q];
    __syncthreads();
    if (threadIdx.x < 9) {
        double a = 0;
#pragma unroll 1
        for (int k = 0; k < 256; ++k) a += sh[k][threadIdx.x];
        S[threadIdx.x] = a;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const double m = (double)res->n_inliers;
    if (res->n_inliers < 3) {
        for (int k = 0; k < 4; ++k) res->refined[k] = (double)res->plane[k];
        return;
    }
    const int64_t a = tri[3 * best];
    const double r0[3] = {p[3 * a], p[3 * a + 1], p[3 * a + 2]};
    const double mu[3] = {S[0] / m, S[1] / m, S[2] / m};
    double A[3][3];
    A[0][0] = S[3] - S[0] * mu[0];
    A[0][1] = A[1][0] = S[4] - S[0] * mu[1];
    A[0][2] = A[2][0] = S[5] - S[0] * mu[2];
    A[1][1] = S[6] - S[1] * mu[1];
    A[1][2] = A[2][1] = S[7] - S[1] * mu[2];
    A[2][2] = S[8] - S[2] * mu[2];
    double V[3][3];
    jacobi3(A, V);
    int k = 0;
    if (A[1][1] < A[k][k]) k = 1;
    if (A[2][2] < A[k][k]) k = 2;
    double nx = V[0][k], ny = V[1][k], nz = V[2][k];
    const double L = sqrt(nx * nx + ny * ny + nz * nz);
    nx /= L; ny /= L; nz /= L;
    if (nz < 0) { nx = -nx; ny = -ny; nz = -nz; }
    const double c[3] = {r0[0] + mu[0], r0[1] + mu[1], r0[2] + mu[2]};
    res->refined[0] = nx;
    res->refined[1] = ny;
    res->refined[2] = nz;
    res->refined[3] = -(nx * c[0] + ny * c[1] + nz * c[2]);
}

__global__ void k_g_fill(int32_t* __restrict__ lab, int64_t n) {
    pdl_prologue();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        lab[i] = -2;
}

__global__ void k_g_expand(const int32_t* __restrict__ kidx, const int32_t* __restrict__ klab,
                           const fec_ground_result_t* __restrict__ res, int32_t* __restrict__ lab) {
    pdl_prologue();
    const int64_t nk = res->n_keep;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nk; j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t l = klab[j];
        lab[kidx[j]] = l < 0 ? -1 : kidx[l];
    }
}

struct GroundEvents {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    bool recorded = false;
};
thread_local GroundEvents g_gev;

fec_status_t g_fail(const char* what, cudaError_t e) {
    set_last_error(std::string(what) + ": " + cudaGetErrorString(e));
    return FEC_ERR_CUDA;
}

}  // namespace
}  // namespace fec

using namespace fec;

extern "C" {

size_t fec_ground_workspace_bytes(int64_t n, int32_t n_hyp) {
    if (n < 0 || n > INT32_MAX || n_hyp < 0 || n_hyp > FEC_GROUND_MAX_HYP) return 0;
    return g_carve(nullptr, n, n_hyp).total;
}

fec_status_t fec_ground_remove(const float* points, int64_t n, const int32_t* triplets, int32_t n_hyp,
                               float threshold, double cos_max_tilt, int64_t min_inliers, float* keep_points,
                               int32_t* keep_idx, int64_t* counts, fec_ground_result_t* result,
                               void* workspace, size_t workspace_bytes, void* stream) {
    if (n < 0 || n > INT32_MAX) { set_last_error("n out of range"); return FEC_ERR_INVALID_ARGUMENT; }
    if (n_hyp < 0 || n_hyp > FEC_GROUND_MAX_HYP) { set_last_error("n_hyp out of range"); return FEC_ERR_INVALID_ARGUMENT; }
    if (!(threshold >= 0.0f) || !isfinite(threshold)) { set_last_error("threshold must be finite and >= 0"); return FEC_ERR_INVALID_ARGUMENT; }
    if (isnan(cos_max_tilt)) { set_last_error("cos_max_tilt is NaN"); return FEC_ERR_INVALID_ARGUMENT; }
    if (min_inliers < 0) { set_last_error("min_inliers < 0"); return FEC_ERR_INVALID_ARGUMENT; }
    if (!result || !workspace || (n > 0 && (!points || !keep_points || !keep_idx)) || (n_hyp > 0 && !triplets)) {
        set_last_error("null pointer");
        return FEC_ERR_INVALID_ARGUMENT;
    }
    if (((uintptr_t)workspace & 255) != 0) { set_last_error("workspace must be 256-B aligned"); return FEC_ERR_INVALID_ARGUMENT; }
    const size_t need = fec_ground_workspace_bytes(n, n_hyp);
    if (workspace_bytes < need) { set_last_error("workspace too small (see fec_ground_workspace_bytes)"); return FEC_ERR_INVALID_ARGUMENT; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    GroundWs w = g_carve(static_cast<char*>(workspace), n, n_hyp);
    const int H = n_hyp;
    const int64_t tiles = g_tiles(n);
    if (H > 0) pdl(k_g_planes, (H + 127) / 128, 128, 0, st)(points, n, triplets, H, cos_max_tilt, w.planes, w.valid, w.cnt);
    if (H > 0 && n > 0) {
        // per-device: SM count and the opt-in shared-memory size already granted to k_g_count
        static int sms_of[64] = {};
        static size_t smem_of[64] = {};
        static std::mutex mu;
        int dev = 0, sms = 0, bps = 0;
        cudaGetDevice(&dev);
        const size_t smem = (size_t)H * (2 * sizeof(float4) + sizeof(unsigned));
        {
            std::lock_guard<std::mutex> lock(mu);
            if (sms_of[dev & 63] == 0) cudaDeviceGetAttribute(&sms_of[dev & 63], cudaDevAttrMultiProcessorCount, dev);
            sms = sms_of[dev & 63];
            if (smem > 48 * 1024 && smem_of[dev & 63] < smem) {
                cudaError_t e = cudaFuncSetAttribute(k_g_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (e != cudaSuccess) return g_fail("cudaFuncSetAttribute(k_g_count)", e);
                smem_of[dev & 63] = smem;
            }
        }
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_g_count, 256, smem);
        const int64_t need_blocks = (n + 256 * kCountPts - 1) / (256 * kCountPts);
        const int64_t grid = std::min<int64_t>(need_blocks, (int64_t)sms * (bps > 0 ? bps : 1));
        const bool timed = timing_enabled();
        if (timed) {
            if (!g_gev.e0) {
                cudaEventCreate(&g_gev.e0);
                cudaEventCreate(&g_gev.e1);
            }
            cudaEventRecord(g_gev.e0, st);
        }
        pdl(k_g_count, (unsigned)grid, 256, smem, st)(points, n, w.planes, H, threshold, w.cnt);
        if (timed) {
            cudaEventRecord(g_gev.e1, st);
            g_gev.recorded = true;
        }
    }
    pdl(k_g_best, 1, 1024, 0, st)(w.planes, w.valid, w.cnt, H, n, min_inliers, counts, result);
    if (n > 0) {
        pdl(k_g_flags, (unsigned)tiles, 256, 0, st)(points, n, triplets, result, threshold, w.tcount, w.part);
        exclusive_scan<uint32_t>(w.tcount, w.tscan, tiles, w.scratch, st);
        pdl(k_g_compact, (unsigned)tiles, 256, 0, st)(points, n, result, threshold, w.tscan, keep_points, keep_idx);
        pdl(k_g_refine, 1, 256, 0, st)(points, triplets, w.part, tiles, result);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return g_fail("fec_ground_remove launch", e);
    return FEC_OK;
}

fec_status_t fec_ground_count_ms(float* ms) {
    if (!ms) { set_last_error("null pointer"); return FEC_ERR_INVALID_ARGUMENT; }
    *ms = -1.0f;
    if (!g_gev.recorded) return FEC_OK;
    cudaError_t e = cudaEventSynchronize(g_gev.e1);
    if (e == cudaSuccess) e = cudaEventElapsedTime(ms, g_gev.e0, g_gev.e1);
    if (e != cudaSuccess) return g_fail("fec_ground_count_ms", e);
    return FEC_OK;
}

fec_status_t fec_ground_expand_labels(const int32_t* keep_idx, const int32_t* keep_labels,
                                      const fec_ground_result_t* result, int64_t n, int32_t* labels_out,
                                      void* stream) {
    if (n < 0 || n > INT32_MAX) { set_last_error("n out of range"); return FEC_ERR_INVALID_ARGUMENT; }
    if (n == 0) return FEC_OK;
    if (!keep_idx || !keep_labels || !result || !labels_out) { set_last_error("null pointer"); return FEC_ERR_INVALID_ARGUMENT; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
    pdl(k_g_fill, g, 256, 0, st)(labels_out, n);
    pdl(k_g_expand, g, 256, 0, st)(keep_idx, keep_labels, result, labels_out);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return g_fail("fec_ground_expand_labels launch", e);
    return FEC_OK;
}

}  // extern "C"
