// Internal device helpers and launch declarations of the FEC sm_100a path.
// Not part of the C ABI (include/fec.h is).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

namespace fec {

// ---- programmatic dependent launch (sm_90+) ---------------------------------------------
// Every kernel of the library starts with pdl_prologue(): wait until the previous kernel of
// the stream has completed and its writes are visible, then let the next kernel launch.
// Launched through pdl() (below), consecutive kernels of one stream overlap their launch
// latency and block rampup with the tail of the previous kernel; launched with <<<>>> the
// wait returns at once.  Dependencies are unchanged: no kernel reads anything before its wait.
__device__ __forceinline__ void pdl_prologue() {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 900
    asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");
#endif
}

bool pdl_enabled();  // FEC_PDL=0 in the environment turns it off (A/B measurements)
// FEC_DEBUG_SYNC=1: synchronise the stream after every launch (outside stream capture) and
// report the first failing kernel by name on stderr and in fec_last_error() (debugging aid)
bool debug_sync_enabled();
cudaError_t debug_sync_after(const void* kernel, cudaStream_t st);

template <typename... KArgs>
struct PdlLaunch {
    void (*k)(KArgs...);
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute attr[1];
    template <typename... Args>
    cudaError_t operator()(Args&&... args) {
        cfg.attrs = attr;
        cfg.numAttrs = pdl_enabled() ? 1 : 0;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
        if (e == cudaSuccess && debug_sync_enabled()) return debug_sync_after(reinterpret_cast<const void*>(k), cfg.stream);
        return e;
    }
};
template <typename... KArgs>
inline PdlLaunch<KArgs...> pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st) {
    PdlLaunch<KArgs...> l;
    l.k = k;
    l.cfg = cudaLaunchConfig_t{};
    l.cfg.gridDim = grid;
    l.cfg.blockDim = block;
    l.cfg.dynamicSmemBytes = smem;
    l.cfg.stream = st;
    l.attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    l.attr[0].val.programmaticStreamSerializationAllowed = 1;
    return l;
}

void set_last_error(const std::string& msg);  // fec_last_error()'s thread-local slot
bool timing_enabled();                         // fec_set_timing()

using u64 = unsigned long long;
constexpr int kWarp = 32;

// ---- the predicate: Eq. 1, readings A1-A3 --------------------------
// Each operation is an explicit round-to-nearest intrinsic, which nvcc never contracts
// into an FMA; the library is additionally compiled with -fmad=false and without
// fast-math / flush-to-zero.
__device__ __forceinline__ float d2_rn(float4 a, float4 b) {
    float dx = __fsub_rn(b.x, a.x);
    float dy = __fsub_rn(b.y, a.y);
    float dz = __fsub_rn(b.z, a.z);
    float s = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
    return __fadd_rn(s, __fmul_rn(dz, dz));
}
__device__ __forceinline__ bool pred(float4 a, float4 b, float t2) { return d2_rn(a, b) <= t2; }

// ---- grid geometry -----------------------------------------------------------------------
// Computed on the DEVICE by the planning block of k_bbox (fec_kernels.cu) from the bbox, or
// uploaded by the host (batch mode); every kernel of the path reads it from the workspace
// (load_grid), so no host round trip sits between a1 and the rest of the pipeline.
struct Grid {
    double lo[3];       // bbox minimum (fp32 values widened)
    double inv_h;       // 1/h (double): sub-cell coordinate = floor((x - lo) * inv_h)
    double h;           // sub-cell edge = c/2, c = d*(1+2^-16)
    double inv_q;       // 2*inv_h (exact): fine sub-cell coordinate = floor((x - lo) * inv_q), edge c/4
    int32_t dims[3];    // cells per axis
    int32_t hashed;     // 0: cell handle = linear cell id (occupancy bitmap over the grid)
                        // 1: cell handle = slot of an open-addressing table of occupied cells
    uint32_t stride[3]; // bitmap mode: linear cell id = sum_a c[a]*stride[a] (smallest dim fastest)
    int32_t perm[3];    // bitmap mode: axes from fastest to slowest
    uint32_t sdiv[2];   // bitmap mode: stride[perm[2]], stride[perm[1]] (for decoding)
    uint32_t hmask;     // hash mode: slots - 1 (slots a power of two >= 2n)
    uint32_t rmask;     // dense records: R - 1 (node ids, fec_kernels.cuh node_of)
    float t2;           // fl32(d*d) (reading A3)
    int32_t status;     // FEC_OK, or the error found by a1 (every later kernel returns at once)
    int32_t key_sort;   // 1: the key-sort binning path runs, 0: the counting path
    int32_t passes;     // key-sort path: 8-bit LSD passes over the linear cell ids
    int32_t key_bits;   // significant bits of the linear cell id (bitmap mode)
    int32_t pad0;
    int64_t words;      // occupancy words: grid cells / 32 (bitmap) or slots / 32 (hash)
    int64_t cells_total;
    u64* hkey;          // hash mode: packed cell coordinates of each slot (~0 = empty)
    // batch mode (fec_cluster_batch_ws): clouds [boff[c], boff[c+1]) with origins blo[3c..3c+2]
    // and z cell offsets bz[c] (device arrays); batch == 0 for a single cloud
    int32_t batch;
    int32_t nclouds;
    const int64_t* boff;
    const double* blo;
    const int32_t* bz;
};

// Every kernel stages the device-resident Grid in shared memory after its PDL wait (one
// thread copies it; all threads then read fields with LDS, which costs no registers: a
// register copy of the whole struct would live through every loop).  Must be reached by
// all threads of the block (it synchronises).
#define FEC_LOAD_GRID(gp)                                       \
    __shared__ Grid fec_grid_sh_;                               \
    if (threadIdx.x == 0) fec_grid_sh_ = *(gp);                 \
    __syncthreads();                                            \
    const Grid& g = fec_grid_sh_

// The same, with the PDL prologue in between: the Grid is written once per call, by a1 (k_bbox)
// or by the host (batch mode, a copy that ends the PDL chain), and a kernel starts only after the
// kernel two places before it has completed (every kernel triggers its dependents after its own
// wait).  So every kernel except the one right after k_bbox (k_zero) may read the Grid BEFORE its
// wait, overlapping that load's latency with the previous kernel's tail.
#define FEC_PROLOGUE_GRID(gp)                                   \
    __shared__ Grid fec_grid_sh_;                               \
    if (threadIdx.x == 0) fec_grid_sh_ = *(gp);                 \
    pdl_prologue();                                             \
    __syncthreads();                                            \
    const Grid& g = fec_grid_sh_

// Sub-cell coordinate on one axis: floor((x - lo) * inv_h).  Cell = sub >> 1 and the octant
// bit = sub & 1, so cell and sub-cell always agree.  Monotone in x (DESIGN.md §4.2 shows
// that pred-true pairs differ by <= 2 sub-cells and <= 1 cell on every axis).
__device__ __forceinline__ uint32_t sub_coord(float x, double lo, double inv_h) {
    return (uint32_t)floor(__dmul_rn(__dadd_rn((double)x, -lo), inv_h));
}

__device__ __forceinline__ u64 pack_cell(uint32_t cx, uint32_t cy, uint32_t cz) {
    return (u64)cx | ((u64)cy << 21) | ((u64)cz << 42);
}
__device__ __forceinline__ u64 hash_cell(u64 pc) {
    pc ^= pc >> 31;
    pc *= 0x7fb5d329728ea185ull;
    pc ^= pc >> 27;
    pc *= 0x81dadef4bc2dd44dull;
    pc ^= pc >> 33;
    return pc;
}

// ---- union-find over sorted positions (ECL-CC style) ----------------------------------
// Invariant: parents are strictly "above" their children in a fixed total order and a root r
// has parent[r] == r.  Hooks attach the lower root under the higher one with atomicCAS
// (performed at L2, always on the current value); path compression only ever moves a parent
// up.  FEC_UF_MINROOT (default): "above" = smaller id, so a set's root is its SMALLEST sorted
// position.  The union kernels sweep the sorted order upwards, so a component's root is
// established early and the points met later hook straight under it: trees stay shallow
// (the opposite order moves the root up with the sweep and deepens the tree at every hook).
// Component nodes (ids above every point) then hang under a point whenever a dense cell's
// component touches a sparse cell's point; nothing depends on roots being nodes.
// Reads are plain (L1-cacheable) loads: a stale value is still an ancestor, so a find may
// return a non-root; the hook's CAS then fails and returns the current parent, and the loop
// continues from there (values move strictly up, so it terminates).  Two finds that return
// the same node prove the inputs are connected, so skipping on equal roots is always
// sound.  The loads/stores are inline PTX so the compiler cannot merge or hoist them.
#ifndef FEC_UF_MINROOT
#define FEC_UF_MINROOT 1
#endif
// true iff `a` lies strictly above `b` in the union-find order
__host__ __device__ __forceinline__ bool uf_above(int a, int b) {
#if FEC_UF_MINROOT
    return a < b;
#else
    return a > b;
#endif
}
// FEC_UF_RELAXED=1 makes the racing parent loads / stores PTX relaxed atomics at GPU scope
// (the memory model's well-defined form of a racy access; they bypass L1), instead of weak
// accesses (L1-cacheable; a stale value is still an ancestor, see above).
#ifndef FEC_UF_RELAXED
#define FEC_UF_RELAXED 0
#endif
__device__ __forceinline__ int ld_parent(const int* p, int x) {
    int v;
#if FEC_UF_RELAXED
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p + x) : "memory");
#else
    asm volatile("ld.global.b32 %0, [%1];" : "=r"(v) : "l"(p + x) : "memory");
#endif
    return v;
}
__device__ __forceinline__ void st_parent(int* p, int x, int v) {
#if FEC_UF_RELAXED
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p + x), "r"(v) : "memory");
#else
    asm volatile("st.global.b32 [%0], %1;" ::"l"(p + x), "r"(v) : "memory");
#endif
}
// The root of v by a read-only walk (no writes: callers store the result themselves).
__device__ __forceinline__ int uf_root(const int* parent, int v) {
    int curr = ld_parent(parent, v), next;
    while (uf_above(next = ld_parent(parent, curr), curr)) curr = next;
    return curr;
}

__device__ __forceinline__ int uf_find(int* parent, int v) {
    int curr = ld_parent(parent, v);
    if (curr != v) {
        int prev = v, next;
        while (uf_above(next = ld_parent(parent, curr), curr)) {
            st_parent(parent, prev, next);  // pointer jumping: prev skips to its grandparent
            prev = curr;
            curr = next;
        }
    }
    return curr;
}

__device__ __forceinline__ void uf_unite(int* parent, int a, int b) {
    int ra = uf_find(parent, a), rb = uf_find(parent, b);
    while (ra != rb) {
        if (uf_above(ra, rb)) { int t = ra; ra = rb; rb = t; }
        int old = atomicCAS(parent + ra, ra, rb);  // hook the lower root under the higher one
        if (old == ra) return;
        ra = uf_find(parent, old);
        rb = uf_find(parent, rb);
    }
}

// ---- device-wide exclusive scan (host recursion over tiles) ---------------------------
template <typename T>
int exclusive_scan(const T* in, T* out, int64_t n, T* scratch, cudaStream_t st);  // returns launches
// same, over the first min(n, *ndev) elements (ndev: device int written by an earlier kernel)
template <typename T>
int exclusive_scan_dn(const T* in, T* out, int64_t n, const int* ndev, T* scratch, cudaStream_t st);
size_t scan_scratch_elems(int64_t n);
// single-pass scan on a look-back state zeroed earlier in the call (no memset node); does
// nothing when *skip0 or *skip1 (optional device ints) is nonzero
int exclusive_scan_lb(const uint32_t* in, uint32_t* out, int64_t n, const int* ndev, unsigned long long* state,
                      unsigned int* counter, int max_blocks, const int* skip0, const int* skip1, cudaStream_t st);
int64_t scan_lb_tiles(int64_t n);

// ---- workspace carving -----------------------------------------------------------------
struct Carver {
    char* base;
    size_t off = 0, cap;
    template <typename T>
    T* take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T* p = reinterpret_cast<T*>(base + off);
        off += count * sizeof(T);
        return p;
    }
};

}  // namespace fec
