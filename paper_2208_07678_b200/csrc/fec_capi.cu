// C ABI (include/fec.h) and host orchestration of the FEC sm_100a pipeline.
#include <float.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "fec.h"
#include "fec_kernels.cuh"
#include "fec_slab.cuh"

using namespace fec;

namespace {

thread_local std::string g_err;
thread_local fec_stats_t g_stats;
thread_local bool g_stats_valid = false;
thread_local int g_instrument = 0;
thread_local Meta* g_pinned_meta = nullptr;
thread_local HostBBox* g_host_bbox = nullptr;  // mapped pinned memory (k_bbox_final writes it)
thread_local int g_bbox_seq = 0;
thread_local int g_timing = 0;
thread_local int g_grid_mode = 0;
thread_local int64_t g_item_cap = 0;  // test hook: cap on the queued uncertain pairs (0 = default)

constexpr int kStages = 10;
const char* const kStageNames[kStages] = {"a1_bbox_validate", "a2_bin_keys",       "a3_sort",
                                          "a4_gather_init",   "a5_tables",    "a6a7_union_sparse",
                                          "a6a7_union_dense", "a8_flatten",        "a9_stats",
                                          "a10_relabel"};  // single-GPU path: a8 = separate flatten (sparse-dominated clouds only), a9 = k_flat_stats
struct StageEvents {
    cudaEvent_t ev[kStages + 1] = {};
    bool created = false;
    bool recorded = false;
};
thread_local StageEvents g_ev;

// Records the boundary event `i` (0 = start ... kStages = end) when timing is enabled.
inline void mark(int i, cudaStream_t st) {
    if (!g_timing) return;
    if (!g_ev.created) {
        for (auto& e : g_ev.ev) cudaEventCreate(&e);
        g_ev.created = true;
    }
    cudaEventRecord(g_ev.ev[i], st);
    if (i == kStages) g_ev.recorded = true;
}

constexpr int kMaxBBoxBlocks = 148 * 8;

fec_status_t fail_cuda(cudaError_t e, const char* where) {
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return FEC_ERR_CUDA;
}
#define FEC_CUDA(call)                                   \
    do {                                                 \
        cudaError_t e_ = (call);                         \
        if (e_ != cudaSuccess) return fail_cuda(e_, #call); \
    } while (0)

struct DevInfo {
    int sms = 0;
    int scan_blocks_per_sm = 0;
    int sparse_blocks_per_sm = 0;
    int wfix_blocks_per_sm = 0;
};
DevInfo dev_info() {
    static DevInfo cache[64];
    int d = 0;
    cudaGetDevice(&d);
    DevInfo& di = cache[d & 63];
    if (di.sms == 0) {
        cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, d);
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_scan_union, SCAN_THREADS, 0);
        di.scan_blocks_per_sm = b > 0 ? b : 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_union_sparse, 256, 0);
        di.sparse_blocks_per_sm = b > 0 ? b : 1;
    }
    return di;
}

// dense-grid mode needs 1/4 B per grid cell (occupancy bitmap + word bases + scan)
int64_t dense_cap(int64_t n) { return 32 * n + (int64_t(1) << 26); }
int64_t dense_max(int64_t n) { return n / (SPARSE_MAX + 1) + 16; }
int64_t nodes_max(int64_t n) { return n + 8 * dense_max(n); }
int64_t hash_cap(int64_t n) {
    int64_t c = 1024;
    while (c < 2 * n) c <<= 1;
    return c;
}

// Workspace = common part + max(radix/hash-mode part, dense-grid-mode part).
struct Layout {
    // common
    Meta* meta;
    float* part;
    float4* spts;
    int *parent, *size, *minidx;
    // radix / hash mode
    u64 *keyA, *keyB;
    int *valA, *valB;
    u64* flags;
    u64* scan64;
    uint32_t* counts;
    uint32_t* scan32;
    Tables T;
    int num_tiles;
    // dense-grid mode (per-cell tables indexed by compact id of the occupied cells)
    uint2* cw;          // [W+1] occupancy bitmap words {bits, occupied cells before the word}
    uint32_t* clin;     // [n]   linear cell id of each compact id
    uint32_t* cstart;   // [n+1] counts, then exclusive prefix (cell start)
    int* crec;          // [n]   dense record id of a dense cell
    uint32_t* dscan;    // scan scratch
    uint32_t* slot;     // [n]
    int* sidx;          // [n] input index of each sorted position
    int* dlist;         // dense record -> compact cell id
    uint32_t* dbits;    // [n/32+2] bitmap of dense compact ids
    uint32_t* dwpos;    // [n/32+2] popcount prefix of the bitmap words
    u64* cocc;          // [n]   fine (4x4x4) occupancy mask of each occupied cell
    u64* ccoord;        // [n]   cell coordinates of each occupied cell, 21 bits each
    int* slist;         // [n]   compact ids of the sparse cells (clouds with few of them)
    int* ncomp;         // per dense record: certain-connected components (<= 8)
    u64* dcoord;        // per dense record: cell coordinates, 21 bits each
    uint32_t* oflag;    // per dense record: slots whose pairs overflowed the queue
    u64* cmask;         // per dense record: 8 component masks
    uint32_t *skey0, *skey1;  // key-sort path: linear cell keys (double buffer)
    int *sval0, *sval1;       // key-sort path: input indices (double buffer)
    uint32_t* scounts;        // key-sort path: digit counts per tile
    int4* items;        // queued component pairs (not certain, possibly within reach)
    int4* items2;       // those still apart after all certain unions (split into slices)
    int4* slices2;      // (slice, slices, queued pair) of each items2 entry
    int* idone;         // per queued pair: a slice found a pred-true pair
    int item_cap;
    size_t total;
};

Layout carve(char* base, int64_t n) {
    Layout L{};
    Carver cv{base, 0, 0};
    L.meta = cv.take<Meta>(1);
    L.part = cv.take<float>(6 * kMaxBBoxBlocks);
    L.spts = cv.take<float4>(n);
    // union-find nodes: the n points, then (dense-grid mode) 8 component nodes per dense cell
    L.parent = cv.take<int>(nodes_max(n));
    L.size = cv.take<int>(nodes_max(n));
    L.minidx = cv.take<int>(nodes_max(n));
    const size_t common = (cv.off + 255) & ~size_t(255);
    // radix / hash mode
    Carver a{base, common, 0};
    L.keyA = a.take<u64>(n);
    L.keyB = a.take<u64>(n);
    L.valA = a.take<int>(n);
    L.valB = a.take<int>(n);
    L.flags = a.take<u64>(n + 1);
    L.scan64 = a.take<u64>(scan_scratch_elems(n + 1));
    L.num_tiles = (int)((n + RS_TILE - 1) / RS_TILE);
    L.counts = a.take<uint32_t>((size_t)256 * L.num_tiles);
    L.scan32 = a.take<uint32_t>(scan_scratch_elems((int64_t)256 * L.num_tiles));
    L.T.gstart = a.take<int>(n + 1);
    L.T.goct = a.take<uint8_t>(n);
    L.T.cell_gstart = a.take<int>(n + 1);
    L.T.cell_pc = a.take<u64>(n);
    const int64_t hc = hash_cap(n);
    L.T.hkey = a.take<u64>(hc);
    L.T.hval = a.take<int>(hc);
    L.T.dense = nullptr;
    // dense-grid mode
    const int64_t dc = dense_cap(n);
    const int64_t W = dc / 32 + 1;
    Carver b{base, common, 0};
    L.cw = b.take<uint2>(W + 1);
    L.clin = b.take<uint32_t>(n);
    L.cstart = b.take<uint32_t>(n + 1);
    L.crec = b.take<int>(n);
    L.dscan = b.take<uint32_t>(
        scan_scratch_elems(std::max<int64_t>(std::max<int64_t>(W + 2, n + 1), 256 * ((n + RS_TILE - 1) / RS_TILE))));
    L.slot = b.take<uint32_t>(n);
    L.sidx = b.take<int>(n);
    L.dlist = b.take<int>(dense_max(n));
    L.dbits = b.take<uint32_t>(n / 32 + 2);
    L.dwpos = b.take<uint32_t>(n / 32 + 2);
    L.cocc = b.take<u64>(n);
    L.skey0 = b.take<uint32_t>(n);
    L.skey1 = b.take<uint32_t>(n);
    L.sval0 = b.take<int>(n);
    L.sval1 = b.take<int>(n);
    L.scounts = b.take<uint32_t>((size_t)256 * ((n + RS_TILE - 1) / RS_TILE));
    L.ccoord = b.take<u64>(n);
    L.slist = b.take<int>(n);
    L.ncomp = b.take<int>(dense_max(n));
    L.dcoord = b.take<u64>(dense_max(n));
    L.oflag = b.take<uint32_t>(dense_max(n));
    L.cmask = b.take<u64>((size_t)8 * dense_max(n));
    L.item_cap = (int)std::min<int64_t>(n / 8 + 65536, INT32_MAX / 2);
    L.items = b.take<int4>(L.item_cap);
    L.items2 = b.take<int4>(2 * (size_t)L.item_cap);
    L.slices2 = b.take<int4>(2 * (size_t)L.item_cap);
    L.idone = b.take<int>(L.item_cap);
    L.total = std::max(a.off, b.off) + 256;
    return L;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int ceil_log2(int64_t v) {
    int b = 0;
    while ((int64_t(1) << b) < v) ++b;
    return b;
}

fec_status_t check_args(int64_t n, float d, int64_t mn, int64_t mx, float* t2_out) {
    if (n < 0 || n > INT32_MAX) { g_err = "n out of range [0, INT32_MAX]"; return FEC_ERR_INVALID_ARGUMENT; }
    if (!(d > 0.0f) || !std::isfinite(d)) { g_err = "d_th must be finite and > 0"; return FEC_ERR_INVALID_ARGUMENT; }
    volatile float dv = d;
    const float t2 = dv * dv;  // one fp32 rounding (reading A3)
    if (!std::isfinite(t2) || t2 < FLT_MIN) {
        g_err = "d_th*d_th must be a finite normal fp32 (reading A13)";
        return FEC_ERR_INVALID_ARGUMENT;
    }
    if (mn < 0 || mx < 1 || mn > mx) { g_err = "need 0 <= min_size <= max_size, max_size >= 1"; return FEC_ERR_INVALID_ARGUMENT; }
    *t2_out = t2;
    return FEC_OK;
}

inline unsigned grid_for(int64_t work, int per_block, int cap) {
    int64_t b = (work + per_block - 1) / per_block;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (unsigned)b;
}

// State of a call after a1..a8 (flattened forest over sorted positions), shared by the
// single-GPU tail (a9, a10) and the slab tail (owned-only stats + boundary records).
struct Core {
    Layout L;
    Grid g;
    int node_stats = 0;        // single-GPU tail: dense points' totals accumulated per component node
    const int* val = nullptr;  // local input index of each sorted position
    int launches = 0;
    int passes = 0;
};

// Batch mode (fec_cluster_batch_ws): clouds [off[c], off[c+1]) clustered independently in one
// pipeline; device arrays live in the batch region after the main workspace.
struct BatchArgs {
    int nclouds = 0;
    const int64_t* off_host = nullptr;
    int64_t* off_dev = nullptr;
    float* bb_dev = nullptr;
    double* blo_dev = nullptr;
    int32_t* bz_dev = nullptr;
};
constexpr fec_status_t kNeedPerCloud = 1;  // internal: the combined grid does not fit, run clouds one by one

thread_local void* g_pinned_batch = nullptr;
thread_local size_t g_pinned_batch_bytes = 0;

// a1..a8 on n > 0 points (arguments already checked, pointers validated).
// word bases + compact cell list in one single-pass look-back kernel (k_cscan); the look-back
// state lives in the scan scratch (counter in the first 256 B)
int cell_scan(const Layout& L, int64_t W, const Grid& g, cudaStream_t st) {
    const int64_t nb = (W + 1 + 2047) / 2048;
    unsigned int* counter = reinterpret_cast<unsigned int*>(L.dscan);
    unsigned long long* state = reinterpret_cast<unsigned long long*>(L.dscan + 64);
    cudaMemsetAsync(L.dscan, 0, 256 + (size_t)nb * 8, st);
    pdl(k_cscan, (unsigned)nb, 256, 0, st)(L.cw, W, L.clin, L.cstart, L.cocc, L.ccoord, g, L.meta, state, counter);
    return 1;
}

fec_status_t run_core(const float* pts, int64_t n, float d, float t2, void* ws, cudaStream_t st, Core& C,
                      const BatchArgs* B = nullptr) {
    Layout& L = C.L;
    L = carve(static_cast<char*>(ws), n);
    int launches = 0;
    if (!g_pinned_meta) FEC_CUDA(cudaMallocHost(&g_pinned_meta, sizeof(Meta)));
    const DevInfo di = dev_info();
    const int cap = di.sms * 8;

    // ---- a1: validate + bbox, then the only host synchronisation ----------------------
    mark(0, st);
    FEC_CUDA(cudaMemsetAsync(L.meta, 0, sizeof(Meta), st));
    const int vec4 = (reinterpret_cast<uintptr_t>(pts) & 15u) == 0;
    const unsigned bb_blocks = grid_for(n, 256 * 4, std::min(cap, kMaxBBoxBlocks));
    const float near = (float)(2.0 * (double)d * (1.0 + std::ldexp(1.0, -16)));
    float* bbh = nullptr;  // batch: per-cloud bboxes on the host
    if (!B) {
        pdl(k_bbox_partial, bb_blocks, 256, 0, st)(pts, n, vec4, L.part, &L.meta->nonfinite, near,
                                                  &L.meta->near_pairs);
        if (!g_host_bbox) FEC_CUDA(cudaHostAlloc(&g_host_bbox, sizeof(HostBBox), cudaHostAllocMapped | cudaHostAllocPortable));
        const int seq = ++g_bbox_seq;
        pdl(k_bbox_final, 1, 256, 0, st)(L.part, (int)bb_blocks, L.meta, g_host_bbox, seq);
        launches += 2;
        FEC_CUDA(cudaGetLastError());
        // wait for the record (no stream synchronisation, no copy); if the stream drains
        // without it, a launch failed: the synchronisation reports the error
        volatile int* vs = &g_host_bbox->seq;
        for (int spins = 0; *vs != seq; ++spins) {
            if ((spins & 1023) == 1023 && cudaStreamQuery(st) != cudaErrorNotReady && *vs != seq) {
                FEC_CUDA(cudaStreamSynchronize(st));
                if (*vs != seq) { g_err = "bbox record missing"; return FEC_ERR_CUDA; }
            }
        }
        std::atomic_thread_fence(std::memory_order_acquire);
        for (int k = 0; k < 6; ++k) g_pinned_meta->bbox[k] = g_host_bbox->bbox[k];
        g_pinned_meta->nonfinite = g_host_bbox->nonfinite;
        g_pinned_meta->near_pairs = g_host_bbox->near_pairs;
    } else {
        const size_t need = (size_t)B->nclouds * (6 * sizeof(float) + 3 * sizeof(double) + sizeof(int32_t)) + 64;
        if (g_pinned_batch_bytes < need) {
            if (g_pinned_batch) cudaFreeHost(g_pinned_batch);
            g_pinned_batch = nullptr;
            g_pinned_batch_bytes = 0;
            FEC_CUDA(cudaMallocHost(&g_pinned_batch, need));
            g_pinned_batch_bytes = need;
        }
        bbh = static_cast<float*>(g_pinned_batch);
        FEC_CUDA(cudaMemcpyAsync(B->off_dev, B->off_host, (size_t)(B->nclouds + 1) * sizeof(int64_t),
                                 cudaMemcpyHostToDevice, st));
        pdl(k_bbox_clouds, B->nclouds, 256, 0, st)(pts, B->off_dev, B->bb_dev, &L.meta->nonfinite, near,
                                                  &L.meta->near_pairs);
        ++launches;
        FEC_CUDA(cudaMemcpyAsync(g_pinned_meta, L.meta, sizeof(Meta), cudaMemcpyDeviceToHost, st));
        FEC_CUDA(cudaMemcpyAsync(bbh, B->bb_dev, (size_t)B->nclouds * 6 * sizeof(float), cudaMemcpyDeviceToHost, st));
    }
    if (B) FEC_CUDA(cudaStreamSynchronize(st));
    const Meta hm = *g_pinned_meta;
    if (hm.nonfinite) { g_err = "non-finite coordinate"; return FEC_ERR_NONFINITE; }

    // ---- grid parameters (reading A6): cell c = d(1+2^-16), sub-cell h = c/2 -----------
    Grid g{};
    const double c = (double)d * (1.0 + std::ldexp(1.0, -16));
    g.h = c * 0.5;
    g.inv_h = 1.0 / g.h;
    g.inv_q = 2.0 * g.inv_h;
    int64_t cells_total = 1;
    int key_bits = 3;
    if (!B) {
        for (int a = 0; a < 3; ++a) {
            g.lo[a] = (double)hm.bbox[a];
            // the same double operations as sub_coord() on the device
            const double smax = std::floor(((double)hm.bbox[3 + a] - g.lo[a]) * g.inv_h);
            if (!(smax < 2097152.0)) { g_err = "bbox extent / cell >= 2^20 (reading A14)"; return FEC_ERR_GRID_RANGE; }
            g.dims[a] = (int32_t)(((int64_t)smax >> 1) + 1);
        }
    } else {
        // each cloud: its own origin and cell dims; stacked along z with one empty layer between
        double* blo = reinterpret_cast<double*>(static_cast<char*>(g_pinned_batch) +
                                                ((size_t)B->nclouds * 6 * sizeof(float) + 7) / 8 * 8);
        int32_t* bz = reinterpret_cast<int32_t*>(blo + 3 * B->nclouds);
        int64_t gx = 1, gy = 1, gz = 0;
        for (int cidx = 0; cidx < B->nclouds; ++cidx) {
            const float* bb = bbh + 6 * cidx;
            bz[cidx] = (int32_t)gz;
            if (B->off_host[cidx + 1] == B->off_host[cidx]) {
                blo[3 * cidx] = blo[3 * cidx + 1] = blo[3 * cidx + 2] = 0.0;
                continue;
            }
            int64_t dm[3];
            for (int a = 0; a < 3; ++a) {
                blo[3 * cidx + a] = (double)bb[a];
                const double smax = std::floor(((double)bb[3 + a] - (double)bb[a]) * g.inv_h);
                if (!(smax < 2097152.0)) { g_err = "a cloud's bbox extent / cell >= 2^20 (reading A14)"; return FEC_ERR_GRID_RANGE; }
                dm[a] = ((int64_t)smax >> 1) + 1;
            }
            gx = std::max(gx, dm[0]);
            gy = std::max(gy, dm[1]);
            gz += dm[2] + 1;
        }
        if (gz < 1) gz = 1;
        if (g_grid_mode == 1 || gx * gy * gz > dense_cap(n) || gx * gy * gz >= (int64_t)0xfffffff0ll || gz >= (1 << 20))
            return kNeedPerCloud;
        FEC_CUDA(cudaMemcpyAsync(B->blo_dev, blo, (size_t)B->nclouds * 3 * sizeof(double), cudaMemcpyHostToDevice, st));
        FEC_CUDA(cudaMemcpyAsync(B->bz_dev, bz, (size_t)B->nclouds * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        g.lo[0] = g.lo[1] = g.lo[2] = 0.0;
        g.dims[0] = (int32_t)gx;
        g.dims[1] = (int32_t)gy;
        g.dims[2] = (int32_t)gz;
        g.batch = 1;
        g.nclouds = B->nclouds;
        g.boff = B->off_dev;
        g.blo = B->blo_dev;
        g.bz = B->bz_dev;
    }
    for (int a = 0; a < 3; ++a) {
        g.bits[a] = ceil_log2(g.dims[a]);
        key_bits += g.bits[a];
        cells_total *= g.dims[a];
    }
    g.key_bits = key_bits;
    g.t2 = t2;
    const int64_t hc = hash_cap(n);
    g.hash_mask = (u64)(hc - 1);
    g.dense = (g_grid_mode != 1 && cells_total <= dense_cap(n) && cells_total < (int64_t)0xfffffff0ll) ? 1 : 0;
    int passes = 0;
    FEC_CUDA(cudaMemsetAsync(&L.meta->instrument, 0, sizeof(int), st));
    if (g_instrument) {
        static const int one = 1;
        FEC_CUDA(cudaMemcpyAsync(&L.meta->instrument, &one, sizeof(int), cudaMemcpyHostToDevice, st));
    }
    const unsigned ew = grid_for(n, 256, cap * 4);
    const unsigned ew4 = grid_for((n + 3) / 4, 256, cap * 4);  // kernels taking 4 points per thread
    const int* val = nullptr;
    DenseCtx dctx{};
    bool key_sort = false;

    if (g.dense) {
        FEC_CUDA(ensure_subcell_tables());
        // smallest dimension fastest in the linear cell id (L2 locality of the slow axis)
        int perm[3] = {0, 1, 2};
        for (int i = 0; i < 3; ++i)
            for (int j = i + 1; j < 3; ++j)
                if (g.dims[perm[j]] < g.dims[perm[i]]) std::swap(perm[i], perm[j]);
        for (int i = 0; i < 3; ++i) g.perm[i] = perm[i];
        g.stride[perm[0]] = 1;
        g.stride[perm[1]] = (uint32_t)g.dims[perm[0]];
        g.stride[perm[2]] = (uint32_t)g.dims[perm[0]] * (uint32_t)g.dims[perm[1]];
        g.sdiv[0] = g.stride[perm[2]];
        g.sdiv[1] = g.stride[perm[1]];
        // dense cells get certain-connected components of their fine occupancy (component nodes)
        dctx.spts = L.spts;
        dctx.cstart = L.cstart;
        dctx.dlist = L.dlist;
        dctx.clin = L.clin;
        dctx.cmask = L.cmask;
        dctx.parent = L.parent;
        dctx.items = L.items;
        dctx.item_cap = g_item_cap > 0 ? (int)std::min<int64_t>(g_item_cap, L.item_cap) : L.item_cap;
        dctx.nbase = (int)n;
        dctx.meta = L.meta;
        const int64_t W = (cells_total + 31) / 32;
        const int64_t dwords = n / 32 + 1;
        const unsigned wb = grid_for(dwords + 1, 256, cap * 4);
        // input order: spatially coherent (LiDAR scan order) -> counting sort; shuffled -> key sort
        const double pairs = 3.0 * (double)(n / 4);
        key_sort = g_grid_mode == 2 || (g_grid_mode != 3 && !(vec4 && (double)hm.near_pairs >= 0.5 * pairs));
        FEC_CUDA(cudaMemsetAsync(L.cw, 0, (size_t)(W + 1) * sizeof(uint2), st));
        FEC_CUDA(cudaMemsetAsync(L.dbits, 0, (size_t)(dwords + 1) * 4, st));
        if (!key_sort) {
            // a2: occupancy bitmap -> compact cell ids; counts per cell -> slots, fine occupancy
            mark(1, st);
            pdl(k_cmark, ew, 256, 0, st)(pts, n, g, L.cw);
            launches += 1 + cell_scan(L, W, g, st);
            const unsigned wt = grid_for((n + kWarp * 4 - 1) / (kWarp * 4) * kWarp, 256, cap * 4);  // warp tiles
            pdl(k_dcount2, wt, 256, 0, st)(pts, n, g, L.cw, L.cstart, L.cocc);
            // a3: counting sort = scan (over the occupied cells only) + cursor scatter
            mark(2, st);
            launches += 2 + exclusive_scan_dn<uint32_t>(L.cstart, L.cstart, n + 1, &L.meta->cells1, L.dscan, st);
            pdl(k_ccount, ew, 256, 0, st)(L.cstart, L.dbits, L.slot, L.meta);
            pdl(k_dbits_popc, wb, 256, 0, st)(L.dbits, dwords, L.dwpos);
            launches += 2 + exclusive_scan<uint32_t>(L.dwpos, L.dwpos, dwords + 1, L.dscan, st);
            pdl(k_dbits_list, wb, 256, 0, st)(L.dbits, dwords, L.dwpos, L.dlist, L.crec, L.meta);
            pdl(k_dcomps, grid_for(dense_max(n), 256, cap), 256, 0, st)(g, L.cocc, L.ccoord, L.ncomp, L.size, L.minidx,
                                                                      L.dcoord, L.oflag, dctx);
            pdl(k_dscatter2, wt, 256, 0, st)(pts, n, g, L.cw, L.slot, L.spts);  // slot = per-cell cursors here
            launches += 3;
        } else {
            // a2: linear cell keys, LSD radix sort over their significant bits
            mark(1, st);
            uint32_t* kin = reinterpret_cast<uint32_t*>(L.skey0);
            uint32_t* kout = reinterpret_cast<uint32_t*>(L.skey1);
            int *vin = L.sval0, *vout = L.sval1;
            pdl(k_lkey, ew4, 256, 0, st)(pts, n, g, kin, vin);
            ++launches;
            const int lbits = std::max(1, ceil_log2(cells_total));
            passes = (lbits + 7) / 8;
            const int tiles = (int)((n + RS_TILE - 1) / RS_TILE);
            for (int pp = 0; pp < passes; ++pp) {
                pdl(k_radix_hist32, tiles, RS_THREADS, 0, st)(kin, n, 8 * pp, L.scounts, tiles);
                launches += exclusive_scan<uint32_t>(L.scounts, L.scounts, (int64_t)256 * tiles, L.dscan, st);
                pdl(k_radix_scatter32l, tiles, RS_THREADS, 0, st)(kin, vin, kout, vout, n, 8 * pp, L.scounts, tiles);
                launches += 2;
                std::swap(kin, kout);
                std::swap(vin, vout);
            }
            // a3: cells = runs of equal keys -> compact ids, starts, fine occupancy; gather points
            mark(2, st);
            pdl(k_smark, ew, 256, 0, st)(kin, n, L.cw);
            launches += 1 + cell_scan(L, W, g, st);
            pdl(k_sgather, ew4, 256, 0, st)(pts, kin, vin, n, g, L.cw, L.spts, L.cstart, L.cocc, L.parent, L.sidx,
                                           L.size, L.minidx, L.meta);
            pdl(k_scount, ew, 256, 0, st)(L.cstart, L.dbits, L.meta);
            pdl(k_dbits_popc, wb, 256, 0, st)(L.dbits, dwords, L.dwpos);
            launches += 4 + exclusive_scan<uint32_t>(L.dwpos, L.dwpos, dwords + 1, L.dscan, st);
            pdl(k_dbits_list, wb, 256, 0, st)(L.dbits, dwords, L.dwpos, L.dlist, L.crec, L.meta);
            pdl(k_dcomps, grid_for(dense_max(n), 256, cap), 256, 0, st)(g, L.cocc, L.ccoord, L.ncomp, L.size, L.minidx,
                                                                      L.dcoord, L.oflag, dctx);
            launches += 2;
        }
        // a4: sorted-order init (parents: self, or the point's component node); the key-sort
        // path wrote parents/indices in k_sgather and only re-parents points of dense cells
        mark(3, st);
        if (key_sort)
            pdl(k_dparent, grid_for(dense_max(n) * 32, 256, cap * 8), 256, 0, st)(L.spts, L.cstart, L.dlist, L.ncomp,
                                                                                L.cmask, g, (int)n, L.parent, L.meta,
                                                                                L.sidx, L.size, L.minidx,
                                                                                C.node_stats, n);
        else
            pdl(k_dinit, ew4, 256, 0, st)(L.spts, n, g, L.cw, L.cstart, L.crec, L.ncomp, L.cmask, (int)n, L.parent,
                                         L.size, L.minidx, L.sidx, L.meta, C.node_stats);
        ++launches;
        mark(4, st);
        // a6+a7: sparse-sparse point pairs; dense cells: certain component unions, then the
        // queued uncertain pairs
        mark(5, st);
        pdl(k_union_sparse, di.sms * di.sparse_blocks_per_sm, 256, 0, st)(L.spts, L.cw, L.ccoord, L.cstart, g,
                                                                         L.parent, L.meta, n);
        pdl(k_slist, grid_for(n, 256, cap * 4), 256, 0, st)(L.cstart, L.slist, L.meta, n);
        pdl(k_union_sparse_local, di.sms * di.sparse_blocks_per_sm, 256, 0, st)(L.spts, L.cw, L.ccoord, L.cstart,
                                                                               L.slist, g, L.parent, L.meta, n);
        mark(6, st);
        const unsigned lx = grid_for(dense_max(n), 256, cap);
        pdl(k_dense_link, dim3(lx, 3), 256, 0, st)(g, L.cw, L.crec, L.ncomp, L.dcoord, L.oflag, dctx, 0);
        pdl(k_dense_link, dim3(lx, 24), 256, 0, st)(g, L.cw, L.crec, L.ncomp, L.dcoord, L.oflag, dctx, 3);
        // almost always a no-op (nothing overflowed): a small grid keeps its launch cheap
        pdl(k_dense_overflow, di.sms, 256, 0, st)(g, L.cw, L.crec, L.ncomp, L.dcoord, L.oflag, dctx);
        pdl(k_flatten_nodes, grid_for(8 * dense_max(n), 256, cap * 4), 256, 0, st)(L.parent, (int)n, L.meta);
        pdl(k_dense_filter, grid_for(L.item_cap, 256, cap * 4), 256, 0, st)(g, dctx, L.items2, L.slices2, L.idone);
        pdl(k_dense_items, di.sms * 8, 256, 0, st)(g, dctx, L.items2, L.slices2, L.idone);
        launches += 9;
        if (g_instrument) {
            pdl(k_dense_count, grid_for(dense_max(n), 256, cap), 256, 0, st)(L.ncomp, L.dlist, L.cstart, dctx);
            ++launches;
        }
        mark(7, st);
        val = L.sidx;
    } else {
        // ---- a2: keys ----------------------------------------------------------------------
        mark(1, st);
        pdl(k_keys, ew, 256, 0, st)(pts, n, g, L.keyA, L.valA);
        ++launches;
        mark(2, st);
        // ---- a3: LSD radix sort over the significant key bits -------------------------------
        passes = (key_bits + 7) / 8;
        u64 *kin = L.keyA, *kout = L.keyB;
        int *vin = L.valA, *vout = L.valB;
        for (int p = 0; p < passes; ++p) {
            const int shift = 8 * p;
            pdl(k_radix_hist, L.num_tiles, RS_THREADS, 0, st)(kin, n, shift, L.counts, L.num_tiles);
            launches += exclusive_scan<uint32_t>(L.counts, L.counts, (int64_t)256 * L.num_tiles, L.scan32, st);
            pdl(k_radix_scatter, L.num_tiles, RS_THREADS, 0, st)(kin, vin, kout, vout, n, shift, L.counts,
                                                                L.num_tiles);
            launches += 2;
            std::swap(kin, kout);
            std::swap(vin, vout);
        }
        const u64* key = kin;
        val = vin;
        // ---- a4: gather ----------------------------------------------------------------------
        mark(3, st);
        pdl(k_gather, ew, 256, 0, st)(pts, val, n, L.spts);
        ++launches;
        mark(4, st);
        // ---- a5: group / cell tables -----------------------------------------------------------
        pdl(k_heads, grid_for(n + 1, 256, cap * 4), 256, 0, st)(key, n, L.flags);
        launches += 1 + exclusive_scan<u64>(L.flags, L.flags, n + 1, L.scan64, st);
        FEC_CUDA(cudaMemsetAsync(L.T.hkey, 0xFF, (size_t)hc * 8, st));
        pdl(k_fill_tables, ew, 256, 0, st)(key, L.flags, n, g, L.T, L.meta);
        pdl(k_init_uf, ew, 256, 0, st)(L.flags, L.T.gstart, n, L.parent, L.size, L.minidx);
        launches += 2;
        mark(5, st);
        mark(6, st);
        // ---- a6+a7: neighbour scan + union (persistent warps, dynamic cell counter) -----------
        pdl(k_scan_union, di.sms * di.scan_blocks_per_sm, SCAN_THREADS, 0, st)(L.spts, g, L.T, L.parent, L.meta);
        ++launches;
        mark(7, st);
    }

    C.g = g;
    C.val = val;
    C.launches = launches;
    C.passes = passes;
    return FEC_OK;
}

// Fills g_stats after a successful call (instrumented counters need one read-back).
fec_status_t finish_stats(const Core& C, int64_t n, cudaStream_t st) {
    const Grid& g = C.g;
    const Layout& L = C.L;
    const int launches = C.launches;
    const int passes = C.passes;
    const int key_bits = g.key_bits;
    std::memset(&g_stats, 0, sizeof(g_stats));
    g_stats.n = n;
    g_stats.cells = g_stats.groups = g_stats.components = g_stats.pair_tests = g_stats.group_pairs = -1;
    g_stats.dense_cells = g_stats.dense_points = g_stats.dense_tests = -1;
    g_stats.key_bits = key_bits;
    g_stats.radix_passes = passes;
    g_stats.dense_table = g.dense;
    for (int a = 0; a < 3; ++a) g_stats.dims[a] = g.dims[a];
    g_stats.launches = launches;
    if (g_instrument) {
        FEC_CUDA(cudaMemcpyAsync(g_pinned_meta, L.meta, sizeof(Meta), cudaMemcpyDeviceToHost, st));
        FEC_CUDA(cudaStreamSynchronize(st));
        g_stats.cells = g_pinned_meta->cells;
        g_stats.groups = g.dense ? -1 : g_pinned_meta->groups;
        g_stats.dense_cells = g.dense ? g_pinned_meta->ndense : -1;
        g_stats.dense_points = g.dense ? (int64_t)g_pinned_meta->dense_points : -1;
        g_stats.components = (int64_t)g_pinned_meta->components;
        g_stats.pair_tests = (int64_t)(g_pinned_meta->pair_tests + g_pinned_meta->dense_tests);
        g_stats.dense_tests = g.dense ? (int64_t)g_pinned_meta->dense_tests : -1;
        g_stats.group_pairs = g.dense ? (int64_t)g_pinned_meta->nitems2 : (int64_t)g_pinned_meta->group_pairs;
        if (g_pinned_meta->internal_error) { g_err = "internal invariant failed (component bound)"; return FEC_ERR_CUDA; }
    }
    g_stats_valid = true;
    return FEC_OK;
}

fec_status_t run(const float* pts, int64_t n, float d, int64_t min_size, int64_t max_size, int32_t* labels,
                 void* ws, size_t ws_bytes, cudaStream_t st, const BatchArgs* B = nullptr) {
    g_stats_valid = false;
    g_ev.recorded = false;
    float t2 = 0.f;
    fec_status_t rc = check_args(n, d, min_size, max_size, &t2);
    if (rc != FEC_OK) return rc;
    if (n == 0) {
        std::memset(&g_stats, 0, sizeof(g_stats));
        g_stats_valid = true;
        return FEC_OK;
    }
    if (!pts || !labels || !ws) { g_err = "null pointer"; return FEC_ERR_INVALID_ARGUMENT; }
    if (!is_device_ptr(pts) || !is_device_ptr(labels) || !is_device_ptr(ws)) {
        g_err = "points, labels_out and workspace must be device pointers";
        return FEC_ERR_INVALID_ARGUMENT;
    }
    if (ws_bytes < carve(nullptr, n).total) { g_err = "workspace too small (see fec_workspace_bytes)"; return FEC_ERR_INVALID_ARGUMENT; }
    Core C;
    C.node_stats = 1;
    rc = run_core(pts, n, d, t2, ws, st, C, B);
    if (rc != FEC_OK) return rc;
    const Layout& L = C.L;
    const unsigned ew = grid_for(n, 256, dev_info().sms * 8 * 4);
    // ---- a8+a9 fused (flatten + stats), a10 -----------------------------------------------------
    // one of each pair below returns at once (device-side choice)
    const unsigned wave = grid_for(n, 256, dev_info().sms * 8);
    pdl(k_flatten_if, wave, 256, 0, st)(L.parent, n, L.meta);
    mark(8, st);
    const int dense = C.g.dense;
    // a9 in one launch (k_stats / node tail / k_flat_stats, chosen on the device)
    // (at least two blocks: the node tail splits the grid in halves)
    pdl(k_tail_stats, std::max(ew, 2u), 256, 0, st)(L.parent, C.val, n, L.size, L.minidx, L.meta, dense, L.ncomp,
                                                   L.cstart, L.slist);
    mark(9, st);
    pdl(k_rootlab, wave, 256, 0, st)(L.parent, L.size, L.minidx, n, (long long)min_size, (long long)max_size, L.meta);
    pdl(k_relabel, grid_for((n + 3) / 4, 256, dev_info().sms * 8 * 4), 256, 0, st)(
        L.parent, C.val, L.size, L.minidx, n, (long long)min_size, (long long)max_size, labels, L.meta,
        B ? B->off_dev : nullptr, B ? B->nclouds : 0);
    C.launches += 4;
    mark(10, st);
    FEC_CUDA(cudaGetLastError());
    return finish_stats(C, n, st);
}


// ---- slab (multi-GPU) path ----------------------------------------------------------------
constexpr int64_t kSlabMagic = 0x46454353'4c414231ll;  // "FECSLAB1"
struct SlabState {       // lives in the caller's fec_slab_state_t (host memory)
    int64_t magic;
    int64_t n_local, n_owned, n_first, rec_cap;
    int64_t val_off;     // byte offset of the sorted-position -> local-index array in the workspace
    int64_t pad[2];
};
static_assert(sizeof(SlabState) == sizeof(fec_slab_state_t), "opaque state size");

int64_t slab_hash_cap(int32_t world, int64_t rec_cap) {
    int64_t c = 1024;
    while (c < 2 * (int64_t)world * rec_cap) c <<= 1;
    return c;
}
struct SlabLayout {
    size_t core;  // fec_workspace_bytes(n_local)
    int* ckey;
    int *hkey, *hpar, *gsize, *gmin;
    size_t total;
};
SlabLayout slab_carve(char* base, int64_t n_local, int32_t world, int64_t rec_cap) {
    SlabLayout S{};
    S.core = n_local > 0 ? carve(nullptr, n_local).total : 0;
    Carver cv{base, S.core, 0};
    S.ckey = cv.take<int>(n_local > 0 ? nodes_max(n_local) : 1);
    const int64_t hc = slab_hash_cap(world, rec_cap);
    S.hkey = cv.take<int>(hc);
    S.hpar = cv.take<int>(hc);
    S.gsize = cv.take<int>(hc);
    S.gmin = cv.take<int>(hc);
    S.total = cv.off + 256;
    return S;
}

// Batch region after the main workspace: offsets, per-cloud bboxes, origins, z offsets.
size_t batch_region_bytes(int32_t nclouds) {
    return (((size_t)(nclouds + 1) * 8 + 255) & ~size_t(255)) + (((size_t)nclouds * 24 + 255) & ~size_t(255)) +
           (((size_t)nclouds * 24 + 255) & ~size_t(255)) + (((size_t)nclouds * 4 + 255) & ~size_t(255)) + 256;
}
BatchArgs batch_carve(char* base, int64_t n, int32_t nclouds, const int64_t* off_host) {
    BatchArgs B;
    B.nclouds = nclouds;
    B.off_host = off_host;
    Carver cv{base, n > 0 ? carve(nullptr, n).total : 0, 0};
    B.off_dev = cv.take<int64_t>(nclouds + 1);
    B.bb_dev = cv.take<float>((size_t)6 * nclouds);
    B.blo_dev = cv.take<double>((size_t)3 * nclouds);
    B.bz_dev = cv.take<int32_t>(nclouds);
    return B;
}
}  // namespace

extern "C" {

size_t fec_workspace_bytes(int64_t n) {
    if (n <= 0) return 0;
    return carve(nullptr, n).total;
}

size_t fec_workspace_bytes_host(int64_t n) {
    if (n <= 0) return 0;
    return fec_workspace_bytes(n) + ((size_t)12 * n + 256) + ((size_t)4 * n + 256);
}

fec_status_t fec_cluster_ws(const float* points, int64_t n, float d_th, int64_t min_size, int64_t max_size,
                            int32_t* labels_out, void* workspace, size_t workspace_bytes, void* stream) {
    return run(points, n, d_th, min_size, max_size, labels_out, workspace, workspace_bytes,
               static_cast<cudaStream_t>(stream));
}

fec_status_t fec_cluster(const float* points, int64_t n, float d_th, int64_t min_size, int64_t max_size,
                         int32_t* labels_out) {
    float t2;
    fec_status_t rc = check_args(n, d_th, min_size, max_size, &t2);
    if (rc != FEC_OK || n == 0) return run(points, n, d_th, min_size, max_size, labels_out, nullptr, 0, 0);
    const size_t b = fec_workspace_bytes(n);
    void* ws = nullptr;
    cudaError_t e = cudaMallocAsync(&ws, b, 0);
    if (e != cudaSuccess) {
        cudaGetLastError();
        g_err = std::string("cudaMallocAsync: ") + cudaGetErrorString(e);
        return FEC_ERR_OUT_OF_MEMORY;
    }
    rc = run(points, n, d_th, min_size, max_size, labels_out, ws, b, 0);
    cudaError_t e2 = cudaStreamSynchronize(0);
    cudaFreeAsync(ws, 0);
    cudaStreamSynchronize(0);
    if (rc == FEC_OK && e2 != cudaSuccess) return fail_cuda(e2, "fec_cluster sync");
    return rc;
}

static fec_status_t cluster_host_impl(const float* points_host, int64_t n, float d_th, int64_t min_size,
                                      int64_t max_size, int32_t* labels_host, void* workspace,
                                      size_t workspace_bytes, void* stream, bool sync);

fec_status_t fec_cluster_host(const float* points_host, int64_t n, float d_th, int64_t min_size, int64_t max_size,
                              int32_t* labels_host, void* workspace, size_t workspace_bytes, void* stream) {
    return cluster_host_impl(points_host, n, d_th, min_size, max_size, labels_host, workspace, workspace_bytes,
                             stream, true);
}

fec_status_t fec_cluster_host_async(const float* points_host, int64_t n, float d_th, int64_t min_size,
                                    int64_t max_size, int32_t* labels_host, void* workspace,
                                    size_t workspace_bytes, void* stream) {
    return cluster_host_impl(points_host, n, d_th, min_size, max_size, labels_host, workspace, workspace_bytes,
                             stream, false);
}

static fec_status_t cluster_host_impl(const float* points_host, int64_t n, float d_th, int64_t min_size,
                                      int64_t max_size, int32_t* labels_host, void* workspace,
                                      size_t workspace_bytes, void* stream, bool sync) {
    float t2;
    fec_status_t rc = check_args(n, d_th, min_size, max_size, &t2);
    if (rc != FEC_OK) return rc;
    if (n == 0) return run(nullptr, 0, d_th, min_size, max_size, nullptr, nullptr, 0, 0);
    if (!points_host || !labels_host || !workspace) { g_err = "null pointer"; return FEC_ERR_INVALID_ARGUMENT; }
    if (workspace_bytes < fec_workspace_bytes_host(n)) { g_err = "workspace too small (see fec_workspace_bytes_host)"; return FEC_ERR_INVALID_ARGUMENT; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t main_b = fec_workspace_bytes(n);
    char* base = static_cast<char*>(workspace);
    float* dpts = reinterpret_cast<float*>(base + ((main_b + 255) & ~size_t(255)));
    int32_t* dlab = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(dpts) + (((size_t)12 * n + 255) & ~size_t(255)));
    FEC_CUDA(cudaMemcpyAsync(dpts, points_host, (size_t)12 * n, cudaMemcpyHostToDevice, st));
    rc = run(dpts, n, d_th, min_size, max_size, dlab, workspace, main_b, st);
    if (rc == FEC_OK) FEC_CUDA(cudaMemcpyAsync(labels_host, dlab, (size_t)4 * n, cudaMemcpyDeviceToHost, st));
    if (sync || rc != FEC_OK) FEC_CUDA(cudaStreamSynchronize(st));
    return rc;
}


int64_t fec_slab_record_words(int64_t rec_cap) { return rec_cap < 0 ? -1 : slab_c_off(rec_cap) + 4 * rec_cap; }

size_t fec_slab_workspace_bytes(int64_t n_local, int32_t world, int64_t rec_cap) {
    if (n_local < 0 || world < 1 || rec_cap < 0) return 0;
    return slab_carve(nullptr, n_local, world, rec_cap).total;
}

fec_status_t fec_slab_local(const float* points, const int32_t* gidx, int64_t n_local, int64_t n_owned,
                            int64_t n_first, float d_th, int32_t* records, int64_t rec_cap, void* workspace,
                            size_t workspace_bytes, fec_slab_state_t* state, void* stream) {
    g_stats_valid = false;
    g_ev.recorded = false;
    float t2 = 0.f;
    fec_status_t rc = check_args(n_local, d_th, 1, 1, &t2);
    if (rc != FEC_OK) return rc;
    if (!state) { g_err = "state is NULL"; return FEC_ERR_INVALID_ARGUMENT; }
    std::memset(state, 0, sizeof(*state));
    if (n_first < 0 || n_owned < n_first || n_local < n_owned) {
        g_err = "need 0 <= n_first <= n_owned <= n_local";
        return FEC_ERR_INVALID_ARGUMENT;
    }
    if (rec_cap < n_first + (n_local - n_owned) || rec_cap > (int64_t)(INT32_MAX - SLAB_HDR) / 6) {
        g_err = "rec_cap must be >= n_first + (n_local - n_owned) (boundary points) and < 2^31/6";
        return FEC_ERR_INVALID_ARGUMENT;
    }
    if (!records || !workspace || (n_local > 0 && (!points || !gidx))) { g_err = "null pointer"; return FEC_ERR_INVALID_ARGUMENT; }
    if (!is_device_ptr(records) || !is_device_ptr(workspace) ||
        (n_local > 0 && (!is_device_ptr(points) || !is_device_ptr(gidx)))) {
        g_err = "points, gidx, records and workspace must be device pointers";
        return FEC_ERR_INVALID_ARGUMENT;
    }
    const SlabLayout S = slab_carve(static_cast<char*>(workspace), n_local, 1, 0);
    if (workspace_bytes < S.total) { g_err = "workspace too small (see fec_slab_workspace_bytes)"; return FEC_ERR_INVALID_ARGUMENT; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    FEC_CUDA(cudaMemsetAsync(records, 0, SLAB_HDR * sizeof(int32_t), st));
    SlabState ss{kSlabMagic, n_local, n_owned, n_first, rec_cap, 0, {0, 0}};
    if (n_local == 0) {
        std::memcpy(state, &ss, sizeof(ss));
        std::memset(&g_stats, 0, sizeof(g_stats));
        g_stats_valid = true;
        return FEC_OK;
    }
    Core C;
    rc = run_core(points, n_local, d_th, t2, workspace, st, C);
    if (rc != FEC_OK) return rc;
    const Layout& L = C.L;
    const unsigned ew = grid_for(n_local, 256, dev_info().sms * 8 * 4);
    pdl(k_flatten, ew, 256, 0, st)(L.parent, n_local, L.size, L.minidx);
    mark(8, st);
    ++C.launches;
    FEC_CUDA(cudaMemsetAsync(S.ckey, 0xFF, (size_t)nodes_max(n_local) * 4, st));
    pdl(k_slab_stats, ew, 256, 0, st)(L.parent, C.val, gidx, n_local, (int)n_owned, (int)n_first, L.size, L.minidx,
                                     S.ckey, L.meta);
    mark(9, st);
    pdl(k_slab_pack, grid_for(nodes_max(n_local), 256, dev_info().sms * 8 * 4), 256, 0, st)(
        L.parent, C.val, gidx, n_local, (int)n_owned, (int)n_first, L.size, L.minidx, S.ckey, records, (int)rec_cap,
        L.meta);
    C.launches += 2;
    mark(10, st);
    FEC_CUDA(cudaGetLastError());
    ss.val_off = reinterpret_cast<const char*>(C.val) - static_cast<const char*>(workspace);
    std::memcpy(state, &ss, sizeof(ss));
    return finish_stats(C, n_local, st);
}

fec_status_t fec_slab_merge(const int32_t* all_records, int32_t world, int32_t rank, int64_t min_size,
                            int64_t max_size, int32_t* labels_owned, void* workspace, size_t workspace_bytes,
                            const fec_slab_state_t* state, void* stream) {
    SlabState ss;
    if (!state) { g_err = "state is NULL"; return FEC_ERR_INVALID_ARGUMENT; }
    std::memcpy(&ss, state, sizeof(ss));
    if (ss.magic != kSlabMagic) { g_err = "state was not filled by a successful fec_slab_local"; return FEC_ERR_INVALID_ARGUMENT; }
    if (world < 1 || rank < 0 || rank >= world) { g_err = "need 0 <= rank < world"; return FEC_ERR_INVALID_ARGUMENT; }
    if (min_size < 0 || max_size < 1 || min_size > max_size) { g_err = "need 0 <= min_size <= max_size, max_size >= 1"; return FEC_ERR_INVALID_ARGUMENT; }
    if ((int64_t)world * ss.rec_cap > INT32_MAX / 2) { g_err = "world * rec_cap too large"; return FEC_ERR_INVALID_ARGUMENT; }
    if (!all_records || !workspace || (ss.n_owned > 0 && !labels_owned)) { g_err = "null pointer"; return FEC_ERR_INVALID_ARGUMENT; }
    if (!is_device_ptr(all_records) || !is_device_ptr(workspace) || (ss.n_owned > 0 && !is_device_ptr(labels_owned))) {
        g_err = "all_records, labels_owned and workspace must be device pointers";
        return FEC_ERR_INVALID_ARGUMENT;
    }
    const SlabLayout S = slab_carve(static_cast<char*>(workspace), ss.n_local, world, ss.rec_cap);
    if (workspace_bytes < S.total) { g_err = "workspace too small (see fec_slab_workspace_bytes)"; return FEC_ERR_INVALID_ARGUMENT; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t hc = slab_hash_cap(world, ss.rec_cap);
    const unsigned mask = (unsigned)(hc - 1);
    const int64_t words = fec_slab_record_words(ss.rec_cap);
    const int cap = dev_info().sms * 8 * 4;
    pdl(k_merge_init, grid_for(hc, 256, cap), 256, 0, st)(S.hkey, S.hpar, S.gsize, S.gmin, hc);
    const int64_t total = (int64_t)world * ss.rec_cap;
    if (total > 0) {
        pdl(k_merge_link, grid_for(total, 256, cap), 256, 0, st)(all_records, world, words, (int)ss.rec_cap, S.hkey,
                                                                mask, S.hpar);
        pdl(k_merge_stats, grid_for(total, 256, cap), 256, 0, st)(all_records, world, words, (int)ss.rec_cap, S.hkey,
                                                                 mask, S.hpar, S.gsize, S.gmin);
    }
    if (ss.n_local > 0) {
        const Layout L = carve(static_cast<char*>(workspace), ss.n_local);
        const int* val = reinterpret_cast<const int*>(static_cast<const char*>(workspace) + ss.val_off);
        if (ss.rec_cap > 0)
            pdl(k_merge_resolve, grid_for(ss.rec_cap, 256, cap), 256, 0, st)(all_records + rank * words, (int)ss.rec_cap,
                                                                            S.hkey, mask, S.hpar, S.gsize, S.gmin,
                                                                            L.size, L.minidx);
        pdl(k_slab_relabel, grid_for(ss.n_local, 256, cap), 256, 0, st)(L.parent, val, L.size, L.minidx, ss.n_local,
                                                                       (int)ss.n_owned, (long long)min_size,
                                                                       (long long)max_size, labels_owned);
    }
    FEC_CUDA(cudaGetLastError());
    return FEC_OK;
}


size_t fec_batch_workspace_bytes(int64_t n_total, int32_t nclouds) {
    if (n_total < 0 || nclouds < 1) return 0;
    return (n_total > 0 ? fec_workspace_bytes(n_total) : 0) + batch_region_bytes(nclouds);
}

fec_status_t fec_cluster_batch_ws(const float* points, const int64_t* offsets, int32_t nclouds, float d_th,
                                  int64_t min_size, int64_t max_size, int32_t* labels_out, void* workspace,
                                  size_t workspace_bytes, void* stream) {
    g_stats_valid = false;
    float t2 = 0.f;
    if (nclouds < 1 || !offsets) { g_err = "need nclouds >= 1 and host offsets[nclouds + 1]"; return FEC_ERR_INVALID_ARGUMENT; }
    if (offsets[0] != 0) { g_err = "offsets[0] must be 0"; return FEC_ERR_INVALID_ARGUMENT; }
    for (int32_t c = 0; c < nclouds; ++c)
        if (offsets[c + 1] < offsets[c]) { g_err = "offsets must be non-decreasing"; return FEC_ERR_INVALID_ARGUMENT; }
    const int64_t n = offsets[nclouds];
    fec_status_t rc = check_args(n, d_th, min_size, max_size, &t2);
    if (rc != FEC_OK) return rc;
    if (n == 0) {
        std::memset(&g_stats, 0, sizeof(g_stats));
        g_stats_valid = true;
        return FEC_OK;
    }
    if (!workspace || workspace_bytes < fec_batch_workspace_bytes(n, nclouds)) {
        g_err = "workspace missing or too small (see fec_batch_workspace_bytes)";
        return FEC_ERR_INVALID_ARGUMENT;
    }
    if (!is_device_ptr(workspace)) { g_err = "workspace must be device memory"; return FEC_ERR_INVALID_ARGUMENT; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const BatchArgs B = batch_carve(static_cast<char*>(workspace), n, nclouds, offsets);
    rc = run(points, n, d_th, min_size, max_size, labels_out, workspace, workspace_bytes, st, &B);
    if (rc != kNeedPerCloud) return rc;
    // the stacked grid does not fit the dense mode: cluster the clouds one after another
    for (int32_t c = 0; c < nclouds; ++c) {
        const int64_t a = offsets[c], nc = offsets[c + 1] - offsets[c];
        if (nc == 0) continue;
        rc = run(points + 3 * a, nc, d_th, min_size, max_size, labels_out + a, workspace, workspace_bytes, st);
        if (rc != FEC_OK) return rc;
    }
    return FEC_OK;
}

fec_status_t fec_get_stats(fec_stats_t* out) {
    if (!out) return FEC_ERR_INVALID_ARGUMENT;
    if (!g_stats_valid) { g_err = "no successful call on this thread"; return FEC_ERR_INVALID_ARGUMENT; }
    *out = g_stats;
    return FEC_OK;
}

void fec_set_instrumentation(int enable) { g_instrument = enable ? 1 : 0; }

void fec_set_timing(int enable) { g_timing = enable ? 1 : 0; }

void fec_set_grid_mode(int mode) { g_grid_mode = mode; }

void fec_set_item_cap(int64_t cap) { g_item_cap = cap > 0 ? cap : 0; }

int32_t fec_get_stage_times(float* ms_out, int32_t max_stages) {
    if (!g_ev.recorded) { g_err = "no timed call on this thread (fec_set_timing(1) first)"; return -1; }
    cudaError_t e = cudaEventSynchronize(g_ev.ev[kStages]);
    if (e != cudaSuccess) { g_err = cudaGetErrorString(e); return -1; }
    for (int i = 0; i < kStages && i < max_stages; ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, g_ev.ev[i], g_ev.ev[i + 1]);
        ms_out[i] = ms;
    }
    return kStages;
}

const char* fec_stage_name(int32_t stage) { return (stage >= 0 && stage < kStages) ? kStageNames[stage] : ""; }

const char* fec_status_string(fec_status_t s) {
    switch (s) {
        case FEC_OK: return "FEC_OK";
        case FEC_ERR_INVALID_ARGUMENT: return "FEC_ERR_INVALID_ARGUMENT";
        case FEC_ERR_NONFINITE: return "FEC_ERR_NONFINITE";
        case FEC_ERR_GRID_RANGE: return "FEC_ERR_GRID_RANGE";
        case FEC_ERR_OUT_OF_MEMORY: return "FEC_ERR_OUT_OF_MEMORY";
        case FEC_ERR_CUDA: return "FEC_ERR_CUDA";
        default: return "FEC_ERR_UNKNOWN";
    }
}

const char* fec_last_error(void) { return g_err.c_str(); }
}  // extern "C"

// the other C-ABI translation units (fec_ground.cu) report through the same thread-local slot
void fec::set_last_error(const std::string& msg) { g_err = msg; }
bool fec::timing_enabled() { return g_timing != 0; }
bool fec::pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FEC_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

extern "C" {

const char* fec_version(void) { return "fec-b200 0.1 sm_100a"; }

fec_status_t fec_debug_pred(const float* a, const float* b, int64_t m, float d_th, uint8_t* out, float* d2_out,
                            void* stream) {
    float t2;
    fec_status_t rc = check_args(0, d_th, 1, 1, &t2);
    if (rc != FEC_OK) return rc;
    if (m <= 0) return FEC_OK;
    if (!is_device_ptr(a) || !is_device_ptr(b) || !is_device_ptr(out)) { g_err = "device pointers required"; return FEC_ERR_INVALID_ARGUMENT; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    pdl(k_debug_pred, grid_for(m, 256, 1024), 256, 0, st)(a, b, m, t2, out, d2_out);
    FEC_CUDA(cudaGetLastError());
    FEC_CUDA(cudaStreamSynchronize(st));
    return FEC_OK;
}

}  // extern "C"
