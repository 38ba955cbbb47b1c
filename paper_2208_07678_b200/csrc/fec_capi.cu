// C ABI (include/fec.h) and host orchestration of the FEC sm_100a pipeline.
#include <float.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "fec.h"
#include "fec_kernels.cuh"
#include "fec_slab.cuh"
#include "fec_part.cuh"

using namespace fec;

namespace {

thread_local std::string g_err;
thread_local fec_stats_t g_stats;
thread_local bool g_stats_valid = false;
thread_local int g_instrument = 0;
thread_local int g_timing = 0;
thread_local int g_grid_mode = 0;
thread_local int64_t g_item_cap = 0;     // test hook: cap on the queued uncertain pairs (0 = default)
thread_local size_t g_alloc_extra = 0;   // test hook: extra bytes asked of the allocator (forced OOM)
struct Snapshot {                        // instrumented calls: Meta + Grid copied back (pinned)
    Meta meta;
    Grid grid;
};
thread_local Snapshot* g_snap = nullptr;
thread_local int32_t* g_status_host = nullptr;  // mapped pinned status word of the synchronous calls
thread_local Meta* g_pinned_meta = nullptr;     // batch mode: the per-cloud pass's Meta
thread_local void* g_pinned_batch = nullptr;
thread_local size_t g_pinned_batch_bytes = 0;
thread_local cudaEvent_t g_batch_copied = nullptr;  // batch mode: the pinned buffer's last H2D copy

// A high-priority side stream per device (thread-local) for latency-bound kernels that can run
// concurrently with bandwidth-bound ones of the same call (fork/join through events: also
// captured into a graph when the caller's stream is being captured).
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr, fork2 = nullptr;
};
// FEC_FULL_SCATTER=1 scatters every point in phase 0 (A/B measurements, debugging)
bool full_scatter() {
    static const bool v = [] {
        const char* e = std::getenv("FEC_FULL_SCATTER");
        return e && e[0] == '1';
    }();
    return v;
}
thread_local SideStream g_side[64];
thread_local int g_side_off = -1;  // FEC_SIDE_STREAM=0 turns the fork off (A/B measurements)
fec_status_t side_stream(SideStream** out) {
    if (g_side_off < 0) {
        const char* e = std::getenv("FEC_SIDE_STREAM");
        g_side_off = (e && e[0] == '0') ? 1 : 0;
    }
    *out = nullptr;
    if (g_side_off) return FEC_OK;
    int d = 0;
    cudaGetDevice(&d);
    SideStream& ss = g_side[d & 63];
    if (!ss.s) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if (cudaStreamCreateWithPriority(&ss.s, cudaStreamNonBlocking, hi) != cudaSuccess ||
            cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ss.fork2, cudaEventDisableTiming) != cudaSuccess) {
            g_err = "side stream creation failed";
            return FEC_ERR_CUDA;
        }
    }
    *out = &ss;
    return FEC_OK;
}

constexpr int kStages = 10;
const char* const kStageNames[kStages] = {"a1_bbox_validate", "a2_bin_keys",       "a3_sort",
                                          "a4_gather_init",   "a5_tables",    "a6a7_union_sparse",
                                          "a6a7_union_dense", "a8_flatten",        "a9_stats",
                                          "a10_relabel"};  // a8 = flatten (sparse-dominated clouds), a9 = k_tail_stats
struct StageEvents {
    cudaEvent_t ev[kStages + 1] = {};
    cudaEvent_t sub[2] = {};  // partial scatter phase 1: a4 work enqueued inside the a6a7 interval
    bool created = false;
    bool recorded = false;
    bool sub_recorded = false;
};
thread_local StageEvents g_ev;

// Records the boundary event `i` (0 = start ... kStages = end) when timing is enabled.
inline void mark(int i, cudaStream_t st) {
    if (!g_timing) return;
    if (!g_ev.created) {
        for (auto& e : g_ev.ev) cudaEventCreate(&e);
        for (auto& e : g_ev.sub) cudaEventCreate(&e);
        g_ev.created = true;
    }
    cudaEventRecord(g_ev.ev[i], st);
    if (i == 0) g_ev.sub_recorded = false;
    if (i == kStages) g_ev.recorded = true;
}
// Sub-interval j (0 = begin, 1 = end) of a4 work enqueued later (counted to a4, not a6a7).
inline void mark_sub(int j, cudaStream_t st) {
    if (!g_timing || !g_ev.created) return;
    cudaEventRecord(g_ev.sub[j], st);
    if (j == 1) g_ev.sub_recorded = true;
}

constexpr int kMaxBBoxBlocks = 148 * 8;
constexpr int64_t kSmallN = int64_t(1) << 17;
constexpr int64_t kRelabelBucketN = int64_t(1) << 22;  // from here: the two-pass bucketed relabel
  // below: the counting path only (no key-sort launches)

fec_status_t fail_cuda(cudaError_t e, const char* where) {
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return FEC_ERR_CUDA;
}
#define FEC_CUDA(call)                                   \
    do {                                                 \
        cudaError_t e_ = (call);                         \
        if (e_ != cudaSuccess) return fail_cuda(e_, #call); \
    } while (0)
#define FEC_CUDA_RC(call)                                \
    do {                                                 \
        fec_status_t r_ = (call);                        \
        if (r_ != FEC_OK) return r_;                     \
    } while (0)

struct DevInfo {
    int sms = 0;
    int sparse_blocks_per_sm = 0;
};
DevInfo dev_info() {
    static DevInfo cache[64];
    int d = 0;
    cudaGetDevice(&d);
    DevInfo& di = cache[d & 63];
    if (di.sms == 0) {
        int sms = 0, b = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_union_sparse, 256, 0);
        di.sparse_blocks_per_sm = b > 0 ? b : 1;
        di.sms = sms > 0 ? sms : 148;
    }
    return di;
}

// bitmap mode needs 1/4 B per grid cell (occupancy bits + word bases)
constexpr int64_t dense_cap(int64_t n) { return 32 * n + (int64_t(1) << 26); }
constexpr int64_t dense_max(int64_t n) { return n / (SPARSE_MAX + 1) + 16; }
// dense-record capacity rounded to a power of two (the node-id permutation, node_of)
constexpr int64_t rec_pow2(int64_t n) {
    int64_t r = 1;
    while (r < dense_max(n)) r <<= 1;
    return r;
}
constexpr int64_t nodes_max(int64_t n) { return n + 8 * rec_pow2(n); }
// the largest n whose node ids (nodes_max) fit in int32 (node_of, union-find)
constexpr int64_t max_points() {
    int64_t lo = 0, hi = INT32_MAX;
    while (hi - lo > 1) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (nodes_max(mid) < (int64_t)INT32_MAX) lo = mid;
        else hi = mid;
    }
    return lo;
}
int64_t hash_slots(int64_t n) {  // hash mode: a power of two >= 2n (load factor <= 1/2)
    int64_t c = 1024;
    while (c < 2 * n) c <<= 1;
    return c;
}
constexpr int CS_TILE_WORDS = 2048;  // k_cscan tile (fec_dense.cu)

// One linear carve of the workspace (fec_workspace_bytes = its total).
struct Layout {
    Meta* meta;
    Grid* grid;
    float* part;
    float4* spts;
    int *parent, *size, *minidx;   // union-find nodes: n points + 8 per dense cell
    // arena zeroed by k_zero every call: counters, look-back states, histograms, dense bits
    uint32_t* arena;
    int64_t arena_words;
    unsigned int* ctr;             // [1] scan A, [2] scan B, [4..7] onesweep passes
    unsigned long long* sa_state;  // cell starts scan
    unsigned long long* sb_state;  // dense-bits popcount scan
    uint32_t* ghist;               // onesweep: [4][256] digit histograms
    uint32_t* dbits;               // [n/32+2] bitmap of dense compact ids
    uint32_t* cneed1;              // [n/32+2] partial scatter phase 1: cells a queued item reads
    unsigned int* rlcur;           // [RL_MAX_BUCKETS] bucketed relabel: per-bucket cursors
    int64_t cs_tiles;              // k_cscan tiles (worst case over both cell-index modes)
    uint32_t* ctile;               // [cs_tiles] occupied cells per k_cscan tile, then their prefix
    uint2* cw;                     // occupancy words {bits, occupied cells before the word}
    u64* hkey;                     // hash mode: packed cell coordinates per slot
    int64_t slots;
    uint32_t* clin;     // [n]   cell handle of each compact id
    uint32_t* cstart;   // [n+1] counts, then exclusive prefix (cell start)
    int* crec;          // [n]   dense record id of a dense cell
    uint32_t* slot;     // [n]   per-cell scatter cursors
    int* sidx;          // [n]   input index of each sorted position
    uint32_t* pcode;    // [n]   counting path: compact cell id << 6 | fine sub-cell per input point
    int* dlist;         // dense record -> compact cell id
    uint32_t* dwpos;    // [n/32+2] popcount prefix of the dense bits
    uint32_t* cneed0;   // [n/32+2] partial scatter phase 0: sparse and multi-component cells
    u64* cocc;          // [n]   fine (4x4x4) occupancy mask of each occupied cell
    int* cmin;          // [n]   counting path: smallest input index in each occupied cell
    u64* ccoord;        // [n]   cell coordinates of each occupied cell, 21 bits each
    int* slist;         // [n]   compact ids of the sparse cells
    int* ncomp;         // per dense record: certain-connected components (<= 8)
    u64* dcoord;        // per dense record: cell coordinates
    uint32_t* oflag;    // per dense record: slots whose pairs overflowed the queue
    u64* cmask;         // per dense record: 8 component masks
    uint4* litems;            // dense link items (k_dcomps -> k_dense_link), aliasing the sort buffers
    int lhalf;                // capacity of each of the two item lists
    uint32_t *skey0, *skey1;  // key-sort path: linear cell keys (double buffer)
    int *sval0, *sval1;       // key-sort path: input indices (double buffer)
    uint32_t* os_state;       // onesweep look-back: 2 x tiles x 256
    int64_t os_tiles;
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
    L.grid = cv.take<Grid>(1);
    L.part = cv.take<float>(6 * kMaxBBoxBlocks);
    L.spts = cv.take<float4>(n);
    L.parent = cv.take<int>(nodes_max(n));
    L.size = cv.take<int>(nodes_max(n));
    L.minidx = cv.take<int>(nodes_max(n));
    L.slots = hash_slots(n);
    const int64_t w_max = std::max<int64_t>((dense_cap(n) + 31) / 32, L.slots / 32);
    L.cs_tiles = (w_max + 1 + CS_TILE_WORDS - 1) / CS_TILE_WORDS;
    const int64_t dwords = n / 32 + 2;
    // arena (u32 words, each part 256-B aligned)
    Carver ar{base, 0, 0};
    ar.off = (cv.off + 255) & ~size_t(255);
    const size_t a0 = ar.off;
    L.arena = reinterpret_cast<uint32_t*>(base + a0);
    L.ctr = ar.take<unsigned int>(64);
    L.sa_state = ar.take<unsigned long long>(scan_lb_tiles(n + 1) + 32);
    L.sb_state = ar.take<unsigned long long>(scan_lb_tiles(dwords + 1) + 32);
    L.ghist = ar.take<uint32_t>(4 * 256);
    L.dbits = ar.take<uint32_t>(dwords + 1);
    L.cneed1 = ar.take<uint32_t>(dwords + 1);
    L.rlcur = ar.take<unsigned int>(n >= kRelabelBucketN ? (size_t)RL_CUR_STRIDE * ((n >> RL_SHIFT) + 1) : 1);
    ar.off = (ar.off + 255) & ~size_t(255);
    L.arena_words = (int64_t)((ar.off - a0) / 4);
    cv.off = ar.off;
    L.cw = cv.take<uint2>(w_max + 4);
    L.ctile = cv.take<uint32_t>(L.cs_tiles + 1);
    L.hkey = cv.take<u64>(L.slots);
    L.clin = cv.take<uint32_t>(n);
    L.cstart = cv.take<uint32_t>(n + 1);
    L.crec = cv.take<int>(n);
    L.slot = cv.take<uint32_t>(n);
    L.sidx = cv.take<int>(n);
    L.pcode = cv.take<uint32_t>(n);
    L.dlist = cv.take<int>(dense_max(n));
    L.dwpos = cv.take<uint32_t>(dwords + 1);
    L.cneed0 = cv.take<uint32_t>(dwords + 1);
    L.cocc = cv.take<u64>(n);
    L.cmin = cv.take<int>(n);
    L.ccoord = cv.take<u64>(n);
    L.slist = cv.take<int>(n);
    L.ncomp = cv.take<int>(dense_max(n));
    L.dcoord = cv.take<u64>(dense_max(n));
    L.oflag = cv.take<uint32_t>(dense_max(n));
    L.cmask = cv.take<u64>((size_t)8 * dense_max(n));
    // key-sort buffers; after binning the same bytes hold the dense link items (2 x n/2 uint4)
    const int64_t n64 = (n + 63) & ~int64_t(63);  // each buffer 256-B aligned (vector stores)
    char* sortbuf = cv.take<char>((size_t)16 * n64 + 1024);
    L.skey0 = reinterpret_cast<uint32_t*>(sortbuf);
    L.skey1 = L.skey0 + n64;
    L.sval0 = reinterpret_cast<int*>(L.skey1 + n64);
    L.sval1 = L.sval0 + n64;
    L.litems = reinterpret_cast<uint4*>(sortbuf);
    L.lhalf = (int)std::min<int64_t>(n64 / 2, INT32_MAX / 2);
    L.os_tiles = (n + RS_TILE - 1) / RS_TILE;
    L.os_state = cv.take<uint32_t>((size_t)2 * L.os_tiles * 256);
    L.item_cap = (int)std::min<int64_t>(n / 8 + 65536, INT32_MAX / 2);
    L.items = cv.take<int4>(L.item_cap);
    L.items2 = cv.take<int4>(2 * (size_t)L.item_cap);
    L.slices2 = cv.take<int4>(2 * (size_t)L.item_cap);
    L.idone = cv.take<int>(L.item_cap);
    L.total = cv.off + 256;
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

// Bound on n: the node ids (n points + 8 per record slot of a power-of-two record capacity)
// must fit in int32.
constexpr int64_t kMaxN = max_points();

fec_status_t check_args(int64_t n, float d, int64_t mn, int64_t mx, float* t2_out) {
    if (n < 0 || n > kMaxN) {
        g_err = "n out of range [0, " + std::to_string(kMaxN) + "] (int32 union-find node ids)";
        return FEC_ERR_INVALID_ARGUMENT;
    }
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

const char* device_status_text(int32_t s) {
    switch (s) {
        case FEC_ERR_NONFINITE: return "non-finite coordinate (reading A12)";
        case FEC_ERR_GRID_RANGE: return "bbox extent / cell >= 2^20 on an axis (reading A14)";
        default: return "device-side error";
    }
}

fec_status_t ensure_status_word() {
    if (!g_status_host) {
        FEC_CUDA(cudaHostAlloc(&g_status_host, sizeof(int32_t), cudaHostAllocMapped | cudaHostAllocPortable));
        *g_status_host = 0;
    }
    return FEC_OK;
}

// Synchronous forms: wait for the stream, then report what the device found.
fec_status_t wait_status(cudaStream_t st, const int32_t* status_host) {
    FEC_CUDA(cudaStreamSynchronize(st));
    const int32_t s = *reinterpret_cast<const volatile int32_t*>(status_host);
    if (s != FEC_OK) {
        g_err = device_status_text(s);
        return s;
    }
    return FEC_OK;
}

// State of a call after a1..a8 (forest over sorted positions), shared by the single-GPU tail
// (a9, a10) and the slab tail (owned-only stats + boundary records).
struct Core {
    Layout L;
    int node_stats = 0;        // single-GPU tail: dense points' totals accumulated per component node
    const int* val = nullptr;  // local input index of each sorted position
    int launches = 0;
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
constexpr fec_status_t kNeedPerCloud = 1;  // internal: the stacked grid cannot be indexed, run clouds one by one

// Batch mode: per-cloud bboxes on the device, then the grid planned on the HOST (the clouds'
// origins and z offsets) and uploaded; one host synchronisation.
fec_status_t plan_batch(const float* pts, int64_t n, const Grid& g0, const Layout& L, const BatchArgs* B,
                        float near, int vec4, cudaStream_t st, bool& key_sort) {
    const size_t need = (size_t)B->nclouds * (6 * sizeof(float) + 3 * sizeof(double) + sizeof(int32_t)) + 64;
    if (!g_batch_copied) FEC_CUDA(cudaEventCreateWithFlags(&g_batch_copied, cudaEventDisableTiming));
    if (g_pinned_batch) FEC_CUDA(cudaEventSynchronize(g_batch_copied));  // the previous call's H2D copies are done
    if (g_pinned_batch_bytes < need) {
        if (g_pinned_batch) cudaFreeHost(g_pinned_batch);
        g_pinned_batch = nullptr;
        g_pinned_batch_bytes = 0;
        FEC_CUDA(cudaMallocHost(&g_pinned_batch, need));
        g_pinned_batch_bytes = need;
    }
    if (!g_pinned_meta) FEC_CUDA(cudaMallocHost(&g_pinned_meta, sizeof(Meta)));
    float* bbh = static_cast<float*>(g_pinned_batch);
    FEC_CUDA(cudaMemcpyAsync(B->off_dev, B->off_host, (size_t)(B->nclouds + 1) * sizeof(int64_t),
                             cudaMemcpyHostToDevice, st));
    pdl(k_bbox_clouds, B->nclouds, 256, 0, st)(pts, B->off_dev, B->bb_dev, &L.meta->nonfinite, near,
                                              &L.meta->near_pairs);
    FEC_CUDA(cudaMemcpyAsync(g_pinned_meta, L.meta, sizeof(Meta), cudaMemcpyDeviceToHost, st));
    FEC_CUDA(cudaMemcpyAsync(bbh, B->bb_dev, (size_t)B->nclouds * 6 * sizeof(float), cudaMemcpyDeviceToHost, st));
    FEC_CUDA(cudaStreamSynchronize(st));
    const Meta hm = *g_pinned_meta;
    if (hm.nonfinite) { g_err = "non-finite coordinate"; return FEC_ERR_NONFINITE; }
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
            const double smax = std::floor(((double)bb[3 + a] - (double)bb[a]) * g0.inv_h);
            if (!(smax < 2097152.0)) { g_err = "a cloud's bbox extent / cell >= 2^20 (reading A14)"; return FEC_ERR_GRID_RANGE; }
            dm[a] = ((int64_t)smax >> 1) + 1;
        }
        gx = std::max(gx, dm[0]);
        gy = std::max(gy, dm[1]);
        gz += dm[2] + 1;
    }
    if (gz < 1) gz = 1;
    if (gz >= (1 << 21)) return kNeedPerCloud;  // packed cell coordinates hold 21 bits per axis
    Grid g = g0;
    g.dims[0] = (int32_t)gx;
    g.dims[1] = (int32_t)gy;
    g.dims[2] = (int32_t)gz;
    const int64_t cells = gx * gy * gz;
    g.cells_total = cells;
    g.hashed = (g_grid_mode == 1 || cells > dense_cap(n) || cells >= (int64_t)0xfffffff0ll) ? 1 : 0;
    if (!g.hashed) {
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
        g.words = (cells + 31) / 32;
        g.key_bits = std::max(1, ceil_log2(cells));
    } else {
        g.words = ((int64_t)g.hmask + 1) / 32;
    }
    const double pairs = 3.0 * (double)(n / 4);
    const bool coherent = vec4 && (double)hm.near_pairs >= 0.5 * pairs;
    key_sort = !g.hashed && (g_grid_mode == 2 || (g_grid_mode != 3 && !coherent));
    g.key_sort = key_sort ? 1 : 0;
    g.passes = key_sort ? (g.key_bits + 7) / 8 : 0;
    g.batch = 1;
    g.nclouds = B->nclouds;
    g.boff = B->off_dev;
    g.blo = B->blo_dev;
    g.bz = B->bz_dev;
    FEC_CUDA(cudaMemcpyAsync(B->blo_dev, blo, (size_t)B->nclouds * 3 * sizeof(double), cudaMemcpyHostToDevice, st));
    FEC_CUDA(cudaMemcpyAsync(B->bz_dev, bz, (size_t)B->nclouds * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    FEC_CUDA(cudaMemcpyAsync(L.grid, &g, sizeof(Grid), cudaMemcpyHostToDevice, st));  // pageable: staged now
    static const int one = 1;
    if (g_instrument) FEC_CUDA(cudaMemcpyAsync(&L.meta->instrument, &one, sizeof(int), cudaMemcpyHostToDevice, st));
    FEC_CUDA(cudaEventRecord(g_batch_copied, st));
    return FEC_OK;
}

// a1..a8 on n > 0 points (arguments already checked, pointers validated).  No host
// synchronisation (single cloud): a1's last block plans the grid on the device and every
// later kernel reads it there; kernels of a path the plan did not choose return at once.
fec_status_t run_core(const float* pts, int64_t n, float d, float t2, void* ws, cudaStream_t st, Core& C,
                      const BatchArgs* B = nullptr, int32_t* status_dev = nullptr) {
    Layout& L = C.L;
    L = carve(static_cast<char*>(ws), n);
    int launches = 0;
    const DevInfo di = dev_info();
    const int cap = di.sms * 8;
    FEC_CUDA(ensure_subcell_tables());

    // ---- a1: validate + bbox + device-side plan ---------------------------------------------
    mark(0, st);
    FEC_CUDA(cudaMemsetAsync(L.meta, 0, sizeof(Meta), st));
    const int vec4 = (reinterpret_cast<uintptr_t>(pts) & 15u) == 0;
    const unsigned bb_blocks = grid_for(n, 256 * 4, std::min(cap, kMaxBBoxBlocks));
    const float near = (float)(2.0 * (double)d * (1.0 + std::ldexp(1.0, -16)));
    Grid g0{};
    const double c = (double)d * (1.0 + std::ldexp(1.0, -16));  // reading A6: cell edge
    g0.h = c * 0.5;
    g0.inv_h = 1.0 / g0.h;
    g0.inv_q = 2.0 * g0.inv_h;
    g0.t2 = t2;
    g0.hmask = (uint32_t)(L.slots - 1);
    g0.hkey = L.hkey;
    g0.rmask = (uint32_t)(rec_pow2(n) - 1);
    bool key_path = g_grid_mode == 2 || (g_grid_mode == 0 && n > kSmallN);
    if (!B) {
        PlanArgs a{};
        a.g0 = g0;
        a.n = n;
        a.dense_cap = dense_cap(n);
        a.grid_mode = g_grid_mode;
        a.key_path = key_path ? 1 : 0;
        a.vec4 = vec4;
        a.instrument = g_instrument;
        a.near = near;
        a.status_dev = status_dev;
        pdl(k_bbox, bb_blocks, 256, 0, st)(pts, a, L.part, L.meta, L.grid);
        ++launches;
    } else {
        bool ks = false;
        fec_status_t rc = plan_batch(pts, n, g0, L, B, near, vec4, st, ks);
        if (rc != FEC_OK) return rc;
        key_path = ks;
        ++launches;
    }
    const Grid* gp = L.grid;
    const int* gstatus = &L.grid->status;
    const int* gkeysort = &L.grid->key_sort;
    // (small clouds: a small grid -- the device-sized words are few and launch latency dominates)
    const bool small = n <= kSmallN;
    const int local_only = small ? 1 : 0;  // sparse cells: always the compact list + k_union_sparse_local
    pdl(k_zero, small ? 64 : di.sms * 4, 256, 0, st)(gp, L.cw, L.hkey, L.slots, L.arena, L.arena_words);
    ++launches;

    const unsigned ew = grid_for(n, 256, cap * 4);
    // k_dinit (4 points per thread, grid-stride): one full-occupancy wave -- on node-tail clouds the
    // device plan turns it into a no-op, and a 4-wave grid of returning blocks cost ~11 us there
    const unsigned ew4 = grid_for((n + 3) / 4, 256, cap);
    const int64_t dwords = n / 32 + 1;
    const unsigned wb = grid_for(dwords + 1, 256, cap * 4);
    const unsigned wt = grid_for((n + kWarp * 4 - 1) / (kWarp * 4) * kWarp, 256, cap * 4);  // warp tiles
    const unsigned cs_blocks = (unsigned)std::min<int64_t>(L.cs_tiles, small ? 32 : di.sms * 8);
    DenseCtx dctx{};
    dctx.spts = L.spts;
    dctx.cstart = L.cstart;
    dctx.dlist = L.dlist;
    dctx.clin = L.clin;
    dctx.cmask = L.cmask;
    dctx.parent = L.parent;
    dctx.items = L.items;
    dctx.item_cap = g_item_cap > 0 ? (int)std::min<int64_t>(g_item_cap, L.item_cap) : L.item_cap;
    dctx.nbase = (int)n;
    dctx.rmask = (uint32_t)(rec_pow2(n) - 1);
    dctx.meta = L.meta;
    dctx.cneed0 = L.cneed0;
    dctx.cneed1 = L.cneed1;
    // single cloud: the counting path is always enqueued (hash mode has no key sort); batch
    // mode planned on the host enqueues only the chosen path
    const bool count_path = !B || !key_path;

    // ---- a2/a3: binning (counting sort for coherent input, key sort for shuffled input) -------
    mark(1, st);
    if (key_path) {
        pdl(k_lkey, grid_for((n + 3) / 4, 256, di.sms * 4), 256, 0, st)(pts, n, gp, L.skey0, L.sval0, L.ghist, L.os_state, L.os_tiles * 256);
        ++launches;
        for (int pass = 0; pass < 4; ++pass) {  // passes beyond the planned count return at once
            pdl(k_onesweep, (unsigned)std::min<int64_t>(L.os_tiles, di.sms * 3), RS_THREADS, 0, st)(gp, pass, L.skey0, L.sval0, L.skey1, L.sval1, n,
                                                                    L.ghist, L.os_state, L.os_tiles, L.ctr + 4);
            ++launches;
        }
    }
    mark(2, st);
    if (count_path) {
        pdl(k_cmark, ew, 256, 0, st)(pts, n, gp, L.cw);
        ++launches;
    }
    if (key_path) {
        pdl(k_smark, grid_for(n, 256, di.sms * 4), 256, 0, st)(L.skey0, L.skey1, n, L.cw, gp);
        ++launches;
    }
    pdl(k_cpop, cs_blocks, 256, 0, st)(L.cw, L.ctile, gp);
    pdl(k_tscan, 1, 1024, 0, st)(L.ctile, gp, L.meta, L.cstart);
    pdl(k_cscan, cs_blocks, 256, 0, st)(L.cw, gp, L.ctile, L.clin, L.cstart, L.cocc, L.cmin, L.ccoord);
    launches += 3;
    if (count_path) {
        pdl(k_dcount2, wt, 256, 0, st)(pts, n, gp, L.cw, L.cstart, L.cocc, L.cmin, L.pcode, L.meta);
        ++launches;
    }
    if (key_path) {
        pdl(k_sgather, grid_for((n + 3) / 4, 256, di.sms * 8), 256, 0, st)(pts, L.skey0, L.sval0, L.skey1, L.sval1, n, gp, L.cw, L.spts, L.cstart, L.cocc,
                                       L.parent, L.sidx, L.size, L.minidx, L.meta);
        ++launches;
    }
    // cell starts + scatter cursors + dense records (dlist, crec) in one scan over the cells
    {
        const unsigned cl_blocks = (unsigned)std::min<int64_t>(scan_lb_tiles(n + 1), small ? 32 : cap);
        pdl(k_cellred, cl_blocks, 256, 0, st)(L.cstart, L.meta, gp, L.sa_state);
        pdl(k_celltscan, 1, 1024, 0, st)(L.sa_state, L.meta, gp, L.cstart);
        pdl(k_cellscan, cl_blocks, 256, 0, st)(L.cstart, L.slot, L.dlist, L.crec, L.cneed0, L.meta, gp, L.sa_state,
                                               L.slist, n, local_only, C.node_stats ? 0 : 1, L.parent, L.size,
                                               L.minidx);
        launches += 3;
    }
    // dense records: their components and nodes
    pdl(k_dcomps, grid_for(dense_max(n), 256, cap), 256, 0, st)(gp, L.cw, L.crec, L.cocc, L.ccoord, L.ncomp, L.size,
                                                              L.minidx, L.dcoord, L.oflag, dctx, L.litems, L.lhalf,
                                                              L.cmin, L.sidx, C.node_stats);
    ++launches;
    // the dense-dense certain unions need no point: they run on the side stream while the
    // points are scattered and initialised
    SideStream* side = nullptr;
    if (!small) FEC_CUDA_RC(side_stream(&side));  // (small clouds: the fork/join would cost more)
    if (side) {
        FEC_CUDA(cudaEventRecord(side->fork, st));
        FEC_CUDA(cudaStreamWaitEvent(side->s, side->fork, 0));
        pdl(k_dense_link, grid_for(dense_max(n) * 4, 256, di.sms * 8), 256, 0, side->s)(
            gp, L.crec, L.ncomp, L.oflag, dctx, L.litems, L.lhalf, 1, L.cw, L.dcoord);
        ++launches;
    }
    // ---- a4: sorted-order init (counting path: scatter + init; key path: dense re-parenting)
    mark(3, st);
    if (count_path) {
        // slot = per-cell cursors here
        pdl(k_dscatter, wt, 256, 0, st)(pts, n, gp, L.cw, L.slot, L.spts, L.pcode, L.meta, L.cneed0, L.cneed1, 0,
                                        C.node_stats && !full_scatter(), dctx.item_cap);
        pdl(k_dinit, ew4, 256, 0, st)(L.spts, n, gp, L.cw, L.crec, L.cmask, (int)n, L.parent, L.size, L.minidx,
                                     L.sidx, L.meta, C.node_stats ? 0 : 1);
        ++launches;
        ++launches;
    }
    // both paths: points of dense cells under their component nodes + node statistics
    pdl(k_dparent, grid_for(dense_max(n) * 32, 256, di.sms * 8), 256, 0, st)(L.spts, L.cstart, L.dlist, L.ncomp,
                                                                        L.cmask, gp, (int)n, L.parent, L.meta,
                                                                        L.sidx, L.size, L.minidx, C.node_stats, n);
    ++launches;
    mark(4, st);
    // ---- a6+a7: sparse-sparse point pairs; dense cells: certain component unions, then the
    // queued uncertain pairs
    mark(5, st);
    // the sparse-cell unions and the dense records' sparse-neighbour links are independent
    // (unions commute): with a side stream the former run there, concurrently with the latter
    // (both are latency-bound chains of dependent loads)
    cudaStream_t us = st;
    if (side) {
        FEC_CUDA(cudaEventRecord(side->fork2, st));
        FEC_CUDA(cudaStreamWaitEvent(side->s, side->fork2, 0));
        us = side->s;
    }
    if (!local_only)
        pdl(k_union_sparse, di.sms * di.sparse_blocks_per_sm, 256, 0, us)(L.spts, L.cw, L.ccoord, L.cstart, gp,
                                                                         L.parent, L.meta, n, local_only);
    pdl(k_union_sparse_local, di.sms * di.sparse_blocks_per_sm, 256, 0, us)(L.spts, L.cw, L.ccoord, L.cstart,
                                                                           L.slist, gp, L.parent, L.meta, n,
                                                                           local_only);
    if (side) FEC_CUDA(cudaEventRecord(side->join, side->s));
    mark(6, st);
    // thread per listed item (k_dcomps): the sparse neighbours and own pairs here, the forward
    // dense pairs on the side stream (forked after k_dcomps); the fallback runs only if a list
    // overflowed
    pdl(k_dense_link, grid_for(dense_max(n) * 4, 256, di.sms * 8), 256, 0, st)(gp, L.crec, L.ncomp, L.oflag, dctx,
                                                                            L.litems, L.lhalf, side ? 2 : 3,
                                                                            L.cw, L.dcoord);
    if (side) FEC_CUDA(cudaStreamWaitEvent(st, side->join, 0));
    // queued pairs still apart after the certain unions (they mark the records whose points
    // they need), then partial scatter phase 1, the item-queue overflow fallback (in-place
    // point tests) and the queued point tests
    pdl(k_dense_filter, grid_for(std::max<int64_t>(L.item_cap, 8 * dense_max(n)), 256, cap * 4), 256, 0, st)(dctx, L.items2, L.slices2, L.idone);
    if (count_path && C.node_stats) {
        mark_sub(0, st);
        pdl(k_dscatter, wt, 256, 0, st)(pts, n, gp, L.cw, L.slot, L.spts, L.pcode, L.meta, L.cneed0, L.cneed1, 1,
                                        C.node_stats && !full_scatter(), dctx.item_cap);
        mark_sub(1, st);
        ++launches;
    }
    // almost always a no-op (nothing overflowed): a small grid keeps its launch cheap
    pdl(k_dense_overflow, di.sms, 256, 0, st)(gp, L.cw, L.crec, L.ncomp, L.dcoord, L.oflag, dctx);
    pdl(k_dense_items, di.sms * 8, 256, 0, st)(gp, dctx, L.items2, L.slices2, L.idone);
    launches += local_only ? 5 : 6;
    if (g_instrument) {
        pdl(k_dense_count, grid_for(dense_max(n), 256, cap), 256, 0, st)(L.ncomp, L.dlist, L.cstart, dctx);
        ++launches;
    }
    mark(7, st);
    C.val = L.sidx;
    C.launches = launches;
    return FEC_OK;
}

// Fills g_stats after an enqueued call.  Fields planned on the device (grid, cells, ...) need
// a read-back, done only for instrumented calls (which therefore synchronise); otherwise -1.
fec_status_t finish_stats(const Core& C, int64_t n, cudaStream_t st) {
    const Layout& L = C.L;
    std::memset(&g_stats, 0, sizeof(g_stats));
    g_stats.n = n;
    g_stats.cells = g_stats.groups = g_stats.components = g_stats.pair_tests = g_stats.group_pairs = -1;
    g_stats.dense_cells = g_stats.dense_points = g_stats.dense_tests = -1;
    g_stats.key_bits = -1;
    g_stats.radix_passes = -1;
    g_stats.dense_table = -1;
    g_stats.binning = -1;
    for (int a = 0; a < 3; ++a) g_stats.dims[a] = -1;
    g_stats.launches = C.launches;
    if (g_instrument) {
        if (!g_snap) FEC_CUDA(cudaMallocHost(&g_snap, sizeof(Snapshot)));
        FEC_CUDA(cudaMemcpyAsync(&g_snap->meta, L.meta, sizeof(Meta), cudaMemcpyDeviceToHost, st));
        FEC_CUDA(cudaMemcpyAsync(&g_snap->grid, L.grid, sizeof(Grid), cudaMemcpyDeviceToHost, st));
        FEC_CUDA(cudaStreamSynchronize(st));
        const Meta& m = g_snap->meta;
        const Grid& g = g_snap->grid;
        if (m.status != FEC_OK) {  // nothing to report (the caller sees the status)
            g_stats_valid = true;
            return FEC_OK;
        }
        g_stats.key_bits = g.key_bits;
        g_stats.radix_passes = g.passes;
        g_stats.dense_table = g.hashed ? 0 : 1;
        g_stats.binning = g.key_sort ? 1 : 0;
        for (int a = 0; a < 3; ++a) g_stats.dims[a] = g.dims[a];
        g_stats.cells = m.cells;
        g_stats.groups = -1;
        g_stats.dense_cells = m.ndense;
        g_stats.dense_points = (int64_t)m.dense_points;
        g_stats.components = (int64_t)m.components;
        g_stats.pair_tests = (int64_t)(m.pair_tests + m.dense_tests);
        g_stats.dense_tests = (int64_t)m.dense_tests;
        g_stats.group_pairs = (int64_t)m.nitems2;
        if (m.internal_error) { g_err = "internal invariant failed (component bound)"; return FEC_ERR_CUDA; }
    }
    g_stats_valid = true;
    return FEC_OK;
}

// Validates and enqueues the whole path (a1..a10).  No host synchronisation for a single cloud
// (status_dev receives what the device finds); batch mode synchronises once after its bboxes.
fec_status_t run(const float* pts, int64_t n, float d, int64_t min_size, int64_t max_size, int32_t* labels,
                 void* ws, size_t ws_bytes, cudaStream_t st, const BatchArgs* B = nullptr,
                 int32_t* status_dev = nullptr, bool ws_own = false) {
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
    // (a workspace the library just took from the stream-ordered pool is not queried: under
    // graph capture it is not mapped yet)
    if (!is_device_ptr(pts) || !is_device_ptr(labels) || (!ws_own && !is_device_ptr(ws))) {
        g_err = "points, labels_out and workspace must be device pointers";
        return FEC_ERR_INVALID_ARGUMENT;
    }
    if (ws_bytes < carve(nullptr, n).total) { g_err = "workspace too small (see fec_workspace_bytes)"; return FEC_ERR_INVALID_ARGUMENT; }
    Core C;
    C.node_stats = 1;
    rc = run_core(pts, n, d, t2, ws, st, C, B, status_dev);
    if (rc != FEC_OK) return rc;
    const Layout& L = C.L;
    const int cap = dev_info().sms * 8;
    const unsigned ew = grid_for(n, 256, cap * 4);
    // ---- a8 (sparse-dominated clouds only), a9 (one launch, variant chosen on the device), a10
    const unsigned wave = grid_for(n, 256, cap);
    pdl(k_flatten_if, wave, 256, 0, st)(L.parent, n, L.meta);
    mark(8, st);
    // (at least two blocks: the node tail splits the grid in halves)
    // large sparse-dominated clouds: the bucket pass of k_relabel_in applies the size filter
    // (k_rootlab returns at once for them), and a filter keeping every size needs no counts
    const bool bucketed = n >= kRelabelBucketN;
    const int count_sizes = (bucketed && min_size <= 1 && max_size >= n) ? 0 : 1;
    uint2* tmp = bucketed ? reinterpret_cast<uint2*>(L.skey0) : nullptr;  // (the sort buffers are free again)
    pdl(k_tail_stats, std::max(ew, 2u), 256, 0, st)(L.parent, C.val, n, L.size, L.minidx, L.meta, L.ncomp,
                                                   L.cstart, L.slist, (uint32_t)(rec_pow2(n) - 1), L.spts,
                                                   count_sizes);
    mark(9, st);
    pdl(k_rootlab, wave, 256, 0, st)(L.parent, L.size, L.minidx, n, (long long)min_size, (long long)max_size, L.meta,
                                     (uint32_t)(rec_pow2(n) - 1), L.cstart, L.slist, L.ncomp, L.dlist, L.crec,
                                     bucketed ? 1 : 0);
    if (bucketed) {
        pdl(k_relabel_b1, wave, 256, 0, st)(L.parent, C.val, L.size, L.minidx, n, (long long)min_size,
                                            (long long)max_size, tmp, L.rlcur, L.meta, L.grid);
        ++C.launches;
    }
    // labels: input order for node-tail clouds, sorted order for sparse-dominated ones (large
    // ones: the bucket pass in k_rootlab, then k_relabel_b2c); the kernels of the variant
    // not chosen return at once
    pdl(k_relabel_in, grid_for((n + 3) / 4, 256, cap * 4), 256, 0, st)(pts, n, L.grid, L.cw, L.crec, L.cmask,
                                                                      L.cstart, L.spts, L.parent, L.minidx, labels,
                                                                      L.meta, L.pcode);
    if (bucketed) {
        static bool attr_set[64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        if (!attr_set[dev & 63]) {
            FEC_CUDA(cudaFuncSetAttribute(k_relabel_b2c, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 << RL_CTA_SHIFT));
            attr_set[dev & 63] = true;
        }
        const int64_t nb = (n + (1 << RL_SHIFT) - 1) >> RL_SHIFT;
        const int64_t clusters = std::min<int64_t>(nb, dev_info().sms / RL_CLUSTER);
        pdl(k_relabel_b2c, (unsigned)(clusters * RL_CLUSTER), 1024, 4 << RL_CTA_SHIFT, st)(tmp, n, labels, L.meta);
    }
    else
        pdl(k_relabel, grid_for((n + 3) / 4, 256, cap * 4), 256, 0, st)(L.parent, C.val, L.minidx, n, labels, L.meta,
                                                                       B ? B->off_dev : nullptr, B ? B->nclouds : 0);
    ++C.launches;
    C.launches += 4;
    mark(10, st);
    FEC_CUDA(cudaGetLastError());
    return finish_stats(C, n, st);
}

// Stream-ordered workspace for the self-allocating calls (the device's default memory pool;
// capturable: a graph gets allocation / free nodes).
fec_status_t alloc_ws(void** ws, size_t bytes, cudaStream_t st) {
    *ws = nullptr;
    cudaError_t e = cudaMallocAsync(ws, bytes + g_alloc_extra, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *ws = nullptr;
        g_err = std::string("cudaMallocAsync(") + std::to_string(bytes + g_alloc_extra) + " B): " + cudaGetErrorString(e);
        return FEC_ERR_OUT_OF_MEMORY;
    }
    return FEC_OK;
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

// ---- multi-GPU Mode B: device-side slab partition of index-sharded input (fec_part.cu) -----
struct PartWs {
    unsigned* state;            // 8 words: bbox (ordered uint) + non-finite flag
    int* info;                  // axis, nlayers, status
    unsigned long long* cnt;    // per destination / category counts (64)
    unsigned long long* cur;    // cursors (64)
    long long* cum;             // kPartMaxLayers + 1 prefix counts
    size_t total;
};
PartWs part_carve(char* base) {
    PartWs W{};
    Carver cv{base, 0, 0};
    W.state = cv.take<unsigned>(8);
    W.info = cv.take<int>(8);
    W.cnt = cv.take<unsigned long long>(64);
    W.cur = cv.take<unsigned long long>(64);
    W.cum = cv.take<long long>((size_t)kPartMaxLayers + 1);
    W.total = cv.off + 256;
    return W;
}
double part_inv_h(float d) { return 1.0 / ((double)d * (1.0 + std::ldexp(1.0, -16)) * 0.5); }
fec_status_t part_check(void* ws, size_t bytes, int32_t world) {
    if (!ws || bytes < part_carve(nullptr).total) { g_err = "workspace missing or too small (see fec_part_workspace_bytes)"; return FEC_ERR_INVALID_ARGUMENT; }
    if (world < 1 || world > 64) { g_err = "need 1 <= world <= 64"; return FEC_ERR_INVALID_ARGUMENT; }
    return FEC_OK;
}
}  // namespace

extern "C" {

size_t fec_part_workspace_bytes(void) { return part_carve(nullptr).total; }
int32_t fec_part_max_layers(void) { return kPartMaxLayers; }

fec_status_t fec_part_bbox(const float* points, int64_t m, float* bbox_out, int32_t* hist, void* workspace,
                           size_t workspace_bytes, void* stream) {
    fec_status_t rc = part_check(workspace, workspace_bytes, 1);
    if (rc != FEC_OK) return rc;
    if (m < 0 || (m > 0 && !points) || !bbox_out || !hist) { g_err = "bad arguments"; return FEC_ERR_INVALID_ARGUMENT; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const PartWs W = part_carve(static_cast<char*>(workspace));
    const int cap = dev_info().sms * 8;
    pdl(k_part_init, cap, 256, 0, st)(W.state, hist);
    if (m > 0) pdl(k_part_bbox, grid_for(m, 256, cap), 256, 0, st)(points, m, W.state);
    pdl(k_part_bbox_out, 1, 32, 0, st)(W.state, bbox_out);
    FEC_CUDA(cudaGetLastError());
    return FEC_OK;
}

fec_status_t fec_part_hist(const float* points, int64_t m, const float* gbbox, float d_th, int32_t* hist,
                           void* workspace, size_t workspace_bytes, void* stream) {
    float t2;
    fec_status_t rc = check_args(0, d_th, 1, 1, &t2);
    if (rc == FEC_OK) rc = part_check(workspace, workspace_bytes, 1);
    if (rc != FEC_OK) return rc;
    if (m < 0 || (m > 0 && !points) || !gbbox || !hist) { g_err = "bad arguments"; return FEC_ERR_INVALID_ARGUMENT; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const PartWs W = part_carve(static_cast<char*>(workspace));
    pdl(k_part_hist, grid_for(std::max<int64_t>(m, 1), 256, dev_info().sms * 8), 256, 0, st)(points, m, gbbox,
                                                                                         part_inv_h(d_th), hist,
                                                                                         W.info);
    FEC_CUDA(cudaGetLastError());
    return FEC_OK;
}

fec_status_t fec_part_plan(const int32_t* ghist, int32_t world, int64_t* plan_out, void* workspace,
                           size_t workspace_bytes, void* stream) {
    fec_status_t rc = part_check(workspace, workspace_bytes, world);
    if (rc != FEC_OK) return rc;
    if (!ghist || !plan_out) { g_err = "bad arguments"; return FEC_ERR_INVALID_ARGUMENT; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const PartWs W = part_carve(static_cast<char*>(workspace));
    pdl(k_part_plan, 1, 1024, 0, st)(ghist, W.info, world, W.cum, reinterpret_cast<long long*>(plan_out));
    pdl(k_part_status, 1, 32, 0, st)(W.info, reinterpret_cast<long long*>(plan_out), world);
    FEC_CUDA(cudaGetLastError());
    return FEC_OK;
}

fec_status_t fec_part_pack(const float* points, const int32_t* gidx, int64_t m, const float* gbbox, float d_th,
                           const int64_t* plan, int32_t world, int64_t* counts, float* send_pts,
                           int32_t* send_gidx, void* workspace, size_t workspace_bytes, void* stream) {
    float t2;
    fec_status_t rc = check_args(0, d_th, 1, 1, &t2);
    if (rc == FEC_OK) rc = part_check(workspace, workspace_bytes, world);
    if (rc != FEC_OK) return rc;
    if (m < 0 || (m > 0 && (!points || !gidx)) || !gbbox || !plan || !counts || (!send_pts != !send_gidx)) {
        g_err = "bad arguments";
        return FEC_ERR_INVALID_ARGUMENT;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const PartWs W = part_carve(static_cast<char*>(workspace));
    const unsigned blocks = grid_for(std::max<int64_t>(m, 1), 256, dev_info().sms * 8);
    auto* c64 = reinterpret_cast<unsigned long long*>(counts);
    if (!send_pts) {  // count pass
        FEC_CUDA(cudaMemsetAsync(counts, 0, (size_t)world * 8, st));
        if (m > 0)
            pdl(k_part_pack, blocks, 256, 0, st)(points, gidx, m, gbbox, part_inv_h(d_th), W.info,
                                                reinterpret_cast<const long long*>(plan), world, 0, c64, nullptr,
                                                nullptr);
    } else if (m > 0) {  // scatter pass: segments in rank order, sizes from the count pass
        pdl(k_part_offsets, 1, 32, 0, st)(c64, world, W.cur);
        pdl(k_part_pack, blocks, 256, 0, st)(points, gidx, m, gbbox, part_inv_h(d_th), W.info,
                                            reinterpret_cast<const long long*>(plan), world, 1, W.cur, send_pts,
                                            send_gidx);
    }
    FEC_CUDA(cudaGetLastError());
    return FEC_OK;
}

fec_status_t fec_part_order(const float* recv_pts, const int32_t* recv_gidx, int64_t k, const float* gbbox,
                            float d_th, const int64_t* plan, int32_t world, int32_t rank, int64_t* counts3,
                            float* out_pts, int32_t* out_gidx, void* workspace, size_t workspace_bytes,
                            void* stream) {
    float t2;
    fec_status_t rc = check_args(0, d_th, 1, 1, &t2);
    if (rc == FEC_OK) rc = part_check(workspace, workspace_bytes, world);
    if (rc != FEC_OK) return rc;
    if (rank < 0 || rank >= world || k < 0 || (k > 0 && (!recv_pts || !recv_gidx || !out_pts || !out_gidx)) ||
        !gbbox || !plan || !counts3) {
        g_err = "bad arguments";
        return FEC_ERR_INVALID_ARGUMENT;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const PartWs W = part_carve(static_cast<char*>(workspace));
    auto* c64 = reinterpret_cast<unsigned long long*>(counts3);
    FEC_CUDA(cudaMemsetAsync(counts3, 0, 3 * 8, st));
    if (k > 0) {
        const unsigned blocks = grid_for(k, 256, dev_info().sms * 8);
        const auto* pl = reinterpret_cast<const long long*>(plan);
        pdl(k_part_order, blocks, 256, 0, st)(recv_pts, recv_gidx, k, gbbox, part_inv_h(d_th), W.info, pl, world,
                                             rank, 0, c64, nullptr, nullptr);
        pdl(k_part_offsets, 1, 32, 0, st)(c64, 3, W.cur);
        pdl(k_part_order, blocks, 256, 0, st)(recv_pts, recv_gidx, k, gbbox, part_inv_h(d_th), W.info, pl, world,
                                             rank, 1, W.cur, out_pts, out_gidx);
    }
    FEC_CUDA(cudaGetLastError());
    return FEC_OK;
}

}  // extern "C"
namespace {
}  // namespace

extern "C" {

size_t fec_workspace_bytes(int64_t n) {
    if (n <= 0 || n > kMaxN) return 0;
    return carve(nullptr, n).total;
}

size_t fec_workspace_bytes_host(int64_t n) {
    if (n <= 0 || n > kMaxN) return 0;
    return fec_workspace_bytes(n) + ((size_t)12 * n + 256) + ((size_t)4 * n + 256);
}

fec_status_t fec_cluster_ws_async(const float* points, int64_t n, float d_th, int64_t min_size, int64_t max_size,
                                  int32_t* labels_out, void* workspace, size_t workspace_bytes, void* stream,
                                  int32_t* status_dev) {
    return run(points, n, d_th, min_size, max_size, labels_out, workspace, workspace_bytes,
               static_cast<cudaStream_t>(stream), nullptr, status_dev);
}

fec_status_t fec_cluster_ws(const float* points, int64_t n, float d_th, int64_t min_size, int64_t max_size,
                            int32_t* labels_out, void* workspace, size_t workspace_bytes, void* stream) {
    float t2;
    fec_status_t rc = check_args(n, d_th, min_size, max_size, &t2);
    if (rc != FEC_OK || n == 0) return run(points, n, d_th, min_size, max_size, labels_out, workspace, 0, 0);
    rc = ensure_status_word();
    if (rc != FEC_OK) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    rc = run(points, n, d_th, min_size, max_size, labels_out, workspace, workspace_bytes, st, nullptr, g_status_host);
    if (rc != FEC_OK || n == 0) return rc;
    return wait_status(st, g_status_host);
}

fec_status_t fec_cluster_async(const float* points, int64_t n, float d_th, int64_t min_size, int64_t max_size,
                               int32_t* labels_out, void* stream, int32_t* status_dev) {
    float t2;
    fec_status_t rc = check_args(n, d_th, min_size, max_size, &t2);
    if (rc != FEC_OK || n == 0) return run(points, n, d_th, min_size, max_size, labels_out, nullptr, 0, 0);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t b = fec_workspace_bytes(n);
    void* ws = nullptr;
    rc = alloc_ws(&ws, b, st);
    if (rc != FEC_OK) return rc;
    rc = run(points, n, d_th, min_size, max_size, labels_out, ws, b, st, nullptr, status_dev, true);
    cudaFreeAsync(ws, st);  // stream-ordered: after the last kernel of the call
    return rc;
}

fec_status_t fec_cluster(const float* points, int64_t n, float d_th, int64_t min_size, int64_t max_size,
                         int32_t* labels_out) {
    float t2;
    fec_status_t rc = check_args(n, d_th, min_size, max_size, &t2);
    if (rc != FEC_OK || n == 0) return run(points, n, d_th, min_size, max_size, labels_out, nullptr, 0, 0);
    rc = ensure_status_word();
    if (rc != FEC_OK) return rc;
    rc = fec_cluster_async(points, n, d_th, min_size, max_size, labels_out, nullptr, g_status_host);
    if (rc != FEC_OK || n == 0) return rc;
    return wait_status(nullptr, g_status_host);
}

static fec_status_t cluster_host_impl(const float* points_host, int64_t n, float d_th, int64_t min_size,
                                      int64_t max_size, int32_t* labels_host, void* workspace,
                                      size_t workspace_bytes, void* stream, bool sync, int32_t* status_dev);

fec_status_t fec_cluster_host(const float* points_host, int64_t n, float d_th, int64_t min_size, int64_t max_size,
                              int32_t* labels_host, void* workspace, size_t workspace_bytes, void* stream) {
    float t2;
    fec_status_t rc = check_args(n, d_th, min_size, max_size, &t2);
    if (rc != FEC_OK || n == 0) return run(nullptr, n, d_th, min_size, max_size, nullptr, nullptr, 0, 0);
    rc = ensure_status_word();
    if (rc != FEC_OK) return rc;
    return cluster_host_impl(points_host, n, d_th, min_size, max_size, labels_host, workspace, workspace_bytes,
                             stream, true, g_status_host);
}

fec_status_t fec_cluster_host_async(const float* points_host, int64_t n, float d_th, int64_t min_size,
                                    int64_t max_size, int32_t* labels_host, void* workspace,
                                    size_t workspace_bytes, void* stream, int32_t* status_dev) {
    return cluster_host_impl(points_host, n, d_th, min_size, max_size, labels_host, workspace, workspace_bytes,
                             stream, false, status_dev);
}

static fec_status_t cluster_host_impl(const float* points_host, int64_t n, float d_th, int64_t min_size,
                                      int64_t max_size, int32_t* labels_host, void* workspace,
                                      size_t workspace_bytes, void* stream, bool sync, int32_t* status_dev) {
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
    rc = run(dpts, n, d_th, min_size, max_size, dlab, workspace, main_b, st, nullptr, status_dev);
    if (rc == FEC_OK) FEC_CUDA(cudaMemcpyAsync(labels_host, dlab, (size_t)4 * n, cudaMemcpyDeviceToHost, st));
    if (rc != FEC_OK) return rc;
    if (sync) return wait_status(st, status_dev);
    return FEC_OK;
}


int64_t fec_slab_record_words(int64_t rec_cap) { return rec_cap < 0 ? -1 : slab_c_off(rec_cap) + 4 * rec_cap; }

size_t fec_slab_workspace_bytes(int64_t n_local, int32_t world, int64_t rec_cap) {
    if (n_local < 0 || world < 1 || rec_cap < 0) return 0;
    return slab_carve(nullptr, n_local, world, rec_cap).total;
}

fec_status_t fec_slab_local(const float* points, const int32_t* gidx, int64_t n_local, int64_t n_owned,
                            int64_t n_first, float d_th, int32_t* records, int64_t rec_cap, void* workspace,
                            size_t workspace_bytes, fec_slab_state_t* state, void* stream, int32_t* status_dev) {
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
    rc = run_core(points, n_local, d_th, t2, workspace, st, C, nullptr, status_dev);
    if (rc != FEC_OK) return rc;
    const Layout& L = C.L;
    const unsigned ew = grid_for(n_local, 256, dev_info().sms * 8 * 4);
    pdl(k_flatten, ew, 256, 0, st)(L.parent, n_local, L.size, L.minidx, L.meta);
    mark(8, st);
    ++C.launches;
    FEC_CUDA(cudaMemsetAsync(S.ckey, 0xFF, (size_t)nodes_max(n_local) * 4, st));
    pdl(k_slab_stats, ew, 256, 0, st)(L.parent, C.val, gidx, n_local, (int)n_owned, (int)n_first, L.size, L.minidx,
                                     S.ckey, L.meta);
    mark(9, st);
    pdl(k_slab_pack, grid_for(nodes_max(n_local), 256, dev_info().sms * 8 * 4), 256, 0, st)(
        L.parent, C.val, gidx, n_local, (int)n_owned, (int)n_first, L.size, L.minidx, S.ckey, records, (int)rec_cap,
        L.meta, (uint32_t)(rec_pow2(n_local) - 1));
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
                                                                       (long long)max_size, labels_owned, L.meta);
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
    rc = ensure_status_word();
    if (rc != FEC_OK) return rc;
    // the stacked grid does not fit the dense mode: cluster the clouds one after another
    for (int32_t c = 0; c < nclouds; ++c) {
        const int64_t a = offsets[c], nc = offsets[c + 1] - offsets[c];
        if (nc == 0) continue;
        rc = run(points + 3 * a, nc, d_th, min_size, max_size, labels_out + a, workspace, workspace_bytes, st, nullptr,
                 g_status_host);
        if (rc == FEC_OK) rc = wait_status(st, g_status_host);
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

void fec_debug_alloc_extra(size_t bytes) { g_alloc_extra = bytes; }

int32_t fec_get_stage_times(float* ms_out, int32_t max_stages) {
    if (!g_ev.recorded) { g_err = "no timed call on this thread (fec_set_timing(1) first)"; return -1; }
    cudaError_t e = cudaEventSynchronize(g_ev.ev[kStages]);
    if (e != cudaSuccess) { g_err = cudaGetErrorString(e); return -1; }
    float sub = 0.f;
    if (g_ev.sub_recorded) cudaEventElapsedTime(&sub, g_ev.sub[0], g_ev.sub[1]);
    for (int i = 0; i < kStages && i < max_stages; ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, g_ev.ev[i], g_ev.ev[i + 1]);
        if (i == 3) ms += sub;  // a4_gather_init: + partial scatter phase 1
        if (i == 6) ms -= sub;  // a6a7_union_dense: - the same interval
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
bool fec::debug_sync_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FEC_DEBUG_SYNC");
        return e && e[0] == '1';
    }();
    return on;
}
cudaError_t fec::debug_sync_after(const void* kernel, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return cudaSuccess;
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        const char* name = "?";
        cudaFuncGetName(&name, kernel);
        std::fprintf(stderr, "[fec] FEC_DEBUG_SYNC: kernel %s failed: %s\n", name, cudaGetErrorString(e));
        g_err = std::string("kernel ") + name + ": " + cudaGetErrorString(e);
    }
    return e;
}
bool fec::pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FEC_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

extern "C" {

const char* fec_version(void) { return "fec-b200 0.2 sm_100a"; }

int64_t fec_max_points(void) { return kMaxN; }

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
