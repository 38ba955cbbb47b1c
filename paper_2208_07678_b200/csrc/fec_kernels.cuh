// Kernel declarations and shared device structs of the FEC path (internal).
#pragma once
#include "fec_internal.cuh"

namespace fec {

constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;
constexpr int SCAN_THREADS = 256;
constexpr int SPARSE_MAX = 6;   // dense-grid mode: cells with <= SPARSE_MAX points are "sparse"

// Small device-resident header at the start of the workspace.
struct Meta {
    float bbox[6];                    // min xyz, max xyz
    int nonfinite;                    // != 0 if any coordinate is NaN / inf
    int status;                       // FEC_OK or the error a1 found (copied from the plan)
    unsigned int ticket;              // a1: blocks done (the last one plans the grid)
    int pad_meta;
    int groups;                       // nonempty sub-cells
    int cells;                        // nonempty cells
    int work;                         // dynamic cell counter of the neighbour scan
    int instrument;                   // gather counters below
    int ndense;                       // dense-grid mode: cells with > SPARSE_MAX points
    unsigned long long pair_tests;
    unsigned long long group_pairs;
    unsigned long long components;
    unsigned long long dense_points;
    unsigned long long dense_tests;
    int nheavy, nlight;               // dense-grid mode: schedule of the dense cells
    int work2;                        // second dynamic work counter
    int cells1;                       // dense-grid mode: occupied cells + 1 (scan length)
    int dwords1;                      // dense-grid mode: words of the dense-cell bitmap + 1 (scan length)
    int nitems;                       // dense-grid mode: uncertain component pairs pushed
    int internal_error;               // != 0: an internal invariant failed (never expected)
    int nitems2;                      // dense-grid mode: queued pairs still apart after the certain unions
    unsigned long long near_pairs;    // a1: consecutive input pairs within 2 cells (input coherence)
    int nsparse;                      // dense-grid mode: occupied cells with <= SPARSE_MAX points
    int nslices_extra;                // dense-grid mode: extra slices of heavy uncertain pairs
    int ndd, nds;                     // dense link items: forward dense pairs / sparse neighbours + own pairs
    int list_overflow;                // != 0: a link item list overflowed (k_dense_link redoes all)
};

// What the host passes to a1 (k_bbox); its last block turns the bbox into the Grid (plan_grid).
struct PlanArgs {
    Grid g0;             // host-known fields: h, inv_h, inv_q, t2, hmask, hkey (the rest is planned)
    int64_t n;
    int64_t dense_cap;   // bitmap mode iff the grid holds <= dense_cap cells
    int32_t grid_mode;   // fec_set_grid_mode: 0 auto, 1 hash, 2 key sort, 3 counting sort
    int32_t key_path;    // the host enqueued the key-sort kernels (else the counting path is taken)
    int32_t vec4;        // points are 16-byte aligned
    int32_t instrument;
    float near;          // coherence test distance (two cells)
    int32_t pad;
    int32_t* status_dev; // optional: the caller's device status word
};

__global__ void k_bbox(const float* p, PlanArgs a, float* part, Meta* meta, Grid* gout);
__global__ void k_zero(const Grid* gp, uint2* cw, u64* hkey, int64_t slots, uint32_t* arena, int64_t arena_words);
__global__ void k_radix_hist(const u64* key, int64_t n, int shift, uint32_t* counts, int num_tiles);
__global__ void k_radix_scatter(const u64* kin, const int* vin, u64* kout, int* vout, int64_t n, int shift,
                                const uint32_t* offs, int num_tiles);
__global__ void k_onesweep(const Grid* gp, int pass, uint32_t* k0, int* v0, uint32_t* k1, int* v1, int64_t n,
                           const uint32_t* ghist, uint32_t* state, int64_t tiles, unsigned int* tile_ctr);
__global__ void k_flatten(int* parent, int64_t n, int* size, int* minidx, const Meta* meta);
__global__ void k_flatten_if(int* parent, int64_t n, const Meta* meta);
__global__ void k_rootlab(const int* parent, const int* size, int* minidx, int64_t n, long long min_size,
                          long long max_size, const Meta* meta, uint32_t rmask, const uint32_t* cstart,
                          const int* slist, const int* ncomp, const int* dlist, int* crec, int bucketed);
__global__ void k_relabel_b1(const int* parent, const int* val, const int* size, const int* minidx, int64_t n,
                             long long min_size, long long max_size, uint2* tmp, unsigned int* cursor,
                             const Meta* meta, const Grid* gp);
__global__ void k_relabel(const int* parent, const int* val, const int* minidx, int64_t n, int* labels,
                          const Meta* meta, const int64_t* boff, int nclouds);
// bucketed relabel (large sparse-dominated clouds): RL_SHIFT bits of input index per bucket
// bucket = input index >> RL_SHIFT: 2^18 labels = 1 MB, staged by k_relabel_b2c in the
// distributed shared memory of a cluster of RL_CLUSTER CTAs (128 KB each)
constexpr int RL_SHIFT = 18;
constexpr int RL_CLUSTER = 8;
constexpr int RL_CTA_SHIFT = 15;  // labels per CTA of the cluster: 2^15 (128 KB)
constexpr int RL_TILE = 2048;
constexpr int RL_MAX_BUCKETS = 4096;  // n <= 2^30 (fec_max_points < 2^30)
constexpr int RL_CUR_STRIDE = 32;     // one bucket cursor per 128-byte line (L2 slices in parallel)
static_assert(RL_CTA_SHIFT + 3 == RL_SHIFT, "a cluster of 8 CTAs holds one bucket");
__global__ void k_relabel_b2c(const uint2* tmp, int64_t n, int* labels, const Meta* meta);
__global__ void k_bbox_clouds(const float* p, const int64_t* off, float* bb, int* nonfinite, float near,
                              unsigned long long* near_pairs);
__global__ void k_cmark(const float* p, int64_t n, const Grid* gp, uint2* cw);
__global__ void k_cpop(const uint2* cw, uint32_t* tsum, const Grid* gp);
__global__ void k_tscan(uint32_t* tsum, const Grid* gp, Meta* meta, uint32_t* count);
__global__ void k_cscan(uint2* cw, const Grid* gp, const uint32_t* tpre, uint32_t* clin, uint32_t* count, u64* cocc,
                        int* cmin, u64* ccoord);
__global__ void k_lkey(const float* p, int64_t n, const Grid* gp, uint32_t* key, int* val, uint32_t* ghist,
                       uint32_t* state0, int64_t state_words);
__global__ void k_smark(const uint32_t* key0, const uint32_t* key1, int64_t n, uint2* cw, const Grid* gp);
__global__ void k_sgather(const float* p, const uint32_t* key0, const int* val0, const uint32_t* key1,
                          const int* val1, int64_t n, const Grid* gp, const uint2* cw, float4* spts, uint32_t* cstart,
                          u64* cocc, int* parent, int* sidx, int* size, int* minidx, const Meta* meta);
// Counting path, per input point: compact cell id << 6 | fine sub-cell, written by k_dcount2
// when the cloud has at most kCodeCells occupied cells (read by k_dscatter and k_relabel_in
// instead of recomputing the cell from the coordinates).
constexpr int kCodeCells = (1 << 26) - 1;  // (the code ~0u >> 6 is never a valid compact id)
__global__ void k_dcount2(const float* p, int64_t n, const Grid* gp, const uint2* cw, uint32_t* count, u64* cocc,
                          int* cmin, uint32_t* pcode, const Meta* meta);
__global__ void k_dscatter(const float* p, int64_t n, const Grid* gp, const uint2* cw, uint32_t* cursor,
                           float4* spts, const uint32_t* pcode, const Meta* meta, const uint32_t* cneed0,
                           const uint32_t* cneed1, int phase, int node_stats, int item_cap);
__global__ void k_dinit(const float4* spts, int64_t n, const Grid* gp, const uint2* cw, const int* crec,
                        const u64* cmask, int nbase, int* parent, int* size, int* minidx, int* sidx, const Meta* meta,
                        int all_parents);
__global__ void k_cellred(const uint32_t* cstart, const Meta* meta, const Grid* gp, unsigned long long* tsum);
__global__ void k_celltscan(unsigned long long* tsum, Meta* meta, const Grid* gp, uint32_t* cstart);
__global__ void k_cellscan(uint32_t* cstart, uint32_t* cursor, int* dlist, int* crec, uint32_t* cneed0, Meta* meta,
                           const Grid* gp, const unsigned long long* tpre, int* slist, int64_t n, int local_only,
                           int all_parents, int* parent, int* size, int* minidx);
// Component node of dense record r, component c (rmask: R - 1 for the record capacity R, a
// power of two; node ids stay below nbase + 8R).
__host__ __device__ __forceinline__ int node_of(int nbase, uint32_t rmask, int r, int c) {
    (void)rmask;
    return nbase + 8 * r + c;
}

// Dense-grid mode: what the component kernels share (item = (P record, P component,
// Q record or point, Q component or -1 for a point)).
struct DenseCtx {
    const float4* spts;
    const uint32_t* cstart;
    const int* dlist;
    const uint32_t* clin;
    u64* cmask;         // [8*nd] component masks
    int* parent;
    int4* items;
    int item_cap;
    int nbase;          // node id of component k of record r: node_of(nbase, rmask, r, k)
    uint32_t rmask;
    Meta* meta;
    uint32_t* cneed0;   // partial scatter: bit per compact id, points written in phase 0
    uint32_t* cneed1;   // ... and in phase 1 (cells a surviving queued item reads)
};
__global__ void k_dcomps(const Grid* gp, const uint2* cw, int* crec, const u64* cocc, const u64* ccoord, int* ncomp, int* size,
                         int* minidx, u64* dcoord, uint32_t* oflags, DenseCtx C, uint4* litems, int lhalf,
                         const int* cmin, const int* sidx, int node_stats);
__global__ void k_dparent(const float4* spts, const uint32_t* cstart, const int* dlist, const int* ncomp,
                          const u64* cmask, const Grid* gp, int nbase, int* parent, const Meta* meta, const int* sidx,
                          int* size, int* minidx, int node_stats, int64_t n);
__global__ void k_tail_stats(int* parent, const int* val, int64_t n, int* size, int* minidx, Meta* meta,
                             const int* ncomp, const uint32_t* cstart, const int* slist, uint32_t rmask,
                             const float4* spts, int count_sizes);
__global__ void k_relabel_in(const float* p, int64_t n, const Grid* gp, const uint2* cw, const int* crec,
                             const u64* cmask, const uint32_t* cstart, const float4* spts, const int* parent,
                             const int* minidx, int* labels, const Meta* meta, const uint32_t* pcode);
// local_only != 0 (small clouds, host-chosen): the sparse cells always go through the compact
// list and k_union_sparse_local (more parallel per cell), whatever their share of the cells.
__global__ void k_union_sparse(const float4* spts, const uint2* cw, const u64* ccoord, const uint32_t* cstart,
                               const Grid* gp, int* parent, Meta* meta, int64_t n, int local_only);
__global__ void k_union_sparse_local(const float4* spts, const uint2* cw, const u64* ccoord, const uint32_t* cstart,
                                     const int* slist, const Grid* gp, int* parent, Meta* meta, int64_t n,
                                     int local_only);
__global__ void k_dense_link(const Grid* gp, const int* crec, const int* ncomp, uint32_t* oflags, DenseCtx C,
                             const uint4* litems, int lhalf, int which, const uint2* cw, const u64* dcoord);
__global__ void k_dense_filter(DenseCtx C, int4* items2, int4* slices2, int* idone);
__global__ void k_dense_overflow(const Grid* gp, const uint2* cw, const int* crec, const int* ncomp,
                                 const u64* dcoord, uint32_t* oflags, DenseCtx C);
__global__ void k_dense_items(const Grid* gp, DenseCtx C, const int4* items2, const int4* slices2, int* idone);
__global__ void k_dense_count(const int* ncomp, const int* dlist, const uint32_t* cstart, DenseCtx C);
cudaError_t ensure_subcell_tables();  // host: upload the fine sub-cell tables (once per device)
__global__ void k_debug_pred(const float* a, const float* b, int64_t m, float t2, uint8_t* out, float* d2out);

}  // namespace fec
