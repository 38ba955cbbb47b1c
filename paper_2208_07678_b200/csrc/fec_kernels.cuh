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
    int nitems;                       // dense-grid mode: uncertain component pairs pushed
    int internal_error;               // != 0: an internal invariant failed (never expected)
    int nitems2;                      // dense-grid mode: queued pairs still apart after the certain unions
    unsigned long long near_pairs;    // a1: consecutive input pairs within 2 cells (input coherence)
    int nsparse;                      // dense-grid mode: occupied cells with <= SPARSE_MAX points
    int nslices_extra;                // dense-grid mode: extra slices of heavy uncertain pairs
};

struct Tables {
    int* gstart;        // [G+1] first sorted position of each group (sub-cell)
    uint8_t* goct;      // [G]   octant of each group within its cell
    int* cell_gstart;   // [U+1] first group of each cell
    u64* cell_pc;       // [U]   packed cell coordinates (21 bits per axis)
    int* dense;         // dense mode: row-major cell -> cell id (-1 empty)
    u64* hkey;          // hash mode: packed coords (~0 empty)
    int* hval;          // hash mode: cell id
};


__global__ void k_bbox_partial(const float* p, int64_t n, int vec4, float* part, int* nonfinite, float near,
                               unsigned long long* near_pairs);
// What the host needs after a1, written by k_bbox_final straight into mapped pinned host
// memory; `seq` last (after a system-scope fence), so the host can spin on it instead of
// copying Meta back and synchronising the stream.
struct HostBBox {
    float bbox[6];
    int nonfinite;
    int pad;
    unsigned long long near_pairs;
    int seq;
    int pad2;
};
__global__ void k_bbox_final(const float* part, int nblocks, Meta* meta, HostBBox* hb, int seq);
__global__ void k_keys(const float* p, int64_t n, Grid g, u64* key, int* val);
__global__ void k_radix_hist(const u64* key, int64_t n, int shift, uint32_t* counts, int num_tiles);
__global__ void k_radix_scatter(const u64* kin, const int* vin, u64* kout, int* vout, int64_t n, int shift,
                                const uint32_t* offs, int num_tiles);
__global__ void k_radix_hist32(const uint32_t* key, int64_t n, int shift, uint32_t* counts, int num_tiles);
__global__ void k_radix_scatter32(const uint32_t* kin, const int* vin, uint32_t* kout, int* vout, int64_t n, int shift,
                                  const uint32_t* offs, int num_tiles);
__global__ void k_radix_scatter32l(const uint32_t* kin, const int* vin, uint32_t* kout, int* vout, int64_t n, int shift,
                                   const uint32_t* offs, int num_tiles);
__global__ void k_gather(const float* p, const int* val, int64_t n, float4* spts);
__global__ void k_heads(const u64* key, int64_t n, u64* flags);
__global__ void k_fill_tables(const u64* key, const u64* ex, int64_t n, Grid g, Tables T, Meta* meta);
__global__ void k_init_uf(const u64* ex, const int* gstart, int64_t n, int* parent, int* size, int* minidx);
__global__ void k_scan_union(const float4* spts, Grid g, Tables T, int* parent, Meta* meta);
__global__ void k_flatten(int* parent, int64_t n, int* size, int* minidx);
__global__ void k_flatten_if(int* parent, int64_t n, const Meta* meta);
__global__ void k_flat_stats(int* parent, const int* val, int64_t n, int* size, int* minidx, Meta* meta, int node_tail);
__global__ void k_stats(const int* parent, const int* val, int64_t n, int* size, int* minidx, Meta* meta, int only_sparse);
__global__ void k_rootlab(const int* parent, const int* size, int* minidx, int64_t n, long long min_size,
                          long long max_size, const Meta* meta);
__global__ void k_relabel(const int* parent, const int* val, const int* size, const int* minidx, int64_t n,
                          long long min_size, long long max_size, int* labels, const Meta* meta, const int64_t* boff,
                          int nclouds);
__global__ void k_bbox_clouds(const float* p, const int64_t* off, float* bb, int* nonfinite, float near,
                              unsigned long long* near_pairs);
__global__ void k_cmark(const float* p, int64_t n, Grid g, uint2* cw);

__global__ void k_cscan(uint2* cw, int64_t words, uint32_t* clin, uint32_t* count, u64* cocc, u64* ccoord, Grid g,
                        Meta* meta, unsigned long long* state, unsigned int* counter);

__global__ void k_lkey(const float* p, int64_t n, Grid g, uint32_t* key, int* val);
__global__ void k_smark(const uint32_t* key, int64_t n, uint2* cw);
__global__ void k_sgather(const float* p, const uint32_t* key, const int* val, int64_t n, Grid g, const uint2* cw,
                          float4* spts, uint32_t* cstart, u64* cocc, int* parent, int* sidx, int* size, int* minidx,
                          const Meta* meta);
__global__ void k_scount(const uint32_t* cstart, uint32_t* dbits, const Meta* meta);
__global__ void k_dcount2(const float* p, int64_t n, Grid g, const uint2* cw, uint32_t* count, u64* cocc);
__global__ void k_dscatter2(const float* p, int64_t n, Grid g, const uint2* cw, uint32_t* cursor, float4* spts);
__global__ void k_ccount(const uint32_t* cstart, uint32_t* dbits, uint32_t* cursor, const Meta* meta);
__global__ void k_dbits_popc(const uint32_t* dbits, int64_t words, uint32_t* wcount);
__global__ void k_dbits_list(const uint32_t* dbits, int64_t words, const uint32_t* wpos, int* dlist, int* crec,
                             Meta* meta);
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
    int nbase;          // node id of component k of record r: nbase + 8r + k
    Meta* meta;
};
__global__ void k_dcomps(Grid g, const u64* cocc, const u64* ccoord, int* ncomp, int* size, int* minidx, u64* dcoord,
                         uint32_t* oflags, DenseCtx C);
__global__ void k_dinit(const float4* spts, int64_t n, Grid g, const uint2* cw, const uint32_t* cstart,
                        const int* crec, const int* ncomp, const u64* cmask, int nbase, int* parent, int* size,
                        int* minidx, int* sidx, const Meta* meta, int node_stats);
__global__ void k_dparent(const float4* spts, const uint32_t* cstart, const int* dlist, const int* ncomp,
                          const u64* cmask, Grid g, int nbase, int* parent, const Meta* meta, const int* sidx,
                          int* size, int* minidx, int node_stats, int64_t n);
__global__ void k_tail_stats(int* parent, const int* val, int64_t n, int* size, int* minidx, Meta* meta, int dense,
                             const int* ncomp, const uint32_t* cstart, const int* slist);
__global__ void k_node_stats(int* parent, const int* ncomp, int* size, int* minidx, int nbase, Meta* meta, int64_t n);
__global__ void k_sparse_stats(int* parent, const uint32_t* cstart, const int* slist, const int* sidx, int* size,
                               int* minidx, Meta* meta, int64_t n);
__global__ void k_union_sparse(const float4* spts, const uint2* cw, const u64* ccoord, const uint32_t* cstart, Grid g,
                               int* parent, Meta* meta, int64_t n);
__global__ void k_union_sparse_local(const float4* spts, const uint2* cw, const u64* ccoord, const uint32_t* cstart,
                                     const int* slist, Grid g, int* parent, Meta* meta, int64_t n);
__global__ void k_slist(const uint32_t* cstart, int* slist, Meta* meta, int64_t n);
__global__ void k_dense_link(Grid g, const uint2* cw, const int* crec, const int* ncomp, const u64* dcoord,
                             uint32_t* oflags, DenseCtx C, int k0);
__global__ void k_dense_overflow(Grid g, const uint2* cw, const int* crec, const int* ncomp, const u64* dcoord,
                                 uint32_t* oflags, DenseCtx C);
__global__ void k_dense_filter(Grid g, DenseCtx C, int4* items2, int4* slices2, int* idone);
__global__ void k_dense_items(Grid g, DenseCtx C, const int4* items2, const int4* slices2, int* idone);
__global__ void k_flatten_nodes(int* parent, int nbase, const Meta* meta);
__global__ void k_dense_count(const int* ncomp, const int* dlist, const uint32_t* cstart, DenseCtx C);
cudaError_t ensure_subcell_tables();  // host: upload the fine sub-cell tables (once per device)
__global__ void k_debug_pred(const float* a, const float* b, int64_t m, float t2, uint8_t* out, float* d2out);

}  // namespace fec
