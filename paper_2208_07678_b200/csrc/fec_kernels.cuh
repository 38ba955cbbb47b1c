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

// Dense-grid mode: a cell holding more than SPARSE_MAX points, re-ordered by octant.
struct DenseRec {
    int cell;    // linear cell id
    int off[9];  // sorted positions: octant k occupies [off[k], off[k+1])
};

__global__ void k_bbox_partial(const float* p, int64_t n, int vec4, float* part, int* nonfinite);
__global__ void k_bbox_final(const float* part, int nblocks, Meta* meta);
__global__ void k_keys(const float* p, int64_t n, Grid g, u64* key, int* val);
__global__ void k_radix_hist(const u64* key, int64_t n, int shift, uint32_t* counts, int num_tiles);
__global__ void k_radix_scatter(const u64* kin, const int* vin, u64* kout, int* vout, int64_t n, int shift,
                                const uint32_t* offs, int num_tiles);
__global__ void k_gather(const float* p, const int* val, int64_t n, float4* spts);
__global__ void k_heads(const u64* key, int64_t n, u64* flags);
__global__ void k_fill_tables(const u64* key, const u64* ex, int64_t n, Grid g, Tables T, Meta* meta);
__global__ void k_init_uf(const u64* ex, const int* gstart, int64_t n, int* parent, int* size, int* minidx);
__global__ void k_scan_union(const float4* spts, Grid g, Tables T, int* parent, Meta* meta);
__global__ void k_flatten(int* parent, int64_t n);
__global__ void k_stats(const int* parent, const int* val, int64_t n, int* size, int* minidx, Meta* meta);
__global__ void k_relabel(const int* parent, const int* val, const int* size, const int* minidx, int64_t n,
                          long long min_size, long long max_size, int* labels);
__global__ void k_dcount(const float* p, int64_t n, Grid g, uint32_t* count, uint32_t* slot, uint32_t* dbits,
                         Meta* meta);
__global__ void k_dbits_popc(const uint32_t* dbits, int64_t words, uint32_t* wcount);
__global__ void k_dbits_list(const uint32_t* dbits, int64_t words, const uint32_t* wpos, int* dlist, int* crec,
                             uint32_t* ocnt, Meta* meta);
__global__ void k_dcount_oct(const float* p, int64_t n, Grid g, const uint32_t* count, const int* crec, uint32_t* ocnt,
                             uint32_t* slot);
__global__ void k_drec_fin(const int* dlist, Meta* meta, const uint32_t* cstart, const uint32_t* ocnt, DenseRec* drec);
__global__ void k_dscatter(const float* p, int64_t n, Grid g, const uint32_t* cstart, const uint32_t* slot,
                           const int* crec, const DenseRec* drec, float4* spts);
__global__ void k_dinit(const float4* spts, int64_t n, Grid g, const uint32_t* cstart, const int* crec,
                        const DenseRec* drec, int* parent, int* size, int* minidx, int* sidx);
__global__ void k_union_sparse(const float4* spts, const uint32_t* cstart, uint32_t cells, Grid g, int* parent,
                               Meta* meta);
__global__ void k_union_dense(const float4* spts, const uint32_t* cstart, const DenseRec* drec, const int* crec,
                              int phase, Grid g, int* parent, Meta* meta);
__global__ void k_debug_pred(const float* a, const float* b, int64_t m, float t2, uint8_t* out, float* d2out);

}  // namespace fec
