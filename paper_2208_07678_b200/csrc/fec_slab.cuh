// Slab (multi-GPU) kernels: declarations (internal; the C ABI is include/fec.h).
#pragma once
#include "fec_kernels.cuh"

namespace fec {

constexpr int SLAB_HDR = 4;  // header words of a record buffer: nP, nC, 0, 0
// word offset of the C region: after rec_cap P pairs, padded to an even count (16-B aligned)
__host__ __device__ __forceinline__ int64_t slab_c_off(int64_t rec_cap) { return SLAB_HDR + 2 * ((rec_cap + 1) & ~int64_t(1)); }

__global__ void k_slab_stats(const int* parent, const int* val, const int* gidx, int64_t n, int n_owned, int n_first,
                             int* size, int* minidx, int* ckey, Meta* meta);
__global__ void k_slab_pack(const int* parent, const int* val, const int* gidx, int64_t n, int n_owned, int n_first,
                            const int* size, const int* minidx, const int* ckey, int* rec, int rec_cap, const Meta* meta,
                            uint32_t rmask);
__global__ void k_merge_init(int* hkey, int* hpar, int* gsize, int* gmin, int64_t hc);
__global__ void k_merge_link(const int* all, int world, int64_t words, int rec_cap, int* hkey, unsigned mask,
                             int* hpar);
__global__ void k_merge_stats(const int* all, int world, int64_t words, int rec_cap, const int* hkey, unsigned mask,
                              int* hpar, int* gsize, int* gmin);
__global__ void k_merge_resolve(const int* own, int rec_cap, const int* hkey, unsigned mask, int* hpar,
                                const int* gsize, const int* gmin, int* size, int* minidx);
__global__ void k_slab_relabel(const int* parent, const int* val, const int* size, const int* minidx, int64_t n,
                               int n_owned, long long min_size, long long max_size, int* labels, const Meta* meta);

}  // namespace fec
