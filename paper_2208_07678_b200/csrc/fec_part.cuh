// Mode B partition kernels (fec_part.cu): declarations (internal; the C ABI is include/fec.h).
#pragma once
#include "fec_kernels.cuh"

namespace fec {

constexpr int kPartMaxLayers = 1 << 20;  // cell layers along the cut axis (reading A14)

__global__ void k_part_init(unsigned* state, int* hist);
__global__ void k_part_bbox(const float* p, int64_t m, unsigned* state);
__global__ void k_part_bbox_out(const unsigned* state, float* out);
__global__ void k_part_status(const int* info, long long* plan, int world);
__global__ void k_part_hist(const float* p, int64_t m, const float* gbb, double inv_h, int* hist, int* info);
__global__ void k_part_plan(const int* hist, const int* info, int world, long long* cum, long long* plan);
__global__ void k_part_pack(const float* p, const int* gidx, int64_t m, const float* gbb, double inv_h, const int* info,
                            const long long* plan, int world, int mode, unsigned long long* cursor, float* send_pts,
                            int* send_gidx);
__global__ void k_part_order(const float* rp, const int* rg, int64_t k, const float* gbb, double inv_h, const int* info,
                             const long long* plan, int world, int rank, int mode, unsigned long long* cursor,
                             float* out_pts, int* out_gidx);

__global__ void k_part_offsets(const unsigned long long* counts, int n, unsigned long long* cursor);

}  // namespace fec
