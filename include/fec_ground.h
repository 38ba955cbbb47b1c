/*
 * fec_ground.h — C ABI of the RANSAC plane-fit ground removal that precedes clustering
 * (SURVEY.md §8(f) N2).  All pointers are CUDA device pointers on the current device
 * unless stated otherwise; every call is enqueued on `stream` (NULL = legacy default stream)
 * and returns without synchronising.
 *
 * The operation (§2.1 "remove the ground surface as a pre-processing",
 * plane fitting being one of the methods it names; SPEC.md L307-310 op remove_ground; the
 * arithmetic readings G1-G7 are in DESIGN.md §8c):
 *
 *   for every hypothesis h (three caller-drawn point indices, reading G1):
 *     plane_h from the three points in binary64 (cross product, normalised, n_z >= 0,
 *     off = -n.p0), rounded to binary32; tilt-valid iff n_z >= cos_max_tilt        (G2)
 *     count_h = #{ i : |fmaf(nz, z_i, fmaf(ny, y_i, fmaf(nx, x_i, off)))| <= threshold } (G3)
 *   best = the tilt-valid h with the largest count, the lowest h among equals      (G4)
 *   ground iff best exists and count_best >= min_inliers (SPEC: ">= 10% inliers")   (G5)
 *   the inliers of plane_best are removed; the survivors keep their input order    (G6)
 *   refined = least-squares plane over those inliers (centroid + smallest-eigenvalue
 *   eigenvector of the scatter matrix, n_z >= 0)                                   (G7)
 */
#ifndef FEC_GROUND_H
#define FEC_GROUND_H

#include <stddef.h>
#include <stdint.h>

#include "fec.h"

#ifdef __cplusplus
extern "C" {
#endif

#define FEC_GROUND_MAX_HYP 4096 /* hypotheses per call (planes live in shared memory) */

typedef struct {
    int32_t best;          /* hypothesis index of the ground plane; -1 = no ground found   */
    int32_t n_valid;       /* hypotheses whose plane exists and is within the tilt bound   */
    int64_t n_inliers;     /* points removed (0 when best == -1)                           */
    int64_t n_keep;        /* survivors written to keep_points / keep_idx (= n - n_inliers)*/
    float plane[4];        /* (nx, ny, nz, off) of hypothesis `best`, binary32; NaN if none */
    double refined[4];     /* least-squares plane over the inliers; NaN if none; the
                              hypothesis plane in binary64 when fewer than 3 inliers        */
} fec_ground_result_t;

/* Device workspace bytes for fec_ground_remove (0 on invalid sizes). */
size_t fec_ground_workspace_bytes(int64_t n, int32_t n_hyp);

/* Ground removal.
 *   points      n x 3 binary32, row-major [n][3] (xyz interleaved), 4-B aligned; read only.
 *   n           0 <= n <= INT32_MAX.
 *   triplets    n_hyp x 3 int32 point indices; a hypothesis with an index outside [0, n) or a
 *               repeated index, or three collinear points, has no plane (never chosen).
 *   n_hyp       0 <= n_hyp <= FEC_GROUND_MAX_HYP.
 *   threshold   finite, >= 0 (metres, compared in binary32).
 *   cos_max_tilt  cos of the largest allowed angle between the plane normal and +z.
 *   min_inliers >= 0; the binding passes ceil(n / 10) by default (SPEC "10% inliers").
 *   keep_points n x 3 binary32 (capacity n): survivors, input order, first n_keep rows.
 *   keep_idx    n int32 (capacity n): the survivors' input indices, increasing.
 *   counts      n_hyp int64 or NULL: inliers of every hypothesis plane (0 if it has none).
 *   result      one fec_ground_result_t, written on the device.
 *   workspace   >= fec_ground_workspace_bytes(n, n_hyp) bytes, 256-B aligned, caller-owned.
 * Points with a NaN/inf coordinate are never inliers (they survive; fec_cluster then rejects
 * them).  Errors (returned before any launch, outputs untouched): FEC_ERR_INVALID_ARGUMENT
 * for bad sizes/threshold/null pointers/too small a workspace; FEC_ERR_CUDA on a launch
 * error (fec_last_error()). */
fec_status_t fec_ground_remove(const float* points, int64_t n, const int32_t* triplets, int32_t n_hyp,
                               float threshold, double cos_max_tilt, int64_t min_inliers, float* keep_points,
                               int32_t* keep_idx, int64_t* counts, fec_ground_result_t* result,
                               void* workspace, size_t workspace_bytes, void* stream);

/* Labels of the whole cloud from the labels of its survivors: labels_out[i] = -2 for a removed
 * (ground) point; for survivor j (input index keep_idx[j]): keep_labels[j] < 0 -> -1, else
 * keep_idx[keep_labels[j]] (the survivor-order minimum maps to the input-order minimum, since
 * keep_idx increases).  keep_labels: n_keep int32 from fec_cluster* on keep_points; result: the
 * fec_ground_result_t of the same fec_ground_remove call (n_keep read on the device);
 * labels_out: n int32.  Errors: FEC_ERR_INVALID_ARGUMENT (n out of range, null pointers),
 * FEC_ERR_CUDA. */
fec_status_t fec_ground_expand_labels(const int32_t* keep_idx, const int32_t* keep_labels,
                                      const fec_ground_result_t* result, int64_t n, int32_t* labels_out,
                                      void* stream);

/* Measurement hook: with fec_set_timing(1), fec_ground_remove records CUDA events around its
 * inlier-counting kernel on `stream`; this returns that kernel's duration in ms for the
 * calling thread's last call (waits for the end event), or -1 if none was recorded.
 * Errors: FEC_ERR_INVALID_ARGUMENT (ms NULL), FEC_ERR_CUDA. */
fec_status_t fec_ground_count_ms(float* ms);

#ifdef __cplusplus
}
#endif

#endif /* FEC_GROUND_H */
