/*
 * fec_metrics.h — C ABI of the segmentation-quality metric: the paper's
 * average precision, Eq. 2 (AP = TP / (TP + FP), "0.75 as the point-wise
 * threshold for true positives"), made concrete as SPEC.md L392-408 (op average_precision)
 * with the readings M1-M4 of DESIGN.md §8e:
 *
 *   M1  points with gt label 0 are excluded from every count; a predicted label -1 (noise) is
 *       not a predicted cluster (its points still count in |G|);
 *   M2  predicted clusters in order of descending |P| (points with gt != 0), ties by label;
 *   M3  each takes the still-unmatched gt cluster of largest IoU = |P n G| / |P u G| among
 *       those it overlaps (ties: smaller gt label), consuming it; TP iff
 *       |P n G| >= threshold * |P u G| (binary64), else FP; no unmatched overlap -> FP;
 *   M4  AP = TP / (TP + FP); 1 if there are neither predicted nor gt clusters; 0 if there are
 *       gt clusters but no predicted ones.
 *
 * All pointers are CUDA device pointers; the call is enqueued on `stream` and does not
 * synchronise.  The (predicted, gt) pair histogram is built by a device radix sort; every
 * predicted cluster's preferred gt cluster is found in parallel, and only when two of them
 * prefer the same gt cluster is the greedy matching (sequential by definition) replayed in
 * order by one warp.
 */
#ifndef FEC_METRICS_H
#define FEC_METRICS_H

#include <stddef.h>
#include <stdint.h>

#include "fec.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int64_t tp;
    int64_t fp;
    int64_t n_pred;   /* predicted clusters (labels >= 0 with at least one gt != 0 point) */
    int64_t n_gt;     /* gt clusters (nonzero gt labels present)                          */
    double ap;        /* NaN when status != 0                                             */
    int32_t status;   /* 0 ok; -1 a label out of range (pred not in {-1} U [0, n), or gt
                         not in [0, n]); then tp = fp = -1                                 */
    int32_t pad;
} fec_ap_result_t;

/* Device workspace bytes for fec_average_precision (0 if n < 0 or n > INT32_MAX - 1). */
size_t fec_ap_workspace_bytes(int64_t n);

/* pred: n int32 (fec_cluster's labels: -1 or a point index); gt: n int32 in [0, n] (0 =
 * unlabelled, e.g. ground); threshold in (0, 1]; result: one fec_ap_result_t on the device;
 * workspace: >= fec_ap_workspace_bytes(n) bytes, 256-B aligned.
 * Errors (host, before any launch): FEC_ERR_INVALID_ARGUMENT (sizes, threshold, null
 * pointers, workspace); FEC_ERR_CUDA.  Out-of-range labels are reported in result->status. */
fec_status_t fec_average_precision(const int32_t* pred, const int32_t* gt, int64_t n, double threshold,
                                   fec_ap_result_t* result, void* workspace, size_t workspace_bytes,
                                   void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FEC_METRICS_H */
