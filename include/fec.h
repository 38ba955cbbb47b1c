/*
 * fec.h — C ABI of the B200 (sm_100a) FEC hot path: fixed-radius connected components
 * of a 3-D point cloud with a cluster-size noise filter and min-index labels.
 *
 * What is computed (PAPER.md = arXiv 2208.07678 text; readings A1..A16 in DESIGN.md §2):
 *
 *   d = fp32(d_th), t2 = fl32(d*d)                                       (reading A3)
 *   pred(i,j) <=> fl(fl(fl(dx*dx) + fl(dy*dy)) + fl(dz*dz)) <= t2,  dx = fl(x_j - x_i) ...
 *       -- Eq. 1, PAPER.md L187-194 (§2.2 "Fast Euclidean Clustering"), boundary inclusive
 *          (reading A1), every operation one fp32 round-to-nearest, no FMA (reading A2).
 *   C(i) = connected component of i in the graph {i~j : pred(i,j)}
 *       -- the clusters Algorithm 1 outputs as P.lab; the paper's loop
 *          is replaced by a grid index + lock-free union-find computing the same partition
 *          as EC.
 *   labels_out[i] = min C(i)  if min_size <= |C(i)| <= max_size,  else -1
 *       -- size filter of the EC interface (reading A7, inclusive),
 *          canonical min-index label (reading A8), -1 = noise (reading A10).
 *
 * Exactly one output is correct for every input (reading A16), so the result is
 * deterministic and bitwise comparable.  There is no CPU fallback: every step runs in the
 * library's sm_100a kernels.
 *
 * Pointers: unless a function says "host", pointers are CUDA device pointers on the
 * calling thread's current device.  `points` is row-major [n][3] fp32 (x,y,z interleaved),
 * 4-byte aligned.  `labels_out` is int32[n], in the caller's input order.
 *
 * Ownership: the caller owns `points`, `labels_out` and `workspace`; the library never
 * frees or retains them past the call.  `workspace` is scratch device memory of at least
 * fec_workspace_bytes(n) bytes, 256-byte aligned (any cudaMalloc / PyTorch allocation).
 *
 * Errors: argument errors are returned before any launch and leave labels_out untouched.
 * FEC_ERR_NONFINITE / FEC_ERR_GRID_RANGE are detected on the device after the first
 * kernel and returned before any write to labels_out.  FEC_ERR_CUDA leaves labels_out
 * unspecified; fec_last_error() then holds the CUDA error string (thread-local).
 */
#ifndef FEC_H_
#define FEC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t fec_status_t;

#define FEC_OK 0
#define FEC_ERR_INVALID_ARGUMENT (-1) /* n<0 or n>fec_max_points(); d_th not finite > 0 or t2 not a
                                         finite normal fp32 (reading A13); min>max;
                                         max<1; min<0; null/host pointer where a device
                                         pointer is required; workspace too small */
#define FEC_ERR_NONFINITE (-2)        /* a coordinate is NaN or +-inf (reading A12) */
#define FEC_ERR_GRID_RANGE (-3)       /* bbox extent / (d_th*(1+2^-16)) >= 2^20 on an axis
                                         (reading A14): cannot be indexed */
#define FEC_ERR_OUT_OF_MEMORY (-4)    /* fec_cluster / fec_cluster_host could not allocate */
#define FEC_ERR_CUDA (-5)             /* a CUDA runtime error; see fec_last_error() */

/* Statistics of the last successful call on this thread (instrumentation). */
typedef struct {
    int64_t n;              /* points */
    int64_t cells;          /* nonempty grid cells (edge c = d_th*(1+2^-16)) */
    int64_t groups;         /* hash mode: nonempty sub-cells (edge c/2: cliques under pred) */
    int64_t components;     /* connected components before the size filter */
    int64_t pair_tests;     /* predicate evaluations in the neighbour scan */
    int64_t group_pairs;    /* sub-cell pairs examined by the neighbour scan */
    int64_t dense_cells;    /* dense-grid mode: cells holding > 16 points (octant-grouped) */
    int64_t dense_points;   /* dense-grid mode: points in those cells */
    int64_t dense_tests;    /* dense-grid mode: predicate evaluations of the dense-cell kernel */
    int64_t key_bits;       /* significant Morton-key bits sorted */
    int32_t radix_passes;   /* LSD passes of the key sort */
    int32_t dense_table;    /* 1: dense cell grid (counting sort), 0: Morton radix sort + hash */
    int32_t dims[3];        /* cells per axis */
    int32_t launches;       /* kernel launches of the call (all of them the library's own) */
    int32_t binning;        /* 0: counting sort (coherent input), 1: key sort (shuffled input
                               above 2^17 points, grid mode 2); -1 unless instrumented */
} fec_stats_t;

/* Bytes of device workspace fec_cluster_ws needs for n points (an upper bound that does
 * not depend on the coordinates).  Returns 0 for n <= 0. */
size_t fec_workspace_bytes(int64_t n);

/* ---- Asynchronous forms: no host round trip ------------------------------
 *
 * The whole path is enqueued on `stream` (cudaStream_t; NULL = legacy default stream) and the
 * call returns at once: the grid (origin, dims, bitmap vs hashed cell index, counting vs key
 * sort) is planned ON THE DEVICE by the validation kernel (a1) and read there by every later
 * kernel, so nothing waits for the host and the call can be captured in a CUDA graph
 * (stream capture; replays recompute everything from the current contents of `points`).
 *
 * status_dev (optional, may be NULL): a device (or mapped host) int32 that receives, in stream
 * order, FEC_OK or what the device found: FEC_ERR_NONFINITE (a coordinate is NaN/inf, reading
 * A12) or FEC_ERR_GRID_RANGE (reading A14).  After such an error every later kernel returns at
 * once and labels_out is left untouched.  The return value covers only what the host can see
 * before enqueueing: argument errors (FEC_ERR_INVALID_ARGUMENT, nothing enqueued), allocation
 * failure (FEC_ERR_OUT_OF_MEMORY) and launch errors (FEC_ERR_CUDA).  n == 0 returns FEC_OK,
 * enqueues nothing and does not write *status_dev.
 *
 * fec_cluster_async: the signature of SURVEY §8(b); the workspace (fec_workspace_bytes(n)) is
 * taken stream-ordered from the device's default memory pool (cudaMallocAsync / cudaFreeAsync
 * on `stream`; under capture these become graph allocation nodes).
 * fec_cluster_ws_async: the same with a caller-provided workspace of at least
 * fec_workspace_bytes(n) bytes (kept alive until the stream has passed the call). */
fec_status_t fec_cluster_async(const float* points, int64_t n, float d_th, int64_t min_size,
                               int64_t max_size, int32_t* labels_out, void* stream, int32_t* status_dev);
fec_status_t fec_cluster_ws_async(const float* points, int64_t n, float d_th, int64_t min_size,
                                  int64_t max_size, int32_t* labels_out, void* workspace,
                                  size_t workspace_bytes, void* stream, int32_t* status_dev);

/* Synchronous form with a caller-provided workspace: fec_cluster_ws_async, then waits for
 * `stream` and returns the device status (FEC_ERR_NONFINITE / FEC_ERR_GRID_RANGE included). */
fec_status_t fec_cluster_ws(const float* points, int64_t n, float d_th, int64_t min_size,
                            int64_t max_size, int32_t* labels_out, void* workspace,
                            size_t workspace_bytes, void* stream);

/* Synchronous convenience form (the north-star signature): fec_cluster_async on the legacy
 * default stream with its own workspace, then waits and returns the device status.  Returns
 * FEC_ERR_OUT_OF_MEMORY if the workspace cannot be allocated. */
fec_status_t fec_cluster(const float* points, int64_t n, float d_th, int64_t min_size,
                         int64_t max_size, int32_t* labels_out);

/* End-to-end form with HOST buffers: points_host [n][3] fp32 and labels_host int32[n] are
 * host memory (pinned memory gives asynchronous copies).  Copies the points into the
 * workspace, clusters, copies the labels back, and synchronises `stream` before
 * returning.  `workspace` must hold fec_workspace_bytes_host(n) bytes of device memory. */
size_t fec_workspace_bytes_host(int64_t n);
fec_status_t fec_cluster_host(const float* points_host, int64_t n, float d_th,
                              int64_t min_size, int64_t max_size, int32_t* labels_host,
                              void* workspace, size_t workspace_bytes, void* stream);

/* Pipelined form of fec_cluster_host for a stream of clouds: the same host->device copy,
 * clustering and device->host copy are enqueued on `stream` and the call returns at once
 * (no host round trip): labels_host is valid after `stream` completes, and status_dev
 * (optional device / mapped int32, as fec_cluster_async) receives the device status.  With PINNED host
 * buffers and two streams (each with its own workspace and host buffers), consecutive calls
 * overlap one cloud's device->host copy and tail kernels with the next cloud's host->device
 * copy (PCIe is full duplex).  The host buffers must stay alive until the stream completes.
 * Errors: as fec_cluster_host. */
fec_status_t fec_cluster_host_async(const float* points_host, int64_t n, float d_th,
                                    int64_t min_size, int64_t max_size, int32_t* labels_host,
                                    void* workspace, size_t workspace_bytes, void* stream,
                                    int32_t* status_dev);

/* Fills *out with the statistics of this thread's last call whose status was FEC_OK.
 * Counters that need a device read-back (components, pair_tests, group_pairs) are
 * gathered only when fec_set_instrumentation(1) was set before that call. */
fec_status_t fec_get_stats(fec_stats_t* out);
void fec_set_instrumentation(int enable);

/* Grid-mode override for testing (thread-local): 0 = automatic (dense cell grid whenever
 * the bbox holds <= 32n + 2^26 cells, else Morton radix sort + hashed cells; in the dense
 * grid, a counting sort for spatially coherent input order and a radix sort of the cell
 * keys otherwise), 1 = hashed mode always, 2 = dense grid with the key sort, 3 = dense grid
 * with the counting sort (when the bbox allows the dense grid).  All modes compute
 * identical labels. */
void fec_set_grid_mode(int mode);

/* Test hook (thread-local): cap the queue of "uncertain" dense component pairs (DESIGN.md
 * §4) at `cap` entries (0 = default, n/8 + 65536).  Pairs beyond the cap are tested in
 * place by one thread each; labels are identical either way. */
void fec_set_item_cap(int64_t cap);

/* Test hook (thread-local): the self-allocating calls (fec_cluster, fec_cluster_async) ask the
 * allocator for `bytes` more than they need; a huge value makes the allocation really fail,
 * exercising the FEC_ERR_OUT_OF_MEMORY path.  0 (default) = off. */
void fec_debug_alloc_extra(size_t bytes);

/* Per-stage device timing.  With fec_set_timing(1), each call records CUDA events on its
 * stream at the stage boundaries (a1 validate+bbox+plan, a2 keys, a3 sort,
 * a4 gather, a5 tables, a6+a7 scan+union, a8 flatten, a9 stats, a10 relabel).
 * fec_get_stage_times() waits for the last event of this thread's last call and writes up
 * to max_stages durations in milliseconds; it returns the number of stages (or <0). */
void fec_set_timing(int enable);
int32_t fec_get_stage_times(float* ms_out, int32_t max_stages);
const char* fec_stage_name(int32_t stage);

/* ---- Batched clouds (the paper's per-scan mode, Table 4)
 *
 * nclouds independent clouds stored back to back: cloud c is points[offsets[c] ..
 * offsets[c+1]) (offsets: HOST array of nclouds + 1 int64, offsets[0] = 0, non-decreasing,
 * empty clouds allowed).  Every cloud is clustered as if by its own fec_cluster call: no edge
 * joins points of different clouds, sizes are per cloud, and labels_out[i] is the minimum
 * index INSIDE the point's cloud (0 .. size-1) of its component, or -1.  One pipeline serves
 * all clouds (each cloud gets its own grid origin and a separate band of cells); if the
 * stacked grid is too large for the dense mode the clouds are run one after another.
 * Device pointers as fec_cluster_ws; workspace of fec_batch_workspace_bytes(n_total,
 * nclouds) bytes.  Errors: as fec_cluster_ws (FEC_ERR_INVALID_ARGUMENT also for bad
 * offsets). */
size_t fec_batch_workspace_bytes(int64_t n_total, int32_t nclouds);
fec_status_t fec_cluster_batch_ws(const float* points, const int64_t* offsets, int32_t nclouds, float d_th,
                                  int64_t min_size, int64_t max_size, int32_t* labels_out, void* workspace,
                                  size_t workspace_bytes, void* stream);

/* ---- Multi-GPU slab path ------------------------------------
 *
 * PAPER.md's FEC is serial (L480 lists a parallel version as future work); the sharding is
 * this library's: the cloud is cut into spatial slabs along one axis at boundaries of a
 * grid whose cell edge exceeds d_th (reading A6), so every edge of the graph of Eq. 1
 * (L187-194) joins points of the same or of adjacent slabs.  Each rank holds its slab plus
 * a one-cell halo (the first cell layer of the next slab) and calls, on its own device:
 *
 *   1. fec_slab_local   clusters owned ∪ halo (a1..a8) and packs boundary records;
 *   2. an all-gather of the record buffers (NCCL, by the caller — the library does no
 *      communication; `world` buffers of fec_slab_record_words(rec_cap) int32 each,
 *      rank r's buffer at offset r);
 *   3. fec_slab_merge   replays the same boundary union-find on every rank and writes the
 *      global labels of the rank's owned points.
 *
 * The result over all ranks equals fec_cluster on the whole cloud: labels_owned[i] = the
 * minimum GLOBAL index (gidx) of the point's component, or -1 when the component's total
 * size (over all slabs) is outside [min_size, max_size].
 *
 * Local input order (caller's contract): points[0 .. n_first) are owned points in the slab's
 * first cell layer (the halo of the previous rank), points[n_first .. n_owned) the other
 * owned points, points[n_owned .. n_local) the halo (owned by the next rank).  gidx[i] is
 * the global input index of local point i (int32, unique over the owned points of all
 * ranks).  rec_cap must be the same on every rank and >= n_first + (n_local - n_owned) on
 * every rank.  Record buffer layout (int32 words): [nP, nC, 0, 0], then rec_cap (gidx, key)
 * pairs (space for rec_cap rounded up to even), then rec_cap (key, owned size, owned min
 * gidx, local root) quads — 16-byte aligned when the buffer is.
 * If the caller's halo/first-layer sets are not exactly one cell layer of a grid with edge
 * > d_th, the result is unspecified (not detected). */
typedef struct {
    int64_t opaque[8]; /* host memory; filled by fec_slab_local, read by fec_slab_merge */
} fec_slab_state_t;

/* int32 words of one rank's record buffer: 4 + 2*(rec_cap rounded up to even) + 4*rec_cap
 * (-1 if rec_cap < 0); a multiple of 4, so gathered buffers stay 16-byte aligned. */
int64_t fec_slab_record_words(int64_t rec_cap);

/* Device workspace for fec_slab_local + fec_slab_merge on n_local points (one buffer for
 * both calls; it carries the local forest from the first call to the second). */
size_t fec_slab_workspace_bytes(int64_t n_local, int32_t world, int64_t rec_cap);

/* Step 1 (device pointers; enqueued on `stream` with no host synchronisation, like
 * fec_cluster_ws_async; status_dev (optional) receives the device status; after an error the
 * records stay empty and fec_slab_merge leaves labels_owned untouched).  Writes the rank's
 * record buffer `records` (fec_slab_record_words(rec_cap) words) and fills *state.  Errors: as fec_cluster_ws, plus FEC_ERR_INVALID_ARGUMENT for
 * n_first/n_owned/n_local out of order or rec_cap too small.  n_local == 0 is valid (the
 * header is zeroed, nothing else is launched). */
fec_status_t fec_slab_local(const float* points, const int32_t* gidx, int64_t n_local, int64_t n_owned,
                            int64_t n_first, float d_th, int32_t* records, int64_t rec_cap, void* workspace,
                            size_t workspace_bytes, fec_slab_state_t* state, void* stream, int32_t* status_dev);

/* Step 3.  all_records: world * fec_slab_record_words(rec_cap) int32 (device), the gathered
 * buffers in rank order.  labels_owned: int32[n_owned] (device), in local order.  The
 * workspace and state must be those of this rank's fec_slab_local, with the workspace
 * sized by fec_slab_workspace_bytes(n_local, world, rec_cap).  Enqueued on `stream`; no
 * host synchronisation. */
fec_status_t fec_slab_merge(const int32_t* all_records, int32_t world, int32_t rank, int64_t min_size,
                            int64_t max_size, int32_t* labels_owned, void* workspace, size_t workspace_bytes,
                            const fec_slab_state_t* state, void* stream);

/* ---- Multi-GPU Mode B: index-sharded input -> spatial slabs, on the device
 *
 * When each rank starts with an arbitrary shard of the cloud (e.g. an index range) instead of
 * its slab, the slab decomposition of the path above is computed from device data: the same
 * rule as the host planner (paper_2208_07678_b200/dist.py plan_slabs): the cut axis is the
 * longest extent of the global bbox (ties: lowest axis), cell layers along it have edge
 * c = d_th*(1+2^-16) (reading A6) and are cut into `world` count-balanced slabs.  Per rank, on
 * `stream`, with one workspace of fec_part_workspace_bytes() bytes kept across the steps:
 *   1. fec_part_bbox   shard bbox -> bbox_out (device float[8]: min xyz, -max xyz, -nonfinite,
 *                      0); also zeroes `hist`.  Caller: all-reduce MIN of the 8 floats.
 *   2. fec_part_hist   histogram of the shard's layers -> hist (device int32[fec_part_max_layers()]).
 *                      Caller: all-reduce SUM.
 *   3. fec_part_plan   the cuts -> plan (device int64[4*world + 3]: cuts[world+1], owned[world],
 *                      first[world], halo[world], rec_cap, status); identical on every rank.
 *                      status = FEC_ERR_NONFINITE / FEC_ERR_GRID_RANGE if the cloud cannot be cut.
 *   4. fec_part_pack   with send_pts == NULL: counts[world] (device int64) of the points each rank
 *                      receives (its owned points, plus the first cell layer of the next slab as
 *                      its halo); then with the send buffers (sum(counts) points): the points and
 *                      gidx packed by destination rank.  Caller: all-to-all of counts, then of the
 *                      points and gidx.
 *   5. fec_part_order  the received points in the local order of fec_slab_local (first-layer
 *                      owned | other owned | halo); counts3 (device int64[3]) gives n_first =
 *                      counts3[0], n_owned = counts3[0] + counts3[1].
 * Then fec_slab_local / all-gather / fec_slab_merge with rec_cap = plan[4*world + 1].
 * Device pointers throughout; nothing synchronises the host (the caller reads counts and the
 * plan for the collectives' sizes). */
size_t fec_part_workspace_bytes(void);
int32_t fec_part_max_layers(void);
fec_status_t fec_part_bbox(const float* points, int64_t m, float* bbox_out, int32_t* hist, void* workspace,
                           size_t workspace_bytes, void* stream);
fec_status_t fec_part_hist(const float* points, int64_t m, const float* gbbox, float d_th, int32_t* hist,
                           void* workspace, size_t workspace_bytes, void* stream);
fec_status_t fec_part_plan(const int32_t* ghist, int32_t world, int64_t* plan_out, void* workspace,
                           size_t workspace_bytes, void* stream);
fec_status_t fec_part_pack(const float* points, const int32_t* gidx, int64_t m, const float* gbbox, float d_th,
                           const int64_t* plan, int32_t world, int64_t* counts, float* send_pts,
                           int32_t* send_gidx, void* workspace, size_t workspace_bytes, void* stream);
fec_status_t fec_part_order(const float* recv_pts, const int32_t* recv_gidx, int64_t k, const float* gbbox,
                            float d_th, const int64_t* plan, int32_t world, int32_t rank, int64_t* counts3,
                            float* out_pts, int32_t* out_gidx, void* workspace, size_t workspace_bytes,
                            void* stream);

/* Human-readable status text (static storage) and the last error detail of this thread. */
const char* fec_status_string(fec_status_t status);
const char* fec_last_error(void);

/* Library version string, e.g. "fec-b200 0.2 sm_100a". */
const char* fec_version(void);

/* The largest n the library accepts: union-find node ids (n points + 8 per dense-record slot,
 * record capacity rounded up to a power of two) must fit in int32.  Larger n is rejected with
 * FEC_ERR_INVALID_ARGUMENT before any launch. */
int64_t fec_max_points(void);

/* Diagnostic: evaluate the device predicate on m point pairs (a[k], b[k]), each [m][3]
 * fp32 device arrays; out[k] = pred (uint8 0/1), d2_out[k] = the fp32 squared distance
 * (d2_out may be NULL).  Exists so tests can check the fp32 operation order / no-FMA
 * contract of Eq. 1 on the GPU itself.  Synchronises `stream`. */
fec_status_t fec_debug_pred(const float* a, const float* b, int64_t m, float d_th, uint8_t* out,
                            float* d2_out, void* stream);

/* Host-only diagnostics of the fine sub-cell relations of the dense-grid path (DESIGN.md
 * §4; no device needed).  A grid cell is split into 4x4x4 sub-cells, bit x + 4y + 16z.
 *   fec_debug_subcell_tables: certain[64*s + a] / reach[64*s + a] (27*64 host uint64 each)
 *     = masks of the sub-cells b of the neighbour cell at slot s (offset (s%3-1, s/3%3-1,
 *     s/9-1)) that are certain-adjacent to / within reach of sub-cell a.  Returns 0.
 *   fec_debug_subcell_dilate(m): m plus every sub-cell certain-adjacent to one of m's.
 *   fec_debug_subcell_components(occ, comps): splits occ into certain-connected components
 *     (comps: 8 host uint64); returns their number, or -1 if more than 8 (never). */
int32_t fec_debug_subcell_tables(unsigned long long* certain, unsigned long long* reach);
unsigned long long fec_debug_subcell_dilate(unsigned long long m);
int32_t fec_debug_subcell_components(unsigned long long occ, unsigned long long* comps);

#ifdef __cplusplus
}
#endif

#endif /* FEC_H_ */
