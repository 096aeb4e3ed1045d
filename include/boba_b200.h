/*
 * boba_b200.h -- C ABI of the B200-native BOBA hot path (libboba_b200.so).
 *
 * This is the drop-in boundary for the reference package's native seam,
 * pkg/src/boba/_parallel.py ("All hot loops live here behind plain-array
 * signatures", _parallel.py:1-5), plus the numpy-level structural ops of
 * graph.py and kernels.py that sit on the same path.  Each entry point names
 * the reference interface it replaces (file:line relative to
 * /root/reference/pkg/src/boba/).  Binding recipes (ctypes / cffi) are in
 * INTEGRATION.md.
 *
 * Conventions (all entry points):
 *   - Vertex ids, positions and CSR offsets are uint32 (n <= 2^32 - 1,
 *     2m <= 2^32 - 2; the reference uses int64, graph.py:31 -- widen with
 *     boba_widen_ids).  First-occurrence "unset" is 0xFFFFFFFF (the
 *     reference's RANK_UNSET = INT64_MAX, _parallel.py:31).
 *   - Pointers are DEVICE pointers unless the name ends in _host.  Inputs are
 *     borrowed read-only (the reference never mutates inputs, graph.py:1-8);
 *     outputs and workspaces are caller-allocated.
 *   - Work is enqueued on `stream` (a cudaStream_t passed as void*); no
 *     entry point synchronises the host except the *_host ones.
 *   - Return 0 on success, a nonzero BOBA_E* code on failure; the message is
 *     in boba_last_error() (thread-local).  Invalid arguments are reported,
 *     never silently clamped.
 *   - Thread-safe across streams and devices (no hidden global state except
 *     per-device kernel attributes).
 */
#ifndef BOBA_B200_H
#define BOBA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BOBA_OK 0
#define BOBA_EINVAL 1   /* bad argument (null pointer, size out of range, small workspace) */
#define BOBA_ECUDA 2    /* CUDA runtime / launch error */
#define BOBA_ERANGE 3   /* an input id is out of [0, n) (reference MalformedGraphError) */
#define BOBA_ENOMEM 4   /* device allocation failed (context API) */

#define BOBA_UNSET_U32 0xFFFFFFFFu

/* Library identity and the last error message of the calling thread. */
int boba_abi_version(void);
const char *boba_last_error(void);

/* --- Phase 1: first occurrence ------------------------------------------
 * first[v] = min{ p : (p < m and I[p] == v) or (p >= m and J[p-m] == v) },
 * BOBA_UNSET_U32 if v never occurs.
 * Replaces _parallel.first_hit_chunked (_parallel.py:139-162) and the rank
 * half of first_hit_order_sequential (_parallel.py:111-136).  relaxed != 0
 * replaces first_hit_racy / run_racy_first_hit (_parallel.py:165-175,44-52):
 * guarded unsynchronised stores; every first[v] still names a position
 * holding v, but the minimum may be lost. */
int boba_first_occurrence(const uint32_t *I, const uint32_t *J, uint64_t m, uint32_t n,
                          uint32_t *first, int relaxed, void *stream);

/* Multi-GPU shard of phase 1: this rank holds edges
 * [e0, e0 + m_local) of a global list of m_global edges; local I[i] is global
 * position e0 + i and local J[i] is m_global + e0 + i.  Merging the per-rank
 * arrays with an elementwise min (NCCL allreduce-MIN after boba_bias_u32)
 * gives exactly boba_first_occurrence of the whole list -- the reference's
 * chunk-local-min merge, _parallel.py:139-162.
 * workspace (may be NULL; boba_first_occurrence_workspace_size() bytes)
 * enables the two-stage sweep with the shared-memory SeenSet of hubs; with
 * boba_first_occurrence_shard_workspace_size(n) bytes, also the prefix count
 * table that fills the SeenSet with the most frequent vertices first, and the
 * wave-guarded sweep the fused single-GPU call uses beyond L2 (n > 2^23). */
size_t boba_first_occurrence_workspace_size(void);
size_t boba_first_occurrence_shard_workspace_size(uint32_t n);
int boba_first_occurrence_shard(const uint32_t *I, const uint32_t *J, uint64_t m_local,
                                uint64_t m_global, uint64_t e0, uint32_t n, uint32_t *first,
                                int relaxed, void *workspace, size_t workspace_bytes, void *stream);

/* --- Phase 2: rank compaction -> permutation --------------------------
 * order[k] = the vertex with the k-th smallest first[] value, then the
 * vertices with first == UNSET in ascending id; label[order[k]] = k.
 * Replaces _parallel.compact_ranks (_parallel.py:178-201) and the label
 * construction of graph.Permutation (graph.py:205-208).  n_seen (device
 * scalar, may be NULL) receives the number of vertices that occur. */
size_t boba_compact_workspace_size(uint64_t m, uint32_t n);
int boba_compact(const uint32_t *first, uint64_t m, uint32_t n, uint32_t *order, uint32_t *label,
                 uint32_t *n_seen, void *workspace, size_t workspace_bytes, void *stream);

/* Phase 1 + 2: the deterministic BOBA permutation of ordering.boba_parallel
 * (ordering.py:99-151; == boba_sequential, ordering.py:59-96).  first
 * (n uint32) is an output too (the reference's return_ranks array). */
size_t boba_order_workspace_size(uint64_t m, uint32_t n);
int boba_order(const uint32_t *I, const uint32_t *J, uint64_t m, uint32_t n, int relaxed,
               uint32_t *first, uint32_t *order, uint32_t *label, void *workspace,
               size_t workspace_bytes, void *stream);

/* --- Phase 3: relabel ---------------------------------------------------
 * I2[e] = label[I[e]], J2[e] = label[J[e]]; edge order unchanged.
 * Replaces graph.apply_permutation (graph.py:280-289).  row_counts (n
 * uint32, may be NULL) additionally receives the out-degree histogram of
 * the relabelled rows (np.bincount of graph.py:270) for boba_coo_to_csr. */
int boba_relabel(const uint32_t *I, const uint32_t *J, uint64_t m, uint32_t n, const uint32_t *label,
                 uint32_t *I2, uint32_t *J2, uint32_t *row_counts, void *stream);

/* Out-degree histogram: replaces graph.degrees (graph.py:292-294). */
int boba_degrees(const uint32_t *I, uint64_t m, uint32_t n, uint32_t *deg, void *stream);

/* --- Phase 4: COO -> CSR, reference within-row order -------------------
 * offsets (n+1) = [0, cumsum(bincount(I2))]; row v of indices holds J2 of
 * the edges with I2 == v in edge-list order; weights (float64, may be NULL)
 * move with their edges bit-exactly.  Replaces graph.coo_to_csr
 * (graph.py:253-277) and _parallel.scatter_rows (_parallel.py:55-88).
 * row_counts may be NULL (computed) or the histogram from boba_relabel. */
size_t boba_coo_to_csr_workspace_size(uint64_t m, uint32_t n, int weighted);
int boba_coo_to_csr(const uint32_t *I2, const uint32_t *J2, const double *weights, uint64_t m,
                    uint32_t n, const uint32_t *row_counts, uint32_t *offsets, uint32_t *indices,
                    double *weights_out, void *workspace, size_t workspace_bytes, void *stream);
/* The same conversion in two steps, so the row keys can be histogrammed while
 * the columns are still in flight (the multi-GPU owner overlaps its column
 * all-to-all this way): boba_coo_to_csr_first_hist(I2, ...) writes the first
 * radix pass's tile histogram into the workspace; a following
 * boba_coo_to_csr_ex(..., first_hist_ready = 1, ...) with the same I2, m, n
 * and workspace skips that pass's upsweep (row_counts must be NULL then).
 * Same results as boba_coo_to_csr. */
int boba_coo_to_csr_first_hist(const uint32_t *I2, uint64_t m, uint32_t n, void *workspace,
                               size_t workspace_bytes, void *stream);
int boba_coo_to_csr_ex(const uint32_t *I2, const uint32_t *J2, const double *weights, uint64_t m,
                       uint32_t n, const uint32_t *row_counts, uint32_t *offsets, uint32_t *indices,
                       double *weights_out, void *workspace, size_t workspace_bytes,
                       int first_hist_ready, void *stream);

/* --- Phase 5: SpMV (fp32) -------------------------------------------------
 * y[v] = sum over row v of weights[k] * x[indices[k]] (weights NULL = 1);
 * empty rows give 0.  Replaces kernels.spmv_pull (kernels.py:30-52; the
 * reference accumulates in float64 -- results agree to fp32 rounding).
 * Deterministic run to run. */
size_t boba_spmv_workspace_size(uint32_t n, uint64_t m);
int boba_spmv(const uint32_t *offsets, const uint32_t *indices, const float *weights,
              const float *x, float *y, uint32_t n, uint64_t m, void *workspace,
              size_t workspace_bytes, void *stream);
/* Same, for iterative callers (the k SpMV iterations of the reference bench,
 * bench.py:152-156): reuse_partition != 0 skips the merge-path partition
 * (one binary search per tile) and uses the one the previous call left in
 * `workspace` -- the caller guarantees that call had the same offsets
 * contents, n and m.  The partition depends on the structure only. */
int boba_spmv_ex(const uint32_t *offsets, const uint32_t *indices, const float *weights, const float *x,
                 float *y, uint32_t n, uint64_t m, void *workspace, size_t workspace_bytes,
                 int reuse_partition, void *stream);
int boba_spmv_f64_ex(const uint32_t *offsets, const uint32_t *indices, const double *weights, const double *x,
                     double *y, uint32_t n, uint64_t m, void *workspace, size_t workspace_bytes,
                     int reuse_partition, void *stream);

/* Same in float64 -- the reference's own precision (kernels.py:30-52); the
 * drop-in spmv_pull uses it.  Same workspace size. */
int boba_spmv_f64(const uint32_t *offsets, const uint32_t *indices, const double *weights,
                  const double *x, double *y, uint32_t n, uint64_t m, void *workspace,
                  size_t workspace_bytes, void *stream);

/* --- Fused device pipeline (reference bench.py:135-149: reorder = BOBA +
 * apply_permutation, convert = coo_to_csr) ------------------------------ */
size_t boba_reorder_to_csr_workspace_size(uint64_t m, uint32_t n, int weighted);
int boba_reorder_to_csr(const uint32_t *I, const uint32_t *J, const double *weights, uint64_t m,
                        uint32_t n, uint32_t *first, uint32_t *order, uint32_t *label, uint32_t *I2,
                        uint32_t *J2, uint32_t *offsets, uint32_t *indices, double *weights_out,
                        void *workspace, size_t workspace_bytes, void *stream);
/* Same, recording events[0..4] (cudaEvent_t, entries may be NULL) on
 * `stream` at the phase boundaries: before first occurrence, before
 * compaction, before relabel, before COO->CSR, after COO->CSR. */
int boba_reorder_to_csr_timed(const uint32_t *I, const uint32_t *J, const double *weights, uint64_t m,
                              uint32_t n, uint32_t *first, uint32_t *order, uint32_t *label,
                              uint32_t *I2, uint32_t *J2, uint32_t *offsets, uint32_t *indices,
                              double *weights_out, void *workspace, size_t workspace_bytes,
                              void *stream, void *const *events);

/* --- Captured pipeline (CUDA graph; the reference's reorder + convert
 * phases, bench.py:135-149, replayed with one launch) ----------------------
 * Records one boba_reorder_to_csr call on these fixed device buffers (after
 * one eager run, which also produces outputs) into a CUDA graph; each
 * boba_graph_launch replays the whole pipeline with a single launch.  The
 * buffers must stay allocated and the input contents may change between
 * launches; (m, n) are fixed.  n >= 2.  Creation synchronises the device
 * first (the eager run uses a private stream, so pending writes of I and J
 * on any caller stream must have landed).  In the captured step COO->CSR
 * chooses its radix plan on the device at every replay (a conditional graph
 * node): one key bit fewer when the relabelled rows allow it, the
 * full-width plan otherwise -- the outputs are the same either way. */
typedef struct boba_graph boba_graph;
int boba_reorder_to_csr_graph_create(const uint32_t *I, const uint32_t *J, uint64_t m, uint32_t n,
                                     uint32_t *first, uint32_t *order, uint32_t *label, uint32_t *I2,
                                     uint32_t *J2, uint32_t *offsets, uint32_t *indices, void *workspace,
                                     size_t workspace_bytes, boba_graph **out);
/* The same graph with event-record nodes at the phase boundaries (events as
 * in boba_reorder_to_csr_timed; each replay records them), for per-phase
 * times of exactly the replayed step. */
int boba_reorder_to_csr_graph_create_timed(const uint32_t *I, const uint32_t *J, uint64_t m, uint32_t n,
                                           uint32_t *first, uint32_t *order, uint32_t *label, uint32_t *I2,
                                           uint32_t *J2, uint32_t *offsets, uint32_t *indices, void *workspace,
                                           size_t workspace_bytes, void *const *events, boba_graph **out);
int boba_graph_launch(boba_graph *graph, void *stream);
void boba_reorder_to_csr_graph_destroy(boba_graph *graph);
/* Number of kernel launches one boba_graph_launch replays (the graph's
 * kernel nodes; memset nodes are not counted). */
int boba_graph_kernel_nodes(const boba_graph *graph, uint64_t *count);

/* --- Host-buffer pipeline (end to end) ----------------------------------
 * A context owns device buffers for graphs up to (max_m, max_n) on the
 * current device plus a stream.  boba_ctx_reorder_to_csr_host copies I, J
 * host -> device, runs the fused pipeline and copies order, label, offsets
 * and indices back (I2/J2 too when non-NULL).  Host buffers may be pageable
 * or pinned (pinned is faster). */
typedef struct boba_ctx boba_ctx;
int boba_ctx_create(uint64_t max_m, uint32_t max_n, boba_ctx **out);
void boba_ctx_destroy(boba_ctx *ctx);
int boba_ctx_reorder_to_csr_host(boba_ctx *ctx, const uint32_t *I_host, const uint32_t *J_host,
                                 uint64_t m, uint32_t n, uint32_t *order_host, uint32_t *label_host,
                                 uint32_t *I2_host, uint32_t *J2_host, uint32_t *offsets_host,
                                 uint32_t *indices_host);
/* Asynchronous form: enqueue one graph and return at once with *ticket.  A
 * context has two buffer slots, so graph k+1's host->device copy and graph
 * k's device->host copy overlap each other and the compute of either (the
 * copies run on their own streams).  The caller keeps the host inputs intact,
 * and does not read the host outputs, until boba_ctx_wait(ticket) returns.
 * Host buffers should be pinned; pageable buffers serialise the copies. */
int boba_ctx_submit_host(boba_ctx *ctx, const uint32_t *I_host, const uint32_t *J_host, uint64_t m,
                         uint32_t n, uint32_t *order_host, uint32_t *label_host, uint32_t *I2_host,
                         uint32_t *J2_host, uint32_t *offsets_host, uint32_t *indices_host,
                         uint64_t *ticket);
int boba_ctx_wait(boba_ctx *ctx, uint64_t ticket);

/* --- Locality metric (reference metrics.py:90-115 nbr) -------------------
 * Mean over rows with neighbours of (distinct index / line_size lines) /
 * (row degree); *out is a device double.  m and n must be positive
 * (the reference raises UndefinedMetricError without edges). */
size_t boba_nbr_workspace_size(uint64_t m, uint32_t n);
int boba_nbr(const uint32_t *offsets, const uint32_t *indices, uint32_t n, uint64_t m, uint32_t line_size,
             double *out, void *workspace, size_t workspace_bytes, void *stream);

/* --- Plumbing and input generators --------------------------------------- */
/* int64 -> uint32 with the reference's range check (graph.py:99-106):
 * returns BOBA_ERANGE and *bad_index (host, may be NULL) = first offending
 * index if any value is outside [0, bound).  Synchronises `stream`. */
int boba_narrow_ids(const int64_t *in, uint64_t count, uint64_t bound, uint32_t *out,
                    int64_t *bad_index, void *stream);
int boba_widen_ids(const uint32_t *in, uint64_t count, int64_t *out, void *stream);
/* Host int64 ids -> device uint32 (narrowed on host threads into pinned
 * staging, chunked so narrowing overlaps the copies), with the same range
 * check as boba_narrow_ids; and device uint32 -> host int64 (widened on host
 * threads while the next chunk copies).  Both return once `host` may be
 * reused / read (synchronous on `stream`).  The drop-in's transfers. */
int boba_host_to_device_ids(const int64_t *host, uint64_t count, uint64_t bound, uint32_t *dev,
                            int64_t *bad_index, void *stream);
int boba_device_to_host_ids(const uint32_t *dev, uint64_t count, int64_t *host, void *stream);
/* boba_device_to_host_ids for a first-occurrence array: 0xFFFFFFFF (never
 * seen) widens to INT64_MAX, the reference's RANK_UNSET (_parallel.py:31), in
 * the same pass (replaces the numpy fix-up of `boba_parallel(...,
 * return_ranks=True)`'s rank array, ordering.py:99-151). */
int boba_device_to_host_ranks(const uint32_t *dev, uint64_t count, int64_t *host, void *stream);
/* offsets[0..n] = exclusive prefix sum of counts[0..n) (offsets[n] = total):
 * np.cumsum of graph.py:270-272 on the device. */
size_t boba_exclusive_scan_workspace_size(uint64_t count);
int boba_exclusive_scan_u32(const uint32_t *counts, uint32_t n, uint32_t *offsets, void *workspace,
                            size_t workspace_bytes, void *stream);
/* out[i] = in[i] ^ 0x80000000: an order-preserving map from uint32 to int32
 * (UNSET stays the maximum), so first[] can be merged with a signed MIN
 * collective. Its own inverse. */
int boba_bias_u32(const uint32_t *in, uint64_t count, uint32_t *out, void *stream);
/* out[i] = in[i] + delta (mod 2^32): shift global row ids to a local range. */
int boba_offset_ids(const uint32_t *in, uint64_t count, uint32_t delta, uint32_t *out, void *stream);
/* Stable partition of (key, val) pairs by key range: part p holds the keys in
 * [bounds[p], bounds[p+1]) (bounds: parts+1 ascending device uint32, only
 * bounds[1..parts-1] are read), in input order; counts_out[p] (device) = pairs
 * in part p.  The send side of the multi-GPU all-to-all by row range. */
/* Compaction of a merged first[] (2 m_global positions) and relabel of a
 * local edge shard (m edges) with the hub label table the compaction builds
 * -- phases 2 and 3 of the multi-GPU pipeline (sharded.py), as in the fused
 * single-GPU call.  Replaces _parallel.compact_ranks (_parallel.py:178-201)
 * + graph.apply_permutation (graph.py:280-289) on one shard. */
size_t boba_compact_relabel_workspace_size(uint64_t m_global, uint32_t n);
int boba_compact_relabel(const uint32_t *first, uint64_t m_global, uint32_t n, const uint32_t *I,
                         const uint32_t *J, uint64_t m, uint32_t *order, uint32_t *label, uint32_t *I2,
                         uint32_t *J2, void *workspace, size_t workspace_bytes, void *stream);

size_t boba_range_partition_workspace_size(uint64_t m, int parts);
int boba_range_partition(const uint32_t *keys, const uint32_t *vals, uint64_t m,
                         const uint32_t *bounds, int parts, uint32_t *keys_out, uint32_t *vals_out,
                         uint32_t *counts_out, void *workspace, size_t workspace_bytes,
                         void *stream);
/* As boba_range_partition; relative_keys != 0 writes each key minus its
 * part's first row (bounds[p]), i.e. row ids local to the owner; counts_out
 * may be NULL. */
int boba_range_partition_ex(const uint32_t *keys, const uint32_t *vals, uint64_t m,
                            const uint32_t *bounds, int parts, int relative_keys, uint32_t *keys_out,
                            uint32_t *vals_out, uint32_t *counts_out, void *workspace,
                            size_t workspace_bytes, void *stream);

/* --- Multi-GPU phases (sharded.py; one process per GPU) -------------------
 * The collectives between these calls belong to the caller: NCCL through
 * torch.distributed in sharded.py; a C/C++ caller issues the same
 * ncclAllReduce / ncclAllGather / ncclSend+ncclRecv on its own ncclComm_t
 * (the sequence is spelled out in INTEGRATION.md §4).  Rank r of P holds the
 * contiguous edges [e0, e0 + m_local) of the m_global-edge list, i.e.
 * positions [e0, e0 + m_local) of I and [m_global + e0, ...) of J.
 *
 * Phase 1: boba_first_occurrence_shard, boba_bias_u32,
 *   [allreduce-MIN over n int32], boba_bias_u32.
 * Phase 2 (compact_ranks, _parallel.py:178-201, split by position window):
 *   boba_compact_shard_mark: marks the vertices whose first position lies in
 *     this rank's windows; counts[2] (device) = how many were first seen in
 *     its I window and in its J window.
 *   [allgather of counts -> all_counts[2P], rank-major]
 *   boba_compact_shard_assign (same workspace, untouched since _mark):
 *     label_partial[v] = global rank of each owned vertex, 0 for the other
 *     seen vertices; never-seen vertices get n_seen + their ascending rank on
 *     rank 0 and 0 elsewhere.
 *   [allreduce-SUM of label_partial over n words -> label, replicated]
 *   boba_order_from_label: order[label[v]] = v, plus (hubs != NULL,
 *     boba_hub_table_bytes()) the hub label table of the smallest labels.
 * Phase 3 (apply_permutation, graph.py:280-289): boba_relabel_hubs.
 * Phase 4 (coo_to_csr, graph.py:253-277, rows split by range):
 *   boba_row_cut_hist: coarse histogram of the local rows
 *     (boba_row_cut_buckets(n) words, bucket = row >> max(0, bits(n-1) - 15)).
 *   [allreduce-SUM of the histogram]
 *   boba_row_cut(global hist, local hist): out[3P+2] = row bounds b[0..P]
 *     (edge-balanced, on bucket boundaries), offsets[b_k] (P+1 words) and the
 *     edges this rank sends to each owner (P words).
 *   boba_range_partition_ex(bounds = out, relative_keys = 1): send buffers.
 *   [all-to-all of keys and of values, in rank order]
 *   boba_coo_to_csr on the received pairs (rows local to [b_r, b_r+1)). */
size_t boba_compact_shard_workspace_size(uint64_t m_local, uint32_t n);
int boba_compact_shard_mark(const uint32_t *first, uint32_t n, uint64_t m_global, uint64_t e0,
                            uint64_t m_local, uint32_t *counts, void *workspace, size_t workspace_bytes,
                            void *stream);
int boba_compact_shard_assign(const uint32_t *first, uint32_t n, uint64_t m_global, uint64_t e0,
                              uint64_t m_local, const uint32_t *all_counts, int world, int rank,
                              uint32_t *label_partial, void *workspace, size_t workspace_bytes, void *stream);
size_t boba_hub_table_bytes(void);
int boba_order_from_label(const uint32_t *label, uint32_t n, uint32_t *order, void *hubs, void *stream);
int boba_relabel_hubs(const uint32_t *I, const uint32_t *J, uint64_t m, uint32_t n, const uint32_t *label,
                      const void *hubs, uint32_t *I2, uint32_t *J2, void *stream);
uint32_t boba_row_cut_buckets(uint32_t n);
int boba_row_cut_hist(const uint32_t *rows, uint64_t m_local, uint32_t n, uint32_t *hist, void *stream);
int boba_row_cut(const uint32_t *hist_global, const uint32_t *hist_local, uint32_t n, uint64_t m_global,
                 int world, uint32_t *out, void *stream);

/* The whole sequence above in one call on the caller's NCCL communicator
 * (nccl_comm: an ncclComm_t; libnccl.so.2 is resolved at first use,
 * preferring the copy already loaded in the process).  Outputs: the
 * replicated first / order / label (n words each), this rank's relabelled
 * shard I2 / J2 (m_local), and its rows of the CSR: offsets (capacity n + 1
 * words, local to the owned rows) and indices (capacity recv_capacity).
 * *out gets the owned row range, the edge count and offsets[row_lo] of the
 * global CSR; bounds_host (may be NULL, world + 1 words) every owner's rows; returns BOBA_EINVAL (with out->nnz set) if recv_capacity is
 * too small.  One host synchronisation.  Replaces, across ranks, the
 * reference's boba_parallel + apply_permutation + coo_to_csr
 * (ordering.py:99-151, graph.py:253-289). */
typedef struct boba_shard_result {
    uint32_t row_lo, row_hi;    /* this rank owns CSR rows [row_lo, row_hi) */
    uint64_t nnz;               /* entries of indices (edges received) */
    uint64_t row_edge_offset;   /* global offsets[row_lo] */
} boba_shard_result;
size_t boba_sharded_workspace_size(uint64_t m_local, uint32_t n, int world, uint64_t recv_capacity);
int boba_sharded_reorder_to_csr_nccl(const uint32_t *I, const uint32_t *J, uint64_t m_local, uint64_t m_global,
                                     uint64_t e0, uint32_t n, void *nccl_comm, uint32_t *first,
                                     uint32_t *order, uint32_t *label, uint32_t *I2, uint32_t *J2,
                                     uint32_t *offsets, uint32_t *indices, uint64_t recv_capacity,
                                     boba_shard_result *out, uint32_t *bounds_host, void *workspace, size_t workspace_bytes,
                                     void *stream);

/* out[i] = src[idx[i]] (permutation application on vertex arrays). */
int boba_gather_u32(const uint32_t *src, const uint32_t *idx, uint64_t count, uint32_t *out,
                    void *stream);
/* --- Orderings and edge sorts beside BOBA ----------------
 * deg[v] = #{e : I[e] == v} + #{e : J[e] == v}: total degree, reference
 * graph.degrees (graph.py:297-300). */
int boba_total_degrees(const uint32_t *I, const uint32_t *J, uint64_t m, uint32_t n, uint32_t *deg,
                       void *stream);
/* Degree ordering: order = vertices by descending total degree, ties by
 * ascending id (np.lexsort((arange(n), -deg))); label[order[k]] = k.
 * Replaces ordering.degree_order (ordering.py:160-164). */
size_t boba_degree_order_workspace_size(uint64_t m, uint32_t n);
int boba_degree_order(const uint32_t *I, const uint32_t *J, uint64_t m, uint32_t n, uint32_t *order,
                      uint32_t *label, void *workspace, size_t workspace_bytes, void *stream);
/* Hub ordering: vertices with total degree above the mean (deg * n > 2m)
 * first by descending degree, ties by id; the rest after them in id order.
 * Workspace as boba_degree_order.  Replaces ordering.hub_order
 * (ordering.py:167-176). */
int boba_hub_order(const uint32_t *I, const uint32_t *J, uint64_t m, uint32_t n, uint32_t *order,
                   uint32_t *label, void *workspace, size_t workspace_bytes, void *stream);
/* Stable sort of the edge list by destination J (ties keep edge order),
 * weights (float64, may be NULL) move bit-exactly.  Replaces
 * graph.sort_coo_by_destination (graph.py:303-307). */
size_t boba_sort_coo_by_destination_workspace_size(uint64_t m, uint32_t n);
int boba_sort_coo_by_destination(const uint32_t *I, const uint32_t *J, const double *w, uint64_t m,
                                 uint32_t n, uint32_t *I_out, uint32_t *J_out, double *w_out,
                                 void *workspace, size_t workspace_bytes, void *stream);

/* PageRank by power iteration on a forward CSR (row v = out-neighbours):
 * uniform teleport, dangling mass redistributed uniformly, stop when the L1
 * change < tol or after max_iters rounds; x (n float64) receives the ranks,
 * *iterations (device uint32, may be NULL) the rounds run.  Fully
 * device-resident (no host synchronisation per round), deterministic.
 * Replaces kernels.pagerank (kernels.py:57-107); BOBA_EINVAL unless
 * 0 < damping < 1 (the reference's ValueError). */
size_t boba_pagerank_workspace_size(uint32_t n, uint64_t m);
int boba_pagerank(const uint32_t *offsets, const uint32_t *indices, const double *w, uint32_t n,
                  uint64_t m, double damping, double tol, int max_iters, double *x,
                  uint32_t *iterations, void *workspace, size_t workspace_bytes, void *stream);

/* Graph500 R-MAT (a,b,c,d = .57,.19,.19,.05), m = edge_factor << scale
 * i.i.d. edges in generation order; identical to oracle_rmat_edges. */
int boba_generate_rmat(int scale, uint64_t m, uint64_t seed, uint32_t *I, uint32_t *J, void *stream);
/* Edges [e0, e0 + count) of the same stream (for per-rank shards). */
int boba_generate_rmat_range(int scale, uint64_t e0, uint64_t count, uint64_t seed, uint32_t *I,
                             uint32_t *J, void *stream);
/* 4-neighbour grid, reference generators.py:100-111 generate_grid. */
int boba_generate_grid(uint32_t rows, uint32_t cols, uint32_t *I, uint32_t *J, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* BOBA_B200_H */
