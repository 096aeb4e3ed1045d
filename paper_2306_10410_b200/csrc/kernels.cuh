// Host-side launchers of the BOBA kernels (internal; the public surface is
// the C ABI in include/boba_b200.h, implemented in api.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace boba {

cudaError_t launch_first_hit(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n, uint32_t* first,
                             bool relaxed, int num_sms, cudaStream_t s);

// seen_ws (first_hit_workspace_bytes(), may be NULL) enables the two-stage sweep
size_t first_hit_workspace_bytes();
// bits_ws (first_hit_bits_workspace_bytes(n), may be NULL): for n > 2^23 the
// two-stage sweep then guards on an L2-resident seen-bitmap in waves
size_t first_hit_bits_workspace_bytes(uint32_t n);
cudaError_t launch_first_hit_shard(const uint32_t* I, const uint32_t* J, uint64_t m, uint64_t m_global, uint64_t e0,
                                   uint32_t n, uint32_t* first, bool relaxed, void* seen_ws, int num_sms,
                                   cudaStream_t s, void* bits_ws = nullptr);

size_t compact_workspace_bytes(uint64_t m, uint32_t n);
// hubs (may be NULL): kHubTableBytes table filled for phase 3 (hubs.cuh)
// rows_bound_out (device word, may be NULL): the number of vertices first seen
// in I -- every relabelled source row is below it
cudaError_t launch_compact(const uint32_t* first, uint64_t m, uint32_t n, uint32_t* order, uint32_t* label,
                           uint32_t* n_seen_out, unsigned long long* hubs, void* ws, size_t ws_bytes, int num_sms,
                           cudaStream_t s, uint32_t* rows_bound_out = nullptr);

// The first radix pass of COO->CSR needs the digit histogram of every
// 4096-row tile of I2; the relabel that writes I2 can produce it on the way
// (csr.cu decides where it lives and which digit; H == NULL: not wanted).
struct RowTileHist {
    uint32_t* H = nullptr;  // digit-major: H[d * tiles + t]
    uint64_t tiles = 0;
    uint32_t mask = 0;      // digit = row & mask (the first pass has shift 0)
    bool done = false;      // set by launch_relabel when it wrote H
};
RowTileHist coo_to_csr_first_hist(void* ws, size_t ws_bytes, uint64_t m, uint32_t n, bool weighted);
// the same histogram computed on its own from the row keys
cudaError_t launch_coo_to_csr_first_hist(const uint32_t* I2, uint64_t m, uint32_t n, void* ws, size_t ws_bytes,
                                         int num_sms, cudaStream_t s);

// counts (may be NULL): also the out-degree histogram of the new rows
cudaError_t launch_relabel(const uint32_t* I, const uint32_t* J, uint64_t m, const uint32_t* label,
                           const unsigned long long* hubs, uint32_t* I2, uint32_t* J2, uint32_t* counts, uint32_t n,
                           int num_sms, cudaStream_t s, RowTileHist* row_hist = nullptr);

cudaError_t launch_hist(const uint32_t* I, uint64_t m, uint32_t n, uint32_t* counts, int num_sms, cudaStream_t s);
cudaError_t launch_row_offsets(const uint32_t* counts, uint32_t n, uint32_t* offsets, unsigned long long* status,
                               unsigned* counter, cudaStream_t s);
size_t coo_to_csr_workspace_bytes(uint64_t m, uint32_t n, bool weighted);
// kernels a graph capture on this thread put inside conditional-node bodies
// (the taken branch's count), reset by the call
uint64_t take_conditional_body_kernels();
// first_hist_ready: the relabel already wrote the first pass's tile histogram
// (coo_to_csr_first_hist of the same workspace)
cudaError_t launch_coo_to_csr(const uint32_t* I2, const uint32_t* J2, const double* w, uint64_t m, uint32_t n,
                              const uint32_t* counts_in, uint32_t* offsets, uint32_t* indices, double* w_out,
                              void* ws, size_t ws_bytes, int num_sms, cudaStream_t s, bool first_hist_ready = false,
                              const uint32_t* rows_bound = nullptr);

size_t spmv_workspace_bytes(uint32_t n, uint64_t m);
cudaError_t launch_spmv(const uint32_t* offsets, const uint32_t* indices, const float* w, const float* x, float* y,
                        uint32_t n, uint64_t m, void* ws, size_t ws_bytes, cudaStream_t s, bool partitioned = false);
cudaError_t launch_spmv_f64(const uint32_t* offsets, const uint32_t* indices, const double* w, const double* x,
                            double* y, uint32_t n, uint64_t m, void* ws, size_t ws_bytes, cudaStream_t s, bool partitioned = false);

cudaError_t launch_rmat(int scale, uint64_t e0, uint64_t count, uint64_t seed, uint32_t* I, uint32_t* J,
                        int num_sms, cudaStream_t s);
cudaError_t launch_grid(uint32_t rows, uint32_t cols, uint32_t* I, uint32_t* J, int num_sms, cudaStream_t s);
cudaError_t launch_narrow(const int64_t* in, uint64_t count, uint64_t bound, uint32_t* out,
                          unsigned long long* first_bad, int num_sms, cudaStream_t s);
cudaError_t launch_widen(const uint32_t* in, uint64_t count, int64_t* out, int num_sms, cudaStream_t s);
cudaError_t launch_bias(const uint32_t* in, uint64_t count, uint32_t* out, int num_sms, cudaStream_t s);
cudaError_t launch_offset_ids(const uint32_t* in, uint64_t count, uint32_t delta, uint32_t* out, int num_sms,
                              cudaStream_t s);
size_t range_partition_workspace_bytes(uint64_t m, int parts);
cudaError_t launch_range_partition(const uint32_t* keys, const uint32_t* vals, uint64_t m, const uint32_t* bounds,
                                   int parts, uint32_t* keys_out, uint32_t* vals_out, uint32_t* counts_out, void* ws,
                                   size_t ws_bytes, int num_sms, cudaStream_t s, bool relative = false);
cudaError_t launch_iota(uint32_t* out, uint64_t count, int num_sms, cudaStream_t s);
size_t sort_pairs_workspace_bytes(uint64_t count, int key_bits);
cudaError_t launch_sort_pairs(const uint32_t* keys, const uint32_t* vals, uint64_t count, int key_bits,
                              uint32_t* keys_out, uint32_t* vals_out, void* ws, size_t ws_bytes, int num_sms,
                              cudaStream_t s);
size_t degree_order_workspace_bytes(uint64_t m, uint32_t n);
cudaError_t launch_total_degrees(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n, uint32_t* deg,
                                 int num_sms, cudaStream_t s);
cudaError_t launch_degree_order(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n, uint32_t* order,
                                uint32_t* label, void* ws, size_t ws_bytes, int num_sms, cudaStream_t s, bool hub);
size_t sort_by_destination_workspace_bytes(uint64_t m, uint32_t n);
cudaError_t launch_sort_by_destination(const uint32_t* I, const uint32_t* J, const double* w, uint64_t m, uint32_t n,
                                       uint32_t* I_out, uint32_t* J_out, double* w_out, void* ws, size_t ws_bytes,
                                       int num_sms, cudaStream_t s);
cudaError_t launch_spmv_f64_iter(const uint32_t* offsets, const uint32_t* indices, const double* w, const double* x,
                                 double* y, uint32_t n, uint64_t m, void* ws, size_t ws_bytes, cudaStream_t s,
                                 const int* stop, bool partitioned);
size_t pagerank_workspace_bytes(uint32_t n, uint64_t m, int num_sms);
cudaError_t launch_pagerank(const uint32_t* offsets, const uint32_t* indices, const double* w, uint32_t n, uint64_t m,
                            double damping, double tol, int max_iters, double* x, uint32_t* iterations, void* ws,
                            size_t ws_bytes, int num_sms, cudaStream_t s);
cudaError_t launch_gather_u32(const uint32_t* src, const uint32_t* idx, uint64_t count, uint32_t* out, int num_sms,
                              cudaStream_t s);

// neighbourhood line ratio (metrics.cu); out: device double
size_t nbr_workspace_bytes(uint64_t m, uint32_t n);
cudaError_t launch_nbr(const uint32_t* offsets, const uint32_t* indices, uint32_t n, uint64_t m, uint32_t line_size,
                       double* out, void* ws, size_t ws_bytes, int num_sms, cudaStream_t s);

// multi-GPU (sharded.py): windowed compaction (compact.cu) and the row cut (shard.cu)
size_t compact_window_workspace_bytes(uint64_t ml, uint32_t n);
cudaError_t launch_compact_window_mark(const uint32_t* first, uint32_t n, uint64_t m, uint64_t e0, uint64_t ml,
                                       uint32_t* counts, void* ws, size_t ws_bytes, int num_sms, cudaStream_t s);
cudaError_t launch_compact_window_assign(const uint32_t* first, uint32_t n, uint64_t m, uint64_t e0, uint64_t ml,
                                         const uint32_t* all_counts, int world, int rank, uint32_t* label, void* ws,
                                         size_t ws_bytes, cudaStream_t s);
cudaError_t launch_order_from_label(const uint32_t* label, uint32_t n, uint32_t* order, unsigned long long* hubs,
                                    int num_sms, cudaStream_t s);
uint32_t row_cut_buckets(uint32_t n);
cudaError_t launch_coarse_hist(const uint32_t* rows, uint64_t m, uint32_t n, uint32_t* hist, int num_sms,
                               cudaStream_t s);
cudaError_t launch_row_cut(const uint32_t* hist_g, const uint32_t* hist_l, uint32_t n, uint64_t m, int parts,
                           uint32_t* out, cudaStream_t s);

// host <-> device id transfers through pinned staging (hostio.cu); synchronous
cudaError_t host_h2d_ids(const int64_t* host, uint64_t count, uint64_t bound, uint32_t* dev, int64_t* bad,
                         cudaStream_t s);
cudaError_t host_d2h_ids(const uint32_t* dev, uint64_t count, int64_t* host, cudaStream_t s, bool unset_to_max = false);

}  // namespace boba
