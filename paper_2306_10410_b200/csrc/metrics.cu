// Neighbourhood line ratio (NBR) of a CSR, the locality score that the
// SpMV's L1/L2 hit rates track.
//
// Reference: pkg/src/boba/metrics.py:90-115 nbr: over rows with at least one
// neighbour, (number of distinct lines index / line_size among the row's
// neighbours) / (row degree as a multiset), averaged.
//
// GPU form: expand the row id of every nonzero, sort (row, line) pairs
// lexicographically with two stable LSD sorts (by line, then by row), count
// the pair boundaries per row, then a fixed-order fp64 reduction of the
// per-row ratios (bitwise deterministic; differs from numpy's pairwise mean
// only in summation order).
#include "common.cuh"
#include "kernels.cuh"

namespace boba {

__global__ void k_expand_rows(const uint32_t* __restrict__ offsets, uint32_t n, uint32_t* rows) {
    const unsigned lane = lane_id();
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < n; r += warps) {
        const uint32_t b = __ldg(offsets + r), e = __ldg(offsets + r + 1);
        for (uint32_t k = b + lane; k < e; k += 32) rows[k] = (uint32_t)r;
    }
}

__global__ void k_lines(const uint32_t* __restrict__ indices, uint64_t m, uint32_t line_size, uint32_t* lines) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += stride)
        lines[k] = __ldg(indices + k) / line_size;
}

// rows/lines sorted by (row, line): one count per first occurrence of a pair
__global__ void k_line_boundaries(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ lines, uint64_t m,
                                  uint32_t* counts) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += stride) {
        const uint32_t r = __ldg(rows + k), l = __ldg(lines + k);
        if (k == 0 || __ldg(rows + k - 1) != r || __ldg(lines + k - 1) != l) atomicAdd(counts + r, 1u);
    }
}

// Per-CTA partial sums of counts[r] / deg[r] over rows with deg > 0 (and
// their number), in row order; the last step folds the partials in order.
constexpr int kNbrNT = 256;
__global__ void __launch_bounds__(kNbrNT) k_nbr_partials(const uint32_t* __restrict__ offsets,
                                                         const uint32_t* __restrict__ counts, uint32_t n,
                                                         double* psum, unsigned long long* pcnt) {
    __shared__ double s_sum[kNbrNT];
    __shared__ unsigned long long s_cnt[kNbrNT];
    const uint64_t r = (uint64_t)blockIdx.x * kNbrNT + threadIdx.x;
    double v = 0.0;
    unsigned long long c = 0;
    if (r < n) {
        const uint32_t d = __ldg(offsets + r + 1) - __ldg(offsets + r);
        if (d) {
            v = (double)__ldg(counts + r) / (double)d;
            c = 1;
        }
    }
    s_sum[threadIdx.x] = v;
    s_cnt[threadIdx.x] = c;
    __syncthreads();
    for (int o = kNbrNT / 2; o > 0; o >>= 1) {  // fixed pairwise tree: deterministic
        if ((int)threadIdx.x < o) {
            s_sum[threadIdx.x] += s_sum[threadIdx.x + o];
            s_cnt[threadIdx.x] += s_cnt[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        psum[blockIdx.x] = s_sum[0];
        pcnt[blockIdx.x] = s_cnt[0];
    }
}

__global__ void k_nbr_final(const double* psum, const unsigned long long* pcnt, uint64_t parts, double* out) {
    __shared__ double s_sum[kNbrNT];
    __shared__ unsigned long long s_cnt[kNbrNT];
    double v = 0.0;
    unsigned long long c = 0;
    for (uint64_t i = threadIdx.x; i < parts; i += kNbrNT) {  // each thread: a fixed strided subsequence
        v += psum[i];
        c += pcnt[i];
    }
    s_sum[threadIdx.x] = v;
    s_cnt[threadIdx.x] = c;
    __syncthreads();
    for (int o = kNbrNT / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            s_sum[threadIdx.x] += s_sum[threadIdx.x + o];
            s_cnt[threadIdx.x] += s_cnt[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = s_cnt[0] ? s_sum[0] / (double)s_cnt[0] : 0.0;
}

static int nbits(uint64_t v) { return v == 0 ? 0 : 64 - __builtin_clzll(v); }

namespace {
struct NbrWs {
    uint32_t *rows, *lines, *a, *b, *counts;
    double* psum;
    unsigned long long* pcnt;
    void* sort_ws;
    size_t sort_bytes, total;
};
NbrWs carve_nbr(void* base, uint64_t m, uint32_t n) {
    NbrWs w{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return base ? static_cast<char*>(base) + o : nullptr;
    };
    w.rows = (uint32_t*)take(m * 4 + 16);
    w.lines = (uint32_t*)take(m * 4 + 16);
    w.a = (uint32_t*)take(m * 4 + 16);
    w.b = (uint32_t*)take(m * 4 + 16);
    w.counts = (uint32_t*)take((size_t)n * 4 + 16);
    const uint64_t parts = ceil_div(n ? n : 1, kNbrNT);
    w.psum = (double*)take(parts * 8);
    w.pcnt = (unsigned long long*)take(parts * 8);
    w.sort_bytes = sort_pairs_workspace_bytes(m, 32);
    w.sort_ws = take(w.sort_bytes);
    w.total = off;
    return w;
}
}  // namespace

size_t nbr_workspace_bytes(uint64_t m, uint32_t n) { return carve_nbr(nullptr, m, n).total; }

cudaError_t launch_nbr(const uint32_t* offsets, const uint32_t* indices, uint32_t n, uint64_t m, uint32_t line_size,
                       double* out, void* ws, size_t ws_bytes, int num_sms, cudaStream_t s) {
    NbrWs W = carve_nbr(ws, m, n);
    if (ws_bytes < W.total || line_size == 0 || m == 0 || n == 0) return cudaErrorInvalidValue;
    const uint64_t cap = (uint64_t)num_sms * 8;
    auto grid = [&](uint64_t work) { const uint64_t b = ceil_div(work, 256); return (unsigned)(b < cap ? b : cap); };
    k_expand_rows<<<grid((uint64_t)n * 32), 256, 0, s>>>(offsets, n, W.rows);
    k_lines<<<grid(m), 256, 0, s>>>(indices, m, line_size, W.lines);
    // (row, line) lexicographic: stable sort by line, then stable sort by row
    const int line_bits = nbits((uint64_t)(n ? n - 1 : 0) / line_size);
    cudaError_t e = launch_sort_pairs(W.lines, W.rows, m, line_bits, W.a, W.b, W.sort_ws, W.sort_bytes, num_sms, s);
    if (e != cudaSuccess) return e;
    e = launch_sort_pairs(W.b, W.a, m, nbits(n ? n - 1 : 0), W.rows, W.lines, W.sort_ws, W.sort_bytes, num_sms, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(W.counts, 0, (size_t)n * 4, s);
    if (e != cudaSuccess) return e;
    k_line_boundaries<<<grid(m), 256, 0, s>>>(W.rows, W.lines, m, W.counts);
    const uint64_t parts = ceil_div(n, kNbrNT);
    k_nbr_partials<<<(unsigned)parts, kNbrNT, 0, s>>>(offsets, W.counts, n, W.psum, W.pcnt);
    k_nbr_final<<<1, kNbrNT, 0, s>>>(W.psum, W.pcnt, parts, out);
    return cudaGetLastError();
}

}  // namespace boba
