// Multi-GPU helpers for the row-partitioned CSR (paper_2306_10410_b200/sharded.py).
//
// Each rank sorts its contiguous edge shard into a local CSR over all n rows
// (the same stable radix COO->CSR as one GPU), so the edges a rank must send
// to the owner of rows [b_k, b_k+1) are one contiguous run of its local
// indices, already in row order and, within a row, in shard order.  The owner
// receives one such run per sender (in rank order) plus each sender's
// per-row counts, and interleaves them row by row: row r = sender 0's
// entries, then sender 1's, ...  Shards are contiguous in edge order, so that
// is global edge order -- the reference's within-row order
// (_parallel.py:55-88) -- and the CSR is bit-exact.
#include "common.cuh"
#include "kernels.cuh"

namespace boba {

__global__ void k_adjacent_diff(const uint32_t* __restrict__ in, uint64_t count, uint32_t* out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
        out[i] = __ldg(in + i + 1) - __ldg(in + i);
}

// Segment s = k * rows + r is sender k's run for row r: it starts at
// src_start[s] in recv (rank-major exclusive scan of the counts) and goes to
// dst[s] = out_off[r] + (entries of senders < k in row r) in the output.
__global__ void k_merge_dst(const uint32_t* __restrict__ counts, int parts, uint32_t rows,
                            const uint32_t* __restrict__ out_off, uint32_t* __restrict__ dst) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += stride) {
        uint32_t d = __ldg(out_off + r);
        for (int k = 0; k < parts; k++) {
            dst[(uint64_t)k * rows + r] = d;
            d += __ldg(counts + (uint64_t)k * rows + r);
        }
    }
}

// Item-balanced copy: each CTA moves kMcTile consecutive recv entries.  The
// segments it spans are located once per CTA (binary search over src_start)
// and their (start, dst) pairs staged in shared memory; each entry then finds
// its segment by a search in shared memory (in global memory if the chunk
// spans more than kMcSegs segments, i.e. runs of empty rows).
constexpr int kMcNT = 256, kMcIPT = 8, kMcTile = kMcNT * kMcIPT, kMcSegs = 4096;

__device__ __forceinline__ uint64_t seg_of(const uint32_t* a, uint64_t lo, uint64_t hi, uint32_t p) {
    // last index i in [lo, hi) with a[i] <= p (a[lo] <= p assumed)
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (a[mid] <= p) lo = mid; else hi = mid;
    }
    return lo;
}

// Segments of every chunk's first and last entry, all chunks in parallel (a
// serial search per CTA would sit on the critical path of every chunk).
__global__ void k_merge_partition(const uint32_t* __restrict__ src_start, uint64_t nseg, uint64_t total,
                                  uint64_t chunks, uint64_t* __restrict__ seg_range) {
    const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= chunks) return;
    const uint64_t p0 = c * kMcTile, p1 = p0 + kMcTile < total ? p0 + kMcTile : total;
    seg_range[2 * c] = seg_of(src_start, 0, nseg + 1, (uint32_t)p0);
    seg_range[2 * c + 1] = seg_of(src_start, 0, nseg + 1, (uint32_t)(p1 - 1));
}

__global__ void __launch_bounds__(kMcNT) k_merge_copy(const uint32_t* __restrict__ recv, uint64_t total,
                                                      const uint32_t* __restrict__ src_start,
                                                      const uint32_t* __restrict__ dst,
                                                      const uint64_t* __restrict__ seg_range,
                                                      uint32_t* __restrict__ out) {
    __shared__ uint32_t s_start[kMcSegs + 1];
    __shared__ uint32_t s_dst[kMcSegs];
    const uint64_t p0 = (uint64_t)blockIdx.x * kMcTile;
    const uint64_t p1 = p0 + kMcTile < total ? p0 + kMcTile : total;
    const uint64_t sa = __ldg(seg_range + 2 * blockIdx.x), sb = __ldg(seg_range + 2 * blockIdx.x + 1);
    const bool staged = sb - sa < (uint64_t)kMcSegs;
    if (staged) {
        for (uint64_t i = threadIdx.x; i <= sb - sa; i += kMcNT) {
            s_start[i] = __ldg(src_start + sa + i);
            s_dst[i] = __ldg(dst + sa + i);
        }
        if (threadIdx.x == 0) s_start[sb - sa + 1] = __ldg(src_start + sb + 1);
    }
    __syncthreads();
    // each warp: 256 consecutive entries, lane-interleaved (coalesced loads and
    // stores); its segment range is found once, then each entry searches it
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const uint64_t w0 = p0 + (uint64_t)warp * 32 * kMcIPT;
    if (w0 >= p1) return;
    const uint64_t w1 = w0 + 32 * kMcIPT < p1 ? w0 + 32 * kMcIPT : p1;
    if (staged) {
        const uint32_t nst = (uint32_t)(sb - sa + 1);
        const uint32_t lo = (uint32_t)seg_of(s_start, 0, nst + 1, (uint32_t)w0);
        const uint32_t hi = (uint32_t)seg_of(s_start, lo, nst + 1, (uint32_t)(w1 - 1)) + 1;
#pragma unroll
        for (int u = 0; u < kMcIPT; u++) {
            const uint64_t p = w0 + (uint64_t)u * 32 + lane;
            if (p < w1) {
                const uint32_t i = (uint32_t)seg_of(s_start, lo, hi, (uint32_t)p);
                out[s_dst[i] + ((uint32_t)p - s_start[i])] = __ldg(recv + p);
            }
        }
    } else {
#pragma unroll
        for (int u = 0; u < kMcIPT; u++) {
            const uint64_t p = w0 + (uint64_t)u * 32 + lane;
            if (p < w1) {
                const uint64_t i = seg_of(src_start, sa, sb + 2, (uint32_t)p);
                out[__ldg(dst + i) + ((uint32_t)p - __ldg(src_start + i))] = __ldg(recv + p);
            }
        }
    }
}

cudaError_t launch_adjacent_diff(const uint32_t* in, uint64_t count, uint32_t* out, int num_sms, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    const uint64_t blocks = ceil_div(count, 256), cap = (uint64_t)num_sms * 8;
    k_adjacent_diff<<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, s>>>(in, count, out);
    return cudaGetLastError();
}

size_t merge_rows_workspace_bytes(int parts, uint32_t rows, uint64_t recv_len) {
    const uint64_t cnt = (uint64_t)parts * rows;
    return 2 * (((cnt + 1) * 4 + 255) / 256 * 256) + (ceil_div(cnt + 1, 2048) + 2) * 8 + 256 +
           (ceil_div(recv_len, kMcTile) + 1) * 16;
}

cudaError_t launch_merge_rows(const uint32_t* recv, uint64_t recv_len, int parts, uint32_t rows,
                              const uint32_t* counts, const uint32_t* out_off, uint32_t* out, void* ws,
                              size_t ws_bytes, int num_sms, cudaStream_t s) {
    if (ws_bytes < merge_rows_workspace_bytes(parts, rows, recv_len)) return cudaErrorInvalidValue;
    if (rows == 0 || parts == 0) return cudaSuccess;
    const uint64_t cnt = (uint64_t)parts * rows;
    const size_t arr = ((cnt + 1) * 4 + 255) / 256 * 256;
    char* p = static_cast<char*>(ws);
    uint32_t* src_start = reinterpret_cast<uint32_t*>(p);
    uint32_t* dst = reinterpret_cast<uint32_t*>(p + arr);
    unsigned long long* st = reinterpret_cast<unsigned long long*>(p + 2 * arr);
    unsigned* counter = reinterpret_cast<unsigned*>(st + ceil_div(cnt + 1, 2048) + 1);
    // rank-major exclusive scan of the counts = segment starts in recv (senders' runs back to back)
    cudaError_t e = launch_row_offsets(counts, (uint32_t)cnt, src_start, st, counter, s);
    if (e != cudaSuccess) return e;
    const uint64_t rb = ceil_div(rows, 256), cap = (uint64_t)num_sms * 8;
    k_merge_dst<<<(unsigned)(rb < cap ? rb : cap), 256, 0, s>>>(counts, parts, rows, out_off, dst);
    if (recv_len == 0) return cudaGetLastError();
    const uint64_t chunks = ceil_div(recv_len, kMcTile);
    uint64_t* seg_range = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(counter) + 256);
    k_merge_partition<<<(unsigned)ceil_div(chunks, 256), 256, 0, s>>>(src_start, cnt, recv_len, chunks, seg_range);
    k_merge_copy<<<(unsigned)chunks, kMcNT, 0, s>>>(recv, recv_len, src_start, dst, seg_range, out);
    return cudaGetLastError();
}

}  // namespace boba
