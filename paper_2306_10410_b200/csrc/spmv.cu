// Phase 5 -- CSR SpMV, fp32: y[v] = sum_{k in row v} w[k] * x[indices[k]].
//
// Reference: pkg/src/boba/kernels.py:30-52 spmv_pull (x[indices] gather,
// optional weights, per-row sums with empty rows = 0; kernels.py:19-27).
// The reference bench passes the FORWARD CSR (bench.py:146-156), so this is a
// row dot product over whatever CSR the caller gives.
//
// Merge-path, perfectly balanced over the n + m "merge items" (row ends and
// nonzeros), so hub rows of skewed graphs cost the same as short rows:
//   * each CTA owns 2048 consecutive merge items; it locates its (row, nnz)
//     start with a binary search on the row-end offsets, stages the row ends
//     and the products x[indices[k]]*w[k] in shared memory with coalesced
//     index loads (the x gathers are all in flight at once -- this is where
//     reordering shows up as L1/L2 hit rate);
//   * each thread folds 8 items sequentially, a warp/CTA segmented scan
//     carries partial rows across threads;
//   * partial rows across CTAs are carried by decoupled lookback whose fold
//     order is canonical (left to right from the CTA that started the row), so
//     results are bitwise deterministic run to run.
#include "common.cuh"
#include "kernels.cuh"

namespace boba {

constexpr int kSpNT = 256, kSpIPT = 8, kSpTile = kSpNT * kSpIPT;
constexpr int kSpMaxRounds = 64;

struct SegVal {
    bool f;
    float v;
};

__device__ __forceinline__ SegVal seg_combine(SegVal a, SegVal b) {
    return b.f ? b : SegVal{a.f, a.v + b.v};
}

// Merge-path search: number of row ends consumed at diagonal `diag` when
// merging row ends a[0..a_len) with nonzero indices b0, b0+1, ... (b_len).
__device__ __forceinline__ uint64_t merge_search(const uint32_t* a, uint64_t a_len, uint64_t b0, uint64_t b_len,
                                                 uint64_t diag) {
    uint64_t lo = diag > b_len ? diag - b_len : 0, hi = diag < a_len ? diag : a_len;
    while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if ((uint64_t)a[mid] <= b0 + (diag - mid - 1))
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// Tile boundaries in merge space, all searched in parallel up front (a
// dependent ~log2(n)-step binary search per CTA would otherwise sit on the
// critical path of every tile).
__global__ void k_spmv_partition(const uint32_t* __restrict__ offsets, uint32_t n, uint64_t m, uint64_t tiles,
                                 uint32_t* coords) {
    const uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b > tiles) return;
    const uint64_t total = (uint64_t)n + m;
    const uint64_t d = b * kSpTile < total ? b * kSpTile : total;
    coords[b] = (uint32_t)merge_search(offsets + 1, n, 0, m, d);
}

__device__ __forceinline__ unsigned long long pack_f(unsigned long long flag, float v) {
    return flag | (unsigned long long)__float_as_uint(v);
}

__global__ void __launch_bounds__(kSpNT) k_spmv_merge(const uint32_t* __restrict__ offsets,
                                                      const uint32_t* __restrict__ indices,
                                                      const float* __restrict__ w, const float* __restrict__ x,
                                                      float* __restrict__ y, uint32_t n, uint64_t m,
                                                      const uint32_t* __restrict__ coords,
                                                      unsigned long long* status, unsigned* tile_counter) {
    __shared__ uint32_t s_end[kSpTile + 1];
    __shared__ float s_val[kSpTile];
    __shared__ uint64_t s_ij[4];
    __shared__ SegVal s_warp[kSpNT / 32];
    __shared__ float s_chain[kSpMaxRounds * 32];
    __shared__ float s_carry;
    __shared__ unsigned s_tile;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t total = (uint64_t)n + m;
    const uint64_t d0 = tile * kSpTile;
    const uint64_t d1 = d0 + kSpTile < total ? d0 + kSpTile : total;
    if (threadIdx.x < 2) {
        const uint64_t d = threadIdx.x == 0 ? d0 : d1;
        const uint64_t i = __ldg(coords + tile + threadIdx.x);
        s_ij[threadIdx.x * 2] = i;
        s_ij[threadIdx.x * 2 + 1] = d - i;
    }
    __syncthreads();
    const uint64_t i0 = s_ij[0], j0 = s_ij[1], i1 = s_ij[2], j1 = s_ij[3];
    const uint32_t nrows = (uint32_t)(i1 - i0), nnz = (uint32_t)(j1 - j0);
    for (uint32_t k = threadIdx.x; k <= nrows; k += kSpNT)
        s_end[k] = (i0 + k < n) ? __ldg(offsets + i0 + 1 + k) : 0xFFFFFFFFu;
    for (uint32_t k = threadIdx.x; k < nnz; k += kSpNT) {
        float p = __ldg(x + __ldg(indices + j0 + k));
        if (w) p *= __ldg(w + j0 + k);
        s_val[k] = p;
    }
    __syncthreads();
    // Per-thread sequential fold over kSpIPT merge items.
    const uint32_t items_tile = (uint32_t)(d1 - d0);
    const uint32_t diag = threadIdx.x * kSpIPT < items_tile ? threadIdx.x * kSpIPT : items_tile;
    uint32_t it = (uint32_t)merge_search(s_end, nrows, j0, nnz, diag);
    uint32_t jt = diag - it;
    const uint32_t items = items_tile - diag < (uint32_t)kSpIPT ? items_tile - diag : (uint32_t)kSpIPT;
    float acc = 0.f, first_val = 0.f;
    uint64_t first_row = 0;
    bool emitted = false;
    for (uint32_t k = 0; k < items; k++) {
        if (j0 + jt < (uint64_t)s_end[it]) {
            acc += s_val[jt];
            jt++;
        } else {
            const uint64_t row = i0 + it;
            if (!emitted) {
                first_row = row;
                first_val = acc;
                emitted = true;
            } else {
                y[row] = acc;
            }
            acc = 0.f;
            it++;
        }
    }
    // CTA segmented scan of (emitted, tail) -> exclusive carry per thread.
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    SegVal mine{emitted, acc};
    SegVal inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        SegVal up;
        up.f = __shfl_up_sync(0xFFFFFFFFu, inc.f, o);
        up.v = __shfl_up_sync(0xFFFFFFFFu, inc.v, o);
        if (lane >= (unsigned)o) inc = seg_combine(up, inc);
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        SegVal wv = lane < kSpNT / 32 ? s_warp[lane] : SegVal{false, 0.f};
        SegVal wi = wv;
#pragma unroll
        for (int o = 1; o < kSpNT / 32; o <<= 1) {
            SegVal up;
            up.f = __shfl_up_sync(0xFFFFFFFFu, wi.f, o);
            up.v = __shfl_up_sync(0xFFFFFFFFu, wi.v, o);
            if (lane >= (unsigned)o) wi = seg_combine(up, wi);
        }
        // exclusive warp prefix
        SegVal we;
        we.f = __shfl_up_sync(0xFFFFFFFFu, wi.f, 1);
        we.v = __shfl_up_sync(0xFFFFFFFFu, wi.v, 1);
        if (lane == 0) we = SegVal{false, 0.f};
        if (lane < kSpNT / 32) s_warp[lane] = we;
        // block aggregate = inclusive of the last warp
        SegVal agg;
        agg.f = __shfl_sync(0xFFFFFFFFu, wi.f, kSpNT / 32 - 1);
        agg.v = __shfl_sync(0xFFFFFFFFu, wi.v, kSpNT / 32 - 1);
        if (lane == 0) {
            if (tile == 0)
                st_volatile_u64(status + tile, pack_f(kFlagInc, agg.v));
            else
                st_volatile_u64(status + tile, pack_f(agg.f ? kFlagInc : kFlagAgg, agg.v));
        }
        // Decoupled lookback with a canonical (left-to-right) fold.
        float carry = 0.f;
        if (tile > 0) {
            long long base = (long long)tile - 1;
            int rounds = 0;
            int stop = 0;
            float overflow = 0.f;
            bool overflowed = false;
            while (true) {
                long long idx = base - (long long)lane;
                unsigned long long s = idx >= 0 ? ld_volatile_u64(status + idx) : kFlagInc;
                unsigned flag = (unsigned)(s >> 62);
                if (__any_sync(0xFFFFFFFFu, flag == 0)) continue;
                unsigned incm = __ballot_sync(0xFFFFFFFFu, flag == 2);
                float v = __uint_as_float((unsigned)(s & 0xFFFFFFFFull));
                if (rounds < kSpMaxRounds) {
                    s_chain[rounds * 32 + lane] = v;
                } else {
                    // pathological row spanning > 64*32 CTAs: fold this round in place
                    overflowed = true;
                    float r = warp_sum(incm ? ((int)lane <= __ffs(incm) - 1 ? v : 0.f) : v);
                    overflow += r;
                }
                __syncwarp();
                if (incm) {
                    stop = __ffs(incm) - 1;
                    break;
                }
                rounds++;
                base -= 32;
            }
            if (lane == 0) {
                float a;
                int r = rounds < kSpMaxRounds ? rounds : kSpMaxRounds - 1;
                if (!overflowed) {
                    a = s_chain[r * 32 + stop];
                    for (int l = stop - 1; l >= 0; l--) a += s_chain[r * 32 + l];
                    r--;
                } else {
                    a = overflow;
                }
                for (; r >= 0; r--)
                    for (int l = 31; l >= 0; l--) a += s_chain[r * 32 + l];
                carry = a;
                if (!agg.f) st_volatile_u64(status + tile, pack_f(kFlagInc, carry + agg.v));
            }
        }
        if (lane == 0) s_carry = carry;
    }
    __syncthreads();
    SegVal lex;
    lex.f = __shfl_up_sync(0xFFFFFFFFu, inc.f, 1);
    lex.v = __shfl_up_sync(0xFFFFFFFFu, inc.v, 1);
    if (lane == 0) lex = SegVal{false, 0.f};
    if (emitted) {
        SegVal ex = seg_combine(s_warp[warp], lex);
        float c = ex.f ? ex.v : s_carry + ex.v;
        y[first_row] = first_val + c;
    }
}

size_t spmv_workspace_bytes(uint32_t n, uint64_t m) {
    const uint64_t tiles = ceil_div((uint64_t)n + m, kSpTile);
    return ((tiles + 1) * 8 + 64 + 255) / 256 * 256 + (tiles + 2) * 4;
}

cudaError_t launch_spmv(const uint32_t* offsets, const uint32_t* indices, const float* w, const float* x, float* y,
                        uint32_t n, uint64_t m, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (ws_bytes < spmv_workspace_bytes(n, m)) return cudaErrorInvalidValue;
    const uint64_t tiles = ceil_div((uint64_t)n + m, kSpTile);
    unsigned long long* status = static_cast<unsigned long long*>(ws);
    unsigned* counter = reinterpret_cast<unsigned*>(status + tiles + 1);
    const size_t head = ((tiles + 1) * 8 + 64 + 255) / 256 * 256;
    uint32_t* coords = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + head);
    cudaError_t e = cudaMemsetAsync(ws, 0, head, s);
    if (e != cudaSuccess) return e;
    k_spmv_partition<<<(unsigned)ceil_div(tiles + 1, 256), 256, 0, s>>>(offsets, n, m, tiles, coords);
    k_spmv_merge<<<(unsigned)tiles, kSpNT, 0, s>>>(offsets, indices, w, x, y, n, m, coords, status, counter);
    return cudaGetLastError();
}

}  // namespace boba
