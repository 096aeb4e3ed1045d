// Phase 5 -- CSR SpMV: y[v] = sum_{k in row v} w[k] * x[indices[k]], in fp32
// (the benchmarked path, north star) or fp64 (the reference's precision, used
// by the drop-in spmv_pull).
//
// Reference: pkg/src/boba/kernels.py:30-52 spmv_pull (x[indices] gather,
// optional weights, per-row sums with empty rows = 0; kernels.py:19-27).
// The reference bench passes the FORWARD CSR (bench.py:146-156), so this is a
// row dot product over whatever CSR the caller gives.
//
// Merge-path, perfectly balanced over the n + m "merge items" (row ends and
// nonzeros), so hub rows of skewed graphs cost the same as short rows:
//   * each CTA owns 1024 consecutive merge items; it locates its (row, nnz)
//     start with a binary search on the row-end offsets, stages the row ends
//     and the products x[indices[k]]*w[k] in shared memory with coalesced
//     index loads (the x gathers are all in flight at once -- this is where
//     reordering shows up as L1/L2 hit rate);
//   * each thread folds 8 items sequentially, a warp/CTA segmented scan
//     carries partial rows across threads;
//   * a row that spans CTAs gets its partial sum from the CTA that ends it and
//     the tails of the CTAs before it from a segmented-scan fix-up over the
//     per-CTA tails (k_spmv_chunk_agg + k_spmv_carry); no CTA waits on another
//     and every sum has a fixed association, so y is bitwise deterministic.
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace boba {

// 128 x 8: measured against 256 x 8 / 512 x 8 / 256 x 16 / 256 x 4 / 64 x 8 / 128 x 16
// (c3 BOBA SpMV 0.219 vs 0.227 / 0.238 / 0.309 / 0.248 / 0.226 / 0.281 ms): smaller
// CTAs lose less to the two block barriers of this latency-bound tile.
constexpr int kSpNT = 128, kSpIPT = 8, kSpTile = kSpNT * kSpIPT;
constexpr int kSpShort = 8;  // longest in-tile row the per-row fold takes (longer: divergent folds)
// Whole-matrix row mode: when no row is longer than kSpRowMax (a mesh / road
// graph), k_spmv_merge skips the merge-path tiling and gives every row one
// thread that sums it sequentially straight from global memory -- no staging,
// no barriers, no carries (profiles/r02_spmv_rowmap.log: on the c3 grid a
// thread per row beats 4/8/16/32 lanes per row and the merge path; on R-MAT
// it is 20x slower).  The longest row is found on the device when the CSR is
// partitioned and the mode travels in the tile coordinates, so one kernel
// serves both modes with no host round trip.  Measured, fp32 per call, c3:
// BOBA order 0.191 -> 0.155 ms, random order 0.361 -> 0.380; R-MAT c2/c5/c4
// unchanged (profiles/r02_spmv_rowmode.log).  Kept at 32 registers: a second
// row per thread (c3 BOBA 0.126 ms) or a separate row kernel beside an idle
// merge launch (0.175) cost the R-MAT path 3-10 %.
constexpr uint32_t kSpRowMax = 8;
constexpr uint32_t kSpRowMode = 0x80000000u;  // flag bit in coords[]

// Streaming loads that must not evict the x vector's hot lines from L1.
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ uint4 ld_stream_u128(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

template <typename T>
struct SegValT {
    bool f;
    T v;
};

template <typename T>
__device__ __forceinline__ SegValT<T> seg_combine(SegValT<T> a, SegValT<T> b) {
    return b.f ? b : SegValT<T>{a.f, a.v + b.v};
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

// Longest row of the CSR (rowmax zeroed beforehand); k_spmv_partition then
// marks row mode in bit 31 of every tile coordinate (row ids < 2^31), so the
// tiles learn the mode from the load they make anyway.
__global__ void k_spmv_rowmax(const uint32_t* __restrict__ offsets, uint32_t n, uint32_t* rowmax) {
    uint32_t mx = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t len = __ldg(offsets + i + 1) - __ldg(offsets + i);
        mx = len > mx ? len : mx;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint32_t v = __shfl_xor_sync(0xFFFFFFFFu, mx, o);
        mx = v > mx ? v : mx;
    }
    if (lane_id() == 0 && mx) atomicMax(rowmax, mx);
}

// Tile boundaries in merge space, all searched in parallel up front (a
// dependent ~log2(n)-step binary search per CTA would otherwise sit on the
// critical path of every tile).
__global__ void k_spmv_partition(const uint32_t* __restrict__ offsets, uint32_t n, uint64_t m, uint64_t tiles,
                                 const uint32_t* __restrict__ rowmax, uint32_t* coords) {
    const uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b > tiles) return;
    const uint64_t total = (uint64_t)n + m;
    const uint64_t d = b * kSpTile < total ? b * kSpTile : total;
    coords[b] = (uint32_t)merge_search(offsets + 1, n, 0, m, d) | (*rowmax <= kSpRowMax ? kSpRowMode : 0u);
}

template <typename T>
__device__ __forceinline__ T row_sum(const uint32_t* __restrict__ indices, const T* __restrict__ w,
                                     const T* __restrict__ x, uint32_t b, uint32_t len) {
    T acc = 0;
#pragma unroll
    for (uint32_t j0 = 0; j0 < kSpRowMax; j0 += 4) {
        if (j0 >= len) break;
        uint32_t c[4];
#pragma unroll
        for (uint32_t j = 0; j < 4; j++) c[j] = j0 + j < len ? __ldg(indices + b + j0 + j) : 0u;
        T v[4];
#pragma unroll
        for (uint32_t j = 0; j < 4; j++) v[j] = j0 + j < len ? __ldg(x + c[j]) : T(0);
#pragma unroll
        for (uint32_t j = 0; j < 4; j++)
            if (j0 + j < len) acc += w ? v[j] * __ldg(w + b + j0 + j) : v[j];
    }
    return acc;
}

// Row mode: one thread per row (grid-stride over the rows), its indices and
// gathers in flight four at a time -- the kernel stays at 32 registers, 16
// CTAs/SM, which the merge path needs (two rows per thread: 40 registers).
template <typename T>
__device__ __forceinline__ void spmv_rows(const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ indices,
                                          const T* __restrict__ w, const T* __restrict__ x, T* __restrict__ y,
                                          uint32_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * kSpNT;
    for (uint64_t r = (uint64_t)blockIdx.x * kSpNT + threadIdx.x; r < n; r += stride) {
        const uint32_t b = __ldg(offsets + r);
        y[r] = row_sum<T>(indices, w, x, b, __ldg(offsets + r + 1) - b);
    }
}

// Merge-path search inside a tile, all tile-relative 32-bit: a[] holds the
// row ends minus the tile's first nonzero index.
__device__ __forceinline__ uint32_t merge_search_rel(const uint32_t* a, uint32_t a_len, uint32_t b_len, uint32_t diag) {
    uint32_t lo = diag > b_len ? diag - b_len : 0, hi = diag < a_len ? diag : a_len;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] <= diag - mid - 1)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// One merge-path tile (kSpTile merge items) processed by a CTA of kSpNT
// threads.  Every row that ends inside the tile is written here; the first
// row the tile ends may have started in earlier tiles -- its partial sum is
// written and fixed up by k_spmv_carry (no tile ever waits on another).
// Inside the tile all indices are 32-bit and relative to the tile's first
// row (i0) and first nonzero (j0); only the global loads and stores use
// 64-bit addresses.
template <typename T, bool VEC>
__device__ __forceinline__ void spmv_tile(uint64_t tile, const uint32_t* __restrict__ offsets,
                                          const uint32_t* __restrict__ indices, const T* __restrict__ w,
                                          const T* __restrict__ x, T* __restrict__ y, uint32_t n, uint64_t m,
                                          uint32_t c_lo, uint32_t c_hi, uint32_t* __restrict__ tile_head,
                                          T* __restrict__ tile_tail, uint32_t* s_end, T* s_val, SegValT<T>* s_warp) {
    using SegVal = SegValT<T>;
    const uint32_t gt = threadIdx.x;
    const uint64_t total = (uint64_t)n + m;
    const uint64_t d0 = tile * kSpTile;
    const uint32_t items_tile = (uint32_t)((d0 + kSpTile < total ? d0 + kSpTile : total) - d0);
    const uint32_t i0 = c_lo & ~kSpRowMode, i1 = c_hi & ~kSpRowMode;
    const uint64_t j0 = d0 - i0;
    // A reused partition (reuse_partition = 1) that does not belong to this
    // CSR could hold any coords: never index s_end / s_val past the tile.
    if (i1 < i0 || i1 - i0 > items_tile || i1 > n) {
        if (gt == 0) {
            tile_head[tile] = 0xFFFFFFFFu;
            tile_tail[tile] = T(0);
        }
        return;
    }
    const uint32_t nrows = i1 - i0, nnz = items_tile - nrows;
    const uint32_t j0_32 = (uint32_t)j0;  // offsets are uint32: relative ends are exact mod 2^32
    for (uint32_t k = gt; k <= nrows; k += kSpNT)
        s_end[k] = (i0 + k < n) ? ld_stream_u32(offsets + i0 + 1 + k) - j0_32 : 0xFFFFFFFFu;
    // VEC (unweighted, 16-byte aligned indices): the tile's indices are
    // read as aligned quads from a0 = j0 & ~3 and the products stored as
    // quads at their a0-relative slot, so s_val[k + sh] holds item k
    const uint32_t sh = VEC ? (uint32_t)(j0 & 3) : 0u;
    if (VEC) {
        const uint64_t a0 = j0 - sh;
        const uint32_t span = nnz + sh, quads = (span + 3) >> 2;
        const uint4* ip4 = reinterpret_cast<const uint4*>(indices + a0);
        constexpr int QPT = kSpIPT / 4 + 1;  // span <= kSpTile + 3: one quad beyond kSpTile / 4
        uint4 c[QPT];
#pragma unroll
        for (int u = 0; u < QPT; u++) {
            const uint32_t q = gt + u * kSpNT;
            c[u] = make_uint4(0, 0, 0, 0);
            if (q < quads) {
                if (a0 + 4ull * q + 4 <= m) {
                    c[u] = ld_stream_u128(ip4 + q);
                } else {  // the array's last partial quad: no read past indices[m)
                    const uint32_t* ip = indices + a0 + 4ull * q;
                    const uint64_t left = m - (a0 + 4ull * q);
                    c[u].x = ld_stream_u32(ip);
                    if (left > 1) c[u].y = ld_stream_u32(ip + 1);
                    if (left > 2) c[u].z = ld_stream_u32(ip + 2);
                }
            }
        }
        // every gather in flight before the first store (the random case is miss-bound)
        T v[QPT][4];
#pragma unroll
        for (int u = 0; u < QPT; u++) {
            const uint32_t r = 4 * (gt + u * kSpNT);
            v[u][0] = r + 0 >= sh && r + 0 < span ? __ldg(x + c[u].x) : T(0);
            v[u][1] = r + 1 >= sh && r + 1 < span ? __ldg(x + c[u].y) : T(0);
            v[u][2] = r + 2 >= sh && r + 2 < span ? __ldg(x + c[u].z) : T(0);
            v[u][3] = r + 3 >= sh && r + 3 < span ? __ldg(x + c[u].w) : T(0);
        }
#pragma unroll
        for (int u = 0; u < QPT; u++) {
            const uint32_t q = gt + u * kSpNT;
            if (q < quads) {
                if constexpr (sizeof(T) == 4) {
                    reinterpret_cast<float4*>(s_val)[q] = make_float4(v[u][0], v[u][1], v[u][2], v[u][3]);
                } else {
                    reinterpret_cast<double2*>(s_val)[2 * q] = make_double2(v[u][0], v[u][1]);
                    reinterpret_cast<double2*>(s_val)[2 * q + 1] = make_double2(v[u][2], v[u][3]);
                }
            }
        }
    } else {
        // all index loads, then all x gathers in flight together (nnz <= kSpTile)
        const uint32_t* ip = indices + j0;
        uint32_t col[kSpIPT];
#pragma unroll
        for (int u = 0; u < kSpIPT; u++) {
            const uint32_t k = gt + u * kSpNT;
            col[u] = k < nnz ? ld_stream_u32(ip + k) : 0u;
        }
        T p[kSpIPT];
#pragma unroll
        for (int u = 0; u < kSpIPT; u++) {
            const uint32_t k = gt + u * kSpNT;
            p[u] = k < nnz ? __ldg(x + col[u]) : T(0);
        }
#pragma unroll
        for (int u = 0; u < kSpIPT; u++) {
            const uint32_t k = gt + u * kSpNT;
            if (k < nnz) s_val[k] = w ? p[u] * __ldg(w + j0 + k) : p[u];
        }
    }
    // Short-row tiles (every row's in-tile part <= kSpShort nonzeros, e.g. a
    // mesh): one thread folds each row straight from s_val -- no merge search,
    // no segmented scan.  Tiles holding a longer row take the balanced
    // merge-path fold below.  The choice depends on the matrix only, so y
    // stays bitwise deterministic.
    __syncthreads();
    const T* sv = s_val + sh;
    // (nnz > (nrows + 1) kSpShort: some row is long by pigeonhole -- skip the check)
    if (nnz <= (nrows + 1) * (uint32_t)kSpShort) {
        bool long_row = false;
        for (uint32_t k = gt; k <= nrows; k += kSpNT) {
            const uint32_t beg = k ? s_end[k - 1] : 0u, end = k < nrows ? s_end[k] : nnz;
            long_row |= end - beg > (uint32_t)kSpShort;
        }
        if (!__syncthreads_or(long_row)) {
            for (uint32_t k = gt; k < nrows; k += kSpNT) {
                const uint32_t beg = k ? s_end[k - 1] : 0u, end = s_end[k];
                T acc = 0;
                for (uint32_t j = beg; j < end; j++) acc += sv[j];
                y[i0 + k] = acc;  // row 0 may have begun in earlier tiles: k_spmv_carry adds their tails
            }
            if (gt == 0) {
                T tail = 0;
                for (uint32_t j = nrows ? s_end[nrows - 1] : 0u; j < nnz; j++) tail += sv[j];
                tile_tail[tile] = tail;
                tile_head[tile] = nrows ? i0 : 0xFFFFFFFFu;
            }
            return;
        }
    }
    // Per-thread sequential fold over kSpIPT merge items.
    const uint32_t diag = gt * kSpIPT < items_tile ? gt * kSpIPT : items_tile;
    uint32_t it = merge_search_rel(s_end, nrows, nnz, diag);
    uint32_t jt = diag - it;
    const uint32_t items = items_tile - diag < (uint32_t)kSpIPT ? items_tile - diag : (uint32_t)kSpIPT;
    T acc = 0, first_val = 0;
    uint32_t first_row = 0;
    bool emitted = false;
    for (uint32_t k = 0; k < items; k++) {
        if (jt < s_end[it]) {
            acc += sv[jt];
            jt++;
        } else {
            if (!emitted) {
                first_row = it;
                first_val = acc;
                emitted = true;
            } else {
                y[i0 + it] = acc;
            }
            acc = 0;
            it++;
        }
    }
    // Segmented scan of (emitted, tail) over the CTA -> exclusive carry per thread.
    const unsigned lane = lane_id(), warp = gt >> 5;
    SegVal inc{emitted, acc};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        SegVal up;
        up.f = __shfl_up_sync(0xFFFFFFFFu, inc.f, o);
        up.v = __shfl_up_sync(0xFFFFFFFFu, inc.v, o);
        if (lane >= (unsigned)o) inc = seg_combine(up, inc);
    }
    SegVal lex;
    lex.f = __shfl_up_sync(0xFFFFFFFFu, inc.f, 1);
    lex.v = __shfl_up_sync(0xFFFFFFFFu, inc.v, 1);
    if (lane == 0) lex = SegVal{false, T(0)};
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        SegVal wi = lane < kSpNT / 32 ? s_warp[lane] : SegVal{false, T(0)};
#pragma unroll
        for (int o = 1; o < kSpNT / 32; o <<= 1) {
            SegVal up;
            up.f = __shfl_up_sync(0xFFFFFFFFu, wi.f, o);
            up.v = __shfl_up_sync(0xFFFFFFFFu, wi.v, o);
            if (lane >= (unsigned)o) wi = seg_combine(up, wi);
        }
        SegVal we;
        we.f = __shfl_up_sync(0xFFFFFFFFu, wi.f, 1);
        we.v = __shfl_up_sync(0xFFFFFFFFu, wi.v, 1);
        if (lane == 0) we = SegVal{false, T(0)};
        __syncwarp();
        if (lane < kSpNT / 32) s_warp[lane] = we;
        if (lane == kSpNT / 32 - 1) {
            tile_tail[tile] = wi.v;                    // tile aggregate (flag = has a head row)
            if (!wi.f) tile_head[tile] = 0xFFFFFFFFu;  // no row ends here
        }
    }
    __syncthreads();
    if (emitted) {
        const SegVal ex = seg_combine(s_warp[warp], lex);
        y[i0 + first_row] = first_val + ex.v;
        if (!ex.f) tile_head[tile] = i0 + first_row;  // partial: earlier tiles add their tails
    }
}

// One merge-path tile per CTA.
template <typename T, bool VEC>
__global__ void __launch_bounds__(kSpNT) k_spmv_merge(const uint32_t* __restrict__ offsets,
                                                      const uint32_t* __restrict__ indices,
                                                      const T* __restrict__ w, const T* __restrict__ x,
                                                      T* __restrict__ y, uint32_t n, uint64_t m,
                                                      const uint32_t* __restrict__ coords,
                                                      uint32_t* __restrict__ tile_head, T* __restrict__ tile_tail,
                                                      const int* stop) {
    if (stop && *(volatile const int*)stop) return;
    // The mode rides in bit 31 of the tile's own coordinate, so merge mode
    // waits on no extra load (measured: a separate mode word, or coords[0],
    // costs the R-MAT SpMV 1-2 %).
    const uint32_t c_lo = __ldg(coords + blockIdx.x), c_hi = __ldg(coords + blockIdx.x + 1);
    if (c_lo & kSpRowMode) {
        spmv_rows<T>(offsets, indices, w, x, y, n);
        return;
    }
    __shared__ uint32_t s_end[kSpTile + 1];
    __shared__ __align__(16) T s_val[kSpTile + 4];
    __shared__ SegValT<T> s_warp[kSpNT / 32];
    spmv_tile<T, VEC>(blockIdx.x, offsets, indices, w, x, y, n, m, c_lo, c_hi, tile_head, tile_tail, s_end, s_val,
                      s_warp);
}

// Chunk aggregates of the per-CTA (has_head, tail) pairs: a segmented sum
// over kSpChunk consecutive CTAs, one thread per CTA.
constexpr int kSpChunk = 1024;

template <typename T>
__device__ __forceinline__ SegValT<T> block_seg_scan(SegValT<T> v, SegValT<T>* s_w, SegValT<T>* total,
                                                     SegValT<T>* excl) {
    using SegVal = SegValT<T>;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    SegVal inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        SegVal up;
        up.f = __shfl_up_sync(0xFFFFFFFFu, inc.f, o);
        up.v = __shfl_up_sync(0xFFFFFFFFu, inc.v, o);
        if (lane >= (unsigned)o) inc = seg_combine(up, inc);
    }
    SegVal lex;
    lex.f = __shfl_up_sync(0xFFFFFFFFu, inc.f, 1);
    lex.v = __shfl_up_sync(0xFFFFFFFFu, inc.v, 1);
    if (lane == 0) lex = SegVal{false, T(0)};
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        SegVal wi = s_w[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            SegVal up;
            up.f = __shfl_up_sync(0xFFFFFFFFu, wi.f, o);
            up.v = __shfl_up_sync(0xFFFFFFFFu, wi.v, o);
            if (lane >= (unsigned)o) wi = seg_combine(up, wi);
        }
        SegVal we;
        we.f = __shfl_up_sync(0xFFFFFFFFu, wi.f, 1);
        we.v = __shfl_up_sync(0xFFFFFFFFu, wi.v, 1);
        if (lane == 0) we = SegVal{false, T(0)};
        __syncwarp();
        s_w[lane] = we;
        if (lane == 31) s_w[32] = wi;
    }
    __syncthreads();
    *excl = seg_combine(s_w[warp], lex);
    *total = s_w[32];
    return inc;
}

template <typename T>
__global__ void __launch_bounds__(kSpChunk) k_spmv_chunk_agg(const uint32_t* __restrict__ tile_head,
                                                             const T* __restrict__ tile_tail, uint64_t tiles,
                                                             unsigned* chunk_flag, T* chunk_val,
                                                             const uint32_t* __restrict__ coords, const int* stop) {
    if ((stop && *(volatile const int*)stop) || (__ldg(coords) & kSpRowMode)) return;
    using SegVal = SegValT<T>;
    __shared__ SegVal s_w[33];
    const uint64_t t = (uint64_t)blockIdx.x * kSpChunk + threadIdx.x;
    SegVal v = t < tiles ? SegVal{tile_head[t] != 0xFFFFFFFFu, tile_tail[t]} : SegVal{false, T(0)};
    SegVal total, excl;
    block_seg_scan<T>(v, s_w, &total, &excl);
    if (threadIdx.x == 0) {
        chunk_flag[blockIdx.x] = total.f;
        chunk_val[blockIdx.x] = total.v;
    }
}

// y[head row of CTA t] += (segmented sum of the tails of the CTAs before t
// back to the last one that ended a row) -- fixed association, so the SpMV
// is bitwise deterministic.
template <typename T>
__global__ void __launch_bounds__(kSpChunk) k_spmv_carry(const uint32_t* __restrict__ tile_head,
                                                         const T* __restrict__ tile_tail, uint64_t tiles,
                                                         const unsigned* __restrict__ chunk_flag,
                                                         const T* __restrict__ chunk_val, T* y,
                                                         const uint32_t* __restrict__ coords, const int* stop) {
    if ((stop && *(volatile const int*)stop) || (__ldg(coords) & kSpRowMode)) return;
    using SegVal = SegValT<T>;
    __shared__ SegVal s_w[33];
    __shared__ T s_cin;
    if (threadIdx.x == 0) {
        // carry into this chunk: fold chunk aggregates left to right from the
        // last chunk that ended a row (normally just the previous chunk)
        long long c = (long long)blockIdx.x - 1;
        while (c > 0 && !chunk_flag[c]) c--;
        T a = 0;
        for (long long k = c < 0 ? 0 : c; k < (long long)blockIdx.x; k++) a += chunk_val[k];
        s_cin = blockIdx.x == 0 ? T(0) : a;
    }
    __syncthreads();
    const uint64_t t = (uint64_t)blockIdx.x * kSpChunk + threadIdx.x;
    const uint32_t head = t < tiles ? tile_head[t] : 0xFFFFFFFFu;
    SegVal v = t < tiles ? SegVal{head != 0xFFFFFFFFu, tile_tail[t]} : SegVal{false, T(0)};
    SegVal total, excl;
    block_seg_scan<T>(v, s_w, &total, &excl);
    if (head != 0xFFFFFFFFu && t > 0) {
        const T carry = excl.f ? excl.v : s_cin + excl.v;
        y[head] += carry;
    }
}

size_t spmv_workspace_bytes(uint32_t n, uint64_t m) {
    const uint64_t tiles = ceil_div((uint64_t)n + m, kSpTile);
    const uint64_t chunks = ceil_div(tiles, kSpChunk);
    const size_t arr = ((tiles + 2) * 8 + 255) / 256 * 256;   // sized for double
    return arr * 3 + ((chunks + 1) * 16 + 255) / 256 * 256 + 256;  // + rowmax
}

template <typename T>
cudaError_t launch_spmv_t(const uint32_t* offsets, const uint32_t* indices, const T* w, const T* x, T* y, uint32_t n,
                          uint64_t m, void* ws, size_t ws_bytes, cudaStream_t s, const int* stop = nullptr,
                          bool partitioned = false) {
    if (n == 0) return cudaSuccess;
    if (ws_bytes < spmv_workspace_bytes(n, m)) return cudaErrorInvalidValue;
    const uint64_t tiles = ceil_div((uint64_t)n + m, kSpTile);
    const uint64_t chunks = ceil_div(tiles, kSpChunk);
    const size_t arr = ((tiles + 2) * 8 + 255) / 256 * 256;
    char* p = static_cast<char*>(ws);
    uint32_t* coords = reinterpret_cast<uint32_t*>(p);
    uint32_t* tile_head = reinterpret_cast<uint32_t*>(p + arr);
    T* tile_tail = reinterpret_cast<T*>(p + 2 * arr);
    unsigned* chunk_flag = reinterpret_cast<unsigned*>(p + 3 * arr);
    T* chunk_val = reinterpret_cast<T*>(p + 3 * arr + ((chunks + 1) * 4 + 15) / 16 * 16);
    uint32_t* rowmax = reinterpret_cast<uint32_t*>(p + 3 * arr + ((chunks + 1) * 16 + 255) / 256 * 256);
    if (!partitioned) {  // coords and the longest row depend on the structure only: computed once
        if (cudaError_t e = cudaMemsetAsync(rowmax, 0, 4, s)) return e;
        const uint64_t blocks = ceil_div(n, 256), cap = 2048;
        k_spmv_rowmax<<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, s>>>(offsets, n, rowmax);
        k_spmv_partition<<<(unsigned)ceil_div(tiles + 1, 256), 256, 0, s>>>(offsets, n, m, tiles, rowmax, coords);
    }
    // (A persistent variant with a 128 KB shared-memory copy of the hub prefix of x
    // was measured slower at c2/c3: the occupancy it costs outweighs the hits.)
    const bool vec = !w && (reinterpret_cast<uintptr_t>(indices) & 15) == 0;
    if (vec) {
        // Pinned shared-memory carveout: left to the driver, the vector kernel's
        // register count buys more resident CTAs at the cost of L1, which the x
        // gathers of poorly ordered graphs depend on.  c3 grid, (BOBA order,
        // random order) per call:
        //   fp32: driver default 0.185 / 0.417 ms, 50 % 0.202 / 0.367 (scalar staging 0.220 / 0.372)
        //   fp64: 50 % 0.298 / 0.722, 66 % 0.271 / 0.775, 75 % 0.265 / 0.973,
        //         100 % 0.277 / 1.79 (scalar staging, driver default: 0.248 / 1.80)
        static PerDeviceOnce carve;
        set_attr_once(carve, k_spmv_merge<T, true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                      sizeof(T) == 4 ? 50 : 66);
    }
    if (vec)
        k_spmv_merge<T, true><<<(unsigned)tiles, kSpNT, 0, s>>>(offsets, indices, w, x, y, n, m, coords, tile_head,
                                                               tile_tail, stop);
    else
        k_spmv_merge<T, false><<<(unsigned)tiles, kSpNT, 0, s>>>(offsets, indices, w, x, y, n, m, coords, tile_head,
                                                                tile_tail, stop);
    if (tiles > 1) {
        k_spmv_chunk_agg<T><<<(unsigned)chunks, kSpChunk, 0, s>>>(tile_head, tile_tail, tiles, chunk_flag, chunk_val,
                                                                 coords, stop);
        k_spmv_carry<T><<<(unsigned)chunks, kSpChunk, 0, s>>>(tile_head, tile_tail, tiles, chunk_flag, chunk_val, y,
                                                             coords, stop);
    }
    return cudaGetLastError();
}

cudaError_t launch_spmv(const uint32_t* offsets, const uint32_t* indices, const float* w, const float* x, float* y,
                        uint32_t n, uint64_t m, void* ws, size_t ws_bytes, cudaStream_t s, bool partitioned) {
    return launch_spmv_t<float>(offsets, indices, w, x, y, n, m, ws, ws_bytes, s, nullptr, partitioned);
}

cudaError_t launch_spmv_f64(const uint32_t* offsets, const uint32_t* indices, const double* w, const double* x,
                            double* y, uint32_t n, uint64_t m, void* ws, size_t ws_bytes, cudaStream_t s,
                            bool partitioned) {
    return launch_spmv_t<double>(offsets, indices, w, x, y, n, m, ws, ws_bytes, s, nullptr, partitioned);
}

cudaError_t launch_spmv_f64_iter(const uint32_t* offsets, const uint32_t* indices, const double* w, const double* x,
                                 double* y, uint32_t n, uint64_t m, void* ws, size_t ws_bytes, cudaStream_t s,
                                 const int* stop, bool partitioned) {
    return launch_spmv_t<double>(offsets, indices, w, x, y, n, m, ws, ws_bytes, s, stop, partitioned);
}

}  // namespace boba
