// Phase 1 -- first occurrence of every vertex in the flattened edge stream
// I||J (positions: I[e] -> e, J[e] -> m + e).
//
// Reference: pkg/src/boba/_parallel.py:139-162 first_hit_chunked (exact
// chunk-local minimum merged exactly) and :165-175 first_hit_racy (guarded
// unsynchronised writes).  Here the minimum is a device-wide atomicMin on
// uint32 (2m <= 2^32 - 2, UNSET = 0xFFFFFFFF), issued only when a plain load
// of first[v] shows the position can still lower it.  The grid sweeps the
// stream in position order (block-cyclic over 16-byte quads), so almost all
// later occurrences of a vertex fail the guard and cost one L2 load, no
// atomic.  Lanes of a warp that hold the same vertex in the same quad slot
// are merged with __match_any_sync first (the lowest lane carries the
// smallest position), which removes the hub collisions of skewed graphs.
#include "common.cuh"
#include "kernels.cuh"

namespace boba {

template <bool RELAXED>
__device__ __forceinline__ void hit(uint32_t* first, uint32_t v, uint32_t pos, bool valid) {
    // Warp-level dedup: among active lanes with equal v, only the lowest lane
    // (smallest position, since positions grow with the lane index) proceeds.
    unsigned peers = __match_any_sync(0xFFFFFFFFu, valid ? v : 0xFFFFFFFFu);
    bool leader = valid && ((peers & lanemask_lt()) == 0);
    if (!leader) return;
    uint32_t cur = *((volatile uint32_t*)(first + v));
    if (pos < cur) {
        if (RELAXED)
            *((volatile uint32_t*)(first + v)) = pos;
        else
            atomicMin(first + v, pos);
    }
}

template <bool RELAXED>
__global__ void __launch_bounds__(256) k_first_hit(const uint32_t* __restrict__ I,
                                                   const uint32_t* __restrict__ J, uint64_t m,
                                                   uint32_t* first) {
    const uint64_t quads = m >> 2;          // full 16-byte quads per array
    const uint64_t total = 2 * quads;
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(I) | reinterpret_cast<uintptr_t>(J)) & 15) == 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    // Uniform trip count across the warp so __match_any_sync sees full warps.
    const uint64_t warp_base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
    for (uint64_t w0 = warp_base; w0 < total; w0 += stride) {
        const uint64_t w = w0 + lane_id();
        const bool valid = w < total;
        uint4 q = make_uint4(0, 0, 0, 0);
        uint32_t pos = 0;
        if (valid) {
            const bool inJ = w >= quads;
            const uint64_t qi = inJ ? w - quads : w;
            const uint32_t* src = inJ ? J : I;
            if (vec_ok) {
                q = __ldg(reinterpret_cast<const uint4*>(src) + qi);
            } else {
                q.x = __ldg(src + 4 * qi); q.y = __ldg(src + 4 * qi + 1);
                q.z = __ldg(src + 4 * qi + 2); q.w = __ldg(src + 4 * qi + 3);
            }
            pos = (uint32_t)(4 * qi + (inJ ? m : 0));
        }
        hit<RELAXED>(first, q.x, pos, valid);
        hit<RELAXED>(first, q.y, pos + 1, valid);
        hit<RELAXED>(first, q.z, pos + 2, valid);
        hit<RELAXED>(first, q.w, pos + 3, valid);
    }
}

// The (m mod 4) tail elements of I and of J.
template <bool RELAXED>
__global__ void k_first_hit_tail(const uint32_t* __restrict__ I, const uint32_t* __restrict__ J,
                                 uint64_t m, uint32_t* first) {
    const uint64_t rem = m & 3, base = m & ~3ull;
    const unsigned t = threadIdx.x;  // 0..7
    if (t >= 2 * rem) return;
    const bool inJ = t >= rem;
    const uint64_t e = base + (inJ ? t - rem : t);
    const uint32_t v = inJ ? J[e] : I[e];
    const uint32_t pos = (uint32_t)(e + (inJ ? m : 0));
    if (RELAXED) {
        if (pos < *((volatile uint32_t*)(first + v))) *((volatile uint32_t*)(first + v)) = pos;
    } else {
        atomicMin(first + v, pos);
    }
}

cudaError_t launch_first_hit(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n,
                             uint32_t* first, bool relaxed, int num_sms, cudaStream_t s) {
    cudaError_t err = cudaMemsetAsync(first, 0xFF, (size_t)n * sizeof(uint32_t), s);
    if (err != cudaSuccess || m == 0) return err;
    const uint64_t total = 2 * (m >> 2);
    if (total) {
        uint64_t blocks = ceil_div(total, 256);
        uint64_t cap = (uint64_t)num_sms * 8;
        int grid = (int)(blocks < cap ? blocks : cap);
        if (relaxed)
            k_first_hit<true><<<grid, 256, 0, s>>>(I, J, m, first);
        else
            k_first_hit<false><<<grid, 256, 0, s>>>(I, J, m, first);
    }
    if (m & 3) {
        if (relaxed)
            k_first_hit_tail<true><<<1, 8, 0, s>>>(I, J, m, first);
        else
            k_first_hit_tail<false><<<1, 8, 0, s>>>(I, J, m, first);
    }
    return cudaGetLastError();
}

}  // namespace boba
