// Phase 1 -- first occurrence of every vertex in the flattened edge stream
// I||J (positions: I[e] -> e, J[e] -> m + e).
//
// Reference: pkg/src/boba/_parallel.py:139-162 first_hit_chunked (exact
// chunk-local minimum merged exactly) and :165-175 first_hit_racy (guarded
// unsynchronised writes).  Here the minimum is a device-wide atomicMin on
// uint32 (2m <= 2^32 - 2, UNSET = 0xFFFFFFFF).
//
// Cost model: the stream is read once (8m bytes, coalesced 16-byte loads);
// the per-endpoint work is a 4-byte random access to first[] (4n bytes,
// L2-resident up to n ~ 25M), and the L2 request rate for those -- not HBM
// bandwidth -- is what bounds a naive kernel.  Two things cut it:
//  * the grid sweeps the stream in position order (persistent CTAs,
//    block-cyclic over 2048-position iterations), so an atomic is issued only
//    when a plain (L1-cacheable; stale values are conservative because
//    first[] only decreases) load shows the position can still lower first[v];
//  * each CTA keeps a 32K-slot shared-memory set of vertices already known
//    to be finalised, i.e. first[v] < the lowest position the CTA will touch
//    from now on.  Hubs of skewed graphs recur early and settle in the set
//    ("insert if the slot is empty"), so most hub endpoints never leave the
//    SM.  Iterations are separated by a CTA barrier so the invariant holds
//    for every warp.
#include "common.cuh"
#include "kernels.cuh"

namespace boba {

constexpr int kFhNT = 1024;              // threads per CTA (one CTA per SM)
constexpr int kFhQuads = 2;              // 16-byte quads per thread per iteration
constexpr int kFhIter = kFhNT * kFhQuads * 4;   // positions per CTA iteration
constexpr int kFhSlotsLog2 = 15;         // 32K-slot finalised-vertex set (128 KB)
constexpr uint32_t kEmpty = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t slot_of(uint32_t v) { return (v * 0x9E3779B1u) >> (32 - kFhSlotsLog2); }

template <bool RELAXED>
__device__ __forceinline__ void hit(uint32_t* first, uint32_t* set, uint32_t v, uint32_t pos, uint32_t iter_lo) {
    const uint32_t s = slot_of(v);
    if (set[s] == v) return;                       // finalised: first[v] < iter_lo <= pos
    const uint32_t cur = first[v];                 // plain load: may be stale (>= true value)
    if (pos < cur) {
        if (RELAXED)
            *((volatile uint32_t*)(first + v)) = pos;
        else
            atomicMin(first + v, pos);
    } else if (cur < iter_lo && set[s] == kEmpty) {
        set[s] = v;                                // benign race: any writer's v is finalised
    }
}

template <bool RELAXED>
__global__ void __launch_bounds__(kFhNT, 1) k_first_hit(const uint32_t* __restrict__ I,
                                                        const uint32_t* __restrict__ J, uint64_t m,
                                                        uint32_t base_i, uint32_t base_j, uint32_t* first) {
    extern __shared__ uint32_t set[];
    for (int i = threadIdx.x; i < (1 << kFhSlotsLog2); i += kFhNT) set[i] = kEmpty;
    const uint64_t quads = m >> 2;          // full 16-byte quads per array
    const uint64_t total_q = 2 * quads;     // quads of I then quads of J
    const uint64_t iters = ceil_div(total_q, (uint64_t)kFhNT * kFhQuads);
    for (uint64_t it = blockIdx.x; it < iters; it += gridDim.x) {
        __syncthreads();  // every warp has left the previous iteration
        const uint64_t q0 = it * kFhNT * kFhQuads;
        // lowest position of this iteration (quads of J start at position m)
        const uint32_t iter_lo = (uint32_t)(q0 < quads ? base_i + 4 * q0 : base_j + 4 * (q0 - quads));
        uint4 q[kFhQuads];
        uint32_t pos[kFhQuads];
        bool ok[kFhQuads];
#pragma unroll
        for (int k = 0; k < kFhQuads; k++) {
            const uint64_t w = q0 + (uint64_t)k * kFhNT + threadIdx.x;
            ok[k] = w < total_q;
            if (ok[k]) {
                const bool inJ = w >= quads;
                const uint64_t qi = inJ ? w - quads : w;
                q[k] = __ldg(reinterpret_cast<const uint4*>(inJ ? J : I) + qi);
                pos[k] = (uint32_t)(4 * qi) + (inJ ? base_j : base_i);
            }
        }
#pragma unroll
        for (int k = 0; k < kFhQuads; k++) {
            if (!ok[k]) continue;
            hit<RELAXED>(first, set, q[k].x, pos[k], iter_lo);
            hit<RELAXED>(first, set, q[k].y, pos[k] + 1, iter_lo);
            hit<RELAXED>(first, set, q[k].z, pos[k] + 2, iter_lo);
            hit<RELAXED>(first, set, q[k].w, pos[k] + 3, iter_lo);
        }
    }
}

// Scalar path: unaligned inputs and the (m mod 4) tails.
template <bool RELAXED>
__global__ void k_first_hit_scalar(const uint32_t* __restrict__ I, const uint32_t* __restrict__ J, uint64_t e0,
                                   uint64_t m, uint32_t base_i, uint32_t base_j, uint32_t* first) {
    const uint64_t cnt = m - e0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < 2 * cnt; t += stride) {
        const bool inJ = t >= cnt;
        const uint64_t e = e0 + (inJ ? t - cnt : t);
        const uint32_t v = inJ ? J[e] : I[e];
        const uint32_t pos = (uint32_t)e + (inJ ? base_j : base_i);
        if (RELAXED) {
            if (pos < *((volatile uint32_t*)(first + v))) *((volatile uint32_t*)(first + v)) = pos;
        } else {
            atomicMin(first + v, pos);
        }
    }
}

cudaError_t launch_first_hit(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n, uint32_t* first,
                             bool relaxed, int num_sms, cudaStream_t s) {
    return launch_first_hit_shard(I, J, m, m, 0, n, first, relaxed, num_sms, s);
}

// A contiguous shard [e0, e0 + m) of a global edge list with m_global edges:
// local I[i] sits at global position e0 + i, local J[i] at m_global + e0 + i.
cudaError_t launch_first_hit_shard(const uint32_t* I, const uint32_t* J, uint64_t m, uint64_t m_global, uint64_t e0,
                                   uint32_t n, uint32_t* first, bool relaxed, int num_sms, cudaStream_t s) {
    const uint32_t base_i = (uint32_t)e0, base_j = (uint32_t)(m_global + e0);
    cudaError_t err = cudaMemsetAsync(first, 0xFF, (size_t)n * sizeof(uint32_t), s);
    if (err != cudaSuccess || m == 0) return err;
    const bool vec = ((reinterpret_cast<uintptr_t>(I) | reinterpret_cast<uintptr_t>(J)) & 15) == 0;
    uint64_t done = 0;
    if (vec && m >= 4) {
        const size_t smem = sizeof(uint32_t) << kFhSlotsLog2;
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_first_hit<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(k_first_hit<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            attr = true;
        }
        const uint64_t iters = ceil_div(2 * (m >> 2), (uint64_t)kFhNT * kFhQuads);
        const int grid = (int)(iters < (uint64_t)num_sms ? iters : (uint64_t)num_sms);
        if (relaxed)
            k_first_hit<true><<<grid, kFhNT, smem, s>>>(I, J, m, base_i, base_j, first);
        else
            k_first_hit<false><<<grid, kFhNT, smem, s>>>(I, J, m, base_i, base_j, first);
        done = m & ~3ull;
    }
    if (done < m) {
        uint64_t work = 2 * (m - done), blocks = ceil_div(work, 256), cap = (uint64_t)num_sms * 8;
        int grid = (int)(blocks < cap ? blocks : cap);
        if (relaxed)
            k_first_hit_scalar<true><<<grid, 256, 0, s>>>(I, J, done, m, base_i, base_j, first);
        else
            k_first_hit_scalar<false><<<grid, 256, 0, s>>>(I, J, done, m, base_i, base_j, first);
    }
    return cudaGetLastError();
}

}  // namespace boba
