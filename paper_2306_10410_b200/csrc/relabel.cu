// Phase 3 -- relabel the edge list through label[] (new id of every old id).
//
// Reference: pkg/src/boba/graph.py:280-289 apply_permutation:
// (label[I], label[J]) with edge order (and weights) unchanged.
//
// One pass: 16-byte loads of I and J, eight read-only-path gathers from
// label[] (4n bytes; L2-resident for n <= ~25M), 16-byte stores of I2 and
// J2.  Optionally fuses the out-degree histogram of the new rows (the
// np.bincount of graph.py:270 for the following COO->CSR) as RED.ADD.
#include "common.cuh"
#include "kernels.cuh"

namespace boba {

template <bool HIST>
__global__ void __launch_bounds__(256) k_relabel(const uint4* __restrict__ I, const uint4* __restrict__ J,
                                                 uint64_t quads, const uint32_t* __restrict__ label,
                                                 uint4* __restrict__ I2, uint4* __restrict__ J2,
                                                 uint32_t* counts) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < quads; q += stride) {
        uint4 a = __ldg(I + q), b = __ldg(J + q);
        uint4 ra, rb;
        ra.x = __ldg(label + a.x); ra.y = __ldg(label + a.y); ra.z = __ldg(label + a.z); ra.w = __ldg(label + a.w);
        rb.x = __ldg(label + b.x); rb.y = __ldg(label + b.y); rb.z = __ldg(label + b.z); rb.w = __ldg(label + b.w);
        I2[q] = ra;
        J2[q] = rb;
        if (HIST) {
            atomicAdd(counts + ra.x, 1u); atomicAdd(counts + ra.y, 1u);
            atomicAdd(counts + ra.z, 1u); atomicAdd(counts + ra.w, 1u);
        }
    }
}

template <bool HIST>
__global__ void k_relabel_scalar(const uint32_t* __restrict__ I, const uint32_t* __restrict__ J,
                                 uint64_t e0, uint64_t m, const uint32_t* __restrict__ label,
                                 uint32_t* I2, uint32_t* J2, uint32_t* counts) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = e0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        uint32_t r = __ldg(label + I[e]);
        I2[e] = r;
        J2[e] = __ldg(label + J[e]);
        if (HIST) atomicAdd(counts + r, 1u);
    }
}

cudaError_t launch_relabel(const uint32_t* I, const uint32_t* J, uint64_t m, const uint32_t* label,
                           uint32_t* I2, uint32_t* J2, uint32_t* counts, uint32_t n, int num_sms,
                           cudaStream_t s) {
    if (counts) {
        cudaError_t err = cudaMemsetAsync(counts, 0, (size_t)n * 4, s);
        if (err != cudaSuccess) return err;
    }
    if (m == 0) return cudaSuccess;
    const bool vec = ((reinterpret_cast<uintptr_t>(I) | reinterpret_cast<uintptr_t>(J) |
                       reinterpret_cast<uintptr_t>(I2) | reinterpret_cast<uintptr_t>(J2)) & 15) == 0;
    uint64_t done = 0;
    const uint64_t cap = (uint64_t)num_sms * 8;
    if (vec && m >= 4) {
        const uint64_t quads = m >> 2;
        uint64_t blocks = ceil_div(quads, 256);
        int grid = (int)(blocks < cap ? blocks : cap);
        if (counts)
            k_relabel<true><<<grid, 256, 0, s>>>((const uint4*)I, (const uint4*)J, quads, label, (uint4*)I2,
                                                 (uint4*)J2, counts);
        else
            k_relabel<false><<<grid, 256, 0, s>>>((const uint4*)I, (const uint4*)J, quads, label, (uint4*)I2,
                                                  (uint4*)J2, counts);
        done = quads * 4;
    }
    if (done < m) {
        uint64_t blocks = ceil_div(m - done, 256);
        int grid = (int)(blocks < cap ? blocks : cap);
        if (counts)
            k_relabel_scalar<true><<<grid, 256, 0, s>>>(I, J, done, m, label, I2, J2, counts);
        else
            k_relabel_scalar<false><<<grid, 256, 0, s>>>(I, J, done, m, label, I2, J2, counts);
    }
    return cudaGetLastError();
}

}  // namespace boba
