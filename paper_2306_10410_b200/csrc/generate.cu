// Input preparation and dtype plumbing (not on the timed BOBA path).
//
//  * R-MAT generator: device twin of oracle/boba_oracle.c oracle_rmat_edges
//    (Graph500 a,b,c,d = .57,.19,.19,.05; i.i.d. edges in generation order,
//    counter-based splitmix64 so any edge range is reproducible anywhere).
//    The reference has no R-MAT.
//  * 4-neighbour grid: reference generators.py:100-111 generate_grid.
//  * narrow / widen: the reference's int64 ids (graph.py:31) <-> the uint32
//    ids the kernels use, with the reference's range check
//    (graph.py:99-106: every endpoint in [0, n)).
#include "common.cuh"
#include "kernels.cuh"

namespace boba {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
constexpr uint32_t kTA = 2448131358u, kTB = 3264175144u, kTC = 4080218931u;

__global__ void k_rmat(int scale, uint64_t e0, uint64_t count, uint64_t seed, uint32_t* I, uint32_t* J) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const uint64_t e = e0 + i;
        uint64_t key = splitmix64(seed ^ splitmix64(e));
        uint32_t u = 0, v = 0;
        for (int lvl = 0; lvl < scale; lvl += 2) {
            uint64_t h = splitmix64(key + (uint64_t)lvl);
#pragma unroll
            for (int k = 0; k < 2; k++) {
                if (lvl + k >= scale) break;
                uint32_t x = (uint32_t)(h >> (32 * k));
                uint32_t bu = x >= kTB;
                uint32_t bv = (x >= kTA && x < kTB) || x >= kTC;
                u = (u << 1) | bu;
                v = (v << 1) | bv;
            }
        }
        I[i] = u;
        J[i] = v;
    }
}

__global__ void k_grid(uint32_t rows, uint32_t cols, uint32_t* I, uint32_t* J) {
    const uint64_t h = (uint64_t)rows * (cols - 1), vt = (uint64_t)(rows - 1) * cols;
    const uint64_t m = 2 * h + 2 * vt;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += stride) {
        uint64_t a, b;
        if (k < 2 * h) {
            uint64_t q = k < h ? k : k - h;
            uint64_t r = q / (cols - 1), c = q % (cols - 1);
            a = r * cols + c;
            b = a + 1;
            if (k >= h) { uint64_t t = a; a = b; b = t; }
        } else {
            uint64_t q = k - 2 * h;
            bool rev = q >= vt;
            if (rev) q -= vt;
            a = q;
            b = q + cols;
            if (rev) { uint64_t t = a; a = b; b = t; }
        }
        I[k] = (uint32_t)a;
        J[k] = (uint32_t)b;
    }
}

__global__ void k_narrow(const int64_t* __restrict__ in, uint64_t count, uint64_t bound, uint32_t* out,
                         unsigned long long* first_bad) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        int64_t v = __ldg(in + i);
        if (v < 0 || (uint64_t)v >= bound) atomicMin(first_bad, (unsigned long long)i);
        out[i] = (uint32_t)v;
    }
}

__global__ void k_widen(const uint32_t* __restrict__ in, uint64_t count, int64_t* out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
        out[i] = (int64_t)__ldg(in + i);
}

__global__ void k_gather_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ idx, uint64_t count,
                             uint32_t* out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
        out[i] = __ldg(src + __ldg(idx + i));
}

__global__ void k_bias(const uint32_t* __restrict__ in, uint64_t count, uint32_t* out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
        out[i] = __ldg(in + i) ^ 0x80000000u;
}

__global__ void k_offset_ids(const uint32_t* __restrict__ in, uint64_t count, uint32_t delta, uint32_t* out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
        out[i] = __ldg(in + i) + delta;
}

static int grid_for(uint64_t work, int num_sms) {
    uint64_t blocks = ceil_div(work, 256), cap = (uint64_t)num_sms * 16;
    blocks = blocks < cap ? blocks : cap;
    return (int)(blocks ? blocks : 1);
}

cudaError_t launch_rmat(int scale, uint64_t e0, uint64_t count, uint64_t seed, uint32_t* I, uint32_t* J,
                        int num_sms, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    k_rmat<<<grid_for(count, num_sms), 256, 0, s>>>(scale, e0, count, seed, I, J);
    return cudaGetLastError();
}

cudaError_t launch_grid(uint32_t rows, uint32_t cols, uint32_t* I, uint32_t* J, int num_sms, cudaStream_t s) {
    uint64_t m = 2ull * rows * (cols - 1) + 2ull * (rows - 1) * cols;
    if (m == 0) return cudaSuccess;
    k_grid<<<grid_for(m, num_sms), 256, 0, s>>>(rows, cols, I, J);
    return cudaGetLastError();
}

cudaError_t launch_narrow(const int64_t* in, uint64_t count, uint64_t bound, uint32_t* out,
                          unsigned long long* first_bad, int num_sms, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(first_bad, 0xFF, 8, s);
    if (e != cudaSuccess || count == 0) return e;
    k_narrow<<<grid_for(count, num_sms), 256, 0, s>>>(in, count, bound, out, first_bad);
    return cudaGetLastError();
}

cudaError_t launch_widen(const uint32_t* in, uint64_t count, int64_t* out, int num_sms, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    k_widen<<<grid_for(count, num_sms), 256, 0, s>>>(in, count, out);
    return cudaGetLastError();
}

cudaError_t launch_bias(const uint32_t* in, uint64_t count, uint32_t* out, int num_sms, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    k_bias<<<grid_for(count, num_sms), 256, 0, s>>>(in, count, out);
    return cudaGetLastError();
}

cudaError_t launch_offset_ids(const uint32_t* in, uint64_t count, uint32_t delta, uint32_t* out, int num_sms,
                              cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    k_offset_ids<<<grid_for(count, num_sms), 256, 0, s>>>(in, count, delta, out);
    return cudaGetLastError();
}

cudaError_t launch_gather_u32(const uint32_t* src, const uint32_t* idx, uint64_t count, uint32_t* out, int num_sms,
                              cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    k_gather_u32<<<grid_for(count, num_sms), 256, 0, s>>>(src, idx, count, out);
    return cudaGetLastError();
}

}  // namespace boba
