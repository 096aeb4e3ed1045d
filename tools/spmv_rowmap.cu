// Row-mapped CSR SpMV kernels (fp32, y = A x, unit weights) -- the forms the
// north star names ("warp- or vector-per-row"), built only to compare against
// the library's merge-path SpMV (tools/spmv_rowmap_ab.py).  Not product code.
//   L = 1:  one thread per row (CSR-scalar)
//   L = 2..32: L lanes per row, strided over the row, shuffle-reduced
//           (CSR-vector; L = 32 is warp-per-row)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//        tools/spmv_rowmap.cu -o ab/libspmv_rowmap.so
#include <cstdint>
#include <cuda_runtime.h>

template <int L>
__global__ void __launch_bounds__(256) k_spmv_rows(const uint32_t* __restrict__ off, const uint32_t* __restrict__ idx,
                                                   const float* __restrict__ x, float* __restrict__ y, uint32_t n) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t groups = (uint64_t)gridDim.x * blockDim.x / L;
    const unsigned lane = threadIdx.x % L;
    for (uint64_t row = tid / L; row < n; row += groups) {
        const uint32_t b = __ldg(off + row), e = __ldg(off + row + 1);
        float s = 0.f;
        for (uint32_t k = b + lane; k < e; k += L) s += __ldg(x + __ldg(idx + k));
#pragma unroll
        for (int w = L / 2; w > 0; w >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, w, L);
        if (lane == 0) y[row] = s;
    }
}

template <int L>
static int launch(const uint32_t* off, const uint32_t* idx, const float* x, float* y, uint32_t n, int sms,
                  cudaStream_t s) {
    const uint64_t want = ((uint64_t)n * L + 255) / 256, cap = (uint64_t)sms * 32;
    const unsigned grid = (unsigned)(want < cap ? (want ? want : 1) : cap);
    k_spmv_rows<L><<<grid, 256, 0, s>>>(off, idx, x, y, n);
    return (int)cudaGetLastError();
}

extern "C" int spmv_rows(int lanes, const uint32_t* off, const uint32_t* idx, const float* x, float* y, uint32_t n,
                         int sms, cudaStream_t s) {
    switch (lanes) {
        case 1: return launch<1>(off, idx, x, y, n, sms, s);
        case 2: return launch<2>(off, idx, x, y, n, sms, s);
        case 4: return launch<4>(off, idx, x, y, n, sms, s);
        case 8: return launch<8>(off, idx, x, y, n, sms, s);
        case 16: return launch<16>(off, idx, x, y, n, sms, s);
        case 32: return launch<32>(off, idx, x, y, n, sms, s);
    }
    return -1;
}
