// PageRank by power iteration on the GPU -- reference kernels.py:57-107
// (SURVEY.md §8f "next": the consumer of the reordered CSR).
//
// Setup (once per call):
//   out_weight[v] = row sums of the forward weights (ones when unweighted),
//   dangling = out_weight == 0; share[e] = w[e] / (dangling ? 1 : ow[src]);
//   rev = COO->CSR of (J, I, share) -- the reference builds exactly this
//   reversed graph (kernels.py:92-95) with its stable coo_to_csr, so rev's
//   rows hold in-edges in forward-CSR order, as there.
// Iterations (all max_iters launched back to back, no host round trip):
//   y = rev * x                                      (merge-path SpMV, fp64)
//   x' = d * (y + dm) + (1 - d) / n;  delta = |x' - x|_1;  dm' = sum x'[dangling] / n
// A device stop flag, raised by the reduction kernel when delta < tol, makes
// every later kernel return at once, so the host never waits per iteration
// and the result is the reference's: same update, same stopping rule.
// Reductions are fixed-grid block partials summed in a fixed order, so the
// result is bitwise deterministic run to run.
#include "common.cuh"
#include "kernels.cuh"

namespace boba {

namespace {

constexpr int kPrNT = 256;

struct PrState {
    int stop;
    uint32_t iters;
    double dm;
    double delta;
};

__device__ __forceinline__ double block_sum(double v, double* s_w) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) s_w[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < (int)(blockDim.x >> 5); k++) t += s_w[k];
    return t;  // valid in thread 0
}

// forward edge -> its source row (upper bound over offsets[1..n])
__global__ void k_edge_src(const uint32_t* __restrict__ offsets, uint32_t n, uint64_t m, uint32_t* src) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        uint32_t lo = 0, hi = n;  // first v with offsets[v + 1] > e
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if ((uint64_t)__ldg(offsets + mid + 1) > e)
                hi = mid;
            else
                lo = mid + 1;
        }
        src[e] = lo;
    }
}

__global__ void k_out_weight_unweighted(const uint32_t* __restrict__ offsets, uint32_t n, double* ow) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride)
        ow[v] = (double)(__ldg(offsets + v + 1) - __ldg(offsets + v));
}

__global__ void k_fill_f64(double* a, uint64_t count, double val) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) a[i] = val;
}

__global__ void k_dangling(const double* __restrict__ ow, uint32_t n, uint8_t* dang) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) dang[v] = ow[v] == 0.0;
}

// share[e] = w[e] / (dangling[src] ? 1 : ow[src])  (kernels.py:94)
__global__ void k_share(const uint32_t* __restrict__ src, const double* __restrict__ w, const double* __restrict__ ow,
                        uint64_t m, double* share) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        const double o = ow[src[e]];
        share[e] = __ddiv_rn(w ? w[e] : 1.0, o == 0.0 ? 1.0 : o);
    }
}

// x = 1/n; partial sums of x over the dangling vertices
__global__ void __launch_bounds__(kPrNT) k_pr_init(double* x, const uint8_t* __restrict__ dang, uint32_t n,
                                                   double inv_n, double* partials) {
    __shared__ double s_w[kPrNT / 32];
    double ds = 0.0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
        x[v] = inv_n;
        if (dang[v]) ds += inv_n;
    }
    const double t = block_sum(ds, s_w);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = 0.0;
        partials[2 * blockIdx.x + 1] = t;
    }
}

// x <- d * (y + dm) + tele in place (y = rev * x already computed); partials
// of |x' - x| and of x' over the dangling vertices.  Explicit _rn ops: no FMA
// contraction, the same roundings as the reference's numpy expression.
__global__ void __launch_bounds__(kPrNT) k_pr_update(double* x, const double* __restrict__ y,
                                                     const uint8_t* __restrict__ dang, uint32_t n, double d,
                                                     double tele, const PrState* st, double* partials) {
    if (*(volatile const int*)&st->stop) return;
    __shared__ double s_w[kPrNT / 32];
    const double dm = st->dm;
    double dl = 0.0, ds = 0.0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
        const double xn = __dadd_rn(__dmul_rn(d, __dadd_rn(y[v], dm)), tele);
        dl += fabs(xn - x[v]);
        x[v] = xn;
        if (dang[v]) ds += xn;
    }
    const double a = block_sum(dl, s_w);
    const double b = block_sum(ds, s_w);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = a;
        partials[2 * blockIdx.x + 1] = b;
    }
}

// one CTA: fold the partials in block order; init == true only sets dm.
__global__ void __launch_bounds__(1024) k_pr_reduce(const double* __restrict__ partials, int G, uint32_t n, double tol,
                                                    PrState* st, bool init) {
    if (*(volatile int*)&st->stop) return;
    __shared__ double s_w[32];
    double dl = 0.0, ds = 0.0;
    for (int b = threadIdx.x; b < G; b += blockDim.x) {
        dl += partials[2 * b];
        ds += partials[2 * b + 1];
    }
    const double a = block_sum(dl, s_w);
    const double c = block_sum(ds, s_w);
    if (threadIdx.x == 0) {
        st->dm = c / (double)n;
        if (!init) {
            st->iters += 1;
            st->delta = a;
            if (a < tol) st->stop = 1;
        }
    }
}

int pr_grid(uint32_t n, int num_sms) {
    const uint64_t b = ceil_div((uint64_t)(n ? n : 1), kPrNT), cap = (uint64_t)num_sms * 4;
    return (int)(b < cap ? b : cap);
}

struct PrWs {
    double *ow, *share, *rev_w, *y, *partials;
    uint8_t* dang;
    uint32_t *src, *rev_off, *rev_idx;
    PrState* st;
    void *csr_ws, *spmv_ws;
    size_t csr_bytes, spmv_bytes, total;
};

PrWs carve_pr(void* base, uint32_t n, uint64_t m, int num_sms) {
    PrWs w{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return base ? static_cast<char*>(base) + o : nullptr;
    };
    w.ow = (double*)take((size_t)n * 8);
    w.y = (double*)take((size_t)n * 8);
    w.dang = (uint8_t*)take(n);
    w.src = (uint32_t*)take(m * 4);
    w.share = (double*)take(m * 8);
    w.rev_off = (uint32_t*)take(((size_t)n + 1) * 4);
    w.rev_idx = (uint32_t*)take(m * 4);
    w.rev_w = (double*)take(m * 8);
    w.partials = (double*)take((size_t)pr_grid(n, num_sms) * 16);
    w.st = (PrState*)take(sizeof(PrState));
    w.csr_bytes = coo_to_csr_workspace_bytes(m, n, true);
    w.csr_ws = take(w.csr_bytes);
    w.spmv_bytes = spmv_workspace_bytes(n, m);
    w.spmv_ws = take(w.spmv_bytes);
    w.total = off;
    return w;
}

int grid_of(uint64_t work, int num_sms) {
    const uint64_t blocks = ceil_div(work ? work : 1, 256), cap = (uint64_t)num_sms * 16;
    return (int)(blocks < cap ? blocks : cap);
}

}  // namespace

size_t pagerank_workspace_bytes(uint32_t n, uint64_t m, int num_sms) { return carve_pr(nullptr, n, m, num_sms).total; }

cudaError_t launch_pagerank(const uint32_t* offsets, const uint32_t* indices, const double* w, uint32_t n, uint64_t m,
                            double damping, double tol, int max_iters, double* x, uint32_t* iterations, void* ws,
                            size_t ws_bytes, int num_sms, cudaStream_t s) {
    PrWs W = carve_pr(ws, n, m, num_sms);
    if (ws_bytes < W.total) return cudaErrorInvalidValue;
    if (n == 0) return iterations ? cudaMemsetAsync(iterations, 0, 4, s) : cudaSuccess;
    cudaError_t e = cudaMemsetAsync(W.st, 0, sizeof(PrState), s);
    if (e != cudaSuccess) return e;
    // out weights and dangling flags (kernels.py:88-89)
    if (w) {
        k_fill_f64<<<grid_of(n, num_sms), 256, 0, s>>>(W.y, n, 1.0);
        e = launch_spmv_f64(offsets, indices, w, W.y, W.ow, n, m, W.spmv_ws, W.spmv_bytes, s);
        if (e != cudaSuccess) return e;
    } else {
        k_out_weight_unweighted<<<grid_of(n, num_sms), 256, 0, s>>>(offsets, n, W.ow);
    }
    k_dangling<<<grid_of(n, num_sms), 256, 0, s>>>(W.ow, n, W.dang);
    // reversed graph with normalised shares (kernels.py:91-95)
    if (m) {
        k_edge_src<<<grid_of(m, num_sms), 256, 0, s>>>(offsets, n, m, W.src);
        k_share<<<grid_of(m, num_sms), 256, 0, s>>>(W.src, w, W.ow, m, W.share);
    }
    e = launch_coo_to_csr(indices, W.src, W.share, m, n, nullptr, W.rev_off, W.rev_idx, W.rev_w, W.csr_ws,
                          W.csr_bytes, num_sms, s);
    if (e != cudaSuccess) return e;
    // x0 = 1/n and the first dangling mass (kernels.py:97-101)
    const int G = pr_grid(n, num_sms);
    k_pr_init<<<G, kPrNT, 0, s>>>(x, W.dang, n, 1.0 / (double)n, W.partials);
    k_pr_reduce<<<1, 1024, 0, s>>>(W.partials, G, n, tol, W.st, true);
    const double tele = (1.0 - damping) / (double)n;
    for (int it = 0; it < max_iters; it++) {
        e = launch_spmv_f64_iter(W.rev_off, W.rev_idx, W.rev_w, x, W.y, n, m, W.spmv_ws, W.spmv_bytes, s, &W.st->stop,
                                 it > 0);
        if (e != cudaSuccess) return e;
        k_pr_update<<<G, kPrNT, 0, s>>>(x, W.y, W.dang, n, damping, tele, W.st, W.partials);
        k_pr_reduce<<<1, 1024, 0, s>>>(W.partials, G, n, tol, W.st, false);
    }
    if (iterations) e = cudaMemcpyAsync(iterations, &W.st->iters, 4, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace boba
