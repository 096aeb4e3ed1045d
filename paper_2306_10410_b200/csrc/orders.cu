// The orderings and edge-list sort that sit next to BOBA on the benchmarked
// pipeline:
//   * degree ordering -- reference ordering.py:160-164: total degree
//     (graph.py:297-300: bincount(I) + bincount(J)) descending, ties by
//     ascending id.  A stable LSD sort of the ids keyed by ~degree gives
//     exactly np.lexsort((arange(n), -deg)).
//   * hub ordering -- reference ordering.py:167-176: vertices with total
//     degree above the mean first (descending degree, ties by id), the rest
//     after them in id order.
//   * sort_coo_by_destination -- reference graph.py:303-307: stable sort of
//     the edge list by J (ties keep edge order), weights moved bit-exactly.
#include "common.cuh"
#include "kernels.cuh"

namespace boba {

__global__ void k_total_degrees(const uint32_t* __restrict__ I, const uint32_t* __restrict__ J, uint64_t m,
                                uint32_t* deg) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        atomicAdd(deg + __ldg(I + e), 1u);
        atomicAdd(deg + __ldg(J + e), 1u);
    }
}

// key = 2m - deg (ascending key == descending degree).  Hub ordering: the
// vertices with deg <= mean (deg * n <= 2m, exact in integers) all get key
// 2m + 1, so the stable sort keeps them after the hubs in id order.
__global__ void k_degree_key(uint32_t* deg, uint64_t n, uint64_t two_m, bool hub) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t d = deg[i];
        deg[i] = (hub && (uint64_t)d * n <= two_m) ? (uint32_t)(two_m + 1) : (uint32_t)(two_m - d);
    }
}

__global__ void k_invert_perm(const uint32_t* __restrict__ order, uint64_t n, uint32_t* label) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride)
        label[__ldg(order + k)] = (uint32_t)k;
}

__global__ void k_gather_edges(const uint32_t* __restrict__ eidx, uint64_t m, const uint32_t* __restrict__ I,
                               const double* __restrict__ w, uint32_t* I_out, double* w_out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += stride) {
        const uint32_t e = __ldg(eidx + k);
        I_out[k] = __ldg(I + e);
        w_out[k] = __ldg(w + e);
    }
}

static int grid_of(uint64_t work, int num_sms) {
    const uint64_t blocks = ceil_div(work ? work : 1, 256), cap = (uint64_t)num_sms * 16;
    return (int)(blocks < cap ? blocks : cap);
}

cudaError_t launch_total_degrees(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n, uint32_t* deg,
                                 int num_sms, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(deg, 0, (size_t)n * 4, s);
    if (e != cudaSuccess || m == 0) return e;
    k_total_degrees<<<grid_of(m, num_sms), 256, 0, s>>>(I, J, m, deg);
    return cudaGetLastError();
}

static int id_bits(uint64_t n) { return n <= 1 ? 0 : 64 - __builtin_clzll(n - 1); }

// keys lie in [0, 2m + 1]: the sort needs only bits(2m + 2) key bits
size_t degree_order_workspace_bytes(uint64_t m, uint32_t n) {
    return (((size_t)n * 4 + 255) & ~size_t(255)) + sort_pairs_workspace_bytes(n, id_bits(2 * m + 2));
}

cudaError_t launch_degree_order(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n, uint32_t* order,
                                uint32_t* label, void* ws, size_t ws_bytes, int num_sms, cudaStream_t s, bool hub) {
    if (ws_bytes < degree_order_workspace_bytes(m, n)) return cudaErrorInvalidValue;
    if (n == 0) return cudaSuccess;
    uint32_t* key = static_cast<uint32_t*>(ws);
    void* rest = static_cast<char*>(ws) + (((size_t)n * 4 + 255) & ~size_t(255));
    cudaError_t e = launch_total_degrees(I, J, m, n, key, num_sms, s);
    if (e != cudaSuccess) return e;
    k_degree_key<<<grid_of(n, num_sms), 256, 0, s>>>(key, n, 2 * m, hub);
    e = launch_sort_pairs(key, nullptr, n, id_bits(2 * m + 2), nullptr, order, rest, ws_bytes - (((size_t)n * 4 + 255) & ~size_t(255)),
                          num_sms, s);
    if (e != cudaSuccess) return e;
    k_invert_perm<<<grid_of(n, num_sms), 256, 0, s>>>(order, n, label);
    return cudaGetLastError();
}

size_t sort_by_destination_workspace_bytes(uint64_t m, uint32_t n) {
    return ((m * 4 + 255) & ~size_t(255)) + sort_pairs_workspace_bytes(m, id_bits(n));
}

cudaError_t launch_sort_by_destination(const uint32_t* I, const uint32_t* J, const double* w, uint64_t m, uint32_t n,
                                       uint32_t* I_out, uint32_t* J_out, double* w_out, void* ws, size_t ws_bytes,
                                       int num_sms, cudaStream_t s) {
    if (ws_bytes < sort_by_destination_workspace_bytes(m, n)) return cudaErrorInvalidValue;
    if (m == 0) return cudaSuccess;
    const size_t head = (m * 4 + 255) & ~size_t(255);
    uint32_t* eidx = static_cast<uint32_t*>(ws);
    void* rest = static_cast<char*>(ws) + head;
    if (!w)  // payload = the source id itself
        return launch_sort_pairs(J, I, m, id_bits(n), J_out, I_out, rest, ws_bytes - head, num_sms, s);
    cudaError_t e = launch_sort_pairs(J, nullptr, m, id_bits(n), J_out, eidx, rest, ws_bytes - head, num_sms, s);
    if (e != cudaSuccess) return e;
    k_gather_edges<<<grid_of(m, num_sms), 256, 0, s>>>(eidx, m, I, w, I_out, w_out);
    return cudaGetLastError();
}

}  // namespace boba
