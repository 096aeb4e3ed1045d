// Multi-GPU row cut for the row-partitioned CSR (paper_2306_10410_b200/sharded.py).
//
// After relabel, rank r holds the relabelled edges of its contiguous shard.
// The CSR rows are split into P contiguous row ranges of ~m/P edges each,
// owned by ranks 0..P-1.  Choosing the cut needs the global row histogram;
// an n-sized allreduce of it (268 MB at s26) is avoided with a coarse one:
//
//   k_coarse_hist  histogram of rows >> shift over B <= 32768 buckets, in
//                  shared memory per CTA, flushed with one atomic per bucket;
//   (allreduce-SUM of the B-word histogram -- 128 KB)
//   k_row_cut      one CTA: prefix sums of the global and the local coarse
//                  histograms; cut k is the first bucket boundary whose global
//                  prefix reaches k*m/P.  Writes the row bounds, each owner's
//                  first global edge offset and this rank's send counts (the
//                  local prefix at the bounds -- exact, since bounds sit on
//                  bucket boundaries).
//
// The send side is then one stable range partition (csr.cu, keys written
// relative to the owner's first row), the exchange an all-to-all, and the
// owner's CSR the one-GPU stable COO->CSR of what it received: senders are
// ranks in order and shards are contiguous in edge order, so the received
// sequence is global edge order restricted to the owner's rows -- the
// reference's within-row order (_parallel.py:55-88), bit-exact.
#include "common.cuh"
#include "kernels.cuh"

namespace boba {

constexpr uint32_t kCutMaxBuckets = 32768;
constexpr int kCutNT = 1024;

int row_cut_shift(uint32_t n) {
    const int bits = n <= 1 ? 0 : 32 - __builtin_clz(n - 1);
    return bits > 15 ? bits - 15 : 0;
}

uint32_t row_cut_buckets(uint32_t n) {
    const int sh = row_cut_shift(n);
    return n == 0 ? 1u : (uint32_t)(((uint64_t)n + (1ull << sh) - 1) >> sh);
}

__global__ void k_coarse_hist(const uint32_t* __restrict__ rows, uint64_t m, int shift, uint32_t B,
                              uint32_t* __restrict__ hist) {
    extern __shared__ uint32_t s_h[];
    for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) s_h[b] = 0;
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t quads = (reinterpret_cast<uintptr_t>(rows) & 15) == 0 ? m >> 2 : 0;
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < quads; q += stride) {
        const uint4 r = __ldg(reinterpret_cast<const uint4*>(rows) + q);
        atomicAdd(s_h + (r.x >> shift), 1u);
        atomicAdd(s_h + (r.y >> shift), 1u);
        atomicAdd(s_h + (r.z >> shift), 1u);
        atomicAdd(s_h + (r.w >> shift), 1u);
    }
    for (uint64_t e = 4 * quads + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride)
        atomicAdd(s_h + (__ldg(rows + e) >> shift), 1u);
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < B; b += blockDim.x)
        if (s_h[b]) atomicAdd(hist + b, s_h[b]);
}

// out (3P + 2 words): [0, P]      row bounds b_0 = 0 <= ... <= b_P = n
//                     [P+1, 2P+1] global edge offset of each bound (offsets[b_k])
//                     [2P+2, 3P+1] edges this rank sends to owner k
__global__ void __launch_bounds__(kCutNT) k_row_cut(const uint32_t* __restrict__ hist_g,
                                                    const uint32_t* __restrict__ hist_l, uint32_t B, int shift,
                                                    uint32_t n, uint64_t m, int P, uint32_t* __restrict__ out) {
    constexpr int kPer = kCutMaxBuckets / kCutNT;  // 32 buckets per thread
    __shared__ unsigned long long s_g[kCutNT], s_l[kCutNT];
    __shared__ unsigned long long s_cut_l[257];
    const uint32_t b0 = threadIdx.x * kPer;
    unsigned long long g = 0, l = 0;
    for (int i = 0; i < kPer; i++)
        if (b0 + i < B) g += hist_g[b0 + i], l += hist_l[b0 + i];
    s_g[threadIdx.x] = g;
    s_l[threadIdx.x] = l;
    __syncthreads();
    // exclusive prefix of the per-thread sums (Hillis-Steele in shared memory, 1024 entries)
    for (int o = 1; o < kCutNT; o <<= 1) {
        unsigned long long a = threadIdx.x >= (unsigned)o ? s_g[threadIdx.x - o] : 0ull;
        unsigned long long c = threadIdx.x >= (unsigned)o ? s_l[threadIdx.x - o] : 0ull;
        __syncthreads();
        s_g[threadIdx.x] += a;
        s_l[threadIdx.x] += c;
        __syncthreads();
    }
    unsigned long long G = s_g[threadIdx.x] - g, L = s_l[threadIdx.x] - l;  // prefixes at b0
    // bucket boundary b (0..B) with prefix G_b: cut k is the smallest b with G_b >= k*m/P
    for (int i = 0; i <= kPer; i++) {
        const uint32_t b = b0 + i;
        if (b > B || (i == kPer && b != B)) break;   // boundary B is checked by its owner only
        const unsigned long long Gprev = G;          // G_b
        for (int k = 1; k < P; k++) {
            const unsigned long long t = (unsigned long long)k * m / (unsigned long long)P;
            // first b with G_b >= t: G_b >= t and (b == 0 or G_{b-1} < t); G_{b-1} = G_b - hist_g[b-1]
            const unsigned long long before = b == 0 ? 0ull : Gprev - hist_g[b - 1];
            if (Gprev >= t && (b == 0 || before < t)) {
                const uint64_t row = (uint64_t)b << shift;
                out[k] = (uint32_t)(row < n ? row : n);
                out[P + 1 + k] = (uint32_t)Gprev;
                s_cut_l[k] = L;
            }
        }
        if (b < B) {
            G += hist_g[b];
            L += hist_l[b];
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        out[0] = 0;
        out[P] = n;
        out[P + 1] = 0;
        out[2 * P + 1] = (uint32_t)m;
        s_cut_l[0] = 0;
        s_cut_l[P] = s_l[kCutNT - 1];  // inclusive total of the local histogram
        for (int k = 0; k < P; k++) out[2 * P + 2 + k] = (uint32_t)(s_cut_l[k + 1] - s_cut_l[k]);
    }
}

cudaError_t launch_coarse_hist(const uint32_t* rows, uint64_t m, uint32_t n, uint32_t* hist, int num_sms,
                               cudaStream_t s) {
    const uint32_t B = row_cut_buckets(n);
    cudaError_t e = cudaMemsetAsync(hist, 0, (size_t)B * 4, s);
    if (e != cudaSuccess || m == 0) return e;
    static PerDeviceOnce attr;
    const int smem = (int)(B * 4);
    if (smem > 48 * 1024) {
        e = set_attr_once(attr, k_coarse_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kCutMaxBuckets * 4));
        if (e != cudaSuccess) return e;
    }
    const uint64_t blocks = ceil_div(m, 4 * 512);
    const int grid = (int)(blocks < (uint64_t)num_sms ? blocks : (uint64_t)num_sms);
    k_coarse_hist<<<grid, 512, smem, s>>>(rows, m, row_cut_shift(n), B, hist);
    return cudaGetLastError();
}

cudaError_t launch_row_cut(const uint32_t* hist_g, const uint32_t* hist_l, uint32_t n, uint64_t m, int parts,
                           uint32_t* out, cudaStream_t s) {
    if (parts < 1 || parts > 256) return cudaErrorInvalidValue;
    k_row_cut<<<1, kCutNT, 0, s>>>(hist_g, hist_l, row_cut_buckets(n), row_cut_shift(n), n, m, parts, out);
    return cudaGetLastError();
}

}  // namespace boba
