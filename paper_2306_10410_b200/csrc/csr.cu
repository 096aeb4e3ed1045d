// Phase 4 -- COO -> CSR with the reference's within-row order.
//
// Reference: pkg/src/boba/graph.py:253-277 coo_to_csr (counts =
// bincount(I), offsets = [0, cumsum(counts)]) and _parallel.py:55-88
// scatter_rows (a cursor per row, edges visited in edge-list order: row v
// holds its destinations in edge-list order -- a STABLE counting sort).
//
// B200 formulation:
//   offsets   exclusive scan of the row histogram (single-pass decoupled
//             lookback), offsets[n] = m.
//   scatter   a stable LSD radix sort of (row, payload) pairs keyed by row,
//             ceil(bits(n-1)/8) passes of reduce-then-scan (radix.cuh): tile
//             digit histograms, one scan over them, then a downsweep that
//             ranks each tile stably in shared memory and writes per-digit
//             runs.  Payload = J2 (unweighted: the last pass writes `indices`
//             directly) or the edge index (weighted: a final gather moves J2
//             and the float64 weights bit-exactly).
#include "common.cuh"
#include "kernels.cuh"

#include <algorithm>
#include <cstdlib>

namespace boba {

// ------------------------------------------------------------- histogram ---
__global__ void k_hist(const uint32_t* __restrict__ I, uint64_t m, uint32_t* counts) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride)
        atomicAdd(counts + __ldg(I + e), 1u);
}

// ---------------------------------------------------------- offsets scan ---
constexpr int kOffNT = 256, kOffIPT = 8, kOffTile = kOffNT * kOffIPT;

__global__ void __launch_bounds__(kOffNT) k_scan_offsets(const uint32_t* __restrict__ counts, uint32_t n,
                                                         uint32_t* offsets, unsigned long long* status,
                                                         unsigned* tile_counter) {
    __shared__ unsigned s_tile;
    __shared__ uint32_t s_scan[kOffNT / 32 + 1];
    __shared__ unsigned long long s_excl;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t r0 = tile * kOffTile + (uint64_t)threadIdx.x * kOffIPT;
    uint32_t c[kOffIPT];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kOffIPT; k++) {
        c[k] = (r0 + k < n) ? __ldg(counts + r0 + k) : 0u;
        sum += c[k];
    }
    uint32_t total;
    uint32_t ex_t = block_exclusive_sum<kOffNT>(sum, s_scan, &total);
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0)
            st_volatile_u64(status + tile, (tile == 0 ? kFlagInc : kFlagAgg) | (unsigned long long)total);
        unsigned long long ex = tile == 0 ? 0ull : warp_lookback(status, (long long)tile);
        if (threadIdx.x == 0) {
            if (tile != 0) st_volatile_u64(status + tile, kFlagInc | (ex + total));
            s_excl = ex;
        }
    }
    __syncthreads();
    uint32_t run = (uint32_t)s_excl + ex_t;
#pragma unroll
    for (int k = 0; k < kOffIPT; k++) {
        if (r0 + k <= n) offsets[r0 + k] = run;  // r0+k == n writes offsets[n] = m
        run += c[k];
    }
}

__global__ void k_set_u32(uint32_t* p, uint32_t v) { *p = v; }

// zeroes words[0, n) and *also (kernel-node replacement for two memsets)
__global__ void k_zero_u32(uint32_t* words, uint64_t n, uint32_t* also) {
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) words[i] = 0u;
    if (threadIdx.x == 0) *also = 0u;
}

static cudaError_t launch_set_u32(uint32_t* p, uint32_t v, cudaStream_t s) {
    k_set_u32<<<1, 1, 0, s>>>(p, v);
    return cudaGetLastError();
}

// ------------------------------------------- offsets from sorted rows ---
// Without a row histogram: after the last radix pass the rows are sorted, so
// offsets[key[g]] = g wherever the key changes (offsets pre-filled with
// 0xFFFFFFFF, offsets[n] = m), then a suffix-min scan gives every empty row
// the start of the next non-empty one.
__global__ void k_row_starts(const uint32_t* __restrict__ keys, uint64_t m, uint32_t n, uint32_t* offsets) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t quads = m >> 2;
    const bool vec = (reinterpret_cast<uintptr_t>(keys) & 15) == 0;
    const uint64_t vq = vec ? quads : 0;
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < vq; q += stride) {
        const uint4 k = __ldg(reinterpret_cast<const uint4*>(keys) + q);
        const uint64_t g = 4 * q;
        const uint32_t p = g ? __ldg(keys + g - 1) : ~k.x;
        if (p != k.x) offsets[k.x] = (uint32_t)g;
        if (k.x != k.y) offsets[k.y] = (uint32_t)(g + 1);
        if (k.y != k.z) offsets[k.z] = (uint32_t)(g + 2);
        if (k.z != k.w) offsets[k.w] = (uint32_t)(g + 3);
    }
    for (uint64_t g = 4 * vq + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < m; g += stride) {
        const uint32_t k = __ldg(keys + g);
        if (g == 0 || __ldg(keys + g - 1) != k) offsets[k] = (uint32_t)g;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) offsets[n] = (uint32_t)m;
}

#ifndef SCAN_IPT
#define SCAN_IPT 64
#endif
#ifndef SMIN_IPT
#define SMIN_IPT SCAN_IPT
#endif
constexpr int kSmNT = 256, kSmIPT = SMIN_IPT, kSmTile = kSmNT * kSmIPT;

// In-place suffix minimum over data[0..count).  Tiles are aligned to
// multiples of kSmTile from the bottom and taken from the top (tile k of T
// covers [(T-1-k) kSmTile, ...)), so every thread's 16 elements are one
// 64-byte aligned run read and written with 16-byte accesses; thread 0 owns
// the topmost run.
__global__ void __launch_bounds__(kSmNT) k_suffix_min(uint32_t* data, uint64_t count, unsigned long long* status,
                                                      unsigned* tile_counter) {
    __shared__ unsigned s_tile;
    __shared__ uint32_t s_w[kSmNT / 32];
    __shared__ unsigned long long s_carry;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t T = ceil_div(count, kSmTile);
    const uint64_t r0 = (T - 1 - tile) * kSmTile + (uint64_t)(kSmNT - 1 - threadIdx.x) * kSmIPT;  // run start
    const bool vec = r0 + kSmIPT <= count && (reinterpret_cast<uintptr_t>(data) & 15) == 0;
    uint32_t v[kSmIPT];
    if (vec) {
#pragma unroll
        for (int q = 0; q < kSmIPT / 4; q++) {
            const uint4 x = reinterpret_cast<const uint4*>(data + r0)[q];
            v[4 * q] = x.x, v[4 * q + 1] = x.y, v[4 * q + 2] = x.z, v[4 * q + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kSmIPT; k++) v[k] = r0 + k < count ? data[r0 + k] : 0xFFFFFFFFu;
    }
    uint32_t run = 0xFFFFFFFFu;
#pragma unroll
    for (int k = 0; k < kSmIPT; k++) run = v[k] < run ? v[k] : run;
    // exclusive suffix-min across threads (thread 0 is the top of the tile)
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    uint32_t inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t u = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= (unsigned)o) inc = u < inc ? u : inc;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t wv = lane < kSmNT / 32 ? s_w[lane] : 0xFFFFFFFFu;
        uint32_t wi = wv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t u = __shfl_up_sync(0xFFFFFFFFu, wi, o);
            if (lane >= (unsigned)o) wi = u < wi ? u : wi;
        }
        const uint32_t total = __shfl_sync(0xFFFFFFFFu, wi, kSmNT / 32 - 1);
        const uint32_t wex = __shfl_up_sync(0xFFFFFFFFu, wi, 1);
        if (lane < kSmNT / 32) s_w[lane] = lane == 0 ? 0xFFFFFFFFu : wex;
        if (lane == 0)
            st_volatile_u64(status + tile, (tile == 0 ? kFlagInc : kFlagAgg) | (unsigned long long)total);
        unsigned long long c = tile == 0 ? kValMask : warp_lookback_min(status, (long long)tile);
        if (lane == 0) {
            const unsigned long long t64 = total;
            if (tile != 0) st_volatile_u64(status + tile, kFlagInc | (c < t64 ? c : t64));
            s_carry = c;
        }
    }
    __syncthreads();
    uint32_t ex = __shfl_up_sync(0xFFFFFFFFu, inc, 1);
    if (lane == 0) ex = 0xFFFFFFFFu;
    ex = s_w[warp] < ex ? s_w[warp] : ex;
    const unsigned long long c = s_carry;
    uint32_t acc = c < (unsigned long long)ex ? (uint32_t)c : ex;
#pragma unroll
    for (int k = kSmIPT - 1; k >= 0; k--) {  // top of the run first
        acc = v[k] < acc ? v[k] : acc;
        v[k] = acc;
    }
    if (vec) {
#pragma unroll
        for (int q = 0; q < kSmIPT / 4; q++)
            reinterpret_cast<uint4*>(data + r0)[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < kSmIPT; k++)
            if (r0 + k < count) data[r0 + k] = v[k];
    }
}

}  // namespace boba

#include "radix.cuh"

namespace boba {

__global__ void k_gather_payload(const uint32_t* __restrict__ eidx, uint64_t m, const uint32_t* __restrict__ J2,
                                 const double* __restrict__ w, uint32_t* indices, double* w_out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += stride) {
        uint32_t e = __ldg(eidx + k);
        indices[k] = __ldg(J2 + e);
        if (w) w_out[k] = __ldg(w + e);
    }
}

// ----------------------------------------------------------------- host ---
namespace {
// Radix passes: 8-bit digits (7- and <=6-bit passes use narrower
// instantiations), 256 threads x 16 items = 4096-item tiles, 4 CTAs/SM.
// Measured slower and removed: 11-bit digits (the tiles x 2048 histogram
// outgrows the scan), 512x8 / 512x16 / 256x8 tiles, a persistent TMA
// double-buffered downsweep, a onesweep (decoupled lookback) variant.
constexpr int kRadixBits = 8;
constexpr uint64_t kRadixTile = RadixCfg<8, 256, 16>::TILE;

struct CsrPlan {
    int passes = 0;
    int shift[4] = {0, 0, 0, 0};
    int bits[4] = {0, 0, 0, 0};
    uint64_t tile = 0;
};

int key_bits(uint32_t n) { return n <= 1 ? 0 : 32 - __builtin_clz(n - 1); }

CsrPlan plan_bits(int kbits) {
    CsrPlan p;
    if (kbits <= 0) return p;
    p.passes = (kbits + kRadixBits - 1) / kRadixBits;
    int sh = 0;
    for (int i = 0; i < p.passes; i++) {
        const int b = kbits / p.passes + (i < kbits % p.passes ? 1 : 0);
        p.shift[i] = sh;
        p.bits[i] = b;
        sh += b;
    }
    p.tile = kRadixTile;
    return p;
}

CsrPlan plan_for(uint32_t n) { return plan_bits(key_bits(n)); }

struct CsrWs {
    uint32_t* counts;
    uint32_t* bufs[4];
    uint32_t* H;
    unsigned long long* scan_status;
    unsigned long long* off_status;
    unsigned* counters;
    size_t total;
};

CsrWs carve(void* base, uint64_t m, uint32_t n) {
    const CsrPlan p = plan_for(n);
    CsrWs w{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return base ? static_cast<char*>(base) + o : nullptr;
    };
    w.counts = (uint32_t*)take((size_t)n * 4 + 4);
    for (int i = 0; i < 4; i++) w.bufs[i] = (uint32_t*)take(m * 4 + 16);
    const uint64_t tiles = p.passes ? ceil_div(m, p.tile) : 1;
    int maxnb = 1;
    for (int i = 0; i < p.passes; i++) maxnb = std::max(maxnb, 1 << p.bits[i]);
    const uint64_t hcount = tiles * (uint64_t)maxnb;
    w.H = (uint32_t*)take(hcount * 4 + 16);
    w.scan_status = (unsigned long long*)take((ceil_div(hcount, kScanTile) + 1) * 8);
    w.off_status = (unsigned long long*)take((ceil_div((uint64_t)n + 1, kOffTile) + ceil_div((uint64_t)n + 1, kSmTile) + 2) * 8);
    w.counters = (unsigned*)take(64);
    w.total = off;
    return w;
}

template <int RB, int NT, int IPT, int MINB, typename Op = DigitShift>
cudaError_t radix_pass_op(const uint32_t* kin, const uint32_t* vin, uint64_t m, Op op, int bits, uint32_t* H,
                          unsigned long long* scan_status, unsigned* counter, uint32_t* kout, uint32_t* vout,
                          int num_sms, cudaStream_t s, uint32_t* row_starts = nullptr, bool h_ready = false,
                          bool zero_by_kernel = false) {
    using C = RadixCfg<RB, NT, IPT>;
    static PerDeviceOnce attr;
    if (cudaError_t e = set_attr_once(attr, k_radix_downsweep<RB, NT, IPT, MINB, Op>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM))
        return e;
    const uint64_t tiles = ceil_div(m, C::TILE);
    const uint64_t hcount = tiles << bits;
    const uint64_t up_grid = tiles < (uint64_t)num_sms * 8 ? tiles : (uint64_t)num_sms * 8;
    if (!h_ready) k_radix_upsweep<RB, NT, IPT, Op><<<(unsigned)up_grid, NT, 0, s>>>(kin, m, op, bits, tiles, H);
    cudaError_t e = cudaSuccess;
    if (zero_by_kernel) {   // inside a conditional graph body: kernel nodes only
        k_zero_u32<<<1, 256, 0, s>>>(reinterpret_cast<uint32_t*>(scan_status), (ceil_div(hcount, kScanTile) + 1) * 2,
                                     counter);
    } else {
        e = cudaMemsetAsync(scan_status, 0, (ceil_div(hcount, kScanTile) + 1) * 8, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(counter, 0, 4, s);
    }
    if (e != cudaSuccess) return e;
    k_scan_u32<<<(unsigned)ceil_div(hcount, kScanTile), kScanTileNT, 0, s>>>(H, hcount, 0u, scan_status, counter);
    k_radix_downsweep<RB, NT, IPT, MINB, Op><<<(unsigned)tiles, NT, C::SMEM, s>>>(kin, vin, m, op, bits, tiles, H,
                                                                                kout, vout, row_starts,
                                                                                (uint32_t)(MINB * num_sms));
    return cudaGetLastError();
}

// RB is the widest digit the pass supports; the ranking spends one ballot per
// bit of RB, so narrower passes (7 or <= 6 bits) use a narrower instantiation.
template <int RB, int NT, int IPT, int MINB>
cudaError_t radix_pass(const uint32_t* kin, const uint32_t* vin, uint64_t m, int shift, int bits, uint32_t* H,
                       unsigned long long* scan_status, unsigned* counter, uint32_t* kout, uint32_t* vout,
                       int num_sms, cudaStream_t s, uint32_t* row_starts, bool h_ready = false,
                       bool zero_by_kernel = false) {
    const DigitShift op{shift, (1u << bits) - 1u};
    if (RB == 8 && bits <= 6)
        return radix_pass_op<6, NT, IPT, MINB, DigitShift>(kin, vin, m, op, bits, H, scan_status, counter, kout, vout,
                                                           num_sms, s, row_starts, h_ready, zero_by_kernel);
    if (RB == 8 && bits == 7)
        return radix_pass_op<7, NT, IPT, MINB, DigitShift>(kin, vin, m, op, bits, H, scan_status, counter, kout, vout,
                                                           num_sms, s, row_starts, h_ready, zero_by_kernel);
    return radix_pass_op<RB, NT, IPT, MINB, DigitShift>(kin, vin, m, op, bits, H, scan_status, counter, kout, vout,
                                                        num_sms, s, row_starts, h_ready, zero_by_kernel);
}

// Kernels captured into the IF body of the last conditional node built on this
// thread (both bodies launch the same number): the captured graph's kernel
// count, which cannot be read back from a conditional node.
thread_local uint64_t t_cond_body_kernels = 0;

// Conditional-graph plan choice: 1 = every row is below 2^(kbits-1), the
// plan with a key bit less is exact (body 0), else the full-width plan.
__global__ void k_plan_cond(const uint32_t* __restrict__ rows_bound, uint32_t half, cudaGraphConditionalHandle h) {
    cudaGraphSetConditional(h, *rows_bound <= half ? 1u : 0u);
}

}  // namespace

size_t coo_to_csr_workspace_bytes(uint64_t m, uint32_t n, bool /*weighted*/) { return carve(nullptr, m, n).total; }

uint64_t take_conditional_body_kernels() {
    const uint64_t k = t_cond_body_kernels;
    t_cond_body_kernels = 0;
    return k;
}

// The first radix pass's tile histogram alone (its upsweep), into the
// workspace launch_coo_to_csr(..., first_hist_ready = true) reads it from: a
// caller can run it as soon as the row keys exist, e.g. while the columns are
// still arriving over the network (sharded.py, nccl_shard.cu).
cudaError_t launch_coo_to_csr_first_hist(const uint32_t* I2, uint64_t m, uint32_t n, void* ws, size_t ws_bytes,
                                         int num_sms, cudaStream_t s) {
    const CsrPlan p = plan_for(n);
    const CsrWs W = carve(ws, m, n);
    if (ws_bytes < W.total) return cudaErrorInvalidValue;
    if (p.passes == 0 || m == 0) return cudaSuccess;
    const uint64_t tiles = ceil_div(m, p.tile);
    const uint64_t up_grid = tiles < (uint64_t)num_sms * 8 ? tiles : (uint64_t)num_sms * 8;
    const DigitShift op{p.shift[0], (1u << p.bits[0]) - 1u};
    k_radix_upsweep<8, 256, 16, DigitShift><<<(unsigned)up_grid, 256, 0, s>>>(I2, m, op, p.bits[0], tiles, W.H);
    return cudaGetLastError();
}

RowTileHist coo_to_csr_first_hist(void* ws, size_t ws_bytes, uint64_t m, uint32_t n, bool /*weighted*/) {
    RowTileHist r;
    const CsrPlan p = plan_for(n);
    const CsrWs W = carve(ws, m, n);
    if (!ws || ws_bytes < W.total || p.passes == 0 || m == 0 || p.tile != 4096) return r;
    r.H = W.H;
    r.tiles = ceil_div(m, p.tile);
    r.mask = (1u << p.bits[0]) - 1u;
    return r;
}


__global__ void k_iota(uint32_t* out, uint64_t count) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) out[i] = (uint32_t)i;
}

cudaError_t launch_iota(uint32_t* out, uint64_t count, int num_sms, cudaStream_t s) {
    const uint64_t blocks = ceil_div(count, 256), cap = (uint64_t)num_sms * 8;
    k_iota<<<(int)(blocks < cap ? blocks : cap), 256, 0, s>>>(out, count);
    return cudaGetLastError();
}

// ------------------------------------------------ generic stable sort ---
// Stable LSD sort of (key, payload) pairs on the low key_bits of the key, 8-bit
// digits (the radix passes of COO->CSR).  vals == NULL: payload = input index.
// Used by the degree ordering (key = ~degree) and by sort_coo_by_destination.
namespace {
struct SortWs {
    uint32_t* bufs[4];
    uint32_t* H;
    unsigned long long* st;
    unsigned* counter;
    size_t total;
};
SortWs carve_sort(void* base, uint64_t count, int key_bits) {
    SortWs w{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return base ? static_cast<char*>(base) + o : nullptr;
    };
    for (int i = 0; i < 4; i++) w.bufs[i] = (uint32_t*)take(count * 4 + 16);
    const uint64_t tiles = ceil_div(count ? count : 1, RadixCfg<8, 256, 16>::TILE);
    const uint64_t hcount = tiles * 256;
    w.H = (uint32_t*)take(hcount * 4 + 16);
    w.st = (unsigned long long*)take((ceil_div(hcount, kScanTile) + 1) * 8);
    w.counter = (unsigned*)take(64);
    w.total = off;
    (void)key_bits;
    return w;
}
}  // namespace

size_t sort_pairs_workspace_bytes(uint64_t count, int key_bits) { return carve_sort(nullptr, count, key_bits).total; }

cudaError_t launch_sort_pairs(const uint32_t* keys, const uint32_t* vals, uint64_t count, int key_bits,
                              uint32_t* keys_out, uint32_t* vals_out, void* ws, size_t ws_bytes, int num_sms,
                              cudaStream_t s) {
    SortWs W = carve_sort(ws, count, key_bits);
    if (ws_bytes < W.total || key_bits < 0 || key_bits > 32) return cudaErrorInvalidValue;
    if (count == 0) return cudaSuccess;
    const int passes = (key_bits + 7) / 8;
    if (passes == 0) {
        cudaError_t e = cudaSuccess;
        if (keys_out) e = cudaMemcpyAsync(keys_out, keys, count * 4, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return e;
        if (vals) return cudaMemcpyAsync(vals_out, vals, count * 4, cudaMemcpyDeviceToDevice, s);
        return launch_iota(vals_out, count, num_sms, s);
    }
    const uint32_t* kin = keys;
    const uint32_t* vin = vals;
    int sh = 0;
    for (int i = 0; i < passes; i++) {
        const int bits = key_bits / passes + (i < key_bits % passes ? 1 : 0);
        const bool last = i == passes - 1;
        uint32_t* kout = last ? keys_out : W.bufs[(i & 1) * 2];
        uint32_t* vout = last ? vals_out : W.bufs[(i & 1) * 2 + 1];
        cudaError_t e = radix_pass<8, 256, 16, RADIX_MINB>(kin, vin, count, sh, bits, W.H, W.st, W.counter, kout, vout,
                                                  num_sms, s, nullptr);
        if (e != cudaSuccess) return e;
        kin = kout;
        vin = vout;
        sh += bits;
    }
    return cudaSuccess;
}

// ------------------------------------------------- row-range partition ---
// Stable partition of (key, payload) pairs by which of `parts` key ranges
// [bounds[p], bounds[p+1]) the key falls in -- the send side of the
// multi-GPU all-to-all by destination row range.  One radix pass whose digit
// is the range index; counts_out[p] = pairs in part p.
__global__ void k_part_counts(const uint32_t* __restrict__ H, uint64_t tiles, int parts, uint64_t m,
                              uint32_t* counts) {
    const int p = threadIdx.x;
    if (p >= parts) return;
    const uint32_t lo = H[(uint64_t)p * tiles];
    const uint32_t hi = p + 1 < parts ? H[(uint64_t)(p + 1) * tiles] : (uint32_t)m;
    counts[p] = hi - lo;
}

namespace {
int part_bits(int parts) { return parts <= 1 ? 1 : 32 - __builtin_clz((unsigned)parts - 1); }
}

size_t range_partition_workspace_bytes(uint64_t m, int parts) {
    const uint64_t tiles = ceil_div(m ? m : 1, RadixCfg<8, 256, 16>::TILE);
    const uint64_t hcount = tiles << part_bits(parts);
    return ((hcount * 4 + 255) / 256 * 256) + (ceil_div(hcount, kScanTile) + 1) * 8 + 256;
}

cudaError_t launch_range_partition(const uint32_t* keys, const uint32_t* vals, uint64_t m, const uint32_t* bounds,
                                   int parts, uint32_t* keys_out, uint32_t* vals_out, uint32_t* counts_out, void* ws,
                                   size_t ws_bytes, int num_sms, cudaStream_t s, bool relative) {
    if (parts < 1 || parts > 256) return cudaErrorInvalidValue;
    if (ws_bytes < range_partition_workspace_bytes(m, parts)) return cudaErrorInvalidValue;
    if (m == 0) return counts_out ? cudaMemsetAsync(counts_out, 0, (size_t)parts * 4, s) : cudaSuccess;
    const int bits = part_bits(parts);
    const uint64_t tiles = ceil_div(m, RadixCfg<8, 256, 16>::TILE);
    const uint64_t hcount = tiles << bits;
    char* p = static_cast<char*>(ws);
    uint32_t* H = reinterpret_cast<uint32_t*>(p);
    unsigned long long* st = reinterpret_cast<unsigned long long*>(p + (hcount * 4 + 255) / 256 * 256);
    unsigned* counter = reinterpret_cast<unsigned*>(st + ceil_div(hcount, kScanTile) + 1);
    cudaError_t e = radix_pass_op<8, 256, 16, RADIX_MINB, DigitRange>(keys, vals, m, DigitRange{bounds, parts, relative}, bits, H, st,
                                                             counter, keys_out, vals_out, num_sms, s);
    if (e != cudaSuccess) return e;
    if (counts_out) k_part_counts<<<1, 256, 0, s>>>(H, tiles, parts, m, counts_out);
    return cudaGetLastError();
}

cudaError_t launch_row_offsets(const uint32_t* counts, uint32_t n, uint32_t* offsets, unsigned long long* status,
                               unsigned* counter, cudaStream_t s) {
    const uint64_t tiles = ceil_div((uint64_t)n + 1, kOffTile);
    cudaError_t e = cudaMemsetAsync(status, 0, tiles * 8, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(counter, 0, 4, s);
    if (e != cudaSuccess) return e;
    k_scan_offsets<<<(unsigned)tiles, kOffNT, 0, s>>>(counts, n, offsets, status, counter);
    return cudaGetLastError();
}

cudaError_t launch_hist(const uint32_t* I, uint64_t m, uint32_t n, uint32_t* counts, int num_sms, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)n * 4, s);
    if (e != cudaSuccess || m == 0) return e;
    const uint64_t blocks = ceil_div(m, 256), cap = (uint64_t)num_sms * 8;
    k_hist<<<(int)(blocks < cap ? blocks : cap), 256, 0, s>>>(I, m, counts);
    return cudaGetLastError();
}

cudaError_t launch_coo_to_csr(const uint32_t* I2, const uint32_t* J2, const double* w, uint64_t m, uint32_t n,
                              const uint32_t* counts_in, uint32_t* offsets, uint32_t* indices, double* w_out,
                              void* ws, size_t ws_bytes, int num_sms, cudaStream_t s, bool first_hist_ready,
                              const uint32_t* rows_bound) {
    const bool weighted = w != nullptr;
    CsrWs W = carve(ws, m, n);
    if (ws_bytes < W.total) return cudaErrorInvalidValue;
    cudaError_t e = cudaSuccess;
    if (counts_in) {
        // caller supplied the row histogram: offsets = exclusive scan of it
        e = launch_row_offsets(counts_in, n, offsets, W.off_status, W.counters + 1, s);
    } else if (m == 0) {
        e = cudaMemsetAsync(offsets, 0, ((size_t)n + 1) * 4, s);
    }
    if (e != cudaSuccess || m == 0) return e;
    const CsrPlan p = plan_for(n);
    if (p.passes == 0) {
        // n == 1: every edge is in row 0; the stable order is the edge order.
        if (!counts_in) {
            const uint32_t h[2] = {0u, (uint32_t)m};
            e = cudaMemcpyAsync(offsets, h, 8, cudaMemcpyHostToDevice, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // h lives on this stack frame
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(indices, J2, m * 4, cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess && weighted) e = cudaMemcpyAsync(w_out, w, m * 8, cudaMemcpyDeviceToDevice, s);
        return e;
    }
    const uint32_t* kin = I2;
    const uint32_t* vin = weighted ? nullptr : J2;
    if (!counts_in) {
        // offsets come from the last pass's sorted output (row starts + suffix-min)
        e = cudaMemsetAsync(offsets, 0xFF, (size_t)n * 4, s);
        if (e == cudaSuccess) e = launch_set_u32(offsets + n, (uint32_t)m, s);
        if (e != cudaSuccess) return e;
    }
    // Under CUDA-graph capture with a device-side row bound: after the first
    // pass, an IF/ELSE conditional node runs either the plan with a key bit
    // less (rows below 2^(kbits-1), decided on the device per replay) or the
    // full-width one; both share that first pass.  Elsewhere: the full plan.
    CsrPlan pa;
    bool cond = false;
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    if (rows_bound && !counts_in && p.passes >= 2 && cudaStreamIsCapturing(s, &cst) == cudaSuccess &&
        cst == cudaStreamCaptureStatusActive) {
        pa = plan_bits(key_bits(n) - 1);
        // the plans share their first pass when its digit is the same; else both
        // run whole inside the branches (not with a first histogram made for p)
        cond = pa.passes == p.passes && (pa.bits[0] == p.bits[0] || !first_hist_ready);
    }
    auto run_passes = [&](const CsrPlan& q, int from, int to, const uint32_t* k0, const uint32_t* v0,
                          cudaStream_t st, bool in_body) -> cudaError_t {
        const uint32_t* ki = k0;
        const uint32_t* vi = v0;
        for (int i = from; i < to; i++) {
            const bool last = i == q.passes - 1;
            // pass i writes bufs[2(i&1)], bufs[2(i&1)+1]; it reads the other parity.
            uint32_t* kout = last ? nullptr : W.bufs[(i & 1) * 2];
            uint32_t* vout = (last && !weighted) ? indices : W.bufs[(i & 1) * 2 + 1];
            cudaError_t r = radix_pass<8, 256, 16, RADIX_MINB>(ki, vi, m, q.shift[i], q.bits[i], W.H, W.scan_status,
                                                      W.counters, kout, vout, num_sms, st,
                                                      (last && !counts_in) ? offsets : nullptr,
                                                      i == 0 && first_hist_ready, in_body);
            if (r != cudaSuccess) return r;
            ki = kout;
            vi = vout;
        }
        kin = ki;
        vin = vi;
        return cudaSuccess;
    };
    if (!cond) {
        e = run_passes(p, 0, p.passes, kin, vin, s, false);
        if (e != cudaSuccess) return e;
    } else {
        const int from = pa.bits[0] == p.bits[0] ? 1 : 0;
        if (from) {
            e = run_passes(p, 0, 1, kin, vin, s, false);   // the shared first pass
            if (e != cudaSuccess) return e;
        }
        const uint32_t* k1 = from ? W.bufs[0] : kin;
        const uint32_t* v1 = from ? W.bufs[1] : vin;
        cudaGraph_t g = nullptr;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        cudaGraphConditionalHandle h;
        e = cudaStreamGetCaptureInfo(s, &cst, nullptr, &g, &deps, &nd);
        if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&h, g, 0, 0);
        if (e != cudaSuccess) return e;
        k_plan_cond<<<1, 1, 0, s>>>(rows_bound, 1u << (key_bits(n) - 1), h);
        e = cudaStreamGetCaptureInfo(s, &cst, nullptr, &g, &deps, &nd);
        if (e != cudaSuccess) return e;
        cudaGraphNodeParams cp{};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeIf;
        cp.conditional.size = 2;
        cudaGraphNode_t cn;
        e = cudaGraphAddNode(&cn, g, deps, nd, &cp);
        if (e == cudaSuccess) e = cudaStreamUpdateCaptureDependencies(s, &cn, 1, cudaStreamSetCaptureDependencies);
        if (e != cudaSuccess) return e;
        for (int body = 0; body < 2; body++) {
            cudaStream_t bs = nullptr;
            e = cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking);
            if (e != cudaSuccess) return e;
            e = cudaStreamBeginCaptureToGraph(bs, cp.conditional.phGraph_out[body], nullptr, nullptr, 0,
                                              cudaStreamCaptureModeRelaxed);
            const CsrPlan& q = body == 0 ? pa : p;
            if (body == 0) t_cond_body_kernels += 4ull * (q.passes - from);   // zero, upsweep, scan, downsweep
            cudaError_t e2 = e == cudaSuccess ? run_passes(q, from, q.passes, k1, v1, bs, true) : e;
            cudaGraph_t done = nullptr;
            if (e == cudaSuccess) e = cudaStreamEndCapture(bs, &done);
            cudaStreamDestroy(bs);
            if (e2 != cudaSuccess) return e2;
            if (e != cudaSuccess) return e;
        }
    }
    if (!counts_in) {
        const uint64_t sm_tiles = ceil_div((uint64_t)n + 1, kSmTile);
        unsigned long long* sm_status = W.off_status + ceil_div((uint64_t)n + 1, kOffTile) + 1;
        e = cudaMemsetAsync(sm_status, 0, sm_tiles * 8, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(W.counters + 2, 0, 4, s);
        if (e != cudaSuccess) return e;
        k_suffix_min<<<(unsigned)sm_tiles, kSmNT, 0, s>>>(offsets, (uint64_t)n + 1, sm_status, W.counters + 2);
    }
    if (weighted) {
        const uint64_t blocks = ceil_div(m, 256), cap = (uint64_t)num_sms * 8;
        k_gather_payload<<<(int)(blocks < cap ? blocks : cap), 256, 0, s>>>(vin, m, J2, w, indices, w_out);
    }
    return cudaGetLastError();
}

}  // namespace boba
