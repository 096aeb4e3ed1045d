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
//             ceil(bits(n-1)/11) passes.  Each pass is one "onesweep" kernel:
//             a tile of 4-8K pairs is ranked per digit inside the CTA with
//             warp match_any multisplit (stable: warp-striped order), the
//             per-digit tile counts are published at once and the global
//             per-digit offsets resolved by decoupled lookback, then the tile
//             is re-sorted in shared memory and written out as contiguous
//             per-digit runs.  Global digit bases come straight from the CSR
//             offsets (no extra histogram pass over the edges).  Payload =
//             J2 (unweighted: the last pass writes `indices` directly) or the
//             edge index (weighted: a final gather moves J2 and the 64-bit
//             weights bit-exactly).
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

// --------------------------------------------- digit bases from offsets ---
// hist_p[d] = sum over rows r with ((r >> shift) & mask) == d of counts[r]
//           = sum_h off(((h << bits) | d) + 1) << shift) - off(((h << bits) | d) << shift)
__global__ void k_digit_hist(const uint32_t* __restrict__ offsets, uint32_t n, int shift, int bits,
                             uint32_t* hist) {
    __shared__ uint32_t s_red[32];
    const uint32_t d = blockIdx.x;
    const uint64_t span = 1ull << shift;
    const uint64_t H = ceil_div((uint64_t)n, span << bits);
    uint32_t acc = 0;
    for (uint64_t h = threadIdx.x; h < H; h += blockDim.x) {
        uint64_t lo = (((h << bits) | d) << shift), hi = lo + span;
        lo = lo < n ? lo : n;
        hi = hi < n ? hi : n;
        acc += __ldg(offsets + hi) - __ldg(offsets + lo);
    }
    acc = warp_sum(acc);
    if (lane_id() == 0) s_red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t v = threadIdx.x < blockDim.x / 32 ? s_red[threadIdx.x] : 0u;
        v = warp_sum(v);
        if (threadIdx.x == 0) hist[d] = v;
    }
}

__global__ void __launch_bounds__(1024) k_digit_base(uint32_t* hist, int nb) {
    // in-place exclusive scan of nb <= 4096 bins with one block of 1024
    __shared__ uint32_t s_scan[33];
    __shared__ uint32_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int c0 = 0; c0 < nb; c0 += 1024) {
        int i = c0 + threadIdx.x;
        uint32_t v = i < nb ? hist[i] : 0u;
        uint32_t tot;
        uint32_t ex = block_exclusive_sum<1024>(v, s_scan, &tot);
        if (i < nb) hist[i] = s_carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += tot;
        __syncthreads();
    }
}

// ------------------------------------------------------- onesweep pass ---
template <int BPT>
__device__ __forceinline__ void multi_lookback(const unsigned long long* status, long long tile, int nb,
                                               const int* d, unsigned long long* excl) {
    long long t[BPT];
    bool done[BPT];
#pragma unroll
    for (int b = 0; b < BPT; b++) {
        t[b] = tile - 1;
        excl[b] = 0;
        done[b] = d[b] < 0 || tile == 0;
    }
    while (true) {
        bool all = true;
#pragma unroll
        for (int b = 0; b < BPT; b++) all &= done[b];
        if (all) break;
        unsigned long long s0[BPT], s1[BPT];
#pragma unroll
        for (int b = 0; b < BPT; b++) {
            if (done[b]) continue;
            s0[b] = ld_volatile_u64(status + (uint64_t)t[b] * nb + d[b]);
            s1[b] = t[b] >= 1 ? ld_volatile_u64(status + (uint64_t)(t[b] - 1) * nb + d[b]) : kFlagInc;
        }
#pragma unroll
        for (int b = 0; b < BPT; b++) {
            if (done[b]) continue;
            unsigned f0 = (unsigned)(s0[b] >> 62);
            if (f0 == 0) continue;
            excl[b] += s0[b] & kValMask;
            if (f0 == 2) { done[b] = true; continue; }
            unsigned f1 = (unsigned)(s1[b] >> 62);
            if (f1 == 0) { t[b] -= 1; continue; }
            excl[b] += s1[b] & kValMask;
            if (f1 == 2) { done[b] = true; continue; }
            t[b] -= 2;
            if (t[b] < 0) done[b] = true;
        }
    }
}

template <int RB, int NT, int IPT>
struct Onesweep {
    static constexpr int B = 1 << RB;
    static constexpr int NW = NT / 32;
    static constexpr int TILE = NT * IPT;
    static constexpr int BPT = B >= NT ? B / NT : 1;
    static constexpr int REGION = (NW * B > 2 * TILE) ? NW * B : 2 * TILE;
    static constexpr size_t SMEM = sizeof(uint32_t) * (size_t)(REGION + 3 * B);
};

template <int RB, int NT, int IPT>
__global__ void __launch_bounds__(NT) k_onesweep(const uint32_t* __restrict__ keys_in,
                                                 const uint32_t* __restrict__ vals_in, uint64_t m, int shift,
                                                 int bits, const uint32_t* __restrict__ base,
                                                 unsigned long long* status, unsigned* tile_counter,
                                                 uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out) {
    using C = Onesweep<RB, NT, IPT>;
    constexpr int B = C::B, NW = C::NW, TILE = C::TILE, BPT = C::BPT;
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t* s_hist = smem;                 // NW x B warp counters (ranking)
    uint32_t* s_stage = smem;                // 2 x TILE staging (aliases s_hist later)
    uint32_t* s_cnt = smem + C::REGION;      // B tile counts
    uint32_t* s_off = s_cnt + B;             // B tile-local exclusive offsets
    uint32_t* s_glob = s_off + B;            // B: global position of the bucket's first tile item - s_off
    __shared__ unsigned s_tile;
    __shared__ uint32_t s_scan[NW + 1];

    const int nb = 1 << bits;
    const uint32_t mask = (uint32_t)nb - 1u;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    for (int i = threadIdx.x; i < NW * B; i += NT) s_hist[i] = 0;
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t tile_base = tile * TILE;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;

    uint32_t key[IPT], val[IPT], rank[IPT];
    const uint64_t wbase = tile_base + (uint64_t)warp * 32 * IPT + lane;
#pragma unroll
    for (int i = 0; i < IPT; i++) {
        uint64_t idx = wbase + (uint64_t)i * 32;
        bool ok = idx < m;
        key[i] = ok ? __ldg(keys_in + idx) : 0u;
        val[i] = ok ? (vals_in ? __ldg(vals_in + idx) : (uint32_t)idx) : 0u;
    }
    // Stable warp multisplit: items are ranked in (i, lane) order == input order.
    uint32_t* wh = s_hist + warp * B;
#pragma unroll
    for (int i = 0; i < IPT; i++) {
        const bool ok = wbase + (uint64_t)i * 32 < m;
        const uint32_t d = ok ? (key[i] >> shift) & mask : 0xFFFFFFFFu;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
        uint32_t pre = 0;
        if (ok) pre = wh[d];
        __syncwarp();
        if (ok) {
            rank[i] = pre + __popc(peers & lanemask_lt());
            if ((peers & lanemask_lt()) == 0) wh[d] = pre + __popc(peers);
        }
        __syncwarp();
    }
    __syncthreads();
    // Per-bucket exclusive scan across warps and tile totals.
    for (int d = threadIdx.x; d < nb; d += NT) {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < NW; w++) {
            uint32_t c = s_hist[w * B + d];
            s_hist[w * B + d] = run;
            run += c;
        }
        s_cnt[d] = run;
        st_volatile_u64(status + tile * nb + d, (tile == 0 ? kFlagInc : kFlagAgg) | (unsigned long long)run);
    }
    __syncthreads();
    // Tile-local exclusive scan over buckets (thread t owns BPT consecutive buckets).
    {
        uint32_t c[BPT];
        uint32_t sum = 0;
#pragma unroll
        for (int b = 0; b < BPT; b++) {
            int d = threadIdx.x * BPT + b;
            c[b] = d < nb ? s_cnt[d] : 0u;
            sum += c[b];
        }
        uint32_t tot;
        uint32_t ex = block_exclusive_sum<NT>(sum, s_scan, &tot);
#pragma unroll
        for (int b = 0; b < BPT; b++) {
            int d = threadIdx.x * BPT + b;
            if (d < nb) s_off[d] = ex;
            ex += c[b];
        }
    }
    __syncthreads();  // s_off is read below by threads that do not own it
    // Decoupled lookback for the global offset of each bucket within this tile.
    {
        int d[BPT];
        unsigned long long excl[BPT];
#pragma unroll
        for (int b = 0; b < BPT; b++) {
            int dd = threadIdx.x + b * NT;
            d[b] = dd < nb ? dd : -1;
        }
        multi_lookback<BPT>(status, (long long)tile, nb, d, excl);
#pragma unroll
        for (int b = 0; b < BPT; b++) {
            if (d[b] < 0) continue;
            if (tile != 0)
                st_volatile_u64(status + tile * nb + d[b], kFlagInc | (excl[b] + s_cnt[d[b]]));
            s_glob[d[b]] = __ldg(base + d[b]) + (uint32_t)excl[b] - s_off[d[b]];
        }
    }
    __syncthreads();
    // Local sorted position of every item, then stage the tile in digit order.
    uint32_t* pos = rank;  // reuse the registers
#pragma unroll
    for (int i = 0; i < IPT; i++) {
        const bool ok = wbase + (uint64_t)i * 32 < m;
        if (ok) {
            const uint32_t d = (key[i] >> shift) & mask;
            pos[i] = s_off[d] + wh[d] + rank[i];
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IPT; i++) {
        const bool ok = wbase + (uint64_t)i * 32 < m;
        if (ok) {
            s_stage[pos[i]] = key[i];
            s_stage[TILE + pos[i]] = val[i];
        }
    }
    __syncthreads();
    const uint64_t rem = m - tile_base;
    const int items = rem < (uint64_t)TILE ? (int)rem : TILE;
    for (int j = threadIdx.x; j < items; j += NT) {
        const uint32_t k = s_stage[j];
        const uint32_t g = s_glob[(k >> shift) & mask] + (uint32_t)j;
        if (keys_out) keys_out[g] = k;
        vals_out[g] = s_stage[TILE + j];
    }
}

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
struct CsrPlan {
    int passes = 0;
    int shift[4] = {0, 0, 0, 0};
    int bits[4] = {0, 0, 0, 0};
    int rb = 8;  // kernel variant
    uint64_t tile = 0;
};

int max_digit_bits() {
    const char* e = getenv("BOBA_RADIX_MAX_BITS");
    int v = e ? atoi(e) : 11;
    return v == 8 ? 8 : 11;
}

CsrPlan plan_for(uint32_t n) {
    CsrPlan p;
    int kbits = n <= 1 ? 0 : 32 - __builtin_clz(n - 1);
    if (kbits == 0) return p;
    const int maxb = max_digit_bits();
    p.passes = (kbits + maxb - 1) / maxb;
    int sh = 0;
    int widest = 0;
    for (int i = 0; i < p.passes; i++) {
        int b = kbits / p.passes + (i < kbits % p.passes ? 1 : 0);
        p.shift[i] = sh;
        p.bits[i] = b;
        sh += b;
        widest = b > widest ? b : widest;
    }
    p.rb = widest <= 8 ? 8 : 11;
    p.tile = p.rb == 8 ? Onesweep<8, 256, 16>::TILE : Onesweep<11, 256, 32>::TILE;
    return p;
}

struct CsrWs {
    uint32_t* counts;
    uint32_t* bufs[4];
    unsigned long long* status;
    unsigned long long* off_status;
    uint32_t* hist;  // 4 x 4096
    unsigned* counters;
    size_t total;
};

CsrWs carve(void* base, uint64_t m, uint32_t n, bool weighted) {
    CsrPlan p = plan_for(n);
    CsrWs w{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return base ? static_cast<char*>(base) + o : nullptr;
    };
    w.counts = (uint32_t*)take((size_t)n * 4 + 4);
    for (int i = 0; i < 4; i++) w.bufs[i] = (uint32_t*)take(m * 4 + 16);
    uint64_t tiles = p.passes ? ceil_div(m, p.tile) : 1;
    int maxnb = 1;
    for (int i = 0; i < p.passes; i++) maxnb = std::max(maxnb, 1 << p.bits[i]);
    w.status = (unsigned long long*)take(tiles * maxnb * 8 + 8);
    w.off_status = (unsigned long long*)take((ceil_div((uint64_t)n + 1, kOffTile) + 1) * 8);
    w.hist = (uint32_t*)take(4 * 4096 * 4);
    w.counters = (unsigned*)take(64);
    w.total = off;
    (void)weighted;
    return w;
}
}  // namespace

size_t coo_to_csr_workspace_bytes(uint64_t m, uint32_t n, bool weighted) {
    return carve(nullptr, m, n, weighted).total;
}

template <int RB, int NT, int IPT>
static cudaError_t run_pass(const uint32_t* kin, const uint32_t* vin, uint64_t m, int shift, int bits,
                            const uint32_t* base, unsigned long long* status, unsigned* counter, uint32_t* kout,
                            uint32_t* vout, cudaStream_t s) {
    using C = Onesweep<RB, NT, IPT>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_onesweep<RB, NT, IPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)C::SMEM);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    uint64_t tiles = ceil_div(m, C::TILE);
    cudaError_t e = cudaMemsetAsync(status, 0, tiles * (1ull << bits) * 8, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(counter, 0, 4, s);
    if (e != cudaSuccess) return e;
    k_onesweep<RB, NT, IPT><<<(unsigned)tiles, NT, C::SMEM, s>>>(kin, vin, m, shift, bits, base, status, counter,
                                                                 kout, vout);
    return cudaGetLastError();
}

cudaError_t launch_row_offsets(const uint32_t* counts, uint32_t n, uint32_t* offsets,
                               unsigned long long* status, unsigned* counter, cudaStream_t s) {
    uint64_t tiles = ceil_div((uint64_t)n + 1, kOffTile);
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
    uint64_t blocks = ceil_div(m, 256), cap = (uint64_t)num_sms * 8;
    k_hist<<<(int)(blocks < cap ? blocks : cap), 256, 0, s>>>(I, m, counts);
    return cudaGetLastError();
}

cudaError_t launch_coo_to_csr(const uint32_t* I2, const uint32_t* J2, const double* w, uint64_t m, uint32_t n,
                              const uint32_t* counts_in, uint32_t* offsets, uint32_t* indices, double* w_out,
                              void* ws, size_t ws_bytes, int num_sms, cudaStream_t s) {
    const bool weighted = w != nullptr;
    CsrWs W = carve(ws, m, n, weighted);
    if (ws_bytes < W.total) return cudaErrorInvalidValue;
    cudaError_t e;
    const uint32_t* counts = counts_in;
    if (!counts) {
        e = launch_hist(I2, m, n, W.counts, num_sms, s);
        if (e != cudaSuccess) return e;
        counts = W.counts;
    }
    e = launch_row_offsets(counts, n, offsets, W.off_status, W.counters + 1, s);
    if (e != cudaSuccess || m == 0) return e;
    CsrPlan p = plan_for(n);
    if (p.passes == 0) {
        // n == 1: every edge is in row 0; the stable order is the edge order.
        if (weighted) {
            e = cudaMemcpyAsync(indices, J2, m * 4, cudaMemcpyDeviceToDevice, s);
            if (e == cudaSuccess) e = cudaMemcpyAsync(w_out, w, m * 8, cudaMemcpyDeviceToDevice, s);
        } else {
            e = cudaMemcpyAsync(indices, J2, m * 4, cudaMemcpyDeviceToDevice, s);
        }
        return e;
    }
    for (int i = 0; i < p.passes; i++)
        k_digit_hist<<<1u << p.bits[i], 256, 0, s>>>(offsets, n, p.shift[i], p.bits[i], W.hist + i * 4096);
    for (int i = 0; i < p.passes; i++) k_digit_base<<<1, 1024, 0, s>>>(W.hist + i * 4096, 1 << p.bits[i]);
    const uint32_t* kin = I2;
    const uint32_t* vin = weighted ? nullptr : J2;
    for (int i = 0; i < p.passes; i++) {
        const bool last = i == p.passes - 1;
        // pass i writes bufs[2(i&1)], bufs[2(i&1)+1]; it reads the other parity.
        uint32_t* kout = last ? nullptr : W.bufs[(i & 1) * 2];
        uint32_t* vout = (last && !weighted) ? indices : W.bufs[(i & 1) * 2 + 1];
        if (p.rb == 8)
            e = run_pass<8, 256, 16>(kin, vin, m, p.shift[i], p.bits[i], W.hist + i * 4096, W.status, W.counters,
                                     kout, vout, s);
        else
            e = run_pass<11, 256, 32>(kin, vin, m, p.shift[i], p.bits[i], W.hist + i * 4096, W.status, W.counters,
                                      kout, vout, s);
        if (e != cudaSuccess) return e;
        kin = kout;
        vin = vout;
    }
    if (weighted) {
        uint64_t blocks = ceil_div(m, 256), cap = (uint64_t)num_sms * 8;
        k_gather_payload<<<(int)(blocks < cap ? blocks : cap), 256, 0, s>>>(vin, m, J2, w, indices, w_out);
    }
    return cudaGetLastError();
}

}  // namespace boba
