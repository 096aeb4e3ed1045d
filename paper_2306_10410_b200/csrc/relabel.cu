// Phase 3 -- relabel the edge list through label[] (new id of every old id).
//
// Reference: pkg/src/boba/graph.py:280-289 apply_permutation:
// (label[I], label[J]) with edge order (and weights) unchanged.
//
// One streaming pass: 16-byte loads of I and J, 16-byte stores of I2 and J2.
// The per-endpoint cost is the random 4-byte gather label[v] (4n bytes,
// L2-resident up to n ~ 25M) -- bounded by the L2 request rate, not HBM.
// Two shared-memory structures cut those requests:
//  * hub label cache: BOBA puts the hubs first, so the vertices with the
//    smallest new labels are exactly the ones most endpoints hit.  Phase 2
//    builds HubLabels (hubs.cuh: 16K buckets x 3 tagged entries, labels <
//    49151); each CTA copies it into shared memory (192 KB) and serves hits
//    from there.
//  * row histogram (the np.bincount of graph.py:270 for the following
//    COO->CSR): rows < 8K -- again the hubs -- are counted in shared memory
//    and flushed once per CTA; other rows use RED.ADD in L2.
#include <cstdlib>

#include "common.cuh"
#include "hubs.cuh"
#include "kernels.cuh"

namespace boba {

constexpr int kRlNT = 1024;
constexpr int kHubHistRows = 8192;

// MODE: 0 relabel only; 1 + out-degree histogram of the new rows (counts, the
// np.bincount of graph.py:270).  (Also writing the first radix pass's tile
// histogram here was measured: the per-tile barrier it needs costs more in
// this latency-bound loop than the upsweep it saves.)
// STREAM (label[] beyond L2): the edge streams are loaded and stored
// evict-first and the label gathers marked evict-last, so the 17 GB of
// streaming traffic at s26 does not push the table's lines out of L2.
// Without the hub table (n > 2^23) the L1 is free to cache hot labels (c5:
// 2.25 -> 2.19 ms); with it, the 192 KB table leaves ~36 KB of L1 and caching
// there costs more than it hits (c2: 0.40 -> 0.43 ms), so the gathers skip L1.
__device__ __forceinline__ uint32_t ld_label(const uint32_t* p, bool stream, unsigned long long pol, bool l1 = false) {
    if (!stream) return l1 ? __ldg(p) : __ldcg(p);
    uint32_t v;
    asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

template <int MODE, bool HUBS, bool STREAM = false>
__global__ void __launch_bounds__(kRlNT, 1) k_relabel(const uint4* __restrict__ I, const uint4* __restrict__ J,
                                                      uint64_t quads, const uint32_t* __restrict__ label,
                                                      const unsigned long long* __restrict__ hubs, HubHash hh,
                                                      uint32_t n, uint4* __restrict__ I2, uint4* __restrict__ J2,
                                                      uint32_t* counts) {
    extern __shared__ uint32_t sm32[];
    uint32_t* s_tab = sm32;                                                       // kHubWays x kHubBuckets
    uint32_t* s_hist = sm32 + (HUBS ? kHubWays * kHubBuckets : 0);                // kHubHistRows
    if (HUBS) {
        const uint4* src = reinterpret_cast<const uint4*>(hubs);
        for (int i = threadIdx.x; i < kHubWays * kHubBuckets / 4; i += kRlNT)
            reinterpret_cast<uint4*>(s_tab)[i] = __ldg(src + i);
    }
    if (MODE == 1)
        for (int i = threadIdx.x; i < kHubHistRows; i += kRlNT) s_hist[i] = 0;
    __syncthreads();
    const uint32_t tmask = hh.tag_bits ? (1u << hh.tag_bits) - 1u : 0u;
    // hub table probe (smem); 0xFFFFFFFF on a miss
    auto probe = [&](uint32_t v) -> uint32_t {
        if (HUBS) {
            uint32_t b, tag;
            hh.split(v, b, tag);
#pragma unroll
            for (int w = 0; w < kHubWays; w++) {   // entries: label << tag_bits | tag, 0xFFFFFFFF = empty
                const uint32_t e = s_tab[w * kHubBuckets + b];
                if (e != 0xFFFFFFFFu && (e & tmask) == tag) return e >> hh.tag_bits;
            }
        }
        return 0xFFFFFFFFu;
    };
    unsigned long long pol = 0;
    if (STREAM) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    auto lookup = [&](uint32_t v) -> uint32_t {
        const uint32_t h = probe(v);
        return h != 0xFFFFFFFFu ? h : ld_label(label + v, STREAM, pol, !HUBS);
    };
    auto count = [&](uint32_t r) {
        if (r < (uint32_t)kHubHistRows)
            atomicAdd(s_hist + r, 1u);
        else
            atomicAdd(counts + r, 1u);
    };
    for (uint64_t t = blockIdx.x; t * kRlNT < quads; t += gridDim.x) {
        const uint64_t q = t * kRlNT + threadIdx.x;
        if (q < quads) {
            const uint4 a = STREAM ? __ldcs(I + q) : __ldg(I + q), b = STREAM ? __ldcs(J + q) : __ldg(J + q);
            uint4 ra, rb;
            ra.x = lookup(a.x); ra.y = lookup(a.y); ra.z = lookup(a.z); ra.w = lookup(a.w);
            rb.x = lookup(b.x); rb.y = lookup(b.y); rb.z = lookup(b.z); rb.w = lookup(b.w);
            if (STREAM) {
                __stcs(I2 + q, ra);
                __stcs(J2 + q, rb);
            } else {
                I2[q] = ra;
                J2[q] = rb;
            }
            if (MODE == 1) {
                count(ra.x); count(ra.y); count(ra.z); count(ra.w);
            }
        }
    }
    if (MODE == 1) {
        __syncthreads();
        for (int i = threadIdx.x; i < kHubHistRows && i < (int)n; i += kRlNT)
            if (s_hist[i]) atomicAdd(counts + i, s_hist[i]);
    }
}

// label[] beyond L2 (s26: 268 MB): gathers over the whole table miss L2 and cost
// a DRAM sector each.  Instead the id space is cut into ranges whose slice of
// label[] stays L2-resident, and the edge streams are passed once per range.
// Pass 0 reads I, J and writes label[v] for v in its range, v | kRlFlag for the
// rest; later passes rewrite I2, J2 in place, resolving the flagged ids in
// their range (n <= 2^31, so the flag bit is free).
constexpr uint32_t kRlFlag = 0x80000000u;

// HIST (last pass only, when every id is final): the CTA's iteration t covers
// edges [4096 t, 4096 t + 4096) -- exactly radix tile t of COO->CSR -- so it
// also counts the first radix digit of its I2 rows in shared memory and
// writes the tile's column of H; the COO->CSR skips its first upsweep.  Two
// alternating histograms: each is flushed and cleared while the next
// iteration counts into the other, one barrier per iteration.
constexpr int kRlHistMax = 256;
static_assert(kRlNT * 4 == 4096, "relabel iteration = radix tile");

template <bool FIRST, bool HIST>
__global__ void __launch_bounds__(kRlNT, 1) k_relabel_range(const uint4* __restrict__ I, const uint4* __restrict__ J,
                                                            uint64_t quads, const uint32_t* __restrict__ label,
                                                            uint32_t lo, uint32_t width, uint4* I2, uint4* J2,
                                                            RowTileHist rh) {
    // HIST: TPI tiles per iteration, so the barrier comes once per 16K edges
#ifndef RL_TPI
#define RL_TPI 1
#endif
    constexpr int TPI = HIST ? 4 : RL_TPI;
    __shared__ uint32_t s_h[2][TPI][HIST ? kRlHistMax : 1];
    if (HIST) {
        for (int i = threadIdx.x; i < 2 * TPI * kRlHistMax; i += kRlNT) (&s_h[0][0][0])[i] = 0;
        __syncthreads();
    }
    int par = 0;
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    auto fix = [&](uint32_t v) -> uint32_t {
        const uint32_t id = FIRST ? v : v ^ kRlFlag;
        if (!FIRST && !(v & kRlFlag)) return v;
        if (id - lo < width) return ld_label(label + id, true, pol);
        return id | kRlFlag;
    };
    for (uint64_t g = blockIdx.x; g * TPI * kRlNT < quads; g += gridDim.x) {
        uint4 a[TPI], b[TPI];
#pragma unroll
        for (int k = 0; k < TPI; k++) {
            const uint64_t q = (g * TPI + k) * kRlNT + threadIdx.x;
            if (q < quads) {
                a[k] = FIRST ? __ldcs(I + q) : __ldcs(I2 + q);
                b[k] = FIRST ? __ldcs(J + q) : __ldcs(J2 + q);
            }
        }
#pragma unroll
        for (int k = 0; k < TPI; k++) {
            const uint64_t q = (g * TPI + k) * kRlNT + threadIdx.x;
            if (q < quads) {
                uint4 ra, rb;
                ra.x = fix(a[k].x); ra.y = fix(a[k].y); ra.z = fix(a[k].z); ra.w = fix(a[k].w);
                rb.x = fix(b[k].x); rb.y = fix(b[k].y); rb.z = fix(b[k].z); rb.w = fix(b[k].w);
                __stcs(I2 + q, ra);
                __stcs(J2 + q, rb);
                if (HIST) {
                    uint32_t* h = s_h[par][k];
                    atomicAdd(h + (ra.x & rh.mask), 1u);
                    atomicAdd(h + (ra.y & rh.mask), 1u);
                    atomicAdd(h + (ra.z & rh.mask), 1u);
                    atomicAdd(h + (ra.w & rh.mask), 1u);
                }
            }
        }
        if (HIST) {
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < (uint32_t)TPI * (rh.mask + 1); i += kRlNT) {
                const uint32_t k = i / (rh.mask + 1), d = i % (rh.mask + 1);
                const uint64_t t = g * TPI + k;
                if (t < rh.tiles) rh.H[(uint64_t)d * rh.tiles + t] = s_h[par][k][d];
                s_h[par][k][d] = 0;
            }
            par ^= 1;
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

template <int MODE, bool HUBS, bool STREAM = false>
static void launch_vec(int grid, size_t smem, cudaStream_t s, const uint32_t* I, const uint32_t* J, uint64_t quads,
                       const uint32_t* label, const unsigned long long* hubs, uint32_t n, uint32_t* I2, uint32_t* J2,
                       uint32_t* counts) {
    static PerDeviceOnce attr;
    set_attr_once(attr, k_relabel<MODE, HUBS, STREAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_relabel<MODE, HUBS, STREAM><<<grid, kRlNT, smem, s>>>((const uint4*)I, (const uint4*)J, quads, label, hubs,
                                                    HubHash::make(n), n, (uint4*)I2, (uint4*)J2, counts);
}

cudaError_t launch_relabel(const uint32_t* I, const uint32_t* J, uint64_t m, const uint32_t* label,
                           const unsigned long long* hubs, uint32_t* I2, uint32_t* J2, uint32_t* counts, uint32_t n,
                           int num_sms, cudaStream_t s, RowTileHist* row_hist) {
    if (row_hist) row_hist->done = false;
    if (counts) {
        cudaError_t err = cudaMemsetAsync(counts, 0, (size_t)n * 4, s);
        if (err != cudaSuccess) return err;
    }
    if (m == 0) return cudaSuccess;
    const bool vec = ((reinterpret_cast<uintptr_t>(I) | reinterpret_cast<uintptr_t>(J) |
                       reinterpret_cast<uintptr_t>(I2) | reinterpret_cast<uintptr_t>(J2)) & 15) == 0;
    uint64_t done = 0;
    if (vec && m >= 4) {
        const uint64_t quads = m >> 2;
        uint64_t blocks = ceil_div(quads, kRlNT);
        const int grid = (int)(blocks < (uint64_t)num_sms ? blocks : (uint64_t)num_sms);
        if (hubs && HubHash::make(n).tag_bits > 16) hubs = nullptr;  // ids too wide for the packed table
        // The table pays off while label[] is L2-resident and the phase is bound by the
        // L2 request rate (measured: c2, n = 2^22, 0.57 -> 0.40 ms).  Beyond 2^23
        // vertices the gathers are DRAM-latency bound and the probe only delays them
        // (c5, n = 2^24: 2.26 ms without, 3.28 ms with).
        if (n > (1u << 23) || getenv("BOBA_NO_HUBS")) hubs = nullptr;
        const size_t smem = (hubs ? kHubTableBytes : 0) + 4 * (counts ? kHubHistRows : 0);
        if (counts) {
            if (hubs) launch_vec<1, true>(grid, smem, s, I, J, quads, label, hubs, n, I2, J2, counts);
            else launch_vec<1, false>(grid, smem, s, I, J, quads, label, hubs, n, I2, J2, counts);
        } else if (n > (1u << 24)) {
            // single pass, measured at s26: 22.6 -> 21.8 ms (with the hub table in shared memory
            // instead: 25.1 ms -- it leaves the L1, which holds the hot labels here, only ~36 KB)
            // range passes keep each slice of label[] <= 128 MiB (measured at s26:
            // 1 pass 21.9 ms, 2 passes 14.1, 3 passes 14.3, 4 passes 16.7)
            const char* e = getenv("BOBA_RL_PASSES");
            const uint32_t passes = e ? (uint32_t)atoi(e) : (uint32_t)ceil_div(n, 1u << 25);
            if (passes <= 1 || n > kRlFlag) {
                launch_vec<0, false, true>(grid, smem, s, I, J, quads, label, hubs, n, I2, J2, counts);
            } else {
                const uint32_t width = (uint32_t)ceil_div(n, passes);
                // the last pass also counts the first radix digit per tile (no scalar tail:
                // every edge is in a quad, so the tiles are complete)
                const bool hist = row_hist && row_hist->H && (m & 3) == 0 && row_hist->mask < kRlHistMax &&
                                  row_hist->tiles == ceil_div(m, 4096);
                const RowTileHist rh = hist ? *row_hist : RowTileHist{};
                for (uint32_t p = 0; p < passes; p++) {
                    const uint32_t lo = p * width;
                    const bool last = p + 1 == passes;
                    if (p == 0)
                        k_relabel_range<true, false><<<grid, kRlNT, 0, s>>>((const uint4*)I, (const uint4*)J, quads,
                                                                            label, lo, width, (uint4*)I2, (uint4*)J2,
                                                                            rh);
                    else if (last && hist)
                        k_relabel_range<false, true><<<grid, kRlNT, 0, s>>>((const uint4*)I2, (const uint4*)J2, quads,
                                                                            label, lo, width, (uint4*)I2, (uint4*)J2,
                                                                            rh);
                    else
                        k_relabel_range<false, false><<<grid, kRlNT, 0, s>>>((const uint4*)I2, (const uint4*)J2,
                                                                             quads, label, lo, width, (uint4*)I2,
                                                                             (uint4*)J2, rh);
                }
                if (hist) row_hist->done = true;
            }
        } else {
            if (hubs) launch_vec<0, true>(grid, smem, s, I, J, quads, label, hubs, n, I2, J2, counts);
            else launch_vec<0, false>(grid, smem, s, I, J, quads, label, hubs, n, I2, J2, counts);
        }
        done = quads * 4;
    }
    if (done < m) {
        uint64_t blocks = ceil_div(m - done, 256), cap = (uint64_t)num_sms * 8;
        int grid = (int)(blocks < cap ? blocks : cap);
        if (counts)
            k_relabel_scalar<true><<<grid, 256, 0, s>>>(I, J, done, m, label, I2, J2, counts);
        else
            k_relabel_scalar<false><<<grid, 256, 0, s>>>(I, J, done, m, label, I2, J2, counts);
    }
    return cudaGetLastError();
}

}  // namespace boba
