// Stable LSD radix pass of (key, payload) uint32 pairs for COO->CSR
// (csr.cu), in reduce-then-scan form -- no CTA ever waits on another:
//
//   k_radix_upsweep    per tile (TILE contiguous items) digit histogram in
//                      shared memory -> H[d * tiles + t] (digit-major);
//   k_scan_u32         exclusive scan of H in place (decoupled lookback over
//                      2K-entry tiles; H is ~nb*tiles words, a few MB);
//   k_radix_downsweep  re-reads the tile, ranks every item stably inside the
//                      CTA and scatters it to H[d * tiles + t] + local rank,
//                      staged through shared memory so each digit's run of
//                      the tile is written contiguously.
//
// Stable in-CTA ranking: items sit in warp-striped order (warp w owns a
// contiguous run, lane l holds items i*32 + l), so (warp, i, lane) order is
// input order.  For each 32-item slot the peers (same digit) are found with
// one ballot per digit bit; the lowest peer bumps the warp's 16-bit counter.
// A per-digit scan across warps then turns warp-local ranks into tile ranks.
#pragma once
#include "common.cuh"

// Independent counter chains per warp in the ranking (RADIX_SUB=2 lets two
// chains' shared-memory read-modify-writes overlap; measured, one chain and
// half the per-warp histograms is faster: c4 20.26 -> 19.74 ms, c5 5.02 ->
// 4.95, c3 1.267 -> 1.257, c2 equal; four chains slower).
#ifndef RADIX_SUB
#define RADIX_SUB 1
#endif
// resident downsweep CTAs per SM the register allocation is bounded for
#ifndef RADIX_MINB
#define RADIX_MINB 4
#endif

namespace boba {

// Digit extractors: the LSD passes use a shift/mask digit; the multi-GPU row
// partition uses the index of the row range a key falls in (bounds[1..parts)).
struct DigitShift {
    int shift;
    uint32_t mask;
    __device__ __forceinline__ uint32_t operator()(uint32_t k) const { return (k >> shift) & mask; }
    __device__ __forceinline__ uint32_t out_key(uint32_t k, uint32_t) const { return k; }
};
struct DigitRange {
    const uint32_t* bounds;  // parts + 1 ascending row boundaries (device)
    int parts;
    bool relative;           // keys written relative to their part's first row
    __device__ __forceinline__ uint32_t operator()(uint32_t k) const {
        uint32_t o = 0;
        for (int p = 1; p < parts; p++) o += k >= __ldg(bounds + p);
        return o;
    }
    __device__ __forceinline__ uint32_t out_key(uint32_t k, uint32_t d) const {
        return relative ? k - __ldg(bounds + d) : k;
    }
};

template <int RB, int NT, int IPT>
struct RadixCfg {
    static constexpr int B = 1 << RB;
    static constexpr int NW = NT / 32;
    static constexpr int TILE = NT * IPT;
    static constexpr int BPT = B >= NT ? B / NT : 1;              // digits per thread in the scans
    static constexpr int SUB = RADIX_SUB;                            // independent counter chains per warp
    static constexpr int VW = NW * SUB;                              // "virtual warps" (warp, chain)
    static constexpr int HIST_BYTES = (VW * B * 2 + 15) / 16 * 16;  // 16-bit counters per virtual warp
    static constexpr int STAGE_BYTES = TILE * 8;                    // staged (key, payload) pairs
    static constexpr int RAW_BYTES = TILE * 4;                      // payloads prefetched by cp.async
    static constexpr size_t SMEM = (size_t)HIST_BYTES + STAGE_BYTES + RAW_BYTES + 2 * B * 4;  // + s_off, s_glob
    static_assert(TILE < 65536, "16-bit counters and packed ranks");
    static_assert(B % NT == 0 || NT >= B, "digit ownership");
};

// ------------------------------------------------------------- upsweep ---
template <int RB, int NT, int IPT, typename Op>
__global__ void __launch_bounds__(NT) k_radix_upsweep(const uint32_t* __restrict__ keys, uint64_t m, Op op,
                                                      int bits, uint64_t tiles, uint32_t* __restrict__ H) {
    using C = RadixCfg<RB, NT, IPT>;
    __shared__ uint32_t s_h[C::B];
    const int nb = 1 << bits;
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        for (int d = threadIdx.x; d < nb; d += NT) s_h[d] = 0;
        __syncthreads();
        const uint64_t base = t * C::TILE;
        if (base + C::TILE <= m && (C::TILE % (4 * NT)) == 0) {
            const uint4* k4 = reinterpret_cast<const uint4*>(keys + base);
#pragma unroll
            for (int i = 0; i < C::TILE / (4 * NT); i++) {
                const uint4 q = __ldg(k4 + i * NT + threadIdx.x);
                atomicAdd(s_h + op(q.x), 1u);
                atomicAdd(s_h + op(q.y), 1u);
                atomicAdd(s_h + op(q.z), 1u);
                atomicAdd(s_h + op(q.w), 1u);
            }
        } else {
            for (uint64_t i = base + threadIdx.x; i < m && i < base + C::TILE; i += NT)
                atomicAdd(s_h + op(__ldg(keys + i)), 1u);
        }
        __syncthreads();
        for (int d = threadIdx.x; d < nb; d += NT) H[(uint64_t)d * tiles + t] = s_h[d];
        __syncthreads();
    }
}

// ------------------------------------------------- exclusive scan (u32) ---
// values per thread of the lookback scans (H scan, suffix-min): 16 -> 64
// measured c2 / c5 COO->CSR 1.085 / 4.524 -> 1.071 / 4.517 ms (fewer tiles
// on the lookback chain)
#ifndef SCAN_IPT
#define SCAN_IPT 64
#endif
constexpr int kScanTileNT = 256, kScanTileIPT = SCAN_IPT, kScanTile = kScanTileNT * kScanTileIPT;

// Each thread owns 16 consecutive words (four 16-byte accesses when the run is
// in bounds and data is 16-byte aligned).
__global__ void __launch_bounds__(kScanTileNT) k_scan_u32(uint32_t* data, uint64_t count, uint32_t add,
                                                          unsigned long long* status, unsigned* tile_counter) {
    __shared__ unsigned s_tile;
    __shared__ uint32_t s_scan[kScanTileNT / 32 + 1];
    __shared__ unsigned long long s_excl;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t i0 = tile * kScanTile + (uint64_t)threadIdx.x * kScanTileIPT;
    const bool vec = i0 + kScanTileIPT <= count && (reinterpret_cast<uintptr_t>(data) & 15) == 0;
    uint32_t c[kScanTileIPT];
    if (vec) {
#pragma unroll
        for (int q = 0; q < kScanTileIPT / 4; q++) {
            const uint4 x = reinterpret_cast<const uint4*>(data + i0)[q];
            c[4 * q] = x.x, c[4 * q + 1] = x.y, c[4 * q + 2] = x.z, c[4 * q + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kScanTileIPT; k++) c[k] = (i0 + k < count) ? data[i0 + k] : 0u;
    }
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kScanTileIPT; k++) sum += c[k];
    uint32_t total;
    uint32_t ex_t = block_exclusive_sum<kScanTileNT>(sum, s_scan, &total);
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
    uint32_t run = add + (uint32_t)s_excl + ex_t;
#pragma unroll
    for (int k = 0; k < kScanTileIPT; k++) {
        const uint32_t x = c[k];
        c[k] = run;
        run += x;
    }
    if (vec) {
#pragma unroll
        for (int q = 0; q < kScanTileIPT / 4; q++)
            reinterpret_cast<uint4*>(data + i0)[q] = make_uint4(c[4 * q], c[4 * q + 1], c[4 * q + 2], c[4 * q + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < kScanTileIPT; k++)
            if (i0 + k < count) data[i0 + k] = c[k];
    }
}

// ----------------------------------------------------------- downsweep ---
// Ranks the warp's IPT 32-item slots: peers (same digit) via one ballot per
// digit bit, the lowest peer bumps the warp's 16-bit counter.  FULL: every
// item of the tile is valid (all tiles but the last), no per-item checks.
template <int RB, int IPT, int SUB, bool FULL, typename Op>
__device__ __forceinline__ void rank_slots(const uint32_t (&key)[IPT], uint32_t (&rank)[IPT], uint16_t* wh,
                                           Op op, uint64_t wslot, uint64_t m) {
    constexpr int B = 1 << RB, SPC = IPT / SUB;
    const unsigned lane = lane_id(), lt = lanemask_lt();
    // SUB chains of consecutive slots, each with its own counters, advance
    // together so their shared-memory read-modify-write latencies overlap.
#pragma unroll
    for (int si = 0; si < SPC; si++) {
#pragma unroll
    for (int c = 0; c < SUB; c++) {
        const int i = c * SPC + si;
        uint16_t* ch = wh + c * B;
        const bool ok = FULL || wslot + (uint64_t)i * 32 + lane < m;
        const uint32_t d = op(key[i]);
        unsigned peers = FULL ? 0xFFFFFFFFu : __ballot_sync(0xFFFFFFFFu, ok);
        // peers &= lanes whose digit bit b equals mine, for every bit b:
        // one predicate test, one ballot and one predicated AND per bit.
#pragma unroll
        for (int b = 0; b < RB; b++) {  // bits >= `bits` are zero in every lane: no effect
            asm("{\n\t"
                ".reg .pred p;\n\t"
                ".reg .b32 bb;\n\t"
                "and.b32 bb, %1, %2;\n\t"
                "setp.ne.u32 p, bb, 0;\n\t"
                "vote.sync.ballot.b32 bb, p, 0xffffffff;\n\t"
                "@!p not.b32 bb, bb;\n\t"
                "and.b32 %0, %0, bb;\n\t"
                "}"
                : "+r"(peers)
                : "r"(d), "r"(1u << b));
        }
        const unsigned below = peers & lt;
        uint32_t pre = 0;
        // counter address = warp base + 2 d: one LEA (the compiler's form was
        // an add of the warp offset and a doubling add of the shared base;
        // c4 COO->CSR 18.20 -> 18.05 ms, c2 1.087 -> 1.083)
        const uint32_t ca = (uint32_t)__cvta_generic_to_shared(ch) + 2u * d;
        if (ok) {
            unsigned short v;
            asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(ca));
            pre = v;
        }
        __syncwarp();
        if (ok && below == 0)
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(ca), "h"((unsigned short)(pre + __popc(peers))));
        rank[i] = ok ? pre + __popc(below) : 0xFFFFFFFFu;
    }
        __syncwarp();
    }
}

// Staging slot of tile rank r.  Sorted or nearly sorted keys (a BOBA-ordered
// grid) give every digit the same count, so a warp's 32 ranks are spaced by a
// multiple of 16 entries -- 16 x 8 B = one full bank cycle -- and all land in
// one bank pair; XOR-ing the low 4 bits with the next 4 spreads them (a
// bijection on every aligned group of 256 slots).
#ifndef RADIX_NO_SWZ
__device__ __forceinline__ uint32_t kv_swz(uint32_t r) { return r ^ ((r >> 4) & 15u); }
#else
__device__ __forceinline__ uint32_t kv_swz(uint32_t r) { return r; }
#endif

template <int RB, int NT, int IPT, int MINB, typename Op>
__global__ void __launch_bounds__(NT, MINB) k_radix_downsweep(const uint32_t* __restrict__ keys_in,
                                                              const uint32_t* __restrict__ vals_in, uint64_t m,
                                                              Op op, int bits, uint64_t tiles,
                                                              const uint32_t* __restrict__ H,
                                                              uint32_t* __restrict__ keys_out,
                                                              uint32_t* __restrict__ vals_out,
                                                              uint32_t* __restrict__ row_starts,
                                                              uint32_t pf_tiles) {
    using C = RadixCfg<RB, NT, IPT>;
    constexpr int B = C::B, NW = C::NW, TILE = C::TILE, BPT = C::BPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint16_t* s_hist = reinterpret_cast<uint16_t*>(smem_raw);                  // NW x B warp counters
    uint2* s_kv = reinterpret_cast<uint2*>(smem_raw + C::HIST_BYTES);          // TILE staged (key, payload)
    uint32_t* s_raw = reinterpret_cast<uint32_t*>(s_kv + TILE);                // TILE payloads, input order
    uint32_t* s_off = s_raw + TILE;                                            // B: tile-local digit offsets
    uint32_t* s_glob = s_off + B;                                              // B: global position - s_off
    __shared__ uint32_t s_scan[NW + 1];

    const int nb = 1 << bits;
    const uint64_t tile = blockIdx.x;
    const uint64_t tile_base = tile * TILE;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const uint64_t wslot = tile_base + (uint64_t)warp * 32 * IPT;
    const bool full = tile_base + TILE <= m;

    // The pass is bound by load latency: pull the keys and payloads of the
    // tile a CTA of the next wave will take (pf_tiles = the resident CTAs of
    // the grid ahead) into L2 with TMA bulk prefetches -- no registers, no
    // shared memory -- so its loads start from L2.  Measured: c4 COO->CSR
    // 19.67 -> 19.19 ms, c2 1.138 -> 1.114 (2x further ahead: slower).
    if (pf_tiles && threadIdx.x == 0) {
        const uint64_t pt = tile + pf_tiles;
        if ((pt + 1) * TILE <= m) {
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(keys_in + pt * TILE), "r"(TILE * 4)
                         : "memory");
            if (vals_in)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(vals_in + pt * TILE), "r"(TILE * 4)
                             : "memory");
        }
    }

    // this tile's scanned digit offsets, read after the ranking: pulled into L1
    // now, so that read does not stall the CTA at the next barrier (no register
    // held; c4 / c5 / c2 COO->CSR 18.77 / 4.580 / 1.0905 -> 18.62 / 4.553 / 1.084 ms)
    if ((int)threadIdx.x < nb)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(H + (uint64_t)threadIdx.x * tiles + tile));
    for (int i = threadIdx.x; i < C::VW * B / 2; i += NT) reinterpret_cast<uint32_t*>(s_hist)[i] = 0;
    // Prefetch this warp's payload run (IPT*32 words) into shared memory with
    // cp.async; it lands while the warp ranks its keys.
    uint32_t* wraw = s_raw + warp * 32 * IPT;
    if (vals_in) {
        if (full && ((reinterpret_cast<uintptr_t>(vals_in + wslot) & 15) == 0)) {
#pragma unroll
            for (int c = lane; c < IPT * 8; c += 32) {
                const unsigned saddr = (unsigned)__cvta_generic_to_shared(wraw + 4 * c);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(vals_in + wslot + 4 * c)
                             : "memory");
            }
        } else {
            for (int c = lane; c < IPT * 32; c += 32) {
                const uint64_t idx = wslot + (uint64_t)c;
                if (idx < m) {
                    const unsigned saddr = (unsigned)__cvta_generic_to_shared(wraw + c);
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(saddr), "l"(vals_in + idx)
                                 : "memory");
                }
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    uint32_t key[IPT], rank[IPT];
    if (full) {
#pragma unroll
        for (int i = 0; i < IPT; i++) key[i] = __ldg(keys_in + wslot + i * 32 + lane);
    } else {
#pragma unroll
        for (int i = 0; i < IPT; i++) {
            const uint64_t idx = wslot + (uint64_t)i * 32 + lane;
            key[i] = idx < m ? __ldg(keys_in + idx) : 0u;
        }
    }
    __syncthreads();
    uint16_t* wh = s_hist + warp * C::SUB * B;
    if (full)
        rank_slots<RB, IPT, C::SUB, true>(key, rank, wh, op, wslot, m);
    else
        rank_slots<RB, IPT, C::SUB, false>(key, rank, wh, op, wslot, m);
    __syncthreads();
    // Per digit: tile offset (block scan of the digit totals), then every
    // warp's counter becomes tile offset + the digit's count in earlier warps,
    // so an item's tile rank is one shared load away.
    uint32_t cnt[BPT];
#pragma unroll
    for (int b = 0; b < BPT; b++) {
        const int d = threadIdx.x * BPT + b;
        uint32_t run = 0;
        if (d < nb) {
#pragma unroll
            for (int w = 0; w < C::VW; w++) run += s_hist[w * B + d];
        }
        cnt[b] = run;
    }
    {
        uint32_t sum = 0;
#pragma unroll
        for (int b = 0; b < BPT; b++) sum += cnt[b];
        uint32_t tot;
        uint32_t ex = block_exclusive_sum<NT>(sum, s_scan, &tot);
#pragma unroll
        for (int b = 0; b < BPT; b++) {
            const int d = threadIdx.x * BPT + b;
            if (d < nb) {
                s_off[d] = ex;
                s_glob[d] = __ldg(H + (uint64_t)d * tiles + tile) - ex;
                uint32_t run = ex;
#pragma unroll
                for (int w = 0; w < C::VW; w++) {
                    const uint32_t c = s_hist[w * B + d];
                    s_hist[w * B + d] = (uint16_t)run;
                    run += c;
                }
            }
            ex += cnt[b];
        }
    }
    __syncthreads();
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
    // shared addresses formed as base + scaled index (one LEA each; measured
    // c4 / c5 COO->CSR 18.25 / 4.540 -> 18.01 / 4.525 ms)
    const uint32_t wh_sa = (uint32_t)__cvta_generic_to_shared(wh);
    const uint32_t kv_sa = (uint32_t)__cvta_generic_to_shared(s_kv);
    auto stage = [&](int i) {
        unsigned short c;
        asm volatile("ld.shared.u16 %0, [%1];"
                     : "=h"(c)
                     : "r"(wh_sa + 2u * ((uint32_t)(i / (IPT / C::SUB)) * B + op(key[i]))));
        const uint32_t r = rank[i] + c;
        const uint32_t v = vals_in ? wraw[i * 32 + lane] : (uint32_t)(wslot + (uint64_t)i * 32 + lane);
        asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(kv_sa + 8u * kv_swz(r)), "r"(key[i]), "r"(v));
    };
    if (full) {
#pragma unroll
        for (int i = 0; i < IPT; i++) stage(i);
    } else {
#pragma unroll
        for (int i = 0; i < IPT; i++)
            if (rank[i] != 0xFFFFFFFFu) stage(i);
    }
    __syncthreads();
    auto emit = [&](int j) {
        const uint2 kv = s_kv[kv_swz(j)];
        const uint32_t d = op(kv.x);
        const uint32_t g = s_glob[d] + (uint32_t)j;
        if (keys_out) keys_out[g] = op.out_key(kv.x, d);
        vals_out[g] = kv.y;
        if (row_starts) {
            // Last (most significant) pass: the output is sorted by key, and this
            // tile's run for digit d is a contiguous segment of it.  A key change
            // inside the run is a first occurrence; the run's first item may
            // continue the previous run, so it only lowers the slot.  Slots start
            // at 0xFFFFFFFF; empty rows are filled by a suffix-min afterwards.
            if (j == (int)s_off[d])
                atomicMin(row_starts + kv.x, g);
            else if (s_kv[kv_swz(j - 1)].x != kv.x)
                row_starts[kv.x] = g;
        }
    };
    // full tiles: a fixed trip count, unrolled (no per-item bound or rank-valid checks)
    if (full) {
#pragma unroll
        for (int k = 0; k < IPT; k++) emit((int)threadIdx.x + k * NT);
    } else {
        const int items = (int)(m - tile_base);
        for (int j = threadIdx.x; j < items; j += NT) emit(j);
    }
}

}  // namespace boba
