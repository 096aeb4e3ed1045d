// Phase 1 -- first occurrence of every vertex in the flattened edge stream
// I||J (positions: I[e] -> e, J[e] -> m + e).
//
// Reference: pkg/src/boba/_parallel.py:139-162 first_hit_chunked (exact
// chunk-local minimum merged exactly) and :165-175 first_hit_racy (guarded
// unsynchronised writes).  Here the minimum is a device-wide atomicMin on
// uint32 (2m <= 2^32 - 2, UNSET = 0xFFFFFFFF).
//
// Cost model: the stream is read once (8m bytes, coalesced 16-byte loads);
// the per-endpoint work is a 4-byte random access to first[] (4n bytes,
// L2-resident up to n ~ 25M), and the L2 request rate for those -- not HBM
// bandwidth -- is what bounds a naive kernel.  What cuts it:
//  * the grid sweeps the stream in position order (persistent CTAs,
//    block-cyclic over 8K-position iterations), so an atomic is issued only
//    when a plain (L1-cacheable; stale values are conservative because
//    first[] only decreases) load shows the position can still lower first[v];
//  * two-stage sweep: stage 1 runs a prefix of I alone (128K positions for
//    ids up to 2^22, 64K beyond); the vertices first seen there -- exactly
//    the first BOBA vertices, i.e. the hubs -- go into a 128K- or 64K-entry
//    tag set (hubs.cuh SeenSet) that every CTA of stage 2 holds in shared
//    memory, and their later endpoints never leave the SM;
//  * when the prefix is too short to matter (small m) or the ids are too wide
//    for 16-bit tags, a single sweep keeps a per-CTA set of vertices already
//    finalised instead (insert-if-empty; CTA barrier per iteration keeps the
//    invariant first[v] < lowest position still to come).
#include "common.cuh"
#include "hubs.cuh"
#include "kernels.cuh"

#include <cstdlib>
#include <type_traits>

namespace boba {

constexpr int kFhNT = 1024;              // threads per CTA (one CTA per SM)
// 16-byte quads per thread per iteration (measured, static sweep, c4 / c5 /
// c3 / c2: 4 quads 7.24 / 1.656 / 0.830 / 0.323 ms, 2 quads 7.19 / 1.627 /
// 0.811 / 0.322, 1 quad 7.17 / 1.621 / 0.797 / 0.348, 8 quads 12.1 / 2.89)
constexpr int kFhQuads = 2;
constexpr int kFhSlotsLog2 = 15;         // 32K-slot finalised-vertex set (128 KB), dynamic mode
constexpr uint32_t kEmpty = 0xFFFFFFFFu;

// Two consecutive position ranges swept in order: A then B (quads of 4 ids).
struct Ranges {
    const uint32_t* a;
    uint64_t qa;      // quads in A
    uint32_t base_a;  // global position of a[0]
    const uint32_t* b;
    uint64_t qb;
    uint32_t base_b;
};

__device__ __forceinline__ uint32_t slot_of(uint32_t v) { return (v * 0x9E3779B1u) >> (32 - kFhSlotsLog2); }
__device__ __forceinline__ uint32_t hash_slot(uint32_t v) { return (v * 0x85EBCA6Bu) ^ (v >> 13); }

template <bool RELAXED>
__device__ __forceinline__ void update(uint32_t* first, uint32_t v, uint32_t pos, uint32_t cur) {
    if (RELAXED)
        *((volatile uint32_t*)(first + v)) = pos;
    else
        atomicMin(first + v, pos);
}

// Dynamic mode: per-CTA set of vertices known finalised.  Reads happen during
// an iteration, inserts between two barriers after it (one candidate per
// thread, by compare-and-swap into an empty slot), so the cache is never
// read and written concurrently; a vertex in the set is finalised, a missing
// one only costs the guarded global check.
template <bool RELAXED>
__device__ __forceinline__ void hit_dyn(uint32_t* first, const uint32_t* set, uint32_t v, uint32_t pos,
                                        uint32_t iter_lo, uint32_t& pending) {
    const uint32_t s = slot_of(v);
    if (set[s] == v) return;                       // finalised: first[v] < iter_lo <= pos
    const uint32_t cur = __ldcg(first + v);        // L2 load: may be stale (>= true value)
    if (pos < cur) {
        update<RELAXED>(first, v, pos, cur);
    } else if (cur < iter_lo && set[s] == kEmpty) {
        pending = v;                               // finalised; cached after the iteration
    }
}

// Dynamic-mode sweep over I||J in position order (block-cyclic 16K-position
// iterations, a CTA barrier per iteration keeps the set invariant).
template <bool RELAXED>
__global__ void __launch_bounds__(kFhNT, 1) k_first_hit(Ranges r, uint32_t* first) {
    extern __shared__ unsigned long long smem_u64[];
    uint32_t* set = reinterpret_cast<uint32_t*>(smem_u64);
    for (int i = threadIdx.x; i < (1 << kFhSlotsLog2); i += kFhNT) set[i] = kEmpty;
    const uint64_t total_q = r.qa + r.qb;
    const uint64_t iters = ceil_div(total_q, (uint64_t)kFhNT * kFhQuads);
    for (uint64_t it = blockIdx.x; it < iters; it += gridDim.x) {
        __syncthreads();  // every warp has left the previous iteration's inserts
        const uint64_t q0 = it * kFhNT * kFhQuads;
        const uint32_t iter_lo = (uint32_t)(q0 < r.qa ? r.base_a + 4 * q0 : r.base_b + 4 * (q0 - r.qa));
        uint4 q[kFhQuads];
        uint32_t pos[kFhQuads];
        bool ok[kFhQuads];
#pragma unroll
        for (int k = 0; k < kFhQuads; k++) {
            const uint64_t w = q0 + (uint64_t)k * kFhNT + threadIdx.x;
            ok[k] = w < total_q;
            if (ok[k]) {
                const bool inB = w >= r.qa;
                const uint64_t qi = inB ? w - r.qa : w;
                q[k] = __ldg(reinterpret_cast<const uint4*>(inB ? r.b : r.a) + qi);
                pos[k] = (uint32_t)(4 * qi) + (inB ? r.base_b : r.base_a);
            }
        }
        uint32_t pending = kEmpty;
#pragma unroll
        for (int k = 0; k < kFhQuads; k++) {
            if (!ok[k]) continue;
            hit_dyn<RELAXED>(first, set, q[k].x, pos[k], iter_lo, pending);
            hit_dyn<RELAXED>(first, set, q[k].y, pos[k] + 1, iter_lo, pending);
            hit_dyn<RELAXED>(first, set, q[k].z, pos[k] + 2, iter_lo, pending);
            hit_dyn<RELAXED>(first, set, q[k].w, pos[k] + 3, iter_lo, pending);
        }
        __syncthreads();  // every read of this iteration is done
        if (pending != kEmpty) atomicCAS(set + slot_of(pending), kEmpty, pending);
    }
}

// Static-mode sweep (stage 2 of the two-stage sweep): each of the two position ranges is walked
// separately (uniform pointer and base, no per-quad range select), and the
// guard load and the atomicMin are predicated instructions, not branches.
// SeenSet membership: a SWAR zero-lane test on each 32-bit word of the bucket
// (planes: word w of bucket b at set[w * kHubBuckets + b]).
template <int TW>
__device__ __forceinline__ bool seen_swar(const uint32_t* set, const HubHash& hh, uint32_t v) {
    constexpr uint32_t kTagMask = (1u << TW) - 1u;
    constexpr uint32_t kOnes = TW == 8 ? 0x01010101u : 0x00010001u;
    constexpr uint32_t kHigh = kOnes << (TW - 1);
    uint32_t b, tag;
    hh.split(v, b, tag);
    const uint32_t rep = tag * kOnes;
    uint32_t z = 0;
#pragma unroll
    for (int w = 0; w < kSeenPlanes; w++) {
        const uint32_t x = set[w * kHubBuckets + b] ^ rep;  // a lane equal to tag -> a zero lane
        z |= (x - kOnes) & ~x;
    }
    return (z & kHigh) != 0 && tag != kTagMask;        // all-ones tags are never inserted (empty marker)
}

#ifndef FH_PROBE_CACHE
#define FH_PROBE_CACHE "cg"
#endif
__device__ __forceinline__ uint32_t ld_cg_pred(const uint32_t* p, bool pred) {
    uint32_t r = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global." FH_PROBE_CACHE ".u32 %0, [%1];\n\t}"
                 : "+r"(r)
                 : "l"(p), "r"((uint32_t)pred));
    return r;
}
__device__ __forceinline__ void red_or_pred(uint32_t* p, uint32_t v, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.relaxed.gpu.global.or.b32 [%0], %1;\n\t}" ::"l"(p),
                 "r"(v), "r"((uint32_t)pred)
                 : "memory");
}
__device__ __forceinline__ void red_min_pred(uint32_t* p, uint32_t v, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.relaxed.gpu.global.min.u32 [%0], %1;\n\t}" ::"l"(p),
                 "r"(v), "r"((uint32_t)pred)
                 : "memory");
}

// BITS (first[] beyond L2, n > 2^23): the guard is not a load of first[v]
// (a DRAM line per access) but a bit of `seenb` (n bits, L2-resident): the
// vertices whose first occurrence lies in an earlier WAVE of positions.  A
// position passes to the red.min only for vertices not seen before its wave,
// and marks them in `newb`, which joins `seenb` after the wave (a bit set
// inside the wave would let a later position hide an earlier one still in
// flight).
template <int TW, bool BITS>
__device__ __forceinline__ void sweep_static(const uint4* __restrict__ src, uint64_t nq, uint32_t base,
                                             uint32_t* first, const uint32_t* set, const HubHash& hh,
                                             const uint32_t* __restrict__ seenb, uint32_t* newb) {
    constexpr uint64_t kIter = (uint64_t)kFhNT * kFhQuads;
    const uint64_t iters = ceil_div(nq, kIter);
    for (uint64_t it = blockIdx.x; it < iters; it += gridDim.x) {
        const uint64_t q0 = it * kIter + threadIdx.x;
        uint4 q[kFhQuads];
        bool ok[kFhQuads];
#pragma unroll
        for (int k = 0; k < kFhQuads; k++) {
            const uint64_t w = q0 + (uint64_t)k * kFhNT;
            ok[k] = w < nq;
            q[k] = ok[k] ? __ldg(src + w) : make_uint4(0, 0, 0, 0);
        }
        bool need[kFhQuads][4];
#pragma unroll
        for (int k = 0; k < kFhQuads; k++) {
            const uint32_t vs[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
#pragma unroll
            for (int j = 0; j < 4; j++) need[k][j] = ok[k] && !seen_swar<TW>(set, hh, vs[j]);
        }
        uint32_t cur[kFhQuads][4];
#pragma unroll
        for (int k = 0; k < kFhQuads; k++) {
            const uint32_t vs[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
#pragma unroll
            for (int j = 0; j < 4; j++)
                cur[k][j] = BITS ? ld_cg_pred(seenb + (vs[j] >> 5), need[k][j]) : ld_cg_pred(first + vs[j], need[k][j]);
        }
#pragma unroll
        for (int k = 0; k < kFhQuads; k++) {
            const uint32_t vs[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
            const uint32_t p0 = base + 4u * (uint32_t)(q0 + (uint64_t)k * kFhNT);
#pragma unroll
            for (int j = 0; j < 4; j++) {
                if (BITS) {
                    const bool go = need[k][j] && !((cur[k][j] >> (vs[j] & 31)) & 1u);
                    red_min_pred(first + vs[j], p0 + j, go);
                    red_or_pred(newb + (vs[j] >> 5), 1u << (vs[j] & 31), go);
                } else {
                    red_min_pred(first + vs[j], p0 + j, need[k][j] && p0 + j < cur[k][j]);
                }
            }
        }
    }
}

template <int TW, bool BITS>
__global__ void __launch_bounds__(kFhNT, 1) k_first_hit_static(Ranges r, uint32_t* first,
                                                               const uint32_t* __restrict__ seen_g,
                                                               HubHash hh, const uint32_t* seenb, uint32_t* newb) {
    extern __shared__ uint4 smem_u128[];
    uint32_t* set = reinterpret_cast<uint32_t*>(smem_u128);
    for (int i = threadIdx.x; i < (int)(kSeenSetBytes / 16); i += kFhNT)
        smem_u128[i] = __ldg(reinterpret_cast<const uint4*>(seen_g) + i);
    __syncthreads();
    sweep_static<TW, BITS>(reinterpret_cast<const uint4*>(r.a), r.qa, r.base_a, first, set, hh, seenb, newb);
    sweep_static<TW, BITS>(reinterpret_cast<const uint4*>(r.b), r.qb, r.base_b, first, set, hh, seenb, newb);
}

template <int TW, bool BITS = false>
static void launch_static(const Ranges& r, uint32_t* first, const uint32_t* seen_g, const HubHash& hh,
                          int num_sms, cudaStream_t s, const uint32_t* seenb = nullptr, uint32_t* newb = nullptr) {
    const size_t smem = kSeenSetBytes;
    static PerDeviceOnce attr;
    set_attr_once(attr, k_first_hit_static<TW, BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_first_hit_static<TW, BITS><<<num_sms, kFhNT, smem, s>>>(r, first, seen_g, hh, seenb, newb);
}

// seenb |= newb; newb = 0 (between waves)
__global__ void k_merge_bits(uint32_t* seenb, uint32_t* newb, uint64_t words) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += stride) {
        const uint32_t b = newb[i];
        if (b) {
            seenb[i] |= b;
            newb[i] = 0;
        }
    }
}

// SeenSet from the counting prefix: a vertex whose first occurrence is one of
// the prefix positions (exactly one thread per vertex) and whose prefix count
// lies in [lo, hi) gets its tag into a free lane of its bucket.  Rounds of
// decreasing count bands (frequent vertices first, then the rest) fill the
// lanes in priority order, each vertex offered once; a full bucket drops the
// vertex: membership only ever saves work, it never changes first[].
// Without counts (cnt == NULL) every such vertex is offered.
template <int TW>
__global__ void k_seen_build(const uint32_t* __restrict__ I, uint32_t count, uint32_t base,
                             const uint32_t* __restrict__ first, HubHash hh, const uint32_t* __restrict__ cnt,
                             uint32_t cmask, uint32_t lo, uint32_t hi, uint32_t* set) {
    constexpr uint32_t kTagMask = (1u << TW) - 1u;
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= count) return;
    const uint32_t v = __ldg(I + p);
    if (__ldg(first + v) != base + p) return;   // not the first occurrence
    if (cnt) {   // this round's count band only: a vertex is offered once
        const uint32_t c = __ldg(cnt + (hash_slot(v) & cmask));
        if (c < lo || c >= hi) return;
    }
    uint32_t b, tag;
    hh.split(v, b, tag);
    if (tag == kTagMask) return;                // reserved for "empty"
    for (int pl = 0; pl < kSeenPlanes; pl++) {
        uint32_t* wp = set + pl * kHubBuckets + b;
        uint32_t w = *wp;
        while (true) {
            int lane = -1;
            for (int l = 0; l < 32 / TW; l++)
                if (((w >> (TW * l)) & kTagMask) == kTagMask) { lane = l; break; }
            if (lane < 0) break;                // word full: next plane
            const uint32_t nw = (w & ~(kTagMask << (TW * lane))) | (tag << (TW * lane));
            const uint32_t old = atomicCAS(wp, w, nw);
            if (old == w) return;
            w = old;
        }
    }
}

// Frequency of every vertex in the counting prefix (hashed slots: a collision
// only merges two counts, which can only change the set's choice).
__global__ void k_prefix_count(const uint32_t* __restrict__ I, uint32_t count, uint32_t cmask, uint32_t* cnt) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < count) atomicAdd(cnt + (hash_slot(__ldg(I + p)) & cmask), 1u);
}

// Stage 1 of the two-stage sweep: guarded atomicMin over the prefix of I, one
// thread per position.
__global__ void k_first_hit_prefix(const uint32_t* __restrict__ I, uint32_t count, uint32_t base, uint32_t* first) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= count) return;
    const uint32_t v = __ldg(I + p);
    const uint32_t cur = __ldcg(first + v);
    if (base + p < cur) atomicMin(first + v, base + p);
}

// Scalar path: unaligned inputs and the (m mod 4) tails.
template <bool RELAXED>
__global__ void k_first_hit_scalar(const uint32_t* __restrict__ I, const uint32_t* __restrict__ J, uint64_t e0,
                                   uint64_t m, uint32_t base_i, uint32_t base_j, uint32_t* first) {
    const uint64_t cnt = m - e0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < 2 * cnt; t += stride) {
        const bool inJ = t >= cnt;
        const uint64_t e = e0 + (inJ ? t - cnt : t);
        const uint32_t v = inJ ? J[e] : I[e];
        const uint32_t pos = (uint32_t)e + (inJ ? base_j : base_i);
        if (RELAXED) {
            if (pos < *((volatile uint32_t*)(first + v))) *((volatile uint32_t*)(first + v)) = pos;
        } else {
            atomicMin(first + v, pos);
        }
    }
}

template <bool RELAXED>
static void launch_sweep(const Ranges& r, uint32_t* first, int num_sms, cudaStream_t s) {
    const size_t smem = sizeof(uint32_t) << kFhSlotsLog2;
    static PerDeviceOnce attr;
    set_attr_once(attr, k_first_hit<RELAXED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint64_t iters = ceil_div(r.qa + r.qb, (uint64_t)kFhNT * kFhQuads);
    if (iters == 0) return;
    const int grid = (int)(iters < (uint64_t)num_sms ? iters : (uint64_t)num_sms);
    k_first_hit<RELAXED><<<grid, kFhNT, smem, s>>>(r, first);
}

cudaError_t launch_first_hit(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n, uint32_t* first,
                             bool relaxed, int num_sms, cudaStream_t s) {
    return launch_first_hit_shard(I, J, m, m, 0, n, first, relaxed, nullptr, num_sms, s);
}

size_t first_hit_workspace_bytes() { return kHubTableBytes; }

// A contiguous shard [e0, e0 + m) of a global edge list with m_global edges:
// local I[i] sits at global position e0 + i, local J[i] at m_global + e0 + i.
// `seen_ws` (kHubTableBytes, may be NULL) enables the two-stage sweep.
// The prefix count table (kCountSlots words + the 256-bin histogram and the
// threshold) shares it: it is dead before the waves clear their bitmaps.
constexpr uint32_t kCountSlots = 1u << 21;
constexpr size_t kCountBytes = (size_t)kCountSlots * 4;
constexpr uint32_t kSeenHot = 4;  // first round: vertices seen at least this often in the prefix
size_t first_hit_bits_workspace_bytes(uint32_t n) {
    const size_t bits = 2 * (((uint64_t)n + 31) / 32 * 4 + 256);
    return bits > kCountBytes ? bits : kCountBytes;
}

// Static sweep of r in waves of positions (BITS mode, see sweep_static).
constexpr uint64_t kFhWaveQuads0 = (1ull << 22) / 4, kFhWaveQuadsMax = (1ull << 30) / 4;

template <int TW>
static cudaError_t launch_static_waves(const Ranges& r, uint32_t* first, const uint32_t* set,
                                       const HubHash& hh, uint32_t n, void* bits_ws, int num_sms, cudaStream_t s) {
    const uint64_t words = ((uint64_t)n + 31) / 32;
    uint32_t* seenb = static_cast<uint32_t*>(bits_ws);
    uint32_t* newb = reinterpret_cast<uint32_t*>(static_cast<char*>(bits_ws) + (words * 4 + 256) / 256 * 256);
    cudaError_t e = cudaMemsetAsync(seenb, 0, words * 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(newb, 0, words * 4, s);
    if (e != cudaSuccess) return e;
    const uint64_t total = r.qa + r.qb;
    const uint64_t mb = ceil_div(words, 256), cap = (uint64_t)num_sms * 8;
    // Geometric waves: 2^22 positions, doubling up to 2^30.  A wave costs a
    // red.min for every position whose vertex is unseen before the wave, so
    // early in the stream (nearly every vertex new) short waves move vertices
    // into the bitmap sooner; later waves are nearly all bitmap hits and long
    // ones save merges.  Measured at s26: fixed 2^26-position waves 8.64 ms,
    // geometric 2^22 -> 2^26 7.73, 2^22 -> 2^28 7.26, 2^22 -> 2^30 7.22.
    uint64_t wq = kFhWaveQuads0;
    for (uint64_t w0 = 0; w0 < total; w0 += wq, wq = wq * 2 < kFhWaveQuadsMax ? wq * 2 : kFhWaveQuadsMax) {
        const uint64_t w1 = w0 + wq < total ? w0 + wq : total;
        Ranges rw{};
        const uint64_t a0 = w0 < r.qa ? w0 : r.qa, a1 = w1 < r.qa ? w1 : r.qa;  // part in A
        rw.a = r.a + 4 * a0;
        rw.qa = a1 - a0;
        rw.base_a = r.base_a + (uint32_t)(4 * a0);
        const uint64_t b0 = w0 > r.qa ? w0 - r.qa : 0, b1 = w1 > r.qa ? w1 - r.qa : 0;  // part in B
        rw.b = r.b + 4 * b0;
        rw.qb = b1 - b0;
        rw.base_b = r.base_b + (uint32_t)(4 * b0);
        launch_static<TW, true>(rw, first, set, hh, num_sms, s, seenb, newb);
        if (w1 < total) k_merge_bits<<<(unsigned)(mb < cap ? mb : cap), 256, 0, s>>>(seenb, newb, words);
    }
    return cudaGetLastError();
}

cudaError_t launch_first_hit_shard(const uint32_t* I, const uint32_t* J, uint64_t m, uint64_t m_global, uint64_t e0,
                                   uint32_t n, uint32_t* first, bool relaxed, void* seen_ws, int num_sms,
                                   cudaStream_t s, void* bits_ws) {
    const uint32_t base_i = (uint32_t)e0, base_j = (uint32_t)(m_global + e0);
    cudaError_t err = cudaMemsetAsync(first, 0xFF, (size_t)n * sizeof(uint32_t), s);
    if (err != cudaSuccess || m == 0) return err;
    const bool vec = ((reinterpret_cast<uintptr_t>(I) | reinterpret_cast<uintptr_t>(J)) & 15) == 0;
    const HubHash hh = HubHash::make(n);
    uint64_t done = 0;
    if (vec && m >= 4) {
        const uint64_t quads = m >> 2;
        // counting prefix: the largest power of two <= min(seen_prefix, m / 256), at least 64K
        uint32_t prefix = seen_prefix(hh.tag_bits);
        while (prefix > 65536u && 256ull * prefix > m) prefix >>= 1;
        const bool two_stage = seen_ws && !relaxed && hh.tag_bits <= 16 && m >= 16ull * prefix;
        if (two_stage) {
            uint32_t* set = static_cast<uint32_t*>(seen_ws);
            const uint64_t qp = prefix / 4;
            // stage 1 fully parallel (the ordered persistent sweep ran on only a few CTAs
            // for a 128K-position prefix: 20 us vs 8 us)
            k_first_hit_prefix<<<(unsigned)ceil_div(prefix, 256), 256, 0, s>>>(I, prefix, base_i, first);
            err = cudaMemsetAsync(set, 0xFF, kSeenSetBytes, s);
            if (err != cudaSuccess) return err;
            // the set's members: the prefix's first-seen vertices, most frequent first
            uint32_t* cnt = bits_ws ? static_cast<uint32_t*>(bits_ws) : nullptr;
            const uint32_t cmask = kCountSlots - 1;
            const unsigned pg = (unsigned)ceil_div(prefix, 256);
            if (cnt) {
                err = cudaMemsetAsync(cnt, 0, kCountBytes, s);
                if (err != cudaSuccess) return err;
                k_prefix_count<<<pg, 256, 0, s>>>(I, prefix, cmask, cnt);
            }
            auto build = [&](auto tw) {
                constexpr int TW = decltype(tw)::value;
                // fill rounds, most frequent first: counts >= 8 (wide ids only), [4, 8), then the rest
                constexpr uint32_t kAll = 0xFFFFFFFFu;
                const uint32_t hot_hi = TW == 16 ? 2 * kSeenHot : kAll;
                if (cnt && TW == 16)
                    k_seen_build<TW><<<pg, 256, 0, s>>>(I, prefix, base_i, first, hh, cnt, cmask, 2 * kSeenHot, kAll,
                                                        set);
                if (cnt)
                    k_seen_build<TW><<<pg, 256, 0, s>>>(I, prefix, base_i, first, hh, cnt, cmask, kSeenHot, hot_hi,
                                                        set);
                k_seen_build<TW><<<pg, 256, 0, s>>>(I, prefix, base_i, first, hh, cnt, cmask, 1u,
                                                    cnt ? kSeenHot : kAll, set);
            };
            Ranges r2{I + prefix, quads - qp, base_i + prefix, J, quads, base_j};
            // first[] beyond L2 (n > 2^23, > 32 MB): guard on a seen-bitmap in geometric waves
            // instead of first[] itself (measured: s26 18.0 -> 7.2 ms; s24 1.70 -> 1.66; s22, first[]
            // L2-resident, 0.32 -> 0.44, so not there)
            const bool waves = bits_ws && n > (1u << 23);
            if (hh.tag_bits <= 8) {
                build(std::integral_constant<int, 8>{});
                if (waves) err = launch_static_waves<8>(r2, first, set, hh, n, bits_ws, num_sms, s);
                else launch_static<8>(r2, first, set, hh, num_sms, s);
            } else {
                build(std::integral_constant<int, 16>{});
                if (waves) err = launch_static_waves<16>(r2, first, set, hh, n, bits_ws, num_sms, s);
                else launch_static<16>(r2, first, set, hh, num_sms, s);
            }
            if (err != cudaSuccess) return err;
        } else {
            Ranges r{I, quads, base_i, J, quads, base_j};
            if (relaxed)
                launch_sweep<true>(r, first, num_sms, s);
            else
                launch_sweep<false>(r, first, num_sms, s);
        }
        done = m & ~3ull;
    }
    if (done < m) {
        uint64_t work = 2 * (m - done), blocks = ceil_div(work, 256), cap = (uint64_t)num_sms * 8;
        int grid = (int)(blocks < cap ? blocks : cap);
        if (relaxed)
            k_first_hit_scalar<true><<<grid, 256, 0, s>>>(I, J, done, m, base_i, base_j, first);
        else
            k_first_hit_scalar<false><<<grid, 256, 0, s>>>(I, J, done, m, base_i, base_j, first);
    }
    return cudaGetLastError();
}

}  // namespace boba
