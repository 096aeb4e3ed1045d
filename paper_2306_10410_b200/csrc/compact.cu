// Phase 2 -- rank compaction: first[] -> (order, label), linear time, no sort.
//
// Reference: pkg/src/boba/_parallel.py:178-201 compact_ranks (presence flag
// per used rank over [0,2m), compaction scan, isolated vertices appended in
// ascending ID order) and graph.py:205-208 (label[order[k]] = k).
//
// B200 formulation (three kernels, all O(n) random or O(m/32) streaming):
//   k_mark          one bit per used position: atomicOr into a 2m-bit map
//                   stored as 32-byte records of 224 bits (7 words) plus, in
//                   the record's 8th word, the number of set bits before it.
//   k_rec_scan      single-pass decoupled-lookback exclusive scan of the
//                   records' popcounts, written into their 8th words; the
//                   total is n_seen (vertices that occur at all).
//   k_assign        per vertex: rank = record prefix + popcount of the bits
//                   below it in its record -- one 32-byte sector, so one
//                   random access per vertex -- or, for a vertex that never
//                   occurs, n_seen + its rank among the isolated vertices (a
//                   second lookback scan over vertex tiles keeps them in
//                   ascending ID order).  Writes label[v] = rank (coalesced)
//                   and order[rank] = v.
// No gather of I||J is needed: position first[v] holds v by definition.
#include "common.cuh"
#include "hubs.cuh"
#include "kernels.cuh"

namespace boba {

constexpr int kScanNT = 256;
constexpr int kRecWords = 7;                            // bitmap words per 32-byte record
constexpr uint32_t kRecBits = 32 * kRecWords;           // 224 positions per record
#ifndef RECS_PER_THREAD
#define RECS_PER_THREAD 4
#endif
constexpr int kRecsPerThread = RECS_PER_THREAD;
constexpr int kRecsPerTile = kScanNT * kRecsPerThread;
// vertices per thread (multiple of 4; measured c4 / c5 P2: 4 -> 2.71 / 0.41 ms,
// 8 -> 2.69 / 0.39, 16 -> 2.74 / 0.41)
constexpr int kAssignVPT = 8;
static_assert(kAssignVPT % 4 == 0, "labels are stored as 16-byte quads");
constexpr int kAssignTile = kScanNT * kAssignVPT;

// word w of the bitmap (position p: w = p >> 5) -> its index in the record array
__device__ __forceinline__ uint32_t rec_of_word(uint32_t w) { return w / kRecWords; }

__global__ void k_mark(const uint32_t* __restrict__ first, uint32_t n, uint32_t* recs) {
    uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
        const uint32_t f = __ldg(first + v);
        if (f != BOBA_UNSET) {
            const uint32_t w = f >> 5, r = rec_of_word(w);
            atomicOr(recs + 8 * r + (w - r * kRecWords), 1u << (f & 31));
        }
    }
}

__global__ void __launch_bounds__(kScanNT) k_rec_scan(uint4* recs, uint64_t nrec, unsigned long long* status,
                                                      unsigned* tile_counter, uint32_t* n_seen) {
    __shared__ unsigned s_tile;
    __shared__ uint32_t s_scan[kScanNT / 32 + 1];
    __shared__ unsigned long long s_excl;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t r0 = tile * kRecsPerTile + (uint64_t)threadIdx.x * kRecsPerThread;
    uint32_t cnt[kRecsPerThread];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kRecsPerThread; k++) {
        uint32_t c = 0;
        if (r0 + k < nrec) {
            const uint4 a = recs[2 * (r0 + k)], b = recs[2 * (r0 + k) + 1];
            c = __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w) + __popc(b.x) + __popc(b.y) + __popc(b.z);
        }
        cnt[k] = c;
        sum += c;
    }
    uint32_t total;
    uint32_t excl_thread = block_exclusive_sum<kScanNT>(sum, s_scan, &total);
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0)
            st_volatile_u64(status + tile, (tile == 0 ? kFlagInc : kFlagAgg) | (unsigned long long)total);
        unsigned long long ex = tile == 0 ? 0ull : warp_lookback(status, (long long)tile);
        if (threadIdx.x == 0) {
            if (tile != 0) st_volatile_u64(status + tile, kFlagInc | (ex + total));
            s_excl = ex;
            if (tile == ceil_div(nrec, kRecsPerTile) - 1) *n_seen = (uint32_t)(ex + total);
        }
    }
    __syncthreads();
    uint32_t run = (uint32_t)s_excl + excl_thread;
    uint32_t* words = reinterpret_cast<uint32_t*>(recs);
#pragma unroll
    for (int k = 0; k < kRecsPerThread; k++) {
        if (r0 + k < nrec) words[8 * (r0 + k) + kRecWords] = run;
        run += cnt[k];
    }
}

__device__ __forceinline__ uint32_t rank_of(uint32_t f, const uint4* __restrict__ recs) {
    const uint32_t w = f >> 5, r = rec_of_word(w), wi = w - r * kRecWords, b = f & 31;
    const uint4 lo = __ldg(recs + 2 * r), hi = __ldg(recs + 2 * r + 1);
    const uint32_t words[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    uint32_t rank = words[kRecWords];
#pragma unroll
    for (int k = 0; k < kRecWords; k++) {
        if ((uint32_t)k < wi) rank += __popc(words[k]);
        else if ((uint32_t)k == wi) rank += __popc(words[k] & ((1u << b) - 1u));
    }
    return rank;
}

// Rank of position f from its record (lo = words 0-3, hi = words 4-6 + the
// record's prefix), branch-free.
__device__ __forceinline__ uint32_t rank_in_record(const uint4& lo, const uint4& hi, uint32_t f) {
    const uint32_t w = f >> 5, wi = w - rec_of_word(w) * kRecWords, below = (1u << (f & 31)) - 1u;
    const uint32_t words[kRecWords] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z};
    uint32_t rank = hi.w;
#pragma unroll
    for (int k = 0; k < kRecWords; k++)
        rank += __popc(words[k] & ((uint32_t)k < wi ? 0xFFFFFFFFu : ((uint32_t)k == wi ? below : 0u)));
    return rank;
}

// Record loads in flight per thread: the lookups are independent DRAM
// round trips (the record array is beyond L2 at s26), so they are issued in
// batches rather than one vertex at a time (measured, P2 c4 / c5 / c2: one
// at a time 2.69 / 0.392 / 0.111 ms, batches of 2 2.61 / 0.371 / 0.101,
// 4: 2.62 / 0.370 / 0.101, all 8: 2.58 / 0.350 / 0.097).
#ifndef ASSIGN_BATCH
#define ASSIGN_BATCH 8
#endif

__global__ void __launch_bounds__(kScanNT) k_assign(const uint32_t* __restrict__ first, uint32_t n,
                                                    const uint4* __restrict__ recs,
                                                    const uint32_t* __restrict__ n_seen_ptr,
                                                    uint32_t* __restrict__ order, uint32_t* __restrict__ label,
                                                    unsigned long long* status, unsigned* tile_counter) {
    __shared__ unsigned s_tile;
    __shared__ uint32_t s_scan[kScanNT / 32 + 1];
    __shared__ unsigned long long s_excl;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t v0 = tile * kAssignTile + (uint64_t)threadIdx.x * kAssignVPT;
    uint32_t f[kAssignVPT];
    uint32_t iso = 0;
#pragma unroll
    for (int k = 0; k < kAssignVPT; k++) {
        f[k] = (v0 + k < n) ? __ldg(first + v0 + k) : 0u;
        iso += (v0 + k < n && f[k] == BOBA_UNSET);
    }
    uint32_t total;
    const uint32_t iso_excl = block_exclusive_sum<kScanNT>(iso, s_scan, &total);
    // publish the tile's aggregate now; the lookback comes after the rank
    // lookups, so its wait overlaps them
    if (threadIdx.x == 0)
        st_volatile_u64(status + tile, (tile == 0 ? kFlagInc : kFlagAgg) | (unsigned long long)total);
    // seen vertices: rank = record prefix + popcount below the position
    uint32_t lab[kAssignVPT];
#pragma unroll
    for (int k0 = 0; k0 < kAssignVPT; k0 += ASSIGN_BATCH) {
        uint4 lo[ASSIGN_BATCH], hi[ASSIGN_BATCH];
#pragma unroll
        for (int j = 0; j < ASSIGN_BATCH; j++) {
            const int k = k0 + j;
            if (v0 + k < n && f[k] != BOBA_UNSET) {
                const uint32_t r = rec_of_word(f[k] >> 5);
                lo[j] = __ldg(recs + 2 * r);
                hi[j] = __ldg(recs + 2 * r + 1);
            } else {
                lo[j] = hi[j] = make_uint4(0, 0, 0, 0);
            }
        }
#pragma unroll
        for (int j = 0; j < ASSIGN_BATCH; j++) {
            const int k = k0 + j;
            lab[k] = rank_in_record(lo[j], hi[j], f[k]);
            if (v0 + k < n && f[k] != BOBA_UNSET) order[lab[k]] = (uint32_t)(v0 + k);
        }
    }
    if (threadIdx.x < 32) {
        unsigned long long ex = tile == 0 ? 0ull : warp_lookback(status, (long long)tile);
        if (threadIdx.x == 0) {
            if (tile != 0) st_volatile_u64(status + tile, kFlagInc | (ex + total));
            s_excl = ex;
        }
    }
    __syncthreads();
    // never-seen vertices: n_seen + their ascending rank among them
    uint32_t iso_rank = __ldg(n_seen_ptr) + (uint32_t)s_excl + iso_excl;
#pragma unroll
    for (int k = 0; k < kAssignVPT; k++) {
        if (v0 + k < n && f[k] == BOBA_UNSET) {
            lab[k] = iso_rank++;
            order[lab[k]] = (uint32_t)(v0 + k);
        }
    }
    if (v0 + kAssignVPT <= n && (reinterpret_cast<uintptr_t>(label) & 15) == 0) {
#pragma unroll
        for (int q = 0; q < kAssignVPT / 4; q++)
            reinterpret_cast<uint4*>(label + v0)[q] = make_uint4(lab[4 * q], lab[4 * q + 1], lab[4 * q + 2], lab[4 * q + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < kAssignVPT; k++)
            if (v0 + k < n) label[v0 + k] = lab[k];
    }
}

// table = kHubWays arrays of kHubBuckets entries holding, per bucket, the
// kHubWays smallest entries (label << tag_bits | tag) in ascending order, in
// one pass: an entry goes through the ways with atomicMin and carries the
// larger of itself and the displaced value on to the next way, so every value
// but a way's final minimum reaches the next way exactly once.
__global__ void k_hub_labels(const uint32_t* __restrict__ order, uint32_t K, HubHash hh, uint32_t* table) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    uint32_t b, tag;
    hh.split(__ldg(order + k), b, tag);
    uint32_t e = (k << hh.tag_bits) | tag;
#pragma unroll
    for (int w = 0; w < kHubWays; w++) {
        const uint32_t old = atomicMin(table + w * kHubBuckets + b, e);
        e = old > e ? old : e;
        if (e == 0xFFFFFFFFu) break;  // filled an empty slot: nothing to carry
    }
}

namespace {
struct CompactWs {
    uint32_t* recs;     // 2m-bit map in 32-byte records (7 words + prefix)
    unsigned long long* st_rec;
    unsigned long long* st_v;
    unsigned* counters;
    size_t total;
};
uint64_t num_recs(uint64_t m) { return ceil_div(2 * m + 1, kRecBits) + 1; }
CompactWs carve_compact(void* base, uint64_t m, uint32_t n) {
    const uint64_t nrec = num_recs(m);
    const uint64_t rec_tiles = ceil_div(nrec, kRecsPerTile);
    const uint64_t v_tiles = ceil_div((uint64_t)n, kAssignTile) + 1;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return base ? static_cast<char*>(base) + o : nullptr;
    };
    CompactWs w;
    w.recs = (uint32_t*)take(nrec * 32);
    w.st_rec = (unsigned long long*)take(rec_tiles * 8);
    w.st_v = (unsigned long long*)take(v_tiles * 8);
    w.counters = (unsigned*)take(64);
    w.total = off;  // all of it is cleared per call
    return w;
}
}  // namespace

size_t compact_workspace_bytes(uint64_t m, uint32_t n) { return carve_compact(nullptr, m, n).total; }

// Vertices whose first occurrence lies in I = set bits of the map before
// position m.  Every CSR row is the label of such a vertex (it occurs in I),
// so this bounds the rows COO->CSR has to sort.
__global__ void k_seen_in_first_half(const uint4* __restrict__ recs, uint64_t m, uint32_t* out) {
    *out = m ? rank_of((uint32_t)m, recs) : 0u;
}

cudaError_t launch_compact(const uint32_t* first, uint64_t m, uint32_t n, uint32_t* order,
                           uint32_t* label, uint32_t* n_seen_out, unsigned long long* hubs, void* ws,
                           size_t ws_bytes, int num_sms, cudaStream_t s, uint32_t* rows_bound_out) {
    if (ws_bytes < compact_workspace_bytes(m, n)) return cudaErrorInvalidValue;
    if (n == 0) return cudaSuccess;
    const uint64_t nrec = num_recs(m);
    const uint64_t rec_tiles = ceil_div(nrec, kRecsPerTile);
    const uint64_t v_tiles = ceil_div((uint64_t)n, kAssignTile);
    CompactWs w = carve_compact(ws, m, n);
    unsigned* counters = w.counters;
    uint32_t* n_seen = counters + 4;
    // clear the records (bits and prefixes), lookback status and counters
    cudaError_t err = cudaMemsetAsync(ws, 0, w.total, s);
    if (err != cudaSuccess) return err;
    {
        uint64_t blocks = ceil_div(n, 256);
        uint64_t cap = (uint64_t)num_sms * 16;
        k_mark<<<(int)(blocks < cap ? blocks : cap), 256, 0, s>>>(first, n, w.recs);
    }
    k_rec_scan<<<(int)rec_tiles, kScanNT, 0, s>>>(reinterpret_cast<uint4*>(w.recs), nrec, w.st_rec, counters + 0,
                                                  n_seen);
    k_assign<<<(int)v_tiles, kScanNT, 0, s>>>(first, n, reinterpret_cast<const uint4*>(w.recs), n_seen, order, label,
                                              w.st_v, counters + 1);
    if (n_seen_out) cudaMemcpyAsync(n_seen_out, n_seen, 4, cudaMemcpyDeviceToDevice, s);
    if (rows_bound_out)
        k_seen_in_first_half<<<1, 1, 0, s>>>(reinterpret_cast<const uint4*>(w.recs), m, rows_bound_out);
    if (hubs) {
        // HubLabels (hubs.cuh) for phase 3: labels [0, kHubMaxLabel), kHubWays
        // slots per bucket, the smallest labels of each bucket (one pass).
        const HubHash hh = HubHash::make(n);
        if (hh.tag_bits <= 16) {
            err = cudaMemsetAsync(hubs, 0xFF, kHubTableBytes, s);
            if (err != cudaSuccess) return err;
            const uint32_t K = n < kHubMaxLabel ? n : kHubMaxLabel;
            k_hub_labels<<<(unsigned)ceil_div(K, 256), 256, 0, s>>>(order, K, hh, reinterpret_cast<uint32_t*>(hubs));
        } else {
            err = cudaMemsetAsync(hubs, 0xFF, kHubTableBytes, s);  // empty table: relabel gathers everything
            if (err != cudaSuccess) return err;
        }
    }
    return cudaGetLastError();
}

// ------------------------------------------------- sharded compaction ---
// Multi-GPU phase 2 (sharded.py).  Rank r of P holds edges [e0, e0 + ml) of
// the m-edge list, i.e. positions [e0, e0 + ml) of I and [m + e0, m + e0 + ml)
// of J.  After the global first[] is known everywhere (allreduce-MIN), rank r
// owns the vertices whose first position lies in one of its two windows and
// compacts only those: a 2 ml-bit map over its windows (I window first), the
// same record scan as above, and for every owned vertex its rank inside the
// map.  The global rank follows from the 2P window counts (an allgather):
// the scan order of [0, 2m) is I0 I1 .. I_{P-1} J0 J1 .. J_{P-1}, so
//   I window of r: base = sum_{j<r} cI[j]
//   J window of r: base = sum_j cI[j] + sum_{j<r} cJ[j] - cI[r]   (local rank counts cI[r] first)
// Never-seen vertices get n_seen + their ascending rank, written by rank 0
// only, so an allreduce-SUM of the per-rank partial labels (0 elsewhere) is
// the global label array.  Reference semantics: _parallel.py:178-201.
__device__ __forceinline__ bool window_pos(uint32_t f, uint64_t m, uint64_t e0, uint64_t ml, uint32_t& q) {
    if (f == BOBA_UNSET) return false;
    if ((uint64_t)f >= e0 && (uint64_t)f < e0 + ml) {
        q = (uint32_t)(f - e0);
        return true;
    }
    if ((uint64_t)f >= m + e0 && (uint64_t)f < m + e0 + ml) {
        q = (uint32_t)(ml + (f - m - e0));
        return true;
    }
    return false;
}

__global__ void k_mark_window(const uint32_t* __restrict__ first, uint32_t n, uint64_t m, uint64_t e0, uint64_t ml,
                              uint32_t* recs) {
    uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
        uint32_t q;
        if (window_pos(__ldg(first + v), m, e0, ml, q)) {
            const uint32_t w = q >> 5, r = rec_of_word(w);
            atomicOr(recs + 8 * r + (w - r * kRecWords), 1u << (q & 31));
        }
    }
}

// counts[0] = owned vertices first seen in the I window, counts[1] = in the J window
__global__ void k_window_counts(const uint4* __restrict__ recs, uint64_t ml, const uint32_t* __restrict__ n_seen,
                                uint32_t* counts) {
    const uint32_t ci = rank_of((uint32_t)ml, recs);
    counts[0] = ci;
    counts[1] = *n_seen - ci;
}

__global__ void __launch_bounds__(kScanNT) k_assign_window(const uint32_t* __restrict__ first, uint32_t n, uint64_t m,
                                                           uint64_t e0, uint64_t ml, const uint4* __restrict__ recs,
                                                           const uint32_t* __restrict__ all_counts, int world,
                                                           int rank, uint32_t* label, unsigned long long* status,
                                                           unsigned* tile_counter) {
    __shared__ unsigned s_tile;
    __shared__ uint32_t s_scan[kScanNT / 32 + 1];
    __shared__ unsigned long long s_excl;
    __shared__ uint32_t s_base[3];  // base_I, base_J, n_seen
    if (threadIdx.x == 0) {
        s_tile = atomicAdd(tile_counter, 1u);
        uint32_t tot_i = 0, tot_j = 0, pre_i = 0, pre_j = 0;
        for (int k = 0; k < world; k++) {
            const uint32_t ci = all_counts[2 * k], cj = all_counts[2 * k + 1];
            if (k < rank) pre_i += ci, pre_j += cj;
            tot_i += ci, tot_j += cj;
        }
        s_base[0] = pre_i;
        s_base[1] = tot_i + pre_j - all_counts[2 * rank];
        s_base[2] = tot_i + tot_j;
    }
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t v0 = tile * kAssignTile + (uint64_t)threadIdx.x * kAssignVPT;
    uint32_t f[kAssignVPT];
    uint32_t iso = 0;
#pragma unroll
    for (int k = 0; k < kAssignVPT; k++) {
        f[k] = (v0 + k < n) ? __ldg(first + v0 + k) : 0u;
        iso += (v0 + k < n && f[k] == BOBA_UNSET);
    }
    uint32_t total;
    uint32_t iso_excl = block_exclusive_sum<kScanNT>(iso, s_scan, &total);
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
    uint32_t iso_rank = s_base[2] + (uint32_t)s_excl + iso_excl;
    uint32_t lab[kAssignVPT];
#pragma unroll
    for (int k = 0; k < kAssignVPT; k++) {
        uint32_t q, r = 0;
        if (f[k] == BOBA_UNSET) {
            r = rank == 0 ? iso_rank : 0u;
            iso_rank++;
        } else if (window_pos(f[k], m, e0, ml, q)) {
            r = (q < ml ? s_base[0] : s_base[1]) + rank_of(q, recs);
        }
        lab[k] = r;
    }
    if (v0 + kAssignVPT <= n && (reinterpret_cast<uintptr_t>(label) & 15) == 0) {
#pragma unroll
        for (int q = 0; q < kAssignVPT / 4; q++)
            reinterpret_cast<uint4*>(label + v0)[q] = make_uint4(lab[4 * q], lab[4 * q + 1], lab[4 * q + 2], lab[4 * q + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < kAssignVPT; k++)
            if (v0 + k < n) label[v0 + k] = lab[k];
    }
}

__global__ void k_order_from_label(const uint32_t* __restrict__ label, uint32_t n, uint32_t* order) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) order[__ldg(label + v)] = v;
}

size_t compact_window_workspace_bytes(uint64_t ml, uint32_t n) { return carve_compact(nullptr, ml, n).total; }

cudaError_t launch_compact_window_mark(const uint32_t* first, uint32_t n, uint64_t m, uint64_t e0, uint64_t ml,
                                       uint32_t* counts, void* ws, size_t ws_bytes, int num_sms, cudaStream_t s) {
    if (ws_bytes < compact_window_workspace_bytes(ml, n)) return cudaErrorInvalidValue;
    CompactWs w = carve_compact(ws, ml, n);
    const uint64_t nrec = num_recs(ml);
    cudaError_t err = cudaMemsetAsync(ws, 0, w.total, s);
    if (err != cudaSuccess) return err;
    if (n) {
        const uint64_t blocks = ceil_div(n, 256), cap = (uint64_t)num_sms * 16;
        k_mark_window<<<(int)(blocks < cap ? blocks : cap), 256, 0, s>>>(first, n, m, e0, ml, w.recs);
    }
    k_rec_scan<<<(int)ceil_div(nrec, kRecsPerTile), kScanNT, 0, s>>>(reinterpret_cast<uint4*>(w.recs), nrec, w.st_rec,
                                                                    w.counters + 0, w.counters + 4);
    k_window_counts<<<1, 1, 0, s>>>(reinterpret_cast<const uint4*>(w.recs), ml, w.counters + 4, counts);
    return cudaGetLastError();
}

cudaError_t launch_compact_window_assign(const uint32_t* first, uint32_t n, uint64_t m, uint64_t e0, uint64_t ml,
                                         const uint32_t* all_counts, int world, int rank, uint32_t* label, void* ws,
                                         size_t ws_bytes, cudaStream_t s) {
    if (ws_bytes < compact_window_workspace_bytes(ml, n)) return cudaErrorInvalidValue;
    if (n == 0) return cudaSuccess;
    CompactWs w = carve_compact(ws, ml, n);
    cudaError_t err = cudaMemsetAsync(w.st_v, 0, (ceil_div((uint64_t)n, kAssignTile) + 1) * 8, s);
    if (err == cudaSuccess) err = cudaMemsetAsync(w.counters + 1, 0, 4, s);
    if (err != cudaSuccess) return err;
    k_assign_window<<<(int)ceil_div((uint64_t)n, kAssignTile), kScanNT, 0, s>>>(
        first, n, m, e0, ml, reinterpret_cast<const uint4*>(w.recs), all_counts, world, rank, label, w.st_v,
        w.counters + 1);
    return cudaGetLastError();
}

cudaError_t launch_order_from_label(const uint32_t* label, uint32_t n, uint32_t* order,
                                    unsigned long long* hubs, int num_sms, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint64_t blocks = ceil_div(n, 256), cap = (uint64_t)num_sms * 16;
    k_order_from_label<<<(int)(blocks < cap ? blocks : cap), 256, 0, s>>>(label, n, order);
    if (hubs) {
        cudaError_t err = cudaMemsetAsync(hubs, 0xFF, kHubTableBytes, s);
        if (err != cudaSuccess) return err;
        const HubHash hh = HubHash::make(n);
        if (hh.tag_bits <= 16) {
            const uint32_t K = n < kHubMaxLabel ? n : kHubMaxLabel;
            k_hub_labels<<<(unsigned)ceil_div(K, 256), 256, 0, s>>>(order, K, hh, reinterpret_cast<uint32_t*>(hubs));
        }
    }
    return cudaGetLastError();
}

}  // namespace boba
