// Shared-memory hub structures for the two L2-request-bound phases.
//
// BOBA orders vertices by first appearance, and on skewed graphs the first
// vertices to appear are the hubs: at c2 (R-MAT s22) the 32K smallest labels
// cover 38% of all edge endpoints and the 64K smallest 51%.  Both structures
// below are keyed by a bijective hash of the vertex id on kk = max(ceil(log2
// n), 14) bits: the top 14 bits pick one of 16K buckets, the remaining
// kk - 14 bits are stored as a tag, so an entry needs no full id.
//
//  * HubLabels (phase 3, relabel): 16K buckets x 3 entries of 32 bits,
//    entry = label << tagbits | tag, for the vertices with labels < 49151;
//    smaller labels win slots (one atomicMin round per slot), 192 KB.
//  * SeenSet (phase 1, first occurrence): 16K buckets of 96 bits (three
//    32-bit planes), each holding 12 8-bit tags (ids up to 2^22) or 6
//    16-bit tags (up to 2^30), 192 KB.  Its members are the most frequent
//    vertices of a counting prefix of I whose first occurrence lies in that
//    prefix: every later position of such a vertex is known not to be its
//    first, so it costs no global access at all.  Chosen by frequency, the
//    set covers far more endpoints than the prefix's first-seen vertices
//    (measured, 64K-position prefix -> top of a 2M-position count:
//    s22 54 -> ~75 %, s26 17 -> ~35 % of all endpoints).
#pragma once
#include <cstdint>

namespace boba {

constexpr int kHubBucketsLog2 = 14;
constexpr int kHubBuckets = 1 << kHubBucketsLog2;
constexpr int kHubWays = 3;                  // HubLabels entries per bucket
constexpr size_t kHubTableBytes = sizeof(uint32_t) * kHubWays << kHubBucketsLog2;  // HubLabels; SeenSet uses 2/3
constexpr uint32_t kHubMaxLabel = 49151;     // labels [0, kHubMaxLabel) go into HubLabels
constexpr int kSeenPlanes = 2;               // SeenSet: 32-bit words per bucket, stored as planes
constexpr size_t kSeenSetBytes = sizeof(uint32_t) * kSeenPlanes << kHubBucketsLog2;
static_assert(kSeenSetBytes <= kHubTableBytes, "the SeenSet lives in the hub table area");
// Stage 1 sweeps I[0, prefix) and counts its vertices; the set takes the most
// frequent of those first seen there, up to ~75% of its capacity.
__host__ __device__ inline uint32_t seen_prefix(int tag_bits) { return tag_bits <= 8 ? (1u << 20) : (1u << 21); }
__host__ __device__ inline uint32_t seen_capacity(int tag_bits) {
    return (uint32_t)kHubBuckets * kSeenPlanes * (tag_bits <= 8 ? 4u : 2u);
}

struct HubHash {
    int kk;          // hashed width, >= kHubBucketsLog2
    int tag_bits;    // kk - kHubBucketsLog2
    uint32_t mask;   // low kk bits

    static HubHash make(uint32_t n) {  // host
        int k = n <= 1 ? 0 : 32 - __builtin_clz(n - 1);
        HubHash h;
        h.kk = k < kHubBucketsLog2 ? kHubBucketsLog2 : k;
        h.tag_bits = h.kk - kHubBucketsLog2;
        h.mask = h.kk >= 32 ? 0xFFFFFFFFu : (1u << h.kk) - 1u;
        return h;
    }
    // bijection on kk bits: odd multiply mod 2^kk (ids are random labels or
    // BOBA ranks, so one multiply mixes enough)
    __device__ __forceinline__ void split(uint32_t v, uint32_t& bucket, uint32_t& tag) const {
        const uint32_t x = (v * 0x9E3779B1u) & mask;
        bucket = x >> tag_bits;
        tag = x & ((1u << tag_bits) - 1u);   // tag_bits < 32
    }
};

}  // namespace boba
