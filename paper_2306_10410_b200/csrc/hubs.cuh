// Hub label table shared by phase 2 (producer, k_assign) and phase 3
// (consumer, k_relabel): a direct-mapped table of 2^kHubSlotsLog2 64-bit
// entries (label << 32 | old id) holding the vertices with the smallest
// BOBA labels -- the hubs -- smallest label wins a slot.  Empty = all ones.
#pragma once
#include <cstdint>

namespace boba {

constexpr int kHubSlotsLog2 = 14;
constexpr size_t kHubTableBytes = sizeof(unsigned long long) << kHubSlotsLog2;

__device__ __forceinline__ uint32_t hub_slot(uint32_t v) { return (v * 0x9E3779B1u) >> (32 - kHubSlotsLog2); }

__device__ __forceinline__ void hub_insert(unsigned long long* table, uint32_t v, uint32_t r) {
    if (table && r < (1u << kHubSlotsLog2)) atomicMin(table + hub_slot(v), ((unsigned long long)r << 32) | v);
}

}  // namespace boba
