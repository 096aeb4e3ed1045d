// Shared device helpers for the BOBA sm_100a kernels: lane intrinsics,
// warp/block scans, and the decoupled-lookback status protocol used by every
// single-pass scan in the library (sector ranks, isolated-vertex ranks, CSR
// offsets, radix bucket offsets and the SpMV row carries).
#pragma once
#include <atomic>
#include <mutex>
#include <cstdint>
#include <cuda_runtime.h>

#define BOBA_UNSET 0xFFFFFFFFu

namespace boba {

__device__ __forceinline__ unsigned lane_id() {
    unsigned r;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// 64-bit relaxed/volatile accessors for lookback status words (flag and
// value live in one word, so no acquire/release pairing is needed for them).
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_volatile_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u32(unsigned* p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_sum(T x) {
    const unsigned lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= (unsigned)o) x += y;
    }
    return x;
}
template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
    return x;
}

// Block-wide exclusive sum for NT threads (NT multiple of 32, <= 1024).
// `scratch` must hold NT/32 + 1 elements; returns the block total in *total.
template <int NT, typename T>
__device__ __forceinline__ T block_exclusive_sum(T x, T* scratch, T* total) {
    constexpr int NW = NT / 32;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    T inc = warp_inclusive_sum(x);
    if (lane == 31) scratch[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = lane < NW ? scratch[lane] : T(0);
        T wi = warp_inclusive_sum(w);
        if (lane < NW) scratch[lane] = wi - w;
        if (lane == NW - 1) scratch[NW] = wi;
    }
    __syncthreads();
    T res = scratch[warp] + inc - x;
    *total = scratch[NW];
    __syncthreads();
    return res;
}

// ---------------------------------------------------------------------------
// Decoupled lookback (single-pass chained scan).  Each tile publishes a
// 64-bit status word: [63:62] flag (0 invalid, 1 aggregate, 2 inclusive),
// [61:0] value.  Tiles take their index from an atomic counter so that every
// predecessor of a tile has already been scheduled (forward progress).
// ---------------------------------------------------------------------------
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagInc = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

// Called by ONE full warp of the tile.  Returns the exclusive prefix of the
// tile (sum of values of all tiles before `tile`).
__device__ __forceinline__ unsigned long long warp_lookback(const unsigned long long* status,
                                                            long long tile) {
    const unsigned lane = lane_id();
    unsigned long long excl = 0;
    long long base = tile - 1;
    while (base >= 0) {
        long long idx = base - (long long)lane;
        unsigned long long s = idx >= 0 ? ld_volatile_u64(status + idx) : kFlagInc;
        unsigned flag = (unsigned)(s >> 62);
        if (__any_sync(0xFFFFFFFFu, flag == 0)) continue;  // a predecessor not yet published
        unsigned inc = __ballot_sync(0xFFFFFFFFu, flag == 2);
        int stop = inc ? __ffs(inc) - 1 : 31;
        unsigned long long v = ((int)lane <= stop) ? (s & kValMask) : 0ull;
        excl += warp_sum(v);
        if (inc) break;
        base -= 32;
    }
    return excl;
}

// Same protocol, combining with min instead of +: returns the min of the
// values of all tiles before `tile` (kValMask if none).
__device__ __forceinline__ unsigned long long warp_lookback_min(const unsigned long long* status, long long tile) {
    const unsigned lane = lane_id();
    unsigned long long acc = kValMask;
    long long base = tile - 1;
    while (base >= 0) {
        long long idx = base - (long long)lane;
        unsigned long long s = idx >= 0 ? ld_volatile_u64(status + idx) : (kFlagInc | kValMask);
        unsigned flag = (unsigned)(s >> 62);
        if (__any_sync(0xFFFFFFFFu, flag == 0)) continue;
        unsigned inc = __ballot_sync(0xFFFFFFFFu, flag == 2);
        int stop = inc ? __ffs(inc) - 1 : 31;
        unsigned long long v = ((int)lane <= stop) ? (s & kValMask) : kValMask;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            unsigned long long u = __shfl_xor_sync(0xFFFFFFFFu, v, o);
            v = u < v ? u : v;
        }
        acc = v < acc ? v : acc;
        if (inc) break;
        base -= 32;
    }
    return acc;
}

__host__ __device__ inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// Kernel attributes (dynamic shared memory limit, carveout) belong to the
// device's context: a call site sets them once per device, tracked here.  The
// device's bit is set only after the attribute call succeeded, under a lock, so
// a second host thread never launches before the attribute is in place and a
// failed call is retried next time.
struct PerDeviceOnce {
    std::mutex mu;
    std::atomic<unsigned long long> done{0};
    template <typename F>
    cudaError_t run(F&& set) {
        int d = 0;
        cudaGetDevice(&d);
        if (d >= 64) return set();  // devices >= 64: no cache, set every time
        const unsigned long long bit = 1ull << d;
        if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
        std::lock_guard<std::mutex> lock(mu);
        if (done.load(std::memory_order_relaxed) & bit) return cudaSuccess;
        const cudaError_t e = set();
        if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
        return e;
    }
};

template <typename K>
inline cudaError_t set_attr_once(PerDeviceOnce& once, K* kernel, cudaFuncAttribute a, int v) {
    return once.run([&] { return cudaFuncSetAttribute(kernel, a, v); });
}

}  // namespace boba
