// Host <-> device id transfers for the reference-shaped (int64 numpy) API.
//
// The reference keeps ids as int64 on the host (graph.py:31); the kernels use
// uint32.  Narrowing on the host halves the PCIe bytes, so each transfer is
// chunked through two pinned staging slots:
//   h2d: host threads narrow chunk k (int64 -> uint32, with the reference's
//        [0, bound) range check, graph.py:99-106) into slot k%2 while chunk
//        k-1's copy runs; the caller's stream gets one async copy per chunk.
//   d2h: chunk k+1's copy runs while host threads widen chunk k into the
//        caller's int64 array.
// Staging is allocated once per device and process (2 x 64 MB pinned) and
// guarded by a mutex, so concurrent callers serialise on it.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <sched.h>

namespace boba {
namespace {

constexpr size_t kChunkIds = size_t(16) << 20;  // 16M ids = 64 MB of uint32 per slot

struct Staging {
    std::mutex mu;
    uint32_t* slot[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    bool ready = false;
};

Staging g_staging[64];

cudaError_t staging_for_device(Staging*& out) {
    int d = 0;
    cudaError_t e = cudaGetDevice(&d);
    if (e != cudaSuccess) return e;
    if (d >= 64) return cudaErrorInvalidDevice;
    out = &g_staging[d];
    return cudaSuccess;
}

cudaError_t ensure(Staging& st) {
    if (st.ready) return cudaSuccess;
    for (int k = 0; k < 2; k++) {
        cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&st.slot[k]), kChunkIds * 4, cudaHostAllocPortable);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&st.done[k], cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    }
    st.ready = true;
    return cudaSuccess;
}

int host_threads() {
    cpu_set_t set;
    int n = 0;
    if (sched_getaffinity(0, sizeof set, &set) == 0) n = CPU_COUNT(&set);
    if (n <= 0) n = (int)std::thread::hardware_concurrency();
    return std::max(1, std::min(n, 32));
}

// fn(lo, hi) over [0, count) split across host threads
template <typename F>
void parallel_for(size_t count, F&& fn) {
    const int T = count < (size_t(1) << 16) ? 1 : host_threads();
    if (T == 1) {
        fn(size_t(0), count);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(T);
    const size_t per = (count + T - 1) / T;
    for (int t = 0; t < T; t++) {
        const size_t lo = std::min(count, t * per), hi = std::min(count, lo + per);
        if (lo < hi) th.emplace_back([&fn, lo, hi] { fn(lo, hi); });
    }
    for (auto& x : th) x.join();
}

}  // namespace

// returns cudaSuccess; *bad = index of the first id outside [0, bound) or -1
cudaError_t host_h2d_ids(const int64_t* host, uint64_t count, uint64_t bound, uint32_t* dev, int64_t* bad,
                         cudaStream_t s) {
    *bad = -1;
    if (count == 0) return cudaSuccess;
    Staging* st = nullptr;
    cudaError_t e = staging_for_device(st);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(st->mu);
    if ((e = ensure(*st)) != cudaSuccess) return e;
    std::atomic<int64_t> first_bad{INT64_MAX};
    for (uint64_t c0 = 0, k = 0; c0 < count; c0 += kChunkIds, k++) {
        const uint64_t len = std::min<uint64_t>(kChunkIds, count - c0);
        uint32_t* buf = st->slot[k & 1];
        if (k >= 2 && (e = cudaEventSynchronize(st->done[k & 1])) != cudaSuccess) return e;
        parallel_for(len, [&](size_t lo, size_t hi) {
            const int64_t* src = host + c0;
            int64_t badi = INT64_MAX;
            for (size_t i = lo; i < hi; i++) {
                const int64_t v = src[i];
                if ((uint64_t)v >= bound && badi == INT64_MAX) badi = (int64_t)(c0 + i);
                buf[i] = (uint32_t)v;
            }
            if (badi != INT64_MAX) {
                int64_t cur = first_bad.load();
                while (badi < cur && !first_bad.compare_exchange_weak(cur, badi)) {
                }
            }
        });
        if ((e = cudaMemcpyAsync(dev + c0, buf, len * 4, cudaMemcpyHostToDevice, s)) != cudaSuccess) return e;
        if ((e = cudaEventRecord(st->done[k & 1], s)) != cudaSuccess) return e;
    }
    // the slots are reused by the next call; the copies must have drained
    for (int k = 0; k < 2; k++)
        if ((e = cudaEventSynchronize(st->done[k])) != cudaSuccess) return e;
    if (first_bad.load() != INT64_MAX) *bad = first_bad.load();
    return cudaSuccess;
}

// unset_to_max: 0xFFFFFFFF widens to INT64_MAX (the reference's RANK_UNSET)
cudaError_t host_d2h_ids(const uint32_t* dev, uint64_t count, int64_t* host, cudaStream_t s, bool unset_to_max) {
    if (count == 0) return cudaSuccess;
    Staging* st = nullptr;
    cudaError_t e = staging_for_device(st);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(st->mu);
    if ((e = ensure(*st)) != cudaSuccess) return e;
    const uint64_t chunks = (count + kChunkIds - 1) / kChunkIds;
    auto issue = [&](uint64_t k) -> cudaError_t {
        const uint64_t c0 = k * kChunkIds, len = std::min<uint64_t>(kChunkIds, count - c0);
        cudaError_t r = cudaMemcpyAsync(st->slot[k & 1], dev + c0, len * 4, cudaMemcpyDeviceToHost, s);
        if (r == cudaSuccess) r = cudaEventRecord(st->done[k & 1], s);
        return r;
    };
    if ((e = issue(0)) != cudaSuccess) return e;
    for (uint64_t k = 0; k < chunks; k++) {
        if ((e = cudaEventSynchronize(st->done[k & 1])) != cudaSuccess) return e;
        if (k + 1 < chunks && (e = issue(k + 1)) != cudaSuccess) return e;
        const uint64_t c0 = k * kChunkIds, len = std::min<uint64_t>(kChunkIds, count - c0);
        const uint32_t* buf = st->slot[k & 1];
        parallel_for(len, [&](size_t lo, size_t hi) {
            int64_t* dst = host + c0;
            if (unset_to_max)
                for (size_t i = lo; i < hi; i++) dst[i] = buf[i] == 0xFFFFFFFFu ? INT64_MAX : (int64_t)buf[i];
            else
                for (size_t i = lo; i < hi; i++) dst[i] = (int64_t)buf[i];
        });
    }
    return cudaSuccess;
}

}  // namespace boba
