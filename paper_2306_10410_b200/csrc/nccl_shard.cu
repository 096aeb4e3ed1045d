// The multi-GPU pipeline behind one C-ABI call that takes
// the caller's ncclComm_t: the same sequence sharded.py drives through
// torch.distributed, issued here on one stream with NCCL directly.
//
//   P1  boba first occurrence of the shard (global positions), allreduce-MIN
//       of the biased array (_parallel.py:139-162's exact chunk merge)
//   P2  windowed compaction: counts allgather, partial labels, allreduce-SUM
//       (_parallel.py:178-201), order = inverse of label
//   P3  relabel of the shard with the hub table (graph.py:280-289)
//   P4  coarse row histogram allreduce-SUM, row cut, stable relative range
//       partition, all-to-all of the rows and then of the columns by grouped
//       send/recv in rank order on a side stream, the owner's first radix
//       histogram of the rows overlapping the column exchange, its stable
//       COO->CSR (graph.py:253-277)
// One host synchronisation per call (the row bounds and the send / receive
// counts the grouped send/recv need).
//
// NCCL is not linked: libnccl.so.2 is looked up at first use, preferring the
// copy already loaded into the process (torch's, whose communicators the
// Python layer passes in), so the communicator and the library always match.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/boba_b200.h"
#include "common.cuh"
#include "hubs.cuh"
#include "kernels.cuh"

namespace boba {
namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    const char* (*error_string)(ncclResult_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*comm_user_rank)(const ncclComm_t, int*) = nullptr;
};

template <typename F>
bool sym(void* h, const char* name, F& fn) {
    fn = reinterpret_cast<F>(dlsym(h, name));
    return fn != nullptr;
}

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("libnccl.so.2 not found: ") + dlerror();
            return;
        }
        api.ok = sym(h, "ncclGetErrorString", api.error_string) && sym(h, "ncclAllReduce", api.all_reduce) &&
                 sym(h, "ncclAllGather", api.all_gather) && sym(h, "ncclSend", api.send) &&
                 sym(h, "ncclRecv", api.recv) && sym(h, "ncclGroupStart", api.group_start) &&
                 sym(h, "ncclGroupEnd", api.group_end) && sym(h, "ncclCommCount", api.comm_count) &&
                 sym(h, "ncclCommUserRank", api.comm_user_rank);
        if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    });
    return api;
}

size_t a256(size_t b) { return (b + 255) & ~size_t(255); }

struct ShardWs {
    void* fh;  // first occurrence (SeenSet + wave bitmaps)
    uint32_t *key, *counts, *all_counts, *hist_l, *hist_g, *cut, *recvc, *keys, *vals, *rk, *rv;
    void* cw;  // window compaction
    void* hubs;
    void* pw;  // range partition
    void* csr; // owner's COO->CSR
    size_t cw_bytes, pw_bytes, csr_bytes, total;
};

ShardWs carve_shard(void* base, uint64_t ml, uint32_t n, int P, uint64_t cap) {
    ShardWs w{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += a256(bytes);
        return base ? static_cast<char*>(base) + o : nullptr;
    };
    const uint32_t B = row_cut_buckets(n);
    w.fh = take(a256(first_hit_workspace_bytes()) + first_hit_bits_workspace_bytes(n));
    w.key = (uint32_t*)take((size_t)n * 4 + 4);
    w.cw_bytes = compact_window_workspace_bytes(ml, n);
    w.cw = take(w.cw_bytes);
    w.counts = (uint32_t*)take(8);
    w.all_counts = (uint32_t*)take((size_t)8 * P);
    w.hubs = take(kHubTableBytes);
    w.hist_l = (uint32_t*)take((size_t)B * 4);
    w.hist_g = (uint32_t*)take((size_t)B * 4);
    w.cut = (uint32_t*)take((size_t)(3 * P + 2) * 4);
    w.recvc = (uint32_t*)take((size_t)P * 4);
    w.keys = (uint32_t*)take(ml * 4 + 16);
    w.vals = (uint32_t*)take(ml * 4 + 16);
    w.rk = (uint32_t*)take(cap * 4 + 16);
    w.rv = (uint32_t*)take(cap * 4 + 16);
    w.pw_bytes = range_partition_workspace_bytes(ml, P);
    w.pw = take(w.pw_bytes);
    w.csr_bytes = coo_to_csr_workspace_bytes(cap, n, false);
    w.csr = take(w.csr_bytes);
    w.total = off;
    return w;
}

}  // namespace
}  // namespace boba

extern "C" {

size_t boba_sharded_workspace_size(uint64_t m_local, uint32_t n, int world, uint64_t recv_capacity) {
    return boba::carve_shard(nullptr, m_local, n, world < 1 ? 1 : world, recv_capacity).total;
}

// defined in api.cu
int boba_sharded_fail(int code, const char* what, const char* detail);

int boba_sharded_reorder_to_csr_nccl(const uint32_t* I, const uint32_t* J, uint64_t m_local, uint64_t m_global,
                                     uint64_t e0, uint32_t n, void* comm_ptr, uint32_t* first, uint32_t* order,
                                     uint32_t* label, uint32_t* I2, uint32_t* J2, uint32_t* offsets,
                                     uint32_t* indices, uint64_t recv_capacity, boba_shard_result* out,
                                     uint32_t* bounds_host, void* ws, size_t ws_bytes, void* stream) {
    using namespace boba;
    const char* what = "boba_sharded_reorder_to_csr_nccl";
    const NcclApi& api = nccl();
    if (!api.ok) return boba_sharded_fail(BOBA_ECUDA, what, api.why.c_str());
    if (!comm_ptr || !out || !ws || !first || !order || !label || !offsets)
        return boba_sharded_fail(BOBA_EINVAL, what, "NULL argument");
    if ((!I || !J || !I2 || !J2) && m_local) return boba_sharded_fail(BOBA_EINVAL, what, "NULL edge arrays");
    if (2 * m_global > 0xFFFFFFFEull || e0 + m_local > m_global || n == 0 || n == 0xFFFFFFFFu)
        return boba_sharded_fail(BOBA_EINVAL, what, "sizes outside the uint32 position space");
    ncclComm_t comm = static_cast<ncclComm_t>(comm_ptr);
    int P = 0, r = 0;
    if (api.comm_count(comm, &P) != ncclSuccess || api.comm_user_rank(comm, &r) != ncclSuccess || P < 1 || P > 256)
        return boba_sharded_fail(BOBA_EINVAL, what, "not a usable communicator (1..256 ranks)");
    if (ws_bytes < carve_shard(nullptr, m_local, n, P, recv_capacity).total)
        return boba_sharded_fail(BOBA_EINVAL, what, "workspace too small (boba_sharded_workspace_size)");
    ShardWs W = carve_shard(ws, m_local, n, P, recv_capacity);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int sms = 148;
    {
        int d = 0;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
    }
    const uint32_t B = row_cut_buckets(n);
    cudaError_t e = cudaSuccess;
    ncclResult_t nr = ncclSuccess;
#define CK(x)                                                                                     \
    do {                                                                                          \
        if ((e = (x)) != cudaSuccess) return boba_sharded_fail(BOBA_ECUDA, what, cudaGetErrorString(e)); \
    } while (0)
#define NK(x)                                                                                     \
    do {                                                                                          \
        if ((nr = (x)) != ncclSuccess) return boba_sharded_fail(BOBA_ECUDA, what, api.error_string(nr)); \
    } while (0)
    // P1
    void* bits = static_cast<char*>(W.fh) + a256(first_hit_workspace_bytes());
    CK(launch_first_hit_shard(I, J, m_local, m_global, e0, n, first, false, W.fh, sms, s, bits));
    CK(launch_bias(first, n, W.key, sms, s));
    NK(api.all_reduce(W.key, W.key, n, ncclInt32, ncclMin, comm, s));
    CK(launch_bias(W.key, n, first, sms, s));
    // P2
    CK(launch_compact_window_mark(first, n, m_global, e0, m_local, W.counts, W.cw, W.cw_bytes, sms, s));
    NK(api.all_gather(W.counts, W.all_counts, 2, ncclUint32, comm, s));
    CK(launch_compact_window_assign(first, n, m_global, e0, m_local, W.all_counts, P, r, label, W.cw, W.cw_bytes,
                                    s));
    NK(api.all_reduce(label, label, n, ncclUint32, ncclSum, comm, s));
    CK(launch_order_from_label(label, n, order, static_cast<unsigned long long*>(W.hubs), sms, s));
    // P3
    CK(launch_relabel(I, J, m_local, label, static_cast<const unsigned long long*>(W.hubs), I2, J2, nullptr, n, sms,
                      s));
    // P4: row cut
    CK(launch_coarse_hist(I2, m_local, n, W.hist_l, sms, s));
    NK(api.all_reduce(W.hist_l, W.hist_g, B, ncclUint32, ncclSum, comm, s));
    CK(launch_row_cut(W.hist_g, W.hist_l, n, m_global, P, W.cut, s));
    NK(api.group_start());
    for (int k = 0; k < P; k++) {
        NK(api.send(W.cut + 2 * P + 2 + k, 1, ncclUint32, k, comm, s));
        NK(api.recv(W.recvc + k, 1, ncclUint32, k, comm, s));
    }
    NK(api.group_end());
    // the partition needs only the device-side bounds: queue it before the host sync
    // (one rank: the shard already is the owner's edges in edge order)
    if (m_local && P > 1)
        CK(launch_range_partition(I2, J2, m_local, W.cut, P, W.keys, W.vals, nullptr, W.pw, W.pw_bytes, sms, s,
                                  true));
    std::vector<uint32_t> h(4 * P + 2);
    CK(cudaMemcpyAsync(h.data(), W.cut, (3 * P + 2) * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h.data() + 3 * P + 2, W.recvc, P * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const uint32_t* bounds = h.data();
    const uint32_t* goff = h.data() + P + 1;
    const uint32_t* sent = h.data() + 2 * P + 2;
    const uint32_t* recvd = h.data() + 3 * P + 2;
    uint64_t total = 0;
    for (int k = 0; k < P; k++) total += recvd[k];
    out->row_lo = bounds[r];
    out->row_hi = bounds[r + 1];
    out->nnz = total;
    out->row_edge_offset = goff[r];
    if (bounds_host)
        for (int k = 0; k <= P; k++) bounds_host[k] = bounds[k];
    if (total > recv_capacity)
        return boba_sharded_fail(BOBA_EINVAL, what, "recv_capacity too small (out->nnz holds the need)");
    // all-to-all of rows, then of columns, in rank order, on a side stream:
    // the owner histograms the rows for its first radix pass while the
    // columns are still in flight
    const uint32_t rows = out->row_hi - out->row_lo;
    const uint32_t* ck = W.rk;
    const uint32_t* cv = W.rv;
    bool hist_ready = false;
    if (P == 1) {
        ck = I2;
        cv = J2;
    } else {
        cudaStream_t cs = nullptr;
        cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};  // partition done, rows in, columns in
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        struct Release {
            cudaStream_t& cs;
            cudaEvent_t* ev;
            ~Release() {
                for (int i = 0; i < 3; i++)
                    if (ev[i]) cudaEventDestroy(ev[i]);
                if (cs) cudaStreamDestroy(cs);
            }
        } release{cs, ev};
        for (auto& evt : ev) CK(cudaEventCreateWithFlags(&evt, cudaEventDisableTiming));
        CK(cudaEventRecord(ev[0], s));
        CK(cudaStreamWaitEvent(cs, ev[0], 0));
        for (int pass = 0; pass < 2; pass++) {
            const uint32_t* src = pass == 0 ? W.keys : W.vals;
            uint32_t* dst = pass == 0 ? W.rk : W.rv;
            NK(api.group_start());
            uint64_t so = 0, ro = 0;
            for (int k = 0; k < P; k++) {
                if (sent[k]) NK(api.send(src + so, sent[k], ncclUint32, k, comm, cs));
                if (recvd[k]) NK(api.recv(dst + ro, recvd[k], ncclUint32, k, comm, cs));
                so += sent[k];
                ro += recvd[k];
            }
            NK(api.group_end());
            CK(cudaEventRecord(ev[1 + pass], cs));
        }
        CK(cudaStreamWaitEvent(s, ev[1], 0));
        CK(launch_coo_to_csr_first_hist(W.rk, total, rows, W.csr, W.csr_bytes, sms, s));
        CK(cudaStreamWaitEvent(s, ev[2], 0));
        hist_ready = true;
    }
    // the owner's stable CSR over rows [row_lo, row_hi) (keys arrive relative to row_lo)
    CK(launch_coo_to_csr(ck, cv, nullptr, total, rows, nullptr, offsets, indices, nullptr, W.csr, W.csr_bytes, sms,
                         s, hist_ready));
#undef CK
#undef NK
    return BOBA_OK;
}

}  // extern "C"
