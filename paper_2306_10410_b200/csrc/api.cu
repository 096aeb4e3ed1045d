// extern "C" boundary of libboba_b200.so -- see include/boba_b200.h for the
// contract and the reference interface each entry point replaces.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/boba_b200.h"
#include "common.cuh"
#include "hubs.cuh"
#include "kernels.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return BOBA_OK;
    if (e == cudaErrorInvalidValue) return fail(BOBA_EINVAL, "%s: invalid value (workspace too small?)", what);
    return fail(BOBA_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

int num_sms() {
    static thread_local int dev = -1, sms = 148;
    int d = 0;
    cudaGetDevice(&d);
    if (d != dev) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
        dev = d;
    }
    return sms;
}

inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

int check_sizes(uint64_t m, uint32_t n, const char* what) {
    if (2 * m > 0xFFFFFFFEull) return fail(BOBA_EINVAL, "%s: 2m = %llu exceeds the uint32 position space", what,
                                           (unsigned long long)(2 * m));
    if (n == 0xFFFFFFFFu) return fail(BOBA_EINVAL, "%s: n must be < 2^32 - 1", what);
    return BOBA_OK;
}

#define REQUIRE(cond, ...)                                  \
    do {                                                    \
        if (!(cond)) return fail(BOBA_EINVAL, __VA_ARGS__); \
    } while (0)

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// Makes `device` current for the scope and restores the caller's device.
struct DeviceGuard {
    int saved = -1;
    explicit DeviceGuard(int device) {
        if (cudaGetDevice(&saved) != cudaSuccess) saved = -1;
        if (saved != device) cudaSetDevice(device);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (saved >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != saved) cudaSetDevice(saved);
    }
};

// SpMV partitions kept in a caller's workspace: which CSR each workspace was
// last partitioned for, so reuse_partition = 1 with a workspace that holds
// another matrix's partition (or none) is an error instead of a wrong walk.
struct SpmvKey {
    const void* offsets;
    const void* indices;
    uint32_t n;
    uint64_t m;
    bool operator==(const SpmvKey& o) const {
        return offsets == o.offsets && indices == o.indices && n == o.n && m == o.m;
    }
};
std::mutex g_spmv_mu;
std::unordered_map<const void*, SpmvKey> g_spmv_parts;

bool spmv_partition_ok(const void* ws, const SpmvKey& k, bool reuse) {
    std::lock_guard<std::mutex> lock(g_spmv_mu);
    if (!reuse) {
        g_spmv_parts[ws] = k;
        return true;
    }
    auto it = g_spmv_parts.find(ws);
    return it != g_spmv_parts.end() && it->second == k;
}

}  // namespace

// Captured pipelines: one fused reorder->CSR call on fixed buffers recorded
// into a CUDA graph, so a repeated step costs one graph launch instead of
// ~21 kernel launches and their gaps.
struct boba_graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    uint64_t body_kernels = 0;  // kernels inside the taken branch of conditional nodes
};

// Host-buffer contexts: two buffer slots so that consecutive graphs overlap
// (H2D of graph k+1 and D2H of graph k run on their own copy streams while
// the compute stream works); the compute-internal arrays (first, I2, J2,
// workspace) are shared because the compute stream serialises the graphs.
struct boba_slot {
    uint32_t *I = nullptr, *J = nullptr, *order = nullptr, *label = nullptr, *offsets = nullptr,
             *indices = nullptr;
    cudaEvent_t h2d_done = nullptr, labels_done = nullptr, compute_done = nullptr, d2h_done = nullptr;
    bool used = false;
};

struct boba_ctx {
    int device = 0;
    uint64_t max_m = 0;
    uint32_t max_n = 0;
    cudaStream_t stream = nullptr;  // compute
    cudaStream_t h2d = nullptr, d2h = nullptr;
    boba_slot slot[2];
    uint32_t *I2 = nullptr, *J2 = nullptr, *first = nullptr;
    void* ws = nullptr;
    size_t ws_bytes = 0;
    uint64_t submitted = 0;
};

extern "C" {

int boba_abi_version(void) { return 1; }

int boba_sharded_fail(int code, const char* what, const char* detail) { return fail(code, "%s: %s", what, detail); }
const char* boba_last_error(void) { return g_err.c_str(); }

int boba_first_occurrence(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n, uint32_t* first,
                          int relaxed, void* stream) {
    if (int rc = check_sizes(m, n, "boba_first_occurrence")) return rc;
    REQUIRE(first || n == 0, "boba_first_occurrence: first is NULL");
    REQUIRE((I && J) || m == 0, "boba_first_occurrence: I/J is NULL");
    if (n == 0) return BOBA_OK;
    return cuda_status(boba::launch_first_hit(I, J, m, n, first, relaxed != 0, num_sms(), S(stream)),
                       "boba_first_occurrence");
}

size_t boba_first_occurrence_workspace_size(void) { return boba::first_hit_workspace_bytes(); }

size_t boba_first_occurrence_shard_workspace_size(uint32_t n) {
    return align256(boba::first_hit_workspace_bytes()) + boba::first_hit_bits_workspace_bytes(n);
}

int boba_first_occurrence_shard(const uint32_t* I, const uint32_t* J, uint64_t m_local, uint64_t m_global,
                                uint64_t e0, uint32_t n, uint32_t* first, int relaxed, void* ws, size_t ws_bytes,
                                void* stream) {
    REQUIRE(!ws || ws_bytes >= boba::first_hit_workspace_bytes(), "boba_first_occurrence_shard: workspace too small");
    if (int rc = check_sizes(m_global, n, "boba_first_occurrence_shard")) return rc;
    REQUIRE(e0 + m_local <= m_global, "boba_first_occurrence_shard: shard [e0, e0+m_local) outside [0, m_global)");
    REQUIRE(first || n == 0, "boba_first_occurrence_shard: first is NULL");
    REQUIRE((I && J) || m_local == 0, "boba_first_occurrence_shard: I/J is NULL");
    if (n == 0) return BOBA_OK;
    void* bits_ws = nullptr;
    if (ws && ws_bytes >= boba_first_occurrence_shard_workspace_size(n))
        bits_ws = static_cast<char*>(ws) + align256(boba::first_hit_workspace_bytes());
    return cuda_status(boba::launch_first_hit_shard(I, J, m_local, m_global, e0, n, first, relaxed != 0, ws,
                                                    num_sms(), S(stream), bits_ws),
                       "boba_first_occurrence_shard");
}

size_t boba_compact_workspace_size(uint64_t m, uint32_t n) { return boba::compact_workspace_bytes(m, n); }

int boba_compact(const uint32_t* first, uint64_t m, uint32_t n, uint32_t* order, uint32_t* label,
                 uint32_t* n_seen, void* ws, size_t ws_bytes, void* stream) {
    if (int rc = check_sizes(m, n, "boba_compact")) return rc;
    if (n == 0) return BOBA_OK;
    REQUIRE(first && order && label && ws, "boba_compact: NULL argument");
    return cuda_status(boba::launch_compact(first, m, n, order, label, n_seen, nullptr, ws, ws_bytes, num_sms(), S(stream)),
                       "boba_compact");
}

size_t boba_order_workspace_size(uint64_t m, uint32_t n) { return boba::compact_workspace_bytes(m, n); }

int boba_order(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n, int relaxed, uint32_t* first,
               uint32_t* order, uint32_t* label, void* ws, size_t ws_bytes, void* stream) {
    if (int rc = boba_first_occurrence(I, J, m, n, first, relaxed, stream)) return rc;
    return boba_compact(first, m, n, order, label, nullptr, ws, ws_bytes, stream);
}

size_t boba_compact_relabel_workspace_size(uint64_t m_global, uint32_t n) {
    return align256(boba::kHubTableBytes) + boba::compact_workspace_bytes(m_global, n);
}

int boba_compact_relabel(const uint32_t* first, uint64_t m_global, uint32_t n, const uint32_t* I, const uint32_t* J,
                         uint64_t m, uint32_t* order, uint32_t* label, uint32_t* I2, uint32_t* J2, void* ws,
                         size_t ws_bytes, void* stream) {
    if (int rc = check_sizes(m_global, n, "boba_compact_relabel")) return rc;
    if (n == 0) return BOBA_OK;
    REQUIRE(m <= m_global, "boba_compact_relabel: shard larger than the graph");
    REQUIRE(first && order && label && ws, "boba_compact_relabel: NULL argument");
    REQUIRE((I && J && I2 && J2) || m == 0, "boba_compact_relabel: NULL edge arrays");
    REQUIRE(ws_bytes >= boba_compact_relabel_workspace_size(m_global, n), "boba_compact_relabel: workspace too small");
    auto* hubs = static_cast<unsigned long long*>(ws);
    void* rest = static_cast<char*>(ws) + align256(boba::kHubTableBytes);
    const size_t rest_bytes = ws_bytes - align256(boba::kHubTableBytes);
    cudaError_t e = boba::launch_compact(first, m_global, n, order, label, nullptr, hubs, rest, rest_bytes, num_sms(),
                                         S(stream));
    if (e == cudaSuccess) e = boba::launch_relabel(I, J, m, label, hubs, I2, J2, nullptr, n, num_sms(), S(stream));
    return cuda_status(e, "boba_compact_relabel");
}

int boba_relabel(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n, const uint32_t* label, uint32_t* I2,
                 uint32_t* J2, uint32_t* row_counts, void* stream) {
    if (int rc = check_sizes(m, n, "boba_relabel")) return rc;
    REQUIRE((I && J && I2 && J2 && label) || m == 0, "boba_relabel: NULL argument");
    return cuda_status(boba::launch_relabel(I, J, m, label, nullptr, I2, J2, row_counts, n, num_sms(), S(stream)),
                       "boba_relabel");
}

int boba_degrees(const uint32_t* I, uint64_t m, uint32_t n, uint32_t* deg, void* stream) {
    if (int rc = check_sizes(m, n, "boba_degrees")) return rc;
    if (n == 0) return BOBA_OK;
    REQUIRE(deg && (I || m == 0), "boba_degrees: NULL argument");
    return cuda_status(boba::launch_hist(I, m, n, deg, num_sms(), S(stream)), "boba_degrees");
}

size_t boba_coo_to_csr_workspace_size(uint64_t m, uint32_t n, int weighted) {
    return boba::coo_to_csr_workspace_bytes(m, n, weighted != 0);
}

int boba_coo_to_csr_ex(const uint32_t* I2, const uint32_t* J2, const double* w, uint64_t m, uint32_t n,
                       const uint32_t* row_counts, uint32_t* offsets, uint32_t* indices, double* w_out, void* ws,
                       size_t ws_bytes, int first_hist_ready, void* stream) {
    if (int rc = check_sizes(m, n, "boba_coo_to_csr")) return rc;
    REQUIRE(offsets && ws, "boba_coo_to_csr: NULL offsets/workspace");
    REQUIRE((I2 && J2 && indices) || m == 0, "boba_coo_to_csr: NULL edge arrays");
    REQUIRE(!w || w_out || m == 0, "boba_coo_to_csr: weights given but weights_out is NULL");
    REQUIRE(!first_hist_ready || !row_counts, "boba_coo_to_csr_ex: first_hist_ready with row_counts");
    return cuda_status(boba::launch_coo_to_csr(I2, J2, w, m, n, row_counts, offsets, indices, w_out, ws, ws_bytes,
                                               num_sms(), S(stream), first_hist_ready != 0),
                       "boba_coo_to_csr");
}

int boba_coo_to_csr(const uint32_t* I2, const uint32_t* J2, const double* w, uint64_t m, uint32_t n,
                    const uint32_t* row_counts, uint32_t* offsets, uint32_t* indices, double* w_out, void* ws,
                    size_t ws_bytes, void* stream) {
    return boba_coo_to_csr_ex(I2, J2, w, m, n, row_counts, offsets, indices, w_out, ws, ws_bytes, 0, stream);
}

int boba_coo_to_csr_first_hist(const uint32_t* I2, uint64_t m, uint32_t n, void* ws, size_t ws_bytes, void* stream) {
    if (int rc = check_sizes(m, n, "boba_coo_to_csr_first_hist")) return rc;
    REQUIRE(ws, "boba_coo_to_csr_first_hist: NULL workspace");
    REQUIRE(I2 || m == 0, "boba_coo_to_csr_first_hist: NULL rows");
    REQUIRE(ws_bytes >= boba::coo_to_csr_workspace_bytes(m, n, false), "boba_coo_to_csr_first_hist: workspace too small");
    return cuda_status(boba::launch_coo_to_csr_first_hist(I2, m, n, ws, ws_bytes, num_sms(), S(stream)),
                       "boba_coo_to_csr_first_hist");
}

size_t boba_spmv_workspace_size(uint32_t n, uint64_t m) { return boba::spmv_workspace_bytes(n, m); }

int boba_spmv_ex(const uint32_t* offsets, const uint32_t* indices, const float* w, const float* x, float* y,
                 uint32_t n, uint64_t m, void* ws, size_t ws_bytes, int reuse_partition, void* stream) {
    if (n == 0) return BOBA_OK;
    REQUIRE(offsets && x && y && ws && (indices || m == 0), "boba_spmv: NULL argument");
    REQUIRE((uint64_t)n + m < 0xFFFFFFFFull * 1024ull, "boba_spmv: too large");
    REQUIRE(spmv_partition_ok(ws, SpmvKey{offsets, indices, n, m}, reuse_partition != 0),
            "boba_spmv: reuse_partition = 1 but this workspace was not partitioned for this CSR");
    return cuda_status(boba::launch_spmv(offsets, indices, w, x, y, n, m, ws, ws_bytes, S(stream), reuse_partition != 0),
                       "boba_spmv");
}

int boba_spmv(const uint32_t* offsets, const uint32_t* indices, const float* w, const float* x, float* y, uint32_t n,
              uint64_t m, void* ws, size_t ws_bytes, void* stream) {
    return boba_spmv_ex(offsets, indices, w, x, y, n, m, ws, ws_bytes, 0, stream);
}

int boba_spmv_f64_ex(const uint32_t* offsets, const uint32_t* indices, const double* w, const double* x, double* y,
                     uint32_t n, uint64_t m, void* ws, size_t ws_bytes, int reuse_partition, void* stream) {
    if (n == 0) return BOBA_OK;
    REQUIRE(offsets && x && y && ws && (indices || m == 0), "boba_spmv_f64: NULL argument");
    REQUIRE((uint64_t)n + m < 0xFFFFFFFFull * 1024ull, "boba_spmv_f64: too large");
    REQUIRE(spmv_partition_ok(ws, SpmvKey{offsets, indices, n, m}, reuse_partition != 0),
            "boba_spmv_f64: reuse_partition = 1 but this workspace was not partitioned for this CSR");
    return cuda_status(
        boba::launch_spmv_f64(offsets, indices, w, x, y, n, m, ws, ws_bytes, S(stream), reuse_partition != 0),
        "boba_spmv_f64");
}

int boba_spmv_f64(const uint32_t* offsets, const uint32_t* indices, const double* w, const double* x, double* y,
                  uint32_t n, uint64_t m, void* ws, size_t ws_bytes, void* stream) {
    return boba_spmv_f64_ex(offsets, indices, w, x, y, n, m, ws, ws_bytes, 0, stream);
}

size_t boba_reorder_to_csr_workspace_size(uint64_t m, uint32_t n, int weighted) {
    size_t a = boba::compact_workspace_bytes(m, n);
    size_t b = boba::coo_to_csr_workspace_bytes(m, n, weighted != 0);
    return align256((size_t)n * 4 + 4) + align256(boba::kHubTableBytes) + (a > b ? a : b);
}

int boba_reorder_to_csr_timed(const uint32_t* I, const uint32_t* J, const double* w, uint64_t m, uint32_t n,
                              uint32_t* first, uint32_t* order, uint32_t* label, uint32_t* I2, uint32_t* J2,
                              uint32_t* offsets, uint32_t* indices, double* w_out, void* ws, size_t ws_bytes,
                              void* stream, void* const* events) {
    if (int rc = check_sizes(m, n, "boba_reorder_to_csr")) return rc;
    REQUIRE(ws && ws_bytes >= boba_reorder_to_csr_workspace_size(m, n, w != nullptr),
            "boba_reorder_to_csr: workspace too small");
    REQUIRE(first && order && label && offsets, "boba_reorder_to_csr: NULL output");
    REQUIRE((I && J && I2 && J2 && indices) || m == 0, "boba_reorder_to_csr: NULL edge arrays");
    REQUIRE(!w || w_out || m == 0, "boba_reorder_to_csr: weights given but weights_out is NULL");
    if (n == 0) return BOBA_OK;
    cudaStream_t s = S(stream);
    // under stream capture a plain record would only order the capture:
    // record external events so each graph replay records them
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    const bool capturing = events && cudaStreamIsCapturing(s, &cst) == cudaSuccess &&
                           cst == cudaStreamCaptureStatusActive;
    auto mark = [&](int i) {
        if (events && events[i])
            cudaEventRecordWithFlags(static_cast<cudaEvent_t>(events[i]), s,
                                     capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
    };
    char* base = static_cast<char*>(ws);
    uint32_t* counts = reinterpret_cast<uint32_t*>(base);
    base += align256((size_t)n * 4 + 4);
    unsigned long long* hubs = reinterpret_cast<unsigned long long*>(base);
    base += align256(boba::kHubTableBytes);
    void* rest = base;
    size_t rest_bytes = ws_bytes - (size_t)(base - static_cast<char*>(ws));
    const int sms = num_sms();
    mark(0);
    // the hub table area doubles as phase 1's SeenSet (dead before phase 2 refills it)
    // the compaction workspace (`rest`, >= 2m bits) is idle during phase 1: it holds the wave bitmaps
    void* bits_ws = rest_bytes >= boba::first_hit_bits_workspace_bytes(n) ? rest : nullptr;
    cudaError_t e = boba::launch_first_hit_shard(I, J, m, m, 0, n, first, false, hubs, sms, s, bits_ws);
    if (e != cudaSuccess) return cuda_status(e, "boba_reorder_to_csr: first occurrence");
    mark(1);
    // counts[0]: the number of vertices first seen in I, which bounds every CSR row
    e = boba::launch_compact(first, m, n, order, label, nullptr, hubs, rest, rest_bytes, sms, s, counts);
    if (e != cudaSuccess) return cuda_status(e, "boba_reorder_to_csr: compact");
    mark(2);
    // the relabel may also count the first radix digit of its rows (the
    // COO->CSR workspace `rest` is idle until then)
    boba::RowTileHist rh = boba::coo_to_csr_first_hist(rest, rest_bytes, m, n, w != nullptr);
    e = boba::launch_relabel(I, J, m, label, hubs, I2, J2, nullptr, n, sms, s, &rh);
    if (e != cudaSuccess) return cuda_status(e, "boba_reorder_to_csr: relabel");
    mark(3);
    e = boba::launch_coo_to_csr(I2, J2, w, m, n, nullptr, offsets, indices, w_out, rest, rest_bytes, sms, s, rh.done,
                                counts);
    if (e != cudaSuccess) return cuda_status(e, "boba_reorder_to_csr: coo_to_csr");
    mark(4);
    return BOBA_OK;
}

int boba_reorder_to_csr(const uint32_t* I, const uint32_t* J, const double* w, uint64_t m, uint32_t n,
                        uint32_t* first, uint32_t* order, uint32_t* label, uint32_t* I2, uint32_t* J2,
                        uint32_t* offsets, uint32_t* indices, double* w_out, void* ws, size_t ws_bytes,
                        void* stream) {
    return boba_reorder_to_csr_timed(I, J, w, m, n, first, order, label, I2, J2, offsets, indices, w_out, ws,
                                     ws_bytes, stream, nullptr);
}

int boba_reorder_to_csr_graph_create_timed(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n,
                                           uint32_t* first, uint32_t* order, uint32_t* label, uint32_t* I2,
                                           uint32_t* J2, uint32_t* offsets, uint32_t* indices, void* ws,
                                           size_t ws_bytes, void* const* events, boba_graph** out) {
    REQUIRE(out, "boba_reorder_to_csr_graph_create: out is NULL");
    REQUIRE(n >= 2, "boba_reorder_to_csr_graph_create: n must be >= 2 (use boba_reorder_to_csr)");
    // the inputs may still be in flight on any of the caller's streams: the
    // eager run below happens on a private stream, so wait for the device first
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_status(e, "boba_reorder_to_csr_graph_create: pending work");
    cudaStream_t st = nullptr;
    e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_status(e, "boba_reorder_to_csr_graph_create: stream");
    // one eager run first: one-time kernel attribute setup happens outside the capture
    int rc = boba_reorder_to_csr(I, J, nullptr, m, n, first, order, label, I2, J2, offsets, indices, nullptr, ws,
                                 ws_bytes, st);
    if (rc == BOBA_OK) e = cudaStreamSynchronize(st);
    boba_graph* g = new boba_graph();
    if (rc == BOBA_OK && e == cudaSuccess) e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    if (rc == BOBA_OK && e == cudaSuccess) {
        boba::take_conditional_body_kernels();
        rc = boba_reorder_to_csr_timed(I, J, nullptr, m, n, first, order, label, I2, J2, offsets, indices, nullptr, ws,
                                       ws_bytes, st, events);
        g->body_kernels = boba::take_conditional_body_kernels();
        cudaError_t e2 = cudaStreamEndCapture(st, &g->graph);
        if (e == cudaSuccess) e = e2;
    }
    if (rc == BOBA_OK && e == cudaSuccess) e = cudaGraphInstantiate(&g->exec, g->graph, 0);
    cudaStreamDestroy(st);
    if (rc != BOBA_OK || e != cudaSuccess) {
        boba_reorder_to_csr_graph_destroy(g);
        return rc != BOBA_OK ? rc : cuda_status(e, "boba_reorder_to_csr_graph_create: capture");
    }
    *out = g;
    return BOBA_OK;
}

int boba_reorder_to_csr_graph_create(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n, uint32_t* first,
                                     uint32_t* order, uint32_t* label, uint32_t* I2, uint32_t* J2, uint32_t* offsets,
                                     uint32_t* indices, void* ws, size_t ws_bytes, boba_graph** out) {
    return boba_reorder_to_csr_graph_create_timed(I, J, m, n, first, order, label, I2, J2, offsets, indices, ws,
                                                  ws_bytes, nullptr, out);
}

int boba_graph_launch(boba_graph* g, void* stream) {
    REQUIRE(g && g->exec, "boba_graph_launch: NULL graph");
    return cuda_status(cudaGraphLaunch(g->exec, S(stream)), "boba_graph_launch");
}

int boba_graph_kernel_nodes(const boba_graph* g, uint64_t* count) {
    REQUIRE(g && g->graph && count, "boba_graph_kernel_nodes: NULL argument");
    size_t num = 0;
    cudaError_t e = cudaGraphGetNodes(g->graph, nullptr, &num);
    if (e != cudaSuccess) return cuda_status(e, "boba_graph_kernel_nodes");
    std::vector<cudaGraphNode_t> nodes(num);
    if (num) e = cudaGraphGetNodes(g->graph, nodes.data(), &num);
    if (e != cudaSuccess) return cuda_status(e, "boba_graph_kernel_nodes");
    uint64_t k = 0;
    for (size_t i = 0; i < num; i++) {
        cudaGraphNodeType t;
        if (cudaGraphNodeGetType(nodes[i], &t) == cudaSuccess)
            k += t == cudaGraphNodeTypeKernel;
        else
            cudaGetLastError();  // a node type this query does not know (conditional): counted below
    }
    *count = k + g->body_kernels;
    return BOBA_OK;
}

void boba_reorder_to_csr_graph_destroy(boba_graph* g) {
    if (!g) return;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
}

int boba_ctx_create(uint64_t max_m, uint32_t max_n, boba_ctx** out) {
    REQUIRE(out, "boba_ctx_create: out is NULL");
    if (int rc = check_sizes(max_m, max_n, "boba_ctx_create")) return rc;
    boba_ctx* c = new boba_ctx();
    c->max_m = max_m;
    c->max_n = max_n;
    cudaGetDevice(&c->device);
    const size_t mb = max_m * 4 + 16, nb = (size_t)max_n * 4 + 16;
    c->ws_bytes = boba_reorder_to_csr_workspace_size(max_m, max_n, 0);
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking);
    for (boba_slot& S : c->slot) {
        if (e == cudaSuccess) e = cudaMalloc(&S.I, mb);
        if (e == cudaSuccess) e = cudaMalloc(&S.J, mb);
        if (e == cudaSuccess) e = cudaMalloc(&S.indices, mb);
        if (e == cudaSuccess) e = cudaMalloc(&S.order, nb);
        if (e == cudaSuccess) e = cudaMalloc(&S.label, nb);
        if (e == cudaSuccess) e = cudaMalloc(&S.offsets, nb + 4);
        for (cudaEvent_t* ev : {&S.h2d_done, &S.labels_done, &S.compute_done, &S.d2h_done})
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaMalloc(&c->I2, mb);
    if (e == cudaSuccess) e = cudaMalloc(&c->J2, mb);
    if (e == cudaSuccess) e = cudaMalloc(&c->first, nb);
    if (e == cudaSuccess) e = cudaMalloc(&c->ws, c->ws_bytes);
    if (e != cudaSuccess) {
        boba_ctx_destroy(c);
        return fail(BOBA_ENOMEM, "boba_ctx_create: %s", cudaGetErrorString(e));
    }
    *out = c;
    return BOBA_OK;
}

void boba_ctx_destroy(boba_ctx* c) {
    if (!c) return;
    DeviceGuard guard(c->device);
    for (cudaStream_t st : {c->stream, c->h2d, c->d2h})
        if (st) cudaStreamSynchronize(st);
    for (boba_slot& S : c->slot) {
        for (void* p : {(void*)S.I, (void*)S.J, (void*)S.indices, (void*)S.order, (void*)S.label, (void*)S.offsets})
            if (p) cudaFree(p);
        for (cudaEvent_t ev : {S.h2d_done, S.labels_done, S.compute_done, S.d2h_done})
            if (ev) cudaEventDestroy(ev);
    }
    for (void* p : {(void*)c->I2, (void*)c->J2, (void*)c->first, c->ws})
        if (p) cudaFree(p);
    for (cudaStream_t st : {c->stream, c->h2d, c->d2h})
        if (st) cudaStreamDestroy(st);
    delete c;
}

int boba_ctx_submit_host(boba_ctx* c, const uint32_t* I_h, const uint32_t* J_h, uint64_t m, uint32_t n,
                         uint32_t* order_h, uint32_t* label_h, uint32_t* I2_h, uint32_t* J2_h, uint32_t* offsets_h,
                         uint32_t* indices_h, uint64_t* ticket) {
    REQUIRE(c, "boba_ctx_submit_host: NULL context");
    DeviceGuard guard(c->device);
    REQUIRE(m <= c->max_m && n <= c->max_n, "boba_ctx_submit_host: graph exceeds the context capacity");
    REQUIRE(order_h && label_h && offsets_h && (indices_h || m == 0) && ((I_h && J_h) || m == 0),
            "boba_ctx_submit_host: NULL host buffer");
    REQUIRE(n > 0, "boba_ctx_submit_host: n must be positive");
    boba_slot& S = c->slot[c->submitted & 1];
    cudaError_t e = cudaSuccess;
    if (S.used) {
        // the slot's previous graph: its compute must be done reading I, J before
        // they are overwritten, and its D2H done before its outputs are
        e = cudaStreamWaitEvent(c->h2d, S.compute_done, 0);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(c->stream, S.d2h_done, 0);
    }
    if (e == cudaSuccess && m) e = cudaMemcpyAsync(S.I, I_h, m * 4, cudaMemcpyHostToDevice, c->h2d);
    if (e == cudaSuccess && m) e = cudaMemcpyAsync(S.J, J_h, m * 4, cudaMemcpyHostToDevice, c->h2d);
    if (e == cudaSuccess) e = cudaEventRecord(S.h2d_done, c->h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->stream, S.h2d_done, 0);
    if (e != cudaSuccess) return cuda_status(e, "boba_ctx_submit_host: H2D");
    // labels_done is recorded after compaction: order and label go home while
    // relabel and COO->CSR run
    void* evs[5] = {nullptr, nullptr, S.labels_done, nullptr, S.compute_done};
    if (int rc = boba_reorder_to_csr_timed(S.I, S.J, nullptr, m, n, c->first, S.order, S.label, c->I2, c->J2,
                                           S.offsets, S.indices, nullptr, c->ws, c->ws_bytes, c->stream, evs))
        return rc;
    e = cudaStreamWaitEvent(c->d2h, S.labels_done, 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(order_h, S.order, (size_t)n * 4, cudaMemcpyDeviceToHost, c->d2h);
    if (e == cudaSuccess) e = cudaMemcpyAsync(label_h, S.label, (size_t)n * 4, cudaMemcpyDeviceToHost, c->d2h);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->d2h, S.compute_done, 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(offsets_h, S.offsets, ((size_t)n + 1) * 4, cudaMemcpyDeviceToHost, c->d2h);
    if (e == cudaSuccess && m) e = cudaMemcpyAsync(indices_h, S.indices, m * 4, cudaMemcpyDeviceToHost, c->d2h);
    // I2/J2 are shared by both slots: their copies finish before the next compute starts
    if (e == cudaSuccess && I2_h && m) e = cudaMemcpyAsync(I2_h, c->I2, m * 4, cudaMemcpyDeviceToHost, c->d2h);
    if (e == cudaSuccess && J2_h && m) e = cudaMemcpyAsync(J2_h, c->J2, m * 4, cudaMemcpyDeviceToHost, c->d2h);
    if (e == cudaSuccess) e = cudaEventRecord(S.d2h_done, c->d2h);
    if (e == cudaSuccess && (I2_h || J2_h)) e = cudaStreamWaitEvent(c->stream, S.d2h_done, 0);
    if (e != cudaSuccess) return cuda_status(e, "boba_ctx_submit_host: D2H");
    S.used = true;
    if (ticket) *ticket = c->submitted;
    c->submitted++;
    return BOBA_OK;
}

int boba_ctx_wait(boba_ctx* c, uint64_t ticket) {
    REQUIRE(c, "boba_ctx_wait: NULL context");
    DeviceGuard guard(c->device);
    REQUIRE(ticket < c->submitted, "boba_ctx_wait: ticket %llu was never submitted", (unsigned long long)ticket);
    // the slot's d2h_done event is the newest graph in that slot; graphs of a
    // slot complete in submission order, so waiting on it covers `ticket`
    return cuda_status(cudaEventSynchronize(c->slot[ticket & 1].d2h_done), "boba_ctx_wait");
}

int boba_ctx_reorder_to_csr_host(boba_ctx* c, const uint32_t* I_h, const uint32_t* J_h, uint64_t m, uint32_t n,
                                 uint32_t* order_h, uint32_t* label_h, uint32_t* I2_h, uint32_t* J2_h,
                                 uint32_t* offsets_h, uint32_t* indices_h) {
    uint64_t t = 0;
    if (n == 0) return BOBA_OK;
    if (int rc = boba_ctx_submit_host(c, I_h, J_h, m, n, order_h, label_h, I2_h, J2_h, offsets_h, indices_h, &t))
        return rc;
    return boba_ctx_wait(c, t);
}

int boba_narrow_ids(const int64_t* in, uint64_t count, uint64_t bound, uint32_t* out, int64_t* bad_index,
                    void* stream) {
    REQUIRE((in && out) || count == 0, "boba_narrow_ids: NULL argument");
    REQUIRE(bound <= 0xFFFFFFFFull, "boba_narrow_ids: bound exceeds uint32");
    if (count == 0) return BOBA_OK;
    unsigned long long* d_bad = nullptr;
    cudaError_t e = cudaMallocAsync(&d_bad, 8, S(stream));
    if (e == cudaSuccess) e = boba::launch_narrow(in, count, bound, out, d_bad, num_sms(), S(stream));
    unsigned long long h_bad = ~0ull;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h_bad, d_bad, 8, cudaMemcpyDeviceToHost, S(stream));
    if (d_bad) cudaFreeAsync(d_bad, S(stream));
    if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
    if (e != cudaSuccess) return cuda_status(e, "boba_narrow_ids");
    if (h_bad != ~0ull) {
        if (bad_index) *bad_index = (int64_t)h_bad;
        return fail(BOBA_ERANGE, "boba_narrow_ids: element %llu out of range [0, %llu)", h_bad,
                    (unsigned long long)bound);
    }
    return BOBA_OK;
}

int boba_host_to_device_ids(const int64_t* host, uint64_t count, uint64_t bound, uint32_t* dev, int64_t* bad_index,
                            void* stream) {
    REQUIRE((host && dev) || count == 0, "boba_host_to_device_ids: NULL argument");
    REQUIRE(bound <= 0x100000000ull, "boba_host_to_device_ids: bound exceeds uint32");
    int64_t bad = -1;
    if (int rc = cuda_status(boba::host_h2d_ids(host, count, bound, dev, &bad, S(stream)), "boba_host_to_device_ids"))
        return rc;
    if (bad >= 0) {
        if (bad_index) *bad_index = bad;
        return fail(BOBA_ERANGE, "boba_host_to_device_ids: element %lld out of range [0, %llu)", (long long)bad,
                    (unsigned long long)bound);
    }
    return BOBA_OK;
}

int boba_device_to_host_ids(const uint32_t* dev, uint64_t count, int64_t* host, void* stream) {
    REQUIRE((host && dev) || count == 0, "boba_device_to_host_ids: NULL argument");
    return cuda_status(boba::host_d2h_ids(dev, count, host, S(stream)), "boba_device_to_host_ids");
}

int boba_device_to_host_ranks(const uint32_t* dev, uint64_t count, int64_t* host, void* stream) {
    REQUIRE((host && dev) || count == 0, "boba_device_to_host_ranks: NULL argument");
    return cuda_status(boba::host_d2h_ids(dev, count, host, S(stream), true), "boba_device_to_host_ranks");
}

int boba_widen_ids(const uint32_t* in, uint64_t count, int64_t* out, void* stream) {
    REQUIRE((in && out) || count == 0, "boba_widen_ids: NULL argument");
    return cuda_status(boba::launch_widen(in, count, out, num_sms(), S(stream)), "boba_widen_ids");
}

size_t boba_exclusive_scan_workspace_size(uint64_t count) {
    return (boba::ceil_div(count + 1, 2048) + 2) * 8 + 256;
}

int boba_exclusive_scan_u32(const uint32_t* counts, uint32_t n, uint32_t* offsets, void* ws, size_t ws_bytes,
                            void* stream) {
    REQUIRE(offsets && ws && (counts || n == 0), "boba_exclusive_scan_u32: NULL argument");
    REQUIRE(n < 0xFFFFFFFFu, "boba_exclusive_scan_u32: n too large");
    REQUIRE(ws_bytes >= boba_exclusive_scan_workspace_size(n), "boba_exclusive_scan_u32: workspace too small");
    unsigned long long* st = static_cast<unsigned long long*>(ws);
    unsigned* counter = reinterpret_cast<unsigned*>(st + boba::ceil_div((uint64_t)n + 1, 2048) + 1);
    return cuda_status(boba::launch_row_offsets(counts, n, offsets, st, counter, S(stream)),
                       "boba_exclusive_scan_u32");
}

int boba_bias_u32(const uint32_t* in, uint64_t count, uint32_t* out, void* stream) {
    REQUIRE((in && out) || count == 0, "boba_bias_u32: NULL argument");
    return cuda_status(boba::launch_bias(in, count, out, num_sms(), S(stream)), "boba_bias_u32");
}

int boba_offset_ids(const uint32_t* in, uint64_t count, uint32_t delta, uint32_t* out, void* stream) {
    REQUIRE((in && out) || count == 0, "boba_offset_ids: NULL argument");
    return cuda_status(boba::launch_offset_ids(in, count, delta, out, num_sms(), S(stream)), "boba_offset_ids");
}

size_t boba_range_partition_workspace_size(uint64_t m, int parts) {
    return boba::range_partition_workspace_bytes(m, parts);
}

int boba_range_partition_ex(const uint32_t* keys, const uint32_t* vals, uint64_t m, const uint32_t* bounds,
                            int parts, int relative_keys, uint32_t* keys_out, uint32_t* vals_out, uint32_t* counts_out,
                            void* ws, size_t ws_bytes, void* stream) {
    REQUIRE(parts >= 1 && parts <= 256, "boba_range_partition: parts must be in [1, 256]");
    REQUIRE(bounds && ws, "boba_range_partition: NULL argument");
    REQUIRE((keys && vals && keys_out && vals_out) || m == 0, "boba_range_partition: NULL edge arrays");
    REQUIRE(m < 0xFFFFFFFFull, "boba_range_partition: m too large");
    return cuda_status(boba::launch_range_partition(keys, vals, m, bounds, parts, keys_out, vals_out, counts_out, ws,
                                                    ws_bytes, num_sms(), S(stream), relative_keys != 0),
                       "boba_range_partition");
}

int boba_range_partition(const uint32_t* keys, const uint32_t* vals, uint64_t m, const uint32_t* bounds, int parts,
                         uint32_t* keys_out, uint32_t* vals_out, uint32_t* counts_out, void* ws, size_t ws_bytes,
                         void* stream) {
    REQUIRE(counts_out, "boba_range_partition: NULL counts_out");
    return boba_range_partition_ex(keys, vals, m, bounds, parts, 0, keys_out, vals_out, counts_out, ws, ws_bytes,
                                   stream);
}

size_t boba_compact_shard_workspace_size(uint64_t m_local, uint32_t n) {
    return boba::compact_window_workspace_bytes(m_local, n);
}

int boba_compact_shard_mark(const uint32_t* first, uint32_t n, uint64_t m_global, uint64_t e0, uint64_t m_local,
                            uint32_t* counts, void* ws, size_t ws_bytes, void* stream) {
    if (int rc = check_sizes(m_global, n, "boba_compact_shard_mark")) return rc;
    REQUIRE(e0 + m_local <= m_global, "boba_compact_shard_mark: shard outside [0, m_global)");
    REQUIRE(counts && ws && (first || n == 0), "boba_compact_shard_mark: NULL argument");
    REQUIRE(ws_bytes >= boba::compact_window_workspace_bytes(m_local, n), "boba_compact_shard_mark: workspace too small");
    return cuda_status(boba::launch_compact_window_mark(first, n, m_global, e0, m_local, counts, ws, ws_bytes,
                                                        num_sms(), S(stream)),
                       "boba_compact_shard_mark");
}

int boba_compact_shard_assign(const uint32_t* first, uint32_t n, uint64_t m_global, uint64_t e0, uint64_t m_local,
                              const uint32_t* all_counts, int world, int rank, uint32_t* label_partial, void* ws,
                              size_t ws_bytes, void* stream) {
    if (int rc = check_sizes(m_global, n, "boba_compact_shard_assign")) return rc;
    REQUIRE(world >= 1 && rank >= 0 && rank < world, "boba_compact_shard_assign: bad rank/world");
    REQUIRE(e0 + m_local <= m_global, "boba_compact_shard_assign: shard outside [0, m_global)");
    REQUIRE(all_counts && ws && ((first && label_partial) || n == 0), "boba_compact_shard_assign: NULL argument");
    REQUIRE(ws_bytes >= boba::compact_window_workspace_bytes(m_local, n),
            "boba_compact_shard_assign: workspace too small");
    return cuda_status(boba::launch_compact_window_assign(first, n, m_global, e0, m_local, all_counts, world, rank,
                                                          label_partial, ws, ws_bytes, S(stream)),
                       "boba_compact_shard_assign");
}

size_t boba_hub_table_bytes(void) { return boba::kHubTableBytes; }

int boba_order_from_label(const uint32_t* label, uint32_t n, uint32_t* order, void* hubs, void* stream) {
    REQUIRE((label && order) || n == 0, "boba_order_from_label: NULL argument");
    return cuda_status(boba::launch_order_from_label(label, n, order, static_cast<unsigned long long*>(hubs),
                                                     num_sms(), S(stream)),
                       "boba_order_from_label");
}

int boba_relabel_hubs(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n, const uint32_t* label,
                      const void* hubs, uint32_t* I2, uint32_t* J2, void* stream) {
    if (int rc = check_sizes(m, n, "boba_relabel_hubs")) return rc;
    REQUIRE((I && J && I2 && J2 && label) || m == 0, "boba_relabel_hubs: NULL argument");
    return cuda_status(boba::launch_relabel(I, J, m, label, static_cast<const unsigned long long*>(hubs), I2, J2,
                                            nullptr, n, num_sms(), S(stream)),
                       "boba_relabel_hubs");
}

uint32_t boba_row_cut_buckets(uint32_t n) { return boba::row_cut_buckets(n); }

int boba_row_cut_hist(const uint32_t* rows, uint64_t m_local, uint32_t n, uint32_t* hist, void* stream) {
    REQUIRE(hist && (rows || m_local == 0), "boba_row_cut_hist: NULL argument");
    return cuda_status(boba::launch_coarse_hist(rows, m_local, n, hist, num_sms(), S(stream)), "boba_row_cut_hist");
}

int boba_row_cut(const uint32_t* hist_global, const uint32_t* hist_local, uint32_t n, uint64_t m_global, int world,
                 uint32_t* out, void* stream) {
    REQUIRE(world >= 1 && world <= 256, "boba_row_cut: world must be in [1, 256]");
    REQUIRE(m_global < 0xFFFFFFFFull, "boba_row_cut: m_global too large");
    REQUIRE(hist_global && hist_local && out, "boba_row_cut: NULL argument");
    return cuda_status(boba::launch_row_cut(hist_global, hist_local, n, m_global, world, out, S(stream)),
                       "boba_row_cut");
}

int boba_gather_u32(const uint32_t* src, const uint32_t* idx, uint64_t count, uint32_t* out, void* stream) {
    REQUIRE((src && idx && out) || count == 0, "boba_gather_u32: NULL argument");
    return cuda_status(boba::launch_gather_u32(src, idx, count, out, num_sms(), S(stream)), "boba_gather_u32");
}

int boba_total_degrees(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n, uint32_t* deg, void* stream) {
    if (int rc = check_sizes(m, n, "boba_total_degrees")) return rc;
    if (n == 0) return BOBA_OK;
    REQUIRE(deg && ((I && J) || m == 0), "boba_total_degrees: NULL argument");
    return cuda_status(boba::launch_total_degrees(I, J, m, n, deg, num_sms(), S(stream)), "boba_total_degrees");
}

size_t boba_degree_order_workspace_size(uint64_t m, uint32_t n) { return boba::degree_order_workspace_bytes(m, n); }

int boba_degree_order(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n, uint32_t* order, uint32_t* label,
                      void* ws, size_t ws_bytes, void* stream) {
    if (int rc = check_sizes(m, n, "boba_degree_order")) return rc;
    if (n == 0) return BOBA_OK;
    REQUIRE(order && label && ws && ((I && J) || m == 0), "boba_degree_order: NULL argument");
    REQUIRE(ws_bytes >= boba::degree_order_workspace_bytes(m, n), "boba_degree_order: workspace too small");
    return cuda_status(boba::launch_degree_order(I, J, m, n, order, label, ws, ws_bytes, num_sms(), S(stream), false),
                       "boba_degree_order");
}

int boba_hub_order(const uint32_t* I, const uint32_t* J, uint64_t m, uint32_t n, uint32_t* order, uint32_t* label,
                   void* ws, size_t ws_bytes, void* stream) {
    if (int rc = check_sizes(m, n, "boba_hub_order")) return rc;
    if (n == 0) return BOBA_OK;
    REQUIRE(order && label && ws && ((I && J) || m == 0), "boba_hub_order: NULL argument");
    REQUIRE(ws_bytes >= boba::degree_order_workspace_bytes(m, n), "boba_hub_order: workspace too small");
    return cuda_status(boba::launch_degree_order(I, J, m, n, order, label, ws, ws_bytes, num_sms(), S(stream), true),
                       "boba_hub_order");
}

size_t boba_sort_coo_by_destination_workspace_size(uint64_t m, uint32_t n) {
    return boba::sort_by_destination_workspace_bytes(m, n);
}

int boba_sort_coo_by_destination(const uint32_t* I, const uint32_t* J, const double* w, uint64_t m, uint32_t n,
                                 uint32_t* I_out, uint32_t* J_out, double* w_out, void* ws, size_t ws_bytes,
                                 void* stream) {
    if (int rc = check_sizes(m, n, "boba_sort_coo_by_destination")) return rc;
    if (m == 0) return BOBA_OK;
    REQUIRE(I && J && I_out && J_out && ws, "boba_sort_coo_by_destination: NULL argument");
    REQUIRE(!w || w_out, "boba_sort_coo_by_destination: weights given but weights_out is NULL");
    REQUIRE(ws_bytes >= boba::sort_by_destination_workspace_bytes(m, n),
            "boba_sort_coo_by_destination: workspace too small");
    return cuda_status(boba::launch_sort_by_destination(I, J, w, m, n, I_out, J_out, w_out, ws, ws_bytes, num_sms(),
                                                        S(stream)),
                       "boba_sort_coo_by_destination");
}

size_t boba_pagerank_workspace_size(uint32_t n, uint64_t m) {
    return boba::pagerank_workspace_bytes(n, m, num_sms());
}

int boba_pagerank(const uint32_t* offsets, const uint32_t* indices, const double* w, uint32_t n, uint64_t m,
                  double damping, double tol, int max_iters, double* x, uint32_t* iterations, void* ws,
                  size_t ws_bytes, void* stream) {
    if (int rc = check_sizes(m, n, "boba_pagerank")) return rc;
    REQUIRE(damping > 0.0 && damping < 1.0, "damping must lie strictly between 0 and 1, got %g", damping);
    REQUIRE(max_iters >= 0, "boba_pagerank: max_iters must be non-negative");
    if (n == 0) return cuda_status(iterations ? cudaMemsetAsync(iterations, 0, 4, S(stream)) : cudaSuccess,
                                   "boba_pagerank");
    REQUIRE(offsets && x && ws && (indices || m == 0), "boba_pagerank: NULL argument");
    REQUIRE(ws_bytes >= boba::pagerank_workspace_bytes(n, m, num_sms()), "boba_pagerank: workspace too small");
    return cuda_status(boba::launch_pagerank(offsets, indices, w, n, m, damping, tol, max_iters, x, iterations, ws,
                                             ws_bytes, num_sms(), S(stream)),
                       "boba_pagerank");
}

size_t boba_nbr_workspace_size(uint64_t m, uint32_t n) { return boba::nbr_workspace_bytes(m, n); }

int boba_nbr(const uint32_t* offsets, const uint32_t* indices, uint32_t n, uint64_t m, uint32_t line_size,
             double* out, void* ws, size_t ws_bytes, void* stream) {
    if (int rc = check_sizes(m, n, "boba_nbr")) return rc;
    REQUIRE(line_size >= 1, "line size must be at least 1, got %u", line_size);
    REQUIRE(m > 0 && n > 0, "boba_nbr: the neighbourhood line ratio is undefined without edges");
    REQUIRE(offsets && indices && out && ws, "boba_nbr: NULL argument");
    REQUIRE(ws_bytes >= boba::nbr_workspace_bytes(m, n), "boba_nbr: workspace too small");
    return cuda_status(boba::launch_nbr(offsets, indices, n, m, line_size, out, ws, ws_bytes, num_sms(), S(stream)),
                       "boba_nbr");
}

int boba_generate_rmat(int scale, uint64_t m, uint64_t seed, uint32_t* I, uint32_t* J, void* stream) {
    REQUIRE(scale >= 0 && scale <= 32, "boba_generate_rmat: scale out of range");
    REQUIRE((I && J) || m == 0, "boba_generate_rmat: NULL argument");
    return cuda_status(boba::launch_rmat(scale, 0, m, seed, I, J, num_sms(), S(stream)), "boba_generate_rmat");
}

int boba_generate_rmat_range(int scale, uint64_t e0, uint64_t count, uint64_t seed, uint32_t* I, uint32_t* J,
                             void* stream) {
    REQUIRE(scale >= 0 && scale <= 32, "boba_generate_rmat_range: scale out of range");
    REQUIRE((I && J) || count == 0, "boba_generate_rmat_range: NULL argument");
    return cuda_status(boba::launch_rmat(scale, e0, count, seed, I, J, num_sms(), S(stream)),
                       "boba_generate_rmat_range");
}

int boba_generate_grid(uint32_t rows, uint32_t cols, uint32_t* I, uint32_t* J, void* stream) {
    REQUIRE(rows >= 1 && cols >= 1, "boba_generate_grid: dimensions must be positive");
    REQUIRE(I && J, "boba_generate_grid: NULL argument");
    return cuda_status(boba::launch_grid(rows, cols, I, J, num_sms(), S(stream)), "boba_generate_grid");
}

}  // extern "C"
