"""Device-resident API: the BOBA path on CUDA tensors (uint32 ids stored as
torch.int32), one C-ABI call per phase on the current torch stream.

This is the layer the numpy-level drop-in (graph.py / ordering.py /
kernels.py) and bench.py are built on.  Every function here runs a kernel
of libboba_b200.so; nothing falls back to the CPU.
"""

from __future__ import annotations

import ctypes

import torch

from . import _native as N
from .errors import MalformedGraphError

ID = torch.int32  # storage dtype of uint32 ids (the kernels read the bits as uint32)


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2306_10410_b200 needs a CUDA device (sm_100a); there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _s():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def as_u32_to_i64(t: torch.Tensor) -> torch.Tensor:
    """uint32 bits (int32 storage) -> int64 values, on the device."""
    out = torch.empty(t.numel(), dtype=torch.int64, device=t.device)
    N.check(N.lib.boba_widen_ids(_p(t), t.numel(), _p(out), _s()))
    return out


def narrow_ids(t: torch.Tensor, bound: int, name: str = "ids") -> torch.Tensor:
    """int64 device tensor -> uint32 ids with the reference's range check
    (graph.py:99-106 raises MalformedGraphError on an id outside [0, n))."""
    out = torch.empty(t.numel(), dtype=ID, device=t.device)
    bad = ctypes.c_int64(-1)
    rc = N.lib.boba_narrow_ids(_p(t), t.numel(), int(bound), _p(out), ctypes.byref(bad), _s())
    if rc == N.BOBA_ERANGE:
        i = int(bad.value)
        raise MalformedGraphError(f"{name}[{i}] = {int(t[i])} out of range for n = {bound}")
    N.check(rc)
    return out


def first_occurrence(I: torch.Tensor, J: torch.Tensor, n: int, relaxed: bool = False) -> torch.Tensor:
    """Phase 1 (reference _parallel.py:139-175)."""
    first = torch.empty(max(n, 1), dtype=ID, device=I.device)[:n]
    N.check(N.lib.boba_first_occurrence(_p(I), _p(J), I.numel(), n, _p(first), int(relaxed), _s()))
    return first


def compact(first: torch.Tensor, m: int, n: int):
    """Phase 2 (reference _parallel.py:178-201, graph.py:205-208) -> (order, label)."""
    dev = first.device
    order = torch.empty(max(n, 1), dtype=ID, device=dev)[:n]
    label = torch.empty(max(n, 1), dtype=ID, device=dev)[:n]
    ws = _ws(N.lib.boba_compact_workspace_size(m, n), dev)
    N.check(N.lib.boba_compact(_p(first), m, n, _p(order), _p(label), None, _p(ws), ws.numel(), _s()))
    return order, label


def boba_order(I: torch.Tensor, J: torch.Tensor, n: int, relaxed: bool = False):
    """Phases 1+2 -> (first, order, label)."""
    first = first_occurrence(I, J, n, relaxed)
    order, label = compact(first, I.numel(), n)
    return first, order, label


def relabel(I: torch.Tensor, J: torch.Tensor, label: torch.Tensor, n: int, with_counts: bool = False):
    """Phase 3 (reference graph.py:280-289) -> (I2, J2[, row_counts])."""
    dev = I.device
    m = I.numel()
    I2 = torch.empty(m, dtype=ID, device=dev)
    J2 = torch.empty(m, dtype=ID, device=dev)
    counts = torch.empty(max(n, 1), dtype=ID, device=dev)[:n] if with_counts else None
    N.check(N.lib.boba_relabel(_p(I), _p(J), m, n, _p(label), _p(I2), _p(J2), _p(counts), _s()))
    return (I2, J2, counts) if with_counts else (I2, J2)


def degrees(I: torch.Tensor, n: int) -> torch.Tensor:
    """reference graph.py:292-294 (uint32 counts)."""
    deg = torch.empty(max(n, 1), dtype=ID, device=I.device)[:n]
    N.check(N.lib.boba_degrees(_p(I), I.numel(), n, _p(deg), _s()))
    return deg


def total_degrees(I: torch.Tensor, J: torch.Tensor, n: int) -> torch.Tensor:
    """reference graph.py:297-300 (in + out degree, uint32 counts)."""
    deg = torch.empty(max(n, 1), dtype=ID, device=I.device)[:n]
    N.check(N.lib.boba_total_degrees(_p(I), _p(J), I.numel(), n, _p(deg), _s()))
    return deg


def degree_order(I: torch.Tensor, J: torch.Tensor, n: int, hub: bool = False):
    """reference ordering.py:160-164 (hub=False) / 167-176 (hub=True) ->
    (order, label)."""
    m = I.numel()
    order = torch.empty(max(n, 1), dtype=ID, device=I.device)[:n]
    label = torch.empty(max(n, 1), dtype=ID, device=I.device)[:n]
    ws = _ws(N.lib.boba_degree_order_workspace_size(m, n), I.device)
    fn = N.lib.boba_hub_order if hub else N.lib.boba_degree_order
    N.check(fn(_p(I), _p(J), m, n, _p(order), _p(label), _p(ws), ws.numel(), _s()))
    return order, label


def sort_coo_by_destination(I: torch.Tensor, J: torch.Tensor, n: int, weights: torch.Tensor | None = None):
    """reference graph.py:303-307: stable sort of the edges by J ->
    (I_out, J_out, weights_out|None)."""
    m = I.numel()
    Io, Jo = torch.empty_like(I), torch.empty_like(J)
    w_out = None
    if weights is not None:
        weights = weights.to(torch.float64).contiguous()
        w_out = torch.empty(m, dtype=torch.float64, device=I.device)
    ws = _ws(N.lib.boba_sort_coo_by_destination_workspace_size(m, n), I.device)
    N.check(N.lib.boba_sort_coo_by_destination(_p(I), _p(J), _p(weights), m, n, _p(Io), _p(Jo), _p(w_out), _p(ws),
                                               ws.numel(), _s()))
    return Io, Jo, w_out


def coo_to_csr(I2: torch.Tensor, J2: torch.Tensor, n: int, weights: torch.Tensor | None = None,
               row_counts: torch.Tensor | None = None):
    """Phase 4 (reference graph.py:253-277, _parallel.py:55-88) ->
    (offsets[n+1], indices[m], weights_out|None)."""
    dev = I2.device
    m = I2.numel()
    offsets = torch.empty(n + 1, dtype=ID, device=dev)
    indices = torch.empty(m, dtype=ID, device=dev)
    w_out = None
    if weights is not None:
        weights = weights.to(torch.float64).contiguous()
        w_out = torch.empty(m, dtype=torch.float64, device=dev)
    ws = _ws(N.lib.boba_coo_to_csr_workspace_size(m, n, int(weights is not None)), dev)
    N.check(N.lib.boba_coo_to_csr(_p(I2), _p(J2), _p(weights), m, n, _p(row_counts), _p(offsets), _p(indices),
                                  _p(w_out), _p(ws), ws.numel(), _s()))
    return offsets, indices, w_out


def spmv(offsets: torch.Tensor, indices: torch.Tensor, x: torch.Tensor,
         weights: torch.Tensor | None = None, out: torch.Tensor | None = None,
         ws: torch.Tensor | None = None, reuse_partition: bool = False) -> torch.Tensor:
    """Phase 5 (reference kernels.py:30-52).  Computes in x's precision:
    float32 (the benchmarked path) or float64 (the reference's).
    reuse_partition: the previous call with this `ws` had the same CSR
    structure; its merge-path partition is reused (iterative callers)."""
    n = offsets.numel() - 1
    m = indices.numel()
    f64 = x.dtype == torch.float64
    dt = torch.float64 if f64 else torch.float32
    x = x.to(dt).contiguous()
    if weights is not None:
        weights = weights.to(dt).contiguous()
    y = out if out is not None else torch.empty(max(n, 1), dtype=dt, device=offsets.device)[:n]
    if reuse_partition and ws is None:
        raise ValueError("reuse_partition needs the workspace of the previous call")
    if ws is None:
        ws = _ws(N.lib.boba_spmv_workspace_size(n, m), offsets.device)
    fn = N.lib.boba_spmv_f64_ex if f64 else N.lib.boba_spmv_ex
    N.check(fn(_p(offsets), _p(indices), _p(weights), _p(x), _p(y), n, m, _p(ws), ws.numel(), int(reuse_partition),
               _s()))
    return y


def pagerank(offsets: torch.Tensor, indices: torch.Tensor, weights: torch.Tensor | None = None,
             damping: float = 0.85, tol: float = 1e-6, max_iters: int = 100):
    """reference kernels.py:57-107 on a forward CSR -> (x float64, iterations
    as a 1-element uint32 device tensor; no host synchronisation)."""
    n = offsets.numel() - 1
    m = indices.numel()
    dev = offsets.device
    if weights is not None:
        weights = weights.to(torch.float64).contiguous()
    x = torch.empty(max(n, 1), dtype=torch.float64, device=dev)[:n]
    iters = torch.zeros(1, dtype=ID, device=dev)
    ws = _ws(N.lib.boba_pagerank_workspace_size(n, m), dev)
    N.check(N.lib.boba_pagerank(_p(offsets), _p(indices), _p(weights), n, m, float(damping), float(tol),
                                int(max_iters), _p(x), _p(iters), _p(ws), ws.numel(), _s()))
    return x, iters


def nbr(offsets: torch.Tensor, indices: torch.Tensor, line_size: int = 32) -> float:
    """Neighbourhood line ratio (reference metrics.py:90-115) on device CSR."""
    n = offsets.numel() - 1
    m = indices.numel()
    out = torch.empty(1, dtype=torch.float64, device=offsets.device)
    ws = _ws(N.lib.boba_nbr_workspace_size(m, n), offsets.device)
    N.check(N.lib.boba_nbr(_p(offsets), _p(indices), n, m, line_size, _p(out), _p(ws), ws.numel(), _s()))
    return float(out.item())


def spmv_workspace(n: int, m: int, device) -> torch.Tensor:
    return _ws(N.lib.boba_spmv_workspace_size(n, m), device)


class Pipeline:
    """Preallocated buffers for the fused reorder -> relabel -> CSR pipeline
    (reference bench.py:135-149) on graphs with up to (m, n)."""

    def __init__(self, m: int, n: int, device=None, weighted: bool = False):
        dev = device or require_cuda()
        self.m, self.n, self.device = m, n, dev
        e = lambda k: torch.empty(max(k, 1), dtype=ID, device=dev)  # noqa: E731
        self.first, self.order, self.label = e(n), e(n), e(n)
        self.I2, self.J2, self.indices = e(m), e(m), e(m)
        self.offsets = e(n + 1)
        self.w_out = torch.empty(max(m, 1), dtype=torch.float64, device=dev) if weighted else None
        self.ws = _ws(N.lib.boba_reorder_to_csr_workspace_size(m, n, int(weighted)), dev)

    def run(self, I: torch.Tensor, J: torch.Tensor, weights: torch.Tensor | None = None):
        m, n = I.numel(), self.n
        if m > self.m:
            raise ValueError(f"graph has {m} edges, pipeline sized for {self.m}")
        N.check(N.lib.boba_reorder_to_csr(
            _p(I), _p(J), _p(weights), m, n, _p(self.first), _p(self.order), _p(self.label), _p(self.I2),
            _p(self.J2), _p(self.offsets), _p(self.indices), _p(self.w_out), _p(self.ws), self.ws.numel(), _s()))
        return self


class CapturedPipeline:
    """A Pipeline's fused call on fixed inputs (I, J) captured into a CUDA
    graph (boba_reorder_to_csr_graph_create); launch() replays the whole
    step with one graph launch.  Creating it runs the pipeline once."""

    def __init__(self, pipe: "Pipeline", I: torch.Tensor, J: torch.Tensor, events=None):
        """events: 5 CUDA event handles recorded at the phase boundaries of
        every replay (boba_reorder_to_csr_graph_create_timed), or None."""
        self.pipe, self.I, self.J = pipe, I, J  # keep the buffers alive
        self._g = ctypes.c_void_p()
        p = pipe
        args = (_p(I), _p(J), I.numel(), p.n, _p(p.first), _p(p.order), _p(p.label), _p(p.I2), _p(p.J2),
                _p(p.offsets), _p(p.indices), _p(p.ws), p.ws.numel())
        if events is None:
            N.check(N.lib.boba_reorder_to_csr_graph_create(*args, ctypes.byref(self._g)))
        else:
            self._events = events
            N.check(N.lib.boba_reorder_to_csr_graph_create_timed(*args, events, ctypes.byref(self._g)))

    def launch(self):
        N.check(N.lib.boba_graph_launch(self._g, _s()))
        return self.pipe

    def kernel_nodes(self) -> int:
        """Kernel launches one replay performs."""
        k = ctypes.c_uint64()
        N.check(N.lib.boba_graph_kernel_nodes(self._g, ctypes.byref(k)))
        return int(k.value)

    def close(self):
        if self._g:
            N.lib.boba_reorder_to_csr_graph_destroy(self._g)
            self._g = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def generate_rmat(scale: int, edge_factor: int, seed: int, device=None):
    """Graph500 R-MAT edges (uint32) on the device; see oracle.rmat_edges."""
    dev = device or require_cuda()
    m = edge_factor << scale
    I = torch.empty(m, dtype=ID, device=dev)
    J = torch.empty(m, dtype=ID, device=dev)
    N.check(N.lib.boba_generate_rmat(scale, m, seed & (2**64 - 1), _p(I), _p(J), _s()))
    return I, J


def generate_rmat_range(scale: int, e0: int, count: int, seed: int, device=None):
    """Edges [e0, e0 + count) of the R-MAT stream of generate_rmat (a shard)."""
    dev = device or require_cuda()
    I = torch.empty(count, dtype=ID, device=dev)
    J = torch.empty(count, dtype=ID, device=dev)
    N.check(N.lib.boba_generate_rmat_range(scale, e0, count, seed & (2**64 - 1), _p(I), _p(J), _s()))
    return I, J


def generate_grid(rows: int, cols: int, device=None):
    """reference generators.py:100-111 on the device."""
    dev = device or require_cuda()
    m = 2 * rows * (cols - 1) + 2 * (rows - 1) * cols
    I = torch.empty(m, dtype=ID, device=dev)
    J = torch.empty(m, dtype=ID, device=dev)
    if m:
        N.check(N.lib.boba_generate_grid(rows, cols, _p(I), _p(J), _s()))
    return I, J


def gather(src: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    out = torch.empty(idx.numel(), dtype=ID, device=idx.device)
    N.check(N.lib.boba_gather_u32(_p(src), _p(idx), idx.numel(), _p(out), _s()))
    return out


class HostPipeline:
    """End-to-end entry with HOST buffers (boba_ctx_* in the C ABI)."""

    def __init__(self, max_m: int, max_n: int):
        require_cuda()
        self._ctx = ctypes.c_void_p()
        N.check(N.lib.boba_ctx_create(max_m, max_n, ctypes.byref(self._ctx)))

    def run(self, I_host, J_host, n, order, label, offsets, indices, I2=None, J2=None):
        """All arguments are host uint32 buffers (numpy arrays or pinned torch
        CPU tensors); outputs are written in place."""
        ptr = lambda a: None if a is None else ctypes.c_void_p(  # noqa: E731
            a.data_ptr() if isinstance(a, torch.Tensor) else a.ctypes.data)
        m = I_host.numel() if isinstance(I_host, torch.Tensor) else I_host.size
        N.check(N.lib.boba_ctx_reorder_to_csr_host(self._ctx, ptr(I_host), ptr(J_host), m, n, ptr(order),
                                                   ptr(label), ptr(I2), ptr(J2), ptr(offsets), ptr(indices)))

    def submit(self, I_host, J_host, n, order, label, offsets, indices, I2=None, J2=None) -> int:
        """Asynchronous run: enqueues the graph and returns a ticket for wait().
        Two graphs can be in flight; their copies overlap each other and the
        compute.  Inputs must stay unchanged and outputs unread until wait()."""
        ptr = lambda a: None if a is None else ctypes.c_void_p(  # noqa: E731
            a.data_ptr() if isinstance(a, torch.Tensor) else a.ctypes.data)
        m = I_host.numel() if isinstance(I_host, torch.Tensor) else I_host.size
        t = ctypes.c_uint64()
        N.check(N.lib.boba_ctx_submit_host(self._ctx, ptr(I_host), ptr(J_host), m, n, ptr(order), ptr(label),
                                           ptr(I2), ptr(J2), ptr(offsets), ptr(indices), ctypes.byref(t)))
        return t.value

    def wait(self, ticket: int) -> None:
        N.check(N.lib.boba_ctx_wait(self._ctx, ticket))

    def close(self):
        if self._ctx:
            N.lib.boba_ctx_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
