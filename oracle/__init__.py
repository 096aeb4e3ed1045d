"""CPU oracle for the BOBA hot path -- TEST INFRASTRUCTURE, not product code.

A ctypes view of ``boba_oracle.c``, a plain-C restatement of the reference
functions on the path (reference ``pkg/src/boba/_parallel.py``, ``graph.py``,
``kernels.py``; file:line in each C function's comment).  Arrays are int64
like the reference's (``graph.py:31`` ``INDEX_DTYPE``).

Allowed importers: ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs -- always as the checker or the
CPU baseline, never as the thing measured for the GPU.  The product package
``paper_2306_10410_b200`` never imports this module.

Parity pinning: ``tests/test_oracle.py`` checks every function here against
the golden vectors in ``tests/golden/`` (made by importing the reference,
``tests/golden/make_golden.py``) and the reference's own known answers.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

RANK_UNSET = np.iinfo(np.int64).max  # reference _parallel.py:31

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc + OpenMP)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "boba_oracle.c"))
    ):
        build()
    lib = ctypes.CDLL(_LIB_PATH)
    sigs = {
        "oracle_num_threads": ([], ctypes.c_int),
        "oracle_first_hit_order_sequential": ([_P, _P, _I64, _I64, _P, _P], None),
        "oracle_first_hit_chunked": ([_P, _P, _I64, _I64, _I64, ctypes.c_int, _P], None),
        "oracle_compact_ranks": ([_P, _P, _P, _I64, _I64, _P], None),
        "oracle_label_from_order": ([_P, _I64, _P], None),
        "oracle_apply_permutation": ([_P, _P, _I64, _P, _P, _P], None),
        "oracle_degrees": ([_P, _I64, _I64, _P], None),
        "oracle_total_degrees": ([_P, _P, _I64, _I64, _P], None),
        "oracle_degree_order": ([_P, _P, _I64, _I64, ctypes.c_int, _P], None),
        "oracle_sort_by_destination": ([_P, _P, _P, _I64, _I64, _P, _P, _P], None),
        "oracle_coo_to_csr": ([_P, _P, _P, _I64, _I64, _P, _P, _P], None),
        "oracle_spmv_pull": ([_P, _P, _P, _P, _I64, _P], None),
        "oracle_rmat_edges": ([ctypes.c_int, _I64, ctypes.c_uint64, _I64, _I64, _P, _P], None),
        "oracle_grid_edges": ([_I64, _I64, _P, _P], None),
        "oracle_verify_pipeline_u32": ([_P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P], ctypes.c_int),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _ptr(a):
    return None if a is None else a.ctypes.data


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def first_hit_order_sequential(I, J, n):
    """reference _parallel.py:111-136 -> (r, order)."""
    I, J = _i64(I), _i64(J)
    r = np.empty(n, np.int64)
    order = np.empty(n, np.int64)
    _load().oracle_first_hit_order_sequential(_ptr(I), _ptr(J), I.size, n, _ptr(r), _ptr(order))
    return r, order


def first_hit_chunked(I, J, n, nchunks, threads=0):
    """reference _parallel.py:139-162 -> r."""
    I, J = _i64(I), _i64(J)
    r = np.empty(n, np.int64)
    _load().oracle_first_hit_chunked(_ptr(I), _ptr(J), I.size, n, int(nchunks), int(threads), _ptr(r))
    return r


def compact_ranks(r, I, J):
    """reference _parallel.py:178-201 -> order."""
    r, I, J = _i64(r), _i64(I), _i64(J)
    order = np.empty(r.size, np.int64)
    _load().oracle_compact_ranks(_ptr(r), _ptr(I), _ptr(J), I.size, r.size, _ptr(order))
    return order


def label_from_order(order):
    """reference graph.py:205-208 -> label."""
    order = _i64(order)
    label = np.empty_like(order)
    _load().oracle_label_from_order(_ptr(order), order.size, _ptr(label))
    return label


def boba_order(I, J, n):
    """reference ordering.py:136-140 (deterministic, thread_hint=None)."""
    return first_hit_order_sequential(I, J, n)[1]


def apply_permutation(I, J, label):
    """reference graph.py:280-289 -> (I2, J2)."""
    I, J, label = _i64(I), _i64(J), _i64(label)
    I2 = np.empty_like(I)
    J2 = np.empty_like(J)
    _load().oracle_apply_permutation(_ptr(I), _ptr(J), I.size, _ptr(label), _ptr(I2), _ptr(J2))
    return I2, J2


def degrees(I, n):
    """reference graph.py:292-294."""
    I = _i64(I)
    d = np.empty(n, np.int64)
    _load().oracle_degrees(_ptr(I), I.size, n, _ptr(d))
    return d


def total_degrees(I, J, n):
    """reference graph.py:297-300."""
    I, J = _i64(I), _i64(J)
    d = np.empty(n, np.int64)
    _load().oracle_total_degrees(_ptr(I), _ptr(J), I.size, n, _ptr(d))
    return d


def degree_order(I, J, n, hub=False):
    """reference ordering.py:160-164 (degree_order) / 167-176 (hub_order) -> order."""
    I, J = _i64(I), _i64(J)
    order = np.empty(n, np.int64)
    _load().oracle_degree_order(_ptr(I), _ptr(J), I.size, n, int(bool(hub)), _ptr(order))
    return order


def sort_coo_by_destination(I, J, n, weights=None):
    """reference graph.py:303-307 -> (I, J, weights)."""
    I, J = _i64(I), _i64(J)
    W = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    I2, J2 = np.empty_like(I), np.empty_like(J)
    W2 = None if W is None else np.empty(I.size, np.float64)
    _load().oracle_sort_by_destination(_ptr(I), _ptr(J), _ptr(W), I.size, n, _ptr(I2), _ptr(J2), _ptr(W2))
    return I2, J2, W2


def coo_to_csr(I, J, n, weights=None):
    """reference graph.py:253-277 + _parallel.py:55-88 -> (offsets, indices, weights)."""
    I, J = _i64(I), _i64(J)
    W = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    offsets = np.empty(n + 1, np.int64)
    indices = np.empty(I.size, np.int64)
    W2 = None if W is None else np.empty(I.size, np.float64)
    _load().oracle_coo_to_csr(_ptr(I), _ptr(J), _ptr(W), I.size, n, _ptr(offsets), _ptr(indices), _ptr(W2))
    return offsets, indices, W2


def spmv_pull(offsets, indices, x, weights=None):
    """reference kernels.py:30-52 (sequential row sums, fp64)."""
    offsets, indices = _i64(offsets), _i64(indices)
    x = np.ascontiguousarray(x, dtype=np.float64)
    W = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    n = offsets.size - 1
    y = np.empty(n, np.float64)
    _load().oracle_spmv_pull(_ptr(offsets), _ptr(indices), _ptr(W), _ptr(x), n, _ptr(y))
    return y


def pagerank(offsets, indices, x0_n, weights=None, damping=0.85, tol=1e-6, max_iters=100):
    """reference kernels.py:57-107, restated with the oracle's own CSR and
    SpMV (sequential row sums) -> (x, iterations)."""
    offsets, indices = _i64(offsets), _i64(indices)
    n = int(x0_n)
    if n == 0:
        return np.zeros(0), 0
    m = indices.size
    fw = np.ones(m) if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    deg = np.diff(offsets)
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    ow = spmv_pull(offsets, indices, np.ones(n), fw)   # row sums of the forward weights (kernels.py:88)
    dangling = ow == 0.0
    share = fw / np.repeat(np.where(dangling, 1.0, ow), deg)
    roff, ridx, rw = coo_to_csr(indices, src, n, share)
    x = np.full(n, 1.0 / n)
    tele = (1.0 - damping) / n
    it = 0
    for it in range(1, max_iters + 1):
        dm = x[dangling].sum() / n
        xn = damping * (spmv_pull(roff, ridx, x, rw) + dm) + tele
        delta = np.abs(xn - x).sum()
        x = xn
        if delta < tol:
            break
    return x, it


def rmat_edges(scale, edge_factor, seed, e0=0, e1=None):
    """Host twin of the device R-MAT generator (input prep, not reference)."""
    m = edge_factor << scale
    e1 = m if e1 is None else e1
    I = np.empty(e1 - e0, np.int64)
    J = np.empty(e1 - e0, np.int64)
    _load().oracle_rmat_edges(int(scale), m, int(seed) & (2**64 - 1), e0, e1, _ptr(I), _ptr(J))
    return I, J


def grid_edges(rows, cols):
    """reference generators.py:100-111 generate_grid (I, J)."""
    m = 2 * rows * (cols - 1) + 2 * (rows - 1) * cols
    I = np.empty(m, np.int64)
    J = np.empty(m, np.int64)
    _load().oracle_grid_edges(rows, cols, _ptr(I), _ptr(J))
    return I, J


def random_labels(n, seed):
    """reference ordering.py:154-157 random_order / io.py:294-301
    randomize_labels: order = default_rng(seed).permutation(n); returns the
    label (inverse) array that relabels the graph."""
    order = np.random.default_rng(seed).permutation(n).astype(np.int64)
    return label_from_order(order)


def pipeline(I, J, n, threads=0, weights=None):
    """The reference bench's reorder + convert phases (bench.py:135-149) with
    the reference's threading: first_hit_chunked over `threads` chunks when
    threads > 1 (ordering.py:141-143), else the fused sequential pass.
    Returns (order, label, I2, J2, offsets, indices, weights2)."""
    if threads and threads > 1:
        r = first_hit_chunked(I, J, n, threads, threads)
        order = compact_ranks(r, I, J)
    else:
        order = first_hit_order_sequential(I, J, n)[1]
    label = label_from_order(order)
    I2, J2 = apply_permutation(I, J, label)
    offsets, indices, w2 = coo_to_csr(I2, J2, n, weights)
    return order, label, I2, J2, offsets, indices, w2


VERIFY_ARRAYS = ("order", "label", "I2", "J2", "offsets", "indices")


def verify_pipeline_u32(I, J, n, order=None, label=None, I2=None, J2=None, offsets=None, indices=None):
    """Streaming uint32 check of a device pipeline result against the
    reference semantics (first_hit_order_sequential -> label ->
    apply_permutation -> coo_to_csr; see oracle_verify_pipeline_u32) at
    sizes where the int64 functions above would not fit in host memory.
    Returns {array name: first differing index} for every array that differs
    (empty dict = bit-exact)."""
    def u32(a):
        return None if a is None else np.ascontiguousarray(a).view(np.uint32)

    I, J = u32(I), u32(J)
    got = [u32(a) for a in (order, label, I2, J2, offsets, indices)]
    for a, size in zip(got, (n, n, I.size, I.size, n + 1, I.size)):
        if a is not None and a.size != size:
            raise ValueError("result array has the wrong size")
    first = np.empty(6, np.int64)
    bad = _load().oracle_verify_pipeline_u32(_ptr(I), _ptr(J), I.size, int(n), *[_ptr(a) for a in got], _ptr(first))
    if bad < 0:
        raise MemoryError("oracle_verify_pipeline_u32: allocation failed")
    return {VERIFY_ARRAYS[k]: int(first[k]) for k in range(6) if bad & (1 << k)}


def nbr(offsets, indices, line_size=32):
    """reference metrics.py:90-115 (neighbourhood line ratio), restated in
    numpy: per row with neighbours, distinct index // line_size values over
    the degree; the mean of those ratios."""
    offsets = np.asarray(offsets, dtype=np.int64)
    indices = np.asarray(indices, dtype=np.int64)
    n = offsets.size - 1
    deg = np.diff(offsets)
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    lines = indices // line_size
    k = np.lexsort((lines, rows))
    rs, ls = rows[k], lines[k]
    boundary = np.empty(rs.size, dtype=bool)
    boundary[0] = True
    boundary[1:] = (rs[1:] != rs[:-1]) | (ls[1:] != ls[:-1])
    counts = np.bincount(rs[boundary], minlength=n)
    mask = deg > 0
    return float(np.mean(counts[mask] / deg[mask]))
