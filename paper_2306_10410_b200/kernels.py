"""CSR SpMV on the GPU with the reference's API (pkg/src/boba/kernels.py).

``spmv_pull`` mirrors kernels.py:30-52: y[v] = sum over row v of
w * x[indices], empty rows 0, ValueError on a length mismatch.  It runs the
merge-path kernel in float64 -- the reference's precision -- so it agrees
with the reference to fp64 rounding (the reference's np.add.reduceat has its
own summation order, so not bit for bit unless the sums are exact).  The
benchmarked path is the fp32 instantiation of the same kernel
(``device.spmv`` with float32 x; 1e-5 relative, SURVEY.md §7 hard part 6).

``pagerank`` mirrors kernels.py:57-107 (power iteration, uniform teleport,
dangling mass spread uniformly, L1 stopping rule) with the whole iteration
device-resident: boba_pagerank launches every round back to back and a
device stop flag ends the work once the L1 change drops below ``tol``.
"""

from __future__ import annotations

import numpy as np

from . import _host
from .validation import check_csr, check_vector

__all__ = ["spmv_pull", "pagerank"]


def spmv_pull(reversed_csr, x) -> np.ndarray:
    csr = check_csr(reversed_csr)
    x = check_vector(x, int(csr.n))
    if int(np.asarray(csr.indices).size) == 0:
        return np.zeros(int(csr.n), dtype=np.float64)
    return _host.spmv(csr.offsets, csr.indices, x, csr.weights)



def pagerank(csr, damping: float = 0.85, tol: float = 1e-6, max_iters: int = 100, return_iterations: bool = False):
    """Reference kernels.py:57-107 on the forward CSR (row v = out-neighbours)."""
    if not 0.0 < damping < 1.0:
        raise ValueError(f"damping must lie strictly between 0 and 1, got {damping}")
    csr = check_csr(csr)
    n = int(csr.n)
    if n == 0:
        empty = np.zeros(0, dtype=np.float64)
        return (empty, 0) if return_iterations else empty
    x, iters = _host.pagerank(csr.offsets, csr.indices, n, csr.weights, float(damping), float(tol), int(max_iters))
    return (x, iters) if return_iterations else x
