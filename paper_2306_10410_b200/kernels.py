"""CSR SpMV on the GPU with the reference's API (pkg/src/boba/kernels.py).

``spmv_pull`` mirrors kernels.py:30-52: y[v] = sum over row v of
w * x[indices], empty rows 0, ValueError on a length mismatch.  It runs the
merge-path kernel in float64 -- the reference's precision -- so it agrees
with the reference to fp64 rounding (the reference's np.add.reduceat has its
own summation order, so not bit for bit unless the sums are exact).  The
benchmarked path is the fp32 instantiation of the same kernel
(``device.spmv`` with float32 x; 1e-5 relative, SURVEY.md §7 hard part 6).
"""

from __future__ import annotations

import numpy as np

from . import _host
from .validation import check_csr, check_vector

__all__ = ["spmv_pull"]


def spmv_pull(reversed_csr, x) -> np.ndarray:
    csr = check_csr(reversed_csr)
    x = check_vector(x, int(csr.n))
    if int(np.asarray(csr.indices).size) == 0:
        return np.zeros(int(csr.n), dtype=np.float64)
    return _host.spmv(csr.offsets, csr.indices, x, csr.weights)

