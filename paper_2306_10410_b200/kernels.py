"""CSR SpMV on the GPU with the reference's API (pkg/src/boba/kernels.py).

``spmv_pull`` mirrors kernels.py:30-52: y[v] = sum over row v of
w * x[indices], empty rows 0, ValueError on a length mismatch.  The
arithmetic is fp32 on the device (merge-path kernel, deterministic); the
result is returned as float64 like the reference's.  Parity with the
reference's float64 sums is a tolerance check (1e-5 relative for
non-negative x; exact when every partial sum is an integer below 2^24).
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

