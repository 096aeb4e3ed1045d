"""Locality metrics on the GPU.

``nbr`` follows the reference's neighbourhood line ratio
(pkg/src/boba/metrics.py:90-115): mean, over vertices with at least one
out-neighbour, of the distinct cache lines (index // line_size) their
neighbour ids span divided by the neighbourhood size as a multiset.  It is
computed by the B200 kernels (csrc/metrics.cu: two stable radix sorts of the
(row, line) pairs and a fixed-order fp64 reduction).  The other scores of the
reference module (nscore, gscore, bandwidth, the brute-force oracle) are off
the BOBA hot path and not provided.
"""

from __future__ import annotations

import numpy as np

from . import _host
from .errors import UndefinedMetricError
from .validation import check_csr

__all__ = ["nbr", "DEFAULT_LINE_SIZE"]

DEFAULT_LINE_SIZE = 32


def nbr(csr, line_size: int = DEFAULT_LINE_SIZE) -> float:
    """Reference metrics.py:90-115.  Lower is better; 1.0 means every
    neighbour sits on its own line.

    Raises
    ------
    ValueError
        line_size < 1.
    UndefinedMetricError
        If the graph has no edges.
    """
    if line_size < 1:
        raise ValueError(f"line size must be at least 1, got {line_size}")
    csr = check_csr(csr)
    if int(np.asarray(csr.indices).size) == 0:
        raise UndefinedMetricError("neighborhood line ratio is undefined without edges")
    return _host.nbr(csr.offsets, csr.indices, int(line_size))
