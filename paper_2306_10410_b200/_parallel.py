"""GPU replacements for the reference's native seam ``boba._parallel``.

The reference keeps "all hot loops ... behind plain-array signatures"
(pkg/src/boba/_parallel.py:1-5) and its callers resolve them through the
module at call time (ordering.py:140-147, graph.py:268).  This module offers
the same names and signatures, returning the same numpy int64 arrays, backed
by libboba_b200.so -- so rebinding ``boba._parallel``'s attributes to these
functions moves the reference's own pipeline onto the GPU.
"""

from __future__ import annotations

import numpy as np

from . import _host

__all__ = ["RANK_UNSET", "clamp_threads", "run_racy_first_hit", "scatter_rows", "first_hit_sequential",
           "first_hit_order_sequential", "first_hit_chunked", "first_hit_racy", "compact_ranks"]

RANK_UNSET = _host.RANK_UNSET  # reference _parallel.py:31


def clamp_threads(k: int | None) -> int:
    """reference _parallel.py:37-41; the GPU ignores host thread counts."""
    return 1 if k is None else max(1, int(k))


def first_hit_sequential(I, J, n):
    """reference _parallel.py:91-108 -> exact ranks."""
    return _host.boba(I, J, int(n))[0]


def first_hit_order_sequential(I, J, n):
    """reference _parallel.py:111-136 -> (ranks, order)."""
    r, order, _, _ = _host.boba(I, J, int(n))
    return r, order


def first_hit_chunked(I, J, n, nchunks):
    """reference _parallel.py:139-162 (exact for every chunk count)."""
    return _host.boba(I, J, int(n))[0]


def first_hit_racy(I, J, n):
    """reference _parallel.py:165-175: guarded racy stores."""
    return _host.boba(I, J, int(n), relaxed=True)[0]


def run_racy_first_hit(I, J, n, threads: int):
    """reference _parallel.py:44-52; one 'thread' is the exact scan."""
    return _host.boba(I, J, int(n), relaxed=clamp_threads(threads) > 1)[0]


def compact_ranks(r, I, J):
    """reference _parallel.py:178-201 -> order."""
    return _host.compact(r, I, J, int(np.asarray(r).size))


def scatter_rows(I, J, weights, offsets):
    """reference _parallel.py:84-88: stable row scatter -> (indices, weights).
    ``offsets`` fixes n; the GPU recomputes the same offsets from I."""
    n = int(np.asarray(offsets).size) - 1
    _, indices, w = _host.coo_to_csr(I, J, n, weights)
    return indices, w
