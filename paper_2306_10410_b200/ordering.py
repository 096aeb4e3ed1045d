"""BOBA vertex ordering on the GPU, with the reference's API.

Drop-in for the hot-path part of ``pkg/src/boba/ordering.py``:

* ``boba_parallel``   reference ordering.py:99-151 -- phases 1+2 on the GPU
  (first occurrence by atomicMin, then bitmap + lookback-scan compaction).
  Deterministic mode is bit-exact with the reference for every
  ``thread_hint`` (the hint only picked a CPU chunk count there).
  Relaxed mode uses guarded racy stores (reference first_hit_racy); with
  ``thread_hint`` None/1 the reference's racy loop is single threaded and
  therefore exact, so the deterministic kernel is used for that case.
* ``boba_sequential`` reference ordering.py:59-96 -- same permutation.
* ``degree_order`` / ``hub_order`` reference ordering.py:160-176 -- total
  degrees by atomics, then a stable radix sort of the ids by degree key.
* ``compute_ordering`` reference ordering.py:334-356 for the methods on the
  path ("boba", "boba-relaxed"), the degree baselines ("degree", "hub") and
  the trivial ones ("random" = numpy PCG64 permutation exactly as the
  reference, "identity").  "rcm" (scipy on a symmetrised CSR) is out of scope.
* ``BobaOrder`` reference ordering.py:273-290 (scikit-learn transformer).
"""

from __future__ import annotations

import numpy as np
from sklearn.base import BaseEstimator, TransformerMixin
from sklearn.exceptions import NotFittedError

from . import _host
from .graph import INDEX_DTYPE, CooGraph, Permutation, apply_permutation
from .validation import check_coo

__all__ = ["RANK_UNSET", "boba_sequential", "boba_parallel", "random_order", "identity_order", "degree_order",
           "hub_order", "compute_ordering", "BobaOrder", "RandomOrder", "IdentityOrder", "DegreeOrder", "HubOrder",
           "ORDERING_CHOICES"]

RANK_UNSET = _host.RANK_UNSET
ORDERING_CHOICES = ("random", "boba", "boba-relaxed", "degree", "hub", "identity")
_MODES = ("deterministic", "relaxed")


def boba_parallel(g, mode: str = "deterministic", thread_hint: int | None = None, return_ranks: bool = False):
    """Order vertices by first appearance in I||J (sources first), isolated
    vertices appended ascending.  Returns a Permutation, or (Permutation,
    ranks) with ranks int64 and RANK_UNSET for isolated vertices."""
    if mode not in _MODES:
        raise ValueError(f"unknown mode: {mode!r}")
    relaxed = mode == "relaxed" and thread_hint is not None and int(thread_hint) > 1
    r, order, label, dlabel = _host.boba(g.I, g.J, int(g.n), relaxed=relaxed, ranks=return_ranks)
    p = Permutation(order, label)
    if dlabel is not None:   # apply_permutation(g, p) reuses the device label
        _host.remember(p.label, dlabel)
    return (p, r) if return_ranks else p


def boba_sequential(g) -> Permutation:
    """Same permutation as the reference's one-pass scan (ordering.py:59-96)."""
    return boba_parallel(g)


def random_order(n: int, seed: int) -> Permutation:
    """Reference ordering.py:154-157 (host numpy PCG64; not a GPU phase)."""
    return Permutation(np.random.default_rng(seed).permutation(n).astype(INDEX_DTYPE))


def identity_order(n: int) -> Permutation:
    return Permutation.identity(n)


def degree_order(g) -> Permutation:
    """Total degree descending, ties by ascending id (reference
    ordering.py:160-164, np.lexsort((arange(n), -deg)))."""
    order, label = _host.degree_order(g.I, g.J, int(g.n))
    return Permutation(order, label)


def hub_order(g) -> Permutation:
    """Vertices of above-mean total degree first by descending degree (ties
    by id), the rest after them in id order (reference ordering.py:167-176)."""
    order, label = _host.degree_order(g.I, g.J, int(g.n), hub=True)
    return Permutation(order, label)


def compute_ordering(g, method: str, seed: int = 0, mode: str = "deterministic",
                     thread_hint: int | None = None) -> Permutation:
    """Dispatch by method name (reference ordering.py:334-356)."""
    if method == "random":
        return random_order(g.n, seed)
    if method == "boba":
        return boba_parallel(g, mode=mode, thread_hint=thread_hint)
    if method == "boba-relaxed":
        return boba_parallel(g, mode="relaxed", thread_hint=thread_hint)
    if method == "degree":
        return degree_order(g)
    if method == "hub":
        return hub_order(g)
    if method == "identity":
        return identity_order(g.n)
    if method == "rcm":
        raise ValueError(f"ordering method {method!r} is outside the B200 hot path; use the reference package")
    raise ValueError(f"unknown ordering method: {method!r}")


class _Reorderer(BaseEstimator, TransformerMixin):
    """fit learns ``permutation_`` from an edge list, transform relabels one
    (reference ordering.py:247-270)."""

    def fit(self, X, y=None):
        X = check_coo(X)
        self.permutation_ = self._permutation(X)
        self.n_vertices_ = X.n
        return self

    def transform(self, X) -> CooGraph:
        if not hasattr(self, "permutation_"):
            raise NotFittedError(f"This {type(self).__name__} instance is not fitted yet.")
        return apply_permutation(check_coo(X), self.permutation_)

    def _permutation(self, X) -> Permutation:
        raise NotImplementedError


class BobaOrder(_Reorderer):
    """Order-by-attachment transformer (reference ordering.py:273-290)."""

    def __init__(self, mode: str = "deterministic", thread_hint: int | None = None):
        self.mode = mode
        self.thread_hint = thread_hint

    def _permutation(self, X):
        return boba_parallel(X, mode=self.mode, thread_hint=self.thread_hint)


class RandomOrder(_Reorderer):
    def __init__(self, seed: int = 0):
        self.seed = seed

    def _permutation(self, X):
        return random_order(X.n, self.seed)


class IdentityOrder(_Reorderer):
    def _permutation(self, X):
        return identity_order(X.n)


class DegreeOrder(_Reorderer):
    """Descending total-degree transformer (reference ordering.py:303-307)."""

    def _permutation(self, X):
        return degree_order(X)


class HubOrder(_Reorderer):
    """Hubs-first transformer (reference ordering.py:310-314)."""

    def _permutation(self, X):
        return hub_order(X)
