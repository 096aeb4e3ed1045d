"""numpy <-> device glue for the reference-shaped API.

The reference works on host int64 arrays; the kernels on device uint32.
Ids cross PCIe as uint32: boba_host_to_device_ids narrows on host threads
into pinned staging (with the reference's [0, n) range check) while earlier
chunks copy, boba_device_to_host_ids widens on host threads while later
chunks copy.

Arrays this package itself returned inside an immutable container (the
relabelled COO of apply_permutation, the label of a Permutation from
boba_parallel) keep a reference to their device copy, so the next call of
the reference pipeline (apply_permutation -> coo_to_csr) does not upload
them again.  Arrays a caller passed in are always uploaded.
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np
import torch

from . import _native as N
from . import device as D
from .errors import MalformedGraphError

RANK_UNSET = np.iinfo(np.int64).max  # reference _parallel.py:31


def _dev():
    return D.require_cuda()


_DEVICE_COPIES: dict = {}


def remember(host_arr, dev: torch.Tensor) -> None:
    """Record that `dev` (uint32 ids on the device) equals the read-only
    host array `host_arr` this package created; forgotten with the array."""
    key = id(host_arr)
    _DEVICE_COPIES[key] = (weakref.ref(host_arr, lambda _r, k=key: _DEVICE_COPIES.pop(k, None)), dev)


def _recall(host_arr):
    e = _DEVICE_COPIES.get(id(host_arr))
    if e is None or e[0]() is not host_arr:
        return None
    t = e[1]
    return t if t.device == _dev() else None


def to_device_ids(a, bound: int, name: str = "ids") -> torch.Tensor:
    cached = _recall(a)
    if cached is not None:
        return cached
    arr = np.ascontiguousarray(a, dtype=np.int64)
    out = torch.empty(arr.size, dtype=D.ID, device=_dev())
    bad = ctypes.c_int64(-1)
    rc = N.lib.boba_host_to_device_ids(ctypes.c_void_p(arr.ctypes.data), arr.size, int(bound), D._p(out),
                                       ctypes.byref(bad), D._s())
    if rc == N.BOBA_ERANGE:
        i = int(bad.value)
        raise MalformedGraphError(f"{name}[{i}] = {int(arr[i])} out of range for n = {bound}")
    N.check(rc)
    return out


def to_host_ids(t: torch.Tensor) -> np.ndarray:
    out = np.empty(t.numel(), dtype=np.int64)
    if t.numel():
        N.check(N.lib.boba_device_to_host_ids(D._p(t), t.numel(), ctypes.c_void_p(out.ctypes.data), D._s()))
    return out


def first_to_ranks(first: torch.Tensor) -> np.ndarray:
    """uint32 first-occurrence array -> the reference's int64 rank array
    (0xFFFFFFFF -> RANK_UNSET, mapped while widening: a numpy masked fix-up
    cost 23 ms of boba_parallel's 59 at c2)."""
    r = np.empty(first.numel(), dtype=np.int64)
    if first.numel():
        N.check(N.lib.boba_device_to_host_ranks(D._p(first), first.numel(), ctypes.c_void_p(r.ctypes.data), D._s()))
    return r


def ranks_to_first(r) -> torch.Tensor:
    r = np.ascontiguousarray(r, dtype=np.int64)
    f = np.where(r == RANK_UNSET, 0xFFFFFFFF, r).astype(np.uint32).view(np.int32)
    return torch.from_numpy(f).to(_dev())


def boba(I, J, n: int, relaxed: bool = False, ranks: bool = True):
    """-> (r int64 with RANK_UNSET or None when not `ranks`, order int64,
    label int64, device label)."""
    if n == 0:
        e = np.empty(0, dtype=np.int64)
        return e, e.copy(), e.copy(), None
    dI, dJ = to_device_ids(I, n, "I"), to_device_ids(J, n, "J")
    first, order, label = D.boba_order(dI, dJ, n, relaxed)
    return first_to_ranks(first) if ranks else None, to_host_ids(order), to_host_ids(label), label


def compact(r, I, J, n: int):
    """reference _parallel.compact_ranks on the GPU -> order int64."""
    if n == 0:
        return np.empty(0, dtype=np.int64)
    first = ranks_to_first(r)
    order, _ = D.compact(first, int(np.asarray(I).size), n)
    return to_host_ids(order)


def relabel(I, J, label, n: int):
    """-> (I2, J2 host int64, I2, J2 on the device)."""
    m = int(np.asarray(I).size)
    if m == 0:
        return np.empty(0, dtype=np.int64), np.empty(0, dtype=np.int64), None, None
    dI, dJ = to_device_ids(I, n, "I"), to_device_ids(J, n, "J")
    dl = to_device_ids(label, max(n, 1), "label")
    I2, J2 = D.relabel(dI, dJ, dl, n)
    return to_host_ids(I2), to_host_ids(J2), I2, J2


def degrees(I, n: int) -> np.ndarray:
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    dI = to_device_ids(I, n, "I")
    return to_host_ids(D.degrees(dI, n))


def total_degrees(I, J, n: int) -> np.ndarray:
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    return to_host_ids(D.total_degrees(to_device_ids(I, n, "I"), to_device_ids(J, n, "J"), n))


def degree_order(I, J, n: int, hub: bool = False):
    """-> (order, label) int64."""
    if n == 0:
        e = np.empty(0, dtype=np.int64)
        return e, e.copy()
    order, label = D.degree_order(to_device_ids(I, n, "I"), to_device_ids(J, n, "J"), n, hub=hub)
    return to_host_ids(order), to_host_ids(label)


def sort_coo_by_destination(I, J, n: int, weights=None):
    m = int(np.asarray(I).size)
    if m == 0:
        e = np.empty(0, dtype=np.int64)
        return e, e.copy(), (None if weights is None else np.empty(0, dtype=np.float64))
    w = None
    if weights is not None:
        w = torch.from_numpy(np.ascontiguousarray(weights, dtype=np.float64)).to(_dev())
    Io, Jo, wo = D.sort_coo_by_destination(to_device_ids(I, n, "I"), to_device_ids(J, n, "J"), n, w)
    return to_host_ids(Io), to_host_ids(Jo), (None if wo is None else wo.cpu().numpy())


def coo_to_csr(I, J, n: int, weights=None):
    dI, dJ = to_device_ids(I, n, "I"), to_device_ids(J, n, "J")
    w = None
    if weights is not None:
        w = torch.from_numpy(np.ascontiguousarray(weights, dtype=np.float64)).to(_dev())
    offsets, indices, w_out = D.coo_to_csr(dI, dJ, n, w)
    return to_host_ids(offsets), to_host_ids(indices), (None if w_out is None else w_out.cpu().numpy())


def spmv(offsets, indices, x, weights=None) -> np.ndarray:
    n = int(np.asarray(offsets).size) - 1
    dev = _dev()
    m = int(np.asarray(indices).size)
    do = to_device_ids(offsets, m + 1, "offsets")
    di = to_device_ids(indices, max(n, 1), "indices") if m else torch.empty(0, dtype=D.ID, device=dev)
    # float64 like the reference (kernels.py:30-52); device.spmv also offers fp32
    dx = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev)
    dw = None if weights is None else torch.from_numpy(np.ascontiguousarray(weights, dtype=np.float64)).to(dev)
    return D.spmv(do, di, dx, dw).cpu().numpy()


def pagerank(offsets, indices, n: int, weights, damping: float, tol: float, max_iters: int):
    m = int(np.asarray(indices).size)
    dev = _dev()
    do = to_device_ids(offsets, m + 1, "offsets")
    di = to_device_ids(indices, max(n, 1), "indices") if m else torch.empty(0, dtype=D.ID, device=dev)
    dw = None if weights is None else torch.from_numpy(np.ascontiguousarray(weights, dtype=np.float64)).to(dev)
    x, it = D.pagerank(do, di, dw, damping, tol, max_iters)
    return x.cpu().numpy(), int(it.cpu()[0])


def nbr(offsets, indices, line_size: int) -> float:
    n = int(np.asarray(offsets).size) - 1
    m = int(np.asarray(indices).size)
    do = to_device_ids(offsets, m + 1, "offsets")
    di = to_device_ids(indices, max(n, 1), "indices")
    return D.nbr(do, di, line_size)
