"""Benchmark records compatible with the reference's ``boba.bench``
(pkg/src/boba/bench.py:37-254): the same timed pipeline --
reorder (ordering + relabel), convert (COO->CSR), kernel -- and the same
``BenchRecord`` rows, order-insensitive kernel checksums and
``compare_records`` speedups, plus a ``device`` column.  Every phase runs
through this package's drop-in API on the B200 (host arrays in, host arrays
out, so the device copies each call makes are inside its time, as the
reference's in-memory timings cover its whole call).

Kernels: ``spmv`` and ``pr``.  The reference's triangle counting and SSSP are
not on the BOBA path and are not provided.  Locality: only the
neighbourhood line ratio (``nbr``) is computed, on the GPU; the other scores
are left ``None``.
"""

from __future__ import annotations

import hashlib
import statistics
import time
from dataclasses import dataclass, fields

import numpy as np

from .errors import BobaError
from .graph import CooGraph, apply_permutation, coo_to_csr
from .kernels import pagerank, spmv_pull
from .metrics import DEFAULT_LINE_SIZE, nbr
from .ordering import ORDERING_CHOICES, compute_ordering

__all__ = ["KERNEL_CHOICES", "BenchRecord", "run_bench", "records_to_frame", "compare_records"]

KERNEL_CHOICES = ("spmv", "pr")


@dataclass(frozen=True)
class BenchRecord:
    """One timed pipeline run (or the median row of its repeats); the
    reference's columns (bench.py:37-66) plus ``device``."""

    dataset: str
    kernel: str
    ordering: str
    mode: str
    seed: int
    threads: int
    repeat: str
    reorder_ms: float
    sort_ms: float | None
    convert_ms: float
    kernel_ms: float
    end_to_end_ms: float
    iterations: int
    kernel_checksum: str
    n: int
    m: int
    nscore: int | None = None
    gscore: int | None = None
    w: int | None = None
    nbr: float | None = None
    bandwidth: int | None = None
    line_size: int | None = None
    device: str = "cuda"

    @classmethod
    def columns(cls) -> list[str]:
        return [f.name for f in fields(cls)]

    def to_row(self) -> list:
        return [getattr(self, c) for c in self.columns()]


def _ms(fn, *args, **kwargs):
    t0 = time.perf_counter_ns()
    out = fn(*args, **kwargs)
    return out, round((time.perf_counter_ns() - t0) / 1e3) / 1e3


def _digest(data: bytes) -> str:
    return hashlib.sha256(data).hexdigest()[:16]


def kernel_checksum(kernel: str, result) -> str:
    """Order-insensitive digest of a kernel's answer (bench.py:80-93)."""
    if kernel == "spmv":
        return _digest(np.sort(result).tobytes())
    if kernel == "pr":
        return _digest(np.round(np.sort(result), 6).tobytes())
    raise ValueError(f"unknown kernel: {kernel!r}")


def run_bench(g: CooGraph, dataset: str, ordering: str, kernel: str, seed: int = 0, threads: int = 1,
              mode: str = "deterministic", repeats: int = 3, w: int = 1, line_size: int = DEFAULT_LINE_SIZE,
              compute_locality: bool = True) -> list[BenchRecord]:
    """reorder -> convert -> kernel, each timed (bench.py:95-223): one record
    per kernel repeat plus a median record."""
    if ordering not in ORDERING_CHOICES:
        raise ValueError(f"unknown ordering: {ordering!r}")
    if kernel not in KERNEL_CHOICES:
        raise ValueError(f"unknown kernel: {kernel!r} (the B200 path runs {', '.join(KERNEL_CHOICES)})")
    if repeats < 1:
        raise ValueError("repeats must be at least 1")
    effective_mode = "relaxed" if ordering == "boba-relaxed" else mode

    def reorder_and_apply():
        p = compute_ordering(g, ordering, seed=seed, mode=mode, thread_hint=threads)
        return p, apply_permutation(g, p)

    (p, relabeled), reorder_ms = _ms(reorder_and_apply)
    csr, convert_ms = _ms(coo_to_csr, relabeled)
    x_ones = np.ones(g.n, dtype=np.float64)

    def run_kernel():
        if kernel == "spmv":
            return spmv_pull(csr, x_ones), 1
        return pagerank(csr, return_iterations=True)

    ratio = nbr(csr, line_size) if (compute_locality and g.m) else None
    base = dict(dataset=dataset, kernel=kernel, ordering=ordering, mode=effective_mode, seed=seed, threads=threads,
                reorder_ms=reorder_ms, sort_ms=None, convert_ms=convert_ms, n=g.n, m=g.m,
                w=w if ratio is not None else None, nbr=ratio, line_size=line_size if ratio is not None else None)
    records, kernel_times = [], []
    for rep in range(repeats):
        (result, iterations), kernel_ms = _ms(run_kernel)
        kernel_times.append(kernel_ms)
        records.append(BenchRecord(repeat=str(rep), kernel_ms=kernel_ms,
                                   end_to_end_ms=round((reorder_ms + convert_ms + kernel_ms) * 1e3) / 1e3,
                                   iterations=iterations, kernel_checksum=kernel_checksum(kernel, result), **base))
    med = round(statistics.median(kernel_times) * 1e3) / 1e3
    records.append(BenchRecord(repeat="median", kernel_ms=med,
                               end_to_end_ms=round((reorder_ms + convert_ms + med) * 1e3) / 1e3,
                               iterations=records[-1].iterations, kernel_checksum=records[-1].kernel_checksum, **base))
    return records


def records_to_frame(records: list[BenchRecord]):
    import pandas as pd

    return pd.DataFrame([r.to_row() for r in records], columns=BenchRecord.columns())


_RATIO_PHASES = ("reorder_ms", "convert_ms", "kernel_ms", "end_to_end_ms")


def compare_records(frame):
    """Median rows normalised against the ``random`` ordering of the same
    (dataset, kernel) (bench.py:229-254); speedup = baseline / observed.

    Raises
    ------
    BobaError
        If there are no median rows, or a group lacks its random baseline.
    """
    import pandas as pd

    med = frame[frame["repeat"].astype(str) == "median"].copy()
    if med.empty:
        raise BobaError("no median rows found in the benchmark records")
    out = []
    for (dataset, kernel), grp in med.groupby(["dataset", "kernel"], sort=True):
        baseline = grp[grp["ordering"] == "random"]
        if baseline.empty:
            raise BobaError(f"missing 'random' baseline row for dataset={dataset!r}, kernel={kernel!r}")
        base = baseline.iloc[0]
        for _, row in grp.iterrows():
            entry = {"dataset": dataset, "kernel": kernel, "ordering": row["ordering"],
                     **{ph: row[ph] for ph in _RATIO_PHASES}}
            for ph in ("convert_ms", "kernel_ms", "end_to_end_ms"):
                entry[ph.replace("_ms", "_speedup")] = float(base[ph]) / float(row[ph]) if row[ph] else float("nan")
            out.append(entry)
    return pd.DataFrame(out)
