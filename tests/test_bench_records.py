"""Benchmark records compatible with the reference's boba.bench (SURVEY §8f
f2): BenchRecord rows, order-insensitive kernel checksums, compare_records
speedups against the random ordering (reference bench.py:37-254 and the
reference's test_bench_cli.py:47-58: identical checksums across orderings)."""

import hashlib

import numpy as np
import pytest

from conftest import has_gpu


def _records_frame():
    from paper_2306_10410_b200.bench import BenchRecord, records_to_frame

    rows = []
    for ordering, conv, kern in (("random", 10.0, 4.0), ("boba", 5.0, 2.0)):
        for rep, k in (("0", kern), ("median", kern)):
            rows.append(BenchRecord(dataset="d", kernel="spmv", ordering=ordering, mode="deterministic", seed=0,
                                    threads=1, repeat=rep, reorder_ms=1.0, sort_ms=None, convert_ms=conv,
                                    kernel_ms=k, end_to_end_ms=1.0 + conv + k, iterations=1, kernel_checksum="x",
                                    n=3, m=2))
    return records_to_frame(rows)


def test_compare_records_speedups():
    from paper_2306_10410_b200.bench import compare_records

    cmp = compare_records(_records_frame())
    boba = cmp[cmp["ordering"] == "boba"].iloc[0]
    assert boba["convert_speedup"] == pytest.approx(2.0) and boba["kernel_speedup"] == pytest.approx(2.0)
    assert boba["end_to_end_speedup"] == pytest.approx(15.0 / 8.0)


def test_compare_records_needs_random_baseline():
    from paper_2306_10410_b200 import BobaError
    from paper_2306_10410_b200.bench import compare_records

    f = _records_frame()
    with pytest.raises(BobaError):
        compare_records(f[f["ordering"] != "random"])
    with pytest.raises(BobaError):
        compare_records(f[f["repeat"] != "median"])


@pytest.mark.gpu
def test_run_bench_checksums_agree_across_orderings(medium):
    if not has_gpu():
        pytest.skip("no CUDA device")
    import paper_2306_10410_b200 as bb
    from paper_2306_10410_b200.bench import compare_records, records_to_frame, run_bench

    c = medium.case(0)
    g = bb.CooGraph(c["n"], c["I"], c["J"])
    recs = []
    for ordering in ("random", "boba", "degree", "identity"):
        r = run_bench(g, "rmat12", ordering, "spmv", seed=3, repeats=2)
        assert len(r) == 3 and r[-1].repeat == "median" and r[-1].device == "cuda"
        assert r[-1].nbr is not None and 0.0 < r[-1].nbr <= 1.0
        recs += r
    sums = {r.kernel_checksum for r in recs}
    # SpMV with x = ones gives the row degrees: the sorted multiset is order independent
    deg = np.sort(np.bincount(c["I"], minlength=c["n"]).astype(np.float64))
    assert sums == {hashlib.sha256(deg.tobytes()).hexdigest()[:16]}
    cmp = compare_records(records_to_frame(recs))
    assert set(cmp["ordering"]) == {"random", "boba", "degree", "identity"}
    pr = run_bench(g, "rmat12", "boba", "pr", repeats=1, compute_locality=False)
    assert pr[-1].iterations > 1 and pr[-1].nbr is None
    with pytest.raises(ValueError):
        run_bench(g, "rmat12", "boba", "tc")
