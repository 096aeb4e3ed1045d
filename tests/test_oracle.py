"""Pin the CPU oracle (oracle/boba_oracle.c) to the reference.

1. Against the golden vectors made by running the reference itself
   (tests/golden/make_golden.py): permutation, ranks, relabelled COO,
   reordered and direct CSR, degrees, SpMV.
2. Against the reference's own known answers (pkg/tests/test_ordering.py,
   test_graph.py, test_kernels.py), restated.
3. Against the live reference package when /root/reference is present
   (build container only; skipped on the GPU box).
"""

import os
import sys

import numpy as np
import pytest

import oracle
from conftest import REFERENCE_SRC

RANK_UNSET = np.iinfo(np.int64).max


def check_case(c):
    I, J, n = c["I"], c["J"], c["n"]
    r, order = oracle.first_hit_order_sequential(I, J, n)
    assert np.array_equal(order, c["order"])
    assert np.array_equal(r, c["r"])
    r2 = oracle.first_hit_chunked(I, J, n, 3, 2)
    assert np.array_equal(r2, c["r"])
    assert np.array_equal(oracle.compact_ranks(r2, I, J), c["order"])
    label = oracle.label_from_order(order)
    assert np.array_equal(label, c["label"])
    I2, J2 = oracle.apply_permutation(I, J, label)
    assert np.array_equal(I2, c["I2"]) and np.array_equal(J2, c["J2"])
    off, idx, w2 = oracle.coo_to_csr(I2, J2, n, c["w"])
    assert np.array_equal(off, c["offsets"]) and np.array_equal(idx, c["indices"])
    if c["w"] is not None:
        assert np.array_equal(w2, c["w2"])
    off0, idx0, w0 = oracle.coo_to_csr(I, J, n, c["w"])
    assert np.array_equal(off0, c["offsets_raw"]) and np.array_equal(idx0, c["indices_raw"])
    if c["w"] is not None:
        assert np.array_equal(w0, c["w2_raw"])
    assert np.array_equal(oracle.degrees(I, n), c["deg"])
    y = oracle.spmv_pull(off, idx, c["x"], w2)
    np.testing.assert_allclose(y, c["y"], rtol=1e-12, atol=1e-12)
    # the orderings and the edge sort beside BOBA
    assert np.array_equal(oracle.total_degrees(I, J, n), c["tdeg"])
    assert np.array_equal(oracle.degree_order(I, J, n), c["deg_order"])
    assert np.array_equal(oracle.degree_order(I, J, n, hub=True), c["hub_order"])
    x, it = oracle.pagerank(off0, idx0, n, w0)
    assert it == c["pr_iters"][0]
    np.testing.assert_allclose(x, c["pr"], rtol=1e-10, atol=1e-14)
    Is, Js, ws = oracle.sort_coo_by_destination(I, J, n, c["w"])
    assert np.array_equal(Is, c["I_sd"]) and np.array_equal(Js, c["J_sd"])
    if c["w"] is not None:
        assert np.array_equal(ws, c["w_sd"])
    if I.size:  # §8f f4: neighbourhood line ratio
        got = [oracle.nbr(off, idx, 32), oracle.nbr(off, idx, 4), oracle.nbr(off0, idx0, 32)]
        np.testing.assert_allclose(got, c["nbr"], rtol=1e-15, atol=0)


def test_known_answers(kat):
    for c in kat:
        check_case(c)


def test_fuzz_cases(fuzz):
    for c in fuzz:
        check_case(c)


def test_medium_cases(medium):
    for c in medium:
        check_case(c)


def test_reference_known_answers_restated():
    # test_ordering.py:37-40 destination scan + isolated append
    _, order = oracle.first_hit_order_sequential([5, 5, 3], [3, 1, 5], 6)
    assert order.tolist() == [5, 3, 1, 0, 2, 4]
    # test_graph.py:40-43 stable row order
    off, idx, _ = oracle.coo_to_csr([1, 1, 1], [3, 0, 2], 4)
    assert idx[off[1]:off[2]].tolist() == [3, 0, 2]
    # test_graph.py:45-47 weights carried
    _, _, w = oracle.coo_to_csr([2, 0], [1, 1], 3, [5.0, 7.0])
    assert w.tolist() == [7.0, 5.0]
    # test_kernels.py:73-76 path
    off, idx, _ = oracle.coo_to_csr([1, 2], [0, 1], 3)   # reversed path 0->1->2
    assert oracle.spmv_pull(off, idx, [1.0, 2.0, 3.0]).tolist() == [0.0, 1.0, 2.0]
    # empty graph
    off, idx, _ = oracle.coo_to_csr([], [], 4)
    assert off.tolist() == [0] * 5 and idx.size == 0
    r, order = oracle.first_hit_order_sequential([], [], 3)
    assert order.tolist() == [0, 1, 2] and np.all(r == RANK_UNSET)


def test_grid_generator_matches_reference_definition():
    I, J = oracle.grid_edges(3, 4)
    # generators.py:100-111 written out with numpy
    ids = np.arange(12).reshape(3, 4)
    rs, rd = ids[:, :-1].ravel(), ids[:, 1:].ravel()
    ds, dd = ids[:-1, :].ravel(), ids[1:, :].ravel()
    assert np.array_equal(I, np.concatenate([rs, rd, ds, dd]))
    assert np.array_equal(J, np.concatenate([rd, rs, dd, ds]))


def test_rmat_generator_properties():
    I, J = oracle.rmat_edges(10, 8, seed=3)
    assert I.size == 8 << 10 and I.min() >= 0 and I.max() < 1024 and J.max() < 1024
    I2, J2 = oracle.rmat_edges(10, 8, seed=3, e0=100, e1=200)
    assert np.array_equal(I2, I[100:200]) and np.array_equal(J2, J[100:200])
    # quadrant frequencies at the top level: P(u bit)=c+d=.24, P(v bit)=b+d=.24
    top_u = (I >> 9) & 1
    top_v = (J >> 9) & 1
    assert abs(top_u.mean() - 0.24) < 0.02 and abs(top_v.mean() - 0.24) < 0.02
    I3, _ = oracle.rmat_edges(10, 8, seed=4)
    assert not np.array_equal(I, I3)


def test_pipeline_matches_parts(medium):
    c = medium.case(0)
    order, label, I2, J2, off, idx, _ = oracle.pipeline(c["I"], c["J"], c["n"], threads=4)
    assert np.array_equal(order, c["order"]) and np.array_equal(idx, c["indices"])


@pytest.mark.skipif(not os.path.isdir(REFERENCE_SRC), reason="reference not mounted (GPU box)")
def test_against_live_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/boba_numba_cache")
    sys.dont_write_bytecode = True
    sys.path.insert(0, REFERENCE_SRC)
    try:
        import boba
    finally:
        sys.path.remove(REFERENCE_SRC)
    rng = np.random.default_rng(2024)
    for _ in range(20):
        n = int(rng.integers(1, 3000))
        m = int(rng.integers(0, 20000))
        I, J = rng.integers(0, n, m), rng.integers(0, n, m)
        g = boba.CooGraph(n, I, J)
        p, r = boba.boba_parallel(g, thread_hint=4, return_ranks=True)
        r2, order = oracle.first_hit_order_sequential(I, J, n)
        assert np.array_equal(order, p.order) and np.array_equal(r2, r)
        csr = boba.coo_to_csr(boba.apply_permutation(g, p))
        I2, J2 = oracle.apply_permutation(I, J, oracle.label_from_order(order))
        off, idx, _ = oracle.coo_to_csr(I2, J2, n)
        assert np.array_equal(off, csr.offsets) and np.array_equal(idx, csr.indices)


def test_streaming_u32_verifier_against_golden(kat, fuzz, medium):
    """oracle.verify_pipeline_u32 (the BASELINE-size checker) accepts the
    reference's own outputs and pinpoints a corrupted entry in each array."""
    u = lambda a: np.asarray(a, dtype=np.int64).astype(np.uint32)  # noqa: E731
    cases = list(kat) + [fuzz.case(i) for i in range(0, fuzz.count, 5)] + list(medium)
    for c in cases:
        n = c["n"]
        got = dict(order=u(c["order"]), label=u(c["label"]), I2=u(c["I2"]), J2=u(c["J2"]),
                   offsets=u(c["offsets"]), indices=u(c["indices"]))
        assert oracle.verify_pipeline_u32(u(c["I"]), u(c["J"]), n, **got) == {}
        for name, arr in got.items():
            if arr.size < 2 or (name == "offsets" and c["I"].size == 0):
                continue
            bad = dict(got)
            bad[name] = arr.copy()
            k = arr.size // 2
            bad[name][k] ^= 1
            res = oracle.verify_pipeline_u32(u(c["I"]), u(c["J"]), n, **bad)
            assert name in res, (name, res)
