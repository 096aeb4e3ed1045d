"""Host-side logic of the reference-shaped API that runs without a GPU:
container invariants and error types (reference graph.py / validation.py /
ordering.py contracts)."""

import numpy as np
import pytest


def test_container_invariants():
    import paper_2306_10410_b200 as bb

    with pytest.raises(bb.MalformedGraphError):
        bb.CooGraph(3, [0, 3], [1, 2])
    with pytest.raises(bb.MalformedGraphError):
        bb.CooGraph(3, [0, -1], [1, 2])
    with pytest.raises(bb.MalformedGraphError):
        bb.CooGraph(3, [0, 1], [1])
    with pytest.raises(bb.MalformedGraphError):
        bb.CooGraph(3, [0], [1], [1.0, 2.0])
    with pytest.raises(bb.MalformedGraphError):
        bb.CsrGraph(2, [0, 1], [0])
    with pytest.raises(bb.MalformedGraphError):
        bb.CsrGraph(2, [0, 2, 1], [0, 1])
    with pytest.raises(bb.MalformedGraphError):
        bb.CsrGraph(2, [0, 1, 2], [0, 5])
    g = bb.CooGraph(3, [0, 1], [1, 2])
    with pytest.raises(ValueError):
        g.I[0] = 2
    assert g.m == 2 and g.reverse().I.tolist() == [1, 2]
    assert issubclass(bb.MalformedGraphError, bb.BobaError)


def test_permutation_contract():
    import paper_2306_10410_b200 as bb

    p = bb.Permutation([2, 0, 1])
    assert p.label.tolist() == [1, 2, 0] and p.is_valid()
    with pytest.raises(bb.MalformedGraphError):
        bb.Permutation.from_order([0, 0, 2])
    q = p.inverse()
    assert q.order.tolist() == [1, 2, 0]
    assert bb.Permutation.identity(4).order.tolist() == [0, 1, 2, 3]


def test_ordering_dispatch_errors_and_estimator_params():
    import paper_2306_10410_b200 as bb
    from sklearn.exceptions import NotFittedError

    g = bb.CooGraph(3, [0, 1], [1, 2])
    with pytest.raises(ValueError):
        bb.compute_ordering(g, "nope")
    with pytest.raises(ValueError):
        bb.boba_parallel(g, mode="yolo")
    with pytest.raises(NotFittedError):
        bb.BobaOrder().transform(g)
    est = bb.BobaOrder(mode="relaxed", thread_hint=4)
    assert est.get_params() == {"mode": "relaxed", "thread_hint": 4}
    est.set_params(mode="deterministic")
    assert est.mode == "deterministic"
    with pytest.raises(TypeError):
        bb.BobaOrder().fit([1, 2, 3])
    # random ordering is numpy PCG64 exactly as the reference's
    assert np.array_equal(bb.random_order(100, 7).order, np.random.default_rng(7).permutation(100))


def test_csr_helpers():
    import paper_2306_10410_b200 as bb

    csr = bb.CsrGraph(3, [0, 2, 2, 3], [1, 2, 0])
    assert csr.row(0).tolist() == [1, 2] and csr.out_degrees().tolist() == [2, 0, 1]
    coo = csr.to_coo()
    assert coo.I.tolist() == [0, 0, 2] and coo.J.tolist() == [1, 2, 0]
