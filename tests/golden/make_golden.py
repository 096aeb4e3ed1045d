"""Generate the golden parity fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package from /root/reference/pkg/src (numba cache
redirected to /tmp so nothing is written into the read-only tree) and the
reference's own test helpers (pkg/tests/conftest.py: the road graph and
``random_coo``), runs the reference's public functions, and stores inputs
and outputs under tests/golden/.  The GPU box never sees /root/reference:
tests there read only these committed fixtures.

Fixtures
--------
kat.npz      the reference's known-answer cases + the road graph
fuzz.npz     random_coo multigraphs from the reference's own fuzz seeds
             (test_ordering.py:64 seed 17, test_graph.py:117 seed 11,
             test_graph.py:140 seed 5 weighted), concatenated
medium.npz   R-MAT s12 ef8 (repo generator), grid 64x64 and LCD(5000,4)
             (reference generator), each randomly relabelled with the
             reference's randomize_labels; outputs stored whole
Every case also stores the reference's neighbourhood line ratio (nbr) of the
BOBA CSR (line sizes 32 and 4) and of the direct CSR (32) when it has edges.
"""

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/boba_numba_cache")
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

import boba  # noqa: E402  (the reference)
from boba import CooGraph  # noqa: E402
from conftest import ROAD_CITIES, ROAD_EDGE_TOKENS, random_coo  # noqa: E402

import oracle  # noqa: E402  (only for the repo's R-MAT input generator)


def run_ref(g: CooGraph, x=None):
    """Everything the hot path produces, straight from the reference."""
    p, r = boba.boba_parallel(g, return_ranks=True)
    seq = boba.boba_sequential(g)
    assert np.array_equal(seq.order, p.order)
    g2 = boba.apply_permutation(g, p)
    csr = boba.coo_to_csr(g2)
    if x is None:
        x = np.random.default_rng(g.n * 7919 + g.m).random(g.n)
    y = boba.spmv_pull(csr, x)
    raw = boba.coo_to_csr(g)                 # direct conversion, no reorder
    out = dict(order=p.order, label=p.label, r=r, I2=g2.I, J2=g2.J,
               offsets=csr.offsets, indices=csr.indices, x=x, y=y,
               deg=boba.degrees(g), offsets_raw=raw.offsets, indices_raw=raw.indices,
               y_raw=boba.spmv_pull(raw, x),
               weighted=np.array([int(g.weights is not None)]),
               tdeg=boba.total_degrees(g), deg_order=boba.degree_order(g).order,
               hub_order=boba.hub_order(g).order)
    out["pr"], it = boba.pagerank(raw, return_iterations=True)
    out["pr_iters"] = np.array([it])
    sd = boba.sort_coo_by_destination(g)
    out["I_sd"], out["J_sd"] = sd.I, sd.J
    if g.m:  # §8f f4: neighbourhood line ratio (metrics.py:90-115), BOBA CSR at 32 and 4, direct CSR at 32
        from boba.metrics import nbr
        out["nbr"] = np.array([nbr(csr, 32), nbr(csr, 4), nbr(raw, 32)])
    if g.weights is not None:
        out["w2"] = csr.weights
        out["w2_raw"] = raw.weights
        out["w_sd"] = sd.weights
    return out


def pack(cases):
    """Concatenate a list of dicts of 1-D arrays with per-case offsets."""
    keys = sorted({k for c in cases for k in c})
    res = {}
    for k in keys:
        arrs = [np.asarray(c.get(k, np.zeros(0))) for c in cases]
        res[k] = np.concatenate(arrs) if arrs else np.zeros(0)
        res[k + "__ptr"] = np.concatenate([[0], np.cumsum([a.size for a in arrs])]).astype(np.int64)
    return res


def case_from(g, name=None, x=None):
    out = run_ref(g, x)
    c = dict(n=np.array([g.n]), I=g.I, J=g.J, **out)
    if g.weights is not None:
        c["w"] = g.weights
    return c


def main():
    kat = []
    ids = {c: k for k, c in enumerate(ROAD_CITIES)}
    road = CooGraph(len(ROAD_CITIES), [ids[u] for u, v in ROAD_EDGE_TOKENS],
                    [ids[v] for u, v in ROAD_EDGE_TOKENS])
    kat.append(case_from(road))                                      # conftest.py:33-40
    kat.append(case_from(CooGraph(3, [0, 1], [1, 2]), x=np.array([1.0, 2.0, 3.0])))  # test_ordering.py:34
    kat.append(case_from(CooGraph(6, [5, 5, 3], [3, 1, 5])))         # test_ordering.py:37-40
    kat.append(case_from(CooGraph(4, [1, 2, 3], [0, 0, 0])))         # test_graph.py:30-33
    kat.append(case_from(CooGraph(3, [2, 0], [1, 1])))               # test_graph.py:35-38
    kat.append(case_from(CooGraph(4, [1, 1, 1], [3, 0, 2])))         # test_graph.py:40-43
    kat.append(case_from(CooGraph(3, [2, 0], [1, 1], [5.0, 7.0])))   # test_graph.py:45-47
    kat.append(case_from(CooGraph(4, [], [])))                       # test_kernels.py:78-80
    kat.append(case_from(CooGraph(1, [0], [0])))                     # self loop
    kat.append(case_from(CooGraph(5, [0, 0, 0, 0], [1, 2, 3, 4])))   # star (test_ordering.py:195)
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **pack(kat))

    fuzz = []
    for seed, count, weighted in ((17, 120, False), (11, 120, False), (5, 100, True)):
        rng = np.random.default_rng(seed)
        for _ in range(count):
            fuzz.append(case_from(random_coo(rng, weighted=weighted)))
    rng = np.random.default_rng(45242 + 5)                           # test_acceptance.py:136-149
    for _ in range(60):
        fuzz.append(case_from(random_coo(rng, n_max=400, m_max=4000)))
    np.savez_compressed(os.path.join(HERE, "fuzz.npz"), **pack(fuzz))

    med = []
    I, J = oracle.rmat_edges(12, 8, seed=1)
    g = CooGraph(1 << 12, I, J)
    g, _ = boba.randomize_labels(g, 7)
    med.append(case_from(g))
    g, _ = boba.randomize_labels(boba.generate_grid(64, 64), 7)
    med.append(case_from(g))
    g = boba.generate_lcd(boba.LcdParams(n=5000, c=4, seed=45242))
    g, _ = boba.randomize_labels(g, 45242 + 60)
    med.append(case_from(g))
    np.savez_compressed(os.path.join(HERE, "medium.npz"), **pack(med))
    for f in ("kat.npz", "fuzz.npz", "medium.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
