"""GPU parity: every phase of the B200 path against the reference's outputs.

Golden fixtures (made by running the reference, tests/golden/) pin the small
cases bit-exactly; the C oracle (oracle/, itself pinned by test_oracle.py)
pins seeded R-MAT / grid graphs up to scale 20; size-independent properties
cover the full BASELINE sizes.  Integer outputs are compared bit-exactly;
SpMV (fp32 on the device vs the reference's fp64) within rtol 1e-5 for
non-negative x, exactly for integer-valued data.
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

RANK_UNSET = np.iinfo(np.int64).max
SPMV_RTOL = 1e-5
PR_RTOL = 1e-10   # fp64 PageRank vs the reference: differs only in summation order


@pytest.fixture(scope="module")
def bb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2306_10410_b200 as bb

    return bb


def run_case(bb, c):
    g = bb.CooGraph(c["n"], c["I"], c["J"], c["w"])
    p, r = bb.boba_parallel(g, return_ranks=True)
    assert np.array_equal(p.order, c["order"]), "order"
    assert np.array_equal(p.label, c["label"]), "label"
    assert np.array_equal(r, c["r"]), "ranks"
    g2 = bb.apply_permutation(g, p)
    assert np.array_equal(g2.I, c["I2"]) and np.array_equal(g2.J, c["J2"]), "relabel"
    csr = bb.coo_to_csr(g2)
    assert np.array_equal(csr.offsets, c["offsets"]), "offsets"
    assert np.array_equal(csr.indices, c["indices"]), "indices"
    raw = bb.coo_to_csr(g)
    assert np.array_equal(raw.offsets, c["offsets_raw"]) and np.array_equal(raw.indices, c["indices_raw"])
    if c["w"] is not None:
        assert np.array_equal(csr.weights, c["w2"]) and np.array_equal(raw.weights, c["w2_raw"])
    assert np.array_equal(bb.degrees(g), c["deg"])
    y = bb.spmv_pull(csr, c["x"])           # float64 path: the reference's precision
    np.testing.assert_allclose(y, c["y"], rtol=1e-12, atol=1e-12)
    y0 = bb.spmv_pull(raw, c["x"])
    np.testing.assert_allclose(y0, c["y_raw"], rtol=1e-12, atol=1e-12)
    # §8f: PageRank on the direct CSR (fp64; tolerance: summation order only)
    x, it = bb.pagerank(raw, return_iterations=True)
    assert it == c["pr_iters"][0], "pagerank iterations"
    np.testing.assert_allclose(x, c["pr"], rtol=PR_RTOL, atol=1e-14)
    # §8f: degree / hub orderings and the destination sort
    assert np.array_equal(bb.total_degrees(g), c["tdeg"]), "total_degrees"
    assert np.array_equal(bb.degree_order(g).order, c["deg_order"]), "degree_order"
    assert np.array_equal(bb.hub_order(g).order, c["hub_order"]), "hub_order"
    sd = bb.sort_coo_by_destination(g)
    assert np.array_equal(sd.I, c["I_sd"]) and np.array_equal(sd.J, c["J_sd"]), "sort_coo_by_destination"
    if c["w"] is not None:
        assert np.array_equal(sd.weights, c["w_sd"])
    # §8f f4: neighbourhood line ratio on the GPU (fp64 mean; summation order differs from numpy)
    if g.m:
        got = [bb.nbr(csr, 32), bb.nbr(csr, 4), bb.nbr(raw, 32)]
        np.testing.assert_allclose(got, c["nbr"], rtol=1e-12, atol=0)
    else:
        with pytest.raises(bb.UndefinedMetricError):
            bb.nbr(csr)


def test_known_answers(bb, kat):
    for c in kat:
        run_case(bb, c)


def test_fuzz(bb, fuzz):
    for c in fuzz:
        run_case(bb, c)


def test_medium(bb, medium):
    for c in medium:
        run_case(bb, c)


def test_thread_hint_never_changes_the_answer(bb, medium):
    c = medium.case(2)
    g = bb.CooGraph(c["n"], c["I"], c["J"])
    for t in (None, 1, 2, 8):
        assert np.array_equal(bb.boba_parallel(g, thread_hint=t).order, c["order"])
    assert np.array_equal(bb.compute_ordering(g, "boba", thread_hint=4).order, c["order"])


def test_relaxed_mode_invariants(bb, fuzz, medium):
    # reference test_ordering.py:79-111 / test_acceptance.py:152-184
    cases = [fuzz.case(i) for i in range(0, fuzz.count, 7)] + list(medium)
    for c in cases:
        g = bb.CooGraph(c["n"], c["I"], c["J"])
        p, r = bb.boba_parallel(g, mode="relaxed", thread_hint=8, return_ranks=True)
        assert p.is_valid()
        flat = np.concatenate([c["I"], c["J"]])
        present = np.zeros(g.n, dtype=bool)
        present[c["I"]] = True
        present[c["J"]] = True
        hit = r != RANK_UNSET
        assert np.array_equal(hit, present)
        k = int(hit.sum())
        assert np.unique(r[hit]).size == k
        assert np.array_equal(flat[r[p.order[:k]]], p.order[:k])
        assert np.all(np.diff(r[p.order[:k]]) > 0)
        assert np.all(np.diff(p.order[k:]) > 0)
        # relaxed with one 'thread' is the exact scan (test_ordering.py:72-77)
        assert np.array_equal(bb.boba_parallel(g, mode="relaxed", thread_hint=1).order, c["order"])


def test_errors(bb):
    with pytest.raises(ValueError):
        bb.boba_parallel(bb.CooGraph(1, [0], [0]), mode="yolo")
    with pytest.raises(bb.MalformedGraphError):
        bb.apply_permutation(bb.CooGraph(3, [0], [1]), bb.Permutation.identity(2))
    csr = bb.coo_to_csr(bb.CooGraph(3, [0], [1]))
    with pytest.raises(ValueError):
        bb.spmv_pull(csr, np.ones(2))
    # the seam's narrowing keeps the reference's range check
    from paper_2306_10410_b200 import _parallel

    with pytest.raises(bb.MalformedGraphError):
        _parallel.first_hit_chunked(np.array([0, 5]), np.array([1, 1]), 3, 4)


def test_seam_functions(bb, medium):
    from paper_2306_10410_b200 import _parallel as P

    c = medium.case(0)
    I, J, n = c["I"], c["J"], c["n"]
    r, order = P.first_hit_order_sequential(I, J, n)
    assert np.array_equal(order, c["order"]) and np.array_equal(r, c["r"])
    assert np.array_equal(P.first_hit_chunked(I, J, n, 8), c["r"])
    assert np.array_equal(P.first_hit_sequential(I, J, n), c["r"])
    assert np.array_equal(P.compact_ranks(c["r"], I, J), c["order"])
    idx, w = P.scatter_rows(c["I2"], c["J2"], None, c["offsets"])
    assert np.array_equal(idx, c["indices"]) and w is None


# ------------------------------------------------------------ device level

@pytest.fixture(scope="module")
def dev(bb):
    from paper_2306_10410_b200 import device

    return device


def to_np(t):
    return t.cpu().numpy().view(np.uint32).astype(np.int64)


@pytest.mark.parametrize("scale,ef", [(10, 8), (14, 4), (16, 8)])
def test_rmat_generator_matches_oracle(dev, scale, ef):
    I, J = dev.generate_rmat(scale, ef, seed=11)
    oI, oJ = oracle.rmat_edges(scale, ef, seed=11)
    assert np.array_equal(to_np(I), oI) and np.array_equal(to_np(J), oJ)


def test_grid_generator_matches_oracle(dev):
    for rows, cols in ((1, 1), (1, 5), (4, 1), (7, 9), (64, 64)):
        I, J = dev.generate_grid(rows, cols)
        oI, oJ = oracle.grid_edges(rows, cols)
        assert np.array_equal(to_np(I), oI) and np.array_equal(to_np(J), oJ)


def pipeline_vs_oracle(dev, I, J, n, threads=8):
    import torch

    pipe = dev.Pipeline(I.numel(), n).run(I, J)
    torch.cuda.synchronize()
    hI, hJ = to_np(I), to_np(J)
    order, label, I2, J2, off, idx, _ = oracle.pipeline(hI, hJ, n, threads=threads)
    m = I.numel()
    assert np.array_equal(to_np(pipe.order[:n]), order), "order"
    assert np.array_equal(to_np(pipe.label[:n]), label), "label"
    assert np.array_equal(to_np(pipe.I2[:m]), I2) and np.array_equal(to_np(pipe.J2[:m]), J2), "relabel"
    assert np.array_equal(to_np(pipe.offsets[: n + 1]), off), "offsets"
    assert np.array_equal(to_np(pipe.indices[:m]), idx), "indices"
    return pipe, off, idx


@pytest.mark.parametrize("scale,ef", [(12, 16), (18, 16), (20, 16)])
def test_rmat_pipeline_bit_exact(dev, scale, ef):
    import torch

    I, J = dev.generate_rmat(scale, ef, seed=1)
    n = 1 << scale
    # randomly relabelled like the BASELINE configs (reference io.py:294-301)
    lab = torch.from_numpy(oracle.random_labels(n, 7).astype(np.int32)).cuda()
    I, J = dev.gather(lab, I), dev.gather(lab, J)
    pipe, off, idx = pipeline_vs_oracle(dev, I, J, n)
    x = np.random.default_rng(5).random(n)
    xs = torch.from_numpy(x).cuda()
    want = oracle.spmv_pull(off, idx, x)
    y = dev.spmv(pipe.offsets[: n + 1], pipe.indices[: I.numel()], xs.float())   # fp32 (bench path)
    np.testing.assert_allclose(y.cpu().numpy(), want, rtol=SPMV_RTOL, atol=1e-5)
    y64 = dev.spmv(pipe.offsets[: n + 1], pipe.indices[: I.numel()], xs)         # fp64 (drop-in path)
    np.testing.assert_allclose(y64.cpu().numpy(), want, rtol=1e-12, atol=1e-12)


def test_grid_pipeline_bit_exact(dev):
    import torch

    I, J = dev.generate_grid(512, 512)
    n = 512 * 512
    lab = torch.from_numpy(oracle.random_labels(n, 7).astype(np.int32)).cuda()
    I, J = dev.gather(lab, I), dev.gather(lab, J)
    pipeline_vs_oracle(dev, I, J, n)


@pytest.mark.parametrize("n", [1, 2, 255, 256, 257, 2048, 2049, 4097, (1 << 22) + 1])
def test_radix_pass_boundaries(dev, n):
    import torch

    rng = np.random.default_rng(n)
    m = 5003
    I = torch.from_numpy(rng.integers(0, n, m).astype(np.int32)).cuda()
    J = torch.from_numpy(rng.integers(0, n, m).astype(np.int32)).cuda()
    pipeline_vs_oracle(dev, I, J, n)


@pytest.mark.parametrize("m", [0, 1, 2, 3, 4, 5, 7, 4099])
def test_tails_and_unaligned(dev, m):
    import torch

    rng = np.random.default_rng(m + 100)
    n = 37
    base = torch.from_numpy(rng.integers(0, n, 2 * m + 2).astype(np.int32)).cuda()
    I, J = base[1: m + 1], base[m + 2: 2 * m + 2]   # 4-byte (not 16-byte) aligned views
    if m == 0:
        I, J = base[:0], base[:0]
    pipeline_vs_oracle(dev, I, J, n)


def test_stability_property_at_scale(dev):
    """Within-row order == edge order at scale 22: carry the edge index as
    a float64 weight; every CSR row's weights must be strictly increasing."""
    import torch

    scale = 22
    I, J = dev.generate_rmat(scale, 16, seed=9)
    n, m = 1 << scale, I.numel()
    first, order, label = dev.boba_order(I, J, n)
    I2, J2 = dev.relabel(I, J, label, n)
    w = torch.arange(m, dtype=torch.float64, device=I.device)
    off, idx, w_out = dev.coo_to_csr(I2, J2, n, weights=w)
    off64 = off.to(torch.int64)
    rows = torch.repeat_interleave(torch.arange(n, device=I.device), off64[1:] - off64[:-1])
    e = w_out.to(torch.int64)
    same = rows[1:] == rows[:-1]
    assert bool(torch.all(e[1:][same] > e[:-1][same]))
    # the moved payload is exactly the edge list sorted by row
    assert bool(torch.all(idx == J2[e]))
    assert bool(torch.all(rows == I2.to(torch.int64)[e]))
    # permutation validity
    lab = label.to(torch.int64)
    assert bool(torch.all(torch.sort(lab).values == torch.arange(n, device=I.device)))
    assert bool(torch.all(lab[order.to(torch.int64)] == torch.arange(n, device=I.device)))


def test_spmv_determinism_and_integer_exactness(dev):
    import torch

    I, J = dev.generate_rmat(18, 16, seed=3)
    n = 1 << 18
    _, _, label = dev.boba_order(I, J, n)
    I2, J2 = dev.relabel(I, J, label, n)
    off, idx, _ = dev.coo_to_csr(I2, J2, n)
    xi = torch.randint(0, 4, (n,), device=I.device).to(torch.float32)
    y1 = dev.spmv(off, idx, xi)
    y2 = dev.spmv(off, idx, xi)
    assert torch.equal(y1, y2)
    want = oracle.spmv_pull(to_np(off), to_np(idx), xi.cpu().numpy().astype(np.float64))
    assert np.array_equal(y1.cpu().numpy().astype(np.float64), want)   # integer sums < 2^24: exact
    xr = torch.rand(n, device=I.device)
    assert torch.equal(dev.spmv(off, idx, xr), dev.spmv(off, idx, xr))
    # iterative form: later calls reuse the first call's partition (boba_spmv_ex)
    for x_ in (xr, xr.double()):
        ws = dev.spmv_workspace(n, I.numel(), I.device)
        dev.spmv(off, idx, x_, ws=ws)
        x2 = x_ * 3 + 1
        assert torch.equal(dev.spmv(off, idx, x2, ws=ws, reuse_partition=True), dev.spmv(off, idx, x2))
    with pytest.raises(ValueError):
        dev.spmv(off, idx, xr, reuse_partition=True)


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("n,mod", [(1, 1), (37, 2), (5000, 3), (70001, 1), (300000, 0)])
def test_spmv_vector_staging_edges(dev, n, mod, dtype):
    """SpMV (fp32 and fp64): the 16-byte staging path (aligned indices) and the scalar
    one (indices one element off alignment) give bitwise the same y, equal to
    the oracle on integer data; m = mod (mod 4) leaves a partial last quad;
    rows mix empty, short and tile-spanning hub rows."""
    import torch

    rng = np.random.default_rng(n + mod)
    deg = rng.choice([0, 1, 2, 3, 4, 7], size=n)
    deg[rng.integers(0, n, max(1, n // 5000))] += rng.integers(1000, 5000)   # hubs across tiles
    m = int(deg.sum())
    deg[0] += (mod - m) % 4
    m = int(deg.sum())
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(deg)
    idx = rng.integers(0, n, m)
    x = rng.integers(0, 4, n).astype(dtype)
    t_off = torch.from_numpy(off.astype(np.uint32).view(np.int32)).cuda()
    aligned = torch.from_numpy(idx.astype(np.uint32).view(np.int32)).cuda()
    buf = torch.empty(m + 1, dtype=torch.int32, device="cuda")
    buf[1:] = aligned
    shifted = buf[1:]                                     # 4 bytes past a 16-byte boundary
    xs = torch.from_numpy(x).cuda()
    y_vec = dev.spmv(t_off, aligned, xs)
    y_sca = dev.spmv(t_off, shifted, xs)
    assert torch.equal(y_vec, y_sca)
    want = oracle.spmv_pull(off, idx, x.astype(np.float64))
    assert np.array_equal(y_vec.cpu().numpy().astype(np.float64), want)


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("maxdeg", [8, 9])
@pytest.mark.parametrize("n", [1, 129, 70001])
def test_spmv_row_mode_switch(dev, n, maxdeg, dtype):
    """Row mode (no row longer than 8: one thread per row) and merge mode
    (a row of 9) on otherwise equal matrices: each equals the oracle exactly on
    integer data, weighted and not, fp32 and fp64; a workspace partitioned for
    one mode and re-partitioned for the other follows the new matrix (the
    mode is decided at partition time), and back."""
    import torch

    rng = np.random.default_rng(n * 10 + maxdeg)
    deg = rng.choice([0, 1, 2, 3, 4, 5, 8], size=n)
    deg[n // 2] = maxdeg
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(deg)
    m = int(off[-1])
    idx = rng.integers(0, n, m)
    x = rng.integers(0, 4, n).astype(dtype)
    wt = rng.integers(1, 3, m).astype(dtype)
    t = lambda a: torch.from_numpy(a.astype(np.uint32).view(np.int32)).cuda()  # noqa: E731
    t_off, t_idx, xs, ws_ = t(off), t(idx), torch.from_numpy(x).cuda(), torch.from_numpy(wt).cuda()
    want = oracle.spmv_pull(off, idx, x.astype(np.float64))
    want_w = oracle.spmv_pull(off, idx, x.astype(np.float64), wt.astype(np.float64))
    ws = dev.spmv_workspace(n, m, "cuda")
    y = dev.spmv(t_off, t_idx, xs, ws=ws)
    assert np.array_equal(y.cpu().numpy().astype(np.float64), want)
    yw = dev.spmv(t_off, t_idx, xs, weights=ws_, ws=ws, reuse_partition=True)
    assert np.array_equal(yw.cpu().numpy().astype(np.float64), want_w)
    # the other mode on the same workspace: one row grows past / shrinks to the bound
    deg2 = deg.copy()
    deg2[n // 2] = 17 - maxdeg
    off2 = np.zeros(n + 1, np.int64)
    off2[1:] = np.cumsum(deg2)
    idx2 = rng.integers(0, n, int(off2[-1]))
    y2 = dev.spmv(t(off2), t(idx2), xs, ws=ws)
    assert np.array_equal(y2.cpu().numpy().astype(np.float64), oracle.spmv_pull(off2, idx2, x.astype(np.float64)))
    y3 = dev.spmv(t_off, t_idx, xs, ws=ws)
    assert torch.equal(y3, y)


def test_spmv_row_mode_grid_float_and_pagerank(bb, dev):
    """The c3-shaped case (a grid: every row <= 4, row mode) with random x:
    fp32 within the north star's 1e-5 of the oracle's fp64 sums, bitwise
    repeatable; PageRank (fp64 SpMV iterations with the device stop flag) on
    the grid matches the oracle."""
    import torch

    I, J = dev.generate_grid(300, 257)
    n = 300 * 257
    off, idx, _ = dev.coo_to_csr(I, J, n)
    x = torch.rand(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
    y = dev.spmv(off, idx, x)
    want = oracle.spmv_pull(to_np(off), to_np(idx), x.cpu().numpy().astype(np.float64))
    np.testing.assert_allclose(y.cpu().numpy(), want, rtol=1e-5, atol=0)
    assert torch.equal(y, dev.spmv(off, idx, x))
    pr, it = dev.pagerank(off, idx)
    ex, eit = oracle.pagerank(to_np(off), to_np(idx), n)
    assert int(it.cpu()[0]) == eit
    np.testing.assert_allclose(pr.cpu().numpy(), ex, rtol=PR_RTOL, atol=1e-15)


def test_host_pipeline_matches_device(dev):
    import torch

    I, J = dev.generate_rmat(16, 8, seed=2)
    n, m = 1 << 16, I.numel()
    pipe = dev.Pipeline(m, n).run(I, J)
    hp = dev.HostPipeline(m, n)
    hI = I.cpu().numpy().view(np.uint32)
    hJ = J.cpu().numpy().view(np.uint32)
    order = np.empty(n, np.uint32)
    label = np.empty(n, np.uint32)
    off = np.empty(n + 1, np.uint32)
    idx = np.empty(m, np.uint32)
    hp.run(hI, hJ, n, order, label, off, idx)
    torch.cuda.synchronize()
    assert np.array_equal(order, pipe.order[:n].cpu().numpy().view(np.uint32))
    assert np.array_equal(off, pipe.offsets[: n + 1].cpu().numpy().view(np.uint32))
    assert np.array_equal(idx, pipe.indices[:m].cpu().numpy().view(np.uint32))
    hp.close()


@pytest.mark.parametrize("relabel_passes", [None, "3"])
def test_first_occurrence_waves_beyond_l2(dev, monkeypatch, relabel_passes):
    """n > 2^24: the fused pipeline's first-occurrence sweep guards on a
    seen-bitmap in waves of 2^26 positions (first[] no longer fits in L2).
    m = 2^26 edges -> 2^27 positions, two waves; the whole pipeline is
    checked against the oracle.  With BOBA_RL_PASSES the relabel runs as
    range passes (the default beyond n = 2^25) over the same graph."""
    import torch

    if relabel_passes:
        monkeypatch.setenv("BOBA_RL_PASSES", relabel_passes)

    scale = 25
    n = 1 << scale
    I, J = dev.generate_rmat(scale, 2, seed=21)
    lab = torch.from_numpy(oracle.random_labels(n, 5).astype(np.int32)).cuda()
    I, J = dev.gather(lab, I), dev.gather(lab, J)
    pipeline_vs_oracle(dev, I, J, n)


def test_relabel_range_passes_ragged(dev):
    """n = 2^25 + 5: the relabel runs as two range passes by default (label[]
    beyond 128 MiB) with a ragged split, and m = 3 mod 4 leaves a scalar tail;
    ids on both sides of the split and at the ends are present."""
    import torch

    n, m = (1 << 25) + 5, 3 * (1 << 20) + 3
    width = -(-n // 2)
    rng = np.random.default_rng(17)
    I = rng.integers(0, n, m, dtype=np.int64)
    J = rng.integers(0, n, m, dtype=np.int64)
    edge = np.array([0, width - 1, width, width + 1, n - 1, n - 2], dtype=np.int64)
    I[: edge.size], J[m - edge.size:] = edge, edge[::-1]
    t = lambda a: torch.from_numpy(a.astype(np.uint32).view(np.int32)).cuda()  # noqa: E731
    pipeline_vs_oracle(dev, t(I), t(J), n)


def test_captured_pipeline_replays_new_inputs(dev):
    """boba_reorder_to_csr_graph_create: the captured step reproduces the
    direct call, and replaying it after new edges are copied into the same
    input buffers gives the new graph's outputs (checked against the oracle)."""
    import torch

    scale = 14
    n = 1 << scale
    I, J = dev.generate_rmat(scale, 8, seed=3)
    m = I.numel()
    pipe = dev.Pipeline(m, n)
    g = dev.CapturedPipeline(pipe, I, J)
    u = lambda t: t.cpu().numpy().view(np.uint32).astype(np.int64)  # noqa: E731
    for seed in (3, 4, 5):
        I_new, J_new = dev.generate_rmat(scale, 8, seed=seed)
        I.copy_(I_new)
        J.copy_(J_new)
        g.launch()
        torch.cuda.synchronize()
        order, label, I2, J2, off, idx, _ = oracle.pipeline(u(I_new), u(J_new), n)
        assert np.array_equal(u(pipe.order[:n]), order) and np.array_equal(u(pipe.label[:n]), label)
        assert np.array_equal(u(pipe.I2[:m]), I2) and np.array_equal(u(pipe.J2[:m]), J2)
        assert np.array_equal(u(pipe.offsets[: n + 1]), off) and np.array_equal(u(pipe.indices[:m]), idx)
    g.close()


def test_host_pipeline_async_graphs_in_flight(dev):
    """boba_ctx_submit_host / boba_ctx_wait: five different graphs (different
    sizes too) submitted back to back through the two buffer slots; each
    graph's host outputs must equal the oracle's for that graph."""
    import torch

    graphs = []
    for k, (scale, ef) in enumerate([(12, 8), (14, 16), (10, 4), (13, 8), (12, 16)]):
        I, J = dev.generate_rmat(scale, ef, seed=10 + k)
        graphs.append((1 << scale, I.cpu().numpy().view(np.uint32).copy(), J.cpu().numpy().view(np.uint32).copy()))
    max_m = max(g[1].size for g in graphs)
    hp = dev.HostPipeline(max_m, 1 << 14)
    outs, tickets = [], []
    for n, hI, hJ in graphs:
        o = (np.empty(n, np.uint32), np.empty(n, np.uint32), np.empty(n + 1, np.uint32), np.empty(hI.size, np.uint32))
        outs.append(o)
        tickets.append(hp.submit(hI, hJ, n, *o))
    for t in tickets:
        hp.wait(t)
    torch.cuda.synchronize()
    for (n, hI, hJ), (order, label, off, idx) in zip(graphs, outs):
        o_order, o_label, _, _, o_off, o_idx, _ = oracle.pipeline(hI.astype(np.int64), hJ.astype(np.int64), n)
        assert np.array_equal(order, o_order) and np.array_equal(label, o_label)
        assert np.array_equal(off, o_off) and np.array_equal(idx, o_idx)
    hp.close()


@pytest.mark.parametrize("scale,ef", [(12, 16), (20, 16)])
def test_degree_orders_and_destination_sort_vs_oracle(bb, dev, scale, ef):
    """R-MAT (heavy ties in degree) through the C ABI vs the oracle."""
    import torch

    I, J = dev.generate_rmat(scale, ef, seed=5)
    n = 1 << scale
    hI, hJ = to_np(I), to_np(J)
    deg = dev.total_degrees(I, J, n)
    assert np.array_equal(to_np(deg), oracle.total_degrees(hI, hJ, n))
    for hub in (False, True):
        order, label = dev.degree_order(I, J, n, hub=hub)
        want = oracle.degree_order(hI, hJ, n, hub=hub)
        assert np.array_equal(to_np(order), want)
        assert np.array_equal(to_np(label), oracle.label_from_order(want))
    w = torch.rand(I.numel(), dtype=torch.float64, device=I.device)
    Io, Jo, wo = dev.sort_coo_by_destination(I, J, n, w)
    eI, eJ, ew = oracle.sort_coo_by_destination(hI, hJ, n, w.cpu().numpy())
    assert np.array_equal(to_np(Io), eI) and np.array_equal(to_np(Jo), eJ)
    assert np.array_equal(wo.cpu().numpy(), ew)
    Io, Jo, _ = dev.sort_coo_by_destination(I, J, n)
    assert np.array_equal(to_np(Io), eI) and np.array_equal(to_np(Jo), eJ)


def test_degree_order_edge_cases(bb):
    g = bb.CooGraph(5, [], [])
    assert bb.degree_order(g).order.tolist() == [0, 1, 2, 3, 4]
    assert bb.hub_order(g).order.tolist() == [0, 1, 2, 3, 4]
    g = bb.CooGraph(1, [0], [0])
    assert bb.degree_order(g).order.tolist() == [0]
    g = bb.CooGraph(0, [], [])
    assert bb.degree_order(g).order.size == 0
    star = bb.CooGraph(5, [0, 0, 0, 0], [1, 2, 3, 4])
    assert bb.compute_ordering(star, "degree").order.tolist() == [0, 1, 2, 3, 4]
    assert bb.compute_ordering(star, "hub").order.tolist() == [0, 1, 2, 3, 4]
    g = bb.CooGraph(4, [3, 3, 2], [1, 1, 3])
    assert bb.compute_ordering(g, "degree").order.tolist() == [3, 1, 2, 0]
    assert bb.DegreeOrder().fit(g).permutation_.order.tolist() == [3, 1, 2, 0]
    assert bb.HubOrder().fit(g).permutation_.order.tolist() == [3, 1, 0, 2]
    sd = bb.sort_coo_by_destination(bb.CooGraph(4, [0, 1, 2, 3], [2, 0, 2, 0], [1.0, 2.0, 3.0, 4.0]))
    assert sd.I.tolist() == [1, 3, 0, 2] and sd.weights.tolist() == [2.0, 4.0, 1.0, 3.0]


@pytest.mark.parametrize("weighted", [False, True])
def test_pagerank_rmat_vs_oracle(bb, dev, weighted):
    import torch

    scale = 16
    I, J = dev.generate_rmat(scale, 8, seed=3)
    n = 1 << scale
    w = torch.rand(I.numel(), dtype=torch.float64, device=I.device) if weighted else None
    off, idx, w2 = dev.coo_to_csr(I, J, n, w)
    x, it = dev.pagerank(off, idx, w2)
    ho, hi = to_np(off), to_np(idx)
    ex, eit = oracle.pagerank(ho, hi, n, None if w2 is None else w2.cpu().numpy())
    assert int(it.cpu()[0]) == eit
    np.testing.assert_allclose(x.cpu().numpy(), ex, rtol=PR_RTOL, atol=1e-15)
    assert abs(x.sum().item() - 1.0) < 1e-9
    x2, _ = dev.pagerank(off, idx, w2)
    assert torch.equal(x, x2), "PageRank must be bitwise deterministic"


def test_pagerank_edge_cases(bb):
    g = bb.CooGraph(3, [0, 1], [1, 2])
    csr = bb.coo_to_csr(g)
    x, it = bb.pagerank(csr, max_iters=0, return_iterations=True)
    assert it == 0 and np.allclose(x, 1 / 3)
    x, it = bb.pagerank(csr, max_iters=1, return_iterations=True)
    ex, eit = oracle.pagerank(csr.offsets, csr.indices, 3, max_iters=1)
    assert it == eit == 1 and np.allclose(x, ex, rtol=1e-14)
    x = bb.pagerank(bb.coo_to_csr(bb.CooGraph(4, [], [])))
    assert np.allclose(x, 0.25)
    assert bb.pagerank(bb.coo_to_csr(bb.CooGraph(0, [], []))).size == 0
    for d in (0.0, 1.0, -0.5):
        with pytest.raises(ValueError):
            bb.pagerank(csr, damping=d)


@pytest.mark.parametrize("scale,with_counts", [(18, True), (18, False), (22, True), (22, False)])
def test_first_occurrence_seen_set_paths(dev, scale, with_counts):
    """The two-stage sweep's SeenSet is filled from a counting prefix (most
    frequent first-seen vertices first) when the caller's workspace has room
    for the count table, and from the prefix's first-seen vertices otherwise
    (boba_first_occurrence_shard with only the SeenSet workspace).  Both are
    pure filters: first[] equals the reference's r either way.  s22 takes the
    8-bit tags, s18 the 16-bit ones (reference _parallel.py:111-136)."""
    import torch

    from paper_2306_10410_b200 import _native as N

    n = 1 << scale
    I, J = dev.generate_rmat(scale, 16, seed=3)
    lab = torch.from_numpy(oracle.random_labels(n, 9).astype(np.int32)).cuda()
    I, J = dev.gather(lab, I), dev.gather(lab, J)
    m = I.numel()
    size = (N.lib.boba_first_occurrence_shard_workspace_size(n) if with_counts
            else N.lib.boba_first_occurrence_workspace_size())
    ws = torch.empty(size, dtype=torch.uint8, device="cuda")
    first = torch.empty(n, dtype=torch.int32, device="cuda")
    N.check(N.lib.boba_first_occurrence_shard(dev._p(I), dev._p(J), m, m, 0, n, dev._p(first), 0, dev._p(ws),
                                              ws.numel(), dev._s()))
    r, _ = oracle.first_hit_order_sequential(to_np(I), to_np(J), n)
    want = np.where(r == oracle.RANK_UNSET, 0xFFFFFFFF, r).astype(np.uint32)
    assert np.array_equal(to_np(first).astype(np.uint32), want)


def test_sixteen_bit_static_sweep_without_waves(dev):
    """n = 2^23: SeenSet tags are 16-bit (ids wider than 2^22) and first[]
    (32 MB) still guards the sweep directly -- no waves (those start above
    2^23).  The whole pipeline against the oracle (reference
    _parallel.py:111-136, graph.py:253-289)."""
    import torch

    scale = 23
    n = 1 << scale
    I, J = dev.generate_rmat(scale, 4, seed=4)
    lab = torch.from_numpy(oracle.random_labels(n, 11).astype(np.int32)).cuda()
    I, J = dev.gather(lab, I), dev.gather(lab, J)
    pipeline_vs_oracle(dev, I, J, n)


@pytest.mark.parametrize("m", [0, 1, 4999, 5000])
def test_many_vertices_few_edges(dev, m):
    """n = 2^25 + 3 with a few thousand edges: nearly every vertex is
    isolated, the range-pass relabel and 26-bit radix keys run on a tiny edge
    list, and the never-seen vertices fill the tail of the order in ascending
    id (reference _parallel.py:132-135, 197-200)."""
    import torch

    n = (1 << 25) + 3
    rng = np.random.default_rng(m + 7)
    I = rng.integers(0, n, m, dtype=np.int64)
    J = rng.integers(0, n, m, dtype=np.int64)
    if m:
        I[0], J[-1] = n - 1, 0
    t = lambda a: torch.from_numpy(a.astype(np.uint32).view(np.int32)).cuda()  # noqa: E731
    pipeline_vs_oracle(dev, t(I), t(J), n)


@pytest.mark.parametrize("logn", [18, 22])
def test_captured_pipeline_picks_the_radix_plan_per_replay(dev, logn):
    """The captured step carries both COO->CSR pass plans behind a conditional
    node: the one with a key bit less when every source row is below
    2^(kbits-1) (decided on the device from the count of vertices first seen
    in I), the full-width one otherwise.  Replays that need each plan, in both
    orders, against the oracle (reference graph.py:253-277).  At n = 2^18 the
    two plans share their first pass (6/6/6 vs 6/6/5 bits); at 2^22 they do
    not (8/7/7 vs 7/7/7) and the whole sort sits in the branches."""
    import torch

    n, m = 1 << logn, 1 << 20
    rng = np.random.default_rng(23)

    def edges(sources):   # the first-seen-in-I count is about `sources`
        I = rng.integers(0, n, sources)[rng.integers(0, sources, m)]
        J = rng.integers(0, n, m)
        return (torch.from_numpy(I.astype(np.uint32).view(np.int32)).cuda(),
                torch.from_numpy(J.astype(np.uint32).view(np.int32)).cuda())

    narrow, wide = edges(n // 4), edges(3 * n // 4)   # rows < n/2 (a key bit less), rows beyond it
    I, J = narrow[0].clone(), narrow[1].clone()
    pipe = dev.Pipeline(m, n)
    g = dev.CapturedPipeline(pipe, I, J)
    u = lambda t: t.cpu().numpy().view(np.uint32).astype(np.int64)  # noqa: E731
    for I_new, J_new in (wide, narrow, wide):
        I.copy_(I_new)
        J.copy_(J_new)
        g.launch()
        torch.cuda.synchronize()
        order, label, I2, J2, off, idx, _ = oracle.pipeline(u(I_new), u(J_new), n)
        assert np.array_equal(u(pipe.order[:n]), order) and np.array_equal(u(pipe.label[:n]), label)
        assert np.array_equal(u(pipe.offsets[: n + 1]), off) and np.array_equal(u(pipe.indices[:m]), idx)
    g.close()
