"""GPU side of the multi-GPU path: every device op the sharded pipeline uses
(shard first occurrence with global offsets, order-preserving bias, windowed
compaction, order from label, coarse row cut, relative range partition)
against its numpy twin with P logical shards emulated on one GPU; the full
sharded pipeline + row-partitioned SpMV through a one-rank NCCL group; and
the whole N > 1 flow with 2 and 3 processes sharing the GPU over gloo."""

import os
import socket

import numpy as np
import pytest

import oracle
from test_sharded_gloo import NumpyOps, check_parts, t32, u32

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2306_10410_b200.sharded import DeviceOps

    return DeviceOps()


def cu(a):
    return t32(a).cuda()


def host(t):
    return u32(t.cpu())


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("P", [2, 4, 7])
def test_shard_first_occurrence_merges_to_global(ops, P):
    from paper_2306_10410_b200.sharded import shard_range

    I, J = oracle.rmat_edges(14, 8, seed=9)
    n, m = 1 << 14, I.size
    r_ref, _ = oracle.first_hit_order_sequential(I, J, n)
    want = np.where(r_ref == np.iinfo(np.int64).max, 0xFFFFFFFF, r_ref).astype(np.uint32)
    npo = NumpyOps()
    merged = None
    for k in range(P):
        e0, e1 = shard_range(m, k, P)
        f = ops.first_occurrence_shard(cu(I[e0:e1]), cu(J[e0:e1]), m, e0, n)
        assert np.array_equal(host(f), u32(npo.first_occurrence_shard(t32(I[e0:e1]), t32(J[e0:e1]), m, e0, n)))
        b = host(ops.bias(f)).view(np.int32)
        merged = b if merged is None else np.minimum(merged, b)   # the allreduce-MIN, signed
    got = host(ops.bias(cu(merged.view(np.uint32))))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("P,scale", [(1, 12), (3, 14), (8, 16)])
def test_windowed_compaction_sums_to_global_label(ops, P, scale):
    """P2 with P emulated ranks: per-window counts, partial labels, their
    SUM == the reference's label; order from label; each piece == its twin."""
    import torch

    from paper_2306_10410_b200.sharded import shard_range

    I, J = oracle.rmat_edges(scale, 4, seed=3)
    n = 1 << scale
    n += 777                                     # isolated vertices beyond the R-MAT id range
    m = I.size
    r, order = oracle.first_hit_order_sequential(I, J, n)
    label = oracle.label_from_order(order)
    first = cu(np.where(r == np.iinfo(np.int64).max, 0xFFFFFFFF, r))
    npo = NumpyOps()
    counts, wss = [], []
    for k in range(P):
        e0, e1 = shard_range(m, k, P)
        c, ws = ops.compact_shard_mark(first, n, m, e0, e1 - e0)
        wc, _ = npo.compact_shard_mark(first.cpu(), n, m, e0, e1 - e0)
        assert np.array_equal(host(c), u32(wc))
        counts.append(host(c))
        wss.append(ws)
    all_counts = np.concatenate(counts)
    total = np.zeros(n, dtype=np.uint64)
    for k in range(P):
        e0, e1 = shard_range(m, k, P)
        part = ops.compact_shard_assign(first, n, m, e0, e1 - e0, cu(all_counts), P, k, wss[k])
        twin = npo.compact_shard_assign(first.cpu(), n, m, e0, e1 - e0, t32(all_counts), P, k, None)
        assert np.array_equal(host(part), u32(twin)), k
        total += host(part)
    assert np.array_equal(total.astype(np.int64), label)
    o, hubs = ops.order_from_label(cu(label), n)
    assert np.array_equal(host(o), order)
    # relabel with the table order_from_label built == the plain gather
    I2, J2 = ops.relabel(cu(I), cu(J), cu(label), hubs, n)
    assert np.array_equal(host(I2), label[I]) and np.array_equal(host(J2), label[J])
    del torch


@pytest.mark.parametrize("n", [5000, 70001, 1 << 22])
def test_row_cut_and_relative_partition(ops, n):
    rng = np.random.default_rng(n)
    P = 5
    rows_g = np.minimum(rng.zipf(1.3, 300001) - 1, n - 1)     # skewed: heavy small rows
    local = rows_g[:120007]
    cols = rng.integers(0, n, local.size)
    npo = NumpyOps()
    hl, hg = ops.row_cut_hist(cu(local), n), ops.row_cut_hist(cu(rows_g), n)
    assert np.array_equal(host(hl), u32(npo.row_cut_hist(t32(local), n)))
    cut = ops.row_cut(hg, hl, n, rows_g.size, P)
    want = u32(npo.row_cut(t32(host(hg)), t32(host(hl)), n, rows_g.size, P))
    assert np.array_equal(host(cut), want)
    b = want[:P + 1].astype(np.int64)
    assert b[0] == 0 and b[P] == n and np.all(np.diff(b) >= 0)
    send = want[2 * P + 2:].astype(np.int64)
    assert send.sum() == local.size
    assert np.array_equal(send, np.bincount(np.searchsorted(b[1:P], local, side="right"), minlength=P))
    ko, vo = ops.range_partition(cu(local), cu(cols), cut[:P + 1], P)
    wk, wv = npo.range_partition(t32(local), t32(cols), t32(b), P)
    assert np.array_equal(host(ko), u32(wk)) and np.array_equal(host(vo), u32(wv))
    # the owner's two-step CSR (row histogram first, while the columns arrive) == one call == numpy
    want_off, want_idx = npo.coo_to_csr(t32(local), t32(cols), n)
    st = ops.coo_to_csr_begin(cu(local), n)
    o2, i2 = ops.coo_to_csr_finish(st, cu(local), cu(cols), n)
    o1, i1 = ops.coo_to_csr(cu(local), cu(cols), n)
    assert np.array_equal(host(o2), u32(want_off)) and np.array_equal(host(i2), u32(want_idx))
    assert np.array_equal(host(o1), host(o2)) and np.array_equal(host(i1), host(i2))


def test_sharded_pipeline_one_rank_nccl(ops):
    import torch
    import torch.distributed as dist

    from paper_2306_10410_b200.sharded import ShardedPipeline, sharded_spmv

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        I, J = oracle.rmat_edges(16, 8, seed=2)
        n = 1 << 16
        lab = oracle.random_labels(n, 7)
        I, J = lab[I], lab[J]
        sp = ShardedPipeline(n, I.size, 0, I.size, torch.device("cuda", 0))
        res = sp.run(cu(I), cu(J))
        order, label, I2, J2, off, idx, _ = oracle.pipeline(I, J, n)
        assert np.array_equal(host(res.order), order) and np.array_equal(host(res.label), label)
        assert np.array_equal(host(res.I2), I2) and np.array_equal(host(res.J2), J2)
        assert (res.row_lo, res.row_hi) == (0, n)
        assert np.array_equal(host(res.offsets), off) and np.array_equal(host(res.indices), idx)
        x = np.random.default_rng(1).random(n, dtype=np.float32)
        y = sharded_spmv(res, torch.from_numpy(x).cuda(), 1).cpu().numpy()
        np.testing.assert_allclose(y, oracle.spmv_pull(off, idx, x.astype(np.float64)), rtol=1e-5, atol=0)
        # the same pipeline through the one-call C-ABI entry on torch's NCCL communicator
        from paper_2306_10410_b200.sharded import native_sharded_reorder_to_csr

        nat = native_sharded_reorder_to_csr(cu(I), cu(J), n, I.size, 0)
        torch.cuda.synchronize()
        assert np.array_equal(host(nat.order), order) and np.array_equal(host(nat.label), label)
        assert np.array_equal(host(nat.I2), I2) and np.array_equal(host(nat.J2), J2)
        assert (nat.row_lo, nat.row_hi, nat.row_edge_offset) == (0, n, 0) and nat.bounds == [0, n]
        assert np.array_equal(host(nat.offsets), off) and np.array_equal(host(nat.indices), idx)
        small = native_sharded_reorder_to_csr(cu(I), cu(J), n, I.size, 0, recv_capacity=100)   # grows and retries
        assert np.array_equal(host(small.indices), idx)
        ph = sp.phase_times(cu(I), cu(J))
        assert set(ph) == set(sp.PHASES) | {"step"}
        assert all(ph[k]["ms"] > 0 and 0 <= ph[k]["comm_ms"] <= ph[k]["ms"] for k in sp.PHASES)
        assert ph["step"]["compute_only_ms"] + ph["step"]["comm_only_ms"] == pytest.approx(ph["step"]["actual_ms"],
                                                                                            abs=1e-3)
        assert sp.spmv_timing(res, 2)["ms_per_iter"] > 0
        # P5 with the slice exchange overlapped piece by piece: the same rows and sums
        yc = sharded_spmv(res, torch.from_numpy(x).cuda(), 1, chunks=4).cpu().numpy()
        np.testing.assert_allclose(yc, oracle.spmv_pull(off, idx, x.astype(np.float64)), rtol=1e-5, atol=0)
        assert sp.spmv_timing(res, 2, chunks=4)["chunks"] == 4
        assert sp.comm_bytes()["total"] >= 0 and sp.kernel_launches_per_step() > 10
    finally:
        dist.destroy_process_group()


def _gpu_worker(rank, world, port, cases, outdir):
    import torch
    import torch.distributed as dist

    from paper_2306_10410_b200.sharded import shard_range, sharded_reorder_to_csr, sharded_spmv

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for name, (I, J, n) in cases.items():
            m = I.size
            e0, e1 = shard_range(m, rank, world)
            res = sharded_reorder_to_csr(cu(I[e0:e1]), cu(J[e0:e1]), n, m, e0)
            x0 = torch.from_numpy((np.arange(n) % 7 + 1).astype(np.float32)).cuda()
            y2 = sharded_spmv(res, x0, 2)
            y2c = sharded_spmv(res, x0, 2, chunks=3)   # exchange overlapped with the multiply
            torch.cuda.synchronize()
            np.savez(os.path.join(outdir, f"{name}_r{rank}.npz"), order=host(res.order), label=host(res.label),
                     I2=host(res.I2), J2=host(res.J2), lo=res.row_lo, hi=res.row_hi, offsets=host(res.offsets),
                     indices=host(res.indices), goff=res.row_edge_offset, bounds=np.array(res.bounds),
                     y2=y2.cpu().numpy(), y2c=y2c.cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_pipeline_ranks_share_one_gpu(ops, world, tmp_path):
    """The whole sharded pipeline with world_size > 1 on the real device ops:
    `world` processes share cuda:0 and exchange over gloo (NCCL refuses two
    ranks on one device), so every kernel of the N > 1 path -- shard first
    occurrence, biased MIN merge, windowed compaction, label SUM, relabel,
    coarse row cut, relative range partition, all-to-all, owner CSR,
    row-partitioned SpMV -- runs on the B200 and the assembled outputs are
    checked against the oracle."""
    import torch.multiprocessing as mp

    I, J = oracle.rmat_edges(15, 8, seed=6)
    n = 1 << 15
    lab = oracle.random_labels(n, 3)
    rng = np.random.default_rng(8)
    cases = {"rmat": (lab[I], lab[J], n),
             "isolated": (rng.integers(0, 3000, 40003), rng.integers(0, 3500, 40003), 5000),
             "coarse_buckets": (rng.integers(0, 90000, 50001), rng.integers(0, 90000, 50001), 90000)}
    mp.spawn(_gpu_worker, args=(world, _port(), cases, str(tmp_path)), nprocs=world, join=True)
    for name, (I, J, n) in cases.items():
        parts = [dict(np.load(os.path.join(tmp_path, f"{name}_r{k}.npz"))) for k in range(world)]
        off, idx = check_parts(parts, I, J, n, name)
        x = (np.arange(n) % 7 + 1).astype(np.float64)
        y = oracle.spmv_pull(off, idx, oracle.spmv_pull(off, idx, x))
        for p in parts:
            np.testing.assert_allclose(p["y2"], y, rtol=1e-5, atol=0)
            np.testing.assert_allclose(p["y2c"], y, rtol=1e-5, atol=0)
