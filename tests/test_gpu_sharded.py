"""GPU side of the multi-GPU path: the device ops the sharded pipeline uses
(shard first-occurrence with global offsets, order-preserving bias, range
partition, id offset, exclusive scan) against their numpy twins, P logical
shards emulated on one GPU, and the full sharded pipeline through a one-rank
NCCL group."""

import os
import socket

import numpy as np
import pytest

import oracle
from test_sharded_gloo import NumpyOps, t32, u32

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


def test_range_partition_and_helpers(ops):
    rng = np.random.default_rng(4)
    n, m = 5000, 40001
    keys = rng.integers(0, n, m)
    vals = rng.integers(0, 1 << 31, m)
    bounds = np.array([0, 0, 1200, 1201, 4000, n])        # includes an empty part
    npo = NumpyOps()
    ko, vo, c = ops.range_partition(cu(keys), cu(vals), cu(bounds), 5)
    wk, wv, wc = npo.range_partition(t32(keys), t32(vals), t32(bounds), 5)
    assert np.array_equal(host(ko), u32(wk)) and np.array_equal(host(vo), u32(wv))
    assert np.array_equal(host(c), u32(wc))
    assert np.array_equal(host(ops.offset_ids(cu(keys), -1200)), u32(npo.offset_ids(t32(keys), -1200)))
    counts = np.bincount(keys, minlength=n)
    assert np.array_equal(host(ops.exclusive_scan(cu(counts))), u32(npo.exclusive_scan(t32(counts))))


@pytest.mark.parametrize("P", [1, 3, 8])
def test_merge_rows_matches_twin(ops, P):
    """Receiver side of the row-range all-to-all: P senders' local CSRs of
    contiguous edge shards, restricted to one owner's row range, interleaved
    row by row in rank order == the single-process CSR of those rows."""
    from paper_2306_10410_b200.sharded import shard_range

    I, J = oracle.rmat_edges(13, 8, seed=11)
    n, m = 1 << 13, I.size
    _, _, _, _, off, idx, _ = oracle.pipeline(I, J, n)
    off_g, idx_g = oracle.coo_to_csr(I, J, n)[:2]
    lo, hi = 1000, 5000                                   # this owner's rows
    npo = NumpyOps()
    runs, rcs = [], []
    for k in range(P):
        e0, e1 = shard_range(m, k, P)
        lo_off, lo_idx = ops.coo_to_csr(cu(I[e0:e1]), cu(J[e0:e1]), n)
        rc = ops.adjacent_diff(lo_off)
        assert np.array_equal(host(rc), u32(npo.adjacent_diff(t32(host(lo_off)))))
        o = host(lo_off).astype(np.int64)
        runs.append(host(lo_idx)[o[lo]:o[hi]])
        rcs.append(host(rc)[lo:hi])
    recv, counts = np.concatenate(runs), np.concatenate(rcs)
    out_off = (off_g[lo:hi + 1] - off_g[lo]).astype(np.uint32)
    got = host(ops.merge_rows(cu(recv), cu(counts), P, hi - lo, cu(out_off)))
    assert np.array_equal(got, u32(npo.merge_rows(t32(recv), t32(counts), P, hi - lo, t32(out_off))))
    assert np.array_equal(got, idx_g[off_g[lo]:off_g[hi]].astype(np.uint32))


def test_sharded_pipeline_one_rank_nccl(ops):
    import torch
    import torch.distributed as dist

    from paper_2306_10410_b200.sharded import sharded_reorder_to_csr

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        I, J = oracle.rmat_edges(16, 8, seed=2)
        n = 1 << 16
        lab = oracle.random_labels(n, 7)
        I, J = lab[I], lab[J]
        res = sharded_reorder_to_csr(cu(I), cu(J), n, I.size, 0)
        order, label, I2, J2, off, idx, _ = oracle.pipeline(I, J, n)
        assert np.array_equal(host(res.order), order) and np.array_equal(host(res.label), label)
        assert np.array_equal(host(res.I2), I2) and np.array_equal(host(res.J2), J2)
        assert (res.row_lo, res.row_hi) == (0, n)
        assert np.array_equal(host(res.offsets), off) and np.array_equal(host(res.indices), idx)
    finally:
        dist.destroy_process_group()


def _gpu_worker(rank, world, port, cases, outdir):
    import torch
    import torch.distributed as dist

    from paper_2306_10410_b200.sharded import shard_range, sharded_reorder_to_csr

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for name, (I, J, n) in cases.items():
            m = I.size
            e0, e1 = shard_range(m, rank, world)
            res = sharded_reorder_to_csr(cu(I[e0:e1]), cu(J[e0:e1]), n, m, e0)
            torch.cuda.synchronize()
            np.savez(os.path.join(outdir, f"{name}_r{rank}.npz"), order=host(res.order), label=host(res.label),
                     I2=host(res.I2), J2=host(res.J2), lo=res.row_lo, hi=res.row_hi, offsets=host(res.offsets),
                     indices=host(res.indices))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_pipeline_ranks_share_one_gpu(ops, world, tmp_path):
    """The whole sharded pipeline with world_size > 1 on the real device ops:
    `world` processes share cuda:0 and exchange over gloo (NCCL refuses two
    ranks on one device), so every kernel of the N > 1 path -- shard first
    occurrence, biased MIN merge, replicated compaction, local CSR, row-range
    partition, all-to-all, row merge -- runs on the B200 and the assembled
    row-partitioned CSR is checked against the oracle."""
    import torch.multiprocessing as mp

    I, J = oracle.rmat_edges(15, 8, seed=6)
    n = 1 << 15
    lab = oracle.random_labels(n, 3)
    rng = np.random.default_rng(8)
    cases = {"rmat": (lab[I], lab[J], n),
             "isolated": (rng.integers(0, 3000, 40003), rng.integers(0, 3500, 40003), 5000)}
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_gpu_worker, args=(world, port, cases, str(tmp_path)), nprocs=world, join=True)
    for name, (I, J, n) in cases.items():
        parts = [dict(np.load(os.path.join(tmp_path, f"{name}_r{k}.npz"))) for k in range(world)]
        order, label, I2, J2, off, idx, _ = oracle.pipeline(I, J, n)
        for p in parts:
            assert np.array_equal(p["order"], order) and np.array_equal(p["label"], label), name
        assert np.array_equal(np.concatenate([p["I2"] for p in parts]), I2), name
        assert np.array_equal(np.concatenate([p["J2"] for p in parts]), J2), name
        assert parts[0]["lo"] == 0 and parts[-1]["hi"] == n, name
        for p in parts:
            lo, hi = int(p["lo"]), int(p["hi"])
            assert np.array_equal(p["offsets"].astype(np.int64) + off[lo], off[lo:hi + 1]), name
            assert np.array_equal(p["indices"], idx[off[lo]:off[hi]]), name
