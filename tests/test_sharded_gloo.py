"""Multi-process check of the sharded (multi-GPU) pipeline's collective logic
on CPU: world_size 2 and 3 over gloo, with the local phases emulated in numpy
(the GPU kernels cannot run here).  The assembled per-rank outputs must equal
the oracle's single-process pipeline bit for bit: replicated permutation,
relabelled COO shards, and the row-partitioned CSR."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
from conftest import ROOT

U32 = np.uint32


def u32(t):
    return t.numpy().view(U32)


def t32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=U32).view(np.int32))


class NumpyOps:
    """The DeviceOps interface of paper_2306_10410_b200.sharded, in numpy."""

    def first_occurrence_shard(self, I, J, m_global, e0, n):
        f = np.full(n, 0xFFFFFFFF, dtype=np.uint64)
        I, J = u32(I).astype(np.int64), u32(J).astype(np.int64)
        pos = np.arange(I.size, dtype=np.uint64)
        np.minimum.at(f, I, pos + e0)
        np.minimum.at(f, J, pos + m_global + e0)
        return t32(f.astype(U32))

    def bias(self, t):
        return t32(u32(t) ^ U32(0x80000000))

    def compact(self, first, m_global, n):
        f = u32(first)
        order = np.argsort(f, kind="stable")  # present by first position, then isolated ascending
        label = np.empty(n, dtype=np.int64)
        label[order] = np.arange(n)
        return t32(order), t32(label)

    def relabel(self, I, J, label, n):
        lab = u32(label)
        return t32(lab[u32(I)]), t32(lab[u32(J)])

    def compact_relabel(self, first, I, J, m_global, n):
        order, label = self.compact(first, m_global, n)
        return (order, label) + self.relabel(I, J, label, n)

    def degrees(self, I2, n):
        return t32(np.bincount(u32(I2), minlength=n))

    def exclusive_scan(self, counts):
        c = u32(counts).astype(np.int64)
        return t32(np.concatenate([[0], np.cumsum(c)]))

    def range_partition(self, keys, vals, bounds, parts):
        k, v = u32(keys), u32(vals)
        b = u32(bounds).astype(np.int64)
        owner = np.searchsorted(b[1:parts], k, side="right")
        o = np.argsort(owner, kind="stable")
        return t32(k[o]), t32(v[o]), t32(np.bincount(owner, minlength=parts))

    def offset_ids(self, t, delta):
        return t32((u32(t).astype(np.int64) + delta) & 0xFFFFFFFF)

    def coo_to_csr(self, rows, cols, n_rows):
        r, c = u32(rows).astype(np.int64), u32(cols)
        o = np.argsort(r, kind="stable")
        off = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=n_rows))])
        return t32(off), t32(c[o])

    def adjacent_diff(self, t):
        a = u32(t).astype(np.int64)
        return t32((a[1:] - a[:-1]) & 0xFFFFFFFF)

    def merge_rows(self, recv, counts, parts, rows, out_offsets):
        rv, cnt = u32(recv), u32(counts).astype(np.int64).reshape(parts, rows)
        off = u32(out_offsets).astype(np.int64)
        src = np.concatenate([[0], np.cumsum(cnt.ravel())])[:-1].reshape(parts, rows)
        out = np.empty(rv.size, dtype=U32)
        for r in range(rows):
            d = off[r]
            for k in range(parts):
                out[d:d + cnt[k, r]] = rv[src[k, r]:src[k, r] + cnt[k, r]]
                d += cnt[k, r]
        return t32(out)


def _worker(rank, world, port, cases, outdir):
    import torch.distributed as dist

    from paper_2306_10410_b200.sharded import shard_range, sharded_reorder_to_csr

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    for name, (I, J, n) in cases.items():
        m = I.size
        e0, e1 = shard_range(m, rank, world)
        res = sharded_reorder_to_csr(t32(I[e0:e1]), t32(J[e0:e1]), n, m, e0, ops=NumpyOps())
        np.savez(os.path.join(outdir, f"{name}_r{rank}.npz"), first=u32(res.first), order=u32(res.order),
                 label=u32(res.label), I2=u32(res.I2), J2=u32(res.J2), lo=res.row_lo, hi=res.row_hi,
                 offsets=u32(res.offsets), indices=u32(res.indices), goff=u32(res.global_offsets))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def make_cases():
    I, J = oracle.rmat_edges(12, 8, seed=5)
    n = 1 << 12
    lab = oracle.random_labels(n, 7)
    rng = np.random.default_rng(3)
    return {
        "rmat": (lab[I], lab[J], n),
        "fuzz_isolated": (rng.integers(0, 600, 5001), rng.integers(0, 700, 5001), 900),  # many isolated
        "tiny": (np.array([5, 5, 3]), np.array([3, 1, 5]), 6),                            # test_ordering.py:37-40
        "fewer_edges_than_ranks": (np.array([1]), np.array([0]), 3),
    }


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_pipeline_matches_oracle(world, tmp_path):
    cases = make_cases()
    mp.spawn(_worker, args=(world, _free_port(), cases, str(tmp_path)), nprocs=world, join=True)
    for name, (I, J, n) in cases.items():
        parts = [dict(np.load(os.path.join(tmp_path, f"{name}_r{k}.npz"))) for k in range(world)]
        order, label, I2, J2, off, idx, _ = oracle.pipeline(I, J, n)
        for p in parts:                                   # replicated results
            assert np.array_equal(p["order"], order) and np.array_equal(p["label"], label), name
            assert np.array_equal(p["goff"], off), name
        assert np.array_equal(np.concatenate([p["I2"] for p in parts]), I2), name
        assert np.array_equal(np.concatenate([p["J2"] for p in parts]), J2), name
        # row-partitioned CSR: contiguous row ranges covering [0, n), bit-exact rows
        assert parts[0]["lo"] == 0 and parts[-1]["hi"] == n, name
        for a, b in zip(parts, parts[1:]):
            assert a["hi"] == b["lo"], name
        for p in parts:
            lo, hi = int(p["lo"]), int(p["hi"])
            assert np.array_equal(p["offsets"].astype(np.int64) + off[lo], off[lo:hi + 1]), name
            assert np.array_equal(p["indices"], idx[off[lo]:off[hi]]), name
