"""Multi-process check of the sharded (multi-GPU) pipeline's collective logic
on CPU: world_size 2 and 3 over gloo, with the local phases emulated in numpy
(the GPU kernels cannot run here).  The assembled per-rank outputs must equal
the oracle's single-process pipeline bit for bit: replicated permutation,
relabelled COO shards, the row-partitioned CSR, and the row-partitioned SpMV
(P5) against the oracle's row sums."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle

U32 = np.uint32
UNSET = 0xFFFFFFFF


def u32(t):
    return t.numpy().view(U32)


def t32(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).astype(np.int64) & 0xFFFFFFFF).astype(U32).view(np.int32))


def _buckets(n):
    bits = 0 if n <= 1 else int(n - 1).bit_length()
    shift = max(bits - 15, 0)
    return shift, max((n + (1 << shift) - 1) >> shift, 1)


class NumpyOps:
    """The DeviceOps interface of paper_2306_10410_b200.sharded, in numpy
    (independent restatements of what each C-ABI call computes)."""

    def first_occurrence_shard(self, I, J, m_global, e0, n):
        f = np.full(n, UNSET, dtype=np.uint64)
        I, J = u32(I).astype(np.int64), u32(J).astype(np.int64)
        pos = np.arange(I.size, dtype=np.uint64)
        np.minimum.at(f, I, pos + e0)
        np.minimum.at(f, J, pos + m_global + e0)
        return t32(f)

    def bias(self, t):
        return t32(u32(t) ^ U32(0x80000000))

    def _windows(self, first, m_global, e0, ml):
        f = u32(first).astype(np.int64)
        in_i = (f >= e0) & (f < e0 + ml) & (f != UNSET)
        in_j = (f >= m_global + e0) & (f < m_global + e0 + ml) & (f != UNSET)
        return f, in_i, in_j

    def compact_shard_mark(self, first, n, m_global, e0, ml):
        f, in_i, in_j = self._windows(first, m_global, e0, ml)
        return t32([int(in_i.sum()), int(in_j.sum())]), (m_global, e0, ml)

    def compact_shard_assign(self, first, n, m_global, e0, ml, all_counts, world, rank, ws):
        f, in_i, in_j = self._windows(first, m_global, e0, ml)
        c = u32(all_counts).astype(np.int64).reshape(world, 2)
        label = np.zeros(n, dtype=np.int64)
        # ranks inside each window follow the position order
        for mask, base in ((in_i, c[:rank, 0].sum()), (in_j, c[:, 0].sum() + c[:rank, 1].sum())):
            v = np.flatnonzero(mask)
            label[v[np.argsort(f[v], kind="stable")]] = base + np.arange(v.size)
        iso = np.flatnonzero(f == UNSET)
        if rank == 0:
            label[iso] = c.sum() + np.arange(iso.size)
        return t32(label)

    def order_from_label(self, label, n):
        lab = u32(label).astype(np.int64)
        order = np.empty(n, dtype=np.int64)
        order[lab] = np.arange(n)
        return t32(order), None

    def relabel(self, I, J, label, hubs, n):
        lab = u32(label)
        return t32(lab[u32(I)]), t32(lab[u32(J)])

    def row_cut_hist(self, rows, n):
        shift, B = _buckets(n)
        return t32(np.bincount(u32(rows).astype(np.int64) >> shift, minlength=B))

    def row_cut(self, hist_g, hist_l, n, m_global, parts):
        shift, B = _buckets(n)
        G = np.concatenate([[0], np.cumsum(u32(hist_g).astype(np.int64))])
        L = np.concatenate([[0], np.cumsum(u32(hist_l).astype(np.int64))])
        cuts = [0] + [int(np.searchsorted(G, k * m_global // parts, side="left")) for k in range(1, parts)] + [B]
        bounds = [min(b << shift, n) for b in cuts]
        goff = [int(G[b]) for b in cuts]
        send = [int(L[cuts[k + 1]] - L[cuts[k]]) for k in range(parts)]
        return t32(bounds + goff + send)

    def range_partition(self, keys, vals, bounds, parts):
        k, v = u32(keys).astype(np.int64), u32(vals)
        b = u32(bounds).astype(np.int64)
        owner = np.searchsorted(b[1:parts], k, side="right")
        o = np.argsort(owner, kind="stable")
        return t32(k[o] - b[owner[o]]), t32(v[o])

    def coo_to_csr(self, rows, cols, n_rows):
        r, c = u32(rows).astype(np.int64), u32(cols)
        o = np.argsort(r, kind="stable")
        off = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=n_rows))])
        return t32(off), t32(c[o])

    def coo_to_csr_begin(self, rows, n_rows):
        return None

    def coo_to_csr_finish(self, state, rows, cols, n_rows):
        return self.coo_to_csr(rows, cols, n_rows)

    def spmv(self, offsets, indices, x, out):
        off, idx = u32(offsets).astype(np.int64), u32(indices).astype(np.int64)
        xs = x.numpy().astype(np.float64)
        y = np.array([xs[idx[off[i]:off[i + 1]]].sum() for i in range(off.size - 1)])
        out.copy_(torch.from_numpy(y.astype(np.float32)))
        return out


def _worker(rank, world, port, cases, outdir):
    import torch.distributed as dist

    from paper_2306_10410_b200.sharded import shard_range, sharded_reorder_to_csr, sharded_spmv

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ops = NumpyOps()
    for name, (I, J, n) in cases.items():
        m = I.size
        e0, e1 = shard_range(m, rank, world)
        res = sharded_reorder_to_csr(t32(I[e0:e1]), t32(J[e0:e1]), n, m, e0, ops=ops)
        x0 = torch.from_numpy((np.arange(n) % 7 + 1).astype(np.float32))
        y2 = sharded_spmv(res, x0, 2, ops=ops)
        y2c = sharded_spmv(res, x0, 2, ops=ops, chunks=3)   # exchange overlapped piece by piece
        np.savez(os.path.join(outdir, f"{name}_r{rank}.npz"), first=u32(res.first), order=u32(res.order),
                 label=u32(res.label), I2=u32(res.I2), J2=u32(res.J2), lo=res.row_lo, hi=res.row_hi,
                 offsets=u32(res.offsets), indices=u32(res.indices), goff=res.row_edge_offset,
                 bounds=np.array(res.bounds), y2=y2.numpy(), y2c=y2c.numpy())
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
    big_n = 70000   # > 32768 rows: the coarse row-cut histogram uses buckets of 4 rows
    return {
        "rmat": (lab[I], lab[J], n),
        "fuzz_isolated": (rng.integers(0, 600, 5001), rng.integers(0, 700, 5001), 900),  # many isolated
        "coarse_buckets": (rng.integers(0, big_n, 20011), rng.integers(0, big_n, 20011), big_n),
        "tiny": (np.array([5, 5, 3]), np.array([3, 1, 5]), 6),                            # test_ordering.py:37-40
        "fewer_edges_than_ranks": (np.array([1]), np.array([0]), 3),
        "no_edges": (np.array([], dtype=np.int64), np.array([], dtype=np.int64), 4),
    }


def check_parts(parts, I, J, n, name):
    order, label, I2, J2, off, idx, _ = oracle.pipeline(I, J, n)
    for p in parts:                                   # replicated results
        assert np.array_equal(p["order"], order) and np.array_equal(p["label"], label), name
        assert np.array_equal(p["bounds"], parts[0]["bounds"]), name
    assert np.array_equal(np.concatenate([p["I2"] for p in parts]), I2), name
    assert np.array_equal(np.concatenate([p["J2"] for p in parts]), J2), name
    # row-partitioned CSR: contiguous row ranges covering [0, n), bit-exact rows
    assert parts[0]["lo"] == 0 and parts[-1]["hi"] == n, name
    for a, b in zip(parts, parts[1:]):
        assert a["hi"] == b["lo"], name
    for p in parts:
        lo, hi = int(p["lo"]), int(p["hi"])
        assert int(p["goff"]) == off[lo], name
        assert np.array_equal(p["offsets"].astype(np.int64) + off[lo], off[lo:hi + 1]), name
        assert np.array_equal(p["indices"], idx[off[lo]:off[hi]]), name
    return off, idx


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_pipeline_matches_oracle(world, tmp_path):
    cases = make_cases()
    mp.spawn(_worker, args=(world, _free_port(), cases, str(tmp_path)), nprocs=world, join=True)
    for name, (I, J, n) in cases.items():
        parts = [dict(np.load(os.path.join(tmp_path, f"{name}_r{k}.npz"))) for k in range(world)]
        off, idx = check_parts(parts, I, J, n, name)
        # P5: two row-partitioned SpMV iterations, replicated result
        x = (np.arange(n) % 7 + 1).astype(np.float64)
        y = oracle.spmv_pull(off, idx, oracle.spmv_pull(off, idx, x))
        for p in parts:
            np.testing.assert_allclose(p["y2"], y, rtol=1e-5, atol=0)
            assert np.array_equal(p["y2c"], p["y2"])   # same rows, same sums: chunking changes only the schedule
        if name == "rmat":   # the edge-balanced cut actually balances
            sizes = [int(off[p["hi"]] - off[p["lo"]]) for p in parts]
            assert max(sizes) <= 1.5 * I.size / world + 64, sizes
