"""Multi-GPU BOBA pipeline over contiguous edge shards.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Rank r
of P holds edges [e0, e0 + ml) of the m-edge list, in order, i.e. positions
[e0, e0 + ml) of I and [m + e0, m + e0 + ml) of J:

  P1  local first occurrence with global positions
      (boba_first_occurrence_shard), then an allreduce-MIN of the n-sized
      array -- the reference's exact chunk-local-min merge
      (_parallel.py:139-162).  uint32 positions are mapped to int32 with the
      order-preserving bias x ^ 0x80000000 so a signed MIN collective is exact.
  P2  compaction split by position window (_parallel.py:178-201): each rank
      ranks only the vertices first seen in its two windows
      (boba_compact_shard_mark / _assign); the global rank adds a prefix over
      the 2P window counts (allgather of 2 words per rank).  The partial
      label arrays (one owner per vertex, 0 elsewhere) are merged by an
      allreduce-SUM; order = inverse of label, built locally.
  P3  relabel of the local shard against the replicated label, with the hub
      label table (graph.py:280-289).
  P4  row-partitioned CSR (graph.py:253-277): a coarse row histogram
      (<= 32768 buckets, allreduce-SUM of 128 KB) fixes P edge-balanced row
      ranges on bucket boundaries and every rank's send counts; one stable
      range partition of (row, col) per rank, an all-to-all of rows and of
      cols, and the owner's stable COO->CSR of what it received.  Senders are
      ranks in order and shards are contiguous in edge order, so the received
      sequence is global edge order restricted to the owner's rows: the
      reference's within-row order (_parallel.py:55-88), bit-exact.  The rows
      are exchanged before the columns, and the owner computes its first radix
      histogram of the rows while the columns are in flight.
  P5  row-partitioned SpMV (kernels.py:30-52): the owner multiplies its rows
      by the replicated x; between iterations every owner broadcasts its y
      slice (an allgather-v) into the next x.

Host synchronisations per step: one (the 3P + 2 + P words of row bounds and
send / receive counts the all-to-all needs on the host).

The algorithm is written against a small ``ops`` object (DeviceOps below:
the C ABI on CUDA tensors).  The multi-process CPU tests substitute a numpy
implementation of the same interface to check the collective logic with the
gloo backend; the GPU path never imports anything but libboba_b200.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _native as N
from . import device as D

_MIN, _SUM = dist.ReduceOp.MIN, dist.ReduceOp.SUM


def _e(k, dev):
    return torch.empty(max(k, 1), dtype=D.ID, device=dev)[:k]


class DeviceOps:
    """Local phases on the current CUDA device (uint32 ids in int32 storage)."""

    def first_occurrence_shard(self, I, J, m_global: int, e0: int, n: int):
        first = _e(n, I.device)
        ws = D._ws(N.lib.boba_first_occurrence_shard_workspace_size(n), I.device)
        N.check(N.lib.boba_first_occurrence_shard(D._p(I), D._p(J), I.numel(), m_global, e0, n, D._p(first), 0,
                                                  D._p(ws), ws.numel(), D._s()))
        return first

    def bias(self, t):
        out = torch.empty_like(t)
        N.check(N.lib.boba_bias_u32(D._p(t), t.numel(), D._p(out), D._s()))
        return out

    def compact_shard_mark(self, first, n: int, m_global: int, e0: int, ml: int):
        """-> (counts[2], workspace to pass to compact_shard_assign)."""
        ws = D._ws(N.lib.boba_compact_shard_workspace_size(ml, n), first.device)
        counts = _e(2, first.device)
        N.check(N.lib.boba_compact_shard_mark(D._p(first), n, m_global, e0, ml, D._p(counts), D._p(ws), ws.numel(),
                                              D._s()))
        return counts, ws

    def compact_shard_assign(self, first, n: int, m_global: int, e0: int, ml: int, all_counts, world: int,
                             rank: int, ws):
        label = _e(n, first.device)
        N.check(N.lib.boba_compact_shard_assign(D._p(first), n, m_global, e0, ml, D._p(all_counts), world, rank,
                                                D._p(label), D._p(ws), ws.numel(), D._s()))
        return label

    def order_from_label(self, label, n: int):
        """-> (order, hub label table for relabel)."""
        order = _e(n, label.device)
        hubs = D._ws(N.lib.boba_hub_table_bytes(), label.device)
        N.check(N.lib.boba_order_from_label(D._p(label), n, D._p(order), D._p(hubs), D._s()))
        return order, hubs

    def relabel(self, I, J, label, hubs, n: int):
        m = I.numel()
        I2, J2 = _e(m, I.device), _e(m, I.device)
        N.check(N.lib.boba_relabel_hubs(D._p(I), D._p(J), m, n, D._p(label), D._p(hubs), D._p(I2), D._p(J2),
                                        D._s()))
        return I2, J2

    def row_cut_hist(self, rows, n: int):
        hist = _e(int(N.lib.boba_row_cut_buckets(n)), rows.device)
        N.check(N.lib.boba_row_cut_hist(D._p(rows), rows.numel(), n, D._p(hist), D._s()))
        return hist

    def row_cut(self, hist_g, hist_l, n: int, m_global: int, parts: int):
        out = _e(3 * parts + 2, hist_g.device)
        N.check(N.lib.boba_row_cut(D._p(hist_g), D._p(hist_l), n, m_global, parts, D._p(out), D._s()))
        return out

    def range_partition(self, keys, vals, bounds, parts: int):
        """Stable partition by row range, keys written relative to their part."""
        m = keys.numel()
        ko, vo = torch.empty_like(keys), torch.empty_like(vals)
        ws = D._ws(N.lib.boba_range_partition_workspace_size(m, parts), keys.device)
        N.check(N.lib.boba_range_partition_ex(D._p(keys), D._p(vals), m, D._p(bounds), parts, 1, D._p(ko), D._p(vo),
                                              None, D._p(ws), ws.numel(), D._s()))
        return ko, vo

    def coo_to_csr(self, rows, cols, n_rows: int):
        offsets, indices, _ = D.coo_to_csr(rows, cols, n_rows)
        return offsets, indices

    def coo_to_csr_begin(self, rows, n_rows: int):
        """The first radix pass's tile histogram of the row keys alone
        (boba_coo_to_csr_first_hist); -> the workspace holding it."""
        m = rows.numel()
        ws = D._ws(N.lib.boba_coo_to_csr_workspace_size(m, n_rows, 0), rows.device)
        N.check(N.lib.boba_coo_to_csr_first_hist(D._p(rows), m, n_rows, D._p(ws), ws.numel(), D._s()))
        return ws

    def coo_to_csr_finish(self, ws, rows, cols, n_rows: int):
        """The rest of the conversion, reusing that histogram."""
        m = rows.numel()
        offsets, indices = _e(n_rows + 1, rows.device), _e(m, rows.device)
        N.check(N.lib.boba_coo_to_csr_ex(D._p(rows), D._p(cols), None, m, n_rows, None, D._p(offsets),
                                         D._p(indices), None, D._p(ws), ws.numel(), 1, D._s()))
        return offsets, indices

    def spmv(self, offsets, indices, x, out):
        return D.spmv(offsets, indices, x, out=out)


@dataclass
class ShardResult:
    first: torch.Tensor       # global first occurrences (replicated)
    order: torch.Tensor       # replicated permutation
    label: torch.Tensor
    I2: torch.Tensor          # this rank's shard of the relabelled COO
    J2: torch.Tensor
    row_lo: int               # this rank owns CSR rows [row_lo, row_hi)
    row_hi: int
    offsets: torch.Tensor     # local CSR offsets (row_hi - row_lo + 1), relative to the local indices
    indices: torch.Tensor     # column ids (global labels)
    row_edge_offset: int      # global offsets[row_lo]: the global CSR offsets are offsets + row_edge_offset
    bounds: list              # all owners' row bounds b_0 = 0 <= ... <= b_P = n
    sent: list                # edges this rank sent to each owner
    received: list            # edges this rank received from each sender


def _alltoallv(send: torch.Tensor, send_counts: list[int], recv_counts: list[int], group=None, async_op=False):
    recv = torch.empty(sum(recv_counts), dtype=send.dtype, device=send.device)
    work = dist.all_to_all_single(recv, send, output_split_sizes=recv_counts, input_split_sizes=send_counts,
                                  group=group, async_op=async_op)
    return (recv, work) if async_op else recv


def sharded_reorder_to_csr(I: torch.Tensor, J: torch.Tensor, n: int, m_global: int, e0: int, group=None,
                           ops=None, mark=None) -> ShardResult:
    """Run the BOBA pipeline on this rank's contiguous shard (see module doc).
    `mark(name)`, if given, is called at every phase boundary (timing) and
    with "+comm" / "-comm" around every collective."""
    ops = ops or DeviceOps()
    mark = mark or (lambda name: None)
    P = dist.get_world_size(group)
    r = dist.get_rank(group)
    ml = I.numel()
    mark("start")
    # P1: local first occurrence, exact global merge
    first = ops.first_occurrence_shard(I, J, m_global, e0, n)
    key = ops.bias(first)
    mark("+comm")
    dist.all_reduce(key, op=_MIN, group=group)
    mark("-comm")
    first = ops.bias(key)
    mark("first_occurrence")
    # P2: compaction of this rank's position windows, global ranks by a prefix over the window counts
    counts, ws = ops.compact_shard_mark(first, n, m_global, e0, ml)
    all_counts = torch.empty(2 * P, dtype=counts.dtype, device=counts.device)
    mark("+comm")
    dist.all_gather_into_tensor(all_counts, counts, group=group)
    mark("-comm")
    label = ops.compact_shard_assign(first, n, m_global, e0, ml, all_counts, P, r, ws)
    del ws
    mark("+comm")
    dist.all_reduce(label, op=_SUM, group=group)
    mark("-comm")
    order, hubs = ops.order_from_label(label, n)
    mark("compact")
    # P3: local relabel
    I2, J2 = ops.relabel(I, J, label, hubs, n)
    mark("relabel")
    # P4: row cut from a coarse histogram, stable partition, all-to-all, owner's CSR
    hist_l = ops.row_cut_hist(I2, n)
    hist_g = hist_l.clone()
    mark("+comm")
    dist.all_reduce(hist_g, op=_SUM, group=group)
    mark("-comm")
    cut = ops.row_cut(hist_g, hist_l, n, m_global, P)
    send_t = cut[2 * P + 2:3 * P + 2].clone()
    recv_t = torch.empty_like(send_t)
    mark("+comm")
    dist.all_to_all_single(recv_t, send_t, group=group)
    mark("-comm")
    meta = torch.cat([cut, recv_t]).cpu().numpy().view("uint32").tolist()   # the step's one host sync
    bounds = meta[:P + 1]
    goff = meta[P + 1:2 * P + 2]
    sent = meta[2 * P + 2:3 * P + 2]
    received = meta[3 * P + 2:]
    lo, hi = bounds[r], bounds[r + 1]
    if P == 1:   # one owner: the shard is already the owner's edges in edge order
        offsets, indices = ops.coo_to_csr(I2, J2, hi - lo)
    else:
        keys, vals = ops.range_partition(I2, J2, cut[:P + 1], P)
        # rows first, then columns (both queued on the collective's stream); the
        # owner histograms the rows for its first radix pass while the columns
        # are still in flight
        mark("+comm")
        rk, wk = _alltoallv(keys, sent, received, group, async_op=True)
        rv, wv = _alltoallv(vals, sent, received, group, async_op=True)
        wk.wait()
        mark("-comm")
        state = ops.coo_to_csr_begin(rk, hi - lo)
        mark("+comm")
        wv.wait()
        mark("-comm")
        del keys, vals
        offsets, indices = ops.coo_to_csr_finish(state, rk, rv, hi - lo)
    mark("coo_to_csr")
    return ShardResult(first, order, label, I2, J2, lo, hi, offsets, indices, goff[r], bounds, sent, received)


def _chunk_rows(b0: int, b1: int, c: int, chunks: int) -> tuple[int, int]:
    """Row range [r0, r1) of chunk c of an owner's rows [b0, b1): equal row
    counts, so every rank knows every owner's chunks from the bounds alone."""
    k = b1 - b0
    return b0 + c * k // chunks, b0 + (c + 1) * k // chunks


def _spmv_pieces(res: ShardResult, chunks: int) -> list:
    """The owner's CSR cut into `chunks` row pieces (offsets re-based to their
    first nonzero), built once per (result, chunks)."""
    cache = res.__dict__.setdefault("_spmv_pieces", {})
    if chunks not in cache:
        pieces = []
        off = res.offsets
        for c in range(chunks):
            r0, r1 = _chunk_rows(0, res.row_hi - res.row_lo, c, chunks)
            if r1 == r0:
                pieces.append(None)
                continue
            o = off[r0:r1 + 1]
            base = o[:1]
            lo_hi = torch.stack([o[0], o[-1]]).to(torch.int64).cpu().tolist()   # setup-time host read
            pieces.append((r0, r1, o - base, res.indices[lo_hi[0] & 0xFFFFFFFF:lo_hi[1] & 0xFFFFFFFF]))
        cache[chunks] = pieces
    return cache[chunks]


def sharded_spmv(res: ShardResult, x: torch.Tensor, iters: int = 1, group=None, ops=None,
                 chunks: int = 1) -> torch.Tensor:
    """P5: `iters` row-partitioned SpMV iterations x <- A x over the CSR that
    sharded_reorder_to_csr left on the ranks (reference kernels.py:30-52 per
    row range).  x (n) is replicated; after each iteration every owner
    broadcasts its slice, so the returned vector is replicated too.

    chunks > 1 overlaps the exchange with the multiply: each
    owner's rows are cut into `chunks` equal row pieces; piece c of every
    owner is broadcast (asynchronously, on the collective's own stream) as
    soon as its owner has computed it, while the owner computes piece c + 1.
    Every rank issues the broadcasts in the same (piece, owner) order."""
    ops = ops or DeviceOps()
    P = dist.get_world_size(group)
    b = res.bounds
    src = [dist.get_global_rank(group, k) if group else k for k in range(P)]
    cur = x
    if chunks <= 1:
        for _ in range(iters):
            nxt = torch.empty_like(x)
            ops.spmv(res.offsets, res.indices, cur, nxt[res.row_lo:res.row_hi])
            works = [dist.broadcast(nxt[b[k]:b[k + 1]], src=src[k], group=group, async_op=True)
                     for k in range(P) if b[k + 1] > b[k]]
            for w in works:
                w.wait()
            cur = nxt
        return cur
    pieces = _spmv_pieces(res, chunks)
    for _ in range(iters):
        nxt = torch.empty_like(x)
        works = []
        for c in range(chunks):
            pc = pieces[c]
            if pc is not None:
                r0, r1, off_c, idx_c = pc
                ops.spmv(off_c, idx_c, cur, nxt[res.row_lo + r0:res.row_lo + r1])
            for k in range(P):
                g0, g1 = _chunk_rows(b[k], b[k + 1], c, chunks)
                if g1 > g0:
                    works.append(dist.broadcast(nxt[g0:g1], src=src[k], group=group, async_op=True))
        for w in works:
            w.wait()
        cur = nxt
    return cur


class _ShardOut(ctypes.Structure):
    _fields_ = [("row_lo", ctypes.c_uint32), ("row_hi", ctypes.c_uint32), ("nnz", ctypes.c_uint64),
                ("row_edge_offset", ctypes.c_uint64)]


def nccl_comm_ptr(group=None) -> int:
    """The raw ncclComm_t of a torch.distributed NCCL process group."""
    pg = group or dist.distributed_c10d._get_default_group()
    return int(pg._get_backend(torch.device("cuda"))._comm_ptr())


def native_sharded_reorder_to_csr(I: torch.Tensor, J: torch.Tensor, n: int, m_global: int, e0: int, group=None,
                                  recv_capacity: int | None = None) -> ShardResult:
    """The same pipeline as sharded_reorder_to_csr in one C-ABI call
    (boba_sharded_reorder_to_csr_nccl) on the group's NCCL communicator: the
    entry a C/C++ caller with its own ncclComm_t uses."""
    P = dist.get_world_size(group)
    r = dist.get_rank(group)
    dev, ml = I.device, I.numel()
    cap = recv_capacity or (2 * m_global) // P + (1 << 20)
    comm = ctypes.c_void_p(nccl_comm_ptr(group))
    first, order, label = _e(n, dev), _e(n, dev), _e(n, dev)
    I2, J2 = _e(ml, dev), _e(ml, dev)
    offsets = _e(n + 1, dev)
    while True:
        indices = _e(cap, dev)
        ws = D._ws(N.lib.boba_sharded_workspace_size(ml, n, P, cap), dev)
        out = _ShardOut()
        bounds = (ctypes.c_uint32 * (P + 1))()
        rc = N.lib.boba_sharded_reorder_to_csr_nccl(
            D._p(I), D._p(J), ml, m_global, e0, n, comm, D._p(first), D._p(order), D._p(label), D._p(I2), D._p(J2),
            D._p(offsets), D._p(indices), cap, ctypes.byref(out), bounds, D._p(ws), ws.numel(), D._s())
        if rc == N.BOBA_EINVAL and out.nnz > cap:
            cap = int(out.nnz)
            continue
        N.check(rc)
        break
    lo, hi = int(out.row_lo), int(out.row_hi)
    return ShardResult(first, order, label, I2, J2, lo, hi, offsets[:hi - lo + 1], indices[:int(out.nnz)],
                       int(out.row_edge_offset), list(bounds), [], [])


def shard_range(m_global: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced edge shard [e0, e1) of rank `rank`."""
    base, extra = divmod(m_global, world)
    e0 = rank * base + min(rank, extra)
    return e0, e0 + base + (1 if rank < extra else 0)


def done_phases(evs, upto) -> set:
    """Names of the phase marks recorded before event `upto` in `evs`."""
    out = set()
    for name, e in evs:
        if e is upto:
            break
        if not name.startswith(("+", "-")):
            out.add(name)
    return out


class ShardedPipeline:
    """The sharded pipeline of one rank on fixed shard geometry, with the
    timing hooks bench.py uses."""

    PHASES = ("first_occurrence", "compact", "relabel", "coo_to_csr")

    def __init__(self, n: int, m_global: int, e0: int, m_local: int, device, group=None):
        self.n, self.m, self.e0, self.ml, self.device, self.group = n, m_global, e0, m_local, device, group
        self.ops = DeviceOps()
        self.last = None

    def run(self, I, J, mark=None) -> ShardResult:
        self.last = sharded_reorder_to_csr(I, J, self.n, self.m, self.e0, self.group, self.ops, mark)
        return self.last

    def phase_times(self, I, J) -> dict:
        """One step with CUDA events at the phase boundaries and around every
        collective: ms per phase (incl. its collectives), of which in
        collectives ("comm_ms"), max over ranks; plus the step's compute-only,
        comm-only and actual (overlapped) totals."""
        evs = []

        def mark(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            evs.append((name, e))

        self.run(I, J, mark)
        torch.cuda.synchronize()
        tot = {k: 0.0 for k in self.PHASES}
        comm = {k: 0.0 for k in self.PHASES}
        prev, c0 = evs[0][1], None
        for name, e in evs[1:]:
            if name == "+comm":
                c0 = e
            elif name == "-comm":
                cur_comm = c0.elapsed_time(e)
                phase = next(k for k in self.PHASES if k not in done_phases(evs, e))
                comm[phase] += cur_comm
            else:
                tot[name] = prev.elapsed_time(e)
                prev = e
        vals = [tot[k] for k in self.PHASES] + [comm[k] for k in self.PHASES]
        t = torch.tensor(vals, dtype=torch.float64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        v = t.tolist()
        K = len(self.PHASES)
        out = {k: {"ms": round(v[i], 4), "comm_ms": round(v[K + i], 4), "compute_ms": round(v[i] - v[K + i], 4)}
               for i, k in enumerate(self.PHASES)}
        out["step"] = {"compute_only_ms": round(sum(v[i] - v[K + i] for i in range(K)), 4),
                       "comm_only_ms": round(sum(v[K:]), 4), "actual_ms": round(sum(v[:K]), 4),
                       "note": "collectives run on NCCL's stream; compute overlaps them in P4 (the owner's row "
                               "histogram while the columns arrive) and in P5 (sharded_spmv chunks)"}
        return out

    def spmv_timing(self, res: ShardResult, iters: int, chunks: int = 1) -> dict:
        """P5: `iters` row-partitioned SpMV iterations (x = ones), ms per
        iteration incl. the slice broadcasts, max over ranks.  chunks > 1:
        the broadcasts overlap the multiply piece by piece (sharded_spmv)."""
        x = torch.ones(self.n, dtype=torch.float32, device=self.device)
        sharded_spmv(res, x, 1, self.group, self.ops, chunks)
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sharded_spmv(res, x, iters, self.group, self.ops, chunks)
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / iters], dtype=torch.float64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        nnz = torch.tensor([res.indices.numel()], dtype=torch.float64, device=self.device)
        dist.all_reduce(nnz, op=dist.ReduceOp.MAX, group=self.group)
        return {"iters": iters, "x": "ones", "chunks": chunks, "ms_per_iter": round(float(t.item()), 4),
                "gedges_per_s": round(self.m / (float(t.item()) / 1e3) / 1e9, 3),
                "max_rows_nnz_per_rank": int(nnz.item()), "balance": round(self.m / self.world / nnz.item(), 4),
                "path": "owner rows x replicated x (boba_spmv), slices broadcast (allgather-v) per iteration"
                        + (f", {chunks} pieces per owner, each broadcast while the next is computed"
                           if chunks > 1 else "")}

    @property
    def world(self) -> int:
        return dist.get_world_size(self.group)

    def comm_bytes(self) -> dict:
        """Bytes each rank moves over NVLink per step, from the
        last step's exchange counts, and the time they take at 900 GB/s per
        direction."""
        P, n = self.world, self.n
        res = self.last
        ring = 2 * (P - 1) / P if P > 1 else 0.0
        sent = 8 * (sum(res.sent) - res.sent[dist.get_rank(self.group)]) if res else 0
        b = {"allreduce_min_first": int(ring * 4 * n), "allgather_window_counts": 8 * P,
             "allreduce_sum_label": int(ring * 4 * n),
             "allreduce_row_hist": int(ring * 4 * int(N.lib.boba_row_cut_buckets(n))),
             "alltoall_rows_cols_sent": int(sent)}
        total = sum(b.values())
        b["total"] = total
        b["nvlink_ms_at_900gbs"] = round(total / 900e9 * 1e3, 4)
        return b

    def kernel_launches_per_step(self) -> int:
        """Kernels one step launches (from the launch plan of each C-ABI call:
        first occurrence 1-4 + 2 bias, window mark 3 + assign 1, order 2,
        relabel 1-3, row-cut 2, partition 3 (+1), COO->CSR 3 per radix pass
        + 2)."""
        rows = max((self.last.row_hi - self.last.row_lo) if self.last else self.n // max(self.world, 1), 2)
        passes = -(-((rows - 1).bit_length()) // 8)
        return 4 + 2 + 4 + 2 + 2 + 2 + 3 + 3 * passes + 2
