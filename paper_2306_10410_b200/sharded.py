"""Multi-GPU BOBA pipeline over contiguous edge shards.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Rank k
holds edges [e0_k, e0_k + m_k) of the global edge list, in order:

  P1  local first occurrence with global positions
      (boba_first_occurrence_shard), then an allreduce-MIN of the n-sized
      array -- the reference's exact chunk-local-min merge
      (_parallel.py:139-162).  uint32 positions are mapped to int32 with the
      order-preserving bias x ^ 0x80000000 so a signed MIN collective is exact
      (UNSET = 0xFFFFFFFF stays the largest, position 2^31-1 stays distinct).
  P2  rank compaction, replicated on every rank (O(n + m/32) work, no
      communication): order and label are identical everywhere.
  P3  relabel of the local shard against the replicated label.
  P4  each rank builds the stable CSR of its shard over all n rows (the
      one-GPU COO->CSR); the sum of the local offsets arrays (allreduce-SUM)
      is the global offsets array.  Rows are cut into P ranges of ~m/P edges.
      The edges rank j owes the owner of rows [b_k, b_k+1) are one contiguous
      run of its local indices, so one all-to-all of column ids (4 bytes per
      edge) and one of per-row counts deliver them; the owner interleaves the
      runs row by row in rank order (boba_merge_rows).  Shards are contiguous
      in edge order, so that is global edge order: the reference's
      within-row order, bit-exact.
  P5  row-partitioned SpMV; x replicated (allgather of y slices to iterate).

The algorithm is written against a small ``ops`` object (DeviceOps below:
the C ABI on CUDA tensors).  The multi-process CPU tests substitute a numpy
implementation of the same interface to check the collective logic with the
gloo backend; the GPU path never imports anything but libboba_b200.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _native as N
from . import device as D

_MIN, _SUM = dist.ReduceOp.MIN, dist.ReduceOp.SUM


class DeviceOps:
    """Local phases on the current CUDA device (uint32 ids in int32 storage)."""

    def first_occurrence_shard(self, I, J, m_global: int, e0: int, n: int):
        first = torch.empty(max(n, 1), dtype=D.ID, device=I.device)[:n]
        ws = D._ws(N.lib.boba_first_occurrence_workspace_size(), I.device)
        N.check(N.lib.boba_first_occurrence_shard(D._p(I), D._p(J), I.numel(), m_global, e0, n, D._p(first), 0,
                                                  D._p(ws), ws.numel(), D._s()))
        return first

    def bias(self, t):
        out = torch.empty_like(t)
        N.check(N.lib.boba_bias_u32(D._p(t), t.numel(), D._p(out), D._s()))
        return out

    def compact(self, first, m_global: int, n: int):
        return D.compact(first, m_global, n)

    def relabel(self, I, J, label, n: int):
        return D.relabel(I, J, label, n)

    def compact_relabel(self, first, I, J, m_global: int, n: int):
        """P2 + P3 with the hub label table, as in the fused one-GPU call."""
        dev = I.device
        m = I.numel()
        e = lambda k: torch.empty(max(k, 1), dtype=D.ID, device=dev)[:k]  # noqa: E731
        order, label, I2, J2 = e(n), e(n), e(m), e(m)
        ws = D._ws(N.lib.boba_compact_relabel_workspace_size(m_global, n), dev)
        N.check(N.lib.boba_compact_relabel(D._p(first), m_global, n, D._p(I), D._p(J), m, D._p(order), D._p(label),
                                           D._p(I2), D._p(J2), D._p(ws), ws.numel(), D._s()))
        return order, label, I2, J2

    def degrees(self, I2, n: int):
        return D.degrees(I2, n)

    def exclusive_scan(self, counts):
        n = counts.numel()
        out = torch.empty(n + 1, dtype=D.ID, device=counts.device)
        ws = D._ws(N.lib.boba_exclusive_scan_workspace_size(n), counts.device)
        N.check(N.lib.boba_exclusive_scan_u32(D._p(counts), n, D._p(out), D._p(ws), ws.numel(), D._s()))
        return out

    def range_partition(self, keys, vals, bounds, parts: int):
        m = keys.numel()
        ko, vo = torch.empty_like(keys), torch.empty_like(vals)
        counts = torch.empty(parts, dtype=D.ID, device=keys.device)
        ws = D._ws(N.lib.boba_range_partition_workspace_size(m, parts), keys.device)
        N.check(N.lib.boba_range_partition(D._p(keys), D._p(vals), m, D._p(bounds), parts, D._p(ko), D._p(vo),
                                           D._p(counts), D._p(ws), ws.numel(), D._s()))
        return ko, vo, counts

    def offset_ids(self, t, delta: int):
        out = torch.empty_like(t)
        N.check(N.lib.boba_offset_ids(D._p(t), t.numel(), delta & 0xFFFFFFFF, D._p(out), D._s()))
        return out

    def coo_to_csr(self, rows, cols, n_rows: int):
        offsets, indices, _ = D.coo_to_csr(rows, cols, n_rows)
        return offsets, indices

    def adjacent_diff(self, t):
        out = torch.empty(max(t.numel() - 1, 1), dtype=D.ID, device=t.device)[: t.numel() - 1]
        N.check(N.lib.boba_adjacent_diff_u32(D._p(t), t.numel() - 1, D._p(out), D._s()))
        return out

    def merge_rows(self, recv, counts, parts: int, rows: int, out_offsets):
        total = recv.numel()
        out = torch.empty(max(total, 1), dtype=D.ID, device=recv.device)[:total]
        ws = D._ws(N.lib.boba_merge_rows_workspace_size(parts, rows, total), recv.device)
        N.check(N.lib.boba_merge_rows(D._p(recv), total, parts, rows, D._p(counts), D._p(out_offsets), D._p(out),
                                      D._p(ws), ws.numel(), D._s()))
        return out


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
    global_offsets: torch.Tensor  # n + 1, replicated


def row_bounds(offsets_g: torch.Tensor, m_global: int, parts: int) -> torch.Tensor:
    """Cut rows so that part k starts at the first row whose global offset is
    >= k * m / parts (edge-balanced ranges; a part may be empty)."""
    n = offsets_g.numel() - 1
    targets = torch.tensor([(k * m_global) // parts for k in range(1, parts)], dtype=torch.int64,
                           device=offsets_g.device)
    offs = offsets_g.to(torch.int64) & 0xFFFFFFFF
    cut = torch.searchsorted(offs, targets, side="left").clamp_(0, n)
    b = torch.empty(parts + 1, dtype=torch.int64, device=offsets_g.device)
    b[0], b[parts] = 0, n
    if parts > 1:
        b[1:parts] = cut
        b = torch.cummax(b, 0).values  # monotone even with empty parts
    return b


def _alltoallv(send: torch.Tensor, send_counts: list[int], recv_counts: list[int], group=None) -> torch.Tensor:
    recv = torch.empty(sum(recv_counts), dtype=send.dtype, device=send.device)
    dist.all_to_all_single(recv, send, output_split_sizes=recv_counts, input_split_sizes=send_counts, group=group)
    return recv


def sharded_reorder_to_csr(I: torch.Tensor, J: torch.Tensor, n: int, m_global: int, e0: int, group=None,
                           ops=None) -> ShardResult:
    """Run the BOBA pipeline on this rank's contiguous shard (see module doc)."""
    ops = ops or DeviceOps()
    P = dist.get_world_size(group)
    r = dist.get_rank(group)
    # P1: local first occurrence, exact global merge
    first = ops.first_occurrence_shard(I, J, m_global, e0, n)
    key = ops.bias(first)
    dist.all_reduce(key, op=_MIN, group=group)
    first = ops.bias(key)
    # P2: replicated compaction; P3: local relabel
    order, label, I2, J2 = ops.compact_relabel(first, I, J, m_global, n)
    # P4: local CSR of the shard over all n rows; global offsets = sum of the local ones
    loc_off, loc_idx = ops.coo_to_csr(I2, J2, n)
    offsets_g = loc_off.clone()
    dist.all_reduce(offsets_g, op=_SUM, group=group)
    bounds64 = row_bounds(offsets_g, m_global, P)
    b = [int(x) for x in bounds64.cpu().tolist()]
    cut = (loc_off.to(torch.int64) & 0xFFFFFFFF)[bounds64].cpu().tolist()     # local run ends per owner
    send_counts = [int(cut[k + 1] - cut[k]) for k in range(P)]
    send_t = torch.tensor(send_counts, dtype=torch.int64, device=I.device)
    recv_t = torch.empty_like(send_t)
    dist.all_to_all_single(recv_t, send_t, group=group)
    recv_counts = [int(c) for c in recv_t.cpu().tolist()]
    lo, hi = b[r], b[r + 1]
    rows_of = [b[k + 1] - b[k] for k in range(P)]
    # per-row counts: owners' row ranges tile [0, n) in rank order, so the send
    # buffer is simply the whole local count array
    row_counts = ops.adjacent_diff(loc_off)
    recv_rc = _alltoallv(row_counts, rows_of, [hi - lo] * P, group)
    recv_idx = _alltoallv(loc_idx, send_counts, recv_counts, group)
    g_lo = int((offsets_g[lo:lo + 1].to(torch.int64) & 0xFFFFFFFF).item())
    offsets = ops.offset_ids(offsets_g[lo:hi + 1].contiguous(), -g_lo)
    # one rank: its run is already the whole CSR
    indices = recv_idx if P == 1 else ops.merge_rows(recv_idx, recv_rc, P, hi - lo, offsets)
    return ShardResult(first, order, label, I2, J2, lo, hi, offsets, indices, offsets_g)


def shard_range(m_global: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced edge shard [e0, e1) of rank `rank`."""
    base, extra = divmod(m_global, world)
    e0 = rank * base + min(rank, extra)
    return e0, e0 + base + (1 if rank < extra else 0)
