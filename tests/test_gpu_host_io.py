"""The drop-in's host <-> device id transfers (boba_host_to_device_ids /
boba_device_to_host_ids: host-thread narrowing / widening through pinned
staging, chunked) and the C-ABI guards added for the advisor's findings
(SpMV partition reuse fingerprint)."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2306_10410_b200 import _host
    from paper_2306_10410_b200 import _native as N
    from paper_2306_10410_b200 import device as D

    return torch, _host, N, D


@pytest.mark.parametrize("count", [0, 1, 5, (16 << 20) - 1, (16 << 20) + 7, (40 << 20) + 3])
def test_round_trip_across_chunks(mods, count):
    torch, H, N, D = mods
    rng = np.random.default_rng(count)
    bound = (1 << 32) if count % 2 else 123457
    a = rng.integers(0, bound, count, dtype=np.int64)
    t = H.to_device_ids(a, bound)
    assert t.numel() == count
    assert np.array_equal(t.cpu().numpy().view(np.uint32), a.astype(np.uint32))
    assert np.array_equal(H.to_host_ids(t), a)


@pytest.mark.parametrize("where", [0, 17, (16 << 20) + 2, (20 << 20) - 2])
def test_range_error_reports_first_offender(mods, where):
    torch, H, N, D = mods
    from paper_2306_10410_b200 import MalformedGraphError

    a = np.zeros(20 << 20, dtype=np.int64)
    a[where] = -3
    a[-1] = 1 << 40          # a later offender must not win
    with pytest.raises(MalformedGraphError, match=rf"I\[{where}\] = -3"):
        H.to_device_ids(a, 10, "I")


def test_dropin_pipeline_reuses_device_copies(mods, medium):
    """apply_permutation -> coo_to_csr through the drop-in returns the same
    result whether or not the device copies are reused."""
    torch, H, N, D = mods
    import paper_2306_10410_b200 as bb

    c = medium.case(0)
    g = bb.CooGraph(c["n"], c["I"], c["J"])
    p = bb.boba_parallel(g)
    assert H._recall(p.label) is not None
    g2 = bb.apply_permutation(g, p)
    assert H._recall(g2.I) is not None and H._recall(g2.J) is not None
    csr = bb.coo_to_csr(g2)
    assert np.array_equal(csr.offsets, c["offsets"]) and np.array_equal(csr.indices, c["indices"])
    # a caller-built container with the same values never hits the cache
    g3 = bb.CooGraph(c["n"], np.array(g2.I), np.array(g2.J))
    assert H._recall(g3.I) is None
    csr3 = bb.coo_to_csr(g3)
    assert np.array_equal(csr3.indices, c["indices"])


def test_spmv_partition_reuse_needs_matching_partition(mods):
    torch, H, N, D = mods
    n, m = 1000, 5000
    rng = np.random.default_rng(0)
    rows = np.sort(rng.integers(0, n, m))
    off = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=n))]).astype(np.int32)
    idx = rng.integers(0, n, m).astype(np.int32)
    o, i = torch.from_numpy(off).cuda(), torch.from_numpy(idx).cuda()
    x = torch.ones(n, device="cuda")
    ws = D.spmv_workspace(n, m, o.device)
    with pytest.raises(Exception, match="reuse_partition"):       # never partitioned
        D.spmv(o, i, x, ws=ws, reuse_partition=True)
    y = D.spmv(o, i, x, ws=ws)
    y2 = D.spmv(o, i, x, ws=ws, reuse_partition=True)
    assert torch.equal(y, y2)
    o2 = o.clone()
    with pytest.raises(Exception, match="reuse_partition"):       # another CSR
        D.spmv(o2, i, x, ws=ws, reuse_partition=True)



GARBAGE_COORDS = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2306_10410_b200 import device as D
n, m = 1000, 5000
rng = np.random.default_rng(0)
rows = np.sort(rng.integers(0, n, m))
o = torch.from_numpy(np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=n))]).astype(np.int32)).cuda()
i = torch.from_numpy(rng.integers(0, n, m).astype(np.int32)).cuda()
x = torch.ones(n, device="cuda")
ws = D.spmv_workspace(n, m, o.device)
D.spmv(o, i, x, ws=ws)
for junk in (0xFF, 0x7F, 0x01):
    ws.fill_(junk)        # coords of nothing: the kernel guard must skip, not write out of bounds
    D.spmv(o, i, x, ws=ws, reuse_partition=True)
    torch.cuda.synchronize()
print("ok")
"""


def test_spmv_garbage_partition_does_not_fault(mods):
    """A corrupted partition in a reused workspace (same CSR pointers, so the
    host fingerprint passes) must not write out of bounds; run in a child
    process so a fault could not take this test session's context down."""
    import subprocess
    import sys

    from conftest import ROOT

    r = subprocess.run([sys.executable, "-c", GARBAGE_COORDS, ROOT], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
