"""BASELINE config 5: the random / BOBA / degree-sort sweep -- reorder time,
COO->CSR time, SpMV time and GFLOP/s per ordering, on the GPU path.

usage: order_sweep.py [rmat SCALE | grid SIDE] [--ncu]

Times are CUDA-event medians (L2 flushed before each sample).  "random" is the
randomly labelled input itself (reorder = 0, as the reference's `identity`);
"boba" runs first occurrence + compaction + relabel; "degree" runs the
degree ordering (total degree descending, ties by id) + relabel.  With --ncu
the script launches exactly one SpMV per ordering, in the order random, boba,
degree, after a marker, for `ncu -k regex:k_spmv_merge` captures of the L1/L2
hit rates (profiles/r01_order_sweep.md).
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2306_10410_b200 import device as D  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "rmat"
size = int(sys.argv[2]) if len(sys.argv) > 2 else 24
ncu = "--ncu" in sys.argv
if kind == "rmat":
    n = 1 << size
    I0, J0 = D.generate_rmat(size, 16, 1)
else:
    n = size * size
    I0, J0 = D.generate_grid(size, size)
lab = torch.from_numpy(oracle.random_labels(n, 7).astype(np.int32)).cuda()
I, J = D.gather(lab, I0), D.gather(lab, J0)
del I0, J0, lab
m = I.numel()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), out


def reorder_boba():
    _, _, label = D.boba_order(I, J, n)
    return D.relabel(I, J, label, n)


def reorder_degree():
    _, label = D.degree_order(I, J, n)
    return D.relabel(I, J, label, n)


rows = {}
csrs = {}
for name, fn in [("random", None), ("boba", reorder_boba), ("degree", reorder_degree)]:
    if fn is None:
        t_re, (I2, J2) = 0.0, (I, J)
    else:
        t_re, (I2, J2) = timed(fn)
    t_csr, (off, idx, _) = timed(lambda: D.coo_to_csr(I2, J2, n))
    x = torch.ones(n, dtype=torch.float32, device="cuda")
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    ws = D.spmv_workspace(n, m, "cuda")
    t_sp, _ = timed(lambda: D.spmv(off, idx, x, out=y, ws=ws), reps=10)
    rows[name] = {"reorder_ms": round(t_re, 4), "coo_to_csr_ms": round(t_csr, 4), "spmv_ms": round(t_sp, 4),
                  "spmv_gflops": round(2 * m / t_sp / 1e6, 1)}
    csrs[name] = (off, idx, x, y, ws)
    del I2, J2
print(json.dumps({"graph": f"{kind} {size}", "n": n, "m": m, "orders": rows}, indent=1))
if ncu:
    torch.cuda.synchronize()
    for name in ["random", "boba", "degree"]:
        off, idx, x, y, ws = csrs[name]
        flush.fill_(1)
        D.spmv(off, idx, x, out=y, ws=ws)
        torch.cuda.synchronize()
