"""Times boba_merge_rows on a c2-sized receive buffer: the local CSR of R-MAT
s22 split into P contiguous 'sender' shards (P = 1, 2, 4, 8), all rows."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2306_10410_b200 import device as D
from paper_2306_10410_b200.sharded import DeviceOps, shard_range
n = 1 << 22
I, J = D.generate_rmat(22, 16, 1)
lab = torch.from_numpy(oracle.random_labels(n, 7).astype(np.int32)).cuda()
I, J = D.gather(lab, I), D.gather(lab, J)
m = I.numel()
ops = DeviceOps()
full_off, full_idx = ops.coo_to_csr(I, J, n)
for P in (1, 2, 4, 8):
    runs, rcs = [], []
    for k in range(P):
        e0, e1 = shard_range(m, k, P)
        o, i = ops.coo_to_csr(I[e0:e1], J[e0:e1], n)
        runs.append(i); rcs.append(ops.adjacent_diff(o))
    recv, counts = torch.cat(runs), torch.cat(rcs)
    out = ops.merge_rows(recv, counts, P, n, full_off)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); out = ops.merge_rows(recv, counts, P, n, full_off); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(P, "merge %.3f ms" % np.median(ts), "exact:", bool(torch.equal(out, full_idx)))
