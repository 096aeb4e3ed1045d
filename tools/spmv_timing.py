"""SpMV per-call time (CUDA events, L2 flushed, median of 20) on the c3 grid
in BOBA order and in random order, fp32 and fp64."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2306_10410_b200 import device as D  # noqa: E402

G0, G1 = D.generate_grid(4096, 4096)
n, m = 4096 * 4096, G0.numel()
lab = torch.from_numpy(oracle.random_labels(n, 7).astype(np.int32)).cuda()
I, J = D.gather(lab, G0), D.gather(lab, G1)
pipe = D.Pipeline(m, n).run(I, J)
csr = {"boba": (pipe.offsets[: n + 1], pipe.indices[:m]), "random": D.coo_to_csr(I, J, n)[:2]}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ws = D.spmv_workspace(n, m, "cuda")
out = {}
for dt in (torch.float32, torch.float64):
    x = torch.ones(n, dtype=dt, device="cuda")
    y = torch.empty(n, dtype=dt, device="cuda")
    for k, (off, idx) in csr.items():
        D.spmv(off, idx, x, out=y, ws=ws)
        ts = []
        for _ in range(20):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            D.spmv(off, idx, x, out=y, ws=ws)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        out[f"{k}_{str(dt).split('.')[-1]}_ms"] = round(statistics.median(ts), 4)
print(json.dumps(out))
