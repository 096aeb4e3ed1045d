"""Times COO->CSR alone (CUDA events, median of R) on the BOBA-relabelled R-MAT
scale S graph.  usage: time_csr.py [S] [R]   (BOBA_LIB_PATH selects the library)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2306_10410_b200 import _native as N  # noqa: E402
from paper_2306_10410_b200 import device as D  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
n = 1 << scale
I, J = D.generate_rmat(scale, 16, 1)
lab = torch.from_numpy(oracle.random_labels(n, 7).astype(np.int32)).cuda()
I, J = D.gather(lab, I), D.gather(lab, J)
m = I.numel()
pipe = D.Pipeline(m, n).run(I, J)
I2, J2 = pipe.I2[:m].clone(), pipe.J2[:m].clone()
offsets = torch.empty(n + 1, dtype=torch.int32, device="cuda")
indices = torch.empty(m, dtype=torch.int32, device="cuda")
ws = torch.empty(N.lib.boba_coo_to_csr_workspace_size(m, n, 0), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for r in range(reps + 3):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    N.check(N.lib.boba_coo_to_csr(D._p(I2), D._p(J2), None, m, n, None, D._p(offsets), D._p(indices), None,
                                  D._p(ws), ws.numel(), D._s()))
    b.record()
    torch.cuda.synchronize()
    if r >= 3:
        ts.append(a.elapsed_time(b))
print(f"coo_to_csr s{scale}: median {np.median(ts):.4f} ms  min {min(ts):.4f} ms  ({os.environ.get('BOBA_LIB_PATH', 'default lib')})")
