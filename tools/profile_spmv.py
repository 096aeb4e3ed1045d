"""SpMV on the c3 grid (4096^2, randomly relabelled) after BOBA, and on the
random labels, for ncu captures: argv[1] = boba|random, argv[2] = reps."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2306_10410_b200 import device as D  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "boba"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
G0, G1 = D.generate_grid(4096, 4096)
n, m = 4096 * 4096, G0.numel()
lab = torch.from_numpy(oracle.random_labels(n, 7).astype(np.int32)).cuda()
I, J = D.gather(lab, G0), D.gather(lab, G1)
del G0, G1, lab
if which == "boba":
    pipe = D.Pipeline(m, n).run(I, J)
    off, idx = pipe.offsets[: n + 1], pipe.indices[:m]
else:
    off, idx = D.coo_to_csr(I, J, n)[:2]
x = torch.ones(n, device="cuda")
y = torch.empty(n, device="cuda")
ws = D.spmv_workspace(n, m, "cuda")
torch.cuda.synchronize()
for _ in range(reps):
    D.spmv(off, idx, x, out=y, ws=ws)
torch.cuda.synchronize()
print("done", which, n, m, float(y.sum()))
