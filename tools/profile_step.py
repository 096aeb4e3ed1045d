"""One pipeline step + one SpMV on R-MAT scale S (default 22) or the c3 grid (arg "grid"), for ncu captures."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2306_10410_b200 import device as D
arg = sys.argv[1] if len(sys.argv) > 1 else "22"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
if arg == "grid":   # c3: 4096^2 grid, random labels
    I, J = D.generate_grid(4096, 4096)
    n = 4096 * 4096
else:
    scale = int(arg)
    n, ef = 1 << scale, 16
    I, J = D.generate_rmat(scale, ef, 1)
lab = torch.from_numpy(oracle.random_labels(n, 7).astype(np.int32)).cuda()
I, J = D.gather(lab, I), D.gather(lab, J)
m = I.numel()
pipe = D.Pipeline(m, n)
x = torch.ones(n, device="cuda")
ws = D.spmv_workspace(n, m, "cuda")
y = torch.empty(n, device="cuda")
torch.cuda.synchronize()
for _ in range(reps):
    pipe.run(I, J)
    D.spmv(pipe.offsets[: n + 1], pipe.indices[:m], x, out=y, ws=ws)
torch.cuda.synchronize()
print("done", n, m)
