"""COO->CSR on the 4096^2 grid, randomly labelled vs BOBA-relabelled, one call
each after a warm-up -- for `ncu --metrics gpu__time_duration.sum` launch lists
that split the phase into its radix passes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2306_10410_b200 import device as D  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
n = side * side
I0, J0 = D.generate_grid(side, side)
lab = torch.from_numpy(oracle.random_labels(n, 7).astype(np.int32)).cuda()
I, J = D.gather(lab, I0), D.gather(lab, J0)
_, _, label = D.boba_order(I, J, n)
I2, J2 = D.relabel(I, J, label, n)
for a, b in [(I, J), (I2, J2), (I, J), (I2, J2)]:
    D.coo_to_csr(a, b, n)
torch.cuda.synchronize()
print("done")
