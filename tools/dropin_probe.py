"""Where the drop-in (int64 numpy) path's time goes at c2: each API call of
the reference pipeline, the id transfers alone, and the host's own copy rates
for the same bytes (numpy, one thread) as a floor reference."""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_10410_b200 as bb  # noqa: E402
from paper_2306_10410_b200 import _host as H  # noqa: E402
from paper_2306_10410_b200 import device as D  # noqa: E402
import bench  # noqa: E402


def t(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return round(statistics.median(ts) * 1e3, 2)


n, I32, J32 = bench.host_input_u32("c2")
I, J = I32.astype(np.int64), J32.astype(np.int64)
g = bb.CooGraph(n, I, J, validate=False)
p = bb.boba_parallel(g)
g2 = bb.apply_permutation(g, p)
out = {"threads": os.cpu_count(),
       "boba_parallel_ms": t(lambda: bb.boba_parallel(g)),
       "apply_permutation_ms": t(lambda: bb.apply_permutation(g, p)),
       "coo_to_csr_ms": t(lambda: bb.coo_to_csr(g2)),
       "h2d_ids_67M_ms": t(lambda: H.to_device_ids(I, n)),
       }
dv = H.to_device_ids(I, n)
out["d2h_ids_67M_ms"] = t(lambda: H.to_host_ids(dv))
buf = np.empty_like(I)
out["numpy_copy_int64_67M_ms_prefaulted"] = t(lambda: np.copyto(buf, I))
out["numpy_narrow_67M_ms"] = t(lambda: I.astype(np.uint32))
out["numpy_empty_and_fill_67M_ms"] = t(lambda: np.empty_like(I).fill(1))
print(json.dumps(out))

# boba_parallel's steps one by one
from paper_2306_10410_b200 import device as D2  # noqa: E402
steps = {}
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dI = H.to_device_ids(g.I, n, "I"); torch.cuda.synchronize(); t1 = time.perf_counter()
    dJ = H.to_device_ids(g.J, n, "J"); torch.cuda.synchronize(); t2 = time.perf_counter()
    first, order, label = D2.boba_order(dI, dJ, n, False); torch.cuda.synchronize(); t3 = time.perf_counter()
    r = H.first_to_ranks(first); t4 = time.perf_counter()
    o = H.to_host_ids(order); lb = H.to_host_ids(label); t5 = time.perf_counter()
    pp = bb.Permutation(o, lb); t6 = time.perf_counter()
    steps = {"h2d_I": t1 - t0, "h2d_J": t2 - t1, "kernels": t3 - t2, "ranks": t4 - t3, "d2h_order_label": t5 - t4,
             "Permutation": t6 - t5}
print(json.dumps({k: round(v * 1e3, 2) for k, v in steps.items()}))

# first_to_ranks pieces
res = {}
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rr = H.to_host_ids(first); t1 = time.perf_counter()
    mask = rr == 0xFFFFFFFF; t2 = time.perf_counter()
    rr[mask] = H.RANK_UNSET; t3 = time.perf_counter()
    oo = H.to_host_ids(order); t4 = time.perf_counter()
    res = {"d2h_first": t1 - t0, "mask": t2 - t1, "assign": t3 - t2, "d2h_order": t4 - t3,
           "n": first.numel(), "unset": int(mask.sum())}
print(json.dumps({k: (round(v * 1e3, 2) if isinstance(v, float) else v) for k, v in res.items()}))
