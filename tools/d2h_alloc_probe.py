"""D2H of 67M ids (int64 host output) by output allocation: numpy default
(2 MB-page madvise), numpy without the madvise (4 KB pages), an anonymous
mmap, and a pre-faulted array (the copy + widen floor)."""
import ctypes
import mmap
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_10410_b200 import _native as N  # noqa: E402
from paper_2306_10410_b200 import device as D  # noqa: E402

n = 67_108_864
dv = torch.randint(0, 1 << 26, (n,), dtype=torch.int32, device="cuda")


def d2h(out):
    N.check(N.lib.boba_device_to_host_ids(D._p(dv), n, ctypes.c_void_p(out.ctypes.data), D._s()))


def timed(alloc, reps=5):
    ts = []
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = alloc()
        d2h(out)
        ts.append(time.perf_counter() - t0)
        del out
    return round(statistics.median(ts[1:]) * 1e3, 2)


def mm():
    buf = mmap.mmap(-1, n * 8)
    return np.frombuffer(buf, dtype=np.int64, count=n)


res = {"numpy_default": timed(lambda: np.empty(n, dtype=np.int64))}
np._core.multiarray._set_madvise_hugepage(False)
res["numpy_4k_pages"] = timed(lambda: np.empty(n, dtype=np.int64))
np._core.multiarray._set_madvise_hugepage(True)
res["mmap_4k"] = timed(mm)
pre = np.empty(n, dtype=np.int64)
pre.fill(0)
res["prefaulted"] = timed(lambda: pre)
print(res, "threads", os.cpu_count())
