"""SpMV per call (CUDA events, L2 flushed, partition reused, median of R) on
the BOBA and random-order CSR of the bench graphs, fp32, for whichever library
BOBA_LIB_PATH selects; prints a digest of y so builds can be compared.
usage: spmv_lib_ab.py CFG[,CFG...] [R]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.csr_ab import graph  # noqa: E402
from paper_2306_10410_b200 import device as D  # noqa: E402

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cfg in cfgs:
    I, J, n = graph(cfg)
    m = I.numel()
    pipe = D.Pipeline(m, n).run(I, J)
    csr = {"boba": (pipe.offsets[: n + 1], pipe.indices[:m]), "random": D.coo_to_csr(I, J, n)[:2]}
    del I, J
    ws = D.spmv_workspace(n, m, "cuda")
    x = torch.rand(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
    out = []
    for k, (off, idx) in csr.items():
        y = torch.empty(n, device="cuda")
        D.spmv(off, idx, x, out=y, ws=ws)
        ts = []
        for _ in range(reps):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            D.spmv(off, idx, x, out=y, ws=ws, reuse_partition=True)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        out.append(f"{k} {statistics.median(ts):.4f} ms (sum {float(y.double().sum()):.6e})")
    print(cfg, os.path.basename(os.environ.get("BOBA_LIB_PATH", "default")), " | ".join(out), flush=True)
    del pipe, csr, ws
    torch.cuda.empty_cache()
