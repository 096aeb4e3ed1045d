"""A/B of COO->CSR variants on the bench graphs: times boba_coo_to_csr (CUDA
events, L2 flushed, median of R) once per variant and checks every variant's
offsets/indices bit for bit against the first one.  A variant is an ENV=value
setting read by the library (e.g. BOBA_RL_PASSES) or a bare label (to compare
library builds run one after another with BOBA_LIB_PATH).
usage: csr_ab.py CFG[,CFG...] [R] [variants]   CFG in c2 c3 c5 c4 sNN"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2306_10410_b200 import _native as N  # noqa: E402
from paper_2306_10410_b200 import device as D  # noqa: E402


def graph(cfg):
    if cfg == "c3":
        n = 4096 * 4096
        I, J = D.generate_grid(4096, 4096)
    else:
        scale = {"c2": 22, "c5": 24, "c4": 26}.get(cfg) or int(cfg[1:])
        n = 1 << scale
        I, J = D.generate_rmat(scale, 16, 1)
    lab = torch.from_numpy(oracle.random_labels(n, 7).astype(np.int32)).cuda()
    return D.gather(lab, I), D.gather(lab, J), n


def main():
    cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2"]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    variants = sys.argv[3].split(",") if len(sys.argv) > 3 else ["default"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for cfg in cfgs:
        I, J, n = graph(cfg)
        m = I.numel()
        pipe = D.Pipeline(m, n).run(I, J)
        I2, J2 = pipe.I2[:m], pipe.J2[:m]
        del I, J
        ref = None
        for v in variants:
            if "=" in v:
                k, val = v.split("=", 1)
                os.environ[k] = val
            ws = torch.empty(N.lib.boba_coo_to_csr_workspace_size(m, n, 0), dtype=torch.uint8, device="cuda")
            offsets = torch.empty(n + 1, dtype=torch.int32, device="cuda")
            indices = torch.empty(m, dtype=torch.int32, device="cuda")
            ts = []
            for r in range(reps + 2):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                N.check(N.lib.boba_coo_to_csr(D._p(I2), D._p(J2), None, m, n, None, D._p(offsets), D._p(indices),
                                              None, D._p(ws), ws.numel(), D._s()))
                b.record()
                torch.cuda.synchronize()
                if r >= 2:
                    ts.append(a.elapsed_time(b))
            if ref is None:
                ref = (offsets, indices)
                same = "ref"
            else:
                same = bool(torch.equal(ref[0], offsets) and torch.equal(ref[1], indices))
            alg = 16 * m + 4 * n + 4
            med = float(np.median(ts))
            print(f"{cfg} n={n} m={m} [{v}]: median {med:.4f} ms min {min(ts):.4f} "
                  f"({alg / med / 1e6:.0f} GB/s alg) same={same}", flush=True)
            del ws
        del pipe, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
