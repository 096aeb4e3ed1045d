"""Per-phase times of the fused pipeline (boba_reorder_to_csr_timed, CUDA
events, L2 flushed, median of R) on the bench graphs, plus an order/CSR digest
so two library builds (BOBA_LIB_PATH) can be compared for speed and output.
usage: phase_ab.py CFG[,CFG...] [R]"""
import ctypes
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.csr_ab import graph  # noqa: E402
from paper_2306_10410_b200 import _native as N  # noqa: E402
from paper_2306_10410_b200 import device as D  # noqa: E402

PHASES = ("first_occurrence", "compact", "relabel", "coo_to_csr")


def main():
    cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2"]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for cfg in cfgs:
        I, J, n = graph(cfg)
        m = I.numel()
        pipe = D.Pipeline(m, n)
        times = {k: [] for k in PHASES}
        for r in range(reps + 2):
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
            for e in evs:
                e.record()
            arr = (ctypes.c_void_p * 5)(*[e.cuda_event for e in evs])
            torch.cuda.synchronize()
            flush.fill_(1)
            N.check(N.lib.boba_reorder_to_csr_timed(
                D._p(I), D._p(J), None, m, n, D._p(pipe.first), D._p(pipe.order), D._p(pipe.label), D._p(pipe.I2),
                D._p(pipe.J2), D._p(pipe.offsets), D._p(pipe.indices), None, D._p(pipe.ws), pipe.ws.numel(), D._s(),
                arr))
            torch.cuda.synchronize()
            if r >= 2:
                for i, k in enumerate(PHASES):
                    times[k].append(evs[i].elapsed_time(evs[i + 1]))
        med = {k: round(statistics.median(v), 4) for k, v in times.items()}
        dig = [int(t[:k].to(torch.int64).mul(torch.arange(1, k + 1, device="cuda") % 1000003).sum().item())
               for t, k in ((pipe.order, n), (pipe.offsets, n + 1), (pipe.indices, m))]
        print(f"{cfg} {os.path.basename(os.environ.get('BOBA_LIB_PATH', 'default'))}: {med} "
              f"total {sum(med.values()):.4f} digest {dig}", flush=True)
        del pipe, I, J
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
