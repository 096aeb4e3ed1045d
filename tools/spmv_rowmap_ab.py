"""The library's merge-path SpMV against the row-mapped forms the north star
names (thread-, 4/8/16-lane vector- and warp-per-row; tools/spmv_rowmap.cu) and
against cuSPARSE (torch CSR @ x), on the BOBA and random-order CSR of the bench
graphs.  fp32, unit weights, the same random x, CUDA-event medians with L2
flushed before each sample; every y's largest relative error against the
library's fp64 SpMV (the oracle's precision) is reported beside its time.  usage: spmv_rowmap_ab.py CFG[,CFG...] [R]   (needs ab/libspmv_rowmap.so)"""
import ctypes
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tools.csr_ab import graph  # noqa: E402
from paper_2306_10410_b200 import device as D  # noqa: E402

rows = ctypes.CDLL(os.path.join(ROOT, "ab", "libspmv_rowmap.so"))
rows.spmv_rows.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 4 + [ctypes.c_uint32, ctypes.c_int, ctypes.c_void_p]
SMS = torch.cuda.get_device_properties(0).multi_processor_count


def timed(fn, reps, flush):
    fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return round(statistics.median(ts), 4)


def main():
    cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2"]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    for cfg in cfgs:
        I, J, n = graph(cfg)
        m = I.numel()
        pipe = D.Pipeline(m, n).run(I, J)
        csr = {"boba": (pipe.offsets[: n + 1], pipe.indices[:m]), "random": D.coo_to_csr(I, J, n)[:2]}
        del I, J
        x = torch.rand(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
        ws = D.spmv_workspace(n, m, "cuda")
        res[cfg] = {}
        for order, (off, idx) in csr.items():
            ref = torch.empty(n, device="cuda")
            y = torch.empty(n, device="cuda")
            st = torch.cuda.current_stream().cuda_stream
            ref64 = D.spmv(off, idx, x.double())
            err = lambda v: float(((v.double() - ref64).abs() / ref64.abs().clamp_min(1e-30)).max())  # noqa: E731
            errs = {}
            r = {"merge_path": timed(lambda: D.spmv(off, idx, x, out=ref, ws=ws, reuse_partition=False), reps, flush)}
            D.spmv(off, idx, x, out=ref, ws=ws)
            r["merge_path_reused_partition"] = timed(lambda: D.spmv(off, idx, x, out=ref, ws=ws, reuse_partition=True),
                                                     reps, flush)
            for L in (1, 4, 8, 16, 32):
                fn = lambda: rows.spmv_rows(L, off.data_ptr(), idx.data_ptr(), x.data_ptr(), y.data_ptr(), n, SMS, st)  # noqa: E731
                t = timed(fn, reps, flush)
                name = {1: "thread_per_row", 32: "warp_per_row"}.get(L, f"vector_{L}_lanes")
                r[name] = t
                errs[name] = err(y)
            try:
                A = torch.sparse_csr_tensor(off.view(torch.int32), idx.view(torch.int32), torch.ones(m, device="cuda"), size=(n, n))
                r["cusparse"] = timed(lambda: torch.mv(A, x), reps, flush)
                errs["cusparse"] = err(torch.mv(A, x))
                del A
            except Exception as e:  # noqa: BLE001
                r["cusparse"] = f"unavailable: {type(e).__name__}: {str(e)[:80]}"
            errs["merge_path"] = err(ref)
            r["max_rel_err_vs_fp64"] = {k: float(f"{v:.2e}") for k, v in errs.items()}
            res[cfg][order] = r
            print(cfg, order, json.dumps(r), flush=True)
        del pipe, csr, ws
        torch.cuda.empty_cache()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
