"""Host-side timing of each stage of sharded_reorder_to_csr on one rank (NCCL),
synchronising after every stage -- to find gaps the CUDA events hide."""
import os, sys, time
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2306_10410_b200 import device as D
from paper_2306_10410_b200 import sharded as S
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29541")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
n = 1 << 22
I, J = D.generate_rmat(22, 16, 1)
lab = torch.from_numpy(oracle.random_labels(n, 7).astype(np.int32)).cuda()
I, J = D.gather(lab, I), D.gather(lab, J)
m = I.numel()
orig_ar, orig_a2a = dist.all_reduce, dist.all_to_all_single
T = {}
def timed(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter(); r = fn(*a, **k); torch.cuda.synchronize()
        T[name] = T.get(name, 0) + time.perf_counter() - t; return r
    return w
ops = S.DeviceOps()
for nm in ["first_occurrence_shard", "bias", "compact_relabel", "coo_to_csr", "adjacent_diff", "offset_ids", "merge_rows"]:
    setattr(ops, nm, timed(nm, getattr(ops, nm)))
S.dist.all_reduce = timed("all_reduce", orig_ar)
S.dist.all_to_all_single = timed("all_to_all", orig_a2a)
S.row_bounds = timed("row_bounds", S.row_bounds)
for it in range(4):
    T.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    S.sharded_reorder_to_csr(I, J, n, m, 0, ops=ops)
    torch.cuda.synchronize(); tt = time.perf_counter() - t0
print("total %.2f ms" % (tt * 1e3), {k: round(v * 1e3, 3) for k, v in T.items()})
# the bench's loop: flush, barrier, events around one plain (untimed-ops) step
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for sampler in (False, True):
    ts = []
    ctx = bench.ClockSampler(0) if sampler else None
    if ctx: ctx.__enter__()
    for _ in range(5):
        flush.fill_(1); torch.cuda.synchronize(); dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); S.sharded_reorder_to_csr(I, J, n, m, 0); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    if ctx: ctx.__exit__(None, None, None)
    print("bench-style loop, clock sampler" if sampler else "bench-style loop", [round(t, 3) for t in ts])
dist.destroy_process_group()
