"""One rank over NCCL: the sharded pipeline per step through the Python
orchestration (ShardedPipeline.run) and through the one-call C ABI
(native_sharded_reorder_to_csr), CUDA events, median of R.
usage: sharded_timing2.py CFG [R]"""
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.csr_ab import graph  # noqa: E402
from paper_2306_10410_b200.sharded import ShardedPipeline, native_sharded_reorder_to_csr  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dev = torch.device("cuda", 0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
I, J, n = graph(cfg)
m = I.numel()
sp = ShardedPipeline(n, m, 0, m, dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, fn in (("python", lambda: sp.run(I, J)), ("native", lambda: native_sharded_reorder_to_csr(I, J, n, m, 0))):
    fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"{cfg} {name}: median {statistics.median(ts):.3f} ms  min {min(ts):.3f}", flush=True)
dist.destroy_process_group()
