"""Pipeline step launched directly vs replayed from a captured CUDA graph
(same buffers), R-MAT s22; CUDA-event medians with the L2 flushed."""
import os, sys, statistics
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2306_10410_b200 import device as D
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
n = 1 << scale
I, J = D.generate_rmat(scale, 16, 1)
lab = torch.from_numpy(oracle.random_labels(n, 7).astype(np.int32)).cuda()
I, J = D.gather(lab, I), D.gather(lab, J)
m = I.numel()
pipe = D.Pipeline(m, n)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        pipe.run(I, J)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    pipe.run(I, J)
torch.cuda.synchronize()
def timeit(fn, reps=20):
    ts = []
    for _ in range(reps):
        with torch.cuda.stream(s):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s); fn(); b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)
for _ in range(2):
    print("direct %.4f ms   graph %.4f ms" % (timeit(lambda: pipe.run(I, J)), timeit(g.replay)))
off = pipe.offsets[: n + 1].clone()
pipe.offsets.zero_()
g.replay(); torch.cuda.synchronize()
print("graph output identical:", bool(torch.equal(off, pipe.offsets[: n + 1])))
