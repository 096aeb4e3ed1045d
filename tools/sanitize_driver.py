"""Exercises every kernel family once at small sizes, for compute-sanitizer
(tools/sanitize.sh): fused pipeline (two-stage first occurrence, compaction,
relabel with the hub table, radix COO->CSR), relaxed first occurrence,
weighted CSR, SpMV fp32/fp64 (vector and scalar staging), PageRank, degree /
hub orders, destination sort, NBR, the multi-GPU ops (windowed compaction,
row cut, relative range partition) and the host transfers.  Argument
"waves": instead, one pipeline at n = 2^25 (wave-guarded first occurrence,
range-pass relabel with the fused first radix histogram).  The default run
also takes one s17 graph through the two-stage first occurrence (counting
prefix, frequency-ordered SeenSet fill) and replays a captured step through
both branches of COO->CSR's conditional radix plan."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_10410_b200 as bb  # noqa: E402
from paper_2306_10410_b200 import _host as H  # noqa: E402
from paper_2306_10410_b200 import device as D  # noqa: E402
from paper_2306_10410_b200.sharded import DeviceOps  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "waves":
    os.environ["BOBA_RL_PASSES"] = "2"   # range-pass relabel, the last pass writing the first radix histogram
    scale = 25
    I, J = D.generate_rmat(scale, 1, 3)
    n = 1 << scale
    p = D.Pipeline(I.numel(), n).run(I, J)
    torch.cuda.synchronize()
    assert int(p.offsets[n].item()) == I.numel()
    print("waves ok")
    sys.exit(0)

# two-stage first occurrence with the counting prefix (m >= 16 x 64K)
I, J = D.generate_rmat(17, 16, 2)
D.Pipeline(I.numel(), 1 << 17).run(I, J)
# the captured step: COO->CSR's conditional radix plan (n = 2^18: both plans share the first pass),
# replayed once on the narrow and once on the wide branch
n18 = 1 << 18
rng = np.random.default_rng(5)
def _edges(src):
    a = rng.integers(0, n18, src)[rng.integers(0, src, 1 << 20)]
    b = rng.integers(0, n18, 1 << 20)
    return (torch.from_numpy(a.astype(np.uint32).view(np.int32)).cuda(),
            torch.from_numpy(b.astype(np.uint32).view(np.int32)).cuda())
In, Jn = _edges(n18 // 4) if not os.environ.get("SKIP_GRAPH") else (None, None)
if In is not None:
    Iw, Jw = _edges(3 * n18 // 4)
    cp = D.Pipeline(1 << 20, n18)
    g = D.CapturedPipeline(cp, In, Jn)
    g.launch()
    In.copy_(Iw)
    Jn.copy_(Jw)
    g.launch()
    torch.cuda.synchronize()
    g.close()
scale = 14
n = 1 << scale
I, J = D.generate_rmat(scale, 8, 1)
m = I.numel()
p = D.Pipeline(m, n).run(I, J)
first = D.first_occurrence(I, J, n, relaxed=True)
w = torch.rand(m, dtype=torch.float64, device="cuda")
off, idx, wo = D.coo_to_csr(p.I2[:m], p.J2[:m], n, w)
x32 = torch.rand(n, device="cuda")
y = D.spmv(p.offsets[:n + 1], p.indices[:m], x32)
y = D.spmv(off, idx, x32, wo.float())
y64 = D.spmv(off, idx, x32.double(), wo)
D.pagerank(off, idx, wo)
D.degree_order(I, J, n, hub=False)
D.degree_order(I, J, n, hub=True)
D.sort_coo_by_destination(I, J, n, w)
D.nbr(p.offsets[:n + 1], p.indices[:m], 32)
ops = DeviceOps()
f = p.first[:n]
c, ws = ops.compact_shard_mark(f, n, m, 1000, m - 3000)
allc = torch.cat([c, c, c])
lab = ops.compact_shard_assign(f, n, m, 1000, m - 3000, allc, 3, 1, ws)
order, hubs = ops.order_from_label(p.label[:n], n)
ops.relabel(I, J, p.label[:n], hubs, n)
hl = ops.row_cut_hist(p.I2[:m], n)
cut = ops.row_cut(hl, hl, n, m, 4)
ops.range_partition(p.I2[:m], p.J2[:m], cut[:5], 4)
h = H.to_host_ids(p.indices[:m])
H.to_device_ids(h, n)
g = bb.CooGraph(n, h % n, h[::-1] % n)
bb.coo_to_csr(bb.apply_permutation(g, bb.boba_parallel(g)))
torch.cuda.synchronize()
print("sanitize driver ok")
