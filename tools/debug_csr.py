import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_10410_b200 import device as D
import oracle
def check(n, m, seed=0):
    rng = np.random.default_rng(seed)
    I = rng.integers(0, n, m).astype(np.int64); J = rng.integers(0, n, m).astype(np.int64)
    dI = torch.from_numpy(I.astype(np.int32)).cuda(); dJ = torch.from_numpy(J.astype(np.int32)).cuda()
    off, idx, _ = D.coo_to_csr(dI, dJ, n)
    torch.cuda.synchronize()
    o, x, _ = oracle.coo_to_csr(I, J, n)
    go = off.cpu().numpy().view(np.uint32).astype(np.int64); gx = idx.cpu().numpy().view(np.uint32).astype(np.int64)
    ok_o = np.array_equal(go, o); ok_x = np.array_equal(gx, x)
    bad = np.flatnonzero(gx != x)
    print(f"n={n} m={m} offsets={ok_o} indices={ok_x} nbad={bad.size} first_bad={bad[:5]}", flush=True)
for n in [int(a) for a in sys.argv[1:]]:
    check(n, 1 << 22)
