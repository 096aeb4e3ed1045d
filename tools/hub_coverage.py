import sys, torch, numpy as np
sys.path.insert(0, '.')
from tools.csr_ab import graph
for cfg in sys.argv[1].split(','):
    I, J, n = graph(cfg)
    deg = torch.zeros(n, dtype=torch.int64, device='cuda')
    for X in (I, J):
        for c in range(0, X.numel(), 1 << 28):
            deg += torch.bincount(X[c:c + (1 << 28)].long(), minlength=n)
    tot = deg.sum().item()
    sd = torch.sort(deg, descending=True).values
    cs = torch.cumsum(sd, 0)
    # current SeenSet: vertices whose first occurrence is in I[0:P]
    for P in (65536, 131072):
        pre = I[:P].long()
        u = torch.unique(pre)
        print(cfg, f"first-seen in I[:{P}]: {u.numel()} vertices cover {deg[u].sum().item()/tot:.3f}")
    for K in (45000, 65536, 90000):
        print(cfg, f"top-{K} by degree cover {cs[K-1].item()/tot:.3f}")
    for L in (1 << 21, 1 << 24):
        cnt = torch.bincount(I[:L].long(), minlength=n)
        top = torch.topk(cnt, 45000).indices
        print(cfg, f"top-45000 by count in I[:{L}] cover {deg[top].sum().item()/tot:.3f}")
    del I, J, deg
    torch.cuda.empty_cache()
