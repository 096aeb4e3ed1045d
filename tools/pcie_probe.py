"""Pinned host<->device copy rates on this box: H2D alone, D2H alone and both
at once on separate streams (the floor under bench.py's e2e number)."""
import json

import torch

def rate(nbytes, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return nbytes * reps / (s.elapsed_time(e) * 1e-3) / 1e9

H = 537 << 20
D = 318 << 20
hi = torch.empty(H, dtype=torch.uint8, pin_memory=True)
di = torch.empty(H, dtype=torch.uint8, device="cuda")
ho = torch.empty(D, dtype=torch.uint8, pin_memory=True)
do = torch.empty(D, dtype=torch.uint8, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
out = {"h2d_GBps": rate(H, lambda: di.copy_(hi, non_blocking=True)),
       "d2h_GBps": rate(D, lambda: ho.copy_(do, non_blocking=True))}

def both():
    cur = torch.cuda.current_stream()
    sa.wait_stream(cur); sb.wait_stream(cur)
    with torch.cuda.stream(sa):
        di.copy_(hi, non_blocking=True)
    with torch.cuda.stream(sb):
        ho.copy_(do, non_blocking=True)
    cur.wait_stream(sa); cur.wait_stream(sb)

t = H / rate(H, both)  # seconds per (H2D + D2H) pair, in GB units
out["concurrent_pair_ms"] = t * 1e3 / 1e9 * 1e9 / 1e9 * 1e9 if False else H / (rate(H, both) * 1e9) * 1e3
out["h2d_only_ms"] = H / (out["h2d_GBps"] * 1e9) * 1e3
print(json.dumps(out))
