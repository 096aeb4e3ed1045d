"""Time the C port (oracle) and the numba reference on the c4 graph / prefixes (host only)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, oracle
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
t0 = time.perf_counter()
n, I, J = bench.host_input_u32(cfg)
print("gen", time.perf_counter() - t0, flush=True)
m = I.size
cores = len(os.sched_getaffinity(0))
for frac in (8, 1):
    ms = m // frac
    a, b = I[:ms].astype(np.int64), J[:ms].astype(np.int64)
    t0 = time.perf_counter()
    r = oracle.first_hit_chunked(a, b, n, cores, cores); t1 = time.perf_counter()
    order = oracle.compact_ranks(r, a, b); t2 = time.perf_counter()
    label = oracle.label_from_order(order); t3 = time.perf_counter()
    I2, J2 = oracle.apply_permutation(a, b, label); t4 = time.perf_counter()
    off, idx, _ = oracle.coo_to_csr(I2, J2, n); t5 = time.perf_counter()
    print(f"port 1/{frac}: first {t1-t0:.2f} compact {t2-t1:.2f} label {t3-t2:.2f} relabel {t4-t3:.2f} csr {t5-t4:.2f} total {t5-t0:.2f} s  {ms/(t5-t0)/1e9:.4f} GE/s", flush=True)
    del r, order, label, I2, J2, off, idx, a, b
