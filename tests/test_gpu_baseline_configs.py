"""Parity at the BASELINE.json sizes, on exactly the graphs bench.py times.

For each benchmarked configuration (c2 R-MAT s22 ef16, c3 grid 4096^2, c5
R-MAT s24 ef16, c4 R-MAT s26 ef16 = the north-star graph) this builds the
bench's device input (bench.device_input), runs the fused pipeline both as
direct launches and as the captured CUDA graph the bench replays, and checks
every output -- order, label, relabelled COO, offsets, indices -- bit for bit
against the oracle's streaming uint32 restatement of the reference
(oracle.verify_pipeline_u32: first_hit_order_sequential, label, apply_
permutation, coo_to_csr with the stable cursor scatter).  The input itself
is rebuilt on the host by the oracle's generators and compared, so the
device generator cannot hide an error.  SpMV (fp32, the bench's precision)
is checked against the oracle's fp64 row sums within rtol 1e-5 on a seeded
U[0,1) vector.

These exercise the size-dependent code paths no small case reaches: the
8-bit SeenSet tags (s22), the 16-bit wave-guarded sweep and the no-hub-table
relabel (n = 2^24), the geometric waves up to 2^30 positions and the two
range passes of relabel with the fused first radix histogram (s26), 3 and 4
radix passes.  (The 16-bit sweep without waves, n in (2^22, 2^23], is
test_gpu_parity.py::test_sixteen_bit_static_sweep_without_waves.)
"""

import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

SPMV_RTOL = 1e-5


def _mem_available_gb():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) / 1e6
    except OSError:
        pass
    return 0.0


@pytest.fixture(scope="module")
def torch_dev():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("cfg", ["c2", "c3", "c5", "c4"])
def test_bench_graph_bit_exact_vs_oracle(torch_dev, cfg):
    torch = torch_dev
    import bench
    from paper_2306_10410_b200 import device as D

    n, m = bench.graph_size(cfg)
    need_host = 24 * m / 1e9 + 8  # u32 inputs + pulled results + oracle scratch, GB
    need_dev = 44 * m / 1e9 + 2
    free_dev = torch.cuda.mem_get_info()[0] / 1e9
    if _mem_available_gb() < need_host or free_dev < need_dev:
        pytest.skip(f"{cfg} needs ~{need_host:.0f} GB host / {need_dev:.0f} GB device memory")
    dev = torch.device("cuda", torch.cuda.current_device())
    n, m, I, J = bench.device_input(cfg, dev)
    hn, hI, hJ = bench.host_input_u32(cfg)
    assert hn == n and hI.size == m
    # the timed input is the oracle's input
    assert np.array_equal(I.cpu().numpy().view(np.uint32), hI), "device generator != host generator (I)"
    assert np.array_equal(J.cpu().numpy().view(np.uint32), hJ), "device generator != host generator (J)"

    pipe = D.Pipeline(m, n, dev).run(I, J)
    torch.cuda.synchronize()
    direct = {k: getattr(pipe, k).clone() for k in ("order", "label", "offsets", "indices")}
    graph = D.CapturedPipeline(pipe, I, J)  # what bench.py replays per step
    for k in ("order", "label", "offsets", "indices", "I2", "J2"):
        getattr(pipe, k).fill_(-1)           # the replay must rewrite every output
    graph.launch()
    graph.launch()
    torch.cuda.synchronize()
    graph.close()
    for k, v in direct.items():
        assert torch.equal(v, getattr(pipe, k)), f"graph replay != direct launch ({k})"
    del direct

    u = lambda t, k: t[:k].cpu().numpy().view(np.uint32)  # noqa: E731
    got = dict(order=u(pipe.order, n), label=u(pipe.label, n), I2=u(pipe.I2, m), J2=u(pipe.J2, m),
               offsets=u(pipe.offsets, n + 1), indices=u(pipe.indices, m))
    bad = oracle.verify_pipeline_u32(hI, hJ, n, **got)
    assert bad == {}, f"{cfg}: first mismatch per array {bad}"

    # SpMV over the reordered CSR (the bench's fp32 path) vs the oracle's fp64 row sums
    rng = np.random.default_rng(1234)
    x = rng.random(n, dtype=np.float32)
    off_t, idx_t = pipe.offsets[: n + 1], pipe.indices[:m]
    y = D.spmv(off_t, idx_t, torch.from_numpy(x).to(dev)).cpu().numpy()
    off, idx = got["offsets"].astype(np.int64), got["indices"].astype(np.int64)
    del pipe, I, J
    torch.cuda.empty_cache()
    y_ref = oracle.spmv_pull(off, idx, x.astype(np.float64))
    np.testing.assert_allclose(y.astype(np.float64), y_ref, rtol=SPMV_RTOL, atol=0)
