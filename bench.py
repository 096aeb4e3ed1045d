#!/usr/bin/env python
"""BOBA reorder + COO->CSR throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4|c2|c3|c5] [--impl ours|reference]

A step = one pass of the hot path over the whole synthetic graph, inputs
already resident in HBM: first occurrence -> rank compaction -> relabel ->
COO->CSR (the reference bench's reorder_ms + convert_ms, bench.py:135-149).
Metric: GEdges/s = m / step time, whole job.

Headline workload (N = 1 and every N of a scaling run): BASELINE config c4,
R-MAT scale 26 edge factor 16 (n = 2^26, m = 2^30), the north-star graph.
N > 1 strong-scales that same graph over contiguous edge shards (sharded.py).
The line also carries, for the smaller BASELINE configs c2 (R-MAT s22), c3
(grid 4096^2) and c5 (R-MAT s24), their own step time and roofline; the
per-phase roofline against MEASURED_PEAKS.json; the end-to-end number through
the host-buffer C-ABI entry; the drop-in (reference API, int64 numpy) end to
end; the SpMV e2e speedup of BOBA vs random labels; and the reference's CPU
path timed on this host (C port and the numba reference itself).

``--impl reference`` times the reference algorithm on the host cores instead
(see run_reference).
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (kind, params, description)
    "c1": ("rmat", dict(scale=16, ef=8), "R-MAT scale 16 edge factor 8"),
    "c2": ("rmat", dict(scale=22, ef=16), "R-MAT scale 22 edge factor 16"),
    "c3": ("grid", dict(rows=4096, cols=4096), "2D grid 4096x4096"),
    "c5": ("rmat", dict(scale=24, ef=16), "R-MAT scale 24 edge factor 16"),
    "c4": ("rmat", dict(scale=26, ef=16), "R-MAT scale 26 edge factor 16"),
}
HEADLINE = "c4"
SUBCONFIGS = ("c2", "c3", "c5")
GEN_SEED, LABEL_SEED = 1, 7
SPMV_ITERS = {"c1": 10, "c2": 10, "c3": 100, "c5": 10, "c4": 10}
METRIC = "BOBA reorder+COO->CSR GEdges/s"
# reference-arm sample: a prefix of the edge stream sized to ~5 s of CPU work per step
REF_SAMPLE_DIV = {"c4": 8, "c5": 2}


def graph_size(cfg):
    kind, p, _ = CONFIGS[cfg]
    if kind == "rmat":
        return 1 << p["scale"], p["ef"] << p["scale"]
    r, c = p["rows"], p["cols"]
    return r * c, 2 * r * (c - 1) + 2 * (r - 1) * c


def alg_bytes(m, n):
    """compulsory bytes per phase (uint32 ids, 4-byte offsets)."""
    return {
        "first_occurrence": 8 * m + 4 * n,
        "compact": m / 2 + 16 * n,
        "relabel": 16 * m + 4 * n,
        "coo_to_csr": 16 * m + 4 * n + 4,
    }


PHASES = ["first_occurrence", "compact", "relabel", "coo_to_csr"]


def config_dict(cfg, world):
    """The `config` object of the JSON line -- identical in both arms."""
    kind, p, desc = CONFIGS[cfg]
    n, m = graph_size(cfg)
    gen = ("Graph500 R-MAT (a,b,c,d)=(.57,.19,.19,.05), generator seed 1" if kind == "rmat"
           else "reference generate_grid (generators.py:100-111)")
    return {"workload": f"{desc}, randomly relabelled", "graph": f"{gen}; randomize_labels seed {LABEL_SEED}",
            "n": n, "m": m, "parallelism": "single" if world == 1 else f"edge-shard{world}",
            "l2": "256 MiB L2 flush before every step; inputs 8m bytes > L2"}


def measured_traffic(cfg):
    """ncu DRAM read+write bytes per phase (profiles/traffic_<cfg>.json,
    from an ncu capture of one step of this config), or {}."""
    for name in (f"traffic_{cfg}.json",):
        if not name:
            continue
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                return json.load(f)["phases"]
        except Exception:
            continue
    return {}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


NOMINAL_HBM_GBS = 8000.0


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons with NVML while running."""

    def __init__(self, index=0, period=0.005):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {
                getattr(pynvml, "nvmlClocksThrottleReasonHwSlowdown", 0x8): "hw_slowdown",
                getattr(pynvml, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
                getattr(pynvml, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
                getattr(pynvml, "nvmlClocksThrottleReasonSwPowerCap", 0x4): "sw_power_cap",
                getattr(pynvml, "nvmlClocksThrottleReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake",
            }

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        for bit, nm in names.items():
                            if r & bit:
                                self.reasons.add(nm)
                    except Exception:
                        pass
                    time.sleep(self.period)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            pass
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "samples": len(self.samples),
            "reasons": sorted(self.reasons),
        }


# ------------------------------------------------------------------ inputs
def device_input(cfg, dev):
    """The bench's input graph for `cfg` on `dev`: the device generator (twin
    of oracle.rmat_edges / generate_grid), then randomize_labels with
    LABEL_SEED (reference io.py:294-301).  Returns (n, m, I, J) as int32
    tensors holding uint32 ids.  Also used by the parity tests, so the graph
    checked there is exactly the graph timed here."""
    import torch

    import oracle
    from paper_2306_10410_b200 import device as D

    kind, p, _ = CONFIGS[cfg]
    n, m = graph_size(cfg)
    if kind == "rmat":
        I0, J0 = D.generate_rmat(p["scale"], p["ef"], GEN_SEED, dev)
    else:
        I0, J0 = D.generate_grid(p["rows"], p["cols"], dev)
    lab = torch.from_numpy(oracle.random_labels(n, LABEL_SEED).astype(np.int32)).to(dev)
    I, J = D.gather(lab, I0), D.gather(lab, J0)
    del I0, J0, lab
    return n, m, I, J


def host_input_u32(cfg, chunk=1 << 26, limit=None):
    """The same graph built on the host by the oracle's generators (uint32,
    generated in chunks so s26 needs 8.6 GB, not 34 GB of int64).  `limit`:
    only the first `limit` edges of the edge stream."""
    import oracle

    kind, p, _ = CONFIGS[cfg]
    n, m = graph_size(cfg)
    m = m if limit is None else min(m, limit)
    lab = oracle.random_labels(n, LABEL_SEED).astype(np.uint32)
    I = np.empty(m, np.uint32)
    J = np.empty(m, np.uint32)
    if kind == "rmat":
        for e0 in range(0, m, chunk):
            e1 = min(m, e0 + chunk)
            a, b = oracle.rmat_edges(p["scale"], p["ef"], GEN_SEED, e0, e1)
            I[e0:e1], J[e0:e1] = lab[a], lab[b]
    else:
        a, b = oracle.grid_edges(p["rows"], p["cols"])
        I[:], J[:] = lab[a[:m]], lab[b[:m]]
    return n, I, J


# ------------------------------------------------------- CPU baselines
def port_pipeline_time(n, I, J, threads):
    """The C port of the reference path (oracle/boba_oracle.c): first-hit
    over `threads` chunks as first_hit_chunked, the rest single-threaded as
    in the reference.  Input int64 arrays."""
    import oracle

    t0 = time.perf_counter()
    oracle.pipeline(I, J, n, threads=threads)
    return time.perf_counter() - t0


def numba_reference_times(n, I, J, cores):
    """The UNMODIFIED reference (numba) from baseline/_ref through its own
    public API: boba_parallel fused (thread_hint=None) and chunked
    (thread_hint=cores), apply_permutation, coo_to_csr.  JIT warmed on a
    small graph first.  Returns {phase: seconds} or {"unavailable": why}."""
    src = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(src, "boba")):
        return {"unavailable": "baseline/_ref not installed (tools/install_reference.sh)"}
    os.environ.setdefault("NUMBA_NUM_THREADS", str(cores))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/boba_numba_cache")
    if src not in sys.path:
        sys.path.insert(0, src)
    try:
        import boba
    except Exception as e:  # pragma: no cover - reported, not fatal
        return {"unavailable": f"import boba failed: {e!r}"}
    small = boba.CooGraph(64, np.arange(64) % 7, (np.arange(64) * 5) % 64, validate=False)
    for th in (None, cores):
        boba.coo_to_csr(boba.apply_permutation(small, boba.boba_parallel(small, thread_hint=th)))
    g = boba.CooGraph(n, I, J, validate=False)
    out = {}
    t0 = time.perf_counter()
    p = boba.boba_parallel(g)
    out["boba_parallel_fused"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    p = boba.boba_parallel(g, thread_hint=cores)
    out["boba_parallel_chunked"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    g2 = boba.apply_permutation(g, p)
    out["apply_permutation"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    boba.coo_to_csr(g2)
    out["coo_to_csr"] = time.perf_counter() - t0
    out["pipeline"] = min(out["boba_parallel_fused"], out["boba_parallel_chunked"]) + out["apply_permutation"] \
        + out["coo_to_csr"]
    out["numba_threads"] = int(os.environ["NUMBA_NUM_THREADS"])
    return out


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def ref_sample(cfg, steps):
    """Edges per reference-arm step: the whole graph, or a prefix of its edge
    stream (same n) where the whole graph would not fit K steps in minutes."""
    n, m = graph_size(cfg)
    div = REF_SAMPLE_DIV.get(cfg, 1)
    return m // div


def run_reference(args):
    """--impl reference: the reference's CPU path on this host's cores.  The
    reference is pure Python + numba (no compiled form to build into
    oracle/_ref), so each step runs the oracle's C port of it (kind "port":
    first-hit on all cores like first_hit_chunked, compaction / relabel / CSR
    scatter single-threaded like the reference).  Under torchrun only rank 0
    works.  The numba reference itself is timed once beside it."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = max(int(os.environ.get("WORLD_SIZE", "1")), args.gpus)
    cfg = args.config
    cores = len(os.sched_getaffinity(0))
    n, m = graph_size(cfg)
    step_m = ref_sample(cfg, args.steps)
    _, I32, J32 = host_input_u32(cfg, limit=step_m)
    I, J = I32.astype(np.int64), J32.astype(np.int64)
    del I32, J32
    port_pipeline_time(n, I, J, cores)  # warm-up (page faults, OpenMP pool)
    ts = [port_pipeline_time(n, I, J, cores) for _ in range(args.steps)]
    t = sum(ts)
    value = step_m * args.steps / t / 1e9
    sample = ("full graph per step" if step_m == m else
              f"first {step_m} of the {m} edges of the edge stream per step (same n = {n}; the n-sized "
              "phases run in full, so the per-edge rate is pessimistic for the CPU)")
    numba = numba_reference_times(n, I, J, cores) if not args.no_numba else {"skipped": "--no-numba"}
    if "pipeline" in numba:
        numba["gedges_per_s"] = round(step_m / numba["pipeline"] / 1e9, 5)
        numba["sample"] = sample.replace(" per step", "")
    line = {
        "metric": METRIC, "value": round(value, 5), "unit": "GEdges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * t / args.steps, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": config_dict(cfg, world), "impl": "reference",
        "cpu_baseline": {"value": round(value, 5), "unit": "GEdges/s", "cores": cores, "kind": "port",
                         "sample": sample, "cpu": cpu_model(),
                         "note": "oracle/boba_oracle.c restates the reference (pure Python + numba); first-hit "
                                 "on all cores (first_hit_chunked), compaction, relabel and CSR scatter "
                                 "single-threaded as in the reference",
                         "numba_reference": numba},
        "e2e": {"value": round(value, 5), "unit": "GEdges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm
def _events(stream, k):
    import ctypes

    import torch

    evs = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
    for e in evs:
        e.record(stream)  # materialise the cudaEvent_t handles
    return evs, (ctypes.c_void_p * k)(*[e.cuda_event for e in evs])


def measure_config(cfg, steps, warmup, flush, dev, clocks=False, keep=False):
    """One config: W warm-up replays, K timed replays of the captured
    pipeline (CUDA events around each replay, L2 flushed before each), then
    the same number of direct launches with events at the phase boundaries.
    Returns (record, state)."""
    import torch

    from paper_2306_10410_b200 import _native as N
    from paper_2306_10410_b200 import device as D

    n, m, I, J = device_input(cfg, dev)
    pipe = D.Pipeline(m, n, dev)
    stream = torch.cuda.current_stream()
    graph = D.CapturedPipeline(pipe, I, J)
    kernels_per_step = graph.kernel_nodes()
    for _ in range(warmup):
        graph.launch()
    torch.cuda.synchronize()
    step_ms = []
    clk = ClockSampler(dev.index or 0) if clocks else None
    if clk:
        clk.__enter__()
    try:
        for _ in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.fill_(1)
            a.record(stream)
            graph.launch()
            b.record(stream)
            torch.cuda.synchronize()
            step_ms.append(a.elapsed_time(b))
    finally:
        if clk:
            clk.__exit__()
    graph.close()
    # per-phase times of the replayed step itself: the same captured graph with
    # event-record nodes at the phase boundaries
    phase_ms = {k: [] for k in PHASES}
    evs, arr = _events(stream, 5)
    tgraph = D.CapturedPipeline(pipe, I, J, events=arr)
    for _ in range(max(min(steps, 10), 3)):
        torch.cuda.synchronize()
        flush.fill_(1)
        tgraph.launch()
        torch.cuda.synchronize()
        for i, k in enumerate(PHASES):
            phase_ms[k].append(evs[i].elapsed_time(evs[i + 1]))
    tgraph.close()
    # and the uncaptured call (direct launches, the full-width radix plan), for reference
    direct_ms = []
    for _ in range(3):
        devs, darr = _events(stream, 5)
        torch.cuda.synchronize()
        flush.fill_(1)
        N.check(N.lib.boba_reorder_to_csr_timed(
            D._p(I), D._p(J), None, m, n, D._p(pipe.first), D._p(pipe.order), D._p(pipe.label), D._p(pipe.I2),
            D._p(pipe.J2), D._p(pipe.offsets), D._p(pipe.indices), None, D._p(pipe.ws), pipe.ws.numel(), D._s(),
            darr))
        torch.cuda.synchronize()
        direct_ms.append(devs[0].elapsed_time(devs[4]))
    # cheap device-side sanity on the timed output (full parity: tests/ and --verify)
    assert int(pipe.offsets[n].item()) == m
    lab = pipe.label[:n].to(torch.int64)
    assert bool(torch.all(torch.sort(lab).values == torch.arange(n, device=dev)))
    del lab
    t_step = statistics.mean(step_ms) / 1e3
    rec = {
        "config": cfg, "workload": CONFIGS[cfg][2] + ", randomly relabelled", "n": n, "m": m,
        "steps": steps, "ms_per_step": round(t_step * 1e3, 4), "value": round(m / t_step / 1e9, 3),
        "unit": "GEdges/s", "step_ms_min": round(min(step_ms), 4), "step_ms_max": round(max(step_ms), 4),
        "ms_per_step_direct": round(statistics.mean(direct_ms), 4), "kernels_per_step": kernels_per_step,
        "roofline": roofline(cfg, m, n, t_step, phase_ms),
    }
    state = dict(n=n, m=m, I=I, J=J, pipe=pipe, phase_ms=phase_ms, clocks=clk.summary() if clk else None)
    if not keep:
        state.pop("pipe")
    return rec, state


def roofline(cfg, m, n, t_step, phase_ms):
    hbm, peak_kind = peaks()
    ab = alg_bytes(m, n)
    traffic = measured_traffic(cfg)
    phases = {}
    for k in PHASES:
        t = statistics.mean(phase_ms[k]) / 1e3
        ach = ab[k] / t / 1e9
        phases[k] = {"ms": round(t * 1e3, 4), "alg_bytes": int(ab[k]), "gbs": round(ach, 1),
                     "frac": round(ach / hbm, 4), "frac_nominal_8tbs": round(ach / NOMINAL_HBM_GBS, 4),
                     "dram_bytes_ncu": traffic.get(k)}
    dom = max(PHASES, key=lambda k: phases[k]["ms"])
    total_alg = sum(ab.values())
    pipe_gbs = total_alg / t_step / 1e9
    return {
        "bound": "hbm", "kernel": dom, "achieved": phases[dom]["gbs"], "peak": hbm, "peak_kind": peak_kind,
        "unit": "GB/s", "frac": phases[dom]["frac"], "traffic": traffic.get(dom),
        "traffic_source": f"profiles/traffic_{cfg}.json (ncu, DRAM read+write per launch of the phase)"
        if traffic else None,
        "pipeline": {"alg_bytes": int(total_alg), "gbs": round(pipe_gbs, 1), "frac": round(pipe_gbs / hbm, 4),
                     "frac_nominal_8tbs": round(pipe_gbs / NOMINAL_HBM_GBS, 4),
                     "roofline_gedges_per_s": round(m / (total_alg / hbm / 1e6) / 1e6, 1)},
        "phases": phases,
    }


def spmv_speedup(cfg, state, flush, dev, k_iters):
    """e2e = (t_reorder + t_convert + k t_spmv) after BOBA vs
    (t_convert + k t_spmv) on the randomly labelled input (reference bench.py
    135-156: reorder_ms, convert_ms, kernel over the forward CSR, x = ones).
    CUDA-event medians, L2 flushed before each sample."""
    import torch

    from paper_2306_10410_b200 import device as D

    n, m, I, J, pipe = state["n"], state["m"], state["I"], state["J"], state["pipe"]
    stream = torch.cuda.current_stream()
    x = torch.ones(n, dtype=torch.float32, device=dev)
    y = torch.empty(n, dtype=torch.float32, device=dev)
    spws = D.spmv_workspace(n, m, dev)

    def time_it(fn, reps):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    t_reorder = sum(statistics.mean(state["phase_ms"][k]) for k in PHASES[:3])
    t_convert = statistics.mean(state["phase_ms"]["coo_to_csr"])
    off_b, idx_b = pipe.offsets[: n + 1], pipe.indices[:m]
    # k iterations: the first call partitions the CSR, the others reuse it (boba_spmv_ex)
    t_spmv_boba = time_it(lambda: [D.spmv(off_b, idx_b, x, out=y, ws=spws, reuse_partition=i > 0)
                                   for i in range(k_iters)], 3) / k_iters
    del pipe, off_b, idx_b
    state.pop("pipe", None)
    rnd = {}

    def convert_random():
        rnd["csr"] = D.coo_to_csr(I, J, n)

    t_conv_rand = time_it(convert_random, 3)
    off_r, idx_r, _ = rnd.pop("csr")
    t_spmv_rand = time_it(lambda: [D.spmv(off_r, idx_r, x, out=y, ws=spws, reuse_partition=i > 0)
                                   for i in range(k_iters)], 3) / k_iters
    e2e_boba = t_reorder + t_convert + k_iters * t_spmv_boba
    e2e_rand = t_conv_rand + k_iters * t_spmv_rand
    return {
        "config": cfg, "iters": k_iters, "x": "ones",
        "spmv_ms_boba": round(t_spmv_boba, 4), "spmv_ms_random": round(t_spmv_rand, 4),
        "spmv_speedup": round(t_spmv_rand / t_spmv_boba, 4),
        "convert_ms_random": round(t_conv_rand, 4), "reorder_ms": round(t_reorder, 4),
        "convert_ms_boba": round(t_convert, 4),
        "e2e_ms_boba": round(e2e_boba, 4), "e2e_ms_random": round(e2e_rand, 4),
        "e2e_speedup_boba_vs_random": round(e2e_rand / e2e_boba, 4),
        "spmv_gflops_boba": round(2 * m / t_spmv_boba / 1e6, 1),
        "spmv_hbm_frac_boba": round((4 * m + 12 * n + 4) / (t_spmv_boba / 1e3) / 1e9 / peaks()[0], 4),
    }


def e2e_host(state, steps, dev):
    """End to end through the host-buffer C-ABI entry (boba_ctx_submit_host /
    boba_ctx_wait): pinned uint32 host inputs in, order/label/CSR out, every
    graph paying its own H2D and D2H; two graphs in flight.  Beside it the
    single synchronous call and the PCIe floor (the same bytes, copies only)."""
    import torch

    from paper_2306_10410_b200 import device as D

    n, m, I, J = state["n"], state["m"], state["I"], state["J"]
    hI = torch.empty(m, dtype=torch.int32, pin_memory=True)
    hJ = torch.empty(m, dtype=torch.int32, pin_memory=True)
    hI.copy_(I)
    hJ.copy_(J)
    outs = [tuple(torch.empty(k, dtype=torch.int32, pin_memory=True) for k in (n, n, n + 1, m)) for _ in range(2)]
    hp = D.HostPipeline(m, n)
    e2e_steps = max(3, min(steps, 10))
    hp.run(hI, hJ, n, *outs[0])
    te = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        hp.run(hI, hJ, n, *outs[0])
        te.append(time.perf_counter() - t0)
    t_single = sum(te) / len(te)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tickets = []
    for k in range(e2e_steps):
        if k >= 2:
            hp.wait(tickets[k - 2])  # its host outputs are about to be reused
        tickets.append(hp.submit(hI, hJ, n, *outs[k & 1]))
    for t in tickets[-2:]:
        hp.wait(t)
    t_batch = (time.perf_counter() - t0) / e2e_steps
    assert int(outs[(e2e_steps - 1) & 1][2][n]) == m
    hp.close()
    # the PCIe floor: the same H2D and D2H bytes, copies only, both directions at once
    src = torch.empty(3 * n + 1 + m, dtype=torch.int32, device=dev)
    sa, sb = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def copies():
        cur = torch.cuda.current_stream(dev)
        sa.wait_stream(cur)
        sb.wait_stream(cur)
        with torch.cuda.stream(sa):
            I.copy_(hI, non_blocking=True)
            J.copy_(hJ, non_blocking=True)
        with torch.cuda.stream(sb):
            o = 0
            for h in outs[0]:
                h.copy_(src[o:o + h.numel()], non_blocking=True)
                o += h.numel()
        cur.wait_stream(sa)
        cur.wait_stream(sb)

    copies()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(e2e_steps):
        copies()
    ev1.record()
    torch.cuda.synchronize()
    t_pcie = ev0.elapsed_time(ev1) / 1e3 / e2e_steps
    del src, hI, hJ, outs
    return {"value": round(m / t_batch / 1e9, 4), "unit": "GEdges/s", "ms_per_step": round(t_batch * 1e3, 3),
            "h2d_bytes_per_step": 8 * m, "d2h_bytes_per_step": 4 * n + 4 * n + 4 * (n + 1) + 4 * m,
            "path": "boba_ctx_submit_host / boba_ctx_wait (pinned host uint32 buffers; outputs order, label, "
                    f"CSR); {e2e_steps} graphs, two in flight",
            "pcie_floor": {"ms_per_step": round(t_pcie * 1e3, 3), "value": round(m / t_pcie / 1e9, 4),
                           "path": "the same H2D and D2H bytes per graph, copies only, both directions concurrent"},
            "single_graph": {"value": round(m / t_single / 1e9, 4), "ms_per_step": round(t_single * 1e3, 3),
                             "path": "boba_ctx_reorder_to_csr_host (one synchronous call per graph)"}}


def e2e_dropin(cfg, reps=3):
    """The reference caller's path: int64 numpy arrays through this package's
    drop-in API, boba_parallel -> apply_permutation -> coo_to_csr (reference
    ordering.py:99-151, graph.py:253-289), host arrays in and out.  Wall
    time per graph, median of `reps` after one warm call."""
    import torch

    import paper_2306_10410_b200 as bb

    n, I32, J32 = host_input_u32(cfg)
    I, J = I32.astype(np.int64), J32.astype(np.int64)
    del I32, J32
    g = bb.CooGraph(n, I, J, validate=False)

    def run():
        p = bb.boba_parallel(g)
        g2 = bb.apply_permutation(g, p)
        return bb.coo_to_csr(g2)

    run()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        csr = run()
        ts.append(time.perf_counter() - t0)
    assert int(csr.offsets[-1]) == I.size
    t = statistics.median(ts)
    m = I.size
    return {"config": cfg, "value": round(m / t / 1e9, 4), "unit": "GEdges/s", "ms_per_graph": round(t * 1e3, 2),
            "path": "paper_2306_10410_b200.boba_parallel -> apply_permutation -> coo_to_csr on int64 numpy "
                    "CooGraph (the reference API); host arrays in, host int64 results out",
            "host_bytes_in": 16 * m, "host_bytes_out": 8 * (3 * n + 2 * m + n + 1 + m)}


def run_ours(args):
    import torch

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = args.config
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    # ---- headline config
    rec, st = measure_config(cfg, args.steps, args.warmup, flush, dev, clocks=True, keep=True)
    n, m = st["n"], st["m"]
    verify = None
    if args.verify:
        verify = verify_state(cfg, st)
    spmv = {cfg: spmv_speedup(cfg, st, flush, dev, SPMV_ITERS[cfg])} if not args.quick else {}
    st.pop("pipe", None)
    torch.cuda.empty_cache()
    e2e = e2e_host(st, args.steps, dev)
    clocks = st["clocks"]
    del st
    gc.collect()
    torch.cuda.empty_cache()

    # ---- the other BASELINE configs, each with its own step time and roofline
    subs = {}
    if not args.quick:
        for c in SUBCONFIGS:
            if c == cfg:
                continue
            r, s = measure_config(c, min(args.steps, 10), min(args.warmup, 3), flush, dev, keep=True)
            if c in ("c2", "c3"):
                spmv[c] = spmv_speedup(c, s, flush, dev, SPMV_ITERS[c])
            subs[c] = r
            del s
            gc.collect()
            torch.cuda.empty_cache()

    dropin = None
    if not args.quick:
        dropin = e2e_dropin("c2")
        torch.cuda.empty_cache()

    # ---- CPU baseline on this host (rank 0, N = 1), same graph
    cpu = None
    if not args.no_cpu:
        cpu = cpu_baseline(cfg, args)

    line = {
        "metric": METRIC, "value": rec["value"], "unit": "GEdges/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": rec["ms_per_step"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic", "config": config_dict(cfg, 1),
        "roofline": rec["roofline"], "cpu_baseline": cpu, "e2e": e2e, "e2e_dropin": dropin, "spmv": spmv,
        "configs": subs, "verify": verify,
        "gpu_launches": rec["kernels_per_step"] * args.steps,
        "launch": {"mode": "CUDA graph replay, one graph launch per step (boba_reorder_to_csr_graph_create); "
                           f"{rec['kernels_per_step']} kernels per replay (boba_graph_kernel_nodes)",
                   "ms_per_step_direct": rec["ms_per_step_direct"],
                   "phases_from": "replays of the captured step with event-record nodes at the phase boundaries "
                                  "(boba_reorder_to_csr_graph_create_timed)"},
        "step_ms_min_max": [rec["step_ms_min"], rec["step_ms_max"]],
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


def verify_state(cfg, st):
    """--verify: the timed step's outputs against the oracle's streaming
    uint32 restatement of the reference (outside the timed region)."""
    import oracle

    n, m, pipe = st["n"], st["m"], st["pipe"]
    _, hI, hJ = host_input_u32(cfg)
    u = lambda t, k: t[:k].cpu().numpy().view(np.uint32)  # noqa: E731
    bad = oracle.verify_pipeline_u32(hI, hJ, n, order=u(pipe.order, n), label=u(pipe.label, n),
                                     I2=u(pipe.I2, m), J2=u(pipe.J2, m), offsets=u(pipe.offsets, n + 1),
                                     indices=u(pipe.indices, m))
    return {"bit_exact": not bad, "mismatch": bad or None,
            "checked": "order, label, I2, J2, offsets, indices vs oracle.verify_pipeline_u32"}


def cpu_baseline(cfg, args):
    """The reference path on this host: the C port on a bounded sample (the
    reference arm's sample) and once on the whole graph, plus the numba
    reference itself on the sample."""
    cores = len(os.sched_getaffinity(0))
    n, m = graph_size(cfg)
    step_m = ref_sample(cfg, args.steps)
    _, I32, J32 = host_input_u32(cfg)
    I, J = I32[:step_m].astype(np.int64), J32[:step_m].astype(np.int64)
    port_pipeline_time(n, I, J, cores)
    ts = [port_pipeline_time(n, I, J, cores) for _ in range(2)]
    t_sample = min(ts)
    full = None
    if step_m != m and not args.no_cpu_full:
        IF, JF = I32.astype(np.int64), J32.astype(np.int64)
        tf = port_pipeline_time(n, IF, JF, cores)
        full = {"value": round(m / tf / 1e9, 5), "ms": round(tf * 1e3, 1), "sample": "full graph, one run"}
        del IF, JF
    del I32, J32
    numba = numba_reference_times(n, I, J, cores) if not args.no_numba else {"skipped": "--no-numba"}
    sample = "full graph" if step_m == m else f"first {step_m} of {m} edges of the edge stream (same n = {n})"
    if "pipeline" in numba:
        numba["gedges_per_s"] = round(step_m / numba["pipeline"] / 1e9, 5)
        numba["sample"] = sample
    return {"value": round(step_m / t_sample / 1e9, 5), "unit": "GEdges/s", "cores": cores, "kind": "port",
            "sample": f"{sample}, best of 2", "ms": round(t_sample * 1e3, 1), "cpu": cpu_model(),
            "note": "oracle/boba_oracle.c (reference restated in C); first-hit on all cores, rest single-threaded "
                    "as in the reference", "full_graph": full, "numba_reference": numba}


# ------------------------------------------------------------ multi-GPU
def run_sharded(args):
    """N GPUs (or --sharded on 1): the multi-GPU pipeline of
    paper_2306_10410_b200.sharded, strong scaling: the config's graph (c4:
    R-MAT s26, BASELINE configs[3]) cut into N contiguous edge shards."""
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2306_10410_b200 import device as D
    from paper_2306_10410_b200.sharded import ShardedPipeline, shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # --share-gpu: every rank on cuda:0 over gloo -- a functional run of the N > 1
    # flow on a one-GPU box (NCCL refuses two ranks per device); not a measurement
    local = 0 if args.share_gpu else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if not dist.is_initialized():
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29511")
        if args.share_gpu:
            dist.init_process_group("gloo", rank=rank, world_size=world)
        else:
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    cfg = args.config
    kind, p, desc = CONFIGS[cfg]
    if kind != "rmat":
        raise SystemExit("the sharded path runs the R-MAT configs")
    n, m = graph_size(cfg)
    e0, e1 = shard_range(m, rank, world)
    I0, J0 = D.generate_rmat_range(p["scale"], e0, e1 - e0, GEN_SEED, dev)
    lab = torch.from_numpy(oracle.random_labels(n, LABEL_SEED).astype(np.int32)).to(dev)
    I, J = D.gather(lab, I0), D.gather(lab, J0)
    del I0, J0, lab
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    sp = ShardedPipeline(n, m, e0, e1 - e0, dev)

    for _ in range(args.warmup):
        sp.run(I, J)
    torch.cuda.synchronize()
    dist.barrier()
    ts = []
    gc.disable()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            res = sp.run(I, J)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
    gc.enable()
    t = torch.tensor([sum(ts)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_total = float(t.item())
    value = m * args.steps / t_total / 1e9
    ms_step = 1e3 * t_total / args.steps
    assert int(res.offsets[-1].item()) == res.indices.numel()
    phases = sp.phase_times(I, J)  # one more step with events at the phase boundaries
    # row-partitioned SpMV (P5): x replicated, y slices allgathered between iterations
    spmv = sp.spmv_timing(res, SPMV_ITERS[cfg])
    # the same iterations with each owner's slice broadcast piece by piece while it computes the next
    spmv["overlapped"] = sp.spmv_timing(res, SPMV_ITERS[cfg], chunks=4)

    # end to end: pinned host shard -> device, sharded pipeline, local CSR back to pinned host buffers
    hI = torch.empty(e1 - e0, dtype=torch.int32, pin_memory=True)
    hJ = torch.empty(e1 - e0, dtype=torch.int32, pin_memory=True)
    hI.copy_(I)
    hJ.copy_(J)
    h_off = torch.empty(res.offsets.numel(), dtype=torch.int32, pin_memory=True)
    h_idx = torch.empty(res.indices.numel(), dtype=torch.int32, pin_memory=True)
    te = []
    d2h = 0
    for _ in range(max(3, min(args.steps, 5))):
        dist.barrier()
        t0 = time.perf_counter()
        I.copy_(hI, non_blocking=True)
        J.copy_(hJ, non_blocking=True)
        r2 = sp.run(I, J)
        h_off[:r2.offsets.numel()].copy_(r2.offsets, non_blocking=True)
        h_idx[:r2.indices.numel()].copy_(r2.indices, non_blocking=True)
        torch.cuda.synchronize()
        te.append(time.perf_counter() - t0)
        d2h = 4 * (r2.offsets.numel() + r2.indices.numel())
    et = torch.tensor([statistics.median(te)], dtype=torch.float64, device=dev)
    dist.all_reduce(et, op=dist.ReduceOp.MAX)
    t_e2e = float(et.item())
    hbm, peak_kind = peaks()
    per_gpu_alg = sum(alg_bytes(m, n).values()) / world
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GEdges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic", "config": config_dict(cfg, world),
        "roofline": {"bound": "hbm", "kernel": "sharded_step",
                     "achieved": round(per_gpu_alg / (ms_step / 1e3) / 1e9, 1), "peak": hbm, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": round(per_gpu_alg / (ms_step / 1e3) / 1e9 / hbm, 4), "traffic": None,
                     "note": "per-GPU share of SURVEY §8d algorithmic bytes over the whole step incl. collectives",
                     "phases": phases, "nvlink": sp.comm_bytes()},
        "step_ms": [round(1e3 * t, 3) for t in ts], "spmv": spmv, "cpu_baseline": None,
        "e2e": {"value": round(m / t_e2e / 1e9, 4), "unit": "GEdges/s", "ms_per_step": round(1e3 * t_e2e, 3),
                "h2d_bytes_per_step": 8 * (e1 - e0), "d2h_bytes_per_step": d2h,
                "path": "pinned host shards -> sharded pipeline -> row-partitioned CSR to host (per rank)"},
        "gpu_launches": sp.kernel_launches_per_step() * args.steps,
        "clocks": clk.summary(),
    }
    if args.share_gpu:
        line["share_gpu"] = "ranks share cuda:0 over gloo: functional run of the N > 1 flow, not a measurement"
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=HEADLINE, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-cpu-full", action="store_true", help="skip the full-graph run of the CPU port")
    ap.add_argument("--no-numba", action="store_true", help="skip the numba reference timing")
    ap.add_argument("--quick", action="store_true", help="headline config only (no sub-configs, SpMV, drop-in)")
    ap.add_argument("--verify", action="store_true", help="check the timed outputs against the oracle")
    ap.add_argument("--sharded", action="store_true", help="use the multi-GPU sharded pipeline even on 1 GPU")
    ap.add_argument("--share-gpu", action="store_true",
                    help="(debug) all torchrun ranks on cuda:0 over gloo: runs the N > 1 flow on one GPU")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.sharded:
        run_sharded(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
