#!/usr/bin/env python
"""BOBA reorder + COO->CSR throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c5|c4] [--impl ours|reference]

A step = one pass of the hot path over the whole synthetic graph, inputs
already resident in HBM: first occurrence -> rank compaction -> relabel ->
COO->CSR (reference bench.py:135-149: reorder_ms + convert_ms).  Metric:
GEdges/s = m / step time, whole job (sum over ranks).  The JSON line also
carries the per-phase roofline against MEASURED_PEAKS.json, the end-to-end
number through the host-buffer C-ABI entry (H2D + pipeline + D2H), the SpMV
e2e speedup of BOBA vs the randomly labelled CSR, and the CPU oracle timed
on this host.  ``--impl reference`` times the reference algorithm's CPU
restatement (oracle/, the reference is pure Python/numba and has no compiled
form to build) on the host cores instead.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (kind, params, human description)
    "c1": ("rmat", dict(scale=16, ef=8), "R-MAT scale 16 edge factor 8"),
    "c2": ("rmat", dict(scale=22, ef=16), "R-MAT scale 22 edge factor 16"),
    "c3": ("grid", dict(rows=4096, cols=4096), "2D grid 4096x4096"),
    "c5": ("rmat", dict(scale=24, ef=16), "R-MAT scale 24 edge factor 16"),
    "c4": ("rmat", dict(scale=26, ef=16), "R-MAT scale 26 edge factor 16"),
}
GEN_SEED, LABEL_SEED = 1, 7
SPMV_ITERS = {"c1": 10, "c2": 10, "c3": 100, "c5": 10, "c4": 10}


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


def measured_traffic(cfg):
    """DRAM bytes per phase from the committed ncu --set full capture
    (profiles/traffic.json; measured on c2 only)."""
    if cfg != "c2":
        return {}
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)["phases"]
    except Exception:
        return {}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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


# ------------------------------------------------------------- CPU (oracle)
def host_graph(cfg):
    """The same synthetic graph on the host, int64 (oracle generator =
    bit-identical twin of the device generator)."""
    import oracle

    kind, p, _ = CONFIGS[cfg]
    n, m = graph_size(cfg)
    if kind == "rmat":
        I, J = oracle.rmat_edges(p["scale"], p["ef"], GEN_SEED)
    else:
        I, J = oracle.grid_edges(p["rows"], p["cols"])
    lab = oracle.random_labels(n, LABEL_SEED)
    return n, lab[I], lab[J]


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


def host_input_u32(cfg, chunk=1 << 26):
    """The same graph built on the host by the oracle's generators (uint32,
    generated in chunks so s26 needs 8.6 GB, not 34 GB of int64)."""
    import oracle

    kind, p, _ = CONFIGS[cfg]
    n, m = graph_size(cfg)
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
        I[:], J[:] = lab[a], lab[b]
    return n, I, J


def cpu_pipeline_time(n, I, J, threads):
    import oracle

    t0 = time.perf_counter()
    oracle.pipeline(I, J, n, threads=threads)
    return time.perf_counter() - t0


def run_reference(args):
    """--impl reference: the reference algorithm on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    cores = len(os.sched_getaffinity(0))
    world = max(int(os.environ.get("WORLD_SIZE", "1")), args.gpus)
    kind, p, desc = CONFIGS[args.config]
    workload = desc + ", randomly relabelled"
    if world > 1 and kind == "rmat":
        # the GPU arm's weak-scaled graph (scale + log2 N); each step times a
        # prefix of its edge stream of one GPU's share (the config's m)
        import math

        scale = p["scale"] + int(round(math.log2(world)))
        n, m = 1 << scale, p["ef"] << scale
        step_m = p["ef"] << p["scale"]
        I, J = oracle.rmat_edges(scale, p["ef"], GEN_SEED, 0, step_m)
        lab = oracle.random_labels(n, LABEL_SEED)
        I, J = lab[I], lab[J]
        workload = f"R-MAT scale {scale} edge factor {p['ef']}, randomly relabelled (weak scaling from {desc})"
    else:
        n, m = graph_size(args.config)
        n, I, J = host_graph(args.config)
        # bound the run: each step is the full graph when K <= 12, else a prefix
        # of the edge stream (same n) sized so K steps stay within a few minutes
        step_m = m if args.steps <= 12 else max(1 << 20, int(m * 12 / args.steps))
    Is, Js = I[:step_m], J[:step_m]
    for _ in range(min(args.warmup, 1)):
        cpu_pipeline_time(n, Is, Js, cores)
    ts = [cpu_pipeline_time(n, Is, Js, cores) for _ in range(args.steps)]
    t = sum(ts)
    value = step_m * args.steps / t / 1e9
    sample = f"{'full graph' if step_m == m else f'first {step_m} edges of the edge stream'} per step, {args.steps} steps"
    line = {
        "metric": "BOBA reorder+COO->CSR GEdges/s",
        "value": round(value, 5),
        "unit": "GEdges/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1e3 * t / args.steps, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int64",
        "data": "synthetic",
        "config": {"workload": workload, "n": n, "m": m},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 5), "unit": "GEdges/s", "cores": cores, "kind": "port",
                         "sample": sample,
                         "note": "oracle/boba_oracle.c restates the reference (pure Python + numba); "
                                 "first-hit uses all cores (reference first_hit_chunked), compaction, "
                                 "relabel and CSR scatter are single-threaded as in the reference"},
        "e2e": {"value": round(value, 5), "unit": "GEdges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def spmv_speedup(D, I, J, pipe, n, m, k_iters, flush, stream, t_reorder=None, t_convert=None):
    """e2e = (t_reorder + t_convert + k t_spmv) after BOBA vs
    (t_convert + k t_spmv) on the randomly labelled input (reference bench.py
    135-156: reorder_ms, convert_ms, kernel over the forward CSR, x = ones).
    Times are CUDA-event medians with the L2 flushed before each sample."""
    import ctypes

    import torch

    from paper_2306_10410_b200 import _native as N

    x = torch.ones(n, dtype=torch.float32, device=I.device)
    y = torch.empty(n, dtype=torch.float32, device=I.device)
    spws = D.spmv_workspace(n, m, I.device)

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

    if t_reorder is None:
        # phase times of the fused pipeline call, from its own events
        ph = {"reorder": [], "convert": []}
        for _ in range(4):
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
            for e in evs:
                e.record(stream)
            arr = (ctypes.c_void_p * 5)(*[e.cuda_event for e in evs])
            torch.cuda.synchronize()
            flush.fill_(1)
            N.check(N.lib.boba_reorder_to_csr_timed(
                D._p(I), D._p(J), None, m, n, D._p(pipe.first), D._p(pipe.order), D._p(pipe.label),
                D._p(pipe.I2), D._p(pipe.J2), D._p(pipe.offsets), D._p(pipe.indices), None, D._p(pipe.ws),
                pipe.ws.numel(), D._s(), arr))
            torch.cuda.synchronize()
            ph["reorder"].append(evs[0].elapsed_time(evs[3]))
            ph["convert"].append(evs[3].elapsed_time(evs[4]))
        t_reorder = statistics.median(ph["reorder"][1:])
        t_convert = statistics.median(ph["convert"][1:])
    off_b, idx_b = pipe.offsets[: n + 1], pipe.indices[:m]
    # k iterations: the first call partitions the CSR, the others reuse it (boba_spmv_ex)
    t_spmv_boba = time_it(lambda: [D.spmv(off_b, idx_b, x, out=y, ws=spws, reuse_partition=i > 0)
                                   for i in range(k_iters)], 3) / k_iters
    rnd = {}

    def convert_random():
        rnd["csr"] = D.coo_to_csr(I, J, n)

    t_conv_rand = time_it(convert_random, 3)
    off_r, idx_r, _ = rnd["csr"]
    t_spmv_rand = time_it(lambda: [D.spmv(off_r, idx_r, x, out=y, ws=spws, reuse_partition=i > 0)
                                   for i in range(k_iters)], 3) / k_iters
    e2e_boba = t_reorder + t_convert + k_iters * t_spmv_boba
    e2e_rand = t_conv_rand + k_iters * t_spmv_rand
    return {
        "n": n, "m": m, "iters": k_iters, "x": "ones",
        "spmv_ms_boba": round(t_spmv_boba, 4), "spmv_ms_random": round(t_spmv_rand, 4),
        "convert_ms_random": round(t_conv_rand, 4), "reorder_ms": round(t_reorder, 4),
        "convert_ms_boba": round(t_convert, 4),
        "e2e_ms_boba": round(e2e_boba, 4), "e2e_ms_random": round(e2e_rand, 4),
        "e2e_speedup_boba_vs_random": round(e2e_rand / e2e_boba, 4),
        "spmv_gflops_boba": round(2 * m / t_spmv_boba / 1e6, 1),
    }


# ----------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2306_10410_b200 import _native as N
    from paper_2306_10410_b200 import device as D

    world = 1  # N > 1 runs the sharded pipeline (run_sharded)
    rank = 0
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = args.config
    kind, p, desc = CONFIGS[cfg]
    n, m = graph_size(cfg)

    # ---- synthetic input, randomly relabelled (reference io.py:294-301)
    if kind == "rmat":
        I0, J0 = D.generate_rmat(p["scale"], p["ef"], GEN_SEED + rank, dev)
    else:
        I0, J0 = D.generate_grid(p["rows"], p["cols"], dev)
    lab = torch.from_numpy(oracle.random_labels(n, LABEL_SEED + rank).astype(np.int32)).to(dev)
    I, J = D.gather(lab, I0), D.gather(lab, J0)
    del I0, J0
    torch.cuda.synchronize()

    pipe = D.Pipeline(m, n, dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()
    s = D._s()
    P = D._p
    lib = N.lib
    import ctypes

    def make_events():
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        for e in evs:
            e.record(stream)  # materialise the cudaEvent_t handles
        return evs, (ctypes.c_void_p * 5)(*[e.cuda_event for e in evs])

    def step(ev=None):
        # one fused C-ABI call: first occurrence -> compaction -> relabel -> COO->CSR
        N.check(lib.boba_reorder_to_csr_timed(
            P(I), P(J), None, m, n, P(pipe.first), P(pipe.order), P(pipe.label), P(pipe.I2), P(pipe.J2),
            P(pipe.offsets), P(pipe.indices), None, P(pipe.ws), pipe.ws.numel(), s, ev[1] if ev else None))

    # The timed step is the whole pipeline captured once into a CUDA graph
    # (boba_reorder_to_csr_graph_create) and replayed: one launch per step.
    graph = D.CapturedPipeline(pipe, I, J)
    for _ in range(args.warmup):
        graph.launch()
    torch.cuda.synchronize()
    phase_names = ["first_occurrence", "compact", "relabel", "coo_to_csr"]
    phase_ms = {k: [] for k in phase_names}
    step_ms, direct_ms = [], []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.fill_(1)  # L2 flush outside the timed events
            a.record(stream)
            graph.launch()
            b.record(stream)
            torch.cuda.synchronize()
            step_ms.append(a.elapsed_time(b))
    torch.cuda.synchronize()
    # per-phase breakdown: the same pipeline launched directly with events at
    # the phase boundaries (boba_reorder_to_csr_timed), same number of steps
    for _ in range(max(args.steps, 3)):
        ev = make_events()
        torch.cuda.synchronize()
        flush.fill_(1)
        step(ev)
        torch.cuda.synchronize()
        ev = ev[0]
        for i, k in enumerate(phase_names):
            phase_ms[k].append(ev[i].elapsed_time(ev[i + 1]))
        direct_ms.append(ev[0].elapsed_time(ev[4]))
    graph.close()
    t_total = sum(step_ms) / 1e3
    if world > 1:
        tt = torch.tensor([t_total], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total = float(tt.item())
        dist.barrier()
    ms_step = 1e3 * t_total / args.steps
    value = m * world * args.steps / t_total / 1e9

    # ---- verify the timed output once (cheap device-side invariants)
    lab_out = pipe.label[:n].to(torch.int64)
    assert int(pipe.offsets[n].item()) == m
    assert bool(torch.all(torch.sort(lab_out).values == torch.arange(n, device=dev)))

    # ---- roofline per phase
    hbm, peak_kind = peaks()
    ab = alg_bytes(m, n)
    traffic = measured_traffic(cfg)
    phases = {}
    for k in phase_names:
        t = statistics.mean(phase_ms[k]) / 1e3
        ach = ab[k] / t / 1e9
        phases[k] = {"ms": round(t * 1e3, 4), "alg_bytes": int(ab[k]), "gbs": round(ach, 1),
                     "frac": round(ach / hbm, 4), "dram_bytes_ncu": traffic.get(k)}
    dom = max(phase_names, key=lambda k: phases[k]["ms"])
    total_alg = sum(ab.values())
    roofline = {
        "bound": "hbm", "kernel": dom, "achieved": phases[dom]["gbs"], "peak": hbm, "peak_kind": peak_kind,
        "unit": "GB/s", "frac": phases[dom]["frac"], "traffic": traffic.get(dom),
        "traffic_source": "profiles/traffic.json (ncu --set full, DRAM read+write per launch)" if traffic else None,
        "pipeline_frac": round(total_alg / (ms_step / 1e3) / 1e9 / hbm, 4),
        "pipeline_alg_bytes": int(total_alg), "phases": phases,
    }

    # ---- SpMV e2e speedup: BOBA (reorder+convert+k SpMV) vs random labels (convert + k SpMV)
    t_reorder = sum(statistics.mean(phase_ms[k]) for k in phase_names[:3])
    t_convert = statistics.mean(phase_ms["coo_to_csr"])
    spmv_info = spmv_speedup(D, I, J, pipe, n, m, SPMV_ITERS[cfg], flush, stream, t_reorder, t_convert)
    spmv_info["config"] = cfg
    if cfg == "c2" and not args.no_spmv_c3:
        # the SURVEY d1 headline pairing: the road-like grid (c3) with 100 SpMV iterations
        del pipe
        torch.cuda.empty_cache()
        n3, m3 = graph_size("c3")
        G0, G1 = D.generate_grid(CONFIGS["c3"][1]["rows"], CONFIGS["c3"][1]["cols"], dev)
        lab3 = torch.from_numpy(oracle.random_labels(n3, LABEL_SEED).astype(np.int32)).to(dev)
        I3, J3 = D.gather(lab3, G0), D.gather(lab3, G1)
        del G0, G1, lab3
        pipe3 = D.Pipeline(m3, n3, dev)
        c3 = spmv_speedup(D, I3, J3, pipe3, n3, m3, SPMV_ITERS["c3"], flush, stream)
        c3["config"] = "c3"
        spmv_info = {"c2": spmv_info, "c3": c3,
                     "headline": "c3 (SURVEY d1: grid, k = 100 SpMV iterations)"}
        del pipe3, I3, J3
        torch.cuda.empty_cache()
        pipe = None

    # ---- end to end through the host-buffer C-ABI entry (pinned buffers)
    hI = torch.empty(m, dtype=torch.int32, pin_memory=True)
    hJ = torch.empty(m, dtype=torch.int32, pin_memory=True)
    hI.copy_(I)
    hJ.copy_(J)
    h_order = torch.empty(n, dtype=torch.int32, pin_memory=True)
    h_label = torch.empty(n, dtype=torch.int32, pin_memory=True)
    h_off = torch.empty(n + 1, dtype=torch.int32, pin_memory=True)
    h_idx = torch.empty(m, dtype=torch.int32, pin_memory=True)
    del pipe
    torch.cuda.empty_cache()
    hp = D.HostPipeline(m, n)
    e2e_steps = max(3, min(args.steps, 10))
    hp.run(hI, hJ, n, h_order, h_label, h_off, h_idx)
    # (a) one graph per call (latency): H2D, pipeline, D2H back to back
    te = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        hp.run(hI, hJ, n, h_order, h_label, h_off, h_idx)
        te.append(time.perf_counter() - t0)
    t_single = sum(te) / len(te)
    # (b) a stream of graphs through the asynchronous API: two in flight, so
    # graph k+1's H2D overlaps graph k's compute and D2H.  Every graph still
    # pays its own H2D and D2H; outputs alternate between two host buffer sets.
    outs = [(h_order, h_label, h_off, h_idx)]
    outs.append(tuple(torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in outs[0]))
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
    # (c) the PCIe floor under (b): the same bytes per graph copied with no compute,
    # H2D and D2H concurrently on their own streams (pinned buffers as above)
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
            for h in (h_order, h_label, h_off, h_idx):
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
    del src
    t_e2e = t_batch
    if world > 1:
        tt = torch.tensor([t_e2e], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    e2e = {"value": round(m * world / t_e2e / 1e9, 4), "unit": "GEdges/s", "ms_per_step": round(t_e2e * 1e3, 3),
           "h2d_bytes_per_step": 8 * m, "d2h_bytes_per_step": 4 * n + 4 * n + 4 * (n + 1) + 4 * m,
           "path": "boba_ctx_submit_host / boba_ctx_wait (pinned host uint32 buffers; outputs order, label, CSR); "
                   f"{e2e_steps} graphs, two in flight",
           "pcie_floor": {"ms_per_step": round(t_pcie * 1e3, 3), "value": round(m / t_pcie / 1e9, 4),
                          "path": "the same H2D and D2H bytes per graph, copies only, both directions concurrent"},
           "single_graph": {"value": round(m / t_single / 1e9, 4), "ms_per_step": round(t_single * 1e3, 3),
                            "path": "boba_ctx_reorder_to_csr_host (one synchronous call per graph)"}}

    # ---- CPU baseline on this host (rank 0, N=1 only), same graph
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = len(os.sched_getaffinity(0))
        hI64 = I.cpu().numpy().view(np.uint32).astype(np.int64)
        hJ64 = J.cpu().numpy().view(np.uint32).astype(np.int64)
        ts = []
        t_start = time.perf_counter()
        while len(ts) < 3 and (time.perf_counter() - t_start) < 25:
            ts.append(cpu_pipeline_time(n, hI64, hJ64, cores))
        tc = statistics.median(ts)
        cpu = {"value": round(m / tc / 1e9, 5), "unit": "GEdges/s", "cores": cores, "kind": "port",
               "sample": f"full graph, {len(ts)} runs (median)", "ms": round(tc * 1e3, 1),
               "note": "oracle/boba_oracle.c (reference restated in C); first-hit on all cores, "
                       "rest single-threaded as in the reference"}

    line = {
        "metric": "BOBA reorder+COO->CSR GEdges/s",
        "value": round(value, 3),
        "unit": "GEdges/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic",
        "config": {"workload": desc + ", randomly relabelled (Graph500 a,b,c=.57,.19,.19; seed 1; labels seed 7)",
                   "n": n, "m": m, "parallelism": f"replicas{world}" if world > 1 else "single",
                   "l2": "256 MiB L2 flush between steps; inputs 8m bytes > L2"},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "spmv": spmv_info,
        "gpu_launches": launches_per_step(m, n) * args.steps,
        "launch": {"mode": "CUDA graph replay, one graph launch per step (boba_reorder_to_csr_graph_create)",
                   "ms_per_step_direct": round(statistics.mean(direct_ms), 4),
                   "phases_from": "direct launches with phase events (boba_reorder_to_csr_timed)"},
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_sharded(args):
    """N GPUs (or --sharded on 1): the multi-GPU pipeline of
    paper_2306_10410_b200.sharded over contiguous edge shards.  Weak scaling
    for R-MAT configs: scale = config scale + log2(N), so every GPU holds the
    config's edge count (c2: 67M edges per GPU)."""
    import math

    import torch
    import torch.distributed as dist

    import oracle
    from paper_2306_10410_b200 import device as D
    from paper_2306_10410_b200.sharded import shard_range, sharded_reorder_to_csr

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
    kind, p, desc = CONFIGS[args.config]
    if kind != "rmat":
        raise SystemExit("the sharded path runs the R-MAT configs")
    scale = p["scale"] + int(round(math.log2(world)))
    n, m = 1 << scale, p["ef"] << scale
    e0, e1 = shard_range(m, rank, world)
    I0, J0 = D.generate_rmat_range(scale, e0, e1 - e0, GEN_SEED, dev)
    lab = torch.from_numpy(oracle.random_labels(n, LABEL_SEED).astype(np.int32)).to(dev)
    I, J = D.gather(lab, I0), D.gather(lab, J0)
    del I0, J0, lab
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        return sharded_reorder_to_csr(I, J, n, m, e0)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    ts = []
    gc.disable()  # no collector pauses between the host-synchronising collectives of a step
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            res = step()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
    gc.enable()
    t = torch.tensor([sum(ts)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_total = float(t.item())
    value = m * args.steps / t_total / 1e9
    ms_step = 1e3 * t_total / args.steps
    # sanity on the last step's output (local, cheap)
    assert int(res.offsets[-1].item()) == res.indices.numel()

    # end to end: pinned host shard -> device, sharded pipeline, local CSR back to host
    hI = torch.empty(e1 - e0, dtype=torch.int32, pin_memory=True)
    hJ = torch.empty(e1 - e0, dtype=torch.int32, pin_memory=True)
    hI.copy_(I)
    hJ.copy_(J)
    h_off = torch.empty(res.offsets.numel() + 4096, dtype=torch.int32, pin_memory=True)
    h_idx = torch.empty(2 * (e1 - e0) + 4096, dtype=torch.int32, pin_memory=True)
    te = []
    for k in range(max(3, min(args.steps, 5))):
        dist.barrier()
        t0 = time.perf_counter()
        I.copy_(hI, non_blocking=True)
        J.copy_(hJ, non_blocking=True)
        r2 = step()
        no, ni = r2.offsets.numel(), r2.indices.numel()
        if no <= h_off.numel():
            h_off[:no].copy_(r2.offsets, non_blocking=True)
        if ni <= h_idx.numel():
            h_idx[:ni].copy_(r2.indices, non_blocking=True)
        torch.cuda.synchronize()
        te.append(time.perf_counter() - t0)
    et = torch.tensor([sum(te) / len(te)], dtype=torch.float64, device=dev)
    dist.all_reduce(et, op=dist.ReduceOp.MAX)
    t_e2e = float(et.item())
    hbm, peak_kind = peaks()
    per_gpu_alg = sum(alg_bytes(m, n).values()) / world
    line = {
        "metric": "BOBA reorder+COO->CSR GEdges/s",
        "value": round(value, 3),
        "unit": "GEdges/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic",
        "config": {"workload": f"R-MAT scale {scale} edge factor {p['ef']} sharded over {world} GPU(s), randomly "
                               f"relabelled (weak scaling from {desc})", "n": n, "m": m,
                   "parallelism": f"edge-shard{world}: allreduce-MIN + all-to-all by row range (NCCL)",
                   "l2": "256 MiB L2 flush between steps"},
        "roofline": {"bound": "hbm", "kernel": "sharded_step", "achieved": round(per_gpu_alg / (ms_step / 1e3) / 1e9, 1),
                     "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": round(per_gpu_alg / (ms_step / 1e3) / 1e9 / hbm, 4), "traffic": None,
                     "note": "per-GPU share of SURVEY §8d algorithmic bytes over the whole step incl. collectives"},
        "step_ms": [round(1e3 * t, 3) for t in ts],
        "cpu_baseline": None,
        "e2e": {"value": round(m / t_e2e / 1e9, 4), "unit": "GEdges/s", "ms_per_step": round(1e3 * t_e2e, 3),
                "h2d_bytes_per_step": 8 * m, "d2h_bytes_per_step": int(4 * (n + world) + 4 * m),
                "path": "pinned host shards -> sharded pipeline -> row-partitioned CSR to host"},
        # first-hit, 2x bias, mark/scan/assign, relabel, degrees, scan, range partition (4),
        # offset ids, local CSR (3 per radix pass + row starts + suffix-min)
        "gpu_launches": args.steps * (1 + 2 + 3 + 1 + 1 + 1 + 4 + 1
                                      + 3 * csr_passes(max(res.row_hi - res.row_lo, 1)) + 2),
        "clocks": clk.summary(),
    }
    if args.share_gpu:
        line["share_gpu"] = "ranks share cuda:0 over gloo: functional run of the N > 1 flow, not a measurement"
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def csr_passes(n):
    bits = 0 if n <= 1 else (n - 1).bit_length()
    return 0 if bits == 0 else -(-bits // 8)


def launches_per_step(m, n):
    """Kernels boba_reorder_to_csr launches (csrc/api.cu): first occurrence
    (two-stage: prefix pass, SeenSet build, main sweep; + scalar tail),
    mark/record-scan/assign + the hub-table build, relabel (+ scalar tail),
    the offsets[n] store, per radix pass upsweep/scan/downsweep, suffix-min."""
    tail = 1 if m % 4 else 0
    kk = max((n - 1).bit_length() if n > 1 else 0, 14)
    prefix = 131072 if kk - 14 <= 8 else 65536
    first_hit = (3 if (kk - 14 <= 16 and m >= 16 * prefix) else 1) + tail
    compact = 3 + (1 if kk - 14 <= 16 else 0)
    return first_hit + compact + (1 + tail) + 1 + 3 * csr_passes(n) + 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-spmv-c3", action="store_true", help="skip the c3 (grid, 100 SpMV) e2e comparison")
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
