#!/usr/bin/env python
"""Power-psi benchmark on B200 (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

A step is one full Power-psi solve (Alg. 2) of the workload to its eps
(1e-9 for config 5): init s_0 = c, T sweeps s <- sA + c with the fused L1 residual
and the device-side stop rule, and the readout psi = (sB + d)/N -- SURVEY §8(a) rows
a2-a5 -- on a graph already ingested (row a1, one-time, reported as ingest_ms).
Inputs are resident in HBM when the timed region starts.

value  = GTEPS over the solve: M * (T + 1) / time-to-eps   (T sweeps + 1 readout pass)
e2e    = same metric through the C-ABI with HOST buffers: psi_build_graph from pinned host
         arrays (H2D copy + ingest), psi_iterate, psi_get_psi to host, all inside the timed region
roofline: the sweep (k_heavy + k_sell or k_tiles + k_fix), algorithmic bytes per sweep
         B_sweep = 4M + 4(N+1) + 8 N_g + 32 N_f / measured sweep time
cpu_baseline / --impl reference: the fp64 oracle (oracle/, Alg. 2 with explicit SciPy
         CSR), single core, on a bounded row-block sample of the same graph.

Multi-GPU (torchrun, N > 1): replicas only -- each rank solves its own independent instance
(seed = rank) with no collective on the data path; value = all ranks' edges / max-over-ranks
time ("scaling": "weak").  See DESIGN.md "Multi-GPU".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_BYTES = 126 * 2**20


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _traffic_from_profiles(kernel="k_tiles", config=5):
    """Per-launch DRAM bytes of the sweep kernel from the committed ncu summary, or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"C{config}", {}).get(kernel)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.idx = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for name, v in zip(names, s[3:7]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------------------------- distributed

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def init_dist(ws, backend):
    import torch.distributed as dist
    if ws > 1 and not dist.is_initialized():
        dist.init_process_group(backend)
    return dist


def max_over_ranks(value: float, ws: int, device=None) -> float:
    """Max of a per-rank float over all ranks (the timing rule: max over ranks)."""
    if ws <= 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, ws: int, device=None) -> float:
    if ws <= 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


# --------------------------------------------------------------------------- workloads

def make_workload(config, seed, pinned):
    import psigen
    alloc = None
    if pinned:
        import torch

        def alloc(shape, dt):
            t = torch.empty(shape, dtype={np.int64: torch.int64, np.int32: torch.int32}[dt],
                            pin_memory=True)
            return t.numpy()
    w = psigen.make_config(config, seed=seed, alloc=alloc)
    if pinned:                              # the activity vectors too: every H2D is from pinned memory
        w.lam = _pinned_copy(w.lam)
        w.mu = _pinned_copy(w.mu)
    return w


def _pinned_copy(a):
    import torch
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    t.numpy()[:] = a
    return t.numpy()


def algorithmic_bytes_per_sweep(n, m, n_g, n_f):
    """4M idx + 4(N+1) offsets + 8 N_g gathered x + 32 N_f (a, g, Wt, x_t)."""
    return 4 * m + 4 * (n + 1) + 8 * n_g + 32 * n_f


# --------------------------------------------------------------------------- CPU baseline

def _row_block(w, target_edges):
    """The leaders [0, r1) of the workload's CSR with ~target_edges follow edges, all other rows
    emptied: a valid follower graph on the same N users (a bounded sample of the workload)."""
    rp = w.row_ptr
    r1 = int(np.searchsorted(rp, min(target_edges, w.m), side="left"))
    r1 = max(1, min(r1, w.n))
    m1 = int(rp[r1])
    rp1 = np.concatenate([rp[: r1 + 1], np.full(w.n - r1, m1, dtype=np.int64)])
    return rp1, w.followers[:m1], r1, m1


def cpu_oracle_sample(w, target_edges=20_000_000, sweeps=3, op=None):
    """The oracle AS IT STANDS (oracle.build_operator + oracle.power_psi: Alg. 2 with explicit
    SciPy CSR A^T, fp64, 1 core) on a bounded sample of the workload -- its leaders [0, r1) with
    ~target_edges edges, on all N users -- run for `sweeps` sweeps (eps = 0, fixed count);
    value = sample edges x sweeps / time of the power_psi call (the operator build is setup;
    pass `op` to reuse one)."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import oracle
    rp1, f1, r1, m1 = _row_block(w, target_edges)
    t0 = time.perf_counter()
    if op is None:
        op = oracle.build_operator(rp1, f1, w.lam, w.mu)
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    r = oracle.power_psi(op=op, eps=0.0, max_iters=sweeps)
    t = (time.perf_counter() - t0) / max(r.iterations, 1)
    return {"value": m1 / t / 1e9, "unit": "GTEPS", "cores": 1, "kind": "oracle",
            "ms_per_sweep": round(t * 1e3, 2), "build_operator_s": round(t_build, 2),
            "sample": f"oracle.power_psi (Alg. 2, explicit SciPy CSR, fp64, 1 thread) on the "
                      f"workload's leaders [0,{r1}) = {m1} edges over all {w.n} users, "
                      f"{r.iterations} sweeps incl. the readout, {t*1e3:.1f} ms per sweep",
            "cpu": _cpu_model(), "host_cpus": os.cpu_count()}


def oracle_time_to_eps(configs=(1, 3)):
    """PAPER.md Table III reports whole solves: the oracle's time-to-eps on
    whole BASELINE configs that fit a CPU core in seconds (oracle.power_psi, 1 thread)."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import oracle
    import psigen
    out = {}
    for k in configs:
        w = psigen.make_config(k)
        t0 = time.perf_counter()
        op = oracle.build_operator(w.row_ptr, w.followers, w.lam, w.mu)
        tb = time.perf_counter() - t0
        t0 = time.perf_counter()
        r = oracle.power_psi(op=op, eps=w.eps)
        t = time.perf_counter() - t0
        out[f"config{k}"] = {"T": r.iterations, "time_to_eps_s": round(t, 3),
                             "build_operator_s": round(tb, 3),
                             "gteps": round(w.m * (r.iterations + 1) / t / 1e9, 4), "cores": 1}
        del op, w
    return out


# Measured gather ceilings of this design (profiles/r1/ubench_gather_r1.txt): random 8-byte
# gathers from an L2-resident vector (the edge stream's gathers) and from shared memory
# (k_heavy's staged segments), per B200, G gathers/s.
GATHER_L2_GPS = 281.0
GATHER_SMEM_GPS = 1040.0


def gather_ceiling(info, sweep_ms):
    """The sweep's design ceiling from psi_get_info counts: k_heavy's entries at the measured
    shared-memory gather rate + the edge stream's gathers at the measured L2 rate (serial,
    as the kernels run), beside the HBM roofline."""
    heavy = info["heavy_entries"]
    stream = info["stream_edges"]                               # gathers of k_sell / k_tiles
    t_ms = heavy / (GATHER_SMEM_GPS * 1e9) * 1e3 + stream / (GATHER_L2_GPS * 1e9) * 1e3
    return {"heavy_entries": heavy, "stream_gathers": stream,
            "rates_gps": {"smem": GATHER_SMEM_GPS, "l2": GATHER_L2_GPS,
                          "source": "profiles/r1/ubench_gather_r1.txt"},
            "ceiling_sweep_ms": round(t_ms, 4), "frac_of_gather_ceiling": round(t_ms / sweep_ms, 4)}


def sweep_kernel(info):
    """The edge-stream kernel the library chose: the sliced-ELL sweep or the tiles."""
    return "k_sell" if info.get("sliced_ell") else "k_tiles"


def knobs(info):
    """Every PSI_* environment override in effect (none by default) and the launch shape the
    library chose, so a number can be traced to its configuration."""
    env = {k: v for k, v in sorted(os.environ.items()) if k.startswith("PSI_")}
    lib = {k: info[k] for k in ("sliced_ell", "tile_edges", "grid", "block", "hot_smem",
                                "heavy_labels", "heavy_panels", "n_heavy", "last_solver")}
    return {"env": env, "library": lib}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# --------------------------------------------------------------------------- arms

def run_reference(args, ws, rank):
    """--impl reference: the oracle as it stands on the host cores (rank 0 only)."""
    if rank != 0:
        return None
    import oracle
    w = make_workload(args.config, seed=0, pinned=False)
    rp1, f1, _, _ = _row_block(w, args.cpu_edges // 4)
    op = oracle.build_operator(rp1, f1, w.lam, w.mu)             # setup, once
    per_step = []
    for i in range(args.warmup + args.steps):
        r = cpu_oracle_sample(w, target_edges=args.cpu_edges // 4, sweeps=1, op=op)
        if i >= args.warmup:
            per_step.append(r)
    val = statistics.median([r["value"] for r in per_step])
    cb = dict(per_step[0])
    cb["value"] = val
    cb["sample"] = cb["sample"] + f"; median of {args.steps} timed steps (one sweep each)"
    ms = statistics.median([r["ms_per_sweep"] for r in per_step])
    return {"metric": METRIC, "value": val, "unit": "GTEPS", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "weak",
            "impl": "reference", "dtype": "f64", "data": "synthetic",
            "config": _config_dict(args, w), "cpu_baseline": cb,
            "e2e": {"value": val, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "vs_baseline": None}


METRIC = "GTEPS per Power-psi sweep & time-to-eps (1e-9) at 1 B200; % HBM roofline"


def _config_dict(args, w):
    import psigen
    return {"workload": f"config{args.config}: {psigen.CONFIG_NAMES[args.config]}",
            "N": w.n, "M": w.m, "eps": w.eps, "norm": "row (kappa_row, reading R1)",
            "l2": "inputs larger than L2 (int32 index stream %.2f GB vs 126 MB L2)" % (4 * w.m / 1e9),
            "parallelism": f"replicas x{args.gpus}"}


def run_ours(args, ws, rank, local):
    import torch
    import paper_2206_09960_b200 as psi

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    w = make_workload(args.config, seed=rank, pinned=True)
    n, m = w.n, w.m
    eps = w.eps
    stream = torch.cuda.current_stream()

    # ---- e2e through the C-ABI with host (pinned) buffers, measured first (before any
    # device-resident copy of the inputs exists), as a user of the public API would run it
    host = [torch.from_numpy(a) for a in (w.row_ptr, w.followers, w.lam, w.mu)]
    psi_host = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h2d = (n + 1) * 8 + m * 4 + 2 * n * 8
    d2h = n * 8
    e2e_steps = max(1, min(args.steps, 5))
    for _ in range(2):             # untimed: the first builds grow the stream-ordered pool
        with psi.PsiGraph(*host) as gh:
            gh.iterate(eps)
            gh.get_psi(out=psi_host)
    barrier(ws)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    Te = []
    parts = []
    for _ in range(e2e_steps):
        h0 = time.perf_counter()
        with psi.PsiGraph(*host) as gh:
            h1 = time.perf_counter()
            _, Tt, _ = gh.iterate(eps)
            h2 = time.perf_counter()
            gh.get_psi(out=psi_host)
            h3 = time.perf_counter()
            Te.append(Tt)
        h4 = time.perf_counter()
        parts.append([round(1e3 * (h1 - h0), 1), round(1e3 * (h2 - h1), 1),
                      round(1e3 * (h3 - h2), 1), round(1e3 * (h4 - h3), 1)])
    b.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(a.elapsed_time(b), ws, dev) / e2e_steps
    e2e_edges = sum_over_ranks(float(m) * (Te[-1] + 1), ws, dev)
    e2e_val = e2e_edges / (e2e_ms * 1e-3) / 1e9

    d_in = [torch.from_numpy(a).to(dev, non_blocking=True) for a in (w.row_ptr, w.followers, w.lam, w.mu)]
    torch.cuda.synchronize()

    g = psi.PsiGraph(*d_in)
    info = g.info()
    psi_dev = torch.empty(n, dtype=torch.float64, device=dev)

    # ---- warm-up
    for _ in range(args.warmup):
        g.iterate(eps)
        g.get_psi(out=psi_dev)
    torch.cuda.synchronize()

    # ---- timed region: K solves to eps, each with the readout's scatter of psi back to the
    # caller's labels (psi_get_psi into a device buffer: the k_unpermute of row a5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    Ts = []
    with ClockSampler(local) as clk:
        barrier(ws)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            st, T, gap = g.iterate(eps)
            g.get_psi(out=psi_dev)
            Ts.append(T)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(ws)
    ms_local = e0.elapsed_time(e1)
    ms_total = max_over_ranks(ms_local, ws, dev)
    ms_step = ms_total / args.steps
    T = Ts[-1]
    edges_local = float(m) * (T + 1) * args.steps
    edges_all = sum_over_ranks(edges_local, ws, dev)
    value = edges_all / (ms_total * 1e-3) / 1e9
    per_sweep = 3 if info["n_heavy"] > 0 else 2
    if g.info()["last_solver"] == 1:          # persistent small-graph solver: one launch per solve
        launches = 2 * len(Ts)
    else:                                     # init + 3 per sweep and readout + unpermute
        launches = sum(per_sweep * (t + 1) + 2 for t in Ts)
    trace = None
    if rank == 0:
        try:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            from launch_trace import trace as _trace
            trace = _trace(g, eps, psi_dev)
            trace["what"] = ("CUPTI (torch.profiler) over one timed step: kernels launched and "
                             "CUDA runtime calls made by psi_iterate + psi_get_psi")
        except Exception as e:   # never lose the main line over the evidence
            trace = {"error": repr(e)}

    # ---- per-launch device time of the sweep kernels: CUDA events on the library's stream
    # around every k_tiles / k_fix launch (psi_time_sweep, direct launches, 20 sweeps)
    # ---- PageRank power method (Eq. (22)) on the same ingested graph:
    # the paper's "as fast as PageRank" comparison (Table IV), alpha = 0.85, same eps
    pr_T, pr_ms = None, []
    for i in range(3):
        e0.record(stream)
        _, pr_T, _ = g.pagerank(0.85, eps)
        e1.record(stream)
        torch.cuda.synchronize()
        if i > 0:
            pr_ms.append(e0.elapsed_time(e1))
    pr_ms = statistics.median(pr_ms)
    g.iterate(eps)   # leave the context at the psi solution

    g.time_sweep(3)
    heavy_ms, tiles_ms, fix_ms = g.time_sweep(20)
    sweep_ms = heavy_ms + tiles_ms + fix_ms
    g.iterate(eps)   # leave the context at the eps solution

    # ---- roofline of the sweep
    peak, peak_kind = _peaks()
    bsweep = algorithmic_bytes_per_sweep(n, m, info["n_g"], info["n_f"])
    achieved = bsweep / (sweep_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": _traffic_from_profiles("sweep", args.config),
            "traffic_source": _traffic_from_profiles("source", args.config),
            "gather": gather_ceiling(info, sweep_ms),
            "kernel": f"one sweep = k_heavy + {sweep_kernel(info)}<sweep> + k_fix<sweep>; each "
                      "launch timed with CUDA events on the library stream (psi_time_sweep, 20 "
                      "sweeps); k_tiles_ms is the edge-stream kernel's time, whichever it is",
            "k_heavy_ms": round(heavy_ms, 4), "k_tiles_ms": round(tiles_ms, 4),
            "k_fix_ms": round(fix_ms, 4),
            "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
            "algorithmic_bytes_per_sweep": bsweep,
            "sweep_ms": round(sweep_ms, 4), "sweep_gteps": round(m / (sweep_ms * 1e-3) / 1e9, 2),
            "frac_of_8TBs_nominal": round(achieved / 8000.0, 4)}

    out = {"metric": METRIC, "value": round(value, 3), "unit": "GTEPS", "n_gpus": ws,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (psigen, seed = rank)", "config": _config_dict(args, w),
           "time_to_eps_ms": round(ms_step, 4), "iterations_T": T,
           "ingest_ms": round(info["ingest_ms"], 2), "gpu_launches": launches,
           "roofline": roof, "clocks": clk.summary(), "launch_trace": trace,
           "knobs": knobs(info),
           "pagerank": {"what": "psi_pagerank: PageRank power method, Eq. (22), alpha = 0.85, "
                                "same graph, eps and kernels (SURVEY 8(f) row 1)",
                        "time_to_eps_ms": round(pr_ms, 3), "iterations_T": pr_T,
                        "gteps": round(float(m) * pr_T / (pr_ms * 1e-3) / 1e9, 2)},
           "graph_info": {k: info[k] for k in ("n_f", "n_g", "n_leaderless", "kappa_row", "kappa_col",
                                               "rho_A", "num_tiles", "num_long_rows", "grid", "block", "hot_smem",
                                               "n_heavy", "heavy_entries", "heavy_panels", "heavy_labels",
                                               "relabeled", "sliced_ell", "sell_long_rows",
                                               "sell_pieces", "sell_words", "stream_edges")}}
    g.close()
    del d_in
    torch.cuda.empty_cache()

    out["e2e"] = {"value": round(e2e_val, 3), "unit": "GTEPS", "ms_per_step": round(e2e_ms, 2),
                  "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                  "what": "psi_build_graph(pinned host CSR) + psi_iterate(eps) + psi_get_psi(host)",
                  "host_ms_build_iterate_get_destroy": parts,
                  "median_step_ms_host": round(statistics.median(sum(p) for p in parts), 2)}
    if rank == 0 and not args.no_batch:
        try:
            out["batch"] = batch_side(w, dev, args.config, sweep_ms)
        except Exception as e:  # never lose the main line over the side measurement
            out["batch"] = {"error": repr(e)}
        torch.cuda.empty_cache()
    if rank == 0:
        try:
            out["table_iii_style"] = paper_comparison(dev)
        except Exception as e:  # never lose the main line over the side measurement
            out["table_iii_style"] = {"error": repr(e)}
    if rank == 0 and not args.no_configs:
        try:
            out["configs"] = configs_side(dev, [k for k in (1, 2, 3, 4) if k != args.config])
        except Exception as e:  # never lose the main line over the side measurement
            out["configs"] = {"error": repr(e)}
        torch.cuda.empty_cache()
    if rank == 0 and not args.no_cpu:
        try:
            out["cpu_baseline"] = cpu_oracle_sample(w, target_edges=args.cpu_edges)
            out["cpu_baseline"]["oracle_time_to_eps"] = oracle_time_to_eps((1, 3))
        except Exception as e:  # never lose the GPU line over the baseline
            out["cpu_baseline"] = {"value": None, "error": repr(e)}
    return out if rank == 0 else None


def configs_side(dev, configs):
    """Every other BASELINE.json config on this GPU (the paper's timings span all its datasets,
    P:476-479): time-to-eps (median of 5 solves + readout, after 3 warm-ups), the sweep time
    (psi_time_sweep, 20 sweeps) and its fraction of the HBM roofline."""
    import torch
    import paper_2206_09960_b200 as psi
    import psigen
    peak, _ = _peaks()
    rows = []
    for k in configs:
        w = psigen.make_config(k)
        d = [torch.from_numpy(a).to(dev) for a in (w.row_ptr, w.followers, w.lam, w.mu)]
        out = torch.empty(w.n, dtype=torch.float64, device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with psi.PsiGraph(*d) as g:
            for _ in range(3):
                g.iterate(w.eps)
                g.get_psi(out=out)
            ts = []
            for _ in range(5):
                torch.cuda.synchronize()
                e0.record()
                _, T, _ = g.iterate(w.eps)
                g.get_psi(out=out)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            g.time_sweep(3)
            hv, ti, fx = g.time_sweep(20)
            inf = g.info()
        sweep = hv + ti + fx
        byt = algorithmic_bytes_per_sweep(w.n, w.m, inf["n_g"], inf["n_f"])
        t = statistics.median(ts)
        rows.append({"config": k, "N": w.n, "M": w.m, "eps": w.eps, "T": T,
                     "time_to_eps_ms": round(t, 4), "solve_gteps": round(w.m * (T + 1) / t / 1e6, 2),
                     "sweep_ms": round(sweep, 4), "k_heavy_ms": round(hv, 4),
                     "k_tiles_ms": round(ti, 4), "k_fix_ms": round(fx, 4),
                     "sweep_kernel": sweep_kernel(inf),
                     "sweep_gteps": round(w.m / sweep / 1e6, 2), "B_sweep": byt,
                     "hbm_frac": round(byt / (sweep * 1e-3) / 1e9 / peak, 4),
                     "solver": inf["last_solver"], "ingest_ms": round(inf["ingest_ms"], 2)})
        del d, out
        torch.cuda.empty_cache()
    return rows


def batch_side(w, dev, config, single_sweep_ms, k=4):
    """k = 4 activity profiles on the same graph in ONE batch context
    (psi_build_graph_batch; x interleaved, one 32-byte gather per edge for four profiles).
    Profile 0 = the workload's own activity, 1..3 = independent draws of the same law."""
    import numpy as np
    import torch
    import paper_2206_09960_b200 as psi
    import psigen
    n, m = w.n, w.m
    lam, mu = psigen.activity_profiles(n, k, "lognormal" if config >= 3 else "uniform",
                                       pure_posters=(config == 5))
    lam[0], mu[0] = w.lam, w.mu
    d = [torch.from_numpy(np.ascontiguousarray(a)).to(dev)
         for a in (w.row_ptr, w.followers, lam, mu)]
    del lam, mu
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with psi.PsiGraph(*d) as g:
        g.time_sweep_batch(3)
        bms = g.time_sweep_batch(20)
        g.iterate(w.eps)
        ts = []
        for _ in range(2):
            torch.cuda.synchronize()
            e0.record()
            g.iterate(w.eps)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        Tp, _ = g.profile_stats()
    del d
    return {"what": "psi_build_graph_batch: 4 activity profiles, one pass over the edge stream "
                    "per sweep (SURVEY 8(f) row 4); profile 0 = this workload's activity",
            "profiles": k, "sweep_ms": round(bms, 4),
            "profile_gteps": round(k * m / (bms * 1e-3) / 1e9, 1),
            "per_profile_sweep_vs_single": round(bms / k / single_sweep_ms, 3),
            "time_to_eps_ms": round(min(ts), 3), "T_profiles": [int(t) for t in Tp]}


def paper_comparison(dev):
    """Tables III-IV of the paper on the config-1 graph (DBLP-sized, N = 10,000):
    time of Power-psi (Alg. 2), the N-systems psi by Power-NF (Alg. 1 x N, psi_nsystems) and
    PageRank (Eq. (22), alpha = 0.85), all on this GPU, eps = 1e-9."""
    import torch
    import paper_2206_09960_b200 as psi
    import psigen
    w = psigen.make_config(1)
    d = [torch.from_numpy(a).to(dev) for a in (w.row_ptr, w.followers, w.lam, w.mu)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {"workload": "config1 graph (ER N=10,000), eps = 1e-9 (P:472)"}
    with psi.PsiGraph(*d) as g:
        for name, fn in (("power_psi", lambda: g.iterate(1e-9)),
                         ("pagerank_0.85", lambda: g.pagerank(0.85, 1e-9)),
                         ("power_nf_nsystems", lambda: g.nsystems(1e-9))):
            fn()
            torch.cuda.synchronize()
            e0.record()
            r = fn()
            e1.record()
            torch.cuda.synchronize()
            res[name + "_ms"] = round(e0.elapsed_time(e1), 3)
            if name == "power_nf_nsystems":
                res["power_nf_matvecs"] = r[2]
            else:
                res[name + "_T"] = r[1]
    res["nsystems_over_power_psi"] = round(res["power_nf_nsystems_ms"] / res["power_psi_ms"], 1)
    res["paper_context"] = ("DBLP (12,591 users) on the authors' CPU, Table III: Power-psi 0.029 s, "
                            "Power-NF 17.805 s (614x)")
    return res


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-edges", type=int, default=20_000_000)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-batch", action="store_true", help="skip the 4-profile batch side line")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1-C4 side record")
    args = ap.parse_args(argv)
    ws, rank, local = dist_env()
    if args.impl == "reference":
        # the oracle runs on rank 0 only; other ranks exit without work (no rendezvous)
        out = run_reference(args, ws, rank)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if ws > 1:
        init_dist(ws, "nccl")
    out = run_ours(args, ws, rank, local)
    if out is not None:
        print(json.dumps(out), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
