#!/usr/bin/env python
"""s-FairSC on B200 — benchmark (contract in the task statement).

Workload (N=1): BASELINE config 4 — normalized s-FairSC on an m-SBM with
n = 4,000,000, h = 10 (Zipf 1.1 groups), k = 50, mean degree 32 (~1.28e8
nnz), tol 1e-8; the configuration the north star's "applies/s & HBM % at
n = 4M" target names (configs 1-3 are parity-test cases).

One STEP = one pass of the whole hot path: build
the operator from the device-resident CSR (validation, degrees, sigma,
factored projector) and run the thick-restart Lanczos eigensolve to the
k = 50 smallest eigenpairs at the residual target, incl. the final true
residual check.  `value` = operator applies L^sigma w executed per second
over the timed steps (whole job); `ms_per_step` = time-to-k-eigenvectors.

The timed solves run with the library's per-launch profiling OFF.  Also
reported: the §8(d) metric-1 apply rate (>= 200 back-to-back single-vector
L^sigma applies, CUDA events on the launching stream, median of 5) and the
paired-apply rate; `roofline` of the dominant kernel from one extra profiled
solve run right after the timed region (CUDA events around every launch on
the library's stream); `e2e` through the C ABI from pinned host buffers; and
`cpu_baseline` = the oracle (Tier S, the paper's matrix-free operator, scipy
SpMV threaded over the host's cores) on a bounded sample, with a host record.

Multi-GPU (torchrun, N > 1): one problem row-partitioned over the ranks
(NCCL INIT logging on, so the rank count is visible in the log).
`--config 5 --max-restarts R` runs the 50M-vertex DC-SBM graph (generated on
each GPU) with a fixed thick-restart budget: applies/s of the same Lanczos
work at every N (the E(P) measurement of §8(d) metric 2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C] [--n N] [--tol T] [--max-restarts R]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback (only if MEASURED_PEAKS.json is absent)

METRIC = "projected-operator applies/s (L^sigma inside the full s-FairSC eigensolve); time-to-k-eigvecs = ms_per_step"


def workload(args, g, normalized, k, tol):
    """The workload string both arms print (same config, same metric)."""
    return (f"BASELINE config {args.config}" + (" (reduced n)" if args.n else "")
            + f": normalized={normalized} m-SBM n={g.n}, nnz={g.nnz}, h={g.h}, k={k}, tol={tol}")


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return FALLBACK_HBM_GBS, "fallback"


# Random 8-byte gathers through the L1tex -> L2 request path: 287 G sectors/s on one B200 whatever the occupancy
# or gathers in flight (scripts/micro/gather_paths.cu, profiles/r2_exp/gather_paths_ABC.txt).
GATHER_SECTORS_PER_S = 287e9


def _gather_ceiling(info, nnz, n, d):
    """The SpMV's own ceiling beside the HBM roofline: one L2 sector per gathered entry plus the
    CSR stream's sectors, at the measured random-sector rate."""
    if 8.0 * n > 1.34 * 48 * 2**20:
        return None  # column-blocked SpMV (gathered vector beyond L2): DESIGN.md §10
    nnz = int(info.get("nnz", nnz))  # this rank's rows (row-partitioned runs)
    stream_bytes = (4 if info.get("unit_weights") else 12) * nnz + 4 * (n + 1)
    sectors = nnz + stream_bytes / 32.0
    floor_us = 1e6 * sectors / GATHER_SECTORS_PER_S
    us = 1e3 * d["ms"] / max(1, d["launches"])
    return {"sectors_per_launch": sectors, "rate_sectors_per_s": GATHER_SECTORS_PER_S, "floor_us": floor_us,
            "us_per_launch": us, "frac": floor_us / us if us > 0 else None,
            "source": "measured random-gather sector rate, profiles/r2_exp/gather_paths_ABC.txt (DESIGN.md §6.1)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [x.strip() for x in out.stdout.strip().split(",")]
                if len(parts) == 6:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_graph(cfg_id, n_override, device="cpu"):
    """The BASELINE config's graph (configs 1-4: numpy m-SBM on the host; config 5: the DC-SBM
    generated on `device`).  Every rank of a row-partitioned run generates the same seeded graph
    and keeps its row block."""
    if cfg_id == 5:
        from synth.dcsbm import config5
        return config5(n=n_override, device=device)
    from synth import baseline_config
    return baseline_config(cfg_id, n=n_override)


def host_record():
    """The CPU the oracle baseline runs on: lscpu summary, affinity, BLAS, RAM."""
    rec = {"logical_cpus": os.cpu_count(), "affinity_cpus": len(os.sched_getaffinity(0))}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "CPU max MHz",
                             "NUMA node(s)"):
                rec[k.strip()] = v.strip()
    except Exception as e:  # noqa: BLE001
        rec["lscpu"] = f"unavailable: {e}"
    try:
        from threadpoolctl import threadpool_info
        rec["blas"] = [{k: d.get(k) for k in ("internal_api", "version", "num_threads", "architecture")}
                       for d in threadpool_info() if d.get("user_api") == "blas"]
    except Exception as e:  # noqa: BLE001
        rec["blas"] = f"unavailable: {e}"
    try:
        with open("/proc/meminfo") as f:
            rec["mem_total_gb"] = round(int(f.readline().split()[1]) / 1048576, 1)
    except Exception:  # noqa: BLE001
        pass
    return rec


def _oracle_applies(op, n, budget_s, max_applies=None):
    w = np.random.default_rng(0).standard_normal(n)
    c0 = time.process_time()
    t0 = time.perf_counter()
    cnt = 0
    while True:
        w = op.apply(w)
        w /= np.linalg.norm(w)
        cnt += 1
        if time.perf_counter() - t0 > budget_s or (max_applies and cnt >= max_applies):
            break
    wall = time.perf_counter() - t0
    return cnt, wall, time.process_time() - c0


def cpu_baseline(g, cfg, budget_s=15.0):
    """The oracle as it stands (Tier S matrix-free L^sigma apply: scipy CSR SpMV cut into
    row blocks on a thread pool over every core of the affinity set, normal-equations projector on
    the threaded BLAS) on a bounded sample: as many applies as fit in ~budget_s.  cores = CPU time /
    wall time actually used."""
    from oracle import sfairsc_cpu
    t0 = time.perf_counter()
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, cfg["normalized"], threads=0)
    t_build = time.perf_counter() - t0
    cnt, wall, cpu = _oracle_applies(op, g.n, budget_s)
    return {"value": cnt / wall, "unit": "applies/s", "cores": max(1, round(cpu / wall)), "kind": "oracle",
            "threads": op.threads,
            "sample": f"{cnt} Tier-S L^sigma applies (scipy CSR SpMV on {op.threads} threads + normal-equations "
                      f"projector, P:799-818) on the same n={g.n} graph in {wall:.1f} s (operator build "
                      f"{t_build:.1f} s excluded); the full ARPACK solve at this size does not finish in minutes",
            "s_per_apply": wall / cnt, "host": host_record()}


def run_reference(args):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return
    g, cfg = make_graph(args.config, args.n)
    if args.config == 5:
        g = g.host()
    from oracle import sfairsc_cpu
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, cfg["normalized"], threads=0)
    per_step = args.ref_applies
    for _ in range(args.warmup):
        _oracle_applies(op, g.n, 1e9, per_step)
    cnt, wall, cpu = 0, 0.0, 0.0
    for _ in range(args.steps):
        c, w_, p_ = _oracle_applies(op, g.n, 1e9, per_step)
        cnt, wall, cpu = cnt + c, wall + w_, cpu + p_
    value = cnt / wall
    cores = max(1, round(cpu / wall))
    line = {"metric": METRIC, "value": value, "unit": "applies/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / max(1, args.steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": workload(args, g, cfg["normalized"], cfg["k_eig"], cfg["tol"]),
                       "step": f"{per_step} oracle applies (the full ARPACK solve does not finish in minutes at this size)"},
            "cpu_baseline": {"value": value, "unit": "applies/s", "cores": cores, "kind": "oracle",
                             "threads": op.threads,
                             "sample": f"{args.steps}x{per_step} Tier-S applies, scipy SpMV on {op.threads} threads, "
                                       f"n={g.n}", "host": host_record()},
            "e2e": {"value": value, "unit": "applies/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n", type=int, default=None, help="override n (reduced-size runs; not a bench value)")
    ap.add_argument("--tol", type=float, default=None)
    ap.add_argument("--max-restarts", type=int, default=0,
                    help="> 0: fixed thick-restart budget (scaling runs; the solve reports applies/s of that work)")
    ap.add_argument("--apply-reps", type=int, default=200)
    ap.add_argument("--ref-applies", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-kmeans", action="store_true")
    ap.add_argument("--quiet", action="store_true")
    ap.add_argument("--apply-only", action="store_true", help="exploration: skip the solves")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    ws, rank, local = _dist_env()
    if ws > 1:  # the rank count of every communicator shows up in the log (driver evidence)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    import torch
    import torch.distributed as dist
    if ws > 1:
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2210_16435_b200 import lib

    t_gen = time.perf_counter()
    g, cfg = make_graph(args.config, args.n, device=dev)
    on_device = args.config == 5
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    k = cfg["k_eig"]
    tol = args.tol if args.tol is not None else cfg["tol"]
    normalized = cfg["normalized"]
    n_glob, nnz_glob = g.n, g.nnz
    # N > 1: one problem row-partitioned across the ranks: each rank holds an nnz-balanced
    # row block of W and of every n-vector; NCCL all-gather / all-reduce inside the solver
    comm, row_kw = None, {}
    if on_device:
        rp_all = g.row_ptr.cpu().numpy() if ws > 1 else None
        r0, r1 = 0, g.n
        if ws > 1:
            comm = lib.comm_from_torch(local)
            cuts = lib.partition_rows(rp_all, ws)
            r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
            row_kw = {"comm": comm, "n_global": g.n, "row_offset": r0}
        a, b = int(g.row_ptr[r0].item()), int(g.row_ptr[r1].item())
        rp = (g.row_ptr[r0:r1 + 1] - a).to(torch.int32).contiguous()
        ci = g.col[a:b].contiguous()
        vv = g.val[a:b].contiguous()
        gr = g.groups[r0:r1].to(torch.int32).contiguous()
        del g
        g = None
        torch.cuda.empty_cache()
        h = cfg["h"] if "h" in cfg else 8
        h_rp = h_ci = h_vv = h_gr = None
    else:
        h_rp, h_ci, h_vv, h_gr = g.row_ptr, g.col, g.val, g.groups.astype(np.int32)
        if ws > 1:
            comm = lib.comm_from_torch(local)
            cuts = lib.partition_rows(g.row_ptr, ws)
            h_rp, h_ci, h_vv, h_gr = lib.row_block(g.row_ptr, g.col, g.val, g.groups, int(cuts[rank]),
                                                   int(cuts[rank + 1]))
            row_kw = {"comm": comm, "n_global": g.n, "row_offset": int(cuts[rank])}
        rp = torch.from_numpy(h_rp).to(dev)
        ci = torch.from_numpy(h_ci).to(dev)
        vv = torch.from_numpy(h_vv).to(dev)
        gr = torch.from_numpy(h_gr).to(dev)
        h = g.h
    n_loc = rp.numel() - 1
    X = torch.empty((k, n_loc), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    budget = {"max_restarts": args.max_restarts} if args.max_restarts > 0 else {}

    def solve(ctx, evecs):
        try:
            ev, _, st = lib.sfairsc_eigs(ctx, k, tol, evecs=evecs, want_evecs=evecs is not None)
        except lib.SfairscError as e:  # a restart budget ends without convergence: the work done is the step
            if not (budget and e.name == "E_NO_CONVERGENCE"):
                raise
            ev, st = np.full(k, np.nan), ctx.last_stats
        return ev, st

    def step(profile=False):
        ctx = lib.sfairsc_build_operator(rp, ci, vv, gr, k, normalized, h=h, cuda_stream=stream.cuda_stream,
                                         **row_kw, **budget)
        if profile:
            lib.profile_enable(ctx, True)
        ev, st = solve(ctx, X)
        prof = lib.profile_read(ctx) if profile else None
        info = ctx.info()
        ctx.close()
        return ev, st, prof, info

    def barrier():
        if ws > 1:
            dist.barrier()

    if args.apply_only:
        args.warmup = 0
        args.steps = 0
    # ---- warm-up ----
    for _ in range(args.warmup):
        step()
    barrier()
    torch.cuda.synchronize()
    # ---- timed region (device clock, CUDA events on the launching stream; library profiling off) ----
    launches0 = lib.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    stats = []
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            ev, st, _, info = step()
            stats.append(st)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = e0.elapsed_time(e1) if args.steps else 0.0
    launches = lib.launch_count() - launches0
    ms_t = torch.tensor([ms], device=dev)
    if ws > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    applies = sum(s["applies"] for s in stats)  # one partitioned problem: every rank counts the same applies
    value = applies / (ms / 1e3) if ms > 0 else 0.0

    # ---- per-kernel roofline: one extra solve with CUDA events around every launch (not timed above) ----
    peak, peak_kind = _peaks()
    roofline = None
    if args.steps:
        p0 = torch.cuda.Event(enable_timing=True)
        p1 = torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        _, pst, prof, _ = step(profile=True)
        p1.record(stream)
        torch.cuda.synchronize()
        prof_ms = p0.elapsed_time(p1)
        kinds = {kk: v for kk, v in prof.items() if v["launches"]}
        tot_kernel_ms = sum(v["ms"] for v in kinds.values())
        dom = max(kinds, key=lambda x: kinds[x]["ms"])
        d = kinds[dom]
        achieved = d["alg_bytes"] / (d["ms"] / 1e3) / 1e9 if d["ms"] > 0 else 0.0
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                traffic = json.load(f).get(dom)
        roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "spmv_variant": ("pattern-only: unit weights detected at build, the implied values are not "
                                     "streamed; bytes still count 12 B per entry (SURVEY §8(d))")
                    if info.get("unit_weights") else "value-streaming CSR",
                    "frac": achieved / peak, "frac_of_8TBps_nominal": achieved / 8000.0,
                    "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs copy bandwidth)",
                    "traffic": traffic, "share_of_step": d["ms"] / prof_ms if prof_ms > 0 else None,
                    "alg_bytes_per_launch": d["alg_bytes"] / max(1, d["launches"]),
                    "us_per_launch": 1e3 * d["ms"] / max(1, d["launches"]),
                    "measured": "one profiled solve right after the timed region: CUDA events around every launch "
                                "on the library's (= the bench's) stream; algorithmic bytes per DESIGN.md §6",
                    "profiled_solve_ms": prof_ms, "profiled_solve_applies": pst["applies"],
                    "gather_ceiling": _gather_ceiling(info, nnz_glob, n_glob, d) if dom == "spmv" else None,
                    "per_kernel": {kk: {"ms": v["ms"], "launches": v["launches"],
                                        "us_per_launch": 1e3 * v["ms"] / v["launches"],
                                        "GBps": (v["alg_bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else None,
                                        "share": v["ms"] / tot_kernel_ms if tot_kernel_ms else None}
                                   for kk, v in sorted(kinds.items(), key=lambda x: -x[1]["ms"])}}

    # ---- applies: §8(d) metric 1 (single-vector, >= 200 back-to-back, median of 5) and paired ----
    ctx = lib.sfairsc_build_operator(rp, ci, vv, gr, k, normalized, h=h, cuda_stream=stream.cuda_stream, **row_kw)
    info = ctx.info()
    reps = max(200, args.apply_reps)
    x1 = torch.randn(n_loc, dtype=torch.float64, device=dev, generator=torch.Generator(dev).manual_seed(7))
    nb = 8 if ws == 1 else 1
    xs = x1.repeat(nb, 1)
    ys = torch.empty_like(xs)
    single = lib.sfairsc_apply_single if ws == 1 else lib.sfairsc_apply
    for _ in range(2):
        single(ctx, xs, ys)
    a0 = torch.cuda.Event(enable_timing=True)
    a1 = torch.cuda.Event(enable_timing=True)
    runs = []
    for _ in range(5):
        barrier()
        a0.record(stream)
        for _ in range(reps // nb):
            single(ctx, xs, ys)
        a1.record(stream)
        torch.cuda.synchronize()
        runs.append(a0.elapsed_time(a1) / ((reps // nb) * nb))
    apply_ms = float(np.median(runs))
    n, nnz = n_glob, nnz_glob
    alg_single = 12.0 * nnz + 4.0 * (n + 1) + 9.0 * n + 16.0 * n  # CSR + (d or s) + g + w + y
    apply_only = {"metric1_single_applies_per_s": 1e3 / apply_ms, "us_per_apply": 1e3 * apply_ms,
                  "alg_bytes_per_apply": alg_single, "alg_GBps": alg_single / (apply_ms / 1e3) / 1e9,
                  "frac_of_peak": alg_single / (apply_ms / 1e3) / 1e9 / peak,
                  "frac_of_8TBps_nominal": alg_single / (apply_ms / 1e3) / 1e9 / 8000.0,
                  "runs_us": [1e3 * r for r in runs], "applies_per_run": (reps // nb) * nb,
                  "how": "sfairsc_apply_ex(SFAIRSC_APPLY_SINGLE) on copies of one seeded vector, one SpMV per apply; "
                         "CUDA events on the launching stream around each run, median of 5 runs"}
    if ws == 1 and h <= 16:  # interleaved pairs: one SpMM per two applies
        for _ in range(2):
            lib.sfairsc_apply(ctx, xs, ys)
        a0.record(stream)
        for _ in range(reps // nb):
            lib.sfairsc_apply(ctx, xs, ys)
        a1.record(stream)
        torch.cuda.synchronize()
        pair_ms = a0.elapsed_time(a1) / ((reps // nb) * nb)
        alg_pair = (12.0 * nnz + 4.0 * (n + 1) + 9.0 * n) / 2.0 + 16.0 * n
        apply_only["paired"] = {"applies_per_s": 1e3 / pair_ms, "us_per_apply": 1e3 * pair_ms,
                                "alg_bytes_per_apply": alg_pair, "alg_GBps": alg_pair / (pair_ms / 1e3) / 1e9}
    ctx.close()

    # ---- e2e through the C ABI from pinned host buffers ----
    e2e = None
    if not args.no_e2e and args.steps:
        if on_device:
            h_rp, h_ci, h_vv, h_gr = rp.cpu().numpy(), ci.cpu().numpy(), vv.cpu().numpy(), gr.cpu().numpy()
        hrp = torch.from_numpy(h_rp).pin_memory()
        hci = torch.from_numpy(h_ci).pin_memory()
        hvv = torch.from_numpy(h_vv).pin_memory()
        hgr = torch.from_numpy(h_gr).pin_memory()
        hX = torch.empty((k, n_loc), dtype=torch.float64).pin_memory()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_app = 0
        for _ in range(args.steps):
            ctx = lib.sfairsc_build_operator(hrp, hci, hvv, hgr, k, normalized, h=h, cuda_stream=stream.cuda_stream,
                                             **row_kw, **budget)
            _, st = solve(ctx, hX)
            e2e_app += st["applies"]
            ctx.close()
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        el_t = torch.tensor([el], device=dev)
        if ws > 1:
            dist.all_reduce(el_t, op=dist.ReduceOp.MAX)
        h2d = h_rp.nbytes + h_ci.nbytes + h_vv.nbytes + h_gr.nbytes  # this rank's block
        d2h = 8 * n_loc * k + 8 * k
        e2e = {"value": e2e_app / float(el_t.item()), "unit": "applies/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * float(el_t.item()) / args.steps,
               "note": "host-timed (perf_counter) with device synchronised; CSR+groups H2D inside build, X D2H inside eigs"}

    # ---- Alg. 3 step 4 (not part of the metric): k-means on the rows of H, labels left on the device ----
    kmeans = None
    if ws == 1 and not args.no_kmeans and not args.apply_only and not budget:
        ctx = lib.sfairsc_build_operator(rp, ci, vv, gr, k, normalized, h=h, cuda_stream=stream.cuda_stream)
        solve(ctx, X)
        lab = torch.empty(n_loc, dtype=torch.int32, device=dev)
        l0 = lib.launch_count()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, wcss = lib.sfairsc_embed_kmeans(ctx, 1, lab)
        torch.cuda.synchronize()
        kmeans = {"s": time.perf_counter() - t0, "wcss": wcss, "gpu_launches": lib.launch_count() - l0,
                  "note": "sfairsc_embed_kmeans(seed 1) on a fresh solve's eigenvectors: k-means++ + Lloyd "
                          "(<= 300 iterations) x 10 restarts (reading R16); outside every timed region"}
        ctx.close()

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not on_device:
        cpu = cpu_baseline(g, cfg)

    if rank == 0 and args.apply_only:
        print(json.dumps({"apply_only": apply_only, "n": n_glob, "nnz": nnz_glob, "spmv_vector": info["spmv_vector"],
                          "generator_s": t_gen}), flush=True)
    elif rank == 0:
        last = stats[-1]
        line = {
            "metric": METRIC,
            "value": value, "unit": "applies/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / max(1, args.steps), "higher_is_better": True,
            "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"BASELINE config {args.config}" + (" (reduced n)" if args.n else "")
                                   + f": normalized={normalized} {'DC-SBM' if args.config == 5 else 'm-SBM'} "
                                     f"n={n_glob}, nnz={nnz_glob}, h={h}, k={k}, tol={tol}"
                                   + (f", thick-restart budget {args.max_restarts}" if budget else ""),
                       "step": "build operator from device CSR (A0-A3) + thick-restart Lanczos to k eigenpairs (A4-A11)"
                               + (f"; stopped after {args.max_restarts} restarts (fixed work per N)" if budget else ""),
                       "l2": f"inputs larger than L2 (CSR {(12 * nnz_glob + 4 * n_glob) / 1e9:.2f} GB, Krylov basis "
                             f"{8 * n_glob * (last['basis_size'] + 1) / 1e9:.2f} GB >> 126 MB)",
                       "parallelism": "1 GPU" if ws == 1 else f"row-partitioned over {ws} GPUs (NCCL all-gather of "
                                                               f"the projected vector + fused all-reduces per step)",
                       "generator_s": t_gen},
            "solve": {"applies_per_step": applies / max(1, args.steps), "steps": last["steps"],
                      "restarts": last["restarts"], "breakdowns": last["breakdowns"],
                      "max_resid_rel": last["max_resid_rel"], "gap_est": last["gap_est"], "sigma": last["sigma"],
                      "converged": last["converged"], "basis": last["basis_size"], "kept": last["kept"],
                      "lambda_k": float(ev[-1]), "lambda_2": float(ev[1]) if len(ev) > 1 else None},
            "apply_only": apply_only,
            "roofline": roofline,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "kmeans": kmeans,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "spmv_vector": info["spmv_vector"],
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
