"""Oracle timing on the host's cores (SURVEY §8(d) "Oracle timing"): a reported
baseline, never the target.  Tier D (Alg. 2, dense FairSC) on configs 1-2 with its phase
times; Tier S (Alg. 3 with ARPACK on the paper's matrix-free apply) time-to-k on configs
1-3; host record (lscpu fields, affinity, BLAS vendor/threads via threadpoolctl, RAM).

    python tests/tools/oracle_timing.py [--tier-d 1,2] [--tier-s 1,2,3] [--out gpurun_out/oracle_timing.json]
"""
import argparse
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from oracle import fairsc, sfairsc_cpu  # noqa: E402
from synth import baseline_config  # noqa: E402


def host_record():
    rec = {"affinity_cpus": len(os.sched_getaffinity(0)), "logical_cpus": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            key, _, val = line.partition(":")
            if key.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "NUMA node(s)"):
                rec[key.strip()] = val.strip()
    except OSError:
        pass
    try:
        from threadpoolctl import threadpool_info
        rec["blas"] = [{k: d.get(k) for k in ("internal_api", "version", "num_threads", "architecture")}
                       for d in threadpool_info()]
    except ImportError:
        pass
    try:
        with open("/proc/meminfo") as f:
            rec["mem_total_gb"] = round(int(f.readline().split()[1]) / 1048576, 1)
    except OSError:
        pass
    return rec


def tier_d(c):
    g, cfg = baseline_config(c)
    k = cfg["k_eig"]
    t0 = time.perf_counter()
    Wd = g.dense()
    t1 = time.perf_counter()
    res = fairsc.fairsc_dense(Wd, g.groups, g.h, k, cfg["normalized"])
    t2 = time.perf_counter()
    return {"config": c, "n": g.n, "k": k, "dense_W_s": t1 - t0, "alg2_s": t2 - t1,
            "what": "oracle.fairsc.fairsc_dense: L, Z = null(F^T) by full SVD, (Z^T D Z)^(1/2), M, eigh (P:465-490)",
            "lambda_k": float(res.evals[k - 1])}


def tier_s(c):
    g, cfg = baseline_config(c)
    k = cfg["k_eig"]
    t0 = time.perf_counter()
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, cfg["normalized"], threads=0)
    t1 = time.perf_counter()
    res = sfairsc_cpu.sfairsc_arpack(op, k, tol=cfg["tol"], seed=1)
    t2 = time.perf_counter()
    return {"config": c, "n": g.n, "nnz": g.nnz, "k": k, "tol": cfg["tol"], "build_s": t1 - t0,
            "eigsh_s": t2 - t1, "matvecs": res.matvecs, "threads": op.threads,
            "what": "oracle.sfairsc_cpu: operator build (scipy) + ARPACK eigsh on the P:803 apply (ncv = max(2k+3, 20))",
            "lambda_k": float(res.evals[k - 1])}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--tier-d", default="1")
    ap.add_argument("--tier-s", default="1,2,3")
    ap.add_argument("--out", default="gpurun_out/oracle_timing.json")
    a = ap.parse_args()
    out = {"host": host_record(), "tier_d": [], "tier_s": []}
    print(json.dumps(out["host"]), flush=True)
    for c in [int(x) for x in a.tier_d.split(",") if x]:
        out["tier_d"].append(tier_d(c))
        print(json.dumps(out["tier_d"][-1]), flush=True)
    for c in [int(x) for x in a.tier_s.split(",") if x]:
        out["tier_s"].append(tier_s(c))
        print(json.dumps(out["tier_s"][-1]), flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
