"""BASELINE config 5 at full size on one GPU (exploration / evidence run, not a
bench value): generate the DC-SBM graph on the GPU (synth/dcsbm.py), build
the operator from the device CSR, run the single-sweep Lanczos with a
restart cap, report timings, per-kernel event times and the solution's
properties.  Properties are checked on the GPU with the library's own apply
(the oracle cannot run at 1.6e9 entries in minutes)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2210_16435_b200 import lib  # noqa: E402
from synth.dcsbm import config5  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--restarts", type=int, default=400)
ap.add_argument("--m", type=int, default=0)
ap.add_argument("--kmeans", action="store_true", help="Alg. 3 step 4 after the solve (no X copy, no property checks)")
args = ap.parse_args()
dev = torch.device("cuda:0")
torch.cuda.set_device(0)
t = time.time()
g, cfg = config5(n=args.n, device="cuda")
torch.cuda.synchronize()
torch.cuda.empty_cache()  # generator intermediates: give the memory back before the library sizes its basis
out = {"n": g.n, "nnz": g.nnz, "gen_s": time.time() - t, "meta": g.meta}
print(json.dumps(out), flush=True)
k = cfg["k_eig"]
t = time.time()
ctx = lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, g.groups, k, False, h=g.h, max_restarts=args.restarts,
                                 max_basis=args.m)
torch.cuda.synchronize()
out["build_s"] = time.time() - t
out["info"] = ctx.info()
groups_dev = g.groups.to(torch.int64)
del g
torch.cuda.empty_cache()
lib.profile_enable(ctx, True)
t = time.time()
Xd = None if args.kmeans else torch.empty((k, out["n"]), dtype=torch.float64, device=dev)
try:
    ev, _, st = lib.sfairsc_eigs(ctx, k, cfg["tol"], evecs=Xd, want_evecs=Xd is not None)
    out["status"] = "OK"
except lib.SfairscError as e:
    st = ctx.last_stats
    out["status"] = e.name
    out["error"] = str(e)
    ev = None
torch.cuda.synchronize()
out["eigs_s"] = time.time() - t
out["stats"] = st
prof = lib.profile_read(ctx)
out["eigs_kernels"] = {kk: {"ms": v["ms"], "launches": v["launches"],
                            "us": 1e3 * v["ms"] / max(1, v["launches"])} for kk, v in prof.items() if v["launches"]}
if args.kmeans and ev is not None:
    lab = torch.empty(out["n"], dtype=torch.int32, device=dev)
    l0 = lib.launch_count()
    torch.cuda.synchronize()
    t = time.time()
    _, wcss = lib.sfairsc_embed_kmeans(ctx, 1, lab)
    torch.cuda.synchronize()
    out["kmeans"] = {"s": time.time() - t, "wcss": wcss, "launches": lib.launch_count() - l0,
                     "cluster_sizes_min_max": [int(torch.bincount(lab.long(), minlength=k).min()),
                                               int(torch.bincount(lab.long(), minlength=k).max())]}
    print(json.dumps(out), flush=True)
    ctx.close()
    sys.exit(0)
print(json.dumps(out), flush=True)  # the solve's record first (the checks below are separate)
ctx.close()  # the checks need the memory the basis held
if ev is not None:
    out["evals"] = [float(x) for x in ev]
    G = Xd @ Xd.T
    out["orth_err"] = float((G - torch.eye(k, device=dev, dtype=torch.float64)).abs().max())
    # fairness F^T X = 0 (unnormalized: C = F = G - 1 z^T, first h-1 columns), computed independently in torch
    h = out["info"]["h"]
    n = out["n"]
    # per-group pairwise (tree) sums, not atomics: the check's own rounding stays ~log(n) eps
    cnt = torch.bincount(groups_dev, minlength=h).to(torch.float64)
    tot = Xd.sum(dim=1)
    FtX = torch.stack([Xd[:, groups_dev == s_].sum(dim=1) - (cnt[s_] / n) * tot for s_ in range(h - 1)])
    out["FtX_rel"] = float(FtX.norm() / Xd.norm())
    Fnorm = float(torch.sqrt(cnt[: h - 1] * (1 - cnt[: h - 1] / n)).max())  # ~ |F|_2 (diagonal-dominant F^T F)
    out["FtX_normwise"] = out["FtX_rel"] / Fnorm
    out["lambda1_rel"] = abs(out["evals"][0]) / st["sigma"]
print(json.dumps(out, indent=1), flush=True)
