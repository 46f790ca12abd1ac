"""§8(f) N2 measured on one B200: the Chebyshev-filtered solve (opts.filter_degree = d, CGS2 solver,
automatic cut) against the default solver (paired lagged steps) on a BASELINE config.  Per run:
status, applies, steps (= basis sweeps of the filtered solve: 3 CGS2 sweeps each), restarts, the cut,
device-synchronised wall time, per-kind kernel time (profiling on), the achieved residual and the
largest eigenvalue difference to the default run (and, at config 4, to the Tier S golden).
Optional --max-restarts bounds a run (config 5: a cost sample; the residual reached is reported).
Evidence run, not a bench value.

    python scripts/filter_eval.py [--config 4] [--degrees 0,2,3,4] [--max-restarts 0]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_16435_b200 import lib  # noqa: E402
from synth import baseline_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--degrees", default="0,2,3,4")
ap.add_argument("--max-restarts", type=int, default=0)
ap.add_argument("--profile", type=int, default=1)
ap.add_argument("--out", default=None)
args = ap.parse_args()
out_path = args.out or f"gpurun_out/filter_cfg{args.config}.json"
dev = torch.device("cuda:0")
g, cfg = baseline_config(args.config)
k = cfg["k_eig"]
rp, ci, vv = (torch.from_numpy(a).to(dev) for a in (g.row_ptr, g.col, g.val))
gr = torch.from_numpy(g.groups.astype(np.int32)).to(dev)
del g.col, g.val
torch.cuda.synchronize()
torch.cuda.empty_cache()
golden = None
gpath = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                     f"cfg{args.config}_tier_s.json")
if os.path.exists(gpath):
    golden = np.array(json.load(open(gpath))["evals"][:k])
res = {"config": args.config, "n": g.n, "k": k, "tol": cfg["tol"], "runs": []}
ref = None
for d in [int(x) for x in args.degrees.split(",")]:
    kw = {"filter_degree": d} if d >= 2 else {}
    if args.max_restarts:
        kw["max_restarts"] = args.max_restarts
    ctx = lib.sfairsc_build_operator(rp, ci, vv, gr, k, cfg["normalized"], h=g.h, **kw)
    if args.profile:
        lib.profile_enable(ctx, True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    status = "OK"
    try:
        ev, _, st = lib.sfairsc_eigs(ctx, k, cfg["tol"], want_evecs=False)
    except lib.SfairscError as e:
        ev, st, status = None, ctx.last_stats, e.name
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    run = {"degree": d, "status": status, "wall_s": wall,
           **{kk: st[kk] for kk in ("applies", "steps", "restarts", "breakdowns", "max_resid_rel", "gap_est",
                                     "filter_cut", "basis_size", "kept")}}
    if args.profile:
        prof = lib.profile_read(ctx)
        run["kernels_ms"] = {kk: round(v["ms"], 1) for kk, v in prof.items() if v["launches"]}
        run["kernel_launches"] = {kk: v["launches"] for kk, v in prof.items() if v["launches"]}
    if ev is not None:
        run["evals"] = [float(x) for x in ev]
        if ref is None and d < 2:
            ref = ev
        if ref is not None:
            run["max_abs_dlambda_vs_default"] = float(np.abs(ev - ref).max())
        if golden is not None:
            run["max_abs_dlambda_vs_tier_s"] = float(np.abs(ev - golden).max())
    ctx.close()
    res["runs"].append(run)
    print(json.dumps({kk: v for kk, v in run.items() if kk != "evals"}), flush=True)
os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
with open(out_path, "w") as f:
    json.dump(res, f, indent=1)
