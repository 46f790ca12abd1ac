"""§8(f) N3: the paper's "s-FairSC is as fast as SC" (at h = 10, n = 1e4,
s-FairSC takes 62 % of SC's time in MATLAB on a laptop) measured on one B200.

For each n and h in {2, 5, 10}: one Experiment-1 graph (k = 5 fair planted clusters,
h equal groups, a, b, c, d = (10, 7, 4, 1)(log n / n)^(2/3), unit weights), generated on the GPU
(synth/msbm_gpu.py).  On that graph, through the C ABI, normalized (the paper's Fig. 8 runs
normalized SC / FairSC):
  * SC        = Alg. 1: the same solver with no constraint (h = 1, every vertex in one group);
  * s-FairSC  = Alg. 3 with the h groups;
each: build, eigensolve to the k = 5 smallest eigenpairs at tol 1e-10 (device-synchronised wall
time, median of `--reps`), applies; then k-means (Alg. 3 step 4) and the error rate against
the planted fair clusters (Eq. err).  Evidence run, not a bench value.

    python scripts/exp1_cost.py [--ns 10000,100000,300000,600000] [--hs 2,5,10] [--reps 3]
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
from synth.msbm_gpu import exp1_msbm_torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ns", default="10000,100000,300000,600000")
ap.add_argument("--hs", default="2,5,10")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--out", default="gpurun_out/exp1_cost.json")
args = ap.parse_args()
dev = torch.device("cuda:0")
k = 5
rows = []


def error_rate(truth, labels, k):
    """Eq. err: (1/n) min over cluster relabellings of ||H^ J - H||_F^2 = 2 (1 - best agreement / n)."""
    from scipy.optimize import linear_sum_assignment
    tab = np.zeros((k, k), dtype=np.int64)
    np.add.at(tab, (np.asarray(truth), np.asarray(labels)), 1)
    r, c = linear_sum_assignment(-tab)
    return 2.0 * (1.0 - tab[r, c].sum() / len(truth))


def run(g, groups, h):
    ts, st = [], None
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx = lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, groups, k, True, h=h)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        ev, _, st = lib.sfairsc_eigs(ctx, k, 1e-10, want_evecs=False)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        ts.append((t1 - t0, t2 - t1))
        lab, _ = lib.sfairsc_embed_kmeans(ctx, 11)
        ctx.close()
    b = float(np.median([x[0] for x in ts]))
    e = float(np.median([x[1] for x in ts]))
    return dict(build_s=b, eigs_s=e, applies=st["applies"], restarts=st["restarts"],
                resid=st["max_resid_rel"], err=float(error_rate(g.clusters, lab, k)), evals=[float(x) for x in ev])


for n in [int(x) for x in args.ns.split(",")]:
    for h in [int(x) for x in args.hs.split(",")]:
        t0 = time.perf_counter()
        g = exp1_msbm_torch(n, h, seed=16435 + h, device="cuda")
        torch.cuda.synchronize()
        gen_s = time.perf_counter() - t0
        torch.cuda.empty_cache()
        gr = torch.from_numpy(g.groups.astype(np.int32)).to(dev)
        sc = run(g, torch.zeros_like(gr), 1)
        fair = run(g, gr, h)
        row = dict(n=n, h=h, nnz=g.nnz, mean_degree=g.nnz / n, gen_s=gen_s, sc=sc, sfairsc=fair,
                   eigs_ratio_sfairsc_over_sc=fair["eigs_s"] / sc["eigs_s"],
                   applies_ratio=fair["applies"] / sc["applies"])
        print(json.dumps(row), flush=True)
        rows.append(row)
        del g, gr
        torch.cuda.empty_cache()
os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
with open(args.out, "w") as f:
    json.dump({"what": __doc__.split("\n")[0], "k": k, "tol": 1e-10, "reps": args.reps, "rows": rows}, f, indent=1)
