"""Probe: a few thick-restart cycles of the config-4 eigensolve with per-kernel
event timing (exploration / ncu target; not a bench value).

    python scripts/probe_cfg4.py [--n N] [--restarts R] [--applies A]
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
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--restarts", type=int, default=2)
ap.add_argument("--applies", type=int, default=20)
ap.add_argument("--vs", type=int, default=0)
ap.add_argument("--bsz", type=int, default=1)
ap.add_argument("--m", type=int, default=0)
ap.add_argument("--keep", type=int, default=0)
ap.add_argument("--skip-apply", action="store_true")
ap.add_argument("--reorth", type=int, default=0)
ap.add_argument("--vparts", type=int, default=0)
args = ap.parse_args()

t = time.time()
g, cfg = baseline_config(args.config, n=args.n)
print(f"generated n={g.n} nnz={g.nnz} in {time.time() - t:.1f}s", file=sys.stderr)
dev = torch.device("cuda:0")
rp, ci, vv = (torch.from_numpy(a).to(dev) for a in (g.row_ptr, g.col, g.val))
gr = torch.from_numpy(g.groups.astype(np.int32)).to(dev)
torch.cuda.synchronize()
torch.cuda.empty_cache()  # generator intermediates (config 5 is generated on the GPU) back before the build
k = cfg["k_eig"]
ctx = lib.sfairsc_build_operator(rp, ci, vv, gr, k, cfg["normalized"], h=g.h, max_restarts=args.restarts,
                                 spmv_vector=args.vs, block_size=args.bsz, max_basis=args.m, keep=args.keep,
                                 reorth=args.reorth, virtual_parts=args.vparts)
out = {"n": g.n, "nnz": g.nnz, "info": ctx.info(), "bsz": args.bsz, "reorth": args.reorth}
# apply-only
x = torch.randn((4, g.n), dtype=torch.float64, device=dev)
y = torch.empty_like(x)
lib.sfairsc_apply(ctx, x, y)
lib.profile_enable(ctx, True)
for _ in range(max(1, args.applies // 4)):
    lib.sfairsc_apply(ctx, x, y)
prof = lib.profile_read(ctx)
out["apply"] = {kk: {"us": 1e3 * v["ms"] / v["launches"], "GBps": v["alg_bytes"] / (v["ms"] * 1e6)}
                for kk, v in prof.items() if v["launches"]}
lib.profile_reset(ctx)
t = time.time()
try:
    ev, X, st = lib.sfairsc_eigs(ctx, k, cfg["tol"], want_evecs=False)
except lib.SfairscError as e:
    st = ctx.last_stats
    out["status"] = e.name
torch.cuda.synchronize()
out["wall_s"] = time.time() - t
prof = lib.profile_read(ctx)
out["stats"] = st
out["eigs"] = {kk: {"ms": v["ms"], "launches": v["launches"], "us": 1e3 * v["ms"] / v["launches"],
                    "GBps": v["alg_bytes"] / (v["ms"] * 1e6)} for kk, v in prof.items() if v["launches"]}
print(json.dumps(out, indent=1))
