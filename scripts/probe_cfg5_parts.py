"""Config 5 (n = 5e7, 1.6e9 entries) with the row-partitioned solver on one GPU (`virtual_parts` P:
P row blocks, the arithmetic of P GPUs run serially) vs P = 1: per-kernel event times of one restart
cycle, for DESIGN.md §9's multi-GPU model.  The graph is generated on the GPU and the torch copy freed
before the build; basis 100 so that P = 8 fits one GPU.  Exploration, not a bench value.

    python scripts/probe_cfg5_parts.py --parts 8
"""
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
ap.add_argument("--parts", type=int, default=8)
ap.add_argument("--m", type=int, default=100)
ap.add_argument("--restarts", type=int, default=1)
a = ap.parse_args()
g, cfg = config5(device="cuda")
torch.cuda.synchronize()
torch.cuda.empty_cache()
k = cfg["k_eig"]
kw = {"virtual_parts": a.parts} if a.parts > 1 else {}
t0 = time.time()
ctx = lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, g.groups, k, False, h=g.h, max_basis=a.m,
                                 max_restarts=a.restarts, **kw)
torch.cuda.synchronize()
out = {"parts": a.parts, "m": a.m, "n": g.n, "nnz": g.nnz, "build_s": time.time() - t0, "info": ctx.info()}
del g
torch.cuda.empty_cache()
lib.profile_enable(ctx, True)
t0 = time.time()
try:
    lib.sfairsc_eigs(ctx, k, cfg["tol"], want_evecs=False)
    out["status"] = "OK"
except lib.SfairscError as e:
    out["status"] = e.name  # the restart budget ends the solve: the work done is what is timed
torch.cuda.synchronize()
out["wall_s"] = time.time() - t0
out["stats"] = ctx.last_stats
prof = lib.profile_read(ctx)
out["kernels"] = {kk: {"ms": v["ms"], "launches": v["launches"], "us": 1e3 * v["ms"] / max(1, v["launches"])}
                  for kk, v in prof.items() if v["launches"]}
ctx.close()
print(json.dumps(out, indent=1))
