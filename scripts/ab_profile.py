"""Exploration: one warm-up config-4 solve, then one full solve with per-kernel CUDA-event profiling; prints
the solve's wall time and per-kind kernel means (the A/B scripts' kernel-level view).  Not a bench value."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_16435_b200 import lib  # noqa: E402
from synth import baseline_config  # noqa: E402

dev = torch.device("cuda:0")
g, cfg = baseline_config(4)
t = lambda a: torch.from_numpy(a).to(dev)
rp, ci, vv, gr = t(g.row_ptr), t(g.col), t(g.val), t(g.groups.astype(np.int32))
k = cfg["k_eig"]
for prof in (False, True):
    ctx = lib.sfairsc_build_operator(rp, ci, vv, gr, k, True, h=g.h)
    if prof:
        lib.profile_enable(ctx, True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev, _, st = lib.sfairsc_eigs(ctx, k, cfg["tol"], want_evecs=False)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if prof:
        p = lib.profile_read(ctx)
        print(json.dumps({"wall_s": round(wall, 3), "applies": st["applies"],
                          "us": {kk: round(v["ms"] * 1e3 / max(1, v["launches"]), 1) for kk, v in p.items()},
                          "ms": {kk: round(v["ms"], 1) for kk, v in p.items()}}), flush=True)
    ctx.close()
