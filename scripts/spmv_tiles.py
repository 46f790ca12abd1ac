"""Exploration (ran while the tile shape was read from SFAIRSC_SPMV_TILE; the shape is now fixed
at 2048 entries / 128 rows / 2 stages in abi.cu, so re-running needs that hook back): tile shape (entries, rows, ring depth) and lane width VS of the TMA SpMV at
config 4 (and 3).  200 back-to-back t = L x per variant, per-launch CUDA events; outputs
compared with the first variant (same rows, same per-lane order => equal to rounding order)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_16435_b200 import lib  # noqa: E402
from synth import baseline_config  # noqa: E402

dev = torch.device("cuda:0")
cfgs = [int(a) for a in sys.argv[1:]] or [4]
shapes = os.environ.get("TILES", "1024,64,2;2048,64,2;2048,128,2;2048,64,3;4096,128,2").split(";")
vss = [int(v) for v in os.environ.get("VSS", "4,2,8").split(",")]
for c in cfgs:
    g, cfg = baseline_config(c)
    t = lambda a: torch.from_numpy(a).to(dev)
    rp, ci, vv, gr = t(g.row_ptr), t(g.col), t(g.val), t(g.groups.astype(np.int32))
    x = torch.randn(g.n, dtype=torch.float64, device=dev)
    ref = None
    for sh in shapes:
        for vs in vss:
            os.environ["SFAIRSC_SPMV_TILE"] = sh
            ctx = lib.sfairsc_build_operator(rp, ci, vv, gr, cfg["k_eig"], cfg["normalized"], h=g.h, spmv_vector=vs)
            y = torch.empty_like(x)
            for _ in range(10):
                lib.sfairsc_laplacian(ctx, x, y)
            lib.profile_enable(ctx, True)
            lib.profile_reset(ctx)
            for _ in range(200):
                lib.sfairsc_laplacian(ctx, x, y)
            pr = lib.profile_read(ctx)["spmv"]
            lib.profile_enable(ctx, False)
            if ref is None:
                ref = y.clone()
            d = ((y - ref).abs().max() / ref.abs().max()).item()
            us = pr["ms"] / pr["launches"] * 1e3
            print(json.dumps({"config": c, "tile": sh, "vs": vs, "us_per_spmv": round(us, 1), "rel_diff": d}), flush=True)
            ctx.close()
