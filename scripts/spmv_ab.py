"""A/B of the single-vector SpMV kernels (A5) at BASELINE sizes on one GPU:
the TMA-fed tile kernel (spmv_tma.cu, default) vs the round-1 LSU kernel
(SFAIRSC_SPMV_TMA=0), and the TMA kernel streaming the values of a unit-weight graph
(SFAIRSC_UNIT=0) vs its pattern-only form.  200 back-to-back t = L x launches per variant, timed by the
library's per-launch CUDA events; algorithmic bytes per DESIGN.md §6."""
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
rows = []
for c in cfgs:
    g, cfg = baseline_config(c)
    t = lambda a: torch.from_numpy(a).to(dev)
    rp, ci, vv, gr = t(g.row_ptr), t(g.col), t(g.val), t(g.groups.astype(np.int32))
    x = torch.randn(g.n, dtype=torch.float64, device=dev)
    outs = {}
    for variant in ("tma", "tma_vals", "tma_vs16", "tma_vs4", "lsu"):
        os.environ["SFAIRSC_SPMV_TMA"] = "0" if variant == "lsu" else "1"
        os.environ["SFAIRSC_UNIT"] = "0" if variant == "tma_vals" else "1"  # tma_vals: stream the values
        kw = {"spmv_vector": int(variant.split("vs")[1])} if "vs" in variant else {}
        ctx = lib.sfairsc_build_operator(rp, ci, vv, gr, cfg["k_eig"], cfg["normalized"], h=g.h, **kw)
        y = torch.empty_like(x)
        for _ in range(10):
            lib.sfairsc_laplacian(ctx, x, y)
        lib.profile_enable(ctx, True)
        lib.profile_reset(ctx)
        for _ in range(200):
            lib.sfairsc_laplacian(ctx, x, y)
        pr = lib.profile_read(ctx)["spmv"]
        lib.profile_enable(ctx, False)
        outs[variant] = y.clone()
        us = pr["ms"] / pr["launches"] * 1e3
        row = {"config": c, "variant": variant, "n": g.n, "nnz": g.nnz, "us_per_spmv": us,
               "alg_GBps": pr["alg_bytes"] / pr["launches"] / (us * 1e-6) / 1e9,
               "unit_weights": ctx.info()["unit_weights"]}
        print(json.dumps(row), flush=True)
        rows.append(row)
        ctx.close()
    d = max((outs[v] - outs["lsu"]).abs().max().item() for v in outs) / max(1e-300, outs["lsu"].abs().max().item())
    print(json.dumps({"config": c, "max_rel_diff_tma_vs_lsu": d}), flush=True)
    assert d < 1e-13, d
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/spmv_ab.json", "w") as f:
    json.dump(rows, f, indent=1)
