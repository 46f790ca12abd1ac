"""Config 5 (n = 5e7, 1.6e9 entries, column-blocked pattern-only SpMV): the TMA-fed column-block kernel
vs the LSU kernel (SFAIRSC_SPMV_TMA=0): per-SpMV time over 20 back-to-back t = L x (library events) and
the relative difference of the outputs.  Exploration, not a bench value.  Optional --n for reduced sizes."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2210_16435_b200 import lib  # noqa: E402
from synth.dcsbm import config5  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
g, cfg = config5(n=a.n, device="cuda")
torch.cuda.synchronize()
torch.cuda.empty_cache()
x = torch.randn(g.n, dtype=torch.float64, device="cuda")
outs = {}
for variant in ("tma", "lsu"):
    os.environ["SFAIRSC_SPMV_TMA"] = "0" if variant == "lsu" else "1"
    ctx = lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, g.groups, cfg["k_eig"], False, h=g.h, max_basis=40)
    y = torch.empty_like(x)
    for _ in range(3):
        lib.sfairsc_laplacian(ctx, x, y)
    lib.profile_enable(ctx, True)
    lib.profile_reset(ctx)
    for _ in range(a.reps):
        lib.sfairsc_laplacian(ctx, x, y)
    pr = lib.profile_read(ctx)["spmv"]
    outs[variant] = y.clone()
    print(json.dumps({"variant": variant, "n": g.n, "nnz": g.nnz, "us_per_spmv": pr["ms"] / pr["launches"] * 1e3,
                      "launches": pr["launches"]}), flush=True)
    ctx.close()
    torch.cuda.empty_cache()
d = ((outs["tma"] - outs["lsu"]).abs().max() / outs["lsu"].abs().max()).item()
print(json.dumps({"max_rel_diff_tma_vs_lsu": d}), flush=True)
