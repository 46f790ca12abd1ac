"""Exploration: column-block size of the config-5 SpMV (SFAIRSC_COLBLK_MB, the test hook of abi.cu):
per-SpMV time over 10 back-to-back t = L x.  Not a bench value."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2210_16435_b200 import lib  # noqa: E402
from synth.dcsbm import config5  # noqa: E402

g, cfg = config5(device="cuda")
torch.cuda.synchronize()
torch.cuda.empty_cache()
x = torch.randn(g.n, dtype=torch.float64, device="cuda")
for mb in sys.argv[1].split(","):
    os.environ["SFAIRSC_COLBLK_MB"] = mb
    ctx = lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, g.groups, cfg["k_eig"], False, h=g.h, max_basis=40)
    y = torch.empty_like(x)
    for _ in range(2):
        lib.sfairsc_laplacian(ctx, x, y)
    lib.profile_enable(ctx, True)
    lib.profile_reset(ctx)
    for _ in range(10):
        lib.sfairsc_laplacian(ctx, x, y)
    pr = lib.profile_read(ctx)["spmv"]
    print(json.dumps({"colblk_mb": float(mb), "us_per_spmv": pr["ms"] / pr["launches"] * 1e3}), flush=True)
    ctx.close()
    torch.cuda.empty_cache()
