"""Profiling target: a few t = L x launches of each SpMV kernel at a BASELINE config
(default 4), for `ncu -k regex:k_spmv_tma|k_spmm`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_16435_b200 import lib  # noqa: E402
from synth import baseline_config  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["tma", "lsu"]
dev = torch.device("cuda:0")
g, cfg = baseline_config(c)
t = lambda a: torch.from_numpy(a).to(dev)
rp, ci, vv, gr = t(g.row_ptr), t(g.col), t(g.val), t(g.groups.astype(np.int32))
x = torch.randn(g.n, dtype=torch.float64, device=dev)
for v in variants:
    os.environ["SFAIRSC_SPMV_TMA"] = "1" if v == "tma" else "0"
    ctx = lib.sfairsc_build_operator(rp, ci, vv, gr, cfg["k_eig"], cfg["normalized"], h=g.h)
    y = torch.empty_like(x)
    for _ in range(3):
        lib.sfairsc_laplacian(ctx, x, y)
    torch.cuda.synchronize()
    ctx.close()
print("ok")
