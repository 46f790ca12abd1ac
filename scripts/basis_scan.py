"""Exploration: (basis m, kept Ritz vectors) scan of the default (paired) solver at config 4:
device-synchronised eigensolve time and applies.  Not a bench value.

    python scripts/basis_scan.py "170,80;186,90;..."
"""
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
for spec in sys.argv[1].split(";"):
    m, keep = (int(x) for x in spec.split(","))
    ctx = lib.sfairsc_build_operator(rp, ci, vv, gr, cfg["k_eig"], True, h=g.h, max_basis=m, keep=keep)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev, _, st = lib.sfairsc_eigs(ctx, cfg["k_eig"], cfg["tol"], want_evecs=False)
    torch.cuda.synchronize()
    print(json.dumps({"m": m, "keep": keep, "eigs_s": round(time.perf_counter() - t0, 3), "applies": st["applies"],
                      "restarts": st["restarts"], "resid": st["max_resid_rel"]}), flush=True)
    ctx.close()
