"""A/B of the single-sweep solver at config 4 (and others): one Lanczos step per basis sweep
(reorth 2) vs two (reorth 3, paired, the default).  Device-synchronised wall time of
sfairsc_eigs, applies, residual, eigenvalue agreement.  Exploration, not a bench value.

    python scripts/pair_ab.py [config ...]
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
for c in [int(a) for a in sys.argv[1:]] or [4]:
    g, cfg = baseline_config(c)
    t = lambda a: torch.from_numpy(a).to(dev)
    rp, ci, vv, gr = t(g.row_ptr), t(g.col), t(g.val), t(g.groups.astype(np.int32))
    k = cfg["k_eig"]
    res = {}
    for reorth in (2, 3, 2, 3):
        ctx = lib.sfairsc_build_operator(rp, ci, vv, gr, k, cfg["normalized"], h=g.h, reorth=reorth)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev, _, st = lib.sfairsc_eigs(ctx, k, cfg["tol"], want_evecs=False)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ctx.close()
        res.setdefault(reorth, []).append(dict(wall_s=wall, applies=st["applies"], restarts=st["restarts"],
                                               resid=st["max_resid_rel"], evals=np.asarray(ev)))
        print(json.dumps({"config": c, "reorth": reorth, "wall_s": round(wall, 3), "applies": st["applies"],
                          "restarts": st["restarts"], "resid": st["max_resid_rel"]}), flush=True)
    d = np.abs(res[3][0]["evals"] - res[2][0]["evals"]).max()
    print(json.dumps({"config": c, "max_abs_dlambda_pair_vs_single": float(d)}), flush=True)
