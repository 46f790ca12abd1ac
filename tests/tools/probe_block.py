"""Probe: block thick-restart Lanczos (block_size 1/2/4) against the dense
FairSC oracle on small cases (exploration; the parity tests are in tests/)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from oracle import fairsc  # noqa: E402
from oracle.metrics import subspace_sin  # noqa: E402
from paper_2210_16435_b200 import lib  # noqa: E402
from synth import baseline_config, planted_cliques, random_graph  # noqa: E402

cases = []
g, cfg = baseline_config(1)
cases.append(("cfg1", g, cfg["k_eig"], cfg["normalized"]))
cases.append(("rand400n", random_graph(400, 3, p=0.02, seed=3, weights="uniform"), 8, True))
cases.append(("planted", planted_cliques(4, 6, 3, seed=7), 4, True))
for name, g, k, norm in cases:
    dense = fairsc.fairsc_dense(g.dense(), g.groups, g.h, k, norm)
    for bsz, ro in ((1, 1), (1, 2), (2, 0)):
        try:
            ctx = lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, g.groups.astype(np.int32), k, norm, h=g.h,
                                             block_size=bsz, reorth=ro)
            ev, Xt, st = lib.sfairsc_eigs(ctx, k, 1e-10)
            info = ctx.info()
            ctx.close()
            err = np.abs(ev - dense.evals[:k]).max()
            sin = subspace_sin(Xt.T, dense.X) if dense.gap > 1e-8 else float("nan")
            print(f"{name:9s} b={bsz} ro={ro} n={g.n} err={err:.2e} sin={sin:.2e} resid={st['max_resid_rel']:.2e} "
                  f"steps={st['steps']} applies={st['applies']} restarts={st['restarts']} bd={st['breakdowns']} "
                  f"m={st['basis_size']} keep={st['kept']} conv={st['converged']}", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"{name:9s} b={bsz} ro={ro} FAILED: {e}", flush=True)
