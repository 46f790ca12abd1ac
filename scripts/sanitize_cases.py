"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck):
every solver variant (single-sweep default, CGS2, block 2), the unit-weight pattern
path, the column-blocked path, the dense projector, the pair apply and k-means, on
BASELINE configs 1-2 sizes or smaller.  Exit code 0 iff every case returned OK.

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py [case ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_16435_b200 import lib  # noqa: E402
from synth import baseline_config, random_graph  # noqa: E402

dev = torch.device("cuda:0")


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def solve(g, k, normalized, **kw):
    ctx = lib.sfairsc_build_operator(t(g.row_ptr), t(g.col), t(g.val), t(g.groups.astype(np.int32)), k, normalized,
                                     h=g.h, **kw)
    X = torch.empty((k, g.n), dtype=torch.float64, device=dev)
    ev, _, st = lib.sfairsc_eigs(ctx, k, 1e-10, evecs=X)
    return ctx, ev, st


def case_cfg1_default():
    g, cfg = baseline_config(1)
    ctx, ev, st = solve(g, 5, False)
    lib.sfairsc_embed_kmeans(ctx, 7)
    x = torch.randn(3, g.n, dtype=torch.float64, device=dev)
    lib.sfairsc_apply(ctx, x)         # pair apply + a single tail
    lib.sfairsc_apply_single(ctx, x)  # metric-1 path
    lib.sfairsc_project(ctx, x)
    ctx.close()


def case_cfg1_cgs2():
    g, _ = baseline_config(1)
    solve(g, 5, False, reorth=1)[0].close()


def case_cfg1_block2():
    g, _ = baseline_config(1)
    solve(g, 5, False, block_size=2)[0].close()


def case_cfg2_default():
    g, cfg = baseline_config(2)
    ctx, ev, st = solve(g, 10, True)
    lib.sfairsc_embed_kmeans(ctx, 3)
    ctx.close()


def case_colblk_unit():
    os.environ["SFAIRSC_COLBLK_MB"] = "0.003"
    try:
        g = random_graph(1500, 3, p=0.01, seed=5, weights="unit")
        solve(g, 6, False)[0].close()
        solve(g, 6, True)[0].close()
    finally:
        del os.environ["SFAIRSC_COLBLK_MB"]


def case_dense_F():
    g = random_graph(1200, 3, p=0.01, seed=4, weights="uniform")
    F = np.random.default_rng(1).standard_normal((g.n, 3))
    ctx = lib.sfairsc_build_operator_dense(t(g.row_ptr), t(g.col), t(g.val), torch.from_numpy(F.T.copy()).to(dev), 6,
                                           True)
    X = torch.empty((6, g.n), dtype=torch.float64, device=dev)
    lib.sfairsc_eigs(ctx, 6, 1e-10, evecs=X)
    ctx.close()


def case_virtual_parts():
    g = random_graph(2000, 4, p=0.008, seed=6, weights="uniform")
    solve(g, 6, True, virtual_parts=3)[0].close()


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        CASES[nm]()
        torch.cuda.synchronize()
        print("case ok:", nm, flush=True)
