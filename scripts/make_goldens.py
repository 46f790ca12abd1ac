"""Write the oracle goldens under tests/golden/ — calls only `oracle/` and `synth/`
(never the CUDA path), so every stored value is the oracle's.

    python scripts/make_goldens.py --config 2   # Tier D (Alg. 2) on BASELINE config 2
    python scripts/make_goldens.py --config 3   # Tier S (Alg. 3 + ARPACK) on config 3
    python scripts/make_goldens.py --config 4   # Tier S on config 4 (about an hour on 8 cores)

Outputs:
  cfg2_tier_d.json (+ cfg2_tier_d_X.npz: the k fair eigenvectors in the orthonormal
  X frame of reading R9, for the subspace angle), cfg3_tier_s.json, cfg4_tier_s.json.
  Each JSON records lambda_1..lambda_{k+1}, gap_k, sigma, the oracle's own residuals
  ||L^sigma x_i - lambda_i x_i|| / sigma through the paper's apply, the
  generator's graph fingerprint (n, nnz, sum of weights, checksum of the column
  indices) and the wall time.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

import numpy as np  # noqa: E402

from oracle import fairsc, sfairsc_cpu  # noqa: E402
from synth import baseline_config  # noqa: E402


def fingerprint(g) -> dict:
    ci = g.col.astype(np.int64)
    return {"n": int(g.n), "nnz": int(g.nnz), "sum_w": float(np.sum(g.val)),
            "col_checksum": int((ci * (np.arange(len(ci), dtype=np.int64) % 1000003 + 1)).sum() % (1 << 61)),
            "groups_checksum": int((g.groups.astype(np.int64) * (np.arange(g.n) % 997 + 1)).sum())}


def tier_d(c: int) -> None:
    g, cfg = baseline_config(c)
    k = cfg["k_eig"]
    t0 = time.time()
    res = fairsc.fairsc_dense(g.dense(), g.groups, g.h, k, cfg["normalized"], extra=1)
    wall = time.time() - t0
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, cfg["normalized"], threads=0)
    resid = [float(np.linalg.norm(op.apply(res.X[:, i]) - res.evals[i] * res.X[:, i]) / op.sigma) for i in range(k)]
    out = {"source": "scripts/make_goldens.py --config %d: oracle.fairsc.fairsc_dense (Tier D, Alg. 2 P:465-490)" % c,
           "config": c, "k": k, "normalized": cfg["normalized"], "evals": [float(x) for x in res.evals[:k + 1]],
           "gap_k": float(res.evals[k] - res.evals[k - 1]), "sigma": op.sigma,
           "resid_rel_via_P803": resid, "graph": fingerprint(g), "wall_s": wall}
    with open(os.path.join(GOLDEN, f"cfg{c}_tier_d.json"), "w") as f:
        json.dump(out, f, indent=1)
    np.savez_compressed(os.path.join(GOLDEN, f"cfg{c}_tier_d_X.npz"), X=res.X[:, :k])
    print(json.dumps({k_: v for k_, v in out.items() if k_ != "resid_rel_via_P803"}))


def tier_s(c: int, ncv: int | None, seed: int, tol: float = 1e-12) -> None:
    g, cfg = baseline_config(c)
    k = cfg["k_eig"]
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, cfg["normalized"], threads=0)
    t0 = time.time()
    _apply, cnt = op.apply, [0]

    def progress_apply(w):  # the oracle's apply, unchanged; a progress line every 500 matvecs
        cnt[0] += 1
        if cnt[0] % 500 == 0:
            print(f"  {cnt[0]} matvecs, {time.time() - t0:.0f} s", file=sys.stderr, flush=True)
        return _apply(w)

    op.apply = progress_apply
    res = sfairsc_cpu.sfairsc_arpack(op, k, tol=tol, ncv=ncv, seed=seed, extra=1)
    wall = time.time() - t0
    op.apply = _apply
    resid = [float(np.linalg.norm(op.apply(res.X[:, i]) - res.evals[i] * res.X[:, i]) / op.sigma) for i in range(k)]
    out = {"source": "scripts/make_goldens.py --config %d: oracle.sfairsc_cpu.sfairsc_arpack (Tier S: Alg. 3 apply "
                     "P:803 with the normal-equations projector P:807-818, ARPACK eigsh, tol %g)" % (c, tol),
           "config": c, "k": k, "normalized": cfg["normalized"], "evals": [float(x) for x in res.evals[:k + 1]],
           "gap_k": float(res.evals[k] - res.evals[k - 1]), "sigma": op.sigma, "matvecs": res.matvecs,
           "ncv": ncv, "seed": seed, "tol": tol, "resid_rel_via_P803": resid, "graph": fingerprint(g), "wall_s": wall,
           "threads": op.threads}
    with open(os.path.join(GOLDEN, f"cfg{c}_tier_s.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k_: v for k_, v in out.items() if k_ != "resid_rel_via_P803"}))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--ncv", type=int, default=None)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--tol", type=float, default=1e-12)
    a = ap.parse_args()
    if a.config in (1, 2):
        tier_d(a.config)
    else:
        tier_s(a.config, a.ncv, a.seed, a.tol)
