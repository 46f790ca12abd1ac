"""Design experiment (not product, not oracle): single-sweep thick-restart
Lanczos with lagged (one-step-delayed) full reorthogonalisation — the
algorithm of csrc/lanczos1.cu written out in numpy, checked against eigh.

Per step only ONE pass over the basis: the update pass forms the corrected
previous vector v_j = (v~_j - V s)/mu and the new residual w, and in the same
pass the dots V^T w that become the next step's correction s.

    python scripts/proto_lagged.py [--n 2000] [--k 10]
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def lagged_trlan(A, n, k, m, keep, target, v0, max_restarts=10000, verbose=False):
    V = np.zeros((n, m + 1))  # corrected basis columns
    H = np.zeros((m + 2, m + 1))  # A V_j = V_j H[:j,:j] + (lagged) v~_j H[j,:j]
    vt = v0 / np.linalg.norm(v0)  # v~_j
    s = np.zeros(0)  # V_j^T v~_j
    omega = vt @ vt
    j = 0
    applies = 0
    restarts = 0
    while True:
        while j < m:
            # ---- coefficient step (device: 1 CTA) ----
            mu = np.sqrt(omega - s @ s)
            bt = H[j, :j].copy()  # b~ (lagged coupling row)
            H[:j, :j] += np.outer(s, bt)  # correction of the previous columns
            H[j, :j] = mu * bt  # b
            # ---- SpMV ----
            y = A(vt)
            applies += 1
            zeta = vt @ y
            Hj = H[:j, :j]
            z = Hj.T @ s + mu * mu * bt
            c = (z - Hj @ s) / mu
            alpha = (zeta - 2 * s @ z + s @ Hj @ s) / (mu * mu)
            kappa = (alpha + bt @ s) / mu
            g = Hj @ s / mu + c - kappa * s
            # ---- update + dots pass ----
            vj = vt / mu - V[:, :j] @ (s / mu)
            w = y / mu - kappa * vt - V[:, :j] @ g
            V[:, j] = vj
            d = V[:, :j + 1].T @ w
            H[:j, j] = c
            H[j, j] = alpha
            # ---- normalize ----
            bnew = np.linalg.norm(w)
            vt = w / bnew
            s = d / bnew
            omega = vt @ vt
            H[j + 1, :j + 1] = 0.0
            H[j + 1, j] = bnew
            j += 1
        # ---- restart sync: correct column m-1 with the lagged s ----
        mu = np.sqrt(omega - s @ s)
        bt = H[m, :m].copy()
        Hm = H[:m, :m] + np.outer(s, bt)
        b = mu * bt
        T = 0.5 * (Hm + Hm.T)
        th, Y = np.linalg.eigh(T)
        est = np.abs(b @ Y)
        maxres = est[:k].max()
        if verbose:
            print(f"  restart {restarts} applies {applies} maxres {maxres:.2e} th_k {th[k-1]:.10f}", flush=True)
        if maxres <= target or restarts >= max_restarts:
            return th[:k], V[:, :m] @ Y[:, :k], dict(applies=applies, restarts=restarts)
        vm = (vt - V[:, :m] @ s) / mu
        Vn = np.zeros_like(V)
        Vn[:, :keep] = V[:, :m] @ Y[:, :keep]
        V = Vn
        vt = vm
        s = np.zeros(keep)
        omega = vt @ vt
        H = np.zeros_like(H)
        H[np.arange(keep), np.arange(keep)] = th[:keep]
        H[keep, :keep] = b @ Y[:, :keep]  # b~ with s = 0, mu = 1
        j = keep
        restarts += 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2000)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--cfg4", type=int, default=0, help="reduced config-4 graph of this n instead")
    args = ap.parse_args()
    from oracle import sfairsc_cpu
    from synth import baseline_config, random_graph
    if args.cfg4:
        g, cfg = baseline_config(4, n=args.cfg4)
        k, norm = 50, True
        m, keep = 150, 110
    else:
        g = random_graph(args.n, 4, p=10 / args.n, seed=1, weights="uniform")
        k, norm = args.k, True
        m, keep = max(2 * k + 10, 3 * k, 20), None
        keep = k + 3 * (m - k) // 5
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, norm)
    rng = np.random.default_rng(0)
    v0 = op.P(rng.standard_normal(g.n))
    th, X, info = lagged_trlan(op.apply, g.n, k, m, keep, 1e-10 * op.sigma, v0, verbose=bool(args.cfg4))
    R = np.stack([op.apply(X[:, i]) for i in range(k)], axis=1) - X * th
    print(f"applies {info['applies']} restarts {info['restarts']} resid {np.linalg.norm(R, axis=0).max()/op.sigma:.2e} "
          f"orth {np.abs(X.T @ X - np.eye(k)).max():.2e}")
    if not args.cfg4:
        from oracle import fairsc
        ref = fairsc.fairsc_dense(g.dense(), g.groups, g.h, k, norm)
        print(f"max |d lambda| {np.abs(th - ref.evals[:k]).max():.2e}")


if __name__ == "__main__":
    main()
