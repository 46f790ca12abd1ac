"""Design experiment (not product, not oracle): the single-sweep lagged thick-restart Lanczos of
proto_lagged.py with TWO Lanczos steps per basis sweep.

Step j runs the lagged coefficient step as before (measured s_j = V_j^T v~_j), but instead of
the sweep it forms the next lagged vector from the three-term part only,
    u = y/mu - kappa v~ - g_{j-1} v_{j-1}         (one basis column read, no pass)
  = w_j + V_j g_far                                (g_far = g with entry j-1 zeroed, O(eps sigma)),
v~_{j+1} = P u / nu, and records column j of H as c - g_far (so that A v_j = V_j (c - g_far) +
alpha v_j + nu v~_{j+1} holds).  Step j+1 uses the ANALYTIC projections
    s_{j+1} = [V_j, v_j]^T v~_{j+1} ~ [g_far / nu ; 0]
(the unmeasured rest, V^T w_j / nu, is rounding-level), and ONE sweep then writes v_j and v_{j+1}
and forms w_{j+1} with the dots [V_{j+2}]^T w_{j+1} (the measured s_{j+2}).  Basis bytes per two
steps: (J + 6) vectors instead of 2 (J + 4).  The first step after a restart (its g couples every
kept Ritz vector) stays a single lagged step.

    python tests/tools/proto_pair.py [--n 3000] [--k 10] [--cfg4 N]
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from proto_lagged import lagged_trlan  # noqa: E402


def pair_trlan(A, P, n, k, m, keep, target, v0, max_restarts=10000, verbose=False):
    """Two Lanczos steps per sweep.  The odd column v'_{j+1} of a pair is finalised with the
    analytic projections; the same sweep measures its defect e = V^T v', and before the next
    coefficient step the bookkeeping moves to the orthonormal basis V'' = V' T^-1
    (T = I but column j+1 = [e; rho]): H <- T H T^-1, b~ <- T^-T b~, s <- T^-T s, and the next
    sweep rewrites column j+1 as v'' = (v' - V e) / rho (one more row combination)."""
    V = np.zeros((n, m + 1))
    H = np.zeros((m + 2, m + 1))
    vt = v0 / np.linalg.norm(v0)
    s = np.zeros(0)
    omega = vt @ vt
    j = 0
    applies = sweeps = restarts = 0
    first = 0  # first step after a (re)start: a single lagged step
    worst = 0.0
    pend = None  # (column, e, rho) of the odd column awaiting its rewrite

    def fix(jj, s):
        """Move the bookkeeping of the jj active columns (+ lagged row jj) to V'' = V' T^-1."""
        nonlocal pend
        if pend is None:
            return s
        col, e, rho = pend
        T = np.eye(jj)
        T[:col, col] = e
        T[col, col] = rho
        Ti = np.linalg.inv(T)
        H[:jj, :jj] = T @ H[:jj, :jj] @ Ti
        H[jj, :jj] = H[jj, :jj] @ Ti
        s = Ti.T @ s
        V[:, col] = (V[:, col] - V[:, :col] @ e) / rho  # (GPU: written by the next sweep)
        pend = None
        return s

    def coef(j, vt, s, omega, y):
        mu = np.sqrt(omega - s @ s)
        bt = H[j, :j].copy()
        H[:j, :j] += np.outer(s, bt)
        H[j, :j] = mu * bt
        zeta = vt @ y
        Hj = H[:j, :j]
        z = Hj.T @ s + mu * mu * bt
        c = (z - Hj @ s) / mu
        alpha = (zeta - 2 * s @ z + s @ Hj @ s) / (mu * mu)
        kappa = (alpha + bt @ s) / mu
        g = Hj @ s / mu + c - kappa * s
        H[:j, j] = c
        H[j, j] = alpha
        return mu, kappa, g

    while True:
        while j < m:
            s = fix(j, s)
            y = A(vt)
            applies += 1
            mu, kappa, g = coef(j, vt, s, omega, y)
            if j == first or j + 1 >= m:  # single lagged step: one sweep
                vj = vt / mu - V[:, :j] @ (s / mu)
                w = y / mu - kappa * vt - V[:, :j] @ g
                V[:, j] = vj
                d = V[:, :j + 1].T @ w
                sweeps += 1
                bnew = np.linalg.norm(w)
                vt, s = P(w / bnew), d / bnew
                omega = vt @ vt
                H[j + 1, :j + 1] = 0.0
                H[j + 1, j] = bnew
                j += 1
                continue
            # ---- pair: step j without a sweep ----
            gfar = g.copy()
            gfar[j - 1] = 0.0
            u = y / mu - kappa * vt - g[j - 1] * V[:, j - 1]  # elementwise + one basis column
            pu = P(u)
            nu = np.linalg.norm(pu)
            vt2 = pu / nu
            H[:j, j] -= gfar  # A v_j = V_j (c - g_far) + alpha v_j + nu v~_{j+1}
            H[j + 1, :j + 1] = 0.0
            H[j + 1, j] = nu
            s2 = np.concatenate([gfar / nu, [0.0]])  # analytic [V_j, v_j]^T v~_{j+1}
            omega2 = vt2 @ vt2
            # ---- step j+1 ----
            y2 = A(vt2)
            applies += 1
            mu2, kappa2, g2 = coef(j + 1, vt2, s2, omega2, y2)
            # ---- the pair's sweep: v_j, v'_{j+1}, w_{j+1}; dots V^T w and the defect V^T v' ----
            vj = vt / mu - V[:, :j] @ (s / mu)
            V[:, j] = vj
            vj1 = vt2 / mu2 - V[:, :j + 1] @ (s2 / mu2)
            w = y2 / mu2 - kappa2 * vt2 - V[:, :j + 1] @ g2
            V[:, j + 1] = vj1
            d = V[:, :j + 2].T @ w
            e = V[:, :j + 1].T @ vj1
            rho = np.sqrt(vj1 @ vj1 - e @ e)
            worst = max(worst, float(np.abs(e).max()))
            pend = (j + 1, e, rho)
            sweeps += 1
            bnew = np.linalg.norm(w)
            vt, s = P(w / bnew), d / bnew  # v~ kept in range(P) (R19; the GPU's k_lz_norm)
            omega = vt @ vt
            H[j + 2, :j + 2] = 0.0
            H[j + 2, j + 1] = bnew
            j += 2
        # ---- restart sync (as proto_lagged, after the pending rewrite) ----
        s = fix(m, s)
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
            info = dict(applies=applies, restarts=restarts, sweeps=sweeps, worst_defect=worst,
                        basis_orth=float(np.abs(V[:, :m].T @ V[:, :m] - np.eye(m)).max()))
            return th[:k], V[:, :m] @ Y[:, :k], info
        vm = (vt - V[:, :m] @ s) / mu
        Vn = np.zeros_like(V)
        Vn[:, :keep] = V[:, :m] @ Y[:, :keep]
        V = Vn
        vt = vm
        s = np.zeros(keep)
        omega = vt @ vt
        H = np.zeros_like(H)
        H[np.arange(keep), np.arange(keep)] = th[:keep]
        H[keep, :keep] = b @ Y[:, :keep]
        j = first = keep
        restarts += 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=3000)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--cfg4", type=int, default=0, help="reduced config-4 graph of this n instead")
    args = ap.parse_args()
    from oracle import sfairsc_cpu
    from synth import baseline_config, random_graph
    if args.cfg4:
        g, cfg = baseline_config(4, n=args.cfg4)
        k, norm = 50, True
        m, keep = 170, 80
    else:
        g = random_graph(args.n, 4, p=10 / args.n, seed=1, weights="uniform")
        k, norm = args.k, True
        m = max(2 * k + 10, 3 * k, 20)
        keep = k + (m - k) // 4
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, norm)
    v0 = op.P(np.random.default_rng(0).standard_normal(g.n))
    for name, fn in (("lagged", lambda: lagged_trlan(op.apply, g.n, k, m, keep, 1e-10 * op.sigma, v0)),
                     ("pair", lambda: pair_trlan(op.apply, op.P, g.n, k, m, keep, 1e-10 * op.sigma, v0))):
        th, X, info = fn()
        R = np.stack([op.apply(X[:, i]) for i in range(k)], axis=1) - X * th
        print(f"{name:7s} {info} resid {np.linalg.norm(R, axis=0).max() / op.sigma:.2e} "
              f"orth {np.abs(X.T @ X - np.eye(k)).max():.2e} CtX {np.linalg.norm(op.C.T @ X):.1e}", flush=True)
        if not args.cfg4:
            from oracle import fairsc
            ref = fairsc.fairsc_dense(g.dense(), g.groups, g.h, k, norm)
            print(f"        max |d lambda| {np.abs(th - ref.evals[:k]).max():.2e}")


if __name__ == "__main__":
    main()
