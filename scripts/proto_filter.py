"""Design experiment (not product, not oracle): Chebyshev-filtered thick-restart
Lanczos vs plain thick-restart Lanczos on a reduced config-4 graph.

Counts operator applies and outer Lanczos steps (each outer step = one set of
CGS2 sweeps over the basis) so the filter degree can be chosen before writing
kernels.  The trivial eigenpair (0, D^{1/2}1) is deflated Hotelling-style
(x -> x - u1 u1^T x inside the operator) so the filter's dynamic range is set
by the non-trivial wanted eigenvalues.

    python scripts/proto_filter.py --n 200000 --deg 1 5 10 20
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def make_op(g, normalized):
    W = g.to_scipy().tocsr()
    n = W.shape[0]
    d = np.asarray(W.sum(axis=1)).ravel()
    s = 1.0 / np.sqrt(d) if normalized else np.ones(n)
    Wh = sp.diags(s) @ W @ sp.diags(s) if normalized else W
    Wh = sp.csr_matrix(Wh)
    diag = np.ones(n) if normalized else d
    grp = g.groups
    h = g.h
    beta = np.bincount(grp, weights=s * s, minlength=h)
    cnt = np.bincount(grp, minlength=h).astype(float)
    isb = 1 / np.sqrt(beta)
    u = cnt * isb
    u /= np.linalg.norm(u)
    u1 = np.sqrt(d) if normalized else np.ones(n)
    u1 = u1 / np.linalg.norm(u1)

    def P(x):  # factored fairness projector (+ deflation of u1)
        bs = np.bincount(grp, weights=s * x, minlength=h)
        c = bs * isb
        gam = (c - u * (u @ c)) * isb
        return x - s * gam[grp]

    sigma = float(np.max(np.abs(diag) + np.asarray(abs(Wh).sum(axis=0)).ravel()))

    def apply(x, deflate):
        p = P(x)
        if deflate:
            p = p - u1 * (u1 @ p)
        t = diag * p - Wh @ p
        y = P(t)
        if deflate:
            y = y - u1 * (u1 @ y)
        return y - sigma * p + sigma * x

    return apply, P, sigma, u1, n


def trlan_op(Op, n, nwant, m, keep, v0, largest, check, verbose=False, max_outer=60000):
    """Thick-restart Lanczos (full CGS2) on the symmetric operator Op; wanted:
    the nwant largest (largest=True) or smallest Ritz pairs.  check(theta, X,
    est) -> (done, info) decides convergence.  Returns (theta, X, outer)."""
    V = np.zeros((n, m + 1))
    V[:, 0] = v0 / np.linalg.norm(v0)
    T = np.zeros((m + 1, m + 1))
    j = 0
    outer = 0
    cyc = 0
    while True:
        while j < m:
            w = Op(V[:, j])
            outer += 1
            cc = np.zeros(j + 1)
            for _ in range(2):
                c_ = V[:, :j + 1].T @ w
                w -= V[:, :j + 1] @ c_
                cc += c_
            b = np.linalg.norm(w)
            T[:j + 1, j] = cc
            T[j + 1, j] = b
            V[:, j + 1] = w / b
            j += 1
        Ts = np.triu(T[:m, :m])
        Ts = Ts + np.triu(Ts, 1).T
        th, Y = np.linalg.eigh(Ts)
        order = np.argsort(-th) if largest else np.arange(m)
        th, Y = th[order], Y[:, order]
        est = np.abs(T[m, m - 1] * Y[m - 1, :nwant])
        X = V[:, :m] @ Y[:, :nwant]
        done, info = check(th[:nwant], X, est)
        if verbose:
            print(f"  cycle {cyc} outer {outer} {info}", flush=True)
        if done or outer > max_outer:
            return th, X, outer
        Vn = np.zeros_like(V)
        Vn[:, :keep] = V[:, :m] @ Y[:, :keep]
        Vn[:, keep] = V[:, m]
        Tn = np.zeros_like(T)
        Tn[np.arange(keep), np.arange(keep)] = th[:keep]
        Tn[keep, :keep] = T[m, m - 1] * Y[m - 1, :keep]
        Tn[:keep, keep] = Tn[keep, :keep]
        V, T, j = Vn, Tn, keep
        cyc += 1


def trlan(apply1, Pproj, n, k, m, keep, target, deg, sigma, u1, seed=0, verbose=False):
    rng = np.random.default_rng(seed)
    applies = [0]

    def A(x):
        applies[0] += 1
        return apply1(x)

    kk = k - 1  # u1 deflated: the k-1 non-trivial wanted
    v0 = Pproj(rng.standard_normal(n))
    v0 -= u1 * (u1 @ v0)
    if deg == 1:
        def check(th, X, est):
            return est.max() <= target, f"applies {applies[0]} est {est.max():.2e} lam_k {th[-1]:.9f}"
        th, X, outer = trlan_op(A, n, kk, m, keep, v0, False, check, verbose)
        return np.sort(np.concatenate([[0.0], th[:kk]])), dict(applies=applies[0], outer=outer)
    # one plain cycle for the cut point, then TRLan on the fixed filter
    res = {}

    def check0(th, X, est):
        res["th"], res["X"] = th, X
        return True, f"plain cycle: lam_keep {th[-1]:.9f}"
    th0, X0, outer0 = trlan_op(A, n, keep, m, keep, v0, False, check0, verbose)
    a_cut = th0[keep - 1]
    c = 0.5 * (a_cut + sigma)
    e = 0.5 * (sigma - a_cut)

    def F(x):
        y0 = x
        y1 = (A(x) - c * x) / e
        for _ in range(2, deg + 1):
            y0, y1 = y1, 2 * (A(y1) - c * y1) / e - y0
        return y1 if deg % 2 == 0 else -y1

    def check(th, X, est):
        # cheap filter-space estimate first; explicit A residuals only when it is small
        if est.max() > 1e-6 * max(abs(th[0]), 1.0):
            return False, f"applies {applies[0]} F-est {est.max():.2e}"
        AX = np.stack([A(X[:, i]) for i in range(X.shape[1])], axis=1)
        lam = np.einsum("ij,ij->j", X, AX)
        rA = np.linalg.norm(AX - X * lam, axis=0).max()
        res["lam"] = lam
        return rA <= target, f"applies {applies[0]} F-est {est.max():.2e} A-res {rA:.2e} lam_max {lam.max():.9f}"
    v1 = X0[:, :kk].sum(axis=1)
    th, X, outer = trlan_op(F, n, kk, m, keep, v1, True, check, verbose)
    lam = np.sort(res["lam"])
    return np.sort(np.concatenate([[0.0], lam])), dict(applies=applies[0], outer=outer + outer0, a_cut=a_cut)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200_000)
    ap.add_argument("--deg", type=int, nargs="+", default=[1, 10])
    ap.add_argument("--m", type=int, default=110)
    ap.add_argument("--keep", type=int, default=80)
    ap.add_argument("--k", type=int, default=50)
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("-v", action="store_true")
    args = ap.parse_args()
    from synth import baseline_config
    t0 = time.time()
    g, cfg = baseline_config(4, n=args.n)
    apply1, P, sigma, u1, n = make_op(g, True)
    print(f"graph n={n} nnz={g.nnz} sigma={sigma:.4f} ({time.time()-t0:.1f}s)", flush=True)
    for deg in args.deg:
        t0 = time.time()
        lam, info = trlan(lambda x: apply1(x, True), P, n, args.k, args.m, args.keep, args.tol * sigma, deg, sigma,
                          u1, verbose=args.v)
        print(f"deg={deg}: applies {info['applies']} outer {info['outer']} "
              f"lam2 {lam[1]:.10f} lamk {lam[-1]:.10f} wall {time.time()-t0:.0f}s "
              f"model_s(0.77ms/apply + 3*95*5.2us/outer) {info['applies']*0.77e-3 + info['outer']*3*95*5.2e-6:.1f}",
              flush=True)


if __name__ == "__main__":
    main()
