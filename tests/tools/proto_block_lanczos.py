"""Design experiment (not product, not oracle): block thick-restart Lanczos
convergence vs block size b on a reduced config-4 graph, numpy/scipy.

Counts operator applies and models GPU time from per-kernel costs so that b,
the basis size m and the kept count can be chosen before writing kernels.

    python scripts/proto_block_lanczos.py --n 200000 --b 1 2 4 --m 110 --keep 80
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def block_trlan(apply, P, n, k, b, m, keep, target, seed=0, max_restarts=100000, verbose=False):
    """Block Krylov-Schur (thick restart) with full CGS2 reorthogonalisation.
    Columns [0,pk) kept Ritz vectors; blocks of b appended; m = basis size at restart."""
    rng = np.random.default_rng(seed)
    V = np.zeros((n, m + b))
    X0 = P(rng.standard_normal((n, b)))
    V[:, :b], _ = np.linalg.qr(X0)
    T = np.zeros((m + b, m + b))
    pk, nv = 0, b
    applies = steps = restarts = 0
    sweepJ = []  # J per step (reorth cost)
    while True:
        while nv < m + b:
            blk = slice(nv - b, nv)
            W = apply(V[:, blk])
            applies += b
            steps += 1
            C = np.zeros((nv, b))
            for _ in range(2):
                c = V[:, :nv].T @ W
                W -= V[:, :nv] @ c
                C += c
            sweepJ.append(nv)
            Q, R = np.linalg.qr(W)
            if np.min(np.abs(np.diag(R))) < 1e-10 * np.max(np.abs(np.diag(R)) + 1e-300):
                raise RuntimeError("rank deficiency (not handled in prototype)")
            T[:nv, blk] = C
            T[nv:nv + b, blk] = R
            V[:, nv:nv + b] = Q
            nv += b
        Tm = np.triu(T[:m, :m])
        Tm = Tm + np.triu(Tm, 1).T
        # the first sub-diagonal blocks are in the lower part: mirror them
        L = np.tril(T[:m, :m], -1)
        Tm = np.triu(Tm) + np.triu(Tm, 1).T
        Tsym = 0.5 * (T[:m, :m] + T[:m, :m].T)
        theta, Y = np.linalg.eigh(Tsym)
        Rlast = T[m:m + b, m - b:m]
        res = np.linalg.norm(Rlast @ Y[m - b:m, :], axis=0)
        maxres = res[:k].max()
        if verbose:
            print(f"restart {restarts} applies {applies} maxres {maxres:.3e} theta_k {theta[k-1]:.10f}")
        if maxres <= target or restarts >= max_restarts:
            X = V[:, :m] @ Y[:, :k]
            return theta[:k], X, dict(applies=applies, steps=steps, restarts=restarts, sweepJ=sweepJ, m=m,
                                      keep=keep, b=b)
        pk = keep
        S = Rlast @ Y[m - b:m, :pk]
        Vn = np.zeros_like(V)
        Vn[:, :pk] = V[:, :m] @ Y[:, :pk]
        Vn[:, pk:pk + b] = V[:, m:m + b]
        V = Vn
        T = np.zeros_like(T)
        T[np.arange(pk), np.arange(pk)] = theta[:pk]
        T[pk:pk + b, :pk] = S
        T[:pk, pk:pk + b] = S.T
        nv = pk + b
        restarts += 1


def model_ms(info, n, nnz, spmm_ms, bw=6.2e12, sweeps=3):
    vb = 8.0 * n
    t = 0.0
    for J in info["sweepJ"]:
        t += spmm_ms[info["b"]] + sweeps * J * vb / bw * 1e3 + 4 * info["b"] * vb / bw * 1e3
    t += info["restarts"] * (info["m"] + info["keep"]) * vb / 1.5e12 * 1e3
    return t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200_000)
    ap.add_argument("--b", type=int, nargs="+", default=[1, 2, 4])
    ap.add_argument("--m", type=int, nargs="+", default=[110])
    ap.add_argument("--keep", type=int, nargs="+", default=[80])
    ap.add_argument("--k", type=int, default=50)
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("-v", action="store_true")
    args = ap.parse_args()
    from synth import baseline_config
    from oracle import sfairsc_cpu
    t0 = time.time()
    g, cfg = baseline_config(4, n=args.n)
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, cfg["normalized"])
    print(f"graph n={g.n} nnz={g.nnz} sigma={op.sigma:.4f} ({time.time()-t0:.1f}s)")
    # per-SpMM ms at cfg-4 size from the GPU probe (filled in from spmm_probe results)
    spmm_ms = {1: 0.90, 2: 0.95, 4: 1.05, 8: 1.6}
    nnz4 = 128e6
    for b in args.b:
        for m in args.m:
            for keep in args.keep:
                mm = args.k + ((m - args.k) // b) * b if False else m
                # m - keep must be a multiple of b
                mm = keep + ((m - keep) // b) * b
                t0 = time.time()
                theta, X, info = block_trlan(op.apply, op.P, g.n, args.k, b, mm, keep, args.tol * op.sigma,
                                             verbose=args.v)
                R = op.apply(X) - X * theta
                rr = np.linalg.norm(R, axis=0).max() / op.sigma
                J = np.mean(info["sweepJ"])
                print(f"b={b} m={mm} keep={keep}: applies {info['applies']} steps {info['steps']} restarts "
                      f"{info['restarts']} meanJ {J:.0f} resid {rr:.1e} theta_k {theta[-1]:.10f} "
                      f"model@4M-per-apply-count {model_ms(info, 4e6, nnz4, spmm_ms)/1e3:.2f}s "
                      f"(wall {time.time()-t0:.0f}s)", flush=True)


if __name__ == "__main__":
    main()
