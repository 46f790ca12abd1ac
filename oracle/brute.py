"""Tier B oracle: 50-digit brute force for tiny graphs (n <= 12) — TEST INFRASTRUCTURE ONLY.

Follows the §3.2 variant in exact-ish arithmetic: X = D^{1/2} H,
L_n = D^{-1/2} L D^{-1/2}, C = D^{-1/2} F; V = orthonormal basis
of null(C^T) from a full Householder QR of C (mpmath.qr); L^v = V^T L_n V
(P:523); eigenpairs by mpmath's Jacobi `eigsy`.  Unnormalized (R1): L, C = F.
Also: exhaustive enumeration for Lemma 2.1(ii).
Pins Tier D (tests/test_oracle_dense.py).
"""
from __future__ import annotations

import itertools

import mpmath as mp
import numpy as np


def brute_fair_eig(W, groups, h, normalized, dps=50, F=None):
    """Return (evals ascending as mpf list, X as mp.matrix n x (n-r)), r = h-1 for
    group fairness, or the columns of an explicit constraint matrix F (n x r)."""
    mp.mp.dps = dps
    W = [[mp.mpf(float(x)) for x in row] for row in np.asarray(W)]
    n = len(W)
    d = [mp.fsum(row) for row in W]
    L = mp.matrix(n, n)
    for i in range(n):
        for j in range(n):
            L[i, j] = (d[i] if i == j else 0) - W[i][j]
    s = [1 / mp.sqrt(x) for x in d] if normalized else [mp.mpf(1)] * n
    Ln = mp.matrix(n, n)
    for i in range(n):
        for j in range(n):
            Ln[i, j] = s[i] * L[i, j] * s[j]
    if F is not None:
        Fa = np.asarray(F, dtype=np.float64).reshape(n, -1)
        r = Fa.shape[1]
    else:
        counts = [sum(1 for g in groups if g == t) for t in range(h)]
        r = h - 1
    if r > 0:
        C = mp.matrix(n, r)
        for i in range(n):
            for t in range(r):
                f = mp.mpf(float(Fa[i, t])) if F is not None else (1 if groups[i] == t else 0) - mp.mpf(counts[t]) / n
                C[i, t] = s[i] * f
        Qf, _ = mp.qr(C, mode="full")
        V = mp.matrix(n, n - r)
        for i in range(n):
            for j in range(n - r):
                V[i, j] = Qf[i, j + r]
    else:
        V = mp.eye(n)
    Lv = V.T * Ln * V
    E, Y = mp.eigsy(Lv)
    order = sorted(range(len(E)), key=lambda i: E[i])
    evals = [E[i] for i in order]
    Ys = mp.matrix(Y.rows, len(order))
    for c, i in enumerate(order):
        for r in range(Y.rows):
            Ys[r, c] = Y[r, i]
    return evals, V * Ys


def all_clusterings(n, k):
    """Every assignment of n vertices to k labelled non-empty clusters."""
    for lab in itertools.product(range(k), repeat=n):
        if len(set(lab)) == k:
            yield np.array(lab)


def is_fair(labels, groups, h, k):
    """Definition 2.1: |V_s ∩ C_l| / |C_l| = |V_s| / |V| for all s, l,
    checked in integers as n |V_s ∩ C_l| = |V_s| |C_l| (Eq. nmz)."""
    n = len(labels)
    for l in range(k):
        cl = labels == l
        for s in range(h):
            if n * np.sum(cl & (groups == s)) != np.sum(groups == s) * np.sum(cl):
                return False
    return True
