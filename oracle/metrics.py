"""Comparison metrics — TEST INFRASTRUCTURE ONLY.

* balance (Eq. bal) and average balance (Eq. avebal);
* count matrix M = G^T H (Eq. mz);
* adjusted Rand index (Hubert & Arabie) — permutation invariant;
* Hungarian matching of cluster labels (scipy linear_sum_assignment);
* largest principal angle between subspaces, sine form (reading R9);
* error rate of a clustering (Eq. err).
"""
from __future__ import annotations

import numpy as np
from scipy.optimize import linear_sum_assignment


def count_matrix(labels, groups, k, h):
    """M = G^T H: m_sl = |V_s ∩ C_l|."""
    M = np.zeros((h, k), dtype=np.int64)
    np.add.at(M, (groups, labels), 1)
    return M


def balance(labels, groups, k, h):
    """Balance(C_l) = min_{s != s'} |V_s ∩ C_l| / |V_s' ∩ C_l| = min_s / max_s."""
    M = count_matrix(labels, groups, k, h)
    out = np.zeros(k)
    for l in range(k):
        col = M[:, l]
        out[l] = 0.0 if col.max() == 0 else col.min() / col.max()
    return out


def ari(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    _, ai = np.unique(a, return_inverse=True)
    _, bi = np.unique(b, return_inverse=True)
    tab = np.zeros((ai.max() + 1, bi.max() + 1), dtype=np.int64)
    np.add.at(tab, (ai, bi), 1)
    comb = lambda x: x * (x - 1) / 2.0
    sij = comb(tab).sum()
    sa = comb(tab.sum(1)).sum()
    sb = comb(tab.sum(0)).sum()
    n = len(a)
    exp = sa * sb / comb(n)
    mx = 0.5 * (sa + sb)
    if mx == exp:
        return 1.0
    return float((sij - exp) / (mx - exp))


def hungarian_match(ref, other, k):
    """Permutation perm with perm[other_label] = ref_label maximising agreement."""
    tab = np.zeros((k, k), dtype=np.int64)
    np.add.at(tab, (ref, other), 1)
    r, c = linear_sum_assignment(-tab)
    perm = np.empty(k, dtype=np.int64)
    perm[c] = r
    return perm


def subspace_sin(Xa, Xb):
    """sin of the largest principal angle between span(Xa) and span(Xb)
    (both orthonormalised first): || (I - Qa Qa^T) Qb ||_2."""
    Qa, _ = np.linalg.qr(Xa)
    Qb, _ = np.linalg.qr(Xb)
    R = Qb - Qa @ (Qa.T @ Qb)
    return float(np.linalg.norm(R, 2))


def error_rate(truth, labels, k):
    """Err(H^ - H) = (1/n) min_{J in Pi_k} ||H^ J - H||_F^2 (Eq. err):
    H, H^ are the n x k cluster indicator matrices; the minimising permutation is
    the assignment maximising the agreement (the squared Frobenius distance of
    indicator matrices is 2 (n - agreement)).  Note this is twice the proportion
    of misclustered vertices (reading R17)."""
    truth = np.asarray(truth)
    labels = np.asarray(labels)
    n = len(truth)
    tab = np.zeros((k, k), dtype=np.int64)
    np.add.at(tab, (labels, truth), 1)
    r, c = linear_sum_assignment(-tab)
    agree = int(tab[r, c].sum())
    return 2.0 * (n - agree) / n
