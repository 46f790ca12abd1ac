"""k-means on the rows of H (Alg. 3 step 4) — TEST INFRASTRUCTURE ONLY.

The paper only says "apply k-means clustering to the rows of H" (P:312,
P:362).  Reading R16 pins the variant, following
SPEC.md S:375-383: k-means++ seeding, Lloyd iterations, best of n_restarts by
WCSS, empty clusters re-seeded at the farthest point, no row normalisation,
ties to the lowest index, Philox4x32-10 draws (counter (t, r, 8, 0)).
Plain loops/numpy in the stated order; pinned by tests/test_oracle_kmeans.py
(brute force over all partitions of 8-12 points, separated blobs).
"""
from __future__ import annotations

import dataclasses

import numpy as np

from .philox import uniform

KMEANS_STREAM = 8


@dataclasses.dataclass
class KMeansResult:
    labels: np.ndarray
    centroids: np.ndarray
    wcss: float
    restart: int


def _sqdist(Y, c):
    # sum over dimensions in index order
    diff = Y - c[None, :]
    out = np.zeros(Y.shape[0])
    for dd in range(Y.shape[1]):
        out += diff[:, dd] * diff[:, dd]
    return out


def _assign(Y, mu):
    n, K = Y.shape[0], mu.shape[0]
    best = np.full(n, np.inf)
    lab = np.zeros(n, dtype=np.int32)
    for c in range(K):
        dc = _sqdist(Y, mu[c])
        better = dc < best  # strict: ties stay with the lower index
        best[better] = dc[better]
        lab[better] = c
    return lab, best


def _means(Y, lab, K, prev):
    mu = prev.copy()
    counts = np.bincount(lab, minlength=K)
    for c in range(K):
        if counts[c] > 0:
            mu[c] = Y[lab == c].sum(axis=0) / counts[c]
    return mu, counts


def kmeanspp_seed(Y, K, seed, r):
    n = Y.shape[0]
    u = uniform(seed, np.arange(K), r, KMEANS_STREAM)
    idx = [min(int(np.floor(u[0] * n)), n - 1)]
    D2 = _sqdist(Y, Y[idx[0]])
    for t in range(1, K):
        prefix = np.cumsum(D2)
        total = prefix[-1]
        if total > 0:
            target = u[t] * total
            hit = np.flatnonzero(prefix > target)
            i = int(hit[0]) if len(hit) else int(np.flatnonzero(D2 > 0)[-1])
        else:
            i = min(int(np.floor(u[t] * n)), n - 1)
        idx.append(i)
        D2 = np.minimum(D2, _sqdist(Y, Y[i]))
    return np.array(idx)


def lloyd(Y, mu, max_iters=300):
    """Lloyd iterations from the centroids mu (R16): assign (ties to the lowest index),
    recompute the means, re-seed every empty cluster (increasing index) at the point
    farthest from its assigned centroid (first index of the maximum, each point used
    once), stop when no label changes.  Returns (labels, centroids, wcss)."""
    Y = np.asarray(Y, dtype=np.float64)
    mu = np.array(mu, dtype=np.float64)
    K = mu.shape[0]
    lab, _ = _assign(Y, mu)
    for _it in range(max_iters):
        mu, counts = _means(Y, lab, K, mu)
        if np.any(counts == 0):
            dist = _sqdist_labels(Y, mu, lab)
            used = np.zeros(len(Y), bool)
            for c in np.flatnonzero(counts == 0):
                dd = np.where(used, -1.0, dist)
                i = int(np.argmax(dd))  # first index of the maximum
                used[i] = True
                mu[c] = Y[i]
        new, _ = _assign(Y, mu)
        if np.array_equal(new, lab):
            break
        lab = new
    mu, _ = _means(Y, lab, K, mu)
    wcss = float(np.sum(_sqdist_labels(Y, mu, lab)))
    return lab, mu, wcss


def kmeans(Y, K, seed, n_restarts=10, max_iters=300) -> KMeansResult:
    Y = np.asarray(Y, dtype=np.float64)
    best = None
    for r in range(n_restarts):
        idx = kmeanspp_seed(Y, K, seed, r)
        lab, mu, wcss = lloyd(Y, Y[idx], max_iters)
        if best is None or wcss < best.wcss:
            best = KMeansResult(lab.copy(), mu.copy(), wcss, r)
    return best


def _sqdist_labels(Y, mu, lab):
    diff = Y - mu[lab]
    out = np.zeros(Y.shape[0])
    for dd in range(Y.shape[1]):
        out += diff[:, dd] * diff[:, dd]
    return out
