"""Modified stochastic block model (m-SBM) generator — inputs only.

Follows PAPER.md App. B.1.2: vertices carry a group (sensitive
attribute) and a planted cluster; an undirected edge {i,j}, i != j,
is present independently with a probability that depends only on whether i,j
share a cluster and whether they share a group (Eq. p-msbm), and
w_ii = 0 (Eq. w-msbm).

Concrete recipe (readings R10-R13 listed in DESIGN.md):
  * groups   : i.i.d. categorical, or exact counts shuffled (config 2);
  * clusters : stratified dealing (R12) — per group, shuffle its vertices and
               deal them round-robin to the k clusters, the dealer continuing
               across groups; every cluster gets n/k (+-1) vertices and every
               (cluster, group) cell is within +-1 of proportional;
  * letters  : BASELINE.json config 1 convention (R10): a = same cluster &
               same group, b = same cluster / different group, c = different
               cluster / same group, d = different both.  `letters="paper"`
               swaps b and c to the paper's Eq. p-msbm convention;
  * edges    : exact independent Bernoulli per pair.  Small n draws every
               pair; large n draws, per (cell, cell) pair, the Binomial edge
               count and then a uniform subset of that many distinct pairs
               (same law, O(nnz) work);
  * weights  : 1.0, or uniform(0.5, 1.5) per undirected edge (config 3, R11);
  * repair   : an isolated vertex is joined to one uniform vertex of its own
               cluster with weight 1 (R13) — the paper assumes D > 0.

Randomness: numpy Generator(PCG64) seeded by SeedSequence([seed, stream]);
streams 0 groups, 1 cluster dealing, 4 edges, 5 weights, 6 repair.
Vertex order is as generated (random with respect to clusters).

Output is CSR (row_ptr int32 n+1, col int32 nnz sorted within rows,
val float64 nnz), symmetric, both triangles stored, zero diagonal.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

_DENSE_PAIR_LIMIT = 30_000  # n at or below which every vertex pair is drawn


def _sorted_unique(x: np.ndarray) -> np.ndarray:
    """np.unique for int64 keys via sort (numpy's hash path is slow at 1e8)."""
    x = np.sort(x)
    if len(x) == 0:
        return x
    keep = np.empty(len(x), dtype=bool)
    keep[0] = True
    np.not_equal(x[1:], x[:-1], out=keep[1:])
    return x[keep]


def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(seed), int(stream)]))


@dataclasses.dataclass
class MSBMGraph:
    n: int
    row_ptr: np.ndarray  # int32 (n+1)
    col: np.ndarray  # int32 (nnz)
    val: np.ndarray  # float64 (nnz)
    groups: np.ndarray  # int32 (n), values in [0, h)
    clusters: np.ndarray  # int32 (n), planted clusters in [0, k) (-1: none)
    h: int
    k: int
    meta: dict

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col, self.row_ptr), shape=(self.n, self.n))

    def dense(self) -> np.ndarray:
        a = np.zeros((self.n, self.n))
        rows = np.repeat(np.arange(self.n), np.diff(self.row_ptr))
        a[rows, self.col] = self.val
        return a


# ----------------------------------------------------------------------------
# building blocks
# ----------------------------------------------------------------------------

def _draw_groups(n, h, seed, group_probs=None, group_counts=None):
    rng = _rng(seed, 0)
    if group_counts is not None:
        counts = np.asarray(group_counts, dtype=np.int64)
        assert counts.sum() == n and len(counts) == h
        g = np.repeat(np.arange(h, dtype=np.int32), counts)
        rng.shuffle(g)
        return g
    probs = np.full(h, 1.0 / h) if group_probs is None else np.asarray(group_probs, float)
    probs = probs / probs.sum()
    for _ in range(1000):
        g = rng.choice(h, size=n, p=probs).astype(np.int32)
        if np.all(np.bincount(g, minlength=h) > 0):
            return g
    raise ValueError("could not draw non-empty groups")


def _deal_clusters(groups, h, k, seed):
    """Stratified dealing (reading R12)."""
    rng = _rng(seed, 1)
    n = len(groups)
    clusters = np.empty(n, dtype=np.int32)
    dealer = 0
    for s in range(h):
        members = np.flatnonzero(groups == s)
        rng.shuffle(members)
        clusters[members] = (dealer + np.arange(len(members))) % k
        dealer += len(members)
    return clusters


def _pair_table(h, k, rates, letters):
    """(kh x kh) table of pair-type rates; cell c = cluster*h + group."""
    a, b, c, d = rates
    if letters == "paper":  # Eq. p-msbm: b diff-cluster/same-group, c same-cluster/diff-group
        b, c = c, b
    C = k * h
    cl = np.arange(C) // h
    gr = np.arange(C) % h
    same_cl = cl[:, None] == cl[None, :]
    same_gr = gr[:, None] == gr[None, :]
    R = np.where(same_cl & same_gr, a, np.where(same_cl, b, np.where(same_gr, c, d)))
    return R.astype(np.float64)


def _sample_dense(n, cell, Pcell, seed):
    """Draw every pair i<j independently: edge iff U_ij < p(cell_i, cell_j)."""
    rng = _rng(seed, 4)
    keys = []
    chunk = max(1, int(4e7 // max(n, 1)))
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        U = rng.random((r1 - r0, n))
        P = Pcell[cell[r0:r1][:, None], cell[None, :]]
        hit = U < P
        ii = np.arange(r0, r1)[:, None]
        hit &= np.arange(n)[None, :] > ii  # strict upper triangle, w_ii = 0
        rr, cc = np.nonzero(hit)
        keys.append((rr.astype(np.int64) + r0) * n + cc.astype(np.int64))
    return np.concatenate(keys) if keys else np.zeros(0, np.int64)


def _sample_sparse(n, cell, Pcell, seed):
    """Per (cell a <= cell b): M ~ Binomial(N_ab, p_ab), then a uniform M-subset
    of the N_ab vertex pairs (draw with replacement, dedupe, top up)."""
    rng = _rng(seed, 4)
    C = Pcell.shape[0]
    order = np.argsort(cell, kind="stable")
    sizes = np.bincount(cell, minlength=C).astype(np.int64)
    off = np.concatenate([[0], np.cumsum(sizes)])
    A, B = np.triu_indices(C)
    A = A.astype(np.int64)
    B = B.astype(np.int64)
    N = np.where(A == B, sizes[A] * (sizes[A] - 1) // 2, sizes[A] * sizes[B])
    M = rng.binomial(N, Pcell[A, B]).astype(np.int64)

    def pair_id(ca, cb):
        lo = np.minimum(ca, cb)
        hi = np.maximum(ca, cb)
        return lo * C - lo * (lo - 1) // 2 + (hi - lo)

    have = np.zeros(0, np.int64)
    need = M.copy()
    for _ in range(200):
        tot = int(need.sum())
        if tot == 0:
            break
        pid = np.repeat(np.arange(len(A)), need)
        ca, cb = A[pid], B[pid]
        i = rng.integers(0, sizes[ca])
        j = rng.integers(0, sizes[cb])
        u = order[off[ca] + i].astype(np.int64)
        v = order[off[cb] + j].astype(np.int64)
        keep = u != v
        u, v = u[keep], v[keep]
        key = np.minimum(u, v) * n + np.maximum(u, v)
        have = _sorted_unique(np.concatenate([have, key]))
        cnt = np.bincount(pair_id(cell[have // n].astype(np.int64), cell[have % n].astype(np.int64)),
                          minlength=len(A))
        need = M - cnt
        assert np.all(need >= 0)
    else:
        raise RuntimeError("sparse sampler did not converge")
    return have


def _to_csr(n, keys, w):
    """Undirected edge list (u<v keys, weights) -> symmetric CSR, rows sorted."""
    u = keys // n
    v = keys % n
    k2 = np.concatenate([u * n + v, v * n + u])
    if np.all(w == w[0]) if len(w) else True:
        k2.sort()
        val = np.full(len(k2), w[0] if len(w) else 1.0)
    else:
        idx = np.argsort(k2, kind="stable")
        k2 = k2[idx]
        val = np.concatenate([w, w])[idx]
    rows = k2 // n
    col = (k2 % n).astype(np.int32)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    assert row_ptr[-1] < 2**31 - 1
    return row_ptr.astype(np.int32), col, val.astype(np.float64)


def _repair_isolated(n, keys, clusters, seed):
    """Reading R13: join each isolated vertex to a uniform vertex of its cluster."""
    touched = np.zeros(n, dtype=bool)
    touched[keys // n] = True
    touched[keys % n] = True
    iso = np.flatnonzero(~touched)
    if len(iso) == 0:
        return keys, 0
    rng = _rng(seed, 6)
    extra = []
    for vtx in iso:
        pool = np.flatnonzero(clusters == clusters[vtx]) if clusters[vtx] >= 0 else np.arange(n)
        pool = pool[pool != vtx]
        if len(pool) == 0:
            pool = np.setdiff1d(np.arange(n), [vtx])
        o = int(pool[rng.integers(0, len(pool))])
        extra.append(min(o, vtx) * n + max(o, vtx))
    keys = _sorted_unique(np.concatenate([keys, np.asarray(extra, np.int64)]))
    return keys, len(iso)


# ----------------------------------------------------------------------------
# public generators
# ----------------------------------------------------------------------------

def msbm(n, h, k, *, seed, probs=None, rel=None, mean_degree=None, group_probs=None,
         group_counts=None, weights="unit", letters="baseline", name="msbm") -> MSBMGraph:
    """m-SBM graph.  Give either absolute `probs`=(a,b,c,d) or a
    relative pattern `rel` scaled so that the expected mean degree is
    `mean_degree` given the realised cell sizes."""
    groups = _draw_groups(n, h, seed, group_probs, group_counts)
    clusters = _deal_clusters(groups, h, k, seed)
    cell = (clusters.astype(np.int64) * h + groups).astype(np.int64)
    C = k * h
    if probs is not None:
        Pcell = _pair_table(h, k, probs, letters)
        t = 1.0
    else:
        R = _pair_table(h, k, rel, letters)
        s = np.bincount(cell, minlength=C).astype(np.float64)
        denom = s @ R @ s - np.sum(s * np.diag(R))
        t = mean_degree * n / denom
        Pcell = R * t
    assert Pcell.max() <= 1.0
    if n <= _DENSE_PAIR_LIMIT:
        keys = _sample_dense(n, cell, Pcell, seed)
    else:
        keys = _sample_sparse(n, cell, Pcell, seed)
    keys, n_repaired = _repair_isolated(n, keys, clusters, seed)
    if weights == "unit":
        w = np.ones(len(keys))
    elif weights == "uniform":
        w = _rng(seed, 5).uniform(0.5, 1.5, size=len(keys))
    else:
        raise ValueError(weights)
    row_ptr, col, val = _to_csr(n, keys, w)
    meta = dict(name=name, seed=seed, t=t, probs=(None if probs is None else list(probs)),
                rel=(None if rel is None else list(rel)), mean_degree=mean_degree,
                weights=weights, letters=letters, repaired=n_repaired)
    return MSBMGraph(n, row_ptr, col, val, groups, clusters, h, k, meta)


def _zipf_probs(h, a):
    p = np.arange(1, h + 1, dtype=np.float64) ** (-a)
    return p / p.sum()


# BASELINE.json "configs".  `normalized` selects L_n
# vs L (reading R1); `k_eig`/`tol` are the eigensolve request.
CONFIGS = {
    1: dict(n=1_000, h=2, k=5, probs=(0.30, 0.20, 0.10, 0.05), weights="unit",
            normalized=False, k_eig=5, tol=1e-10),
    2: dict(n=20_000, h=5, k=10, group_counts=(2000, 3000, 4000, 5000, 6000), rel=(8, 6, 2, 1),
            mean_degree=100, weights="unit", normalized=True, k_eig=10, tol=1e-10),
    3: dict(n=500_000, h=5, k=20, rel=(8, 6, 2, 1), mean_degree=64, weights="uniform",
            normalized=False, k_eig=20, tol=1e-8),
    4: dict(n=4_000_000, h=10, k=50, group_probs=tuple(_zipf_probs(10, 1.1)), rel=(8, 6, 2, 1),
            mean_degree=32, weights="unit", normalized=True, k_eig=50, tol=1e-8),
}


def baseline_config(c: int, n: int | None = None) -> tuple[MSBMGraph, dict]:
    """Graph for BASELINE config `c` (seed 16435 + c).  `n` optionally rescales
    the vertex count (same law, same mean degree / literal probabilities) for
    reduced-size tests; group counts are rescaled proportionally."""
    if c == 5:  # DC-SBM law (synth/dcsbm.py); generated with torch on the GPU when one is visible
        import torch
        from .dcsbm import config5
        g, cfg = config5(n=n, device="cuda" if torch.cuda.is_available() else "cpu")
        return g.host(), cfg
    cfg = dict(CONFIGS[c])
    params = {kk: cfg[kk] for kk in ("probs", "rel", "mean_degree", "group_probs", "group_counts", "weights") if kk in cfg}
    nn = cfg["n"] if n is None else int(n)
    if n is not None and "group_counts" in params:
        gc = np.asarray(cfg["group_counts"], dtype=np.float64) * nn / cfg["n"]
        gi = np.floor(gc).astype(np.int64)
        gi[: nn - gi.sum()] += 1
        params["group_counts"] = tuple(int(x) for x in gi)
    g = msbm(nn, cfg["h"], cfg["k"], seed=16435 + c, name=f"cfg{c}", **params)
    return g, cfg


def exp1_msbm(n, h, *, k=5, seed=0) -> MSBMGraph:
    """The paper's Experiment-1 / Fig. 8 m-SBM: k = 5
    fair planted clusters, h equal groups, a,b,c,d = (10, 7, 4, 1) (log n / n)^(2/3)
    with the paper's letters (b: different cluster / same group, c: same
    cluster / different group, Eq. p-msbm), unit weights (the
    caption gives no alpha, beta; reading R11).  §8(f) N3."""
    base = (np.log(n) / n) ** (2.0 / 3.0)
    probs = tuple(float(x * base) for x in (10, 7, 4, 1))
    counts = np.full(h, n // h, dtype=np.int64)
    counts[: n - counts.sum()] += 1
    return msbm(n, h, k, seed=seed, probs=probs, group_counts=tuple(int(c) for c in counts), weights="unit",
                letters="paper", name=f"exp1-h{h}")


def planted_cliques(k, m, h, seed=0, shuffle=True) -> MSBMGraph:
    """k disjoint complete graphs K_m, each holding every group in exact
    proportion m/h (SURVEY §8(c) P-closed-1).  Unit weights."""
    assert m % h == 0
    n = k * m
    clusters = np.repeat(np.arange(k, dtype=np.int32), m)
    groups = np.tile(np.repeat(np.arange(h, dtype=np.int32), m // h), k)
    perm = _rng(seed, 0).permutation(n) if shuffle else np.arange(n)
    # vertex perm[i] plays the role of position i
    cl = np.empty(n, np.int32)
    gr = np.empty(n, np.int32)
    cl[perm] = clusters
    gr[perm] = groups
    keys = []
    for c in range(k):
        mem = np.sort(perm[c * m:(c + 1) * m]).astype(np.int64)
        a, b = np.triu_indices(m, 1)
        keys.append(mem[a] * n + mem[b])
    keys = np.sort(np.concatenate(keys))
    row_ptr, col, val = _to_csr(n, keys, np.ones(len(keys)))
    return MSBMGraph(n, row_ptr, col, val, gr, cl, h, k, dict(name="planted_cliques", m=m, seed=seed))


def random_laplacian(n, density, r, *, seed=0):
    """Experiment 4's random Laplacian: a random symmetric weight matrix
    W of prescribed sparsity `density` (uniform(0.5,1.5) weights, isolated vertices
    repaired, R13) and a random constraint matrix F (n x r, standard normal, PCG64
    stream 7) that "is not for group-membership information but only acts as a
    placeholder".  Returns (graph with h = 1, F)."""
    g = random_graph(n, 1, p=density, seed=seed, weights="uniform")
    F = _rng(seed, 7).standard_normal((n, r))
    return g, F


def random_graph(n, h, *, p=0.3, seed=0, weights="uniform", group_counts=None) -> MSBMGraph:
    """Erdos-Renyi G(n,p) with random groups and (optionally) random weights;
    isolated vertices repaired (R13).  For small oracle pins."""
    groups = _draw_groups(n, h, seed, None, group_counts)
    clusters = np.full(n, -1, np.int32)
    rng = _rng(seed, 4)
    iu, ju = np.triu_indices(n, 1)
    hit = rng.random(len(iu)) < p
    keys = iu[hit].astype(np.int64) * n + ju[hit]
    keys, _ = _repair_isolated(n, keys, clusters, seed)
    w = np.ones(len(keys)) if weights == "unit" else _rng(seed, 5).uniform(0.5, 1.5, len(keys))
    row_ptr, col, val = _to_csr(n, keys, w)
    return MSBMGraph(n, row_ptr, col, val, groups, clusters, h, 0, dict(name="random", p=p, seed=seed))


def hub_graph(n, h, *, hub_degrees=(1500, 5000), p=0.004, seed=0, weights="uniform") -> MSBMGraph:
    """G(n, p) plus hub vertices 0, 1, ... joined to hub_degrees[i] distinct random vertices:
    rows longer than any SpMV tile (edge cases of the row-aligned tiling).  For oracle pins."""
    groups = _draw_groups(n, h, seed, None, None)
    clusters = np.full(n, -1, np.int32)
    rng = _rng(seed, 4)
    iu, ju = np.triu_indices(n, 1)
    hit = rng.random(len(iu)) < p
    keys = [iu[hit].astype(np.int64) * n + ju[hit]]
    for hub, deg in enumerate(hub_degrees):
        nb = rng.choice(np.arange(hub + 1, n), size=min(deg, n - hub - 1), replace=False)
        keys.append(hub * n + nb.astype(np.int64))
    keys = _sorted_unique(np.concatenate(keys))
    keys, _ = _repair_isolated(n, keys, clusters, seed)
    w = np.ones(len(keys)) if weights == "unit" else _rng(seed, 5).uniform(0.5, 1.5, len(keys))
    row_ptr, col, val = _to_csr(n, keys, w)
    return MSBMGraph(n, row_ptr, col, val, groups, clusters, h, 0, dict(name="hub", seed=seed))
