"""Degree-corrected modified SBM (BASELINE config 5) — inputs only.

BASELINE.json config 5: "Unnormalized s-FairSC on a degree-skewed modified
SBM: n = 50,000,000, h = 8 uniform groups, k = 64 clusters with sizes
proportional to Dirichlet(alpha = 2); vertex degree propensities follow
Pareto(shape 2.5), DC-SBM style, at mean degree 32".  The m-SBM pair-type
pattern of App. B.1.2 (letters per reading R10, rates
(a,b,c,d) = t (8,6,2,1)) is multiplied by theta_i theta_j:

  * groups    : i.i.d. uniform over h                      (stream 0)
  * clusters  : sizes = largest-remainder rounding of n q, q ~ Dirichlet(2 1_k)
                (stream 2, numpy), labels dealt in a random order (stream 1)
  * theta_i   : Pareto(x_m = 1, shape 2.5) = (1-U)^(-1/2.5)  (stream 3)
  * edges     : per cell pair (a <= b) (cell = cluster * h + group),
                M_ab ~ Poisson(t R_ab Theta_a Theta_b (1/2 if a = b)), endpoints
                drawn within the cells with probability proportional to theta
                (stream 4); self-pairs dropped, multi-edges collapsed, so
                P(edge ij) = 1 - exp(-t theta_i theta_j R) ~ t theta_i theta_j R;
                t = 32 n / (Theta^T R Theta) gives expected mean degree 32 before
                the collapse
  * weights   : 1.0 (reading R11)
  * repair    : isolated vertices joined to a uniform vertex of their cluster
                (reading R13; stream 6)

At n = 5e7 the graph has ~1.6e9 stored entries (19 GB as CSR), beyond what
numpy builds in minutes, so the whole generator is written in torch and runs
on the GPU (or on the CPU for small n).  Randomness: torch.Generator(device)
seeded with hash(seed, stream); results are deterministic for a fixed device
type, seed and n (CUDA and CPU streams differ — tests compare both sides on
the same generated graph, never across devices).
"""
from __future__ import annotations

import numpy as np

from .msbm import MSBMGraph, _pair_table


def _gen(seed: int, stream: int, device):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(np.random.SeedSequence([int(seed), int(stream)]).generate_state(1, np.uint64)[0] >> 1))
    return g


def _cluster_sizes(n, k, seed):
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), 2]))
    q = rng.dirichlet(np.full(k, 2.0))
    raw = q * n
    sz = np.floor(raw).astype(np.int64)
    rem = n - int(sz.sum())
    order = np.argsort(-(raw - sz), kind="stable")
    sz[order[:rem]] += 1
    sz = np.maximum(sz, 1)
    while sz.sum() > n:  # (only if the max(.,1) bumped a tiny cluster)
        sz[np.argmax(sz)] -= 1
    return sz


def dcsbm(n, h, k, *, seed, rel=(8, 6, 2, 1), mean_degree=32.0, pareto_shape=2.5, device="cuda",
          chunk=200_000_000, name="dcsbm") -> MSBMGraph:
    import torch
    dev = torch.device(device)
    f64 = torch.float64
    groups = torch.randint(0, h, (n,), generator=_gen(seed, 0, dev), device=dev, dtype=torch.int64)
    sizes = _cluster_sizes(n, k, seed)
    labels = torch.repeat_interleave(torch.arange(k, device=dev), torch.as_tensor(sizes, device=dev))
    perm = torch.randperm(n, generator=_gen(seed, 1, dev), device=dev)
    clusters = torch.empty(n, dtype=torch.int64, device=dev)
    clusters[perm] = labels
    del labels, perm
    u = torch.rand(n, generator=_gen(seed, 3, dev), device=dev, dtype=f64)
    theta = (1.0 - u).pow(-1.0 / pareto_shape)
    del u
    C = k * h
    cell = clusters * h + groups
    R = torch.as_tensor(_pair_table(h, k, rel, "baseline"), device=dev, dtype=f64)
    Theta = torch.zeros(C, device=dev, dtype=f64).index_add_(0, cell, theta)
    t = mean_degree * n / float(Theta @ R @ Theta)
    # vertices sorted by cell; cumulative theta for proportional endpoint draws
    order = torch.argsort(cell, stable=True)
    cth = torch.cumsum(theta[order], 0)
    counts = torch.bincount(cell, minlength=C)
    ends = torch.cumsum(counts, 0)
    starts = ends - counts
    cstart = torch.where(starts > 0, cth[(starts - 1).clamp(min=0)], torch.zeros_like(Theta))
    # edge counts per cell pair (a <= b)
    A, B = torch.triu_indices(C, C, device=dev)
    lam = t * R[A, B] * Theta[A] * Theta[B] * torch.where(A == B, 0.5, 1.0).to(f64)
    M = torch.poisson(lam, generator=_gen(seed, 4, dev)).to(torch.int64)
    g4 = _gen(seed, 5, dev)  # endpoint draws (stream 5 of this generator family)
    keys = []
    pid = torch.repeat_interleave(torch.arange(len(A), device=dev), M)
    for lo in range(0, len(pid), chunk):
        p = pid[lo:lo + chunk]
        ca, cb = A[p], B[p]
        ua = torch.rand(len(p), generator=g4, device=dev, dtype=f64)
        ub = torch.rand(len(p), generator=g4, device=dev, dtype=f64)
        va = torch.searchsorted(cth, cstart[ca] + ua * Theta[ca], right=True).clamp(max=n - 1)
        vb = torch.searchsorted(cth, cstart[cb] + ub * Theta[cb], right=True).clamp(max=n - 1)
        # guard the float boundary: keep the draw inside its cell's segment
        va = torch.minimum(torch.maximum(va, starts[ca]), ends[ca] - 1)
        vb = torch.minimum(torch.maximum(vb, starts[cb]), ends[cb] - 1)
        x, y = order[va], order[vb]
        keep = x != y
        x, y = x[keep], y[keep]
        keys.append(torch.unique(torch.minimum(x, y) * n + torch.maximum(x, y)))
        del ua, ub, va, vb, x, y, keep, ca, cb, p
    del pid, cth, order
    key = torch.unique(torch.cat(keys)) if keys else torch.zeros(0, dtype=torch.int64, device=dev)
    del keys
    # isolated repair (R13): a uniform vertex of the same cluster
    deg = torch.bincount(key // n, minlength=n) + torch.bincount(key % n, minlength=n)
    iso = torch.nonzero(deg == 0).flatten()
    n_rep = int(iso.numel())
    if n_rep:
        g6 = _gen(seed, 6, dev)
        ordc = torch.argsort(clusters, stable=True)
        csz = torch.bincount(clusters, minlength=k)
        cst = torch.cumsum(csz, 0) - csz
        ci = clusters[iso]
        r = (torch.rand(n_rep, generator=g6, device=dev, dtype=f64) * csz[ci].to(f64)).to(torch.int64)
        r = torch.minimum(r, csz[ci] - 1)
        o = ordc[cst[ci] + r]
        o = torch.where(o == iso, ordc[cst[ci] + (r + 1) % csz[ci]], o)
        key = torch.unique(torch.cat([key, torch.minimum(o, iso) * n + torch.maximum(o, iso)]))
    # symmetric CSR, rows sorted
    both = torch.cat([key, (key % n) * n + key // n])
    del key
    both = torch.sort(both).values
    rows = both // n
    col = (both % n).to(torch.int32)
    del both
    rp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    rp[1:] = torch.cumsum(torch.bincount(rows, minlength=n), 0)
    del rows
    nnz = int(rp[-1])
    assert nnz < 2**31 - 1
    val = torch.ones(nnz, dtype=f64, device=dev)
    meta = dict(name=name, seed=seed, t=t, rel=list(rel), mean_degree=mean_degree, pareto_shape=pareto_shape,
                weights="unit", letters="baseline", repaired=n_rep, device=str(dev))
    return _TorchGraph(n, rp.to(torch.int32), col, val, groups.to(torch.int32), clusters.to(torch.int32), h, k,
                       meta)


class _TorchGraph:
    """The generated CSR kept as torch tensors on the generating device; .host()
    gives the numpy MSBMGraph used by the oracle side."""

    def __init__(self, n, row_ptr, col, val, groups, clusters, h, k, meta):
        self.n, self.row_ptr, self.col, self.val = n, row_ptr, col, val
        self.groups, self.clusters, self.h, self.k, self.meta = groups, clusters, h, k, meta

    @property
    def nnz(self):
        return int(self.col.numel())

    def host(self) -> MSBMGraph:
        return MSBMGraph(self.n, self.row_ptr.cpu().numpy(), self.col.cpu().numpy(), self.val.cpu().numpy(),
                         self.groups.cpu().numpy(), self.clusters.cpu().numpy(), self.h, self.k, dict(self.meta))


CONFIG5 = dict(n=50_000_000, h=8, k=64, rel=(8, 6, 2, 1), mean_degree=32, pareto_shape=2.5, weights="unit",
               normalized=False, k_eig=64, tol=1e-8)


def config5(n: int | None = None, device="cuda"):
    """BASELINE config 5 graph (seed 16435 + 5); `n` rescales the vertex count
    (same law, same mean degree) for reduced-size tests."""
    c = CONFIG5
    g = dcsbm(c["n"] if n is None else int(n), c["h"], c["k"], seed=16435 + 5, rel=c["rel"],
              mean_degree=c["mean_degree"], pareto_shape=c["pareto_shape"], device=device, name="cfg5")
    return g, dict(c)
