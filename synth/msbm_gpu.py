"""The m-SBM law of synth/msbm.py written in torch so that it runs on the GPU — inputs only.

Same law as `msbm.msbm` (App. B.1.2): groups and the
stratified cluster dealing (reading R12) are drawn exactly as there (numpy, streams 0 and 1,
O(n)); the edges are exact independent Bernoulli per vertex pair, sampled per (cell, cell)
pair as M_ab ~ Binomial(N_ab, p_ab) (numpy, stream 4) followed by a uniform M_ab-subset of
the N_ab pairs: random pairs drawn on the device with replacement, deduplicated by a sort,
topped up until every cell pair holds exactly M_ab distinct edges.  Isolated vertices are
repaired as in reading R13.  Unit weights.

The device sampler's random stream (torch.Generator seeded by (seed, 4)) differs from
numpy's, so for a given seed the graphs differ from `msbm.msbm`'s (same law, different
draw); tests pin the law on the CPU device.  Used for the §8(f) N3 cost sweep at sizes the
numpy sampler does not reach in minutes (the Experiment-1 law's degree grows as n^(1/3)).
"""
from __future__ import annotations

import numpy as np

from .msbm import MSBMGraph, _deal_clusters, _draw_groups, _pair_table, _rng


def _gen(seed: int, stream: int, device):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(np.random.SeedSequence([int(seed), int(stream), 7]).generate_state(1, np.uint64)[0] >> 1))
    return g


class DeviceGraph:
    """CSR on a torch device (row_ptr / col int32, val float64) + host groups / clusters."""

    def __init__(self, n, row_ptr, col, val, groups, clusters, h, k, meta):
        self.n, self.row_ptr, self.col, self.val = n, row_ptr, col, val
        self.groups, self.clusters, self.h, self.k, self.meta = groups, clusters, h, k, meta

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1].item())

    def host(self) -> MSBMGraph:
        return MSBMGraph(self.n, self.row_ptr.cpu().numpy(), self.col.cpu().numpy(), self.val.cpu().numpy(),
                         self.groups, self.clusters, self.h, self.k, dict(self.meta))


def msbm_torch(n, h, k, *, seed, probs, group_counts=None, letters="paper", device="cuda",
               name="msbm_gpu") -> DeviceGraph:
    """m-SBM with absolute pair-type probabilities `probs` = (a, b, c, d) (letters per R10)."""
    import torch
    groups = _draw_groups(n, h, seed, None, group_counts)
    clusters = _deal_clusters(groups, h, k, seed)
    cell_np = clusters.astype(np.int64) * h + groups
    C = k * h
    P = _pair_table(h, k, probs, letters)
    assert P.max() <= 1.0
    sizes = np.bincount(cell_np, minlength=C).astype(np.int64)
    A, B = np.triu_indices(C)
    N = np.where(A == B, sizes[A] * (sizes[A] - 1) // 2, sizes[A] * sizes[B])
    M = _rng(seed, 4).binomial(N, P[A, B]).astype(np.int64)
    dev = torch.device(device)
    gen = _gen(seed, 4, dev)
    cell = torch.from_numpy(cell_np).to(dev)
    order = torch.argsort(cell, stable=True)
    off = torch.from_numpy(np.concatenate([[0], np.cumsum(sizes)])).to(dev)
    sz = torch.from_numpy(sizes).to(dev)
    Ad, Bd = torch.from_numpy(A.astype(np.int64)).to(dev), torch.from_numpy(B.astype(np.int64)).to(dev)
    Md = torch.from_numpy(M).to(dev)
    npairs = len(A)

    def pair_id(ca, cb):
        lo, hi = torch.minimum(ca, cb), torch.maximum(ca, cb)
        return lo * C - lo * (lo - 1) // 2 + (hi - lo)

    have = torch.zeros(0, dtype=torch.int64, device=dev)
    need = Md.clone()
    for _ in range(200):
        tot = int(need.sum().item())
        if tot == 0:
            break
        pid = torch.repeat_interleave(torch.arange(npairs, device=dev), need)
        ca, cb = Ad[pid], Bd[pid]
        del pid
        i = (torch.rand(tot, generator=gen, device=dev, dtype=torch.float64) * sz[ca]).long().clamp_max_(sz[ca] - 1)
        j = (torch.rand(tot, generator=gen, device=dev, dtype=torch.float64) * sz[cb]).long().clamp_max_(sz[cb] - 1)
        u, v = order[off[ca] + i], order[off[cb] + j]
        del i, j, ca, cb
        keep = u != v
        u, v = u[keep], v[keep]
        key = torch.minimum(u, v) * n + torch.maximum(u, v)
        del u, v, keep
        have = torch.unique(torch.cat([have, key]), sorted=True)
        del key
        cnt = torch.bincount(pair_id(cell[have // n], cell[have % n]), minlength=npairs)
        need = Md - cnt
        assert bool((need >= 0).all())
    else:
        raise RuntimeError("device sampler did not converge")
    # reading R13: an isolated vertex is joined to a uniform vertex of its own cluster
    deg = torch.bincount(have // n, minlength=n) + torch.bincount(have % n, minlength=n)
    iso = torch.nonzero(deg == 0).flatten().cpu().numpy()
    repaired = len(iso)
    if repaired:
        rng = _rng(seed, 6)
        extra = []
        for vtx in iso:
            pool = np.flatnonzero(clusters == clusters[vtx])
            pool = pool[pool != vtx]
            o = int(pool[rng.integers(0, len(pool))])
            extra.append(min(o, vtx) * n + max(o, vtx))
        have = torch.unique(torch.cat([have, torch.tensor(extra, dtype=torch.int64, device=dev)]), sorted=True)
    # symmetric CSR, rows sorted
    u, v = have // n, have % n
    k2 = torch.cat([u * n + v, v * n + u])
    del u, v, have
    k2, _ = torch.sort(k2)
    rows = k2 // n
    col = (k2 % n).to(torch.int32)
    del k2
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    row_ptr[1:] = torch.cumsum(torch.bincount(rows, minlength=n), 0)
    del rows
    assert int(row_ptr[-1].item()) < 2**31 - 1
    val = torch.ones(col.numel(), dtype=torch.float64, device=dev)
    meta = dict(name=name, seed=seed, probs=list(probs), letters=letters, weights="unit", repaired=repaired,
                device=str(dev.type))
    return DeviceGraph(n, row_ptr.to(torch.int32), col, val, groups, clusters, h, k, meta)


def exp1_msbm_torch(n, h, *, k=5, seed=0, device="cuda") -> DeviceGraph:
    """The paper's Experiment-1 / Fig. 8 law (synth.exp1_msbm): k = 5
    fair planted clusters, h equal groups, a, b, c, d = (10, 7, 4, 1) (log n / n)^(2/3) with the
    paper's letters, unit weights."""
    base = (np.log(n) / n) ** (2.0 / 3.0)
    probs = tuple(float(x * base) for x in (10, 7, 4, 1))
    counts = np.full(h, n // h, dtype=np.int64)
    counts[: n - counts.sum()] += 1
    return msbm_torch(n, h, k, seed=seed, probs=probs, group_counts=tuple(int(c) for c in counts),
                      letters="paper", device=device, name=f"exp1-h{h}-gpu")
