"""The torch m-SBM sampler (synth/msbm_gpu.py, the §8(f) N3 cost sweep's generator) draws the
same law as synth/msbm.py: pinned on the CPU device (same code path as on the GPU)."""
import numpy as np
import pytest

from synth.msbm import _pair_table
from synth.msbm_gpu import exp1_msbm_torch, msbm_torch


def test_structure_and_pair_type_frequencies():
    n, h, k = 3000, 3, 4
    probs = (0.08, 0.05, 0.03, 0.01)
    g = msbm_torch(n, h, k, seed=11, probs=probs, letters="paper", device="cpu").host()
    rp, col = g.row_ptr.astype(np.int64), g.col.astype(np.int64)
    rows = np.repeat(np.arange(n), np.diff(rp))
    assert np.all(rows != col)  # zero diagonal (Eq. w-msbm)
    key = rows * n + col
    assert np.all(np.diff(key) > 0)  # rows sorted, no duplicates
    assert np.array_equal(np.sort(col * n + rows), key)  # symmetric
    assert np.all(np.diff(rp) > 0)  # no isolated vertex (R13)
    # every (cell, cell) pair holds exactly its Binomial count: compare the per pair-type edge
    # frequency with p (5 standard deviations of the binomial proportion)
    cell = g.clusters.astype(np.int64) * h + g.groups
    P = _pair_table(h, k, probs, "paper")
    up = rows < col
    ca, cb = cell[rows[up]], cell[col[up]]
    same_cl = (ca // h) == (cb // h)
    same_gr = (ca % h) == (cb % h)
    cl = g.clusters.astype(np.int64)
    for sc, sg in [(True, True), (True, False), (False, True), (False, False)]:
        m = np.sum((same_cl == sc) & (same_gr == sg))
        same_c = cl[:, None] == cl[None, :]
        same_g = g.groups[:, None] == g.groups[None, :]
        mask = np.triu((same_c == sc) & (same_g == sg), 1)
        npairs = int(mask.sum())
        p = P[0, 0] if sc and sg else (P[0, 1] if sc else (P[0, h] if sg else P[0, h + 1]))
        sd = np.sqrt(npairs * p * (1 - p))
        assert abs(m - npairs * p) <= 5 * sd + 1, (sc, sg, m, npairs * p)


def test_exp1_law_and_determinism():
    a = exp1_msbm_torch(2000, 2, seed=3, device="cpu")
    b = exp1_msbm_torch(2000, 2, seed=3, device="cpu")
    assert a.nnz == b.nnz and bool((a.col == b.col).all())
    assert np.bincount(a.groups).tolist() == [1000, 1000]
    assert np.bincount(a.clusters).tolist() == [400] * 5
    assert a.meta["letters"] == "paper"
