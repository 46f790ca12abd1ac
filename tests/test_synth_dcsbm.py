"""The config-5 input law (synth/dcsbm.py: DC-SBM m-SBM, BASELINE config 5,
SURVEY §8(d)) at reduced n on CPU: the generated graph is a valid fair-SC
input (symmetric, zero diagonal, unit weights, no isolated vertex, every
group present), its mean degree matches the target, its degrees are
Pareto-skewed, its cluster sizes follow the largest-remainder rounding of a
Dirichlet draw, and the generator is deterministic per seed and device."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def g20k():
    from synth.dcsbm import config5
    g, cfg = config5(n=20_000, device="cpu")
    return g.host(), cfg


def test_valid_input(g20k):
    g, cfg = g20k
    W = g.to_scipy()
    assert abs(W - W.T).sum() == 0
    assert W.diagonal().sum() == 0
    assert np.all(g.val == 1.0)
    deg = np.diff(g.row_ptr)
    assert deg.min() >= 1
    assert np.all(np.bincount(g.groups, minlength=8) > 0) and g.groups.max() < 8
    # sorted, unique columns per row
    for i in range(0, g.n, 997):
        c = g.col[g.row_ptr[i]:g.row_ptr[i + 1]]
        assert np.all(np.diff(c) > 0)


def test_mean_degree_and_skew(g20k):
    g, cfg = g20k
    deg = np.diff(g.row_ptr)
    # expected mean degree 32 before multi-edge collapse; collapse removes a little
    assert 29.0 <= deg.mean() <= 32.5
    # Pareto(2.5) propensities: heavy right tail (max >> mean), median below mean
    assert deg.max() > 10 * deg.mean()
    assert np.median(deg) < deg.mean()


def test_cluster_sizes_dirichlet(g20k):
    from synth.dcsbm import _cluster_sizes
    g, cfg = g20k
    sz = np.bincount(g.clusters, minlength=64)
    assert np.array_equal(np.sort(sz), np.sort(_cluster_sizes(20_000, 64, 16440)))
    assert sz.sum() == 20_000 and sz.min() >= 1
    # Dirichlet(2) sizes are uneven: largest / smallest well above 1
    assert sz.max() / sz.min() > 3


def test_deterministic():
    from synth.dcsbm import dcsbm
    a = dcsbm(3000, 3, 5, seed=1, device="cpu").host()
    b = dcsbm(3000, 3, 5, seed=1, device="cpu").host()
    c = dcsbm(3000, 3, 5, seed=2, device="cpu").host()
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col, b.col)
    assert not (len(a.col) == len(c.col) and np.array_equal(a.col, c.col))
