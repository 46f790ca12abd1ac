"""Pins for the Tier S oracle (paper's matrix-free s-FairSC + ARPACK), the
Philox generator, k-means and the metrics (CPU only)."""
import itertools
import json
import os

import numpy as np
import pytest
from sklearn.metrics import adjusted_rand_score

from conftest import GOLDEN
from oracle import fairsc, sfairsc_cpu
from oracle.kmeans import kmeans, kmeanspp_seed
from oracle.metrics import ari, balance, hungarian_match, subspace_sin
from oracle.philox import philox4x32_10, uniform
from synth import baseline_config, planted_cliques, random_graph


# --- Tier S vs Tier D ----------------------------------------------------------

@pytest.mark.parametrize("normalized,h,n,k", [(False, 2, 300, 5), (True, 5, 400, 6), (True, 3, 250, 4),
                                              (False, 1, 200, 3)])
def test_tier_s_matches_tier_d(normalized, h, n, k):
    g = random_graph(n, h, p=0.05, seed=n + h, weights="uniform")
    W = g.dense()
    dense = fairsc.fairsc_dense(W, g.groups, h, k, normalized, extra=1)
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, h, normalized)
    assert np.isclose(op.sigma, dense.sigma, rtol=1e-14)
    # operator: matrix-free formula vs dense L^sigma (Eq. asigma)
    A, _ = fairsc.deflated_operator(W, g.groups, h, normalized)
    w = np.random.default_rng(1).standard_normal((n, 2))
    assert np.allclose(op.apply(w), A @ w, atol=1e-12 * op.sigma)
    res = sfairsc_cpu.sfairsc_arpack(op, k, tol=1e-13, seed=3)
    assert np.allclose(res.evals[:k], dense.evals[:k], atol=1e-10 * op.sigma)
    if dense.gap > 1e-4 * op.sigma:
        assert subspace_sin(res.X, dense.X) < 1e-7


def test_tier_s_config1_against_tier_d():
    g, cfg = baseline_config(1)
    W = g.dense()
    k = cfg["k_eig"]
    dense = fairsc.fairsc_dense(W, g.groups, g.h, k, cfg["normalized"])
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, cfg["normalized"])
    res = sfairsc_cpu.sfairsc_arpack(op, k, tol=1e-13, seed=1)
    assert np.allclose(res.evals[:k], dense.evals[:k], rtol=1e-10, atol=1e-12 * op.sigma)
    assert subspace_sin(res.X, dense.X) < 1e-7
    # sigma closed form for R1: ||L||_1 = 2 max_j d_j
    d = W.sum(1)
    assert op.sigma == pytest.approx(2 * d.max(), rel=1e-15)


def test_sigma_closed_form_normalized():
    g = random_graph(80, 3, p=0.1, seed=4)
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, 3, True)
    d = g.dense().sum(1)
    s = 1 / np.sqrt(d)
    expect = np.max(1 + s * (g.dense() @ s))  # ||L_n||_1 = max_j (1 + s_j (W s)_j)
    assert op.sigma == pytest.approx(expect, rel=1e-14)


# --- Philox (Random123 KAT) ----------------------------------------------------

def test_philox_known_answers():
    with open(os.path.join(GOLDEN, "philox_kat.json")) as f:
        kat = json.load(f)
    for v in kat["vectors"]:
        ctr = np.array([int(x, 16) for x in v["ctr"]], np.uint64)
        key = np.array([int(x, 16) for x in v["key"]], np.uint64)
        out = philox4x32_10(ctr, key)
        assert [int(x) for x in out] == [int(x, 16) for x in v["out"]]


def test_uniform_range_and_moments():
    u = uniform(12345, np.arange(200000), 7, 8)
    assert u.min() >= 0 and u.max() < 1
    assert abs(u.mean() - 0.5) < 3e-3 and abs(u.var() - 1 / 12) < 2e-3


# --- k-means -------------------------------------------------------------------

def _brute_wcss(Y, K):
    best = np.inf
    for lab in itertools.product(range(K), repeat=len(Y)):
        lab = np.array(lab)
        if len(set(lab)) < K:
            continue
        w = sum(((Y[lab == c] - Y[lab == c].mean(0)) ** 2).sum() for c in range(K))
        best = min(best, w)
    return best


@pytest.mark.parametrize("seed,n,K", [(1, 8, 2), (2, 9, 3), (3, 10, 3)])
def test_kmeans_vs_bruteforce(seed, n, K):
    rng = np.random.default_rng(seed)
    Y = rng.standard_normal((n, 2))
    res = kmeans(Y, K, seed=seed)
    # Lloyd fixed point: centroids are means, each point at its nearest centroid
    for c in range(K):
        assert np.allclose(res.centroids[c], Y[res.labels == c].mean(0))
    dist = ((Y[:, None, :] - res.centroids[None]) ** 2).sum(-1)
    assert np.all(dist[np.arange(n), res.labels] <= dist.min(1) + 1e-15)
    bw = _brute_wcss(Y, K)
    assert res.wcss >= bw - 1e-12
    assert res.wcss == pytest.approx(bw, rel=1e-9)  # 10 k-means++ restarts find it here


def test_kmeans_blobs_and_seeding():
    rng = np.random.default_rng(0)
    centers = np.array([[0, 0], [10, 0], [0, 10], [10, 10]], float)
    truth = np.repeat(np.arange(4), 50)
    Y = centers[truth] + 0.1 * rng.standard_normal((200, 2))
    res = kmeans(Y, 4, seed=99)
    assert ari(res.labels, truth) == 1.0
    idx = kmeanspp_seed(Y, 4, 99, 0)
    assert idx[0] == int(np.floor(uniform(99, [0], 0, 8)[0] * 200))
    assert len(set(truth[idx])) == 4  # D^2 seeding lands in distinct blobs here


# --- metrics -------------------------------------------------------------------

def test_ari_matches_sklearn():
    rng = np.random.default_rng(5)
    for _ in range(10):
        a = rng.integers(0, 5, 300)
        b = np.where(rng.random(300) < 0.7, a, rng.integers(0, 5, 300))
        assert ari(a, b) == pytest.approx(adjusted_rand_score(a, b), abs=1e-12)


def test_balance_example_b2_and_hungarian():
    with open(os.path.join(GOLDEN, "example_b2.json")) as f:
        g = json.load(f)
    groups = np.array([0 if a == 1 else 1 for a in g["g1"]])
    labels = np.array(g["H_T"]).T.argmax(1)
    assert np.allclose(balance(labels, groups, 3, 2), 1.0)  # fair clustering: max balance
    perm = np.array([2, 0, 1])
    other = perm[labels]
    m = hungarian_match(labels, other, 3)
    assert np.array_equal(m[other], labels)


def test_error_rate_definition():
    """Eq. err: (1/n) min_J ||H^ J - H||_F^2 — brute force over all
    k! permutations on small cases, and the closed values 0 and 2/n."""
    import itertools
    from oracle.metrics import error_rate
    rng = np.random.default_rng(0)
    for trial in range(20):
        n, k = 12, 3
        t = rng.integers(0, k, n)
        l = rng.integers(0, k, n)
        H = np.eye(k)[t]
        Hh = np.eye(k)[l]
        best = min(np.sum((Hh @ np.eye(k)[list(p)] - H) ** 2) for p in itertools.permutations(range(k))) / n
        assert error_rate(t, l, k) == pytest.approx(best)
    t = np.array([0, 0, 1, 1, 2, 2])
    assert error_rate(t, (t + 1) % 3, 3) == 0.0  # relabelled: no error
    l = t.copy()
    l[0] = 1
    assert error_rate(t, l, 3) == pytest.approx(2.0 / 6)
