"""Pins of the oracle's comparison metrics and k-means branches (CPU, `-m "not gpu"`).

* `subspace_sin` — the checker of the north star's <= 1e-6 angle contract (reading
  R9): closed-form principal angles of constructed subspaces (down to 1e-8, where an
  acos-of-cosines form returns 0), scipy's independent `subspace_angles`, basis
  invariance, orthogonal and identical spans.
* `balance` (Eq. bal) — hand-computed count matrices whose answers are not 1,
  and the upper bound Eq. bal-upper with equality for a fair clustering.
* the R16 k-means' tie rule and empty-cluster re-seed, on constructed inputs whose
  outcome was traced by hand.
"""
import math

import numpy as np
import pytest
import scipy.linalg as sla

from oracle import kmeans as km
from oracle.metrics import balance, count_matrix, subspace_sin


def _rotated_pair(n, thetas, seed):
    """span(Xa) = U[:, :k]; span(Xb) = U [cos Θ; sin Θ; 0]: principal angles = thetas exactly."""
    k = len(thetas)
    U, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, n)))
    E = np.zeros((n, k))
    E[np.arange(k), np.arange(k)] = np.cos(thetas)
    E[k + np.arange(k), np.arange(k)] = np.sin(thetas)
    return U[:, :k], U @ E


@pytest.mark.parametrize("theta", [1e-8, 3e-7, 1e-4, 0.3, 1.2])
def test_subspace_sin_single_angle_closed_form(theta):
    # exact in floating point when the spans are coordinate planes
    Xa = np.zeros((5, 1))
    Xa[0, 0] = 1.0
    Xb = np.zeros((5, 1))
    Xb[0, 0], Xb[1, 0] = math.cos(theta), math.sin(theta)
    assert subspace_sin(Xa, Xb) == pytest.approx(math.sin(theta), rel=1e-12)
    # the same angle inside a random rotation of R^40
    Xa, Xb = _rotated_pair(40, np.array([theta]), seed=1)
    assert abs(subspace_sin(Xa, Xb) - math.sin(theta)) <= 1e-14


def test_subspace_sin_is_the_largest_principal_angle():
    thetas = np.array([2e-9, 5e-7, 1e-3, 0.2])
    Xa, Xb = _rotated_pair(60, thetas, seed=2)
    s = subspace_sin(Xa, Xb)
    assert abs(s - math.sin(0.2)) <= 1e-14
    # scipy's independent routine (SVD-based, with its own small-angle branch)
    assert abs(s - math.sin(np.max(sla.subspace_angles(Xa, Xb)))) <= 1e-12
    # only the small angles: the largest is 5e-7 (the contract's regime)
    Xa, Xb = _rotated_pair(60, thetas[:2], seed=3)
    assert abs(subspace_sin(Xa, Xb) - math.sin(5e-7)) <= 1e-14


def test_subspace_sin_basis_invariance_and_extremes():
    rng = np.random.default_rng(4)
    Xa, Xb = _rotated_pair(30, np.array([1e-6, 2e-6, 4e-6]), seed=5)
    G = rng.standard_normal((3, 3)) + 3 * np.eye(3)  # any basis of the same span
    assert abs(subspace_sin(Xa @ G, Xb) - subspace_sin(Xa, Xb)) <= 1e-14
    assert abs(subspace_sin(Xa, Xb @ G) - math.sin(4e-6)) <= 1e-14
    assert subspace_sin(Xa, Xa @ G) <= 1e-15  # identical spans
    I = np.eye(6)
    assert subspace_sin(I[:, :2], I[:, 2:4]) == pytest.approx(1.0, abs=1e-15)  # orthogonal spans
    assert subspace_sin(I[:, :2], I[:, 1:3]) == pytest.approx(1.0, abs=1e-15)  # one shared direction


def _labels_groups(M):
    """labels/groups realising the h x k count matrix M (m_sl = |V_s ∩ C_l|)."""
    lab, grp = [], []
    for s in range(M.shape[0]):
        for l in range(M.shape[1]):
            lab += [l] * int(M[s, l])
            grp += [s] * int(M[s, l])
    perm = np.random.default_rng(0).permutation(len(lab))
    return np.array(lab)[perm], np.array(grp)[perm]


def test_balance_hand_computed():
    # h = 2, k = 3: cluster 0 has (2, 4) -> 2/4; cluster 1 (3, 1) -> 1/3; cluster 2 (0, 5) -> 0
    M = np.array([[2, 3, 0], [4, 1, 5]])
    lab, grp = _labels_groups(M)
    assert np.array_equal(count_matrix(lab, grp, 3, 2), M)
    b = balance(lab, grp, 3, 2)
    assert b[0] == 0.5 and b[1] == pytest.approx(1 / 3, abs=0) and b[2] == 0.0
    assert b.mean() == pytest.approx((0.5 + 1 / 3) / 3, rel=1e-15)  # Average_Balance (Eq. avebal)
    # h = 3: (2, 3, 6) -> min over ordered pairs s != s' = 2/6; (5, 5, 5) -> 1; (7, 2, 4) -> 2/7
    M = np.array([[2, 5, 7], [3, 5, 2], [6, 5, 4]])
    lab, grp = _labels_groups(M)
    b = balance(lab, grp, 3, 3)
    assert b[0] == pytest.approx(1 / 3, abs=0) and b[1] == 1.0 and b[2] == pytest.approx(2 / 7, abs=0)


def test_balance_upper_bound_and_fair_equality():
    """Eq. bal-upper: min_l Balance(C_l) <= min_{s != s'} |V_s| / |V_s'|, with
    equality when every cluster holds the groups in the global proportions (Eq. gfair-equiv)."""
    rng = np.random.default_rng(7)
    for _ in range(50):
        h, k = rng.integers(2, 5), rng.integers(1, 6)
        n = 200
        grp = rng.integers(0, h, n)
        lab = rng.integers(0, k, n)
        sizes = np.bincount(grp, minlength=h)
        if sizes.min() == 0:
            continue
        assert balance(lab, grp, k, h).min() <= sizes.min() / sizes.max() + 1e-15
    # fair: group proportions (1 : 2 : 3) in every cluster
    M = np.array([[2, 3, 1], [4, 6, 2], [6, 9, 3]])
    lab, grp = _labels_groups(M)
    b = balance(lab, grp, 3, 3)
    assert np.allclose(b, 1 / 3, rtol=0, atol=1e-15)


def test_kmeans_ties_go_to_the_lowest_index():
    Y = np.array([[0.0], [2.0], [1.0]])
    lab, _ = km._assign(Y, np.array([[0.0], [2.0]]))
    assert lab.tolist() == [0, 1, 0]  # point 1 is equidistant: lower index
    # through Lloyd: with ties to the higher index the answer would be [0, 1, 1] (means 0 and 1.5)
    lab, mu, wcss = km.lloyd(Y, np.array([[0.0], [2.0]]))
    assert lab.tolist() == [0, 1, 0] and mu.ravel().tolist() == [0.5, 2.0] and wcss == 0.5


def test_kmeans_empty_cluster_reseed_at_farthest_point():
    """Hand trace: Y = (0, 1, 10, 13), mu0 = (0.5, 100, 11.5).  Cluster 1 starts empty;
    the distances to the assigned centroids are (0.25, 0.25, 2.25, 2.25), the first
    farthest point is Y[2] = 10, so mu1 = 10; then labels (0, 0, 1, 2), stable."""
    Y = np.array([[0.0], [1.0], [10.0], [13.0]])
    lab, mu, wcss = km.lloyd(Y, np.array([[0.5], [100.0], [11.5]]))
    assert lab.tolist() == [0, 0, 1, 2]
    assert mu.ravel().tolist() == [0.5, 10.0, 13.0]
    assert wcss == 0.5
    # two empty clusters: re-seeded in increasing index at distinct points (each point used once)
    Y = np.array([[0.0], [4.0], [5.0], [9.0]])
    lab, mu, wcss = km.lloyd(Y, np.array([[4.5], [100.0], [200.0]]))
    # assigned distances to 4.5: (20.25, 0.25, 0.25, 20.25) -> cluster 1 at Y[0] = 0, cluster 2 at Y[3] = 9
    assert lab.tolist() == [1, 0, 0, 2]
    assert mu.ravel().tolist() == [4.5, 0.0, 9.0]


def test_kmeanspp_degenerate_total_zero_branch():
    """All points identical: the D^2 weights vanish and the seeding falls back to
    floor(u n) (R16); every restart then has WCSS 0 and k-means returns one cluster's
    worth of points in cluster 0 (ties to the lowest index)."""
    Y = np.ones((7, 2))
    idx = km.kmeanspp_seed(Y, 3, seed=11, r=0)
    assert idx.min() >= 0 and idx.max() < 7
    res = km.kmeans(Y, 3, seed=11, n_restarts=2)
    assert res.wcss == 0.0 and np.all(res.labels == 0)
