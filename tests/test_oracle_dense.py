"""Pins for the Tier D / Tier B oracle (CPU only).

Each test checks the oracle against something other than itself: the paper's
printed Example B.2, exhaustive enumeration, 50-digit brute force, a library
routine for the h = 1 special case, closed-form spectra (planted cliques,
expected-graph quotient), Prop. 3.1 / Eq. asigma and Ky Fan (Thm 2.2).
"""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla
from scipy.sparse.csgraph import laplacian as csgraph_laplacian

from conftest import GOLDEN
from oracle import brute, fairsc
from oracle.metrics import subspace_sin
from synth import planted_cliques, random_graph, random_laplacian


def _golden_b2():
    with open(os.path.join(GOLDEN, "example_b2.json")) as f:
        return json.load(f)


# --- Lemma 2.1 and Example B.2 ----------------------

def test_example_b2_FtH_zero():
    g = _golden_b2()
    groups = np.array([0 if a == 1 else 1 for a in g["g1"]])
    assert np.array_equal(np.array(g["g2"]), 1 - np.array(g["g1"]))
    H = np.array(g["H_T"], dtype=float).T
    F = fairsc.fairness_matrix(groups, g["h"])
    assert F.shape == (10, 1)
    assert np.all(F.T @ H == 0.0)  # exact: entries are +-1/2
    labels = H.argmax(1)
    assert brute.is_fair(labels, groups, g["h"], g["k"])
    # the printed block vector u = [(2,2),(2,2),(1,1)]
    for l, (u1, u2) in enumerate(g["u"]):
        assert np.sum((labels == l) & (groups == 0)) == u1
        assert np.sum((labels == l) & (groups == 1)) == u2


@pytest.mark.parametrize("h", [2, 3, 4])
def test_lemma21_rank_and_null(h):
    rng = np.random.default_rng(h)
    groups = np.concatenate([np.arange(h), rng.integers(0, h, 13)])
    n = len(groups)
    G = fairsc.group_indicator(groups, h)
    z = G.T @ np.ones(n) / n
    F0 = G - np.outer(np.ones(n), z)
    assert np.allclose(F0 @ np.ones(h), 0)  # F_0 1_h = 0
    assert np.linalg.matrix_rank(F0) == h - 1  # Lemma 2.1(i)
    F = fairsc.fairness_matrix(groups, h)
    assert np.linalg.matrix_rank(F) == h - 1
    assert np.allclose(F, F0[:, : h - 1])


@pytest.mark.parametrize("groups,k", [([0, 0, 1, 1, 0, 1], 2), ([0, 0, 1, 1, 0, 1], 3),
                                      ([0, 1, 2, 0, 1, 2], 2), ([0, 0, 0, 1, 1, 1, 0, 1], 2)])
def test_lemma21_exhaustive_fair_iff_FtH0(groups, k):
    """Lemma 2.1(ii): clustering fair (Def. 2.1) <=> F^T H = 0, every clustering."""
    groups = np.array(groups)
    h = groups.max() + 1
    F = fairsc.fairness_matrix(groups, h)
    n = len(groups)
    n_fair = 0
    for lab in brute.all_clusterings(n, k):
        H = np.zeros((n, k))
        H[np.arange(n), lab] = 1
        fair = brute.is_fair(lab, groups, h, k)
        n_fair += fair
        assert fair == bool(np.allclose(F.T @ H, 0, atol=1e-12))
    assert n_fair > 0


# --- brute force (Tier B) pins Tier D ----------------------------------------

@pytest.mark.parametrize("n,h,normalized,seed", [(6, 2, False, 1), (7, 2, True, 2), (8, 3, False, 3),
                                                 (9, 3, True, 4), (10, 2, True, 5), (12, 4, False, 6),
                                                 (11, 1, True, 7)])
def test_dense_matches_bruteforce(n, h, normalized, seed):
    g = random_graph(n, h, p=0.5, seed=seed, weights="uniform")
    W = g.dense()
    k = min(3, n - h + 1)
    res = fairsc.fairsc_dense(W, g.groups, h, k, normalized, extra=n)
    ev_b, X_b = brute.brute_fair_eig(W, list(g.groups), h, normalized)
    ev_b = np.array([float(x) for x in ev_b])
    assert len(res.evals) == n - h + 1
    assert np.max(np.abs(res.evals - ev_b)) <= 1e-13 * max(1.0, res.sigma)
    # subspace of the k smallest where separated by a gap
    if ev_b[k] - ev_b[k - 1] > 1e-6:
        Xb = np.array(X_b.tolist(), dtype=float)[:, :k]
        assert subspace_sin(res.X, Xb) < 1e-10


# --- h = 1 reduces to plain SC (Alg. 1) ----------------------------

@pytest.mark.parametrize("normalized", [False, True])
def test_h1_is_spectral_clustering(normalized):
    g = random_graph(60, 1, p=0.2, seed=11, weights="uniform")
    W = g.dense()
    res = fairsc.fairsc_dense(W, g.groups, 1, 5, normalized, extra=3)
    Lref = csgraph_laplacian(W, normed=normalized)  # library routine
    ev = sla.eigh(Lref, eigvals_only=True)[:8]
    assert np.allclose(res.evals, ev, atol=1e-12, rtol=0)


# --- planted disjoint cliques (P-closed-1) -----------------------

@pytest.mark.parametrize("normalized", [False, True])
def test_planted_cliques_closed_form(normalized):
    k, m, h = 3, 6, 3
    g = planted_cliques(k, m, h, seed=5)
    W = g.dense()
    res = fairsc.fairsc_dense(W, g.groups, h, k, normalized, extra=g.n)
    n = g.n
    expect_hi = m / (m - 1) if normalized else float(m)
    assert np.allclose(res.evals[:k], 0, atol=1e-12)
    assert np.allclose(res.evals[k:], expect_hi, atol=1e-12)
    assert len(res.evals) == n - h + 1
    # fair eigenspace = span{1_{C_l}} (normalized: span{D^{1/2} 1_{C_l}})
    d = W.sum(1)
    E = np.zeros((n, k))
    E[np.arange(n), g.clusters] = 1.0
    if normalized:
        E *= np.sqrt(d)[:, None]
    assert subspace_sin(res.X, E) < 1e-12


# --- expected-graph quotient (P-closed-2) ------------------------

def _quotient_spectrum(sizes, cell_group, Pc, h, normalized):
    """Closed form for W_bar with block-constant off-diagonal entries Pc[a,b]:
    within-cell eigenvalue dbar_c + p_cc (or 1 + p_cc/dbar_c), multiplicity
    |c|-1, plus the spectrum of the constrained (C x C) quotient."""
    s = np.asarray(sizes, float)
    C = len(s)
    dbar = np.array([sum((s[b] - (a == b)) * Pc[a, b] for b in range(C)) for a in range(C)])
    Aq = np.zeros((C, C))
    for a in range(C):
        for b in range(C):
            Aq[a, b] = ((a == b) * s[a] * dbar[a] - s[a] * (s[b] - (a == b)) * Pc[a, b]) / np.sqrt(s[a] * s[b])
    n = s.sum()
    z = np.array([s[cell_group == t].sum() / n for t in range(h)])
    Phi = np.zeros((C, h - 1))
    for c in range(C):
        for t in range(h - 1):
            Phi[c, t] = np.sqrt(s[c]) * ((cell_group[c] == t) - z[t])
    if normalized:
        Aq = Aq / np.sqrt(np.outer(dbar, dbar))
        Phi = Phi / np.sqrt(dbar)[:, None]
        within = 1 + np.diag(Pc) / dbar
    else:
        within = dbar + np.diag(Pc)
    N = sla.null_space(Phi.T)
    quot = np.linalg.eigvalsh(N.T @ Aq @ N)
    ev = list(quot)
    for c in range(C):
        ev += [within[c]] * int(s[c] - 1)
    return np.sort(ev)


@pytest.mark.parametrize("normalized", [False, True])
def test_expected_graph_quotient(normalized):
    rng = np.random.default_rng(3)
    k, h = 3, 2
    sizes = np.array([5, 4, 6, 3, 7, 5])  # cells c = cluster*h + group
    cell_group = np.arange(k * h) % h
    Pc = rng.uniform(0.05, 0.9, (k * h, k * h))
    Pc = 0.5 * (Pc + Pc.T)
    cell = np.repeat(np.arange(k * h), sizes)
    perm = rng.permutation(len(cell))
    cell = cell[perm]
    groups = cell_group[cell]
    W = Pc[cell[:, None], cell[None, :]]
    np.fill_diagonal(W, 0.0)
    res = fairsc.fairsc_dense(W, groups, h, 3, normalized, extra=len(cell))
    expect = _quotient_spectrum(sizes, cell_group, Pc, h, normalized)
    assert len(res.evals) == len(expect)
    assert np.max(np.abs(res.evals - expect)) < 1e-12 * max(1, expect.max())


# --- Prop. 3.1, Eq. asigma, Prop. 3.4, Ky Fan ----------------------------------

@pytest.mark.parametrize("normalized,h", [(False, 2), (True, 3), (True, 5)])
def test_prop31_deflated_spectrum(normalized, h):
    g = random_graph(40, h, p=0.25, seed=20 + h, weights="uniform")
    W = g.dense()
    lam_v = fairsc.variant_evals(W, g.groups, h, normalized)  # §3.2
    res = fairsc.fairsc_dense(W, g.groups, h, 4, normalized, extra=100)
    assert np.allclose(res.evals, lam_v, atol=1e-12)  # Alg. 2 == §3.2 variant
    A, sigma = fairsc.deflated_operator(W, g.groups, h, normalized)
    assert np.isclose(sigma, res.sigma)
    ev = np.linalg.eigvalsh(A)
    expect = np.sort(np.concatenate([lam_v, np.full(h - 1, sigma)]))
    assert np.allclose(ev, expect, atol=1e-12 * sigma)
    # Prop. 3.4 precondition holds with sigma = ||L||_1 (every lambda <= sigma)
    assert lam_v.max() <= sigma * (1 + 1e-14)
    # ||L^sigma||_2 = sigma exactly for h >= 2
    assert np.isclose(np.abs(ev).max(), sigma, rtol=1e-13)
    # matrix-free apply formula equals the dense operator
    w = np.random.default_rng(0).standard_normal((g.n, 3))
    assert np.allclose(fairsc.apply_deflated(W, g.groups, h, normalized, w), A @ w, atol=1e-12 * sigma)


@pytest.mark.parametrize("normalized", [False, True])
def test_invariants_and_kyfan(normalized):
    h, k = 3, 4
    g = random_graph(50, h, p=0.2, seed=9, weights="uniform")
    W = g.dense()
    res = fairsc.fairsc_dense(W, g.groups, h, k, normalized)
    d = W.sum(1)
    F = fairsc.fairness_matrix(g.groups, h)
    assert np.abs(F.T @ res.H).max() < 1e-12  # F^T H = 0 (Eq. fairmath)
    if normalized:
        assert np.allclose(res.H.T @ (d[:, None] * res.H), np.eye(k), atol=1e-12)  # H^T D H = I
    else:
        assert np.allclose(res.H.T @ res.H, np.eye(k), atol=1e-12)
    assert np.allclose(res.X.T @ res.X, np.eye(k), atol=1e-12)
    # lambda_1 = 0 with eigenvector prop. to 1 (D^{1/2} 1): F^T 1 = 0
    assert abs(res.evals[0]) < 1e-12 * res.sigma
    one = np.sqrt(d) if normalized else np.ones(g.n)
    assert subspace_sin(res.X[:, :1], one[:, None]) < 1e-10
    # Ky Fan (Thm 2.2): tr(X^T A X) over feasible orthonormal X >= sum lambda_i
    A = fairsc.operator_laplacian(W, normalized)
    assert np.isclose(np.trace(res.X.T @ A @ res.X), res.evals[:k].sum(), atol=1e-12)
    C = fairsc.constraint_matrix(W, g.groups, h, normalized)
    V = fairsc.nullspace_basis(C)
    rng = np.random.default_rng(1)
    for _ in range(20):
        Y, _ = np.linalg.qr(rng.standard_normal((V.shape[1], k)))
        Xr = V @ Y
        assert np.trace(Xr.T @ A @ Xr) >= res.evals[:k].sum() - 1e-12


def test_validation_rejects_bad_inputs():
    g = random_graph(10, 2, p=0.5, seed=1)
    W = g.dense()
    bad = W.copy()
    bad[0, 1] += 1.0
    with pytest.raises(fairsc.OracleInputError):
        fairsc.fairsc_dense(bad, g.groups, 2, 2, False)
    bad = W.copy()
    bad[:, 0] = 0
    bad[0, :] = 0
    with pytest.raises(fairsc.OracleInputError):
        fairsc.fairsc_dense(bad, g.groups, 2, 2, False)
    with pytest.raises(fairsc.OracleInputError):
        fairsc.fairsc_dense(W, np.zeros(10, int), 2, 2, False)


# --- explicit constraint matrix F (§8(f) N4; Experiment 4's random F) -------------

@pytest.mark.parametrize("normalized", [False, True])
@pytest.mark.parametrize("n,r,seed", [(9, 2, 1), (11, 3, 2), (12, 1, 3)])
def test_dense_F_matches_bruteforce(normalized, n, r, seed):
    """Alg. 2 with an explicit random F equals the 50-digit brute force (QR null space + Jacobi)."""
    from oracle import brute
    from synth import random_laplacian
    g, F = random_laplacian(n, 0.6, r, seed=seed)
    W = g.dense()
    res = fairsc.fairsc_dense_F(W, F, n - r - 1, normalized, extra=0)
    ev, _ = brute.brute_fair_eig(W, None, 1, normalized, F=F)
    ref = np.array([float(x) for x in ev])[: n - r - 1]
    assert np.allclose(res.evals, ref, atol=1e-13 * max(1.0, np.abs(ref).max()))


@pytest.mark.parametrize("normalized", [False, True])
def test_dense_F_range_invariance_variant_and_prop31(normalized):
    """Only range(F) matters (F and F R agree); Alg. 2 = the §3.2 variant;
    spec L^sigma = spec L^v U {sigma}^r (Prop. 3.1, Eq. asigma) for an explicit F."""
    from synth import random_laplacian
    n, r, k = 60, 4, 8
    g, F = random_laplacian(n, 0.15, r, seed=4)
    W = g.dense()
    a = fairsc.fairsc_dense_F(W, F, k, normalized)
    R = np.random.default_rng(1).standard_normal((r, r)) + 3 * np.eye(r)
    b = fairsc.fairsc_dense_F(W, F @ R, k, normalized)
    assert np.allclose(a.evals, b.evals, atol=1e-12)
    var = fairsc.variant_evals_F(W, F, normalized)
    assert np.allclose(a.evals, var[: len(a.evals)], atol=1e-12)
    A, sigma = fairsc.deflated_operator_F(W, F, normalized)
    full = np.sort(np.concatenate([var, np.full(r, sigma)]))
    assert np.allclose(np.linalg.eigvalsh(A), full, atol=1e-11 * sigma)
    # X is fair: C^T X = 0, and orthonormal in the comparison frame
    C = fairsc.constraint_matrix_F(W, F, normalized)
    assert np.linalg.norm(C.T @ a.X) <= 1e-12 * np.linalg.norm(C) * np.linalg.norm(a.X)
    assert np.allclose(a.X.T @ a.X, np.eye(k), atol=1e-12)


def test_dense_F_tier_s_matches_tier_d():
    """Tier S (the paper's matrix-free operator with the normal-equations projector) with an
    explicit F equals Tier D."""
    from oracle import sfairsc_cpu
    from synth import random_laplacian
    g, F = random_laplacian(400, 0.03, 5, seed=6)
    for normalized in (False, True):
        d = fairsc.fairsc_dense_F(g.dense(), F, 6, normalized)
        op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, 1, normalized, F=F)
        s = sfairsc_cpu.sfairsc_arpack(op, 6, tol=1e-13, seed=1)
        assert np.allclose(s.evals[:6], d.evals[:6], atol=1e-10 * op.sigma)


@pytest.mark.parametrize("normalized", [False, True])
def test_rank_deficient_F_null_space_reading_R21(normalized):
    """Reading R21 (rank-deficient F, §8(f) N4): Z = null(F^T) at the numerical rank.  Appending
    linear combinations of the columns leaves range(F), hence null(F^T) and every fair eigenpair,
    unchanged; without rank_tol the oracle refuses (Lemma 2.1(i) check)."""
    g, F0 = random_laplacian(60, 0.2, 3, seed=2)
    W = g.dense()
    F = np.hstack([F0, F0 @ np.array([[1.0, -2.0], [0.5, 0.0], [0.0, 3.0]])])
    a = fairsc.fairsc_dense_F(W, F, 6, normalized, rank_tol=1e-7)
    b = fairsc.fairsc_dense_F(W, F0, 6, normalized)
    assert np.allclose(a.evals, b.evals, rtol=1e-11, atol=1e-12)
    assert subspace_sin(a.X, b.X) <= 1e-9
    Z = fairsc.nullspace_basis(F, 1e-7)
    assert Z.shape == (60, 57) and np.abs(F.T @ Z).max() <= 1e-12 * np.abs(F).max()
    with pytest.raises(fairsc.OracleInputError):
        fairsc.fairsc_dense_F(W, F, 6, normalized)
