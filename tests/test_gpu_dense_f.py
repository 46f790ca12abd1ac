"""GPU parity of the dense-constraint path (§8(f) N4, sfairsc_build_operator_dense):
general constraints C^T H = 0 with an explicit F (Experiment 4's random Laplacian with
a random F), against the explicit-F oracle (Alg. 2 with F as input)."""
import numpy as np
import pytest

from oracle import fairsc
from oracle.metrics import subspace_sin
from synth import baseline_config, random_laplacian

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("normalized", [False, True])
@pytest.mark.parametrize("n,r,k", [(1500, 5, 6), (2011, 12, 10), (700, 1, 4)])
def test_dense_F_vs_oracle(gpu_lib, normalized, n, r, k):
    g, F = random_laplacian(n, 8.0 / n, r, seed=n + r)
    W = g.dense()
    ref = fairsc.fairsc_dense_F(W, F, k, normalized)
    ctx = gpu_lib.sfairsc_build_operator_dense(g.row_ptr, g.col, g.val, F, k, normalized)
    ev, Xt, st = gpu_lib.sfairsc_eigs(ctx, k, 1e-10)
    # operator apply against the dense deflated operator (P:799-803 with P from F)
    A, sigma = fairsc.deflated_operator_F(W, F, normalized)
    x = np.random.default_rng(1).standard_normal((3, n))
    y = gpu_lib.sfairsc_apply(ctx, x)
    ctx.close()
    assert st["sigma"] == pytest.approx(sigma, rel=1e-14)
    assert np.abs(y - x @ A.T).max() <= 1e-12 * sigma * np.abs(x).max()
    X = Xt.T
    assert st["converged"] == 1 and st["max_resid_rel"] <= 1e-9
    assert np.all(np.abs(ev - ref.evals[:k]) <= 1e-8 * np.abs(ref.evals[:k]) + 1e-12 * sigma)
    assert np.abs(X.T @ X - np.eye(k)).max() <= 1e-12
    C = fairsc.constraint_matrix_F(W, F, normalized)
    assert np.linalg.norm(C.T @ X) <= 1e-10 * np.linalg.norm(C) * np.linalg.norm(X)
    bound = 2 * (st["max_resid_rel"] * sigma * np.sqrt(k) + 1e-12 * sigma) / ref.gap
    assert subspace_sin(X, ref.X) <= max(1e-6, bound)


def test_dense_F_with_group_F_equals_group_path(gpu_lib):
    """F = F_0(:, 1:h-1) of Lemma 2.1 through the dense path reproduces the group path."""
    g, cfg = baseline_config(1)
    F = fairsc.fairness_matrix(g.groups, g.h)
    k = cfg["k_eig"]
    a = gpu_lib.sfairsc_build_operator_dense(g.row_ptr, g.col, g.val, F, k, cfg["normalized"])
    ev_a, Xa, st_a = gpu_lib.sfairsc_eigs(a, k, cfg["tol"])
    a.close()
    b = gpu_lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, g.groups.astype(np.int32), k, cfg["normalized"],
                                       h=g.h)
    ev_b, Xb, st_b = gpu_lib.sfairsc_eigs(b, k, cfg["tol"])
    b.close()
    assert np.all(np.abs(ev_a - ev_b) <= 1e-8 * np.abs(ev_b) + 1e-12 * st_b["sigma"])
    assert subspace_sin(Xa.T, Xb.T) <= 1e-6


@pytest.mark.parametrize("normalized", [False, True])
@pytest.mark.parametrize("n,r,extra,k", [(900, 3, 2, 5), (1300, 12, 12, 8)])
def test_dense_F_rank_deficient_vs_oracle(gpu_lib, normalized, n, r, extra, k):
    """Reading R21: F with r independent columns plus `extra` linear combinations of them
    (24 columns of rank 12 in the second case: wider than the 16-wide projector rows) gives
    the projector of range(F) (P = I - C C^+), the same eigenpairs as the oracle's
    Alg. 2 with Z = null(F^T) at the numerical rank."""
    g, F0 = random_laplacian(n, 8.0 / n, r, seed=n + r)
    M = np.random.default_rng(r).standard_normal((r, extra))
    F = np.hstack([F0, F0 @ M])  # rank r, r + extra columns
    W = g.dense()
    ref = fairsc.fairsc_dense_F(W, F, k, normalized, rank_tol=1e-7)
    ref0 = fairsc.fairsc_dense_F(W, F0, k, normalized)  # range(F) = range(F0)
    assert np.allclose(ref.evals, ref0.evals, rtol=1e-10, atol=1e-12)
    ctx = gpu_lib.sfairsc_build_operator_dense(g.row_ptr, g.col, g.val, F, k, normalized)
    assert ctx.info()["constraint_rank"] == r
    ev, Xt, st = gpu_lib.sfairsc_eigs(ctx, k, 1e-10)
    ctx.close()
    sigma = st["sigma"]
    X = Xt.T
    assert st["converged"] == 1 and st["max_resid_rel"] <= 1e-9
    assert np.all(np.abs(ev - ref.evals[:k]) <= 1e-8 * np.abs(ref.evals[:k]) + 1e-12 * sigma)
    C = fairsc.constraint_matrix_F(W, F0, normalized)
    assert np.linalg.norm(C.T @ X) <= 1e-10 * np.linalg.norm(C) * np.linalg.norm(X)
    bound = 2 * (st["max_resid_rel"] * sigma * np.sqrt(k) + 1e-12 * sigma) / ref.gap
    assert subspace_sin(X, ref.X) <= max(1e-6, bound)


def test_dense_F_rank_limits(gpu_lib):
    g, F = random_laplacian(400, 0.05, 17, seed=1)
    with pytest.raises(gpu_lib.SfairscError) as e:  # numerical rank 17 > 16
        gpu_lib.sfairsc_build_operator_dense(g.row_ptr, g.col, g.val, F, 4, True)
    assert e.value.name == "E_INVALID_ARG"
    with pytest.raises(gpu_lib.SfairscError) as e:  # more than 64 columns
        gpu_lib.sfairsc_build_operator_dense(g.row_ptr, g.col, g.val, np.hstack([F[:, :1]] * 65), 4, True)
    assert e.value.name == "E_INVALID_ARG"
    # all-zero F: no constraint (rank 0), the plain spectral problem
    ctx = gpu_lib.sfairsc_build_operator_dense(g.row_ptr, g.col, g.val, np.zeros((g.n, 3)), 4, False)
    assert ctx.info()["constraint_rank"] == 0
    ctx.close()
