"""§8(f) N2 on the GPU: thick-restart Lanczos on the Chebyshev filter -p(L^sigma) (opts.filter_degree,
DESIGN.md §10a; every kernel of the filtered solve is still an SpMV or a
vector pass).  Parity against the dense oracle (Alg. 2) with the same bars as the
unfiltered solvers (R6 eigenvalues, R8 subspaces, residual <= 1e-9 sigma, C^T X = 0), the
automatic and a fixed cut, odd and even degrees, h > 16 (the extra group-sum passes), breakdowns
on the planted cliques, and the option errors.
"""
import numpy as np
import pytest

from oracle import fairsc
from oracle.metrics import subspace_sin
from synth import baseline_config, planted_cliques, random_graph

pytestmark = pytest.mark.gpu


def _ctx(lib, g, k, normalized, **kw):
    return lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, g.groups.astype(np.int32), k, normalized,
                                      h=g.h, **kw)


def _check(lib, g, k, normalized, dense, tol=1e-10, **kw):
    ctx = _ctx(lib, g, k, normalized, **kw)
    ev, Xt, st = lib.sfairsc_eigs(ctx, k, tol)
    ctx.close()
    X = Xt.T
    sigma = st["sigma"]
    assert st["converged"] == 1
    assert st["max_resid_rel"] <= 1e-9
    assert 0.0 < st["filter_cut"] < sigma
    ref = dense.evals[:k]
    assert np.all(np.abs(ev - ref) <= 1e-8 * np.abs(ref) + 1e-12 * sigma), (ev, ref)
    assert np.all(np.diff(ev) >= 0)
    assert np.abs(X.T @ X - np.eye(k)).max() <= 1e-12
    C = fairsc.constraint_matrix(g.dense(), g.groups, g.h, normalized)
    assert np.linalg.norm(C.T @ X) <= 1e-10 * np.linalg.norm(X)
    if dense.gap > 0:
        bound = 2 * (st["max_resid_rel"] * sigma * np.sqrt(k) + 1e-12 * sigma) / dense.gap
        assert subspace_sin(X, dense.X) <= max(1e-6, bound)
    return ev, X, st


@pytest.mark.parametrize("deg", [2, 3, 5])
@pytest.mark.parametrize("n,h,normalized,k,seed", [(600, 2, True, 5, 1), (1031, 5, False, 8, 2),
                                                   (1500, 20, True, 6, 3)])
def test_filtered_eigs_match_dense_oracle(gpu_lib, n, h, normalized, k, seed, deg):
    g = random_graph(n, h, p=min(0.5, 8.0 / n), seed=seed, weights="uniform")
    dense = fairsc.fairsc_dense(g.dense(), g.groups, h, k, normalized)
    _check(gpu_lib, g, k, normalized, dense, filter_degree=deg)


def test_filtered_config1_and_fixed_cut(gpu_lib):
    """Config 1 (P:1565 shift) with the automatic cut, then with a fixed cut a between lambda_k and
    lambda_{k+4} of the oracle (the filter's wanted part is everything below a)."""
    g, cfg = baseline_config(1)
    k = cfg["k_eig"]
    dense = fairsc.fairsc_dense(g.dense(), g.groups, g.h, k + 6, cfg["normalized"])
    d6 = fairsc.fairsc_dense(g.dense(), g.groups, g.h, k, cfg["normalized"])
    _check(gpu_lib, g, k, cfg["normalized"], d6, tol=cfg["tol"], filter_degree=3)
    cut = 0.5 * (dense.evals[k] + dense.evals[k + 3])
    ev, X, st = _check(gpu_lib, g, k, cfg["normalized"], d6, tol=cfg["tol"], filter_degree=4, filter_cut=cut)
    assert st["filter_cut"] == cut


def test_filtered_unit_weights_unnormalized(gpu_lib):
    g = random_graph(2500, 4, p=0.004, seed=11, weights="unit")
    dense = fairsc.fairsc_dense(g.dense(), g.groups, g.h, 7, False)
    _check(gpu_lib, g, 7, False, dense, filter_degree=2)


@pytest.mark.parametrize("normalized", [False, True])
def test_filtered_planted_cliques_breakdown(gpu_lib, normalized):
    """Disconnected planted graph (spectrum {0^k, ...}, eigenspace span{1_{C_l}}): invariant subspaces
    are hit inside the filtered Krylov space too."""
    k, m, h = 4, 6, 3
    g = planted_cliques(k, m, h, seed=7)
    ctx = _ctx(gpu_lib, g, k, normalized, filter_degree=3)
    ev, Xt, st = gpu_lib.sfairsc_eigs(ctx, k, 1e-10)
    ctx.close()
    assert st["converged"] == 1 and st["max_resid_rel"] <= 1e-9
    assert np.abs(ev).max() <= 1e-12 * st["sigma"]
    d = np.diff(g.row_ptr).astype(float)
    E = np.zeros((g.n, k))
    E[np.arange(g.n), g.clusters] = 1.0
    if normalized:
        E *= np.sqrt(d)[:, None]
    assert subspace_sin(Xt.T, E) <= 1e-8


def test_filtered_matches_unfiltered_and_counts_applies(gpu_lib):
    """Same eigenpairs as the default solver; applies count every L^sigma application (d per step)."""
    g = random_graph(3000, 3, p=10.0 / 3000, seed=21, weights="uniform")
    k = 10
    c0 = _ctx(gpu_lib, g, k, True)
    ev0, X0, st0 = gpu_lib.sfairsc_eigs(c0, k, 1e-10)
    c0.close()
    c3 = _ctx(gpu_lib, g, k, True, filter_degree=3)
    ev3, X3, st3 = gpu_lib.sfairsc_eigs(c3, k, 1e-10)
    c3.close()
    assert np.all(np.abs(ev3 - ev0) <= 1e-9 * np.abs(ev0) + 1e-12 * st0["sigma"])
    assert st3["applies"] >= 3 * (st3["steps"] - st3["basis_size"]) + k
    assert st0["filter_cut"] == 0.0


def test_filter_option_errors(gpu_lib):
    g = random_graph(600, 3, p=0.02, seed=5, weights="uniform")
    for kw in ({"filter_degree": 3, "reorth": 2}, {"filter_degree": 3, "reorth": 3},
               {"filter_degree": 2, "block_size": 2}, {"filter_degree": 65}, {"filter_degree": -1},
               {"filter_degree": 2, "virtual_parts": 2}):
        with pytest.raises(gpu_lib.SfairscError) as e:
            _ctx(gpu_lib, g, 4, True, **kw)
        assert e.value.name == "E_INVALID_ARG", kw
    F = np.random.default_rng(0).standard_normal((g.n, 2))
    with pytest.raises(gpu_lib.SfairscError) as e:  # dense-F builds keep the single-sweep solver
        gpu_lib.sfairsc_build_operator_dense(g.row_ptr, g.col, g.val, F, 4, True, filter_degree=2)
    assert e.value.name == "E_INVALID_ARG"
    ctx = _ctx(gpu_lib, g, 4, True, filter_degree=2, filter_cut=1e9)  # a >= sigma: refused at eigs
    with pytest.raises(gpu_lib.SfairscError) as e:
        gpu_lib.sfairsc_eigs(ctx, 4, 1e-10)
    assert e.value.name == "E_INVALID_ARG"
    ctx.close()
    ctx = _ctx(gpu_lib, g, 4, True, filter_degree=1)  # degree 1 = no filter
    ev, _, st = gpu_lib.sfairsc_eigs(ctx, 4, 1e-10)
    assert st["filter_cut"] == 0.0
    ctx.close()
