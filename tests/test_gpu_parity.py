"""GPU parity: the CUDA path (through the C ABI) against the oracle on the
same seeded inputs.

Tolerances:
  * operator pieces (SpMV, P, L^sigma): fp64 with a different summation
    order -> |y - y_ref|_inf <= 1e-13 * sigma * |x|_inf (n <= 1e5 terms of a
    row are <= deg ~ 1e2; 1e-13 is ~500 ulps of slack);
  * eigenvalues: |d lambda_i| <= 1e-8 |lambda_i| + 1e-12 sigma (north star
    relative 1e-8, floor for lambda_1 = 0, reading R6);
  * subspace: sin(angle) <= 1e-6 when the Davis-Kahan bound
    (|R_gpu| + |R_oracle|) / gap permits (reading R8);
  * residual |L^sigma x - lambda x| / sigma <= 1e-9 (north star).
"""
import numpy as np
import pytest

from oracle import fairsc, sfairsc_cpu
from oracle.metrics import subspace_sin
from synth import baseline_config, planted_cliques, random_graph

pytestmark = pytest.mark.gpu


def _ctx(lib, g, k, normalized, **kw):
    return lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, g.groups.astype(np.int32), k, normalized,
                                      h=g.h, **kw)


def _graphs():
    # (graph, normalized) — ragged sizes (not multiples of 256), h = 1, 2, 5, 20 (> 16 fused groups)
    return [
        (random_graph(37, 2, p=0.3, seed=1), False),
        (random_graph(300, 3, p=0.05, seed=2), True),
        (random_graph(1031, 5, p=0.01, seed=3), False),
        (random_graph(777, 1, p=0.02, seed=4), True),
        (random_graph(2000, 20, p=0.01, seed=5), True),
        (random_graph(2000, 20, p=0.01, seed=6), False),
    ]


@pytest.mark.parametrize("idx", range(6))
def test_operator_pieces_match_oracle(gpu_lib, idx):
    g, normalized = _graphs()[idx]
    lib = gpu_lib
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, normalized)
    ctx = _ctx(lib, g, 1, normalized)
    info = ctx.info()
    assert info["sigma"] == pytest.approx(op.sigma, rel=1e-14)
    rng = np.random.default_rng(idx)
    X = rng.standard_normal((3, g.n))
    tol = 1e-13 * op.sigma * np.abs(X).max()
    # bare Laplacian (A5)
    y = lib.sfairsc_laplacian(ctx, np.ascontiguousarray(X[0]))
    assert np.abs(y - op.Ln @ X[0]).max() <= tol
    # projector (A4): P x by the factored form vs the normal-equations form
    Y = lib.sfairsc_project(ctx, X)
    ref = np.stack([op.P(x) for x in X])
    assert np.abs(Y - ref).max() <= 1e-13 * np.abs(X).max() * 10
    # full operator L^sigma
    Y = lib.sfairsc_apply(ctx, X)
    ref = np.stack([op.apply(x) for x in X])
    assert np.abs(Y - ref).max() <= tol
    ctx.close()


@pytest.mark.parametrize("n,h,p,normalized,colblk", [(37, 2, 0.3, False, None), (1031, 5, 0.01, True, None),
                                                     (2000, 20, 0.01, False, None), (3001, 3, 0.004, True, "0.01"),
                                                     (2500, 4, 0.006, False, "0.01")])
def test_unit_weight_spmv_matches_oracle(gpu_lib, monkeypatch, n, h, p, normalized, colblk):
    """Unit-weight graphs take the pattern-only SpMV (no value stream; normalized, when
    column-blocked: gathers of s o x, row sums scaled by s_i).  L x and L^sigma x
    against the oracle; the last two cases run column-blocked."""
    if colblk:
        monkeypatch.setenv("SFAIRSC_COLBLK_MB", colblk)
    g = random_graph(n, h, p=p, seed=n, weights="unit")
    lib = gpu_lib
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, normalized)
    ctx = _ctx(lib, g, 1, normalized)
    assert ctx.info()["unit_weights"] == 1
    x = np.random.default_rng(n).standard_normal(g.n)
    tol = 1e-13 * op.sigma * np.abs(x).max()
    assert np.abs(lib.sfairsc_laplacian(ctx, x) - op.Ln @ x).max() <= tol
    assert np.abs(lib.sfairsc_apply(ctx, x) - op.apply(x)).max() <= tol
    ctx.close()
    gw = random_graph(n, h, p=p, seed=n, weights="uniform")
    ctx = _ctx(lib, gw, 1, normalized)
    assert ctx.info()["unit_weights"] == 0
    ctx.close()


@pytest.mark.parametrize("normalized", [False, True])
def test_unit_pattern_eigs_match_scaled_weights(gpu_lib, normalized):
    """The same graph as unit weights (pattern-only SpMV) and with every weight 2
    (value-streaming SpMV): L_n is invariant under W -> 2W, L = D - W doubles
    (P:123), so the eigenvalues agree (normalized) or double (unnormalized)
    and the eigenvector subspaces coincide."""
    g = random_graph(3000, 4, p=0.004, seed=11, weights="unit")
    lib = gpu_lib
    k = 6
    ctx = _ctx(lib, g, k, normalized)
    assert ctx.info()["unit_weights"] == 1
    ev1, X1, st1 = lib.sfairsc_eigs(ctx, k, 1e-10)
    ctx.close()
    ctx = lib.sfairsc_build_operator(g.row_ptr, g.col, 2.0 * g.val, g.groups.astype(np.int32), k, normalized, h=g.h)
    assert ctx.info()["unit_weights"] == 0
    ev2, X2, st2 = lib.sfairsc_eigs(ctx, k, 1e-10)
    ctx.close()
    scale = 1.0 if normalized else 2.0
    assert np.allclose(ev2[1:], scale * ev1[1:], rtol=1e-8, atol=0)
    assert abs(ev1[0]) <= 1e-10 * st1["sigma"] and abs(ev2[0]) <= 1e-10 * st2["sigma"]
    assert subspace_sin(X1.T, X2.T) <= 1e-6


def test_operator_device_tensors(gpu_lib):
    import torch
    g, _ = baseline_config(1)
    lib = gpu_lib
    d = torch.device("cuda:0")
    ctx = lib.sfairsc_build_operator(torch.from_numpy(g.row_ptr).to(d), torch.from_numpy(g.col).to(d),
                                     torch.from_numpy(g.val).to(d), torch.from_numpy(g.groups.astype(np.int32)).to(d),
                                     5, False)
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, False)
    x = torch.randn(2, g.n, dtype=torch.float64, device=d)
    y = lib.sfairsc_apply(ctx, x)
    ref = np.stack([op.apply(v) for v in x.cpu().numpy()])
    assert np.abs(y.cpu().numpy() - ref).max() <= 1e-13 * op.sigma * x.abs().max().item()
    ctx.close()


# eigensolver variants of the C ABI (sfairsc_opts): the default (paired steps: two Lanczos steps per
# basis sweep, reorth 3, where allowed), one lagged step per sweep (reorth 2), three-sweep CGS2, and block
# Lanczos with b = 2, and the Chebyshev-filtered CGS2 solver of degree 3 (§8(f) N2)
SOLVERS = {"default": {}, "lagged1": {"reorth": 2}, "cgs2": {"reorth": 1}, "block2": {"block_size": 2},
           "cheb3": {"filter_degree": 3}}


def _check_eigs(lib, g, k, normalized, tol, dense=None, ref_evals=None, ref_X=None, gap=None, **kw):
    ctx = _ctx(lib, g, k, normalized, **kw)
    ev, Xt, st = lib.sfairsc_eigs(ctx, k, tol)
    X = Xt.T
    sigma = st["sigma"]
    assert st["converged"] == 1
    assert st["max_resid_rel"] <= 1e-9
    if dense is not None:
        ref_evals, ref_X, gap = dense.evals[:k], dense.X, dense.gap
    assert np.all(np.abs(ev - ref_evals) <= 1e-8 * np.abs(ref_evals) + 1e-12 * sigma), (ev, ref_evals)
    # orthonormal, fair (C^T X = 0)
    assert np.abs(X.T @ X - np.eye(k)).max() <= 1e-12
    W = g.to_scipy()
    C = fairsc.constraint_matrix(W.toarray(), g.groups, g.h, normalized) if g.n <= 3000 else None
    if C is not None:
        assert np.linalg.norm(C.T @ X) <= 1e-10 * np.linalg.norm(X)
    if ref_X is not None and gap is not None and gap > 0:
        bound = 2 * (st["max_resid_rel"] * sigma * np.sqrt(k) + 1e-12 * sigma) / gap
        sin = subspace_sin(X, ref_X)
        assert sin <= max(1e-6, bound), (sin, bound)
        if bound <= 1e-7:
            assert sin <= 1e-6
    ctx.close()
    return ev, X, st


@pytest.mark.parametrize("solver", list(SOLVERS))
def test_eigs_config1_vs_dense_fairsc(gpu_lib, solver):
    g, cfg = baseline_config(1)
    dense = fairsc.fairsc_dense(g.dense(), g.groups, g.h, cfg["k_eig"], cfg["normalized"])
    _check_eigs(gpu_lib, g, cfg["k_eig"], cfg["normalized"], cfg["tol"], dense=dense, **SOLVERS[solver])


@pytest.mark.parametrize("n,h,normalized,k,seed", [(200, 2, True, 4, 1), (513, 5, False, 6, 2),
                                                   (400, 3, True, 8, 3), (300, 1, False, 5, 4),
                                                   (1500, 20, True, 5, 5)])
@pytest.mark.parametrize("solver", list(SOLVERS))
def test_eigs_random_vs_dense(gpu_lib, n, h, normalized, k, seed, solver):
    g = random_graph(n, h, p=min(0.5, 8.0 / n), seed=seed, weights="uniform")
    if SOLVERS[solver].get("reorth") == 2 and h > 16:  # the lagged solver's fused epilogues carry <= 16 groups
        with pytest.raises(gpu_lib.SfairscError) as e:
            _ctx(gpu_lib, g, k, normalized, **SOLVERS[solver])
        assert e.value.name == "E_INVALID_ARG"
        return
    dense = fairsc.fairsc_dense(g.dense(), g.groups, h, k, normalized)
    _check_eigs(gpu_lib, g, k, normalized, 1e-10, dense=dense, **SOLVERS[solver])


@pytest.mark.parametrize("solver", list(SOLVERS))
@pytest.mark.parametrize("normalized", [False, True])
def test_eigs_planted_cliques_closed_form(gpu_lib, normalized, solver):
    """Disconnected planted graph (P-closed-1): spec = {0^k, m or m/(m-1)},
    eigenspace span{1_{C_l}} (D^{1/2} 1_{C_l}).  Exercises Lanczos breakdown."""
    k, m, h = 4, 6, 3
    g = planted_cliques(k, m, h, seed=7)
    ev, X, st = _check_eigs(gpu_lib, g, k, normalized, 1e-10, ref_evals=np.zeros(k), **SOLVERS[solver])
    d = np.diff(g.row_ptr).astype(float)
    E = np.zeros((g.n, k))
    E[np.arange(g.n), g.clusters] = 1.0
    if normalized:
        E *= np.sqrt(d)[:, None]
    assert subspace_sin(X, E) <= 1e-8
    assert st["breakdowns"] >= 1


def test_eigs_h1_is_spectral_clustering(gpu_lib):
    g = random_graph(400, 1, p=0.03, seed=8)
    dense = fairsc.fairsc_dense(g.dense(), g.groups, 1, 6, True)
    _check_eigs(gpu_lib, g, 6, True, 1e-10, dense=dense)


def test_eigs_deterministic(gpu_lib):
    g, cfg = baseline_config(1)
    a = _check_eigs(gpu_lib, g, 5, False, 1e-10, dense=fairsc.fairsc_dense(g.dense(), g.groups, g.h, 5, False))
    b = _check_eigs(gpu_lib, g, 5, False, 1e-10, dense=fairsc.fairsc_dense(g.dense(), g.groups, g.h, 5, False))
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.fixture(scope="module")
def config2_ref():
    g, cfg = baseline_config(2)
    k = cfg["k_eig"]
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, True)
    return g, cfg, sfairsc_cpu.sfairsc_arpack(op, k, tol=1e-13, seed=2)


@pytest.mark.parametrize("solver", list(SOLVERS))
def test_eigs_config2_vs_tier_s(gpu_lib, config2_ref, solver):
    g, cfg, ref = config2_ref
    k = cfg["k_eig"]
    gap = ref.evals[k] - ref.evals[k - 1]
    _check_eigs(gpu_lib, g, k, True, cfg["tol"], ref_evals=ref.evals[:k], ref_X=ref.X, gap=gap, **SOLVERS[solver])


# --- error vocabulary ----------------------------------------------------------

def test_errors(gpu_lib):
    lib = gpu_lib
    g = random_graph(50, 2, p=0.2, seed=1)
    grp = g.groups.astype(np.int32)
    # asymmetric
    v = g.val.copy()
    v[0] += 1.0
    with pytest.raises(lib.SfairscError) as e:
        lib.sfairsc_build_operator(g.row_ptr, g.col, v, grp, 2, False)
    assert e.value.name == "E_ASYMMETRIC"
    # negative weight (symmetric)
    v = -g.val
    with pytest.raises(lib.SfairscError) as e:
        lib.sfairsc_build_operator(g.row_ptr, g.col, v, grp, 2, False)
    assert e.value.name == "E_NEGATIVE_WEIGHT"
    # empty group
    with pytest.raises(lib.SfairscError) as e:
        lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, np.zeros(50, np.int32), 2, False, h=2)
    assert e.value.name == "E_EMPTY_GROUP"
    # k too large
    with pytest.raises(lib.SfairscError) as e:
        lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, grp, 50, False)
    assert e.value.name == "E_K_TOO_LARGE"
    # isolated vertex: drop all edges of vertex 0 (both directions)
    import scipy.sparse as sp
    W = g.to_scipy().tolil()
    W[0, :] = 0
    W[:, 0] = 0
    W = sp.csr_matrix(W)
    W.eliminate_zeros()
    with pytest.raises(lib.SfairscError) as e:
        lib.sfairsc_build_operator(W.indptr.astype(np.int32), W.indices.astype(np.int32), W.data, grp, 2, False)
    assert e.value.name == "E_ISOLATED_VERTEX"
    # call order
    ctx = lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, grp, 2, False)
    with pytest.raises(lib.SfairscError) as e:
        lib.sfairsc_embed_kmeans(ctx, 1)
    assert e.value.name == "E_STATE"
    ctx.close()


# --- Alg. 3 step 4: k-means on H (reading R16) ---------------------------------

def _kmeans_parity(lib, g, k, normalized, tol, H_oracle, seed=2024):
    from oracle.kmeans import kmeans
    from oracle.metrics import ari, balance, hungarian_match
    ctx = _ctx(lib, g, k, normalized)
    lib.sfairsc_eigs(ctx, k, tol)
    lab_gpu, wcss_gpu = lib.sfairsc_embed_kmeans(ctx, seed)
    ctx.close()
    ref = kmeans(H_oracle, k, seed)
    a = ari(ref.labels, lab_gpu)
    assert a >= 0.99, a
    perm = hungarian_match(ref.labels, lab_gpu, k)
    b_ref = balance(ref.labels, g.groups, k, g.h)
    b_gpu = balance(perm[lab_gpu], g.groups, k, g.h)
    assert np.abs(b_ref - b_gpu).max() <= 1e-3
    return a, lab_gpu, ref


def test_kmeans_config1_vs_oracle(gpu_lib):
    g, cfg = baseline_config(1)
    dense = fairsc.fairsc_dense(g.dense(), g.groups, g.h, cfg["k_eig"], cfg["normalized"])
    _kmeans_parity(gpu_lib, g, cfg["k_eig"], cfg["normalized"], cfg["tol"], dense.H)


def test_kmeans_normalized_random_vs_oracle(gpu_lib):
    g = random_graph(600, 3, p=0.02, seed=31, weights="uniform")
    dense = fairsc.fairsc_dense(g.dense(), g.groups, 3, 6, True)
    _kmeans_parity(gpu_lib, g, 6, True, 1e-10, dense.H)


def test_kmeans_planted_recovers_truth(gpu_lib):
    from oracle.metrics import ari
    g = planted_cliques(5, 8, 4, seed=3)
    ctx = _ctx(gpu_lib, g, 5, True)
    gpu_lib.sfairsc_eigs(ctx, 5, 1e-10)
    lab, wcss = gpu_lib.sfairsc_embed_kmeans(ctx, 7)
    ctx.close()
    assert ari(lab, g.clusters) == 1.0
    assert wcss < 1e-20


def test_kmeans_device_labels_and_determinism(gpu_lib):
    import torch
    g, cfg = baseline_config(1)
    ctx = _ctx(gpu_lib, g, 5, False)
    gpu_lib.sfairsc_eigs(ctx, 5, 1e-10)
    a, w1 = gpu_lib.sfairsc_embed_kmeans(ctx, 99)
    b = torch.empty(g.n, dtype=torch.int32, device="cuda:0")
    _, w2 = gpu_lib.sfairsc_embed_kmeans(ctx, 99, labels=b)
    ctx.close()
    assert np.array_equal(a, b.cpu().numpy()) and w1 == w2


@pytest.mark.parametrize("n,k", [(37, 1), (50, 3), (130, 4), (300, 9)])
def test_kmeans_small_edge_cases_match_oracle_on_same_embedding(gpu_lib, n, k):
    """Edge cases of the k-means kernels (k = 1, n below one 128-row tile, a ragged
    last tile): the oracle's R16 k-means run on the GPU's own embedding H = X
    (unnormalized) gives the same partition and WCSS."""
    from oracle.kmeans import kmeans
    from oracle.metrics import ari
    g = random_graph(n, 2, p=min(1.0, 8.0 / n), seed=n, weights="uniform")
    ctx = _ctx(gpu_lib, g, k, False)
    _, Xt, _ = gpu_lib.sfairsc_eigs(ctx, k, 1e-12)
    lab, wcss = gpu_lib.sfairsc_embed_kmeans(ctx, 5)
    ctx.close()
    ref = kmeans(np.ascontiguousarray(Xt.T), k, 5)
    assert lab.min() >= 0 and lab.max() < k
    assert ari(ref.labels, lab) == 1.0 if k > 1 else np.all(lab == 0)
    assert abs(wcss - ref.wcss) <= 1e-10 * max(1.0, abs(ref.wcss))


@pytest.mark.parametrize("n,h,k,normalized", [(3001, 3, 13, True), (2500, 4, 8, False), (4000, 2, 64, True)])
def test_kmeans_tensor_core_assignment_is_exact(gpu_lib, monkeypatch, n, h, k, normalized):
    """The tensor-core assignment (DMMA distances + exact guard) must reproduce the
    direct R16 assignment bit for bit: same labels, same WCSS (k = 13: ragged DMMA
    tiles; k = 64: the widest embedding)."""
    g = random_graph(n, h, p=8.0 / n, seed=k, weights="uniform")
    ctx = _ctx(gpu_lib, g, k, normalized)
    gpu_lib.sfairsc_eigs(ctx, k, 1e-10)
    try:
        monkeypatch.setenv("SFAIRSC_KM_MMA", "0")
        lab0, w0 = gpu_lib.sfairsc_embed_kmeans(ctx, 7)
        monkeypatch.setenv("SFAIRSC_KM_MMA", "1")
        lab1, w1 = gpu_lib.sfairsc_embed_kmeans(ctx, 7)
    finally:
        monkeypatch.setenv("SFAIRSC_KM_MMA", "1")
        ctx.close()
    assert np.array_equal(lab0, lab1)
    assert w0 == w1


@pytest.mark.parametrize("n,h,k,normalized", [(30000, 3, 12, True), (20000, 2, 5, False), (6000, 3, 64, True)])
def test_kmeans_bound_pruned_assignment_is_exact(gpu_lib, monkeypatch, n, h, k, normalized):
    """Rows whose Hamerly bounds (with a 1e-12 relative margin) prove the assigned
    centroid strictly nearest are skipped: the labels and WCSS must equal the
    unpruned assignment's bit for bit."""
    g = random_graph(n, h, p=8.0 / n, seed=k + 1, weights="uniform")
    ctx = _ctx(gpu_lib, g, k, normalized)
    gpu_lib.sfairsc_eigs(ctx, k, 1e-10)
    try:
        monkeypatch.setenv("SFAIRSC_KM_PRUNE", "0")
        lab0, w0 = gpu_lib.sfairsc_embed_kmeans(ctx, 11)
        monkeypatch.setenv("SFAIRSC_KM_PRUNE", "1")
        lab1, w1 = gpu_lib.sfairsc_embed_kmeans(ctx, 11)
    finally:
        monkeypatch.delenv("SFAIRSC_KM_PRUNE")
        ctx.close()
    assert np.array_equal(lab0, lab1)
    assert w0 == w1


def test_kmeans_incremental_sums_match_full(gpu_lib, monkeypatch):
    """Lloyd iterations with few changed labels update the cluster sums from the
    changed rows only (full recomputation every 16 iterations): same clustering as
    recomputing every iteration, WCSS equal to rounding."""
    from oracle.metrics import ari
    g = random_graph(30000, 3, p=8.0 / 30000, seed=5, weights="uniform")
    ctx = _ctx(gpu_lib, g, 12, True)
    gpu_lib.sfairsc_eigs(ctx, 12, 1e-10)
    try:
        monkeypatch.setenv("SFAIRSC_KM_INCR", "0")
        lab0, w0 = gpu_lib.sfairsc_embed_kmeans(ctx, 3)
        monkeypatch.setenv("SFAIRSC_KM_INCR", "1")
        lab1, w1 = gpu_lib.sfairsc_embed_kmeans(ctx, 3)
    finally:
        monkeypatch.setenv("SFAIRSC_KM_INCR", "1")
        ctx.close()
    assert ari(lab0, lab1) >= 0.999
    assert abs(w0 - w1) <= 1e-9 * abs(w0)


# --- BASELINE configs 3 and 4 ------------------------------------------------------

def test_eigs_config3_reduced_vs_tier_s(gpu_lib):
    """Config 3 law (unnormalized, h=5, k=20, U(0.5,1.5) weights) at n = 50,000
    against the Tier S oracle (ARPACK on the paper's matrix-free operator)."""
    g, cfg = baseline_config(3, n=50_000)
    k = cfg["k_eig"]
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, False)
    ref = sfairsc_cpu.sfairsc_arpack(op, k, tol=1e-12, seed=3)
    gap = ref.evals[k] - ref.evals[k - 1]
    _check_eigs(gpu_lib, g, k, False, cfg["tol"], ref_evals=ref.evals[:k], ref_X=ref.X, gap=gap)


def _full_size_properties(lib, c, n_sample=3):
    """Full BASELINE size in the launch configuration bench.py times: the GPU
    solve (device-resident CSR) checked by properties that hold at any size
    and by oracle applies of sampled eigenvectors (Tier S, one by one)."""
    import torch
    g, cfg = baseline_config(c)
    k = cfg["k_eig"]
    dev = torch.device("cuda:0")
    t = lambda a: torch.from_numpy(a).to(dev)
    ctx = lib.sfairsc_build_operator(t(g.row_ptr), t(g.col), t(g.val), t(g.groups.astype(np.int32)), k,
                                     cfg["normalized"], h=g.h)
    Xd = torch.empty((k, g.n), dtype=torch.float64, device=dev)
    ev, _, st = lib.sfairsc_eigs(ctx, k, cfg["tol"], evecs=Xd)
    ctx.close()
    X = Xd.T.cpu().numpy()
    del Xd
    sigma = st["sigma"]
    assert st["converged"] == 1 and st["max_resid_rel"] <= 1e-9
    assert np.all(np.diff(ev) >= -1e-12 * sigma) and ev[-1] < sigma
    assert abs(ev[0]) <= 1e-12 * sigma  # lambda_1 = 0 (F^T 1 = 0)
    assert np.abs(X.T @ X - np.eye(k)).max() <= 1e-11  # orthonormal
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, cfg["normalized"])
    assert op.sigma == pytest.approx(sigma, rel=1e-14)
    assert np.linalg.norm(op.C.T @ X) <= 1e-10 * np.linalg.norm(X)  # fair: C^T X = 0
    one = np.sqrt(op.d) if cfg["normalized"] else np.ones(g.n)
    # the lambda = 0 eigenvector is D^{1/2} 1 (normalized) / 1: it lies in span(X)
    assert subspace_sin(X, one[:, None]) <= 1e-8
    rng = np.random.default_rng(c)
    for i in sorted(rng.choice(k, size=n_sample, replace=False)):
        r = op.apply(X[:, i]) - ev[i] * X[:, i]  # oracle apply, one vector at a time
        assert np.linalg.norm(r) / sigma <= 1e-9, (i, np.linalg.norm(r) / sigma)
        rq = X[:, i] @ op.apply(X[:, i])
        assert abs(rq - ev[i]) <= 1e-8 * abs(ev[i]) + 1e-12 * sigma
    return ev, st


def test_config3_full_size_properties(gpu_lib):
    _full_size_properties(gpu_lib, 3)


def test_config4_full_size_properties(gpu_lib):
    ev, st = _full_size_properties(gpu_lib, 4, n_sample=2)
    assert st["steps"] > 0


# --- column-blocked SpMV (the config-5 path: gathered vector larger than L2) ------------------

@pytest.mark.parametrize("weights", ["uniform", "unit"])
@pytest.mark.parametrize("normalized", [False, True])
def test_column_blocked_spmv_matches_oracle(gpu_lib, normalized, weights, monkeypatch):
    """Force the block-major CSR (normally chosen for n > ~8M) on a small graph:
    SpMV, L^sigma and the eigensolve must equal the oracle as for the plain CSR
    (unit weights: pattern-only SpMV, the value array dropped after the build)."""
    monkeypatch.setenv("SFAIRSC_COLBLK_MB", "0.003")  # 3 KB column blocks -> several blocks at n ~ 1000
    g = random_graph(1031, 5, p=0.02, seed=21, weights=weights)
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, normalized)
    ctx = _ctx(gpu_lib, g, 6, normalized)
    monkeypatch.delenv("SFAIRSC_COLBLK_MB")
    x = np.random.default_rng(5).standard_normal((2, g.n))
    tol = 1e-13 * op.sigma * np.abs(x).max()
    assert np.abs(gpu_lib.sfairsc_laplacian(ctx, np.ascontiguousarray(x[0])) - op.Ln @ x[0]).max() <= tol
    assert np.abs(gpu_lib.sfairsc_apply(ctx, x) - np.stack([op.apply(v) for v in x])).max() <= tol
    ev, Xt, st = gpu_lib.sfairsc_eigs(ctx, 6, 1e-10)
    ctx.close()
    dense = fairsc.fairsc_dense(g.dense(), g.groups, g.h, 6, normalized)
    assert st["converged"] == 1 and st["max_resid_rel"] <= 1e-9
    assert np.all(np.abs(ev - dense.evals[:6]) <= 1e-8 * np.abs(dense.evals[:6]) + 1e-12 * st["sigma"])


# --- BASELINE config 5 (DC-SBM, reading R20) ---------------------------------------

def test_eigs_config5_reduced_vs_tier_s(gpu_lib):
    """Config 5 law (unnormalized, h=8, k=64, Pareto(2.5) degree propensities,
    Dirichlet(2) cluster sizes) at n = 20,000 against the Tier S oracle (ARPACK
    on the paper's matrix-free operator).  The full-size (n = 5e7) solve is an
    evidence run (scripts/run_cfg5.py, profiles/) — ARPACK cannot finish there."""
    from synth.dcsbm import config5
    g, cfg = config5(n=20_000, device="cuda")
    g = g.host()
    k = cfg["k_eig"]
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, False)
    ref = sfairsc_cpu.sfairsc_arpack(op, k, tol=1e-12, seed=5, ncv=160)
    gap = ref.evals[k] - ref.evals[k - 1]
    _check_eigs(gpu_lib, g, k, False, cfg["tol"], ref_evals=ref.evals[:k], ref_X=ref.X, gap=gap)


# --- §8(f) N3: the paper's Experiment-1 m-SBM (fair vs unconstrained SC) ---------------------

@pytest.mark.parametrize("h", [2, 5])
def test_exp1_fair_recovers_planted_sc_fails(gpu_lib, h):
    """Fig. 8 setting: with a,b,c,d = (10,7,4,1)(log n/n)^(2/3)
    group membership dominates the edges, so SC (Alg. 1, h = 1) splits by group while
    s-FairSC recovers the fair planted clusters; the error rate (Eq. err) of the GPU
    clustering equals the oracle's (dense FairSC + oracle k-means) on the same graph."""
    from oracle.kmeans import kmeans
    from oracle.metrics import error_rate
    from synth import exp1_msbm
    n, k = 3000, 5
    g = exp1_msbm(n, h, seed=3)
    ctx = _ctx(gpu_lib, g, k, True)
    gpu_lib.sfairsc_eigs(ctx, k, 1e-10)
    lab_fair, _ = gpu_lib.sfairsc_embed_kmeans(ctx, 11)
    ctx.close()
    ctx = gpu_lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, np.zeros(n, np.int32), k, True, h=1)
    gpu_lib.sfairsc_eigs(ctx, k, 1e-10)
    lab_sc, _ = gpu_lib.sfairsc_embed_kmeans(ctx, 11)
    ctx.close()
    err_fair = error_rate(g.clusters, lab_fair, k)
    err_sc = error_rate(g.clusters, lab_sc, k)
    dense = fairsc.fairsc_dense(g.dense(), g.groups, h, k, True)
    err_or = error_rate(g.clusters, kmeans(dense.H, k, 11).labels, k)
    assert err_fair <= 0.05, err_fair
    assert err_sc >= 0.3, err_sc
    assert abs(err_fair - err_or) <= 2.0 / n * 5  # a handful of borderline vertices at most


def test_pair_apply_matches_single(gpu_lib):
    """sfairsc_apply on several device vectors runs them in pairs through one SpMM of the
    interleaved pair: equal to the oracle and to the one-vector path (odd count: last alone)."""
    import torch
    g = random_graph(1500, 4, p=0.01, seed=31, weights="uniform")
    for normalized in (False, True):
        op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, normalized)
        ctx = _ctx(gpu_lib, g, 3, normalized)
        x = torch.from_numpy(np.random.default_rng(3).standard_normal((5, g.n))).cuda()
        y = gpu_lib.sfairsc_apply(ctx, x).cpu().numpy()
        ref = np.stack([op.apply(v) for v in x.cpu().numpy()])
        assert np.abs(y - ref).max() <= 1e-13 * op.sigma * float(x.abs().max())
        y1 = np.stack([gpu_lib.sfairsc_apply(ctx, np.ascontiguousarray(v)) for v in x.cpu().numpy()])
        assert np.abs(y - y1).max() <= 1e-13 * op.sigma * float(x.abs().max())
        ctx.close()


def test_kmeans_config2_vs_oracle(gpu_lib, config2_ref):
    """Config 2 (normalized, n = 20,000, h = 5, k = 10): fair clustering of the GPU
    (eigs + embed_kmeans) against the oracle's k-means on the Tier-S embedding
    H = D^{-1/2} X (ARI >= 0.99, per-cluster balance within 1e-3; north star)."""
    from oracle.kmeans import kmeans
    from oracle.metrics import ari, balance, hungarian_match
    g, cfg, ref = config2_ref
    k = cfg["k_eig"]
    d = np.diff(g.row_ptr).astype(float)
    d = np.asarray(g.to_scipy().sum(axis=1)).ravel()
    H_or = ref.X / np.sqrt(d)[:, None]
    ctx = _ctx(gpu_lib, g, k, True)
    gpu_lib.sfairsc_eigs(ctx, k, cfg["tol"])
    lab, _ = gpu_lib.sfairsc_embed_kmeans(ctx, 2024)
    ctx.close()
    r = kmeans(H_or, k, 2024)
    assert ari(r.labels, lab) >= 0.99
    perm = hungarian_match(r.labels, lab, k)
    assert np.abs(balance(r.labels, g.groups, k, g.h) - balance(perm[lab], g.groups, k, g.h)).max() <= 1e-3


@pytest.mark.parametrize("blocked", [False, True])
def test_skewed_degree_spmv(gpu_lib, blocked, monkeypatch):
    """Heavy-tailed degrees (config-5 law: Pareto(2.5) propensities): rows longer than
    32 VS slots go to a whole warp; L x and L^sigma x equal the oracle, with and
    without the column-blocked CSR."""
    from synth.dcsbm import config5
    g, cfg = config5(n=30_000, device="cpu")
    g = g.host()
    deg = np.diff(g.row_ptr)
    assert deg.max() > 16 * deg.mean()  # the long-row path is exercised
    if blocked:
        monkeypatch.setenv("SFAIRSC_COLBLK_MB", "0.05")
    ctx = _ctx(gpu_lib, g, 4, False)
    if blocked:
        monkeypatch.delenv("SFAIRSC_COLBLK_MB")
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, False)
    x = np.random.default_rng(9).standard_normal((2, g.n))
    tol = 1e-13 * op.sigma * np.abs(x).max()
    assert np.abs(gpu_lib.sfairsc_laplacian(ctx, np.ascontiguousarray(x[0])) - op.Ln @ x[0]).max() <= tol
    assert np.abs(gpu_lib.sfairsc_apply(ctx, x) - np.stack([op.apply(v) for v in x])).max() <= tol
    ctx.close()


# --- edge cases: the whole constrained spectrum, tiny graphs, empty input --------------------

@pytest.mark.parametrize("normalized", [False, True])
def test_eigs_full_constrained_spectrum(gpu_lib, normalized):
    """k = n - h + 1 = dim null(C^T): every eigenpair of the fair problem (the Krylov space
    exhausts null(C^T); the solver must stop on the invariant subspace, not fail)."""
    g = random_graph(31, 3, p=0.3, seed=41, weights="uniform")
    k = g.n - g.h + 1
    dense = fairsc.fairsc_dense(g.dense(), g.groups, g.h, k, normalized, extra=0)
    _check_eigs(gpu_lib, g, k, normalized, 1e-10, ref_evals=dense.evals[:k], ref_X=dense.X, gap=None)


def test_eigs_tiny_graph_k1(gpu_lib):
    """n = 4, h = 2, k = 1: the trivial pair lambda_1 = 0 only."""
    g = random_graph(4, 2, p=1.0, seed=3, weights="unit", group_counts=(2, 2))
    ev, X, st = _check_eigs(gpu_lib, g, 1, True, 1e-10, ref_evals=np.zeros(1))
    assert abs(ev[0]) <= 1e-12 * st["sigma"]


def test_empty_and_invalid_inputs(gpu_lib):
    lib = gpu_lib
    with pytest.raises(lib.SfairscError) as e:  # n = 0
        lib.sfairsc_build_operator(np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0), np.zeros(0, np.int32),
                                   1, False, h=1)
    assert e.value.name == "E_INVALID_ARG"
    g = random_graph(20, 2, p=0.3, seed=2)
    with pytest.raises(lib.SfairscError) as e:  # k = 0
        lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, g.groups.astype(np.int32), 0, False)
    assert e.value.name == "E_INVALID_ARG"
    ctx = lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, g.groups.astype(np.int32), 3, False)
    with pytest.raises(lib.SfairscError) as e:  # eigs k above the build k
        lib.sfairsc_eigs(ctx, 4, 1e-10)
    assert e.value.name == "E_K_TOO_LARGE"
    with pytest.raises(lib.SfairscError) as e:  # tol <= 0
        lib.sfairsc_eigs(ctx, 2, 0.0)
    assert e.value.name == "E_INVALID_ARG"
    ctx.close()
    col = g.col.copy()
    col[0] = g.n + 5  # column out of range
    with pytest.raises(lib.SfairscError) as e:
        lib.sfairsc_build_operator(g.row_ptr, col, g.val, g.groups.astype(np.int32), 2, False)
    assert e.value.name == "E_CSR_INVALID"


@pytest.mark.parametrize("normalized", [False, True])
@pytest.mark.parametrize("n,k,m", [(1800, 6, 0), (2400, 9, 23), (3000, 12, 17)])
def test_paired_steps_match_single_steps_and_oracle(gpu_lib, normalized, n, k, m):
    """two Lanczos steps per basis sweep (reorth 3, the default) against one (reorth 2) and
    the dense oracle: the same eigenvalues (R6), subspaces within the Davis-Kahan bound, an orthonormal
    fair basis; small bases (m = 17 = k + 5: one pair per cycle after the single first steps) included."""
    g = random_graph(n, 4, p=8.0 / n, seed=n + k, weights="uniform")
    dense = fairsc.fairsc_dense(g.dense(), g.groups, g.h, k, normalized)
    kw = {"max_basis": m} if m else {}
    ev3, X3, st3 = _check_eigs(gpu_lib, g, k, normalized, 1e-10, dense=dense, reorth=3, **kw)
    ev2, X2, st2 = _check_eigs(gpu_lib, g, k, normalized, 1e-10, dense=dense, reorth=2, **kw)
    assert np.all(np.abs(ev3 - ev2) <= 1e-9 * np.abs(ev2) + 1e-12 * st2["sigma"])
    assert abs(st3["applies"] - st2["applies"]) <= 0.1 * st2["applies"] + 10


def test_paired_steps_option_errors(gpu_lib):
    g = random_graph(600, 3, p=0.02, seed=5, weights="uniform")
    with pytest.raises(gpu_lib.SfairscError) as e:  # reorth 3 needs the single-vector lagged solver
        _ctx(gpu_lib, g, 4, True, reorth=3, block_size=2)
    assert e.value.name == "E_INVALID_ARG"
    with pytest.raises(gpu_lib.SfairscError) as e:
        _ctx(gpu_lib, g, 4, True, reorth=4)
    assert e.value.name == "E_INVALID_ARG"


def test_binding_rejects_wrong_output_shapes(gpu_lib):
    """Advisor r1: the binding checks the caller's output buffers before handing pointers to the library
    (which writes k x n doubles / n labels / vectors of length n)."""
    g = random_graph(300, 3, p=0.05, seed=2, weights="uniform")
    ctx = _ctx(gpu_lib, g, 4, True)
    with pytest.raises(ValueError):
        gpu_lib.sfairsc_eigs(ctx, 4, 1e-10, evecs=np.zeros((3, g.n)))
    with pytest.raises(ValueError):
        gpu_lib.sfairsc_eigs(ctx, 4, 1e-10, evecs=np.zeros((4, g.n - 1)))
    gpu_lib.sfairsc_eigs(ctx, 4, 1e-10)
    with pytest.raises(ValueError):
        gpu_lib.sfairsc_embed_kmeans(ctx, 1, labels=np.zeros(g.n - 1, np.int32))
    x = np.random.default_rng(0).standard_normal(g.n)
    with pytest.raises(ValueError):
        gpu_lib.sfairsc_apply(ctx, x[:-1])
    with pytest.raises(ValueError):
        gpu_lib.sfairsc_apply(ctx, x, np.zeros(g.n + 1))
    y = gpu_lib.sfairsc_apply(ctx, x)
    assert y.shape == x.shape
    ctx.close()


@pytest.mark.parametrize("parts", [1, 3])
def test_paired_row_partitioned_matches_single_gpu(gpu_lib, parts):
    """Paired steps in the row-partitioned solver (virtual parts) against the single-GPU paired solver and
    the one-step partitioned solver: the same eigenvalues (R6) on a ragged n."""
    g = random_graph(1777, 4, p=0.006, seed=21, weights="uniform")
    k = 7
    ctx = _ctx(gpu_lib, g, k, True)
    ev1, _, st1 = gpu_lib.sfairsc_eigs(ctx, k, 1e-10)
    ctx.close()
    kw = {"virtual_parts": parts} if parts > 1 else {}
    for reorth in (3, 2):
        ctx = _ctx(gpu_lib, g, k, True, reorth=reorth, **kw)
        ev, _, st = gpu_lib.sfairsc_eigs(ctx, k, 1e-10)
        ctx.close()
        assert st["converged"] == 1 and st["max_resid_rel"] <= 1e-9
        assert np.all(np.abs(ev - ev1) <= 1e-8 * np.abs(ev1) + 1e-12 * st1["sigma"])
