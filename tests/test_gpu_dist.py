"""GPU parity of the row-partitioned solver.

One GPU is available, so the partitioned arithmetic is exercised with
`virtual_parts` (P row blocks in one process: padded column remap, gathered
projected vector, fixed-order reductions) and the NCCL transport with a
1-rank communicator (the same calls a multi-GPU job makes).  Results are
checked against the oracle with the tolerances of tests/test_gpu_parity.py
and across part counts (agreement to rounding, reading R8)."""
import numpy as np
import pytest

from oracle import fairsc
from oracle.metrics import subspace_sin
from synth import baseline_config, random_graph

pytestmark = pytest.mark.gpu


def _solve(lib, g, k, normalized, tol, **kw):
    ctx = lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, g.groups.astype(np.int32), k, normalized, h=g.h, **kw)
    ev, Xt, st = lib.sfairsc_eigs(ctx, k, tol)
    info = ctx.info()
    return ctx, ev, Xt.T, st, info


@pytest.mark.parametrize("blocked", ["0", "1"])
@pytest.mark.parametrize("parts", [2, 3])
@pytest.mark.parametrize("case", ["cfg1", "rand_norm"])
def test_virtual_parts_vs_dense(gpu_lib, parts, case, blocked, monkeypatch):
    if case == "cfg1":
        g, cfg = baseline_config(1)
        k, normalized, tol = cfg["k_eig"], cfg["normalized"], cfg["tol"]
    else:
        g = random_graph(900, 4, p=0.015, seed=11, weights="uniform")
        k, normalized, tol = 6, True, 1e-10
    dense = fairsc.fairsc_dense(g.dense(), g.groups, g.h, k, normalized)
    monkeypatch.setenv("SFAIRSC_DIST_BLOCK", blocked)  # owner-segment column blocks (config-5 path) or not
    ctx, ev, X, st, info = _solve(gpu_lib, g, k, normalized, tol, virtual_parts=parts)
    monkeypatch.delenv("SFAIRSC_DIST_BLOCK")
    sigma = st["sigma"]
    assert st["converged"] == 1 and st["max_resid_rel"] <= 1e-9
    assert np.all(np.abs(ev - dense.evals[:k]) <= 1e-8 * np.abs(dense.evals[:k]) + 1e-12 * sigma)
    assert np.abs(X.T @ X - np.eye(k)).max() <= 1e-12
    C = fairsc.constraint_matrix(g.dense(), g.groups, g.h, normalized)
    assert np.linalg.norm(C.T @ X) <= 1e-10 * np.linalg.norm(X)
    bound = 2 * (st["max_resid_rel"] * sigma * np.sqrt(k) + 1e-12 * sigma) / dense.gap
    assert subspace_sin(X, dense.X) <= max(1e-6, bound)
    # the partitioned operator apply equals the single-GPU one (same arithmetic up to reduction order)
    x = np.random.default_rng(parts).standard_normal((2, g.n))
    ref_ctx = gpu_lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, g.groups.astype(np.int32), k, normalized,
                                             h=g.h)
    y_ref = gpu_lib.sfairsc_apply(ref_ctx, x)
    y = gpu_lib.sfairsc_apply(ctx, x)
    assert np.abs(y - y_ref).max() <= 1e-13 * sigma * np.abs(x).max()
    ref_ctx.close()
    ctx.close()


def test_virtual_parts_agree_across_part_counts(gpu_lib):
    g, cfg = baseline_config(2)
    k = cfg["k_eig"]
    res = {}
    for P in (1, 2, 4):
        kw = {"virtual_parts": P} if P > 1 else {}
        ctx, ev, X, st, _ = _solve(gpu_lib, g, k, True, cfg["tol"], **kw)
        ctx.close()
        assert st["converged"] == 1 and st["max_resid_rel"] <= 1e-9
        res[P] = (ev, X, st)
    ev1, X1, st1 = res[1]
    for P in (2, 4):
        ev, X, st = res[P]
        assert np.all(np.abs(ev - ev1) <= 1e-8 * np.abs(ev1) + 1e-12 * st["sigma"])
        gap = st["gap_est"]
        bound = 2 * ((st["max_resid_rel"] + st1["max_resid_rel"]) * st["sigma"] * np.sqrt(k)) / gap
        assert subspace_sin(X, X1) <= max(1e-6, bound)


def test_virtual_parts_deterministic(gpu_lib):
    g, cfg = baseline_config(1)
    a = _solve(gpu_lib, g, 5, False, 1e-10, virtual_parts=3)
    b = _solve(gpu_lib, g, 5, False, 1e-10, virtual_parts=3)
    a[0].close()
    b[0].close()
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


def test_virtual_parts_kmeans(gpu_lib):
    from oracle.kmeans import kmeans
    from oracle.metrics import ari
    g, cfg = baseline_config(1)
    dense = fairsc.fairsc_dense(g.dense(), g.groups, g.h, cfg["k_eig"], cfg["normalized"])
    ctx, ev, X, st, _ = _solve(gpu_lib, g, cfg["k_eig"], cfg["normalized"], cfg["tol"], virtual_parts=2)
    lab, wcss = gpu_lib.sfairsc_embed_kmeans(ctx, 2024)
    ctx.close()
    ref = kmeans(dense.H, cfg["k_eig"], 2024)
    assert ari(ref.labels, lab) >= 0.99


def test_nccl_one_rank(gpu_lib):
    """The NCCL transport with a 1-rank communicator: the calls and the row-block
    ABI (row_offset, n_global) a multi-GPU job uses."""
    import torch
    torch.cuda.set_device(0)
    g, cfg = baseline_config(1)
    comm = gpu_lib.Comm(gpu_lib.comm_unique_id(), 0, 1, 0)
    cuts = gpu_lib.partition_rows(g.row_ptr, 1)
    rp, ci, vv, gr = gpu_lib.row_block(g.row_ptr, g.col, g.val, g.groups, int(cuts[0]), int(cuts[1]))
    ctx = gpu_lib.sfairsc_build_operator(rp, ci, vv, gr, cfg["k_eig"], cfg["normalized"], h=g.h, comm=comm,
                                         n_global=g.n, row_offset=int(cuts[0]))
    ev, Xt, st = gpu_lib.sfairsc_eigs(ctx, cfg["k_eig"], cfg["tol"])
    ctx.close()
    comm.close()
    dense = fairsc.fairsc_dense(g.dense(), g.groups, g.h, cfg["k_eig"], cfg["normalized"])
    assert st["converged"] == 1 and st["max_resid_rel"] <= 1e-9
    assert np.all(np.abs(ev - dense.evals[:5]) <= 1e-8 * np.abs(dense.evals[:5]) + 1e-12 * st["sigma"])
    assert subspace_sin(Xt.T, dense.X) <= 1e-6


def test_nccl_failed_rank_agreement(gpu_lib):
    """Advisor r1: a rank whose own input checks fail takes part in the build's agreement all-reduce
    (dist_agree) before returning, so the other ranks fail with it instead of blocking in the first
    all-gather.  With one rank: the local status comes back (not a hang, not E_NCCL), the message is this
    rank's, and the communicator is still usable for a correct build afterwards (the collective matched)."""
    import torch
    torch.cuda.set_device(0)
    g, cfg = baseline_config(1)
    comm = gpu_lib.Comm(gpu_lib.comm_unique_id(), 0, 1, 0)
    cuts = gpu_lib.partition_rows(g.row_ptr, 1)
    rp, ci, vv, gr = gpu_lib.row_block(g.row_ptr, g.col, g.val, g.groups, int(cuts[0]), int(cuts[1]))
    bad = np.array(gr, copy=True)
    bad[3] = g.h + 7  # group id out of [0, h): a per-rank check before any collective
    with pytest.raises(gpu_lib.SfairscError) as ei:
        gpu_lib.sfairsc_build_operator(rp, ci, vv, bad, cfg["k_eig"], cfg["normalized"], h=g.h, comm=comm,
                                       n_global=g.n, row_offset=int(cuts[0]))
    assert ei.value.status == 1 and "group id" in str(ei.value)
    ctx = gpu_lib.sfairsc_build_operator(rp, ci, vv, gr, cfg["k_eig"], cfg["normalized"], h=g.h, comm=comm,
                                         n_global=g.n, row_offset=int(cuts[0]))
    ev, _, st = gpu_lib.sfairsc_eigs(ctx, cfg["k_eig"], cfg["tol"])
    ctx.close()
    comm.close()
    assert st["converged"] == 1
