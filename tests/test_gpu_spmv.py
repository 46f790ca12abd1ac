"""GPU parity of the TMA-fed tile SpMV (spmv_tma.cu, A5) against the oracle and
against the round-1 LSU kernel (SFAIRSC_SPMV_TMA=0).

Edge cases of the row-aligned tiling: rows longer than a tile (hubs of degree 1.5k
and 5k, read by the whole CTA), graphs smaller than one tile, ragged n, every lane
width VS, unit and non-unit weights, both operators.  Tolerance as in
test_gpu_parity.py: |y - y_ref|_inf <= 1e-13 sigma |x|_inf, for both kernels; the TMA
kernel is deterministic (bitwise-identical on repeated launches).
"""
import numpy as np
import pytest

from oracle import sfairsc_cpu
from synth import hub_graph, random_graph

pytestmark = pytest.mark.gpu


def _build(lib, g, normalized, tma=True, monkeypatch=None, **kw):
    monkeypatch.setenv("SFAIRSC_SPMV_TMA", "1" if tma else "0")
    ctx = lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, g.groups.astype(np.int32), 3, normalized, h=g.h, **kw)
    monkeypatch.delenv("SFAIRSC_SPMV_TMA")
    return ctx


@pytest.mark.parametrize("weights", ["uniform", "unit"])
@pytest.mark.parametrize("normalized", [False, True])
@pytest.mark.parametrize("vs", [2, 8, 32])
def test_spmv_tma_long_rows(gpu_lib, monkeypatch, weights, normalized, vs):
    g = hub_graph(6000, 3, hub_degrees=(1500, 5000), seed=vs, weights=weights)
    assert np.diff(g.row_ptr).max() > 4096  # longer than a tile
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, normalized)
    ctx = _build(gpu_lib, g, normalized, monkeypatch=monkeypatch, spmv_vector=vs)
    x = np.random.default_rng(3).standard_normal((2, g.n))
    tol = 1e-13 * op.sigma * np.abs(x).max()
    assert np.abs(gpu_lib.sfairsc_laplacian(ctx, np.ascontiguousarray(x[0])) - op.Ln @ x[0]).max() <= tol
    assert np.abs(gpu_lib.sfairsc_apply(ctx, x) - np.stack([op.apply(v) for v in x])).max() <= tol
    ev, _, st = gpu_lib.sfairsc_eigs(ctx, 3, 1e-10)
    assert st["converged"] == 1 and st["max_resid_rel"] <= 1e-9
    ctx.close()


@pytest.mark.parametrize("n,p,h,normalized", [(5, 1.0, 2, False), (37, 0.3, 2, True), (70, 0.2, 3, False),
                                              (1031, 0.01, 5, True), (4099, 0.008, 4, False)])
def test_spmv_tma_small_and_ragged_vs_lsu(gpu_lib, monkeypatch, n, p, h, normalized):
    g = random_graph(n, h, p=p, seed=n, weights="uniform")
    op = sfairsc_cpu.build_operator(g.to_scipy(), g.groups, g.h, normalized)
    x = np.random.default_rng(n).standard_normal(g.n)
    tol = 1e-13 * op.sigma * np.abs(x).max()
    ys = []
    for tma in (True, False):
        ctx = _build(gpu_lib, g, normalized, tma=tma, monkeypatch=monkeypatch)
        y = gpu_lib.sfairsc_laplacian(ctx, x)
        assert np.abs(y - op.Ln @ x).max() <= tol
        assert np.array_equal(y, gpu_lib.sfairsc_laplacian(ctx, x))  # deterministic
        ys.append(y)
        ctx.close()
    assert np.abs(ys[0] - ys[1]).max() <= tol
