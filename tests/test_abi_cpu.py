"""CPU-only checks of the C-ABI library: it loads without a GPU, exports every
symbol include/sfairsc.h declares, and its host-side Rayleigh-Ritz
eigensolver (A10) is pinned against LAPACK."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "sfairsc.h")


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(sfairsc_[a-z_0-9]+)\s*\(", text)
    return sorted(set(names))


def test_header_declares_boundary():
    names = _declared_functions()
    for required in ("sfairsc_build_operator", "sfairsc_eigs", "sfairsc_embed_kmeans", "sfairsc_apply",
                     "sfairsc_destroy", "sfairsc_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2210_16435_b200 import lib
    so = ctypes.CDLL(lib.LIB_PATH)
    missing = [n for n in _declared_functions() if not hasattr(so, n)]
    assert not missing, missing
    assert "sm_100a" in lib.version()


def test_struct_mirrors_match_library_layout():
    """The binding's ctypes mirrors of sfairsc_csr / _opts / _stats / _info have the library's sizes
    (the binding also checks this at load time) and the default options match the header's defaults."""
    from paper_2210_16435_b200 import lib
    for which, st in enumerate((lib.CSR, lib.Opts, lib.Stats, lib.Info)):
        assert lib._lib.sfairsc_struct_size(which) == ctypes.sizeof(st), st.__name__
    assert lib._lib.sfairsc_struct_size(9) == -1
    o = lib.default_opts()
    assert (o.reorth, o.block_size, o.filter_degree, o.filter_cut, o.tol_eff_cap) == (0, 0, 0, 0.0, 1e-10)


def test_library_is_sm100a_cubin():
    import subprocess
    from paper_2210_16435_b200 import lib
    out = subprocess.run(["cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("m,seed", [(1, 0), (2, 1), (7, 2), (40, 3), (130, 4)])
def test_host_symeig_vs_lapack(m, seed):
    from paper_2210_16435_b200 import lib
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, m))
    A = A + A.T
    ev, V = lib.host_symeig(A)
    ref = np.linalg.eigvalsh(A)
    scale = max(1.0, np.abs(ref).max())
    assert np.allclose(ev, ref, atol=1e-13 * scale * m)
    assert np.allclose(V.T @ V, np.eye(m), atol=1e-13 * m)
    assert np.allclose(A @ V, V * ev, atol=1e-12 * scale * m)


def test_host_symeig_arrowhead_degenerate():
    """Thick-restart T: diagonal Ritz block + arrow + tridiagonal tail, with
    repeated eigenvalues (planted-clique case)."""
    from paper_2210_16435_b200 import lib
    p, m = 5, 12
    T = np.zeros((m, m))
    T[np.arange(p), np.arange(p)] = [0, 0, 0, 6, 6]
    T[:p, p] = T[p, :p] = [1e-3, 0, 2e-3, 0, 1e-9]
    rng = np.random.default_rng(0)
    for i in range(p, m):
        T[i, i] = rng.uniform(0, 10)
        if i + 1 < m:
            T[i, i + 1] = T[i + 1, i] = rng.uniform(0, 1)
    ev, V = lib.host_symeig(T)
    assert np.allclose(ev, np.linalg.eigvalsh(T), atol=1e-13 * 10)
    assert np.allclose(T @ V, V * ev, atol=1e-12)


@pytest.mark.parametrize("m,nvec,seed", [(1, 1, 0), (2, 1, 1), (7, 3, 2), (40, 0, 3), (40, 17, 4), (130, 60, 5),
                                         (170, 81, 6), (170, 170, 7)])
def test_host_symeig_sel_vs_lapack(m, nvec, seed):
    """The thick restart's selected-vector Rayleigh-Ritz (row-contiguous Householder reduction with the
    reflectors kept, QL rotations applied in reverse to the selected unit vectors, reflectors applied after):
    all eigenvalues and the nvec smallest eigenpairs against LAPACK (numpy eigh), and the same pairs as the
    full solver (eigenvalues to rounding, vectors up to sign where the eigenvalues are simple)."""
    from paper_2210_16435_b200 import lib
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, m))
    A = A + A.T
    ev, V = lib.host_symeig_sel(A, nvec)
    ref, U = np.linalg.eigh(A)
    scale = max(1.0, np.abs(ref).max())
    assert np.allclose(ev, ref, atol=1e-13 * scale * m)
    assert V.shape == (m, nvec)
    assert np.allclose(V.T @ V, np.eye(nvec), atol=1e-13 * m)
    assert np.allclose(A @ V, V * ev[:nvec], atol=1e-12 * scale * m)
    evf, Vf = lib.host_symeig(A)  # the full solver (EISPACK tred2/tql2): same pairs to rounding
    assert np.allclose(ev, evf, atol=1e-13 * scale * m)
    sgn = np.sign(np.sum(V * Vf[:, :nvec], axis=0))
    gaps = np.diff(ref)
    if nvec and (nvec == m or gaps[:nvec].min() > 1e-3):  # vectors are unique up to sign for simple eigenvalues
        assert np.allclose(V * sgn, Vf[:, :nvec], atol=1e-10 * m)


def test_host_symeig_sel_thick_restart_structure():
    """Thick-restart shape (diagonal Ritz block + arrow + tridiagonal tail) with repeated and tightly
    clustered eigenvalues (config 4's lambda_2..lambda_50 lie within 2.4e-4 of each other), and a
    zero-scale Householder step (an exact zero row below the diagonal)."""
    from paper_2210_16435_b200 import lib
    rng = np.random.default_rng(11)
    p, m = 80, 170
    T = np.zeros((m, m))
    T[np.arange(p), np.arange(p)] = 0.6515 + 2.4e-4 * np.sort(rng.random(p))
    T[:3, :3] = np.diag([0.0, 0.0, 0.0])
    T[:p, p] = T[p, :p] = 1e-6 * rng.standard_normal(p)
    for i in range(p, m):
        T[i, i] = rng.uniform(0.6, 1.4)
        if i + 1 < m:
            T[i, i + 1] = T[i + 1, i] = rng.uniform(0, 0.2)
    T[m - 1, m - 2] = T[m - 2, m - 1] = 0.0
    ev, V = lib.host_symeig_sel(T, p)
    assert np.allclose(ev, np.linalg.eigvalsh(T), atol=1e-14)
    assert np.allclose(V.T @ V, np.eye(p), atol=1e-13)
    assert np.allclose(T @ V, V * ev[:p], atol=1e-14)


def test_host_symeig_sel_bad_args():
    from paper_2210_16435_b200 import lib
    with pytest.raises(Exception):
        lib.host_symeig_sel(np.eye(4), 5)
