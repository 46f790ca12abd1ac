"""Tier S oracle: the paper's matrix-free s-FairSC on CPU — TEST INFRASTRUCTURE ONLY.

Algorithm 3 literally, with the implementation choices the paper
states in "Implementation issues":
  (i)   eigensolver = ARPACK (scipy `eigsh`, implicitly restarted Lanczos —
        the symmetric sibling of MATLAB eigs' Arnoldi), accessing
        L^sigma only through  L^sigma w = P(L_n(P w)) - sigma P w + sigma w;
  (ii)  P w = w - C z, z = argmin ||C z - w||, solved directly for small h
         — here via the normal equations / Cholesky of C^T C;
  (iii) sigma = ||L_n||_1.
This projector is deliberately NOT the GPU's factored form.  Pinned against
Tier D (tests/test_oracle_sparse.py) at n <= 2000.
"""
from __future__ import annotations

import dataclasses
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla


@dataclasses.dataclass
class SparseOperator:
    n: int
    Ln: sp.csr_matrix  # L_n (normalized) or L (R1)
    C: np.ndarray  # n x (h-1)
    cho: object  # Cholesky factor of C^T C (None when h = 1)
    sigma: float
    d: np.ndarray
    normalized: bool
    threads: int = 1  # > 1: L_n x by row blocks on a thread pool (scipy releases the GIL; same rows, same sums)
    _blocks: list = dataclasses.field(default=None, repr=False)
    _pool: object = dataclasses.field(default=None, repr=False)

    def spmv(self, x: np.ndarray) -> np.ndarray:
        """L_n x (or L x).  With threads > 1 the rows are cut into contiguous blocks,
        each block's products computed by scipy exactly as in the single call."""
        if self.threads <= 1 or x.ndim != 1:
            return self.Ln @ x
        if self._blocks is None:
            cuts = np.linspace(0, self.n, self.threads + 1).astype(np.int64)
            self._blocks = [self.Ln[cuts[i]:cuts[i + 1]] for i in range(self.threads)]
            self._pool = ThreadPoolExecutor(self.threads)
        return np.concatenate(list(self._pool.map(lambda B: B @ x, self._blocks)))

    def P(self, w: np.ndarray) -> np.ndarray:
        """P w = w - C z with z = (C^T C)^{-1} C^T w."""
        if self.C.shape[1] == 0:
            return w.copy()
        z = sla.cho_solve(self.cho, self.C.T @ w)
        return w - self.C @ z

    def apply(self, w: np.ndarray) -> np.ndarray:
        """L^sigma w = P(L_n(P w)) - sigma P w + sigma w."""
        Pw = self.P(w)
        return self.P(self.spmv(Pw)) - self.sigma * Pw + self.sigma * w

    def linear_operator(self) -> spla.LinearOperator:
        return spla.LinearOperator((self.n, self.n), matvec=self.apply, matmat=self.apply,
                                   dtype=np.float64)


def build_operator(W: sp.csr_matrix, groups: np.ndarray, h: int, normalized: bool,
                   sigma: float | None = None, F: np.ndarray | None = None,
                   threads: int = 1) -> SparseOperator:
    """Alg. 3 steps 1-2: L = D - W; L_n = D^{-1/2} L D^{-1/2}; C = D^{-1/2} F."""
    W = sp.csr_matrix(W)
    n = W.shape[0]
    d = np.asarray(W.sum(axis=1)).ravel()
    L = sp.diags(d) - W
    if normalized:
        s = 1.0 / np.sqrt(d)
        Ln = sp.diags(s) @ L @ sp.diags(s)
    else:
        s = np.ones(n)
        Ln = L
    Ln = sp.csr_matrix(Ln)
    # F = F_0(:, 1:h-1), F_0 = G - 1 z^T, z = G^T 1/n
    if F is None:  # group fairness: F = F_0(:, 1:h-1)
        counts = np.bincount(groups, minlength=h).astype(np.float64)
        z = counts / n
        F = np.zeros((n, max(h - 1, 0)))
        for col in range(h - 1):
            F[:, col] = (groups == col).astype(np.float64) - z[col]
    else:  # an explicit constraint matrix (Exp. 4's random F)
        F = np.asarray(F, dtype=np.float64).reshape(n, -1)
    C = s[:, None] * F
    cho = sla.cho_factor(C.T @ C) if C.shape[1] > 0 else None
    if sigma is None:
        sigma = float(abs(Ln).sum(axis=0).max())  # ||L_n||_1, max column sum
    if threads == 0:
        threads = len(os.sched_getaffinity(0))
    return SparseOperator(n, Ln, C, cho, float(sigma), d, normalized, threads)


@dataclasses.dataclass
class ArpackResult:
    evals: np.ndarray
    X: np.ndarray
    sigma: float
    matvecs: int


def sfairsc_arpack(op: SparseOperator, k: int, tol: float = 1e-12, ncv: int | None = None,
                   seed: int = 0, extra: int = 1, maxiter: int | None = None) -> ArpackResult:
    """Alg. 3 step 3: the k smallest eigenpairs of L^sigma with ARPACK."""
    count = [0]

    def mv(w):
        count[0] += 1 if w.ndim == 1 else w.shape[1]
        return op.apply(w)

    A = spla.LinearOperator((op.n, op.n), matvec=mv, dtype=np.float64)
    kk = k + extra
    if ncv is None:
        ncv = min(op.n, max(2 * kk + 1, 20))
    v0 = np.random.default_rng(seed).standard_normal(op.n)
    lam, X = spla.eigsh(A, k=kk, which="SA", tol=tol, ncv=ncv, v0=v0, maxiter=maxiter)
    order = np.argsort(lam)
    return ArpackResult(lam[order], X[:, order][:, :k], op.sigma, count[0])
