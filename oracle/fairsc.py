"""Tier D oracle: dense FairSC (Algorithm 2) — TEST INFRASTRUCTURE ONLY.

Every step follows PAPER.md in the paper's order and notation; numpy/scipy
dense LAPACK routines serve as steps (SVD, eigh, solve).  fp64 throughout.
Pinned by tests/test_oracle_dense.py (brute force, h=1 -> SC, planted cliques,
expected-graph quotient, Prop. 3.1, Example B.2, Ky Fan).

Readings: R1 unnormalized = D -> I in §3 (RatioCut
relaxation, H^T H = I); R2 normalized projects with C = D^{-1/2} F; R4
sigma = ||L||_1 of the operator's Laplacian; R14 drop the last column of F_0.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import scipy.linalg as sla


class OracleInputError(ValueError):
    pass


def validate(W: np.ndarray, groups: np.ndarray, h: int) -> None:
    """w_ij >= 0, w_ii = 0, W symmetric, no isolated vertex (D > 0);
    P:152: every group non-empty."""
    if W.shape[0] != W.shape[1] or W.shape[0] != len(groups):
        raise OracleInputError("dimension mismatch")
    if np.any(W < 0):
        raise OracleInputError("negative weight")
    if np.any(np.diag(W) != 0):
        raise OracleInputError("nonzero diagonal")
    if not np.array_equal(W, W.T):
        raise OracleInputError("asymmetric W")
    if np.any(W.sum(axis=1) <= 0):
        raise OracleInputError("isolated vertex")
    if np.any(np.bincount(groups, minlength=h)[:h] == 0) or groups.min() < 0 or groups.max() >= h:
        raise OracleInputError("empty group / group id out of range")


def group_indicator(groups: np.ndarray, h: int) -> np.ndarray:
    """G of Eq. (group-vec): g_is = 1 iff v_i in V_s."""
    n = len(groups)
    G = np.zeros((n, h))
    G[np.arange(n), groups] = 1.0
    return G


def fairness_matrix(groups: np.ndarray, h: int) -> np.ndarray:
    """F = F_0(:, 1:h-1), F_0 = G - 1_n z^T, z = G^T 1_n / n (Lemma 2.1)."""
    G = group_indicator(groups, h)
    n = len(groups)
    z = G.T @ np.ones(n) / n
    F0 = G - np.outer(np.ones(n), z)
    return F0[:, : h - 1]


def laplacian(W: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """d_i = sum_j w_ij; L = D - W (Alg. 2 step 1 P:477)."""
    d = W.sum(axis=1)
    return np.diag(d) - W, d


def nullspace_basis(F: np.ndarray, rank_tol: float | None = None) -> np.ndarray:
    """Z = U(:, h:n) from the full SVD F = U Sigma V^T (Alg. 2 step 2).

    rank_tol (reading R21, a rank-deficient F of §8(f) N4): Z = null(F^T) = U(:, r:n) with
    r = #{i : Sigma_i > rank_tol Sigma_1}, the numerical rank (the textbook null space
    from the SVD).  None: F must have full column rank (Lemma 2.1(i) for group F)."""
    n, q = F.shape
    if q == 0:
        return np.eye(n)
    U, S, Vt = np.linalg.svd(F, full_matrices=True)
    if rank_tol is not None:
        r = int(np.sum(S > rank_tol * S[0])) if S[0] > 0 else 0
        return U[:, r:]
    if S[-1] <= 1e-12 * S[0]:
        raise OracleInputError("F rank deficient (Lemma 2.1(i) violated)")
    return U[:, q:]


@dataclasses.dataclass
class FairSCResult:
    evals: np.ndarray  # ascending, k_out values (k + extra)
    X: np.ndarray  # n x k, orthonormal comparison frame (R9)
    H: np.ndarray  # n x k, Alg. 2 step 6 output (normalized) or X (unnormalized)
    sigma: float
    gap: float  # lambda_{k+1} - lambda_k (nan when unavailable)


def sigma_norm1(L: np.ndarray) -> float:
    """sigma = ||L||_1, the max absolute column sum (reading R4)."""
    return float(np.max(np.abs(L).sum(axis=0)))


def fairsc_dense(W: np.ndarray, groups: np.ndarray, h: int, k: int, normalized: bool,
                 extra: int = 1) -> FairSCResult:
    """Algorithm 2 with the group-fairness F of Lemma 2.1."""
    validate(W, groups, h)
    return fairsc_dense_F(W, fairness_matrix(groups, h), k, normalized, extra)


def validate_W(W: np.ndarray) -> None:
    """w_ij >= 0, w_ii = 0, W symmetric, no isolated vertex (D > 0)."""
    if W.shape[0] != W.shape[1]:
        raise OracleInputError("dimension mismatch")
    if np.any(W < 0) or np.any(np.diag(W) != 0) or not np.array_equal(W, W.T) or np.any(W.sum(axis=1) <= 0):
        raise OracleInputError("W is not a valid weighted adjacency matrix")


def fairsc_dense_F(W: np.ndarray, F: np.ndarray, k: int, normalized: bool, extra: int = 1,
                   rank_tol: float | None = None) -> FairSCResult:
    """Algorithm 2 (FairSC), for a given constraint matrix F (n x r;
    the paper's algorithm takes F as its input).  Returns the k smallest
    eigenpairs of the fair-SC problem plus `extra` further eigenvalues.

    normalized (Alg. 2 as printed):
      1. L = D - W;  2. Z = null(F^T);  3. Q = (Z^T D Z)^{1/2};
      4. M = Q^{-1} Z^T L Z Q^{-1};  5. k smallest eigenpairs (lam, X_M) of M;
      6. H = Z Q^{-1} X_M.   Comparison frame X = D^{1/2} H (R9).
    unnormalized (R1, D -> I): eigenpairs of Z^T L Z, X = H = Z Y.
    """
    validate_W(W)
    n = W.shape[0]
    L, d = laplacian(W)  # step 1
    Z = nullspace_basis(np.asarray(F, dtype=np.float64).reshape(n, -1), rank_tol)  # step 2: Z = null(F^T)
    A = Z.T @ L @ Z
    A = 0.5 * (A + A.T)
    kk = min(k + extra, Z.shape[1])
    if normalized:
        S = Z.T @ (d[:, None] * Z)  # Z^T D Z (SPD)
        S = 0.5 * (S + S.T)
        ws, Es = np.linalg.eigh(S)
        Q = (Es * np.sqrt(ws)) @ Es.T  # step 3: principal square root (SPD)
        Qi_A = np.linalg.solve(Q, A)
        M = np.linalg.solve(Q, Qi_A.T).T  # step 4: Q^{-1} A Q^{-1}
        M = 0.5 * (M + M.T)
        lam, XM = np.linalg.eigh(M)  # step 5
        H = Z @ np.linalg.solve(Q, XM[:, :k])  # step 6
        X = np.sqrt(d)[:, None] * H
        Ln = L / np.sqrt(np.outer(d, d))
        sigma = sigma_norm1(Ln)
    else:
        lam, Y = np.linalg.eigh(A)
        X = Z @ Y[:, :k]
        H = X
        sigma = sigma_norm1(L)
    gap = float(lam[k] - lam[k - 1]) if len(lam) > k else float("nan")
    return FairSCResult(lam[:kk].copy(), X, H, sigma, gap)


# ----------------------------------------------------------------------------
# cross-check formulations (§3.2 variant and the deflated operator)
# ----------------------------------------------------------------------------

def operator_laplacian(W: np.ndarray, normalized: bool) -> np.ndarray:
    """L_n = D^{-1/2} L D^{-1/2} or L (R1)."""
    L, d = laplacian(W)
    if normalized:
        s = 1.0 / np.sqrt(d)
        return s[:, None] * L * s[None, :]
    return L


def constraint_matrix(W: np.ndarray, groups: np.ndarray, h: int, normalized: bool) -> np.ndarray:
    """C = D^{-1/2} F (Alg. 3 step 2 P:780-781); C = F for R1."""
    F = fairness_matrix(groups, h)
    if normalized:
        d = W.sum(axis=1)
        return F / np.sqrt(d)[:, None]
    return F


def variant_evals(W, groups, h, normalized) -> np.ndarray:
    """§3.2 variant: eigenvalues of L^v = V^T L_n V, V = orth. basis of null(C^T)."""
    C = constraint_matrix(W, groups, h, normalized)
    V = nullspace_basis(C)
    A = V.T @ operator_laplacian(W, normalized) @ V
    return np.linalg.eigvalsh(0.5 * (A + A.T))


def projector(C: np.ndarray) -> np.ndarray:
    """P = I - C (C^T C)^{-1} C^T."""
    n = C.shape[0]
    if C.shape[1] == 0:
        return np.eye(n)
    return np.eye(n) - C @ np.linalg.solve(C.T @ C, C.T)


def deflated_operator(W, groups, h, normalized, sigma=None) -> tuple[np.ndarray, float]:
    """L^sigma = P L_n P + sigma (I - P) (Eq. asigma); sigma = ||L_n||_1."""
    Ln = operator_laplacian(W, normalized)
    if sigma is None:
        sigma = sigma_norm1(Ln)
    P = projector(constraint_matrix(W, groups, h, normalized))
    n = W.shape[0]
    A = P @ Ln @ P + sigma * (np.eye(n) - P)
    return 0.5 * (A + A.T), float(sigma)


def apply_deflated(W, groups, h, normalized, w, sigma=None) -> np.ndarray:
    """L^sigma w = P(L_n(P w)) - sigma P w + sigma w, dense, one vector/column."""
    Ln = operator_laplacian(W, normalized)
    if sigma is None:
        sigma = sigma_norm1(Ln)
    P = projector(constraint_matrix(W, groups, h, normalized))
    Pw = P @ w
    return P @ (Ln @ Pw) - sigma * Pw + sigma * w


def constraint_matrix_F(W: np.ndarray, F: np.ndarray, normalized: bool) -> np.ndarray:
    """C = D^{-1/2} F or C = F (R1) for an explicit F."""
    if normalized:
        return F / np.sqrt(W.sum(axis=1))[:, None]
    return np.asarray(F, dtype=np.float64)


def variant_evals_F(W, F, normalized) -> np.ndarray:
    """§3.2 variant with an explicit F: eigenvalues of V^T L_n V, V = null(C^T)."""
    V = nullspace_basis(constraint_matrix_F(W, F, normalized))
    A = V.T @ operator_laplacian(W, normalized) @ V
    return np.linalg.eigvalsh(0.5 * (A + A.T))


def deflated_operator_F(W, F, normalized, sigma=None) -> tuple[np.ndarray, float]:
    """L^sigma = P L_n P + sigma (I - P) (Eq. asigma) with P from an explicit F."""
    Ln = operator_laplacian(W, normalized)
    if sigma is None:
        sigma = sigma_norm1(Ln)
    P = projector(constraint_matrix_F(W, F, normalized))
    A = P @ Ln @ P + sigma * (np.eye(W.shape[0]) - P)
    return 0.5 * (A + A.T), float(sigma)
