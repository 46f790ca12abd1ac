"""Config 5 at full size (n = 5e7, 1.6e9 stored entries): the SURVEY §8(c) host certificate
of the GPU eigensolve, plus two-seed agreement (reading R8).  Evidence run, not a bench value.

1. Generate the DC-SBM graph on the GPU (synth/dcsbm.py), copy the CSR to the host.
2. Two GPU solves (Alg. 3 steps 1-3 through the C ABI) from different start vectors
   (start_seed default and 0xC0FFEE); X_A, X_B copied to the host.
3. Oracle certificate on the host's cores, through the oracle's own operator (Tier S:
   the paper's apply P:803 with the normal-equations projector, scipy CSR):
     * every residual ||L^sigma x_i - lambda_i x_i|| / sigma, i = 1..64 (contract <= 1e-9);
     * the Rayleigh-Ritz values of X_A^T L^sigma X_A against lambda (reading R6);
     * ||C^T X|| / ||X|| (fairness, Lemma 2.1) and max |X^T X - I|;
     * sigma recomputed by the oracle (||L||_1) against the library's.
4. Two-seed agreement: lambda_A vs lambda_B (R6), sin angle(span X_A, span X_B) against
   the Davis-Kahan bound (||R_A|| + ||R_B||) sqrt(k) / gap (R8), gap = the solver's gap_est
   (theta_65 - theta_64 of its last Rayleigh-Ritz; no host solver reaches lambda_65 at this size).

    python tests/tools/cfg5_certificate.py [--n N] [--out profiles/r2_cfg5_certificate.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402
import torch  # noqa: E402

from oracle import sfairsc_cpu  # noqa: E402
from paper_2210_16435_b200 import lib  # noqa: E402
from synth.dcsbm import config5  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--out", default="gpurun_out/cfg5_certificate.json")
ap.add_argument("--seed-b", type=lambda s: int(s, 0), default=0xC0FFEE)
args = ap.parse_args()
dev = torch.device("cuda:0")
out = {"what": __doc__.split("\n")[0]}
T0 = time.time()


def log(**kw):
    out.update(kw)
    print(json.dumps({k: v for k, v in kw.items()}), flush=True)


t = time.time()
g, cfg = config5(n=args.n, device="cuda")
torch.cuda.synchronize()
k, n, h = cfg["k_eig"], g.n, g.h
host = {"row_ptr": g.row_ptr.cpu().numpy(), "col": g.col.cpu().numpy(), "groups": g.groups.cpu().numpy()}
log(n=n, nnz=int(g.nnz), h=h, k=k, gen_s=time.time() - t)


del g
torch.cuda.empty_cache()


def gpu_solve(seed):
    # the graph is regenerated on the GPU for each solve (same seed, same graph) and freed after the build, so
    # the library sizes its Krylov basis with the generator's memory returned (as in scripts/run_cfg5.py)
    g, _ = config5(n=args.n, device="cuda")
    torch.cuda.synchronize()
    torch.cuda.empty_cache()  # generator intermediates back to the driver before the library sizes its basis
    ctx = lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, g.groups, k, False, h=h, start_seed=seed)
    del g
    torch.cuda.empty_cache()
    X = torch.empty((k, n), dtype=torch.float64, device=dev)
    t0 = time.time()
    ev, _, st = lib.sfairsc_eigs(ctx, k, cfg["tol"], evecs=X)
    torch.cuda.synchronize()
    st = dict(st, eigs_wall_s=time.time() - t0)
    ctx.close()
    Xh = X.cpu().numpy()  # (k, n): rows are the eigenvectors
    del X
    torch.cuda.empty_cache()
    return np.asarray(ev), Xh, st


evA, XA, stA = gpu_solve(0)
log(solve_A={kk: stA[kk] for kk in ("applies", "restarts", "max_resid_rel", "gap_est", "sigma", "eigs_wall_s",
                                    "basis_size", "kept", "converged")})
evB, XB, stB = gpu_solve(args.seed_b)
log(solve_B={kk: stB[kk] for kk in ("applies", "restarts", "max_resid_rel", "gap_est", "sigma", "eigs_wall_s",
                                    "basis_size", "kept", "converged")})
# ---- two-seed agreement (before the oracle build: X_B is freed afterwards) ----
# sin of the largest principal angle = ||X_B - X_A (X_A^T X_B)||_2 (oracle.metrics.subspace_sin's formula, with the
# QR skipped: both bases are orthonormal to ~1e-12, checked below); R^T R accumulated over row chunks so that no
# n x k temporary is formed (n = 5e7)
sigma_lib = stA["sigma"]
M = XA @ XB.T  # (k, k) = X_A^T X_B in column form
RtR = np.zeros((k, k))
for r0 in range(0, n, 1 << 22):
    R = XB[:, r0:r0 + (1 << 22)] - M.T @ XA[:, r0:r0 + (1 << 22)]
    RtR += R @ R.T
sin = float(np.sqrt(max(0.0, np.linalg.eigvalsh(RtR)[-1])))
r6ab = np.abs(evB - evA) <= 1e-8 * np.abs(evA) + 1e-12 * sigma_lib
gap = float(stA["gap_est"])
bound = (stA["max_resid_rel"] + stB["max_resid_rel"]) * sigma_lib * np.sqrt(k) / gap
log(lambda_A=[float(x) for x in evA], lambda_B_minus_A=[float(x) for x in evB - evA], seeds_r6_ok=bool(r6ab.all()),
    sin_angle_AB=sin, davis_kahan_bound=float(bound), gap_est_solver=gap,
    angle_within_bound=bool(sin <= max(1e-6, 2 * bound)), orth_err_B=float(np.abs(XB @ XB.T - np.eye(k)).max()))
del XB, R

# ---- oracle certificate (host) ----
t = time.time()
W = sp.csr_matrix((np.ones(len(host["col"])), host["col"], host["row_ptr"]), shape=(n, n))
op = sfairsc_cpu.build_operator(W, host["groups"].astype(np.int64), h, False, threads=0)
del W
log(oracle_build_s=time.time() - t, oracle_threads=op.threads, oracle_sigma=op.sigma,
    sigma_rel_diff=abs(op.sigma - stA["sigma"]) / op.sigma)
sigma = op.sigma
t = time.time()
res, XtAX = [], np.empty((k, k))
AX_cols = []
for i in range(k):
    x = np.ascontiguousarray(XA[i])
    ax = op.apply(x)
    res.append(float(np.linalg.norm(ax - evA[i] * x) / sigma))
    AX_cols.append(XA @ ax)  # column i of X^T A X (k-vector)
XtAX = np.stack(AX_cols, axis=1)
theta = np.linalg.eigvalsh(0.5 * (XtAX + XtAX.T))
r6 = np.abs(theta - evA) <= 1e-8 * np.abs(evA) + 1e-12 * sigma
G = XA @ XA.T
CtX = op.C.T @ XA.T
log(oracle_apply_s=time.time() - t, resid_max=max(res), resid_all=res,
    rr_vs_lambda_max_abs=float(np.max(np.abs(theta - evA))), rr_r6_ok=bool(r6.all()),
    orth_err=float(np.abs(G - np.eye(k)).max()),
    CtX_rel=float(np.linalg.norm(CtX) / np.linalg.norm(XA)), lambda1_rel=float(abs(evA[0]) / sigma),
    total_s=time.time() - T0)

out["contract"] = {"resid<=1e-9": max(res) <= 1e-9, "rr_r6": bool(r6.all()), "seeds_r6": bool(r6ab.all()),
                   "angle<=max(1e-6,2*DK)": bool(sin <= max(1e-6, 2 * bound)),
                   "CtX_rel<=1e-10": out["CtX_rel"] <= 1e-10, "orth<=1e-11": out["orth_err"] <= 1e-11}
os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
with open(args.out, "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out["contract"]), flush=True)
