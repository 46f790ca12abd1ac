// libsfairsc — block thick-restart Lanczos driver (A7-A11 for
// b vectors at a time).  Alg. 3 step 3 computes the k smallest
// eigenpairs of L^sigma; the paper uses MATLAB eigs and leaves the
// Krylov method free ("modern Krylov subspace eigensolver").
//
// Basis V (column-major, ld = ldv): columns [0, pk) kept Ritz vectors, then
// blocks of b.  One expansion step on the newest block W = V[:, nv-b:nv]:
//   T  = L P W           spmm (P W is kept interleaved in bP by the previous step)
//   R  = finish(T)       = L^sigma W, fused with C1 = V^T R     (sweep 0)
//   R -= V C1, C2 = V^T R                                                   (sweep 1)
//   R -= V C2, Gram R^T R, B^T R                                            (sweep 2)
//   R = Q U (CholQR2), Q -> V[:, nv:nv+b], P Q -> bP                        (bqr1, bqr2)
// The projected matrix is recorded as the CGS coefficients: T[0:nv, nv-b:nv]
// = C1 + C2 = V^T L^sigma W (up to rounding), T[nv:nv+b, nv-b:nv] = U.  The
// Rayleigh-Ritz matrix is the symmetric completion of the upper block
// triangle (each column block's coefficients against all earlier columns), so
// thick restarts need no special arrow bookkeeping: the coupling of the
// residual block to the kept Ritz vectors is measured by the next step's C1.
// No host synchronisation inside a restart cycle; breakdowns (rank-deficient
// residual block) are flagged per step on the device and handled at the sync
// by rolling back to the step and injecting a random block.
#include "ctx.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <vector>

namespace sfz {

void symeig(int m, std::vector<double>& A, std::vector<double>& evals);

namespace {

struct BlockLanczos {
  sfairsc_ctx* c;
  int b, m, keep, k;
  int64_t applies = 0, steps = 0, restarts = 0, breakdowns = 0;
  unsigned inject = 0;
  double bd_tol = 0.0;

  BlockSweepArgs sargs(int J, const double* xin, double* xout, const double* coef) const {
    BlockSweepArgs a{};
    a.V = c->V;
    a.ld = c->ldv;
    a.J = J;
    a.xin = xin;
    a.xout = xout;
    a.coef = coef;
    a.bsum_t = c->bs_t;
    a.bsum_w = c->bs_v;
    a.sigma = c->sigma;
    a.partials = c->partials;
    a.counter = c->counters + 2;
    a.out = c->nb;
    return a;
  }

  double vb() const { return c->vb(); }

  // CGS2 of the block in bR against V[:, 0:J] and CholQR2 into V[:, J:J+b] / bP.
  // from_t: bR = finish(bT) fused into the first sweep (an expansion step, T recorded).
  sfairsc_status orth(int J, bool from_t) {
    const GraphDev g = c->g();
    const ProjDesc pd = c->pd();
    const int G = bsweep_grid(c->n);
    if (J > 0) {
      {
        ProfScope ps(c, K_DOTS, J * vb() + (from_t ? 2 * b * vb() + c->sgb() : b * vb()));
        launch_bsweep(from_t ? 0 : 3, b, g, pd, sargs(J, from_t ? c->bT : c->bR, c->bR, nullptr), G, c->st);
        launch_reduce_cols(c->partials, G, J * b, c->c1, c->st);
      }
      {
        ProfScope ps(c, K_UPDDOT, J * vb() + 2 * b * vb());
        launch_bsweep(1, b, g, pd, sargs(J, c->bR, c->bR, c->c1), G, c->st);
        launch_reduce_cols(c->partials, G, J * b, c->c2, c->st);
      }
    }
    {
      ProfScope ps(c, K_UPDNORM, J * vb() + 2 * b * vb() + c->sgb());
      launch_bsweep(2, b, g, pd, sargs(J, c->bR, c->bR, c->c2), G, c->st);
    }
    {
      ProfScope ps(c, K_NORMALIZE, (b > 1 ? 4 : 2) * b * vb() + b * vb() + c->sgb());
      if (b > 1) launch_bqr1(b, c->n, c->bR, c->nb, c->partials, c->counters + 5, c->g2, c->st);
      BlockQRArgs qa{};
      qa.nbo = c->nb;
      qa.g2 = b > 1 ? c->g2 : nullptr;
      qa.J = J;
      qa.T = from_t ? c->Tdev : nullptr;
      qa.ldT = c->ldT;
      qa.c1 = c->c1;
      qa.c2 = c->c2;
      qa.bs_v = c->bs_v;
      qa.flag = from_t ? c->bflags + J / b : c->bflags + kMaxJ;
      qa.bd_tol = bd_tol;
      qa.rel_tol = 1e-7;
      launch_bqr2(b, g, pd, c->bR, qa, c->V, c->ldv, c->bP, c->st);
    }
    CHECK_LAUNCH();
    return SFAIRSC_OK;
  }

  // random block orthogonalised against V[:, 0:J] into V[:, J:J+b] (start / breakdown)
  sfairsc_status random_block(int J) {
    for (int attempt = 0; attempt < 5; ++attempt) {
      launch_brandom(c->bR, c->n, b, c->seed, 1024u * inject++, 7u, c->st);
      launch_bgsum(b, c->g(), c->bR, c->partials, c->counters + 3, c->bs_w, c->st);
      launch_bproject(b, c->g(), c->pd(), c->bR, c->bs_w, c->bR, c->st);
      TRY(orth(J, false));
      int flag = 0;
      CU(cudaMemcpyAsync(c->hp, c->bflags + kMaxJ, sizeof(int), cudaMemcpyDeviceToHost, c->st));
      CU(cudaStreamSynchronize(c->st));
      std::memcpy(&flag, c->hp, sizeof(int));
      if (!flag) return SFAIRSC_OK;
    }
    return fail(SFAIRSC_E_NO_CONVERGENCE, "could not generate a random block outside the Krylov basis");
  }

  // one expansion step of the block at columns [nv - b, nv)
  sfairsc_status expand(int nv) {
    {
      ProfScope ps(c, K_SPMV, c->csr_bytes() + 2.0 * b * vb() + vb() + 1.0 * c->n);
      launch_spmm(c->g(), b, c->vs, c->row_split, c->spmv_grid, c->bP, c->bT, c->partials, c->counters + 1, c->bs_t,
                  c->st);
    }
    TRY(orth(nv, true));
    applies += b;
    steps++;
    return SFAIRSC_OK;
  }
};

}  // namespace

sfairsc_status eigs_block(sfairsc_ctx* c, int k, double tol, double* evals_out, double* evecs_out,
                          int evecs_memspace, sfairsc_stats* stats) {
  const double t0 = now_s();
  c->have_eigs = false;
  BlockLanczos L;
  L.c = c;
  L.b = c->bsz;
  L.m = c->m;
  L.k = k;
  L.keep = c->keep;
  const int b = L.b, mmax = L.m;
  const double tol_eff = std::min(tol, c->tol_cap);
  const double target = tol_eff * c->sigma;
  L.bd_tol = std::min(1e-12, 0.01 * tol_eff) * c->sigma;
  const int n = c->n;
  const int ldT = c->ldT;
  std::vector<double> Th((size_t)ldT * ldT, 0.0);  // host copy of the projected matrix (column-major)
  CU(cudaMemsetAsync(c->bflags, 0, sizeof(int) * (kMaxJ + 8), c->st));
  CU(cudaMemsetAsync(c->Tdev, 0, sizeof(double) * ldT * ldT, c->st));

  L.inject = 0;
  TRY(L.random_block(0));
  int nv = b;       // basis columns present (the newest block is not yet expanded)
  int pk = 0;       // kept Ritz vectors heading the basis
  int nsync = 0;    // first column whose T entries are not yet on the host
  bool converged = false, unreliable = false;
  std::vector<double> theta, Y;
  double gap = std::numeric_limits<double>::quiet_NaN();
  double max_resid = std::numeric_limits<double>::infinity();
  for (;;) {
    const int m = pk + b * ((mmax - pk) / b);  // this cycle's basis size ((m - pk) % b == 0)
    while (nv < m + b) {
      TRY(L.expand(nv));
      nv += b;
    }
    // ---- sync: T columns [nsync, m), per-step flags ----
    {
      const int c0 = std::max(nsync - b, pk);  // first expanded column since the last sync
      const int cols = m - c0;
      if (cols > 0)
        CU(cudaMemcpyAsync(Th.data() + (size_t)c0 * ldT, c->Tdev + (size_t)c0 * ldT, sizeof(double) * ldT * cols,
                           cudaMemcpyDeviceToHost, c->st));
      CU(cudaMemcpyAsync(c->hp, c->bflags, sizeof(int) * (kMaxJ / 1), cudaMemcpyDeviceToHost, c->st));
      CU(cudaStreamSynchronize(c->st));
      if (c->prof.on) c->prof.resolve();
    }
    int bad_nv = -1;
    {
      const int* fl = reinterpret_cast<const int*>(c->hp);
      for (int j = std::max(nsync, pk + b); j <= m; j += b)
        if (fl[j / b]) {
          bad_nv = j;
          break;
        }
    }
    if (bad_nv >= 0) {  // rank-deficient residual block at columns [bad_nv, bad_nv + b): roll back, inject
      if (c->debug) fprintf(stderr, "[sfairsc] block breakdown at column %d\n", bad_nv);
      L.breakdowns++;
      unreliable = true;
      CU(cudaMemsetAsync(c->bflags, 0, sizeof(int) * (kMaxJ + 8), c->st));
      TRY(L.random_block(bad_nv));
      nv = bad_nv + b;
      nsync = nv;
      continue;
    }
    nsync = m + b;

    // ---- Rayleigh-Ritz: symmetric completion of the upper block triangle ----
    std::vector<double> A((size_t)m * m, 0.0);
    for (int j = 0; j < m; ++j) {
      const int jb = j < pk ? j : pk + ((j - pk) / b) * b;  // first column of j's block
      for (int i = 0; i < m; ++i) {
        double v;
        const int ib = i < pk ? i : pk + ((i - pk) / b) * b;
        if (ib == jb) v = (j < pk) ? (i == j ? Th[(size_t)j * ldT + i] : 0.0)
                                   : 0.5 * (Th[(size_t)j * ldT + i] + Th[(size_t)i * ldT + j]);
        else if (i < j) v = (j < pk) ? 0.0 : Th[(size_t)j * ldT + i];
        else v = (i < pk) ? 0.0 : Th[(size_t)i * ldT + j];
        A[(size_t)i * m + j] = v;  // row-major for symeig
      }
    }
    Y = A;
    symeig(m, Y, theta);  // Y row-major: Y[l*m + col]
    // residual estimates ||U_last Y[m-b:m, i]||, U_last = T[m:m+b, m-b:m]
    double maxres = 0.0;
    for (int i = 0; i < k; ++i) {
      double ss = 0.0;
      for (int r = 0; r < b; ++r) {
        double acc = 0.0;
        for (int cc = r; cc < b; ++cc) acc += Th[(size_t)(m - b + cc) * ldT + m + r] * Y[(size_t)(m - b + cc) * m + i];
        ss += acc * acc;
      }
      maxres = std::max(maxres, std::sqrt(ss));
    }
    if (k < m) gap = theta[k] - theta[k - 1];
    bool done = maxres <= target;
    if (c->debug)
      fprintf(stderr, "[sfairsc] block RR restarts=%lld steps=%lld maxres=%g target=%g theta_k=%.17g\n",
              (long long)L.restarts, (long long)L.steps, maxres, target, theta[k - 1]);
    if (done || L.restarts >= c->max_restarts) {
      std::vector<double> Yc((size_t)m * k);
      for (int cc = 0; cc < k; ++cc)
        for (int l = 0; l < m; ++l) Yc[(size_t)cc * m + l] = Y[(size_t)l * m + cc];
      CU(cudaMemcpyAsync(c->Ydev, Yc.data(), sizeof(double) * Yc.size(), cudaMemcpyHostToDevice, c->st));
      {
        ProfScope ps(c, K_RITZ, (double)(m + k) * c->vb());
        launch_ritz(c->V, c->ldv, n, m, c->Ydev, k, c->X, c->st);
      }
      CHECK_LAUNCH();
      TRY(true_residuals(c, theta.data(), k, &max_resid));
      L.applies += k;
      // after a breakdown the cheap estimates miss the discarded residual: trust only the true residuals
      if (!unreliable || max_resid <= 10.0 * tol_eff || L.restarts >= c->max_restarts) {
        converged = done && (!unreliable || max_resid <= 10.0 * tol_eff);
        break;
      }
    }
    // ---- thick restart: keep the `keep` smallest Ritz pairs, the residual block follows ----
    pk = L.keep;
    std::vector<double> Yc((size_t)m * pk);
    for (int cc = 0; cc < pk; ++cc)
      for (int l = 0; l < m; ++l) Yc[(size_t)cc * m + l] = Y[(size_t)l * m + cc];
    CU(cudaMemcpyAsync(c->Ydev, Yc.data(), sizeof(double) * Yc.size(), cudaMemcpyHostToDevice, c->st));
    {
      ProfScope ps(c, K_RITZ, (double)(m + pk) * c->vb());
      launch_ritz(c->V, c->ldv, n, m, c->Ydev, pk, c->Vb, c->st);
    }
    CU(cudaMemcpyAsync(c->Vb + (long long)pk * c->ldv, c->V + (long long)m * c->ldv, sizeof(double) * c->ldv * b,
                       cudaMemcpyDeviceToDevice, c->st));
    CHECK_LAUNCH();
    std::swap(c->V, c->Vb);
    std::fill(Th.begin(), Th.end(), 0.0);
    for (int i = 0; i < pk; ++i) Th[(size_t)i * ldT + i] = theta[i];
    nv = pk + b;
    nsync = nv;
    L.restarts++;
  }

  if (c->prof.on) c->prof.resolve();
  c->evals.assign(theta.begin(), theta.begin() + k);
  c->k_eigs = k;
  c->have_eigs = true;
  for (int i = 0; i < k; ++i) evals_out[i] = theta[i];
  if (evecs_out) {
    const cudaMemcpyKind kind = evecs_memspace == SFAIRSC_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CU(cudaMemcpy2DAsync(evecs_out, sizeof(double) * n, c->X, sizeof(double) * c->ldv, sizeof(double) * n, k, kind,
                         c->st));
    CU(cudaStreamSynchronize(c->st));
  }
  sfairsc_stats S{};
  S.applies = L.applies;
  S.steps = L.steps;
  S.restarts = L.restarts;
  S.breakdowns = L.breakdowns;
  S.sigma = c->sigma;
  S.max_resid_rel = max_resid;
  S.gap_est = gap;
  S.t_build_s = c->t_build;
  S.t_eigs_s = now_s() - t0;
  S.converged = converged ? 1 : 0;
  S.basis_size = mmax;
  S.kept = L.keep;
  c->last = S;
  if (stats) *stats = S;
  if (!converged) return fail(SFAIRSC_E_NO_CONVERGENCE, "no convergence after %lld restarts", (long long)L.restarts);
  if (theta[k - 1] >= c->sigma * (1.0 - 1e-8))
    return fail(SFAIRSC_E_SHIFT_TOO_SMALL, "lambda_k=%g >= sigma(1-1e-8)=%g (Prop. 3.4)", theta[k - 1], c->sigma);
  return SFAIRSC_OK;
}

}  // namespace sfz
