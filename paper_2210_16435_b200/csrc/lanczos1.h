// Single-sweep (lagged) Lanczos kernels (lanczos1.cu), shared with the
// row-partitioned driver (dist.cu).  Internal, not part of the C ABI.
#pragma once
#include "kernels.cuh"

#include <vector>

namespace sfz {

// scalar slots of the device state `lz`
enum { LZ_OMEGA = 0, LZ_PNORM2 = 1, LZ_AY = 2, LZ_AV = 3, LZ_MU = 4, LZ_INVMU = 5, LZ_BETA = 6,
       // paired steps (two Lanczos steps per basis sweep): the stored odd column
       // LZ_PEND (-1: none) awaits its move to the orthonormal basis (defect e in epend, rho in
       // LZ_PRHO); LZ_CONV (-1: none) = the column the next sweep rewrites (econv, LZ_CRHO), while the
       // coefficient vectors are converted to the stored basis; LZ_INVMU_A = 1/mu of the pair's first step
       LZ_PEND = 7, LZ_PRHO = 8, LZ_CONV = 9, LZ_CRHO = 10, LZ_INVMU_A = 11 };

struct LzDev {
  double* H;       // (ldH x ldH) column-major; A V_j = V_j H[:j,:j] + v~_j H[j,:j] (lagged)
  int ldH;
  double* s;       // V_j^T v~_j (j entries)
  double* lz;      // scalars (LZ_*)
  double* cs;      // s / mu        (update coefficients of v_j)
  double* cg;      // g             (update coefficients of w)
  const double* bs_t;  // B^T t [kHB], p~^T t at [kHB]
  const double* bs_v;  // B^T v~ [kHB]
  int* flag;       // breakdown flag of this step
  double sigma;
  double bd_tol;
  double* epend;   // paired steps: defect V^T v' of the pending odd column (LZ_PEND)
  double* econv;   // the defect of the column being rewritten (LZ_CONV)
};

struct LzSweepArgs {
  const double* V;
  long long ld;
  int J;
  const double* vt;   // v~
  const double* t;    // L p~
  double* vj_out;     // V column J
  double* w_out;
  const double* cs;
  const double* cg;
  const double* lz;
  const double* bs_t;
  const double* bs_v;
  double sigma;
  double* partials;   // [grid][J+1]
  double* partials2;  // [grid][1+kHB]
  unsigned* counter;
  double* nb;         // out: |w|^2, B^T w
};

// coefficient step (one CTA): reads s, H, lz, bs_t[kHB] = p~^T t; writes H column j, cs, cg, lz
void launch_lz_coef(const LzDev& d, int j, cudaStream_t st);
// the one basis sweep of step J = a.J (TMA-fed): v_J, w, partial dots -> a.partials, |w|^2 and B^T w -> a.nb
void launch_lz_update(const GraphDev& g, const ProjDesc& pd, const LzSweepArgs& a, int grid, cudaStream_t st);
// v~ = p~ = P(w/|w|) -> vt, p; s = dots/|w| (nd entries); H row jrow (jrow >= 0); B^T v~ -> bs_v
void launch_lz_norm(const GraphDev& g, const ProjDesc& pd, const double* w, const double* nb, const double* dots,
                    int nd, const LzDev& d, int jrow, double* vt, double* p, double* bs_v, cudaStream_t st,
                    double* q = nullptr);

// the pair sweep of two Lanczos steps (k_lz_pair)
struct LzPairArgs {
  const double* V;
  long long ld;
  int J;
  const double* vtA;  // v~_j
  const double* vtB;  // v~_{j+1}
  const double* t;    // L p~_{j+1}
  double* vj_out;     // V[:, J]
  double* vj1_out;    // V[:, J + 1]
  double* w_out;
  double* conv_out;   // V[:, conv] (nullptr: no rewrite)
  const double* cA;   // step j: s/mu (stored basis, J)
  const double* cB;   // step j+1: s/mu (J + 1)
  const double* gB;   // step j+1: g (J + 1)
  const double* tr;   // rewrite coefficients (J; zero beyond the rewritten column)
  const double* lz;
  const double* bs_t;
  const double* bs_v;
  double sigma;
  double* partials;   // [grid][2J + 3]
  double* partials2;  // [grid][2 + kHB]
  unsigned* counter;
  double* nb;
};

// paired steps: the three-term vector of the pair's first step (+ its g_far dots; fix_h:
// this call owns the replicated H / lz updates), the pair sweep, and the post-sweep dot bookkeeping
void launch_lz_three(const GraphDev& g, const ProjDesc& pd, const double* t, const double* vt, const double* vprev,
                     const LzDev& d, int j, double* u_out, double* dots, double* cA, double* tr, double* partials,
                     unsigned* counter, double* nb, int grid, bool fix_h, cudaStream_t st);
void launch_lz_pair(const GraphDev& g, const ProjDesc& pd, const LzPairArgs& a, int grid, cudaStream_t st);
void launch_lz_pairpost(const LzDev& d, int J, const double* dd2, double* dd, const double* nb, const int* flags,
                        cudaStream_t st);
// host side of the pending odd column's basis change at a restart sync (H, lagged row, s), and the Ritz
// coefficients back to the stored columns
void pair_pending_to_orthonormal(int m, int ldH, std::vector<double>& Hh, std::vector<double>& sh, const double* e,
                                 double rho);
void pair_coef_to_stored(int m, double* x, const double* e, double rho);

}  // namespace sfz
