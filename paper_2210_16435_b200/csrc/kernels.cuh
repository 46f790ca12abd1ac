// Internal kernel launch interface of libsfairsc (not part of the C ABI).
// All launches are asynchronous on `st`; callers check errors.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace sfz {

constexpr int kThreads = 256;  // CTA size of every streaming kernel
constexpr int kHB = 16;        // group sums fused per kernel (h > 16: extra gsum passes)
constexpr int kMaxJ = 512;
constexpr int kPairMaxM = 186;  // paired Lanczos steps (lanczos1.cu): basis size limit of the pair sweep     // max Krylov basis columns handled by the sweep kernels
constexpr int kBT = kHB + 1;   // per-vector stride of the SpMV epilogue output: B^T t (kHB) and p^T t

// Factored projector coefficients (DESIGN.md §Factored projector).
//   b_s   = sum_{i in V_s} s_i x_i          (B^T x, B = [s o g_1 ... s o g_h])
//   c_s   = scale * b_s * isb_s              (isb_s = beta_s^{-1/2}, beta_s = sum_{i in V_s} s_i^2)
//   pi    = sum_s uh_s c_s                   (uh = u/|u|, u_s = |V_s| isb_s)
//   gam_s = (c_s - uh_s pi) * isb_s          so that  Q Q^T x = s o gam_{g(i)}
// Dense mode (§8(f) N4, general constraints C^T H = 0 with a dense F): Q (n x r, row-major, ld = ldq,
// orthonormal columns spanning range(C)) replaces the group structure; h = r, QQ^T x = Q gam with
// gam = Q^T x (gamma_serial is the identity), B^T x := Q^T x.
struct ProjDesc {
  int h;
  const double* isb;  // device, h
  const double* uh;   // device, h
  const double* Q = nullptr;  // dense mode: n x r row-major
  int ldq = 0;
};

struct GraphDev {
  int n;
  int nnz;
  const int* rp;
  const int* ci;
  const double* vv;   // normalized: s_i w_ij s_j ; unnormalized: w_ij
  const double* dg;   // degrees d (unnormalized diagonal of L)
  const double* s;    // d^{-1/2} (normalized only; nullptr otherwise)
  const uint8_t* grp;
  bool normalized;
  // dense projector (§8(f) N4): Q (n x qr, row-major, ld = ldq); nullptr: group-factored projector
  const double* Q = nullptr;
  int ldq = 0, qr = 0;
  bool skewed = false;  // heavy-tailed degrees: the SpMV gives rows longer than 32 VS slots a whole warp
  // unit weights (every stored w_ij = 1, no diagonal entries): the single-vector SpMV streams only the
  // column indices; normalized graphs then gather q = s o p and scale the row sum by s_i
  bool unit = false;
};

// ---- build-time kernels -----------------------------------------------------
void launch_validate_csr(const GraphDev& g, int check_sym, int* flags, cudaStream_t st);
void launch_degrees(const GraphDev& g, double* d, int* flags, cudaStream_t st);
void launch_scale_values(const int* rp, const int* ci, double* vv, const double* s, int n, cudaStream_t st);
void launch_inv_sqrt(const double* d, double* s, int n, cudaStream_t st);
// q = s o p (normalized unit-weight SpMV input)
void launch_scale_vec(const double* s, const double* p, double* q, int n, cudaStream_t st);
// row sums of |L| columns -> max into *out (sigma = ||L||_1)
void launch_sigma(const GraphDev& g, double* partials, unsigned* counter, double* out, cudaStream_t st);
void launch_group_check(const int32_t* groups, int n, int h, uint8_t* grp, int* flags, cudaStream_t st);

// ---- per-apply kernels --------------------------------------------------------
// bsum[g_base .. g_base+16) = sum over V_s of (s_i) x_i
void launch_gsum(const GraphDev& g, const double* x, int g_base, double* partials, unsigned* counter,
                 double* bsum, cudaStream_t st);
// p = x - s o gam(bsum, scale)_g
void launch_project(const GraphDev& g, const ProjDesc& pd, const double* x, const double* bsum, double scale,
                    double* p, cudaStream_t st);
// t = L p ; bsum_t[0..16) = B^T t, bsum_t[16] = p^T t (fused epilogue)
void launch_spmv(const GraphDev& g, int vs, const int* row_split, int grid, const double* p, double* t,
                 double* partials, unsigned* counter, double* bsum_t, cudaStream_t st);
// y = t - s o (gam_t - sigma gam_w)_g ;  optional dot w^T y -> *dot
void launch_finish(const GraphDev& g, const ProjDesc& pd, const double* t, const double* bsum_t,
                   const double* bsum_w, double sigma, double* y, cudaStream_t st);

// ---- Krylov kernels -------------------------------------------------------------
// mode 0: r = finish(t); partial dots V[:,0:J]^T r
// mode 1: r' = r - V c ; partial dots V^T r'
// mode 2: r'' = r - V c ; partial |r''|^2 and B^T r''  (ticket-reduced into norm_bsum[0..17))
// mode 3: partial dots V^T x (x unchanged)
struct SweepArgs {
  const double* V;
  long long ld;
  int J;
  const double* xin;   // mode 0: t ; else r
  double* xout;        // r out (modes 0,1,2)
  const double* coef;  // device coef (modes 1,2)
  const double* bsum_t;
  const double* bsum_w;
  double sigma;
  double* partials;    // [grid][J] (modes 0,1,3) or [grid][17] (mode 2)
  unsigned* counter;
  double* norm_bsum;   // mode 2 output: [0] = |r''|^2, [1..17) = B^T r''
};
int sweep_grid(int n, int num_sms);
long long launch_count();  // kernels launched by this process so far
void launch_sweep(int mode, const GraphDev& g, const ProjDesc& pd, const SweepArgs& a, int grid, cudaStream_t st);
// TMA-fed persistent sweeps (krylov.cu); J <= 192, grid <= #SMs
bool sweep_tma_ok(int J);
int sweep_tma_grid(int n, int num_sms);
void launch_sweep_tma(int mode, const GraphDev& g, const ProjDesc& pd, const SweepArgs& a, int grid, cudaStream_t st);
void launch_ritz_rb(const double* V, long long ld, int n, int m, const double* Y, int p, double* Vout,
                    cudaStream_t st);
// out[l] = sum_b partials[b*J + l], fixed order
void launch_reduce_cols(const double* partials, int G, int J, double* out, cudaStream_t st);
// v = r / beta -> vout ; bsum_v = bsum_r / beta ; p = v - s o gam(bsum_v)
struct NormArgs {
  const double* nb;   // [0] = |r|^2, [1..1+h) = B^T r
  double beta_host;   // > 0: use this beta instead of sqrt(nb[0])
  double bd_tol;      // beta <= bd_tol -> breakdown flag
  int j;              // Lanczos index: records alpha_dev[j], beta_dev[j]
  const double* c1;   // CGS coefficients (alpha_j = c1[j] + c2[j])
  const double* c2;
  double* alpha_dev;  // nullptr: do not record
  double* beta_dev;
  int* flag;
};
void launch_normalize(const GraphDev& g, const ProjDesc& pd, const double* r, const NormArgs& na, double* vout,
                      double* bsum_v, double* p, cudaStream_t st);
// x_i = u_i - 1/2, u = Philox4x32-10(key=seed, ctr=(i, c1, stream, 0))
void launch_random(double* x, int n, uint64_t seed, unsigned c1, unsigned stream, cudaStream_t st);
// Vout[:, c] = sum_l V[:, l] Y[l, c]   (c < p, l < m), Y column-major m x p on device
void launch_ritz(const double* V, long long ld, int n, int m, const double* Y, int p, double* Vout,
                 cudaStream_t st);
// out = |y - theta x|^2 (ticket reduced)
void launch_resid(const double* y, const double* x, double theta, int n, double* partials, unsigned* counter,
                  double* out, cudaStream_t st);
// the same with theta read on the device (*theta_dev)
void launch_resid_dev(const double* y, const double* x, const double* theta_dev, int n, double* partials,
                      unsigned* counter, double* out, cudaStream_t st);
// out = x^T y (ticket reduced)
void launch_dot(const double* x, const double* y, int n, double* partials, unsigned* counter, double* out,
                cudaStream_t st);
// Chebyshev step (§8(f) N2): y_new = a (L^sigma y_cur - cc y_cur) + b y_prev, L^sigma y_cur = finish(t) with
// t = L P y_cur (bsum_t = B^T t, bsum_w = B^T y_cur); group projector only; y_new may alias y_prev
void launch_finish_cheb(const GraphDev& g, const ProjDesc& pd, const double* t, const double* bsum_t,
                        const double* bsum_w, double sigma, const double* ycur, const double* yprev, double a,
                        double cc, double b, double* ynew, cudaStream_t st);

// ---- block Krylov kernels (block.cu) ---------------------------------
// NB in {1, 2, 4}; blocks of NB n-vectors are interleaved (row-major, ldv rows x NB).
constexpr int kBMaxJ = 192;  // max basis columns of a block sweep (TMA box + smem ring)
struct BlockSweepArgs {
  const double* V;     // basis, column-major, ld
  long long ld;
  int J;               // columns of V swept (0 allowed)
  const double* xin;   // interleaved block in (mode 0: T = L P)
  double* xout;        // interleaved block out (modes 0, 1, 2)
  const double* coef;  // [J][NB] (modes 1, 2)
  const double* bsum_t;  // [NB][kBT] B^T T (+ P^T T)   (mode 0)
  const double* bsum_w;  // [NB][kHB] B^T W   (mode 0, W = current basis block)
  double sigma;
  double* partials;    // [grid][J*NB] dots, or [grid][NB*(NB+kHB)] (mode 2)
  unsigned* counter;
  double* out;         // mode 2: [c*(NB+kHB) + j]: Gram row c (j < NB), B^T r_c (j = NB + s)
};
struct BlockQRArgs {
  const double* nbo;   // mode-2 sweep output (Gram, B^T R)
  const double* g2;    // Gram after pass 1 (NB*NB) or nullptr (single pass)
  int J;               // first new basis column (= nv, columns orthogonalised against)
  double* T;           // projected matrix (column-major, ldT) or nullptr (no record)
  int ldT;
  const double* c1;    // [nv][NB] CGS coefficients (pass 1, pass 2 may be nullptr)
  const double* c2;
  double* bs_v;        // out: B^T Q, [NB][kHB]
  int* flag;           // breakdown flag
  double bd_tol;       // absolute pivot tolerance
  double rel_tol;      // relative pivot tolerance (ill-conditioned block)
};
// p: the gathered vector indexed by ci; p_self (nullptr: p): this part's own rows (diagonal term)
void launch_spmm(const GraphDev& g, int nb, int vs, const int* split, int grid, const double* p, double* t,
                 double* partials, unsigned* counter, double* bsum_t, cudaStream_t st,
                 const double* p_self = nullptr);
int bsweep_grid(int n);
// column-blocked single-vector SpMV (cmode 1 first, 2 middle, 3 last block; g.rp = the block's row offsets)
void launch_spmv_colblock(const GraphDev& g, int vs, const int* split, int grid, const double* p, double* t,
                          double* partials, unsigned* counter, double* bsum_t, int cmode, cudaStream_t st,
                          const double* p_self = nullptr);
void launch_colblk_starts(const int* rp, const int* ci, int n, int nblk, int cb, int* cnt, cudaStream_t st);
void launch_colblk_scatter(const int* rp, const int* ci, const double* vv, int n, int nblk, const int* rpb, int* ci2,
                           double* vv2, cudaStream_t st);
void launch_bsweep(int mode, int nb, const GraphDev& g, const ProjDesc& pd, const BlockSweepArgs& a, int grid,
                   cudaStream_t st);
void launch_bqr1(int nb, int n, double* R, const double* nbo, double* partials, unsigned* counter, double* g2,
                 cudaStream_t st);
void launch_bqr2(int nb, const GraphDev& g, const ProjDesc& pd, const double* R, const BlockQRArgs& qa, double* V,
                 long long ld, double* p, cudaStream_t st);
void launch_bgsum(int nb, const GraphDev& g, const double* x, double* partials, unsigned* counter, double* out,
                  cudaStream_t st);
void launch_bproject(int nb, const GraphDev& g, const ProjDesc& pd, const double* x, const double* bsum, double* y,
                     cudaStream_t st);
void launch_brandom(double* x, int n, int nb, uint64_t seed, unsigned c1, unsigned stream, cudaStream_t st);
// pair apply (two vectors through one b = 2 SpMM): out[c*kHB + s] = B^T x_c; p = (P x0, P x1) interleaved;
// y_c = t_c - s o (gam(B^T t_c) - sigma gam(B^T x_c))_g unpacked
void launch_pair_gsum(const GraphDev& g, const double* x0, const double* x1, double* partials, unsigned* counter,
                      double* out, cudaStream_t st);
void launch_pair_project(const GraphDev& g, const ProjDesc& pd, const double* x0, const double* x1,
                         const double* bsum, double* p, cudaStream_t st);
void launch_pair_finish(const GraphDev& g, const ProjDesc& pd, const double* t, const double* bsum_t,
                        const double* bsum_x, double sigma, double* y0, double* y1, cudaStream_t st);

// TMA-fed single-vector SpMV (spmv_tma.cu): t = L p + epilogue B^T t, p^T t (same outputs as launch_spmv)
struct SpmvTileShape {  // row-aligned tiles of <= tn padded entries and <= tr rows; `stages`-deep smem ring
  int tn = 2048, tr = 128, stages = 2;
  int val_off = 0, col_off = 0, rp_off = 0, ps_off = 0, ds_off = 0, gr_off = 0, stage_bytes = 0;
};
SpmvTileShape spmv_tile_shape(int tn, int tr, int stages, bool unit);
int spmv_tma_ctas_per_sm(int vs, bool normalized, bool unit, const SpmvTileShape& S);
void spmv_tma_layout(const int* hrp, int n, int G, const SpmvTileShape& S, std::vector<int>& prp,
                     std::vector<int2>& tiles, std::vector<int>& cta_tiles);
void launch_pad_csr(const int* rp, const int* ci, const double* vv, int n, const int* prp, int* pci, double* pvv,
                    cudaStream_t st);
void launch_spmv_tma(const GraphDev& g, int vs, const SpmvTileShape& S, const int2* tiles, const int* cta_tiles,
                     int grid, const double* p, const double* p_self, double* t, double* partials, unsigned* counter,
                     double* bsum_t, cudaStream_t st);

// ---- dense constraint basis (§8(f) N4) -----------------------------------------------
// out[a*r + b] (a <= b) = sum_i M(i,a) M(i,b), M(i,a) = M[i*rs + a*cs] (fixed-order block reduction)
void launch_gram_pairs(const double* M, long long rs, long long cs, int n, int r, double* out, cudaStream_t st);
void launch_scale_rows(double* M, long long ld, int n, int r, const double* s, cudaStream_t st);
constexpr int kMaxFCols = 64;  // dense constraint matrix F: at most 64 columns (numerical rank <= kHB)
// Qout (row-major, ldq; columns rq..ldq zeroed) = M T, T: r x rq row-major (device), r <= 64, rq <= 16
void launch_rows_times(const double* Min, long long rs, long long cs, int n, int r, int rq, const double* T,
                       double* Qout, int ldq, cudaStream_t st);

// ---- k-means ----------------------------------------------------------------------
void launch_build_rows(const double* X, long long ldx, int n, int k, const double* s, double* H, cudaStream_t st);
void launch_d2_update(const double* H, int n, int k, const double* center, int first, double* D2, double* blocksum,
                      int nblk, cudaStream_t st);
void launch_pp_select(const double* D2, const double* blocksum, int nblk, int n, double u, int* chosen,
                      cudaStream_t st);
void launch_gather_center(const double* H, int k, const int* idx, double* center, cudaStream_t st);
void launch_assign(const double* H, int n, int k, int K, const double* mu, int* labels, double* dist,
                   int* changes, cudaStream_t st);
void launch_centroid_partials(const double* H, int n, int k, int K, const int* labels, double* partials, int grid,
                              cudaStream_t st);
int centroid_grid(int n, int num_sms);
void launch_centroid_finish(const double* partials, int grid, int k, int K, double* mu, double* counts,
                            cudaStream_t st);
void launch_argmax_excluding(const double* dist, const int* used_mask, int n, int* out, double* scratch,
                             cudaStream_t st);
void launch_sum(const double* x, int n, double* partials, unsigned* counter, double* out, cudaStream_t st);

}  // namespace sfz
