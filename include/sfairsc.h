/*
 * sfairsc.h — C ABI of the B200 (sm_100a) s-FairSC eigensolver library.
 *
 * Method: Scalable FairSC, Wang, Lu, Davidson, Bai (arXiv 2210.16435),
 * Algorithm 3.  The library computes the k smallest
 * eigenpairs of the Hotelling-deflated, nullspace-projected fair-SC operator
 *
 *     L^sigma = P L P + sigma (I - P)                       Eq. asigma
 *     L^sigma w = P(L(P w)) - sigma P w + sigma w
 *
 * with P = I - Q Q^T the orthogonal projector onto null(C^T) (Eq. pmat2,
 * P:566-569; P = I - C (C^T C)^{-1} C^T) and
 *   normalized: L = L_n = D^{-1/2}(D - W)D^{-1/2}, C = D^{-1/2} F;
 *   unnormalized (reading R1): L = D - W, C = F;
 * F = F_0(:, 1:h-1), F_0 = G - 1_n z^T, z = G^T 1_n / n (Lemma 2.1);
 * sigma = ||L||_1.  By Prop. 3.4 the k smallest
 * eigenvectors X of L^sigma solve the fair-SC problem, with
 * H = D^{-1/2} X (H = X for R1).
 *
 * Conventions for every entry point
 *  - Return value: SFAIRSC_OK or an error status; on error, outputs are left
 *    untouched (exception: SFAIRSC_E_NO_CONVERGENCE still fills the best
 *    Ritz values/vectors and stats).  sfairsc_last_error() gives
 *    a thread-local message for the last non-OK status.
 *  - Ownership: input arrays are borrowed for the duration of the call only;
 *    the context copies what it needs into library-owned device memory and
 *    owns it until sfairsc_destroy().  Output arrays are caller-allocated.
 *  - memspace: SFAIRSC_MEM_HOST = ordinary host pointer (pinned or pageable),
 *    SFAIRSC_MEM_DEVICE = CUDA device pointer on the context's device.
 *  - Matrices of n-vectors are column-major with leading dimension n.
 *  - All work is enqueued on the context's stream (opts.cuda_stream, or a
 *    stream the library creates); every call returns with that stream
 *    synchronised.  Calls on one context must not run concurrently.
 *  - Determinism: for fixed inputs, options and GPU, results are bitwise
 *    reproducible (fixed-order reductions, no floating-point atomics).
 *  - Precision: fp64 arithmetic throughout (indices int32).
 */
#ifndef SFAIRSC_H
#define SFAIRSC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sfairsc_ctx sfairsc_ctx; /* opaque; owns all device memory */
typedef struct sfairsc_comm sfairsc_comm; /* opaque NCCL communicator of a row-partitioned job */

typedef enum {
  SFAIRSC_OK = 0,
  SFAIRSC_E_INVALID_ARG = 1,      /* bad scalar argument / null pointer / group id out of [0,h) */
  SFAIRSC_E_DIM_MISMATCH = 2,     /* n_rows != n_cols, ... */
  SFAIRSC_E_CSR_INVALID = 3,      /* row_ptr not monotone / col out of range / unsorted or duplicate columns / nonzero diagonal (w_ii = 0) */
  SFAIRSC_E_ASYMMETRIC = 4,       /* W != W^T (undirected graph) */
  SFAIRSC_E_NEGATIVE_WEIGHT = 5,  /* w_ij < 0 */
  SFAIRSC_E_ISOLATED_VERTEX = 6,  /* d_i = 0; the paper assumes D > 0 */
  SFAIRSC_E_EMPTY_GROUP = 7,      /* some V_s empty */
  SFAIRSC_E_RANK_DEFICIENT = 8,   /* rank F < h-1 (cannot happen for non-empty groups, Lemma 2.1(i)) */
  SFAIRSC_E_K_TOO_LARGE = 9,      /* k > n - h + 1 (dimension of null(C^T)) or k > build k */
  SFAIRSC_E_SHIFT_TOO_SMALL = 10, /* some wanted lambda_i >= sigma (1 - 1e-8): Prop. 3.4 precondition violated */
  SFAIRSC_E_NO_CONVERGENCE = 11,  /* max_restarts reached; best Ritz pairs returned */
  SFAIRSC_E_STATE = 12,           /* call order (build -> eigs -> embed_kmeans) violated */
  SFAIRSC_E_OOM = 13,             /* device allocation failed */
  SFAIRSC_E_CUDA = 14,            /* CUDA runtime error (message in sfairsc_last_error) */
  SFAIRSC_E_NCCL = 15             /* reserved: multi-GPU communicator error */
} sfairsc_status;

enum { SFAIRSC_MEM_HOST = 0, SFAIRSC_MEM_DEVICE = 1 };

/* Weighted adjacency W as CSR: row_ptr[n_rows+1], col_idx[nnz],
 * values[nnz]; both triangles stored; columns strictly increasing within a
 * row; w_ij >= 0; no stored nonzero diagonal.  Single-GPU: n_rows == n_cols,
 * row_offset == 0.  int32 indices: nnz < 2^31. */
typedef struct {
  int64_t n_rows, n_cols, nnz, row_offset;
  const int32_t *row_ptr;
  const int32_t *col_idx;
  const double *values;
  int32_t memspace;
} sfairsc_csr;

/* Options of the extended build.  sfairsc_default_opts() fills defaults. */
typedef struct {
  double sigma_override;  /* <= 0: sigma = ||L||_1; > 0: use this shift (must exceed lambda_k, Prop. 3.4) */
  int32_t max_basis;      /* Lanczos basis size m; 0: min(192, max(2k+10, 3.4k, 20)) (SPEC S:342 suggests 2k+10), capped at n and to fit HBM */
  int32_t keep;           /* Ritz vectors kept at a thick restart; 0: k + (m-k)/4 (block: k + (m-k)/2) */
  int32_t max_restarts;   /* 0: 100000 */
  uint64_t start_seed;    /* Philox key for the Lanczos start / breakdown vectors */
  double tol_eff_cap;     /* residual target = min(tol, tol_eff_cap) * sigma; <= 0: 1e-10 (reading R7) */
  void *cuda_stream;      /* cudaStream_t to run on (e.g. torch.cuda.current_stream()); NULL: library-created */
  int32_t check_symmetry; /* 1 (default): verify W == W^T at build (one O(nnz log deg) pass) */
  int32_t spmv_vector;    /* 0: auto; else lanes per row in the SpMV (2,4,8,16,32) */
  int32_t block_size;     /* Lanczos block size b: 1 = single-vector thick-restart Lanczos; 2 or 4 = block
                             thick-restart Lanczos (SpMM on b interleaved vectors, block CGS2, CholQR2;
                             requires h <= 16); 0 = auto (DESIGN.md §Block Lanczos) */
  int32_t reorth;         /* single-vector full reorthogonalisation: 1 = CGS2 (three basis sweeps per step),
                             2 = lagged single sweep (one basis sweep per step, DESIGN.md §6.2;
                             needs h <= 16, k < m <= min(192, n-h)), 3 = paired steps (one basis sweep per
                             TWO steps; single GPU, group constraints, k + 4 <= m <= 186);
                             0 = auto (3 where allowed, else 2, else 1) */
  struct sfairsc_comm *comm; /* NULL: single GPU.  Else row-partitioned across the communicator's ranks
                             (SURVEY §8(e)): each rank passes its contiguous row block of W (row_offset,
                             n_rows, global n_cols; blocks tile [0, n) in rank order) and the groups of its
                             rows; h must be given; evecs/labels/apply vectors hold the rank's rows */
  int32_t virtual_parts;  /* > 1 (test/emulation): split the full W into this many nnz-balanced row blocks
                             inside one process and GPU and run the row-partitioned solver over them */
  int32_t filter_degree;  /* SURVEY §8(f) N2 (every kernel stays an SpMV): 0 or 1 = no
                             filter; d >= 2 (<= 64) = thick-restart Lanczos on the Chebyshev filter
                             -p(L^sigma), p(x) = (-1)^d T_d((x - c)/e), c = (a + sigma)/2, e = (sigma - a)/2,
                             which maps [a, sigma] into [-1, 1] and the wanted eigenvalues below a, in the
                             same order, below -1.  Each Lanczos step applies L^sigma d times
                             (three-term recurrence fused into the apply's last kernel).  Eigenvalues are the
                             Rayleigh quotients x^T L^sigma x of the filter's Ritz vectors; convergence is
                             decided on their explicit L^sigma residuals.  Needs a group-fairness build,
                             block_size 0/1, reorth 0/1 (the CGS2 solver runs), single GPU; else
                             SFAIRSC_E_INVALID_ARG */
  double filter_cut;      /* the filter's a: > 0 fixed (must be < sigma); <= 0 automatic: one unfiltered
                             cycle of m steps, a = its keep-th Ritz value, and the filtered solve restarts
                             from the sum of the cycle's k lowest Ritz vectors */
} sfairsc_opts;

typedef struct {
  int64_t applies;       /* operator applications L^sigma w performed by eigs (incl. final residual check) */
  int64_t steps;         /* Lanczos expansion steps */
  int64_t restarts;      /* thick restarts */
  int64_t breakdowns;    /* invariant-subspace breakdowns (fresh random vector injected) */
  double sigma;          /* the shift used */
  double max_resid_rel;  /* max_i ||L^sigma x_i - lambda_i x_i||_2 / sigma, recomputed with k fresh applies */
  double gap_est;        /* theta_{k+1} - theta_k from the final Rayleigh-Ritz (NaN if unavailable) */
  double t_build_s;      /* wall time of the build call */
  double t_eigs_s;       /* wall time of the last eigs call */
  int32_t converged;     /* 1 if the residual target was met */
  int32_t basis_size;    /* m used */
  int32_t kept;          /* Ritz vectors kept per restart */
  int32_t reserved;
  double filter_cut;     /* the Chebyshev filter's a used (opts.filter_degree >= 2), else 0 */
} sfairsc_stats;

typedef struct {
  int64_t n, nnz;
  int32_t h, k_build, normalized, spmv_vector;
  double sigma;
  int32_t device, num_sms;
  int32_t unit_weights;   /* 1: every stored w_ij = 1 (no diagonal entries): the single-vector SpMV
                             streams only column indices (normalized: gathers s o x, row sums scaled by s_i) */
  int32_t constraint_rank; /* rank of C: h - 1 for group fairness; the numerical rank of C for a dense F */
} sfairsc_info;

void sfairsc_default_opts(sfairsc_opts *opts);

/* Alg. 3 steps 1-2 + shift: validate W and
 * groups (A0), copy them into library-owned device memory, compute degrees
 * d = W 1, the scaling s = d^{-1/2} (normalized: stored values
 * become s_i w_ij s_j), sigma = ||L||_1, and the factored basis Q of
 * range(C) (DESIGN.md §Factored projector; no dense Q is formed).
 * groups[n] in the same memspace as W, values in [0, h); h = 0 infers
 * h = max(groups)+1; 1 <= h <= 255.  k = number of eigenpairs the context
 * must be able to return (sizes the Krylov basis).  *out receives a new
 * context on success. */
sfairsc_status sfairsc_build_operator(const sfairsc_csr *W, const int32_t *groups, int32_t h,
                                      int32_t k, int32_t normalized, sfairsc_ctx **out);
sfairsc_status sfairsc_build_operator_ex(const sfairsc_csr *W, const int32_t *groups, int32_t h,
                                         int32_t k, int32_t normalized, const sfairsc_opts *opts,
                                         sfairsc_ctx **out);

/* §8(f) N4 — general linear constraints C^T H = 0 with a dense constraint matrix F (n x r,
 * column-major, 0 <= r <= 64; e.g. the random-F Laplacian of Experiment 4, or
 * overlapping groups; P:465-490 take F as input): C = D^{-1/2} F (normalized) or F.
 * P = I - C C^+ (C^+ the pseudo-inverse, i.e. the minimum-norm least-squares solve
 * of P:815-820, so a rank-deficient C is allowed): Q = an orthonormal basis of range(C) from
 * the eigendecomposition of C^T C with numerical rank rq = #{eigenvalues > 1e-14 x the largest}
 * (reading R21), then one Cholesky-QR step; rq must be <= 16 (SFAIRSC_E_INVALID_ARG otherwise),
 * k <= n - rq (SFAIRSC_E_K_TOO_LARGE).  Every projector step applies P = I - Q Q^T with the
 * dense rows of Q (Q^T x fused into the SpMV epilogue and the basis sweep, x - Q (Q^T x) into
 * the normalisation).  sfairsc_info.constraint_rank reports rq.  F in W's memspace.  Single GPU,
 * single-sweep solver.  sfairsc_eigs / sfairsc_apply / embed_kmeans as usual. */
sfairsc_status sfairsc_build_operator_dense(const sfairsc_csr *W, const double *F, int32_t r, int32_t k,
                                            int32_t normalized, const sfairsc_opts *opts, sfairsc_ctx **out);

/* Alg. 3 step 3: the k smallest eigenpairs of L^sigma by
 * thick-restart Lanczos with full CGS2 reorthogonalisation (replaces
 * MATLAB eigs / ARPACK).  Stops when every wanted Ritz pair has
 * ||L^sigma x - theta x|| <= min(tol, tol_eff_cap) * sigma.
 * evals_out[k] (host, ascending); evecs_out = X (n x k, column-major,
 * orthonormal, C^T X = 0) in evecs_memspace, or NULL.  stats may be NULL. */
sfairsc_status sfairsc_eigs(sfairsc_ctx *ctx, int32_t k, double tol, double *evals_out,
                            double *evecs_out, int32_t evecs_memspace, sfairsc_stats *stats);

/* Alg. 3 step 4: k-means on the rows of H = D^{-1/2} X (normalized)
 * or H = X (unnormalized) from the last eigs call, with the k-means variant
 * of reading R16 (k-means++ seeding, Lloyd, best of 10 restarts by WCSS,
 * Philox4x32-10 draws keyed by `seed`).  labels_out[n] in memspace;
 * objective_out (host, may be NULL) = best WCSS. */
sfairsc_status sfairsc_embed_kmeans(sfairsc_ctx *ctx, uint64_t seed, int32_t *labels_out,
                                    int32_t memspace, double *objective_out);

/* y = L^sigma x for nvec column vectors: four fused kernels —
 * group sums B^T x, p = P x, SpMV t = L p with B^T t in its epilogue,
 * y = t - s o (gamma_t - sigma gamma_x)_g.  x, y: n x nvec, same memspace. */
sfairsc_status sfairsc_apply(sfairsc_ctx *ctx, const double *x, double *y, int32_t nvec,
                             int32_t memspace);
/* sfairsc_apply with flags: SFAIRSC_APPLY_SINGLE = every vector through its own
 * single-vector SpMV (no interleaved pairs) — the §8(d) metric-1 apply, one L^sigma
 * application at a time.  Same arguments, ownership and errors as sfairsc_apply. */
#define SFAIRSC_APPLY_SINGLE 1
sfairsc_status sfairsc_apply_ex(sfairsc_ctx *ctx, const double *x, double *y, int32_t nvec,
                                int32_t memspace, int32_t flags);

/* y = P x (P:807-818 in factored form) for nvec column vectors. */
sfairsc_status sfairsc_project(sfairsc_ctx *ctx, const double *x, double *y, int32_t nvec,
                               int32_t memspace);

/* y = L x (normalized: L_n; unnormalized: D - W) — the bare SpMV, for tests. */
sfairsc_status sfairsc_laplacian(sfairsc_ctx *ctx, const double *x, double *y, int32_t memspace);

sfairsc_status sfairsc_get_info(const sfairsc_ctx *ctx, sfairsc_info *info);

/* Per-kernel device timing with CUDA events on the context stream (for the
 * bench roofline); one event pair brackets each profiled launch group.  kind: 0 spmv, 1 reorth sweep (dots), 2 reorth sweep
 * (update+dots), 3 reorth sweep (update+norm), 4 normalize, 5 ritz gemm,
 * 6 project/group-sum, 7 apply-finish, 8 kmeans, 9 other.  Enabling adds
 * one event pair per launch. */
sfairsc_status sfairsc_profile_enable(sfairsc_ctx *ctx, int32_t enable);
sfairsc_status sfairsc_profile_read(sfairsc_ctx *ctx, int32_t kind, double *total_ms,
                                    int64_t *launches, double *alg_bytes);
/* alg_bytes = sum over the kind's launches of its algorithmic bytes (each
 * operand read or written once; SpMV: CSR 12 nnz + 4(n+1) + p, t, d or s,
 * group ids; sweeps: J basis columns + the vectors). */

/* Total kernel launches issued by this library in this process (all
 * contexts) — the bench's gpu_launches evidence. */
int64_t sfairsc_launch_count(void);
sfairsc_status sfairsc_profile_reset(sfairsc_ctx *ctx);

/* Host-only utility: the dense symmetric eigensolver of the Rayleigh-Ritz step
 * (Householder tridiagonalisation + implicit QL).  A: m x m row-major
 * symmetric; evals[m] ascending; evecs (m x m row-major, column c = vector c,
 * may be NULL).  Returns 0 on success.  Exported so tests can pin it on CPU. */
int sfairsc_host_symeig(int32_t m, const double *A, double *evals, double *evecs);
/* Same, with only the eigenvectors of the nvec smallest eigenvalues (what a thick restart keeps): all m
 * evals ascending; evecs m x m row-major with columns c < nvec written (the others untouched).
 * 0 <= nvec <= m.  Returns 0 on success, 1 on bad arguments. */
int sfairsc_host_symeig_sel(int32_t m, const double *A, double *evals, double *evecs, int32_t nvec);

/* Multi-GPU bootstrap: rank 0 calls sfairsc_comm_unique_id and
 * broadcasts the 128 bytes (e.g. with torch.distributed); every rank then calls
 * sfairsc_comm_init with its rank, the rank count and its CUDA device.  NCCL
 * (libnccl.so.2) is loaded at run time; SFAIRSC_E_NCCL if it is missing or fails. */
sfairsc_status sfairsc_comm_unique_id(uint8_t id_out[128]);
sfairsc_status sfairsc_comm_init(const uint8_t id[128], int32_t rank, int32_t nranks, int32_t device,
                                 sfairsc_comm **out);
void sfairsc_comm_destroy(sfairsc_comm *comm);

/* Host-only: sizeof of the ABI structs (0 sfairsc_csr, 1 sfairsc_opts, 2 sfairsc_stats, 3 sfairsc_info;
 * -1 otherwise), so that a binding can verify its struct mirrors at load time. */
int64_t sfairsc_struct_size(int32_t which);

void sfairsc_destroy(sfairsc_ctx *ctx);
const char *sfairsc_last_error(void);
const char *sfairsc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SFAIRSC_H */
