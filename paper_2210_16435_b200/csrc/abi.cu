// libsfairsc — C ABI (include/sfairsc.h): context, operator build (A0-A3),
// operator apply (A4-A6), thick-restart Lanczos driver (A7-A11).
#include "ctx.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

namespace sfz {
void symeig(int m, std::vector<double>& A, std::vector<double>& evals);
void symeig(int m, std::vector<double>& A, std::vector<double>& evals, int nvec);
sfairsc_status eigs_block(sfairsc_ctx* c, int k, double tol, double* evals_out, double* evecs_out,
                          int evecs_memspace, sfairsc_stats* stats);
sfairsc_status eigs_lagged(sfairsc_ctx* c, int k, double tol, double* evals_out, double* evecs_out,
                           int evecs_memspace, sfairsc_stats* stats);
sfairsc_status dist_build(sfairsc_ctx* c, const sfairsc_csr* W, const int32_t* groups, int hh,
                          const std::vector<int64_t>& cnt_local, const sfairsc_opts& opts);
sfairsc_status dist_agree(sfairsc_comm* comm, int local_status, cudaStream_t st);
sfairsc_status dist_eigs(sfairsc_ctx* c, int k, double tol, double* evals_out, double* evecs_out, int evecs_memspace,
                         sfairsc_stats* stats);
sfairsc_status dist_apply(sfairsc_ctx* c, const double* x, double* y);
sfairsc_status dist_kmeans(sfairsc_ctx* c, uint64_t seed, int32_t* labels_out, int32_t memspace, double* objective);
long long dist_local_rows(const sfairsc_ctx* c);
void dist_free(DistCtx* D);
sfairsc_status kmeans_run(sfairsc_ctx* ctx, uint64_t seed, int32_t* labels_out, int32_t memspace, double* objective);
}  // namespace sfz

using namespace sfz;

static thread_local std::string g_err;

sfairsc_status sfz::fail(sfairsc_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}


// accessors used by kmeans.cu
namespace sfz {
cudaStream_t ctx_stream(sfairsc_ctx* c) { return c->st; }
int ctx_n(sfairsc_ctx* c) { return c->n; }
int ctx_k(sfairsc_ctx* c) { return c->k_eigs; }
bool ctx_have_eigs(sfairsc_ctx* c) { return c->have_eigs; }
const double* ctx_X(sfairsc_ctx* c, long long* ld) {
  *ld = c->ldv;
  return c->X;
}
const double* ctx_s(sfairsc_ctx* c) { return c->normalized ? c->s : nullptr; }
int ctx_num_sms(sfairsc_ctx* c) { return c->num_sms; }
void** ctx_km(sfairsc_ctx* c, void (**freer)(void*)) {
  *freer = c->km_free;
  return &c->km;
}
void ctx_set_km_free(sfairsc_ctx* c, void (*f)(void*)) { c->km_free = f; }
void ctx_prof_begin(sfairsc_ctx* c, cudaEvent_t* a);
void ctx_prof_end(sfairsc_ctx* c, int kind, cudaEvent_t a);
sfairsc_status ctx_fail(sfairsc_status st, const char* msg) { return fail(st, "%s", msg); }
}  // namespace sfz

namespace sfz {
void ctx_prof_begin(sfairsc_ctx* c, cudaEvent_t* a) {
  *a = nullptr;
  if (c->prof.on) {
    *a = c->prof.get();
    cudaEventRecord(*a, c->st);
  }
}
void ctx_prof_end(sfairsc_ctx* c, int kind, cudaEvent_t a) {
  if (c->prof.on && a) {
    cudaEvent_t b = c->prof.get();
    cudaEventRecord(b, c->st);
    c->prof.pending.push_back({kind, a, b, 0.0});
  }
}
}  // namespace sfz

template <typename T>
static cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T));
}

static void free_ctx(sfairsc_ctx* c) {
  if (!c) return;
  if (c->dist) dist_free(c->dist);
  if (c->km && c->km_free) c->km_free(c->km);
  void* ptrs[] = {c->tiles, c->cta_tiles, c->prp, c->pci, c->pvv, c->rp, c->ci, c->row_split, c->vv, c->dg, c->s, c->grp, c->isb, c->uh, c->partials, c->counters,
                  c->bs_w, c->bs_t, c->bs_v, c->nb, c->scal, c->c1, c->c2, c->vp, c->vt, c->vr, c->vy, c->V,
                  c->Vb, c->Ydev, c->X, c->flags, c->talpha, c->tbeta,
                  c->bP, c->bT, c->bR, c->Tdev, c->g2, c->bflags, c->Hdev, c->sdev, c->lz, c->partials2, c->dd, c->rpb,
                  c->pairP, c->pairT, c->pairY, c->Qr, c->vq, c->vq_lz, c->vrB, c->lzp, c->fbuf, c->fth};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->hp) cudaFreeHost(c->hp);
  if (c->own_stream && c->st) cudaStreamDestroy(c->st);
  delete c;
}

double sfz::now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// --------------------------------------------------------------------------
// options / info
// --------------------------------------------------------------------------
extern "C" void sfairsc_default_opts(sfairsc_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->sigma_override = 0.0;
  o->max_basis = 0;
  o->keep = 0;
  o->max_restarts = 0;
  o->start_seed = 0x5F41C5EEDull;
  o->tol_eff_cap = 1e-10;
  o->cuda_stream = nullptr;
  o->check_symmetry = 1;
  o->spmv_vector = 0;
  o->block_size = 0;
  o->reorth = 0;
  o->comm = nullptr;
  o->virtual_parts = 0;
  o->filter_degree = 0;
  o->filter_cut = 0.0;
}

extern "C" const char* sfairsc_last_error(void) { return g_err.c_str(); }
extern "C" const char* sfairsc_version(void) { return "sfairsc-b200 0.1 (sm_100a, fp64)"; }

extern "C" sfairsc_status sfairsc_get_info(const sfairsc_ctx* c, sfairsc_info* info) {
  if (!c || !info) return fail(SFAIRSC_E_INVALID_ARG, "null argument");
  info->n = c->n;
  info->nnz = c->nnz;
  info->h = c->h;
  info->k_build = c->k_build;
  info->normalized = c->normalized;
  info->spmv_vector = c->vs;
  info->sigma = c->sigma;
  info->device = c->device;
  info->num_sms = c->num_sms;
  info->unit_weights = c->unit ? 1 : 0;
  info->constraint_rank = c->Qr || c->rank_in > 0 ? c->qr : std::max(0, c->h - 1);
  return SFAIRSC_OK;
}

// --------------------------------------------------------------------------
// group sums for h > 16 (the fused epilogues cover groups [0,16))
// --------------------------------------------------------------------------
static void extra_gsums(sfairsc_ctx* c, const double* x, double* bsum) {
  for (int gb = kHB; gb < c->h; gb += kHB)
    launch_gsum(c->g(), x, gb, c->partials, c->counters + 3, bsum, c->st);
}

static void gsum_all(sfairsc_ctx* c, const double* x, double* bsum) {
  for (int gb = 0; gb < c->h; gb += kHB) launch_gsum(c->g(), x, gb, c->partials, c->counters + 3, bsum, c->st);
}

// y = L^sigma x on device vectors (4 kernels; A4-A6)
sfairsc_status sfz::apply_dev(sfairsc_ctx* c, const double* x, double* y) {
  {
    ProfScope ps(c, K_PROJ, c->gpasses() * (c->vb() + c->sgb()) + 2 * c->vb() + c->sgb());
    gsum_all(c, x, c->bs_w);
    launch_project(c->g(), c->pd(), x, c->bs_w, 1.0, c->vp, c->st);
  }
  {
    ProfScope ps(c, K_SPMV, c->csr_bytes() + 3 * c->vb() + 1.0 * c->n);
    ctx_spmv(c, c->vp, c->vt);
  }
  if (c->h > kHB) extra_gsums(c, c->vt, c->bs_t);
  {
    ProfScope ps(c, K_FINISH, 2 * c->vb() + c->sgb());
    launch_finish(c->g(), c->pd(), c->vt, c->bs_t, c->bs_w, c->sigma, y, c->st);
  }
  CHECK_LAUNCH();
  return SFAIRSC_OK;
}


// y0, y1 = L^sigma x0, x1 through one SpMM of the interleaved pair (h <= 16, plain CSR); the pair
// buffers are allocated on first use (2 interleaved n x 2 blocks)
sfairsc_status sfz::apply_pair_dev(sfairsc_ctx* c, const double* x0, const double* x1, double* y0, double* y1) {
  if (!c->pairP) {
    CU(cudaMalloc(&c->pairP, sizeof(double) * 2 * c->ldv));
    CU(cudaMalloc(&c->pairT, sizeof(double) * 2 * c->ldv));
  }
  {
    ProfScope ps(c, K_PROJ, 2 * (2 * c->vb() + c->sgb()) + 2 * c->vb());
    launch_pair_gsum(c->g(), x0, x1, c->partials, c->counters + 3, c->bs_w, c->st);
    launch_pair_project(c->g(), c->pd(), x0, x1, c->bs_w, c->pairP, c->st);
  }
  {
    ProfScope ps(c, K_SPMV, c->csr_bytes() + 4 * c->vb() + c->vb() + 1.0 * c->n);
    launch_spmm(c->g(), 2, c->vs, c->row_split, c->spmv_grid, c->pairP, c->pairT, c->partials, c->counters + 1,
                c->bs_t, c->st);
  }
  {
    ProfScope ps(c, K_FINISH, 4 * c->vb() + c->sgb());
    launch_pair_finish(c->g(), c->pd(), c->pairT, c->bs_t, c->bs_w, c->sigma, y0, y1, c->st);
  }
  CHECK_LAUNCH();
  return SFAIRSC_OK;
}
static bool pair_ok(const sfairsc_ctx* c) { return c->h <= kHB && c->nblk <= 1 && !c->dist && !c->Qr; }

// set by the dense-constraint build around its inner build: the DQ SpMV streams the values
static thread_local bool g_build_keep_values = false;

void sfz::ctx_spmv(sfairsc_ctx* c, const double* p, double* t, const double* q_pre) {
  // unit weights, normalized: gather q = s o p (the row sum is scaled by s_i in the kernel)
  const double* pg = p;
  if (c->unit_spmv() && c->normalized && q_pre) {
    pg = q_pre;
  } else if (c->unit_spmv() && c->normalized) {
    launch_scale_vec(c->s, p, c->vq, c->n, c->st);
    pg = c->vq;
  }
  if (c->nblk <= 1 && c->tiles && !c->Qr) {
    GraphDev g = c->gs();
    g.rp = c->prp;
    g.ci = c->pci;
    g.vv = c->pvv;
    g.nnz = c->nnz_pad;
    launch_spmv_tma(g, c->vs, c->spmv_shape, c->tiles, c->cta_tiles, c->tma_grid, pg, p, t, c->partials, c->counters + 1, c->bs_t,
                    c->st);
    return;
  }
  if (c->nblk <= 1) {
    launch_spmm(c->gs(), 1, c->vs, c->row_split, c->spmv_grid, pg, t, c->partials, c->counters + 1, c->bs_t, c->st, p);
    return;
  }
  for (int b = 0; b < c->nblk; ++b) {  // p restricted to block b (8n/nblk bytes) stays in L2 while W_b streams
    GraphDev g = c->gs();
    g.rp = c->rpb + (size_t)b * (c->n + 1);
    const int cmode = (b == 0) ? 1 : (b + 1 < c->nblk ? 2 : 3);
    launch_spmv_colblock(g, c->vs_blk, c->row_split, c->spmv_grid, pg, t, c->partials, c->counters + 1, c->bs_t, cmode,
                         c->st, p);
  }
}

// max_i ||L^sigma x_i - theta_i x_i|| / sigma over the k columns of X (A11), k fresh applies
sfairsc_status sfz::true_residuals(sfairsc_ctx* c, const double* theta, int k, double* max_out) {
  NvtxRange nv("sfairsc.true_residuals");
  std::vector<double> res(k);
  if (pair_ok(c) && !c->pairY) CU(cudaMalloc(&c->pairY, sizeof(double) * c->ldv));
  for (int i = 0; i < k; ++i) {
    const double* xi = c->X + (long long)i * c->ldv;
    if (pair_ok(c) && i + 1 < k && i % 64 != 63) {  // two residuals per SpMM (the pair stays in one 64-batch)
      const double* xj = xi + c->ldv;
      TRY(apply_pair_dev(c, xi, xj, c->vy, c->pairY));
      launch_resid(c->vy, xi, theta[i], c->n, c->partials, c->counters + 4, c->scal + 8 + i % 64, c->st);
      launch_resid(c->pairY, xj, theta[i + 1], c->n, c->partials, c->counters + 4, c->scal + 8 + (i + 1) % 64, c->st);
      CHECK_LAUNCH();
      ++i;
    } else {
      TRY(apply_dev(c, xi, c->vy));
      launch_resid(c->vy, xi, theta[i], c->n, c->partials, c->counters + 4, c->scal + 8 + i % 64, c->st);
      CHECK_LAUNCH();
    }
    if (i % 64 == 63 || i == k - 1) {
      const int base = i - i % 64;
      CU(cudaMemcpyAsync(c->hp, c->scal + 8, sizeof(double) * (i - base + 1), cudaMemcpyDeviceToHost, c->st));
      CU(cudaStreamSynchronize(c->st));
      for (int q = base; q <= i; ++q) res[q] = std::sqrt(c->hp[q - base]) / c->sigma;
    }
  }
  double mx = 0.0;
  for (int i = 0; i < k; ++i) mx = std::max(mx, res[i]);
  *max_out = mx;
  return SFAIRSC_OK;
}

// --------------------------------------------------------------------------
// build (A0-A3)
// --------------------------------------------------------------------------
extern "C" sfairsc_status sfairsc_build_operator(const sfairsc_csr* W, const int32_t* groups, int32_t h, int32_t k,
                                                 int32_t normalized, sfairsc_ctx** out) {
  return sfairsc_build_operator_ex(W, groups, h, k, normalized, nullptr, out);
}

static sfairsc_status build_impl(const sfairsc_csr* W, const int32_t* groups, int32_t h, int32_t k,
                                 int32_t normalized, const sfairsc_opts* opts_in, sfairsc_ctx** out,
                                 bool* reached_dist);

extern "C" sfairsc_status sfairsc_build_operator_ex(const sfairsc_csr* W, const int32_t* groups, int32_t h,
                                                    int32_t k, int32_t normalized, const sfairsc_opts* opts_in,
                                                    sfairsc_ctx** out) {
  NvtxRange nv("sfairsc.build");
  bool reached_dist = false;
  const sfairsc_status st = build_impl(W, groups, h, k, normalized, opts_in, out, &reached_dist);
  if (st != SFAIRSC_OK && !reached_dist && opts_in && opts_in->comm) {
    // this rank failed before the row-partitioned build's first collective: take part in the agreement the
    // other ranks wait in (dist_build), so that they fail too instead of blocking; keep this rank's message
    const std::string msg = g_err;
    dist_agree(opts_in->comm, (int)st, (cudaStream_t)opts_in->cuda_stream);
    g_err = msg;
  }
  return st;
}

static sfairsc_status build_impl(const sfairsc_csr* W, const int32_t* groups, int32_t h, int32_t k,
                                 int32_t normalized, const sfairsc_opts* opts_in, sfairsc_ctx** out,
                                 bool* reached_dist) {
  const double t0 = now_s();
  if (!W || !groups || !out) return fail(SFAIRSC_E_INVALID_ARG, "null argument");
  *out = nullptr;
  sfairsc_opts opts;
  sfairsc_default_opts(&opts);
  if (opts_in) opts = *opts_in;
  if (W->memspace != SFAIRSC_MEM_HOST && W->memspace != SFAIRSC_MEM_DEVICE)
    return fail(SFAIRSC_E_INVALID_ARG, "bad memspace");
  // row-partitioned: NCCL ranks pass their own contiguous row block; virtual parts: the full matrix
  const bool is_nccl = opts.comm != nullptr;
  const bool is_dist = is_nccl || opts.virtual_parts > 1;
  if (opts.virtual_parts < 0 || opts.virtual_parts > 64) return fail(SFAIRSC_E_INVALID_ARG, "virtual_parts in [0, 64]");
  if (!is_nccl && W->n_rows != W->n_cols) return fail(SFAIRSC_E_DIM_MISMATCH, "n_rows != n_cols (row blocks need opts.comm)");
  if (!is_nccl && W->row_offset != 0) return fail(SFAIRSC_E_INVALID_ARG, "row_offset must be 0 without opts.comm");
  if (is_nccl && (W->row_offset < 0 || W->row_offset + W->n_rows > W->n_cols || W->n_rows < 1))
    return fail(SFAIRSC_E_DIM_MISMATCH, "row block [row_offset, row_offset + n_rows) outside [0, n_cols)");
  if (is_nccl && h < 1) return fail(SFAIRSC_E_INVALID_ARG, "h must be given (> 0) for a row-partitioned build");
  if (W->n_cols < 1 || W->n_cols >= (1LL << 31) - 1024) return fail(SFAIRSC_E_INVALID_ARG, "n out of range");
  if (W->nnz < 0 || W->nnz >= (1LL << 31) - 1) return fail(SFAIRSC_E_INVALID_ARG, "nnz out of int32 range");
  if (W->nnz > 0 && (!W->col_idx || !W->values)) return fail(SFAIRSC_E_INVALID_ARG, "null CSR arrays");
  if (!W->row_ptr) return fail(SFAIRSC_E_INVALID_ARG, "null row_ptr");
  if (k < 1) return fail(SFAIRSC_E_INVALID_ARG, "k must be >= 1");
  if (h < 0 || h > 255) return fail(SFAIRSC_E_INVALID_ARG, "h must be in [0, 255]");
  const int n = (int)W->n_cols, nnz = (int)W->nnz;  // n: global vertex count
  const int n_rows = (int)W->n_rows;                  // rows passed (= n unless an NCCL row block)
  const bool dev_in = W->memspace == SFAIRSC_MEM_DEVICE;

  // groups on host: counts, inferred h, range check
  std::vector<int32_t> hg(n_rows);
  if (dev_in) {
    cudaError_t e = cudaMemcpy(hg.data(), groups, sizeof(int32_t) * n_rows, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return fail(SFAIRSC_E_CUDA, "groups copy: %s", cudaGetErrorString(e));
  } else {
    std::memcpy(hg.data(), groups, sizeof(int32_t) * n_rows);
  }
  int hh = h;
  if (hh == 0) {
    int mx = -1;
    for (int i = 0; i < n_rows; ++i) mx = std::max(mx, hg[i]);
    hh = mx + 1;
    if (hh < 1 || hh > 255) return fail(SFAIRSC_E_INVALID_ARG, "inferred h out of range");
  }
  std::vector<int64_t> cnt(hh, 0);
  for (int i = 0; i < n_rows; ++i) {
    if (hg[i] < 0 || hg[i] >= hh) return fail(SFAIRSC_E_INVALID_ARG, "group id %d out of [0,%d) at vertex %d", hg[i], hh, i);
    cnt[hg[i]]++;
  }
  if (!is_nccl)  // a rank's row block may miss a group: checked globally in dist_build
    for (int s = 0; s < hh; ++s)
      if (cnt[s] == 0) return fail(SFAIRSC_E_EMPTY_GROUP, "group %d is empty (P:152)", s);
  if ((int64_t)k > (int64_t)n - hh + 1) return fail(SFAIRSC_E_K_TOO_LARGE, "k=%d > n-h+1=%lld", k, (long long)n - hh + 1);

  sfairsc_ctx* c = new sfairsc_ctx();
  c->n = n;
  c->nnz = nnz;
  c->h = hh;
  c->k_build = k;
  c->normalized = normalized != 0;
  c->groups_host = hg;
  c->group_count = cnt;
  c->tol_cap = opts.tol_eff_cap > 0 ? opts.tol_eff_cap : 1e-10;
  c->seed = opts.start_seed;
  c->max_restarts = opts.max_restarts > 0 ? opts.max_restarts : 100000;
  c->check_symmetry = opts.check_symmetry;
  c->debug = getenv("SFAIRSC_DEBUG") ? atoi(getenv("SFAIRSC_DEBUG")) : 0;
  auto bail = [&](sfairsc_status st) {
    free_ctx(c);
    return st;
  };
#define CUB(expr)                                                                                          \
  do {                                                                                                     \
    cudaError_t e_ = (expr);                                                                               \
    if (e_ != cudaSuccess)                                                                                 \
      return bail(fail(e_ == cudaErrorMemoryAllocation ? SFAIRSC_E_OOM : SFAIRSC_E_CUDA, "%s: %s (%s:%d)", \
                       #expr, cudaGetErrorString(e_), __FILE__, __LINE__));                                 \
  } while (0)

  CUB(cudaGetDevice(&c->device));
  CUB(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
  if (opts.cuda_stream) {
    c->st = (cudaStream_t)opts.cuda_stream;
  } else {
    CUB(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  c->ldv = ((long long)n + 255) / 256 * 256;
  // Krylov basis size (SPEC S:342 default), capped so that v_{m+1} exists
  // default basis: m = max(2k + 10, 3.4k, 20) (SPEC S:342 suggests 2k + 10; 3.4k measured fastest at config 4,
  // profiles/r1_exp/cfg4_restart_scan.json), keep k + (m - k)/4 Ritz vectors per thick restart
  int m = opts.max_basis > 0 ? opts.max_basis : std::min(192, std::max(std::max(2 * k + 10, 17 * k / 5), 20));
  m = std::min(m, kMaxJ - 1);
  m = std::min(m, std::max(n - 1, 1));
  m = std::max(m, std::min(k + 1, n));
  if (m > n) m = n;
  c->m = m;
  c->keep = opts.keep > 0 ? opts.keep : k + (m - k) / 4;
  c->keep = std::max(std::min(c->keep, m - 1), std::min(k, m - 1));
  const int m_pref = m;  // the basis the HBM budget below may shrink (and a dropped value array may regrow)
  // block Lanczos sizing: m + b <= kBMaxJ, m + b <= dim null(C^T) = n - h + 1, keep >= k, (m - keep) % b == 0
  c->bsz = opts.block_size > 0 ? opts.block_size : 1;
  if (c->bsz != 1 && c->bsz != 2 && c->bsz != 4)
    return bail(fail(SFAIRSC_E_INVALID_ARG, "block_size must be 0, 1, 2 or 4"));
  if (hh > kHB) c->bsz = 1;  // the fused block epilogues carry at most kHB group sums
  if (c->bsz > 1) {
    const int b = c->bsz;
    int mb = opts.max_basis > 0 ? opts.max_basis : std::max(2 * k + 10, 20);
    mb = std::min(mb, kBMaxJ - b);
    mb = std::min(mb, n - hh + 1 - b);
    if (mb < k + b) {
      c->bsz = 1;  // too small for a block basis: single-vector Lanczos
    } else {
      int kp = opts.keep > 0 ? opts.keep : k + (mb - k) / 2;
      kp = std::max(k, std::min(kp, mb - b));
      mb = kp + b * ((mb - kp) / b);
      c->m = m = mb;
      c->keep = kp;
    }
  }
  // HBM budget (single GPU, default basis only): the two basis buffers (m+1 columns each) plus the CSR copy,
  // X and ~12 work vectors must fit in free device memory (config 5 on one GPU: n = 5e7, 400 MB per vector)
  if (opts.max_basis <= 0 && !(opts.comm || opts.virtual_parts > 1)) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess && fr > 0) {
      const double vbytes = 8.0 * (double)c->ldv * (c->bsz > 1 ? 1 : 1);
      const double fixed = 12.0 * nnz + 4.0 * n + ((double)k + 12.0 + 3.0 * c->bsz) * vbytes + 256.0 * (1 << 20);
      const double avail = 0.97 * (double)fr - fixed;
      const int mfit = (int)std::floor(avail / (2.0 * vbytes)) - std::max(1, c->bsz);
      if (mfit < m) {
        const int mnew = std::max(mfit, k + std::max(2, c->bsz));
        if (mnew < k + 2) return bail(fail(SFAIRSC_E_OOM, "Krylov basis for k=%d does not fit in device memory", k));
        const int b = std::max(1, c->bsz);
        int kp = opts.keep > 0 ? opts.keep : k + (mnew - k) / 4;
        kp = std::max(k, std::min(kp, mnew - b));
        c->m = m = (b > 1) ? kp + b * ((mnew - kp) / b) : mnew;
        c->keep = kp;
      }
    }
  }
  // single-vector reorthogonalisation: 0 auto (= paired lagged sweeps where allowed, else lagged), 1 CGS2 (three
  // sweeps per step), 2 lagged (one sweep per step), 3 paired (one sweep per two steps)
  if (opts.reorth < 0 || opts.reorth > 3) return bail(fail(SFAIRSC_E_INVALID_ARG, "reorth must be 0, 1, 2 or 3"));
  // Chebyshev filter (§8(f) N2): the CGS2 solver on -p(L^sigma); group-fairness builds, single GPU
  if (opts.filter_degree < 0 || opts.filter_degree > 64)
    return bail(fail(SFAIRSC_E_INVALID_ARG, "filter_degree must be in [0, 64]"));
  if (opts.filter_degree >= 2) {
    if (opts.reorth > 1 || opts.block_size > 1 || is_dist || g_build_keep_values)
      return bail(fail(SFAIRSC_E_INVALID_ARG,
                       "filter_degree >= 2 needs a group-fairness build, block_size 0/1, reorth 0/1 and one GPU"));
    c->filter_deg = opts.filter_degree;
    c->filter_cut = opts.filter_cut;
    c->bsz = 1;
    opts.reorth = 1;
  }
  c->lagged = c->bsz == 1 && opts.reorth != 1 && hh <= kHB && m <= 192 && m <= n - hh && m > k;
  if ((opts.reorth == 2 || opts.reorth == 3) && !c->lagged)
    return bail(fail(SFAIRSC_E_INVALID_ARG, "reorth=2/3 need block_size 1, h <= 16 and k < m <= min(192, n-h)"));
  // paired steps: single GPU, group projector (the dense projector and row-partitioned builds keep one step
  // per sweep); they need room for a pair after the first step of a cycle
  c->paired = c->lagged && opts.reorth != 2 && !g_build_keep_values && m >= k + 4 &&
              (!(opts.comm || opts.virtual_parts > 1) || m <= kPairMaxM);  // (dist: the basis size is final here)
  if (opts.reorth == 3 && !c->paired)
    return bail(fail(SFAIRSC_E_INVALID_ARG, "reorth=3 needs a group-fairness build and k + 4 <= m (<= 186)"));
  if (is_dist) {  // row-partitioned single-sweep Lanczos (dist.cu)
    if (!c->lagged) return bail(fail(SFAIRSC_E_INVALID_ARG, "row-partitioned builds need h <= 16, block_size 1, reorth 0/2/3"));
    {
      const double mean_deg = (double)W->nnz / std::max(1, n_rows);
      int vs = 2;
      while (vs < 32 && vs * 4 < mean_deg) vs *= 2;
      c->vs = opts.spmv_vector > 0 ? opts.spmv_vector : vs;
    }
    *reached_dist = true;
    sfairsc_status ds = dist_build(c, W, groups, hh, cnt, opts);
    if (ds != SFAIRSC_OK) return bail(ds);
    c->t_build = now_s() - t0;
    *out = c;
    return SFAIRSC_OK;
  }

  // device allocations
  // CSR padded by 8 entries: the TMA SpMV's bulk copies round their ranges out to 16-byte boundaries
  CUB(dalloc(&c->rp, n + 1 + 8));
  CUB(dalloc(&c->ci, nnz + 8));
  CUB(dalloc(&c->vv, nnz + 8));
  // per-vertex arrays padded to ldv rows (the TMA sweeps stage whole 64-row chunks)
  CUB(dalloc(&c->dg, c->ldv));
  CUB(cudaMemset(c->dg, 0, sizeof(double) * c->ldv));
  if (c->normalized) {
    CUB(dalloc(&c->s, c->ldv));
    CUB(cudaMemset(c->s, 0, sizeof(double) * c->ldv));
  }
  CUB(dalloc(&c->grp, c->ldv));
  CUB(cudaMemset(c->grp, 0, c->ldv));
  CUB(dalloc(&c->isb, 256));
  CUB(dalloc(&c->uh, 256));
  CUB(dalloc(&c->counters, 16));
  CUB(cudaMemset(c->counters, 0, 16 * sizeof(unsigned)));
  CUB(dalloc(&c->flags, 4));
  CUB(cudaMemset(c->flags, 0, 4 * sizeof(int)));
  for (double** p : {&c->bs_w, &c->bs_t, &c->bs_v, &c->nb, &c->scal}) {
    CUB(dalloc(p, 512));
    CUB(cudaMemset(*p, 0, 512 * sizeof(double)));
  }
  CUB(dalloc(&c->c1, 4 * kMaxJ));
  CUB(dalloc(&c->c2, 4 * kMaxJ));
  for (double** p : {&c->vp, &c->vt, &c->vr, &c->vy}) {
    CUB(dalloc(p, c->ldv));
    CUB(cudaMemsetAsync(*p, 0, c->ldv * sizeof(double), c->st));
  }
  CUB(cudaMallocHost((void**)&c->hp, 4096 * sizeof(double)));

  // A0: library-owned copies of W and groups
  const cudaMemcpyKind kind = dev_in ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CUB(cudaMemcpyAsync(c->rp, W->row_ptr, sizeof(int) * (n + 1), kind, c->st));
  if (nnz > 0) {
    CUB(cudaMemcpyAsync(c->ci, W->col_idx, sizeof(int) * nnz, kind, c->st));
    CUB(cudaMemcpyAsync(c->vv, W->values, sizeof(double) * nnz, kind, c->st));
  }
  {
    int32_t* dgroups = nullptr;
    CUB(dalloc(&dgroups, n));
    CUB(cudaMemcpyAsync(dgroups, hg.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->st));
    launch_group_check(dgroups, n, hh, c->grp, c->flags, c->st);
    CUB(cudaStreamSynchronize(c->st));
    cudaFree(dgroups);
  }
  // row_ptr on host (nnz-balanced SpMV partition)
  std::vector<int32_t> hrp(n + 1);
  if (dev_in) {
    CUB(cudaMemcpy(hrp.data(), W->row_ptr, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost));
  } else {
    std::memcpy(hrp.data(), W->row_ptr, sizeof(int32_t) * (n + 1));
  }
  launch_validate_csr(c->g(), c->check_symmetry, c->flags, c->st);
  CUB(cudaGetLastError());
  int hflags = 0;
  CUB(cudaMemcpyAsync(&hflags, c->flags, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  CUB(cudaStreamSynchronize(c->st));
  if (hflags & 1) return bail(fail(SFAIRSC_E_CSR_INVALID, "CSR invalid (row_ptr/col range, unsorted or duplicate columns, or nonzero diagonal)"));
  if (hflags & 2) return bail(fail(SFAIRSC_E_NEGATIVE_WEIGHT, "negative or NaN weight (P:121)"));
  if (hflags & 4) return bail(fail(SFAIRSC_E_ASYMMETRIC, "W is not symmetric"));
  // unit-weight pattern (every stored w_ij = 1): the single-vector SpMV needs no value stream
  // (env SFAIRSC_UNIT=0 keeps the value-streaming kernel, for A/B measurements)
  c->unit = nnz > 0 && !(hflags & 32) && !(getenv("SFAIRSC_UNIT") && atoi(getenv("SFAIRSC_UNIT")) == 0);
  // A1: degrees d = W 1
  launch_degrees(c->g(), c->dg, c->flags, c->st);
  CUB(cudaMemcpyAsync(&hflags, c->flags, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  CUB(cudaStreamSynchronize(c->st));
  if (hflags & 8) return bail(fail(SFAIRSC_E_ISOLATED_VERTEX, "isolated vertex: d_i = 0 (P:127-128)"));
  if (c->normalized) {
    launch_inv_sqrt(c->dg, c->s, n, c->st);                   // s = d^{-1/2}
    launch_scale_values(c->rp, c->ci, c->vv, c->s, n, c->st);  // stored values s_i w_ij s_j
  }
  // A2: sigma = ||L||_1
  launch_sigma(c->g(), c->vt, c->counters + 0, c->scal, c->st);
  CUB(cudaGetLastError());
  double hsig = 0.0;
  CUB(cudaMemcpyAsync(&hsig, c->scal, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CUB(cudaStreamSynchronize(c->st));
  c->sigma = opts.sigma_override > 0 ? opts.sigma_override : hsig;

  // column blocking (single GPU, single-vector solvers): when 8n bytes of the gathered vector exceed what
  // L2 keeps across the CSR stream (~48 MB), the SpMV runs per column block on a block-major copy of W
  {
    const double pbytes = 8.0 * n;
    const double blk_bytes = getenv("SFAIRSC_COLBLK_MB") ? atof(getenv("SFAIRSC_COLBLK_MB")) * 1048576.0 : 48.0 * 1048576.0;
    if (c->bsz == 1 && pbytes > 1.34 * blk_bytes && nnz > 0) {
      const int nb = (int)std::ceil(pbytes / blk_bytes);
      const int cb = (n + nb - 1) / nb;
      int* cnt = nullptr;
      CUB(dalloc(&cnt, (size_t)nb * n));
      launch_colblk_starts(c->rp, c->ci, n, nb, cb, cnt, c->st);
      std::vector<int32_t> hc((size_t)nb * n);
      CUB(cudaMemcpyAsync(hc.data(), cnt, sizeof(int32_t) * hc.size(), cudaMemcpyDeviceToHost, c->st));
      CUB(cudaStreamSynchronize(c->st));
      cudaFree(cnt);
      std::vector<int32_t> hr((size_t)nb * (n + 1));
      long long base = 0;
      for (int b = 0; b < nb; ++b) {
        int32_t* r = hr.data() + (size_t)b * (n + 1);
        const int32_t* q = hc.data() + (size_t)b * n;
        r[0] = (int32_t)base;
        for (int i = 0; i < n; ++i) r[i + 1] = r[i] + q[i];
        base = r[n];
      }
      if (base != nnz) return bail(fail(SFAIRSC_E_CUDA, "column blocking lost entries (%lld vs %d)", base, nnz));
      CUB(dalloc(&c->rpb, hr.size()));
      CUB(cudaMemcpyAsync(c->rpb, hr.data(), sizeof(int32_t) * hr.size(), cudaMemcpyHostToDevice, c->st));
      // unit weights: after the build only the single-vector SpMV reads W here, and it streams column
      // indices only (pairs need an unblocked CSR, block Lanczos and the dense projector keep the values)
      const bool drop_vals = c->unit && c->bsz == 1 && !g_build_keep_values;
      int* ci2 = nullptr;
      double* vv2 = nullptr;
      CUB(dalloc(&ci2, nnz));
      if (!drop_vals) CUB(dalloc(&vv2, nnz));
      launch_colblk_scatter(c->rp, c->ci, drop_vals ? nullptr : c->vv, n, nb, c->rpb, ci2, vv2, c->st);
      CUB(cudaGetLastError());
      CUB(cudaStreamSynchronize(c->st));
      cudaFree(c->ci);
      cudaFree(c->vv);
      c->ci = ci2;
      c->vv = vv2;
      // the value array's HBM (8 nnz bytes) goes back to the Krylov basis, up to the preferred size
      if (drop_vals && opts.max_basis <= 0 && c->m < m_pref && !(opts.comm || opts.virtual_parts > 1)) {
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) == cudaSuccess && fr > 0) {
          const double vbytes = 8.0 * (double)c->ldv;
          const double fixed = ((double)k + 15.0) * vbytes + 256.0 * (1 << 20);
          const int mfit = (int)std::floor((0.97 * (double)fr - fixed) / (2.0 * vbytes)) - 1;
          int mnew = std::min(m_pref, mfit);
          if (c->lagged) mnew = std::min(mnew, std::min(192, n - hh));
          if (mnew > c->m) {
            c->m = m = mnew;
            c->keep = opts.keep > 0 ? opts.keep : k + (m - k) / 4;
            c->keep = std::max(std::min(c->keep, m - 1), std::min(k, m - 1));
          }
        }
      }
      c->nblk = nb;
      const double mdb = (double)nnz / n / nb;
      int vsb = 2;
      while (vsb < 32 && vsb * 4 < mdb) vsb *= 2;
      c->vs_blk = vsb;
    }
  }
  // the single-vector SpMV is the TMA-fed tile kernel unless column-blocked or dense-projected
  c->spmv_tma = c->nblk <= 1 && nnz > 0 && !c->Qr && !(getenv("SFAIRSC_SPMV_TMA") && atoi(getenv("SFAIRSC_SPMV_TMA")) == 0);
  // normalized pattern-only SpMV: its gathered vector s o p (vq_lz: the lagged solver's, written by its
  // normalisation kernel)
  if (c->unit_spmv() && c->normalized) {
    CUB(dalloc(&c->vq, c->ldv));
    CUB(dalloc(&c->vq_lz, c->ldv));
    CUB(cudaMemsetAsync(c->vq, 0, sizeof(double) * c->ldv, c->st));
    CUB(cudaMemsetAsync(c->vq_lz, 0, sizeof(double) * c->ldv, c->st));
  }
  // A3: factored basis of range(C): beta_s = sum_{V_s} s_i^2, u_s = |V_s| beta_s^{-1/2}
  c->sgrid = sweep_grid(n, c->num_sms);
  // SpMV partition: CTA b owns rows with cumulative (nnz + 4 rows) weight in [b, b+1)/G
  {
    const long long total = (long long)nnz + 4LL * n;
    // 8 CTAs per SM (5 and 10 measured slower)
    int G = std::max(1, std::min(c->num_sms * 8, (n + 31) / 32));
    std::vector<int32_t> split(G + 1);
    split[0] = 0;
    split[G] = n;
    for (int b = 1; b < G; ++b) {
      const long long target = total * b / G;
      int lo = 0, hi = n;
      while (lo < hi) {
        const int mid = lo + ((hi - lo) >> 1);
        if ((long long)hrp[mid] + 4LL * mid < target) lo = mid + 1; else hi = mid;
      }
      split[b] = std::max(split[b - 1], lo);
    }
    c->spmv_grid = G;
    CUB(dalloc(&c->row_split, G + 1));
    CUB(cudaMemcpyAsync(c->row_split, split.data(), sizeof(int32_t) * (G + 1), cudaMemcpyHostToDevice, c->st));

    const double mean_deg = n > 0 ? (double)nnz / n : 0.0;
    {
      int maxdeg = 0;
      for (int i = 0; i < n; ++i) maxdeg = std::max(maxdeg, hrp[i + 1] - hrp[i]);
      c->skewed = maxdeg > 16.0 * std::max(1.0, mean_deg);
    }
    int vs = 2;
    while (vs < 32 && vs * 4 < mean_deg) vs *= 2;
    const bool tma = c->spmv_tma;
    if (tma) {  // the TMA SpMV's lane reads 4-entry blocks, two per pass: VS = largest power of two <= mean degree / 16
      vs = 2;    // (config 4, mean degree 32: VS 2 525 us, VS 4 543 us; config 3, 64: VS 4 170 us, VS 2 272 us)
      while (vs < 32 && vs * 32 <= mean_deg) vs *= 2;
    }
    c->vs = opts.spmv_vector > 0 ? opts.spmv_vector : vs;
    if (c->vs != 2 && c->vs != 4 && c->vs != 8 && c->vs != 16 && c->vs != 32)
      return bail(fail(SFAIRSC_E_INVALID_ARG, "spmv_vector must be 2,4,8,16 or 32"));
    // TMA-fed SpMV (spmv_tma.cu): row-aligned tiles
    // padded CSR copy (rows start at multiples of 4 entries) + tiles; the plain CSR stays for the other kernels
    if (tma) {
      std::vector<int2> tiles;
      std::vector<int> cta, prp;
      // tiles of <= 2048 padded entries / 128 rows, 2-deep ring: config 4 SpMV 579 -> 525 us against 1024 / 64
      // (profiles/r2_exp/spmv_tile_sweep.jsonl; 1536-4096 entries, 64-128 rows, 3 stages and 12 gathers per lane
      // in flight measured equal or slower)
      c->spmv_shape = spmv_tile_shape(2048, 128, 2, c->unit_spmv());
      spmv_tma_layout(hrp.data(), n, spmv_tma_ctas_per_sm(c->vs, c->normalized, c->unit_spmv(), c->spmv_shape) * c->num_sms,
                      c->spmv_shape, prp, tiles, cta);
      c->tma_grid = (int)cta.size() - 1;
      CUB(dalloc(&c->tiles, tiles.size()));
      CUB(dalloc(&c->cta_tiles, cta.size()));
      CUB(dalloc(&c->prp, prp.size() + 8));
      c->nnz_pad = prp[n];
      CUB(dalloc(&c->pci, (size_t)prp[n]));
      if (!c->unit_spmv()) CUB(dalloc(&c->pvv, (size_t)prp[n]));
      CUB(cudaMemcpyAsync(c->tiles, tiles.data(), sizeof(int2) * tiles.size(), cudaMemcpyHostToDevice, c->st));
      CUB(cudaMemcpyAsync(c->cta_tiles, cta.data(), sizeof(int) * cta.size(), cudaMemcpyHostToDevice, c->st));
      CUB(cudaMemcpyAsync(c->prp, prp.data(), sizeof(int) * prp.size(), cudaMemcpyHostToDevice, c->st));
      launch_pad_csr(c->rp, c->ci, c->pvv ? c->vv : nullptr, n, c->prp, c->pci, c->pvv, c->st);
      CUB(cudaGetLastError());
      CUB(cudaStreamSynchronize(c->st));  // the host vectors die here
    }
  }
  // partial buffers: max over users
  {
    size_t need = std::max<size_t>((size_t)c->sgrid * (kMaxJ + 1), (size_t)c->spmv_grid * kHB);
    need = std::max<size_t>(need, (size_t)c->num_sms * 16 * (kHB + 1));
    need = std::max<size_t>(need, (size_t)c->sgrid * (kHB + 1));
    c->partials_cnt = need;
    CUB(dalloc(&c->partials, need));
  }
  {
    std::vector<double> beta(hh), isb(hh), uh(hh);
    if (c->normalized) {
      gsum_all(c, c->s, c->bs_w);  // B^T s = sum_{V_s} s_i^2
      CUB(cudaGetLastError());
      CUB(cudaMemcpyAsync(c->hp, c->bs_w, sizeof(double) * hh, cudaMemcpyDeviceToHost, c->st));
      CUB(cudaStreamSynchronize(c->st));
      for (int s = 0; s < hh; ++s) beta[s] = c->hp[s];
    } else {
      for (int s = 0; s < hh; ++s) beta[s] = (double)cnt[s];
    }
    double un = 0.0;
    for (int s = 0; s < hh; ++s) {
      if (!(beta[s] > 0)) return bail(fail(SFAIRSC_E_RANK_DEFICIENT, "group %d has zero weight", s));
      isb[s] = 1.0 / std::sqrt(beta[s]);
      uh[s] = (double)cnt[s] * isb[s];
      un += uh[s] * uh[s];
    }
    un = std::sqrt(un);
    for (int s = 0; s < hh; ++s) uh[s] /= un;
    CUB(cudaMemcpyAsync(c->isb, isb.data(), sizeof(double) * hh, cudaMemcpyHostToDevice, c->st));
    CUB(cudaMemcpyAsync(c->uh, uh.data(), sizeof(double) * hh, cudaMemcpyHostToDevice, c->st));
  }
  // Krylov basis (double-buffered for thick restarts) and eigenvector block
  const int vcols = m + std::max(1, c->bsz);
  CUB(dalloc(&c->V, (size_t)vcols * c->ldv));
  CUB(dalloc(&c->Vb, (size_t)vcols * c->ldv));
  CUB(cudaMemsetAsync(c->V, 0, sizeof(double) * vcols * c->ldv, c->st));
  CUB(cudaMemsetAsync(c->Vb, 0, sizeof(double) * vcols * c->ldv, c->st));
  CUB(dalloc(&c->Ydev, (size_t)(m + 1) * (m + 1)));
  CUB(dalloc(&c->talpha, m + 1));
  CUB(dalloc(&c->tbeta, m + 1));
  CUB(dalloc(&c->X, (size_t)k * c->ldv));
  CUB(cudaMemsetAsync(c->X, 0, sizeof(double) * k * c->ldv, c->st));
  if (c->lagged) {
    c->ldT = m + 2;
    CUB(dalloc(&c->Hdev, (size_t)c->ldT * c->ldT));
    CUB(dalloc(&c->sdev, m + 2));
    CUB(dalloc(&c->lz, 16));
    CUB(cudaMemsetAsync(c->lz, 0, sizeof(double) * 16, c->st));
    CUB(dalloc(&c->partials2, (size_t)c->num_sms * (kHB + 2) + 64));
    c->paired = c->paired && m <= kPairMaxM;  // the pair sweep's 2-stage ring fits up to J = m - 1 <= 185
    if (c->paired) {
      CUB(dalloc(&c->vrB, c->ldv));
      CUB(cudaMemsetAsync(c->vrB, 0, sizeof(double) * c->ldv, c->st));
      CUB(dalloc(&c->lzp, 8 * kMaxJ));
      CUB(cudaMemsetAsync(c->lzp, 0, sizeof(double) * 8 * kMaxJ, c->st));
    }
    CUB(dalloc(&c->dd, kMaxJ + 8));
    CUB(dalloc(&c->bflags, kMaxJ + 8));
    CUB(cudaMemsetAsync(c->bflags, 0, sizeof(int) * (kMaxJ + 8), c->st));
  }
  if (c->filter_deg >= 2) {
    CUB(dalloc(&c->fbuf, 2 * (size_t)c->ldv));
    CUB(cudaMemsetAsync(c->fbuf, 0, sizeof(double) * 2 * c->ldv, c->st));
    CUB(dalloc(&c->fth, kMaxJ));
  }
  if (c->bsz > 1) {  // block Lanczos buffers (m + bsz basis columns: V/Vb above hold m + 1 <= m + bsz)
    const int nbz = c->bsz;
    for (double** p : {&c->bP, &c->bT, &c->bR}) {
      CUB(dalloc(p, (size_t)c->ldv * nbz));
      CUB(cudaMemsetAsync(*p, 0, sizeof(double) * c->ldv * nbz, c->st));
    }
    c->ldT = m + nbz;
    CUB(dalloc(&c->Tdev, (size_t)c->ldT * c->ldT));
    CUB(cudaMemsetAsync(c->Tdev, 0, sizeof(double) * c->ldT * c->ldT, c->st));
    CUB(dalloc(&c->g2, 64));
    CUB(dalloc(&c->bflags, kMaxJ + 8));
    CUB(cudaMemsetAsync(c->bflags, 0, sizeof(int) * (kMaxJ + 8), c->st));
  }
  CUB(cudaStreamSynchronize(c->st));
  c->t_build = now_s() - t0;
  *out = c;
#undef CUB
  return SFAIRSC_OK;
}

// §8(f) N4: general constraints C^T H = 0 with a dense F (n x r).  Builds the operator with the group
// machinery switched off (h = 1: P = I), then forms Q = orth(C), C = D^{-1/2} F (normalized) or F, by
// CholQR2 and switches every projector kernel to the dense rows of Q.
extern "C" sfairsc_status sfairsc_build_operator_dense(const sfairsc_csr* W, const double* F, int32_t r, int32_t k,
                                                       int32_t normalized, const sfairsc_opts* opts_in,
                                                       sfairsc_ctx** out) {
  if (!W || !out || (r > 0 && !F)) return fail(SFAIRSC_E_INVALID_ARG, "null argument");
  if (r < 0 || r > kMaxFCols) return fail(SFAIRSC_E_INVALID_ARG, "r must be in [0, %d]", kMaxFCols);
  *out = nullptr;
  sfairsc_opts opts;
  sfairsc_default_opts(&opts);
  if (opts_in) opts = *opts_in;
  if (opts.comm || opts.virtual_parts > 1) return fail(SFAIRSC_E_INVALID_ARG, "dense constraints: single GPU only");
  if (opts.block_size > 1 || opts.reorth == 1)
    return fail(SFAIRSC_E_INVALID_ARG, "dense constraints use the single-sweep solver (block_size 0/1, reorth 0/2)");
  const long long n = W->n_rows;
  if (n < 2 || k < 1 || (long long)k > n - 1) return fail(SFAIRSC_E_K_TOO_LARGE, "k=%d > n - 1 = %lld", k, n - 1);
  opts.block_size = 1;
  opts.reorth = 2;
  if (opts.max_basis <= 0) {
    int m = std::min(192, std::max(std::max(2 * k + 10, 17 * k / 5), 20));
    opts.max_basis = (int)std::min<long long>(m, n - std::min<long long>(r, kHB) - 1);
  }
  std::vector<int32_t> zeros((size_t)n, 0);
  int32_t* gz = zeros.data();
  int32_t* gzd = nullptr;
  if (W->memspace == SFAIRSC_MEM_DEVICE) {
    CU(cudaMalloc(&gzd, sizeof(int32_t) * n));
    CU(cudaMemset(gzd, 0, sizeof(int32_t) * n));
    gz = gzd;
  }
  sfairsc_ctx* c = nullptr;
  g_build_keep_values = true;
  sfairsc_status st0 = sfairsc_build_operator_ex(W, gz, 1, k, normalized, &opts, &c);
  g_build_keep_values = false;
  if (gzd) cudaFree(gzd);
  if (st0 != SFAIRSC_OK) return st0;
  if (r == 0) {
    *out = c;
    return SFAIRSC_OK;
  }
  auto bail = [&](sfairsc_status s) {
    sfairsc_destroy(c);
    return s;
  };
  const int ni = (int)n;
  double *Cd = nullptr, *Q1 = nullptr, *G = nullptr, *Td = nullptr;
  auto cleanup = [&]() {
    if (Cd) cudaFree(Cd);
    if (Q1) cudaFree(Q1);
    if (G) cudaFree(G);
    if (Td) cudaFree(Td);
  };
#define CUD(expr)                                                                                       \
  do {                                                                                                  \
    cudaError_t e_ = (expr);                                                                            \
    if (e_ != cudaSuccess) {                                                                            \
      cleanup();                                                                                        \
      return bail(fail(e_ == cudaErrorMemoryAllocation ? SFAIRSC_E_OOM : SFAIRSC_E_CUDA, "%s: %s", #expr, \
                       cudaGetErrorString(e_)));                                                        \
    }                                                                                                   \
  } while (0)
  CUD(cudaMalloc(&Cd, sizeof(double) * (size_t)n * r));
  CUD(cudaMemcpyAsync(Cd, F, sizeof(double) * (size_t)n * r,
                      W->memspace == SFAIRSC_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->st));
  if (c->normalized) launch_scale_rows(Cd, n, ni, r, c->s, c->st);  // C = D^{-1/2} F
  CUD(cudaMalloc(&G, sizeof(double) * r * r));
  CUD(cudaMalloc(&Td, sizeof(double) * r * kHB));
  // pass 0, rank revealing (reading R21; P:819-822 allow any C whose least-squares problem min ||C z - w|| the
  // projector solves): G = C^T C = V diag(lam) V^T; the numerical rank rq = #{lam_i > 1e-14 lam_max} (singular
  // values above 1e-7 of the largest: what a Gram matrix resolves in fp64); Q1 = C V_rq diag(lam_rq)^{-1/2} spans
  // range(C) = the range of the P:809 projector's C (C^+ of a rank-deficient C: the minimum-norm LS solution)
  std::vector<double> Gh((size_t)r * r), lam;
  CUD(cudaMemsetAsync(G, 0, sizeof(double) * r * r, c->st));
  launch_gram_pairs(Cd, 1, n, ni, r, G, c->st);
  CUD(cudaMemcpyAsync(Gh.data(), G, sizeof(double) * r * r, cudaMemcpyDeviceToHost, c->st));
  CUD(cudaStreamSynchronize(c->st));
  for (int a = 0; a < r; ++a)
    for (int b = 0; b < a; ++b) Gh[(size_t)a * r + b] = Gh[(size_t)b * r + a];
  symeig(r, Gh, lam);  // ascending; Gh[a * r + c] = component a of eigenvector c
  const double lmax = lam[r - 1];
  int rq = 0;
  for (int i = r - 1; i >= 0; --i)
    if (lmax > 0.0 && lam[i] > 1e-14 * lmax) ++rq;
  if (rq > kHB) {
    cleanup();
    return bail(fail(SFAIRSC_E_INVALID_ARG, "numerical rank %d of C exceeds %d (the projector's row width)", rq, kHB));
  }
  if ((long long)k > n - rq) {
    cleanup();
    return bail(fail(SFAIRSC_E_K_TOO_LARGE, "k=%d > n - rank(C) = %lld", k, n - rq));
  }
  c->qr = rq;
  c->rank_in = r;  // dense-F context (constraint_rank = qr)
  if (rq == 0) {  // C = 0: no constraint (P = I)
    cleanup();
    *out = c;
    return SFAIRSC_OK;
  }
  c->ldq = (rq + 1) / 2 * 2;  // 16-byte rows for the TMA bulk copies
  CUD(cudaMalloc(&Q1, sizeof(double) * (size_t)c->ldv * c->ldq));
  CUD(cudaMemsetAsync(Q1, 0, sizeof(double) * (size_t)c->ldv * c->ldq, c->st));
  CUD(cudaMalloc(&c->Qr, sizeof(double) * (size_t)c->ldv * c->ldq));
  CUD(cudaMemsetAsync(c->Qr, 0, sizeof(double) * (size_t)c->ldv * c->ldq, c->st));
  {
    std::vector<double> T((size_t)r * rq);
    for (int j = 0; j < rq; ++j) {  // largest eigenvalue first
      const int col = r - 1 - j;
      const double is = 1.0 / std::sqrt(lam[col]);
      for (int a = 0; a < r; ++a) T[(size_t)a * rq + j] = Gh[(size_t)a * r + col] * is;
    }
    CUD(cudaMemcpyAsync(Td, T.data(), sizeof(double) * T.size(), cudaMemcpyHostToDevice, c->st));
    launch_rows_times(Cd, 1, n, ni, r, rq, Td, Q1, c->ldq, c->st);
    CUD(cudaGetLastError());
    CUD(cudaStreamSynchronize(c->st));
  }
  // pass 1: one Cholesky-QR step Q = Q1 U^{-1} (Q1^T Q1 = I up to cond(C)^2 eps: CholQR2 in total)
  {
    const int q = rq;
    std::vector<double> Gq((size_t)q * q), U((size_t)q * q, 0.0), Ui((size_t)q * q, 0.0);
    CUD(cudaMemsetAsync(G, 0, sizeof(double) * q * q, c->st));
    launch_gram_pairs(Q1, c->ldq, 1, ni, q, G, c->st);
    CUD(cudaMemcpyAsync(Gq.data(), G, sizeof(double) * q * q, cudaMemcpyDeviceToHost, c->st));
    CUD(cudaStreamSynchronize(c->st));
    for (int a = 0; a < q; ++a)
      for (int b = 0; b < a; ++b) Gq[(size_t)a * q + b] = Gq[(size_t)b * q + a];
    for (int j = 0; j < q; ++j) {  // G = U^T U (U upper)
      double d = Gq[(size_t)j * q + j];
      for (int p = 0; p < j; ++p) d -= U[(size_t)p * q + j] * U[(size_t)p * q + j];
      if (!(d > 0.25)) {  // Q1 is orthonormal to far better than this unless the rank decision was wrong
        cleanup();
        return bail(fail(SFAIRSC_E_RANK_DEFICIENT, "constraint basis lost orthogonality (rank decision %d of %d)", q, r));
      }
      U[(size_t)j * q + j] = std::sqrt(d);
      for (int i = j + 1; i < q; ++i) {
        double v = Gq[(size_t)j * q + i];
        for (int p = 0; p < j; ++p) v -= U[(size_t)p * q + j] * U[(size_t)p * q + i];
        U[(size_t)j * q + i] = v / U[(size_t)j * q + j];
      }
    }
    for (int j = 0; j < q; ++j) {
      Ui[(size_t)j * q + j] = 1.0 / U[(size_t)j * q + j];
      for (int i = j - 1; i >= 0; --i) {
        double v = 0.0;
        for (int p = i + 1; p <= j; ++p) v += U[(size_t)i * q + p] * Ui[(size_t)p * q + j];
        Ui[(size_t)i * q + j] = -v / U[(size_t)i * q + i];
      }
    }
    CUD(cudaMemcpyAsync(Td, Ui.data(), sizeof(double) * Ui.size(), cudaMemcpyHostToDevice, c->st));
    launch_rows_times(Q1, c->ldq, 1, ni, q, q, Td, c->Qr, c->ldq, c->st);
    CUD(cudaGetLastError());
    CUD(cudaStreamSynchronize(c->st));
  }
  cleanup();
#undef CUD
  *out = c;
  return SFAIRSC_OK;
}

extern "C" void sfairsc_destroy(sfairsc_ctx* c) {
  if (!c) return;
  if (c->st) cudaStreamSynchronize(c->st);
  free_ctx(c);
}

// --------------------------------------------------------------------------
// apply / project / laplacian entry points
// --------------------------------------------------------------------------
static sfairsc_status vec_io(sfairsc_ctx* c, const double* x, double* y, int32_t nvec, int32_t memspace,
                             sfairsc_status (*op)(sfairsc_ctx*, const double*, double*), bool allow_pairs = true) {
  if (!c || !x || !y || nvec < 0) return fail(SFAIRSC_E_INVALID_ARG, "null argument");
  if (memspace != SFAIRSC_MEM_HOST && memspace != SFAIRSC_MEM_DEVICE) return fail(SFAIRSC_E_INVALID_ARG, "memspace");
  if (c->dist) {  // row-partitioned: vectors hold this process's rows; only the operator apply is offered
    if (op != apply_dev) return fail(SFAIRSC_E_INVALID_ARG, "only sfairsc_apply is available on a row-partitioned context");
    const long long nl = dist_local_rows(c);
    double *dx = nullptr, *dy = nullptr;
    CU(cudaMalloc(&dx, sizeof(double) * std::max(nl, 1LL)));
    CU(cudaMalloc(&dy, sizeof(double) * std::max(nl, 1LL)));
    sfairsc_status rs = SFAIRSC_OK;
    const cudaMemcpyKind kin = memspace == SFAIRSC_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    const cudaMemcpyKind kout = memspace == SFAIRSC_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    for (int v = 0; v < nvec && rs == SFAIRSC_OK; ++v) {
      cudaMemcpyAsync(dx, x + (size_t)v * nl, sizeof(double) * nl, kin, c->st);
      rs = dist_apply(c, dx, dy);
      if (rs == SFAIRSC_OK) cudaMemcpyAsync(y + (size_t)v * nl, dy, sizeof(double) * nl, kout, c->st);
    }
    cudaStreamSynchronize(c->st);
    cudaFree(dx);
    cudaFree(dy);
    return rs;
  }
  const size_t nb = sizeof(double) * c->n;
  int v0 = 0;
  if (op == apply_dev && allow_pairs && pair_ok(c) && nvec >= 2 && memspace == SFAIRSC_MEM_DEVICE) {
    for (; v0 + 1 < nvec; v0 += 2)
      TRY(apply_pair_dev(c, x + (size_t)v0 * c->n, x + (size_t)(v0 + 1) * c->n, y + (size_t)v0 * c->n,
                         y + (size_t)(v0 + 1) * c->n));
  }
  for (int v = v0; v < nvec; ++v) {
    const double* xv = x + (size_t)v * c->n;
    double* yv = y + (size_t)v * c->n;
    if (memspace == SFAIRSC_MEM_HOST) {
      CU(cudaMemcpyAsync(c->vr, xv, nb, cudaMemcpyHostToDevice, c->st));
      TRY(op(c, c->vr, c->vy));
      CU(cudaMemcpyAsync(yv, c->vy, nb, cudaMemcpyDeviceToHost, c->st));
    } else {
      TRY(op(c, xv, yv));
    }
  }
  CU(cudaStreamSynchronize(c->st));
  if (c->prof.on) c->prof.resolve();
  return SFAIRSC_OK;
}

static sfairsc_status project_dev(sfairsc_ctx* c, const double* x, double* y) {
  ProfScope ps(c, K_PROJ, c->gpasses() * (c->vb() + c->sgb()) + 2 * c->vb() + c->sgb());
  gsum_all(c, x, c->bs_w);
  launch_project(c->g(), c->pd(), x, c->bs_w, 1.0, y, c->st);
  CHECK_LAUNCH();
  return SFAIRSC_OK;
}

static sfairsc_status lap_dev(sfairsc_ctx* c, const double* x, double* y) {
  ProfScope ps(c, K_SPMV, c->csr_bytes() + 3 * c->vb() + 1.0 * c->n);
  ctx_spmv(c, x, y);
  CHECK_LAUNCH();
  return SFAIRSC_OK;
}

extern "C" sfairsc_status sfairsc_apply(sfairsc_ctx* c, const double* x, double* y, int32_t nvec, int32_t memspace) {
  return vec_io(c, x, y, nvec, memspace, apply_dev);
}
extern "C" sfairsc_status sfairsc_apply_ex(sfairsc_ctx* c, const double* x, double* y, int32_t nvec,
                                           int32_t memspace, int32_t flags) {
  NvtxRange nv("sfairsc.apply");
  if (flags & ~SFAIRSC_APPLY_SINGLE) return fail(SFAIRSC_E_INVALID_ARG, "unknown apply flags");
  return vec_io(c, x, y, nvec, memspace, apply_dev, (flags & SFAIRSC_APPLY_SINGLE) == 0);
}
extern "C" sfairsc_status sfairsc_project(sfairsc_ctx* c, const double* x, double* y, int32_t nvec,
                                          int32_t memspace) {
  return vec_io(c, x, y, nvec, memspace, project_dev);
}
extern "C" sfairsc_status sfairsc_laplacian(sfairsc_ctx* c, const double* x, double* y, int32_t memspace) {
  if (c && x == y) return fail(SFAIRSC_E_INVALID_ARG, "x and y must not alias");
  return vec_io(c, x, y, 1, memspace, lap_dev);
}

// --------------------------------------------------------------------------
// profiling
// --------------------------------------------------------------------------
extern "C" sfairsc_status sfairsc_profile_enable(sfairsc_ctx* c, int32_t enable) {
  if (!c) return fail(SFAIRSC_E_INVALID_ARG, "null ctx");
  CU(cudaStreamSynchronize(c->st));
  c->prof.resolve();
  c->prof.on = enable != 0;
  return SFAIRSC_OK;
}
extern "C" sfairsc_status sfairsc_profile_read(sfairsc_ctx* c, int32_t kind, double* total_ms, int64_t* launches,
                                               double* alg_bytes) {
  if (!c || kind < 0 || kind >= 10) return fail(SFAIRSC_E_INVALID_ARG, "bad argument");
  CU(cudaStreamSynchronize(c->st));
  c->prof.resolve();
  if (total_ms) *total_ms = c->prof.total_ms[kind];
  if (launches) *launches = c->prof.launches[kind];
  if (alg_bytes) *alg_bytes = c->prof.bytes[kind];
  return SFAIRSC_OK;
}
extern "C" sfairsc_status sfairsc_profile_reset(sfairsc_ctx* c) {
  if (!c) return fail(SFAIRSC_E_INVALID_ARG, "null ctx");
  CU(cudaStreamSynchronize(c->st));
  c->prof.resolve();
  for (int i = 0; i < 10; ++i) {
    c->prof.total_ms[i] = 0;
    c->prof.launches[i] = 0;
    c->prof.bytes[i] = 0;
  }
  return SFAIRSC_OK;
}

// --------------------------------------------------------------------------
// thick-restart Lanczos (A7-A11)
// --------------------------------------------------------------------------
struct Lanczos {
  sfairsc_ctx* c;
  int m, keep, k;
  int pk = 0;  // number of kept Ritz vectors heading the basis (arrow part of T)
  std::vector<double> alpha, beta, arrow;
  int64_t applies = 0, steps = 0, restarts = 0, breakdowns = 0;
  unsigned inject = 0;
  double bd_tol = 0.0;

  double* col(int j) const { return c->V + (long long)j * c->ldv; }

  SweepArgs sargs(int J, const double* xin, double* xout, const double* coef) const {
    SweepArgs a{};
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
    a.norm_bsum = c->nb;
    return a;
  }

  // one sweep; returns the grid used (= number of partial rows)
  int sweep(int mode, const SweepArgs& a) {
    // dots-type modes: TMA-fed persistent sweep; update + norm (mode 2): the register kernel (measured faster)
    if (sweep_tma_ok(a.J) && mode != 2) {
      const int G = sweep_tma_grid(c->n, c->num_sms);
      launch_sweep_tma(mode, c->g(), c->pd(), a, G, c->st);
      return G;
    }
    launch_sweep(mode, c->g(), c->pd(), a, c->sgrid, c->st);
    return c->sgrid;
  }

  // CGS2 of r against V[:, 0:J]: |r''|^2 and B^T r'' land in nb.
  // from_t: r = finish(t) (= L^sigma v_j) fused into the first sweep.
  sfairsc_status cgs2(int J, bool from_t) {
    GraphDev g = c->g();
    ProjDesc pd = c->pd();
    if (J > 0) {
      {
        ProfScope ps(c, K_DOTS, J * c->vb() + (from_t ? 2 * c->vb() + c->sgb() : c->vb()));
        const int G = sweep(from_t ? 0 : 3, sargs(J, from_t ? c->vt : c->vr, c->vr, nullptr));
        launch_reduce_cols(c->partials, G, J, c->c1, c->st);
      }
      {
        ProfScope ps(c, K_UPDDOT, J * c->vb() + 2 * c->vb());
        const int G = sweep(1, sargs(J, c->vr, c->vr, c->c1));
        launch_reduce_cols(c->partials, G, J, c->c2, c->st);
      }
    } else if (from_t) {
      ProfScope ps(c, K_DOTS, 2 * c->vb() + c->sgb());
      launch_finish(g, pd, c->vt, c->bs_t, c->bs_v, c->sigma, c->vr, c->st);
    }
    {
      ProfScope ps(c, K_UPDNORM, J * c->vb() + 2 * c->vb() + c->sgb());
      sweep(2, sargs(J, c->vr, c->vr, c->c2));
    }
    if (c->h > kHB) extra_gsums(c, c->vr, c->nb + 1);
    CHECK_LAUNCH();
    return SFAIRSC_OK;
  }

  // v_{j+1} = r''/beta into column j+1 (beta from device), recording T entries
  sfairsc_status normalize_step(int j) {
    ProfScope ps(c, K_NORMALIZE, 3 * c->vb() + c->sgb());
    NormArgs na{};
    na.nb = c->nb;
    na.beta_host = 0.0;
    na.bd_tol = bd_tol;
    na.j = j;
    na.c1 = c->c1;
    na.c2 = c->c2;
    na.alpha_dev = c->talpha;
    na.beta_dev = c->tbeta;
    na.flag = c->flags + 1;
    launch_normalize(c->g(), c->pd(), c->vr, na, col(j + 1), c->bs_v, c->vp, c->st);
    CHECK_LAUNCH();
    return SFAIRSC_OK;
  }

  // §8(f) N2: r = -p(L^sigma) x0 into vr, p(x) = (-1)^d T_d((x - cc)/e), by the Chebyshev three-term
  // recurrence y_1 = (A x0 - cc x0)/e, y_{i+1} = 2 (A y_i - cc y_i)/e - y_{i-1} (d applies; each apply's
  // finish kernel carries the recurrence)
  sfairsc_status filter_apply(const double* x0, double cut) {
    const int d = c->filter_deg;
    const double cc = 0.5 * (cut + c->sigma), e = 0.5 * (c->sigma - cut);
    const double sign = (d % 2 == 0) ? -1.0 : 1.0;  // -p = (-1)^(d+1) T_d
    double* F0 = c->fbuf;
    double* F1 = c->fbuf + c->ldv;
    const double* ycur = x0;
    const double* yprev = x0;
    for (int i = 1; i <= d; ++i) {
      {
        ProfScope ps(c, K_PROJ, c->gpasses() * (c->vb() + c->sgb()) + 2 * c->vb() + c->sgb());
        gsum_all(c, ycur, c->bs_w);
        launch_project(c->g(), c->pd(), ycur, c->bs_w, 1.0, c->vp, c->st);
      }
      {
        ProfScope ps(c, K_SPMV, c->csr_bytes() + 3 * c->vb() + 1.0 * c->n);
        ctx_spmv(c, c->vp, c->vt);
      }
      if (c->h > kHB) extra_gsums(c, c->vt, c->bs_t);
      double a = (i == 1 ? 1.0 : 2.0) / e, b = (i == 1 ? 0.0 : -1.0);
      if (i == d) {
        a *= sign;
        b *= sign;
      }
      // y_new: F0, then F1, then in place over y_{i-1} (never over x0, a basis column); the last into vr
      double* ynew = (i == d) ? c->vr : (i == 1 ? F0 : (i == 2 ? F1 : const_cast<double*>(yprev)));
      {
        ProfScope ps(c, K_FINISH, 4 * c->vb() + c->sgb());
        launch_finish_cheb(c->g(), c->pd(), c->vt, c->bs_t, c->bs_w, c->sigma, ycur, yprev, a, cc, b, ynew, c->st);
      }
      yprev = ycur;
      ycur = ynew;
    }
    CHECK_LAUNCH();
    applies += d;
    return SFAIRSC_OK;
  }

  // random vector orthogonalised (CGS2 twice) against V[:, 0:J], normalised into column J
  sfairsc_status random_vector(int J, bool project_first, bool from_vr = false) {
    for (int attempt = 0; attempt < 5; ++attempt) {
      if (from_vr && attempt == 0) {  // the caller's vector already in vr (filtered start, N2)
      } else if (project_first) {  // r = P u
        launch_random(c->vt, c->n, c->seed, inject++, 7u, c->st);
        gsum_all(c, c->vt, c->bs_w);
        launch_project(c->g(), c->pd(), c->vt, c->bs_w, 1.0, c->vr, c->st);
      } else {
        launch_random(c->vr, c->n, c->seed, inject++, 7u, c->st);
      }
      TRY(cgs2(J, false));
      if (J > 0) TRY(cgs2(J, false));
      CU(cudaMemcpyAsync(c->hp, c->nb, sizeof(double), cudaMemcpyDeviceToHost, c->st));
      CU(cudaStreamSynchronize(c->st));
      const double b = std::sqrt(c->hp[0]);
      if (b > 1e-8) {
        ProfScope ps(c, K_NORMALIZE, 3 * c->vb() + c->sgb());
        NormArgs na{};
        na.nb = c->nb;
        na.beta_host = b;
        na.bd_tol = 0.0;
        launch_normalize(c->g(), c->pd(), c->vr, na, col(J), c->bs_v, c->vp, c->st);
        CHECK_LAUNCH();
        return SFAIRSC_OK;
      }
    }
    return fail(SFAIRSC_E_NO_CONVERGENCE, "could not generate a random vector outside the Krylov basis");
  }

  // sync point: T entries [from, to) and the breakdown flag to the host
  sfairsc_status fetch_T(int from, int to, int* flag) {
    const int cnt = to - from;
    if (cnt > 0) {
      CU(cudaMemcpyAsync(c->hp, c->talpha + from, sizeof(double) * cnt, cudaMemcpyDeviceToHost, c->st));
      CU(cudaMemcpyAsync(c->hp + 1024, c->tbeta + from, sizeof(double) * cnt, cudaMemcpyDeviceToHost, c->st));
    }
    CU(cudaMemcpyAsync(c->hp + 2048, c->flags + 1, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    if (c->prof.on) c->prof.resolve();
    for (int i = 0; i < cnt; ++i) {
      alpha[from + i] = c->hp[i];
      beta[from + i] = c->hp[1024 + i];
    }
    std::memcpy(flag, c->hp + 2048, sizeof(int));
    return SFAIRSC_OK;
  }
};

// §8(f) N2: for the k columns of X (Ritz vectors of the filter, unit norm), theta_i = x_i^T L^sigma x_i and
// max_i ||L^sigma x_i - theta_i x_i|| / sigma (k applies); X's columns are put in increasing theta order
static sfairsc_status filter_check(sfairsc_ctx* c, int k, std::vector<double>* th, double* max_out) {
  std::vector<double> res(k);
  th->assign(k, 0.0);
  for (int i = 0; i < k; ++i) {
    const double* xi = c->X + (long long)i * c->ldv;
    TRY(apply_dev(c, xi, c->vy));
    launch_dot(xi, c->vy, c->n, c->partials, c->counters + 4, c->fth + i, c->st);
    launch_resid_dev(c->vy, xi, c->fth + i, c->n, c->partials, c->counters + 4, c->scal + 8 + i % 64, c->st);
    CHECK_LAUNCH();
    if (i % 64 == 63 || i == k - 1) {
      const int base = i - i % 64;
      CU(cudaMemcpyAsync(c->hp, c->scal + 8, sizeof(double) * (i - base + 1), cudaMemcpyDeviceToHost, c->st));
      CU(cudaStreamSynchronize(c->st));
      for (int q = base; q <= i; ++q) res[q] = std::sqrt(c->hp[q - base]) / c->sigma;
    }
  }
  CU(cudaMemcpyAsync(c->hp, c->fth, sizeof(double) * k, cudaMemcpyDeviceToHost, c->st));
  CU(cudaStreamSynchronize(c->st));
  std::vector<int> idx(k);
  for (int i = 0; i < k; ++i) {
    (*th)[i] = c->hp[i];
    idx[i] = i;
  }
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return (*th)[a] < (*th)[b]; });
  bool ident = true;
  for (int i = 0; i < k; ++i) ident = ident && idx[i] == i;
  if (!ident) {  // reorder X (Vb is free scratch at a convergence check)
    CU(cudaMemcpyAsync(c->Vb, c->X, sizeof(double) * (size_t)k * c->ldv, cudaMemcpyDeviceToDevice, c->st));
    std::vector<double> t2(k), r2(k);
    for (int i = 0; i < k; ++i) {
      CU(cudaMemcpyAsync(c->X + (long long)i * c->ldv, c->Vb + (long long)idx[i] * c->ldv, sizeof(double) * c->ldv,
                         cudaMemcpyDeviceToDevice, c->st));
      t2[i] = (*th)[idx[i]];
      r2[i] = res[idx[i]];
    }
    CU(cudaStreamSynchronize(c->st));
    *th = t2;
    res = r2;
  }
  double mx = 0.0;
  for (int i = 0; i < k; ++i) mx = std::max(mx, res[i]);
  *max_out = mx;
  return SFAIRSC_OK;
}

extern "C" sfairsc_status sfairsc_eigs(sfairsc_ctx* c, int32_t k, double tol, double* evals_out, double* evecs_out,
                                       int32_t evecs_memspace, sfairsc_stats* stats) {
  NvtxRange nv("sfairsc.eigs");
  const double t0 = now_s();
  if (c && c->debug) fprintf(stderr, "[sfairsc] eigs enter k=%d tol=%g\n", k, tol);
  if (!c || !evals_out) return fail(SFAIRSC_E_INVALID_ARG, "null argument");
  if (k < 1 || k > c->k_build) return fail(SFAIRSC_E_K_TOO_LARGE, "k=%d must be in [1, build k=%d]", k, c->k_build);
  if ((int64_t)k > (int64_t)c->n - c->h + 1) return fail(SFAIRSC_E_K_TOO_LARGE, "k > n-h+1");
  if (!(tol > 0)) return fail(SFAIRSC_E_INVALID_ARG, "tol must be > 0");
  if (evecs_out && evecs_memspace != SFAIRSC_MEM_HOST && evecs_memspace != SFAIRSC_MEM_DEVICE)
    return fail(SFAIRSC_E_INVALID_ARG, "memspace");
  if (c->bsz > 1) return eigs_block(c, k, tol, evals_out, evecs_out, evecs_memspace, stats);
  if (c->dist) return dist_eigs(c, k, tol, evals_out, evecs_out, evecs_memspace, stats);
  if (c->lagged) return eigs_lagged(c, k, tol, evals_out, evecs_out, evecs_memspace, stats);
  c->have_eigs = false;
  Lanczos L;
  L.c = c;
  L.m = c->m;
  L.k = k;
  L.keep = std::max(std::min(c->keep, L.m - 1), std::min(k, L.m - 1));
  L.alpha.assign(L.m + 1, 0.0);
  L.beta.assign(L.m + 1, 0.0);
  L.arrow.assign(L.m + 1, 0.0);
  const double tol_eff = std::min(tol, c->tol_cap);
  const double target = tol_eff * c->sigma;
  L.bd_tol = std::min(1e-12, 0.01 * tol_eff) * c->sigma;
  const int n = c->n;
  CU(cudaMemsetAsync(c->flags + 1, 0, sizeof(int), c->st));

  // start vector v_0 = P u / |P u|, u from Philox stream 7
  L.inject = 0;
  if (c->debug) fprintf(stderr, "[sfairsc] eigs start m=%d keep=%d\n", L.m, L.keep);
  TRY(L.random_vector(0, true));
  if (c->debug) fprintf(stderr, "[sfairsc] start vector ok\n");
  int j = 0;       // column being expanded
  int jsync = 0;   // first T index not yet fetched
  bool converged = false, complete = false;
  std::vector<double> theta, Y;
  int m_eff = 0;
  double gap = std::numeric_limits<double>::quiet_NaN();
  // §8(f) N2: Lanczos on B = -p(L^sigma); automatic cut: one unfiltered cycle first
  const bool filter = c->filter_deg >= 2;
  double cut = c->filter_cut;
  bool filtering = filter && cut > 0.0;
  if (filter && cut >= c->sigma) return fail(SFAIRSC_E_INVALID_ARG, "filter_cut=%g must be below sigma=%g", cut, c->sigma);
  double fthr = 0.0;        // filtered: B-residual estimate below which the explicit L^sigma check runs
  double fres = 0.0;        // filtered: the explicit check's max residual / sigma
  std::vector<double> thA;  // filtered: Rayleigh quotients x^T L^sigma x of the check
  for (;;) {
    // ---- expand column j: r = L^sigma v_j (filtered: -p(L^sigma) v_j), CGS2 against V[:, 0:j+1],
    // v_{j+1} = r/|r| (no host synchronisation inside the expansion; breakdowns are detected at the next sync)
    if (filtering) {
      TRY(L.filter_apply(L.col(j), cut));
      TRY(L.cgs2(j + 1, false));
    } else {
      {
        ProfScope ps(c, K_SPMV, c->csr_bytes() + 3 * c->vb() + 1.0 * c->n);
        ctx_spmv(c, c->vp, c->vt);
      }
      if (c->h > kHB) extra_gsums(c, c->vt, c->bs_t);
      TRY(L.cgs2(j + 1, true));
      L.applies++;
    }
    TRY(L.normalize_step(j));
    L.steps++;
    if (c->debug > 1) {
      cudaError_t e = cudaStreamSynchronize(c->st);
      fprintf(stderr, "[sfairsc] step j=%d done (%s)\n", j, cudaGetErrorString(e));
    }
    ++j;
    if (j < L.m) continue;

    // ---- sync: fetch T, handle a breakdown by rolling back to it ----
    int flag = 0;
    const int jfrom = jsync;  // T entries [jfrom, m) are new since the last sync
    TRY(L.fetch_T(jsync, L.m, &flag));
    if (c->debug)
      fprintf(stderr, "[sfairsc] sync restarts=%lld jsync=%d m=%d pk=%d flag=%d steps=%lld\n", (long long)L.restarts,
              jsync, L.m, L.pk, flag, (long long)L.steps);
    jsync = L.m;
    m_eff = L.m;
    if (flag) {
      int jb = -1;
      for (int i = jfrom; i < L.m; ++i)
        if (!(L.beta[i] > L.bd_tol)) {
          jb = i;
          break;
        }
      if (jb < 0) return fail(SFAIRSC_E_CUDA, "breakdown flag without a small beta");
      if (c->debug) fprintf(stderr, "[sfairsc] breakdown at j=%d beta=%g\n", jb, L.beta[jb]);
      L.breakdowns++;
      L.beta[jb] = 0.0;
      CU(cudaMemsetAsync(c->flags + 1, 0, sizeof(int), c->st));
      if (jb + 1 >= n) {
        complete = true;
        m_eff = jb + 1;
      } else {
        TRY(L.random_vector(jb + 1, false));
        j = jb + 1;
        jsync = j;
        if (j < L.m) continue;
        m_eff = L.m;
      }
    }

    // ---- Rayleigh-Ritz on T (m_eff x m_eff): arrowhead + tridiagonal ----
    const int me = m_eff;
    std::vector<double> T((size_t)me * me, 0.0);
    for (int i = 0; i < me; ++i) T[(size_t)i * me + i] = L.alpha[i];
    for (int i = 0; i < L.pk && L.pk < me; ++i) {
      T[(size_t)i * me + L.pk] = L.arrow[i];
      T[(size_t)L.pk * me + i] = L.arrow[i];
    }
    for (int i = L.pk; i + 1 < me; ++i) {
      T[(size_t)i * me + i + 1] = L.beta[i];
      T[(size_t)(i + 1) * me + i] = L.beta[i];
    }
    Y = T;
    symeig(me, Y, theta);
    const double bm = complete ? 0.0 : L.beta[me - 1];
    double maxres = 0.0;
    for (int i = 0; i < k; ++i) maxres = std::max(maxres, std::fabs(bm * Y[(size_t)(me - 1) * me + i]));
    if (k < me) gap = theta[k] - theta[k - 1];
    converged = complete || maxres <= target;
    if (filter && !filtering && !converged) {
      // end of the unfiltered cycle: a = the keep-th Ritz value (>= lambda_keep > lambda_k by interlacing),
      // restart the filtered solve from the sum of the k lowest Ritz vectors (tests/tools: proto_filter.py)
      const int q = std::min(L.keep, me) - 1;
      cut = std::min(theta[q], 0.5 * c->sigma);
      if (!(cut > theta[k - 1])) cut = 0.5 * (theta[k - 1] + c->sigma);
      filtering = true;
      std::vector<double> ys(me, 0.0);
      for (int cc = 0; cc < k; ++cc)
        for (int l = 0; l < me; ++l) ys[l] += Y[(size_t)l * me + cc];
      CU(cudaMemcpyAsync(c->Ydev, ys.data(), sizeof(double) * me, cudaMemcpyHostToDevice, c->st));
      launch_ritz(c->V, c->ldv, n, me, c->Ydev, 1, c->vr, c->st);
      CU(cudaStreamSynchronize(c->st));
      TRY(L.random_vector(0, false, true));
      L.pk = 0;
      j = 0;
      jsync = 0;
      L.restarts++;
      if (c->debug) fprintf(stderr, "[sfairsc] filter cut a=%.17g (theta_%d), degree %d\n", cut, q, c->filter_deg);
      continue;
    }
    if (filtering && !complete) {
      // the B-estimate is in units of B's spectrum (|p| <= 1 on [a, sigma]); below the threshold, decide on
      // the explicit L^sigma residuals of the Ritz vectors (k applies) and tighten the threshold if they miss
      if (fthr == 0.0) fthr = 1e-6 * std::max(1.0, std::fabs(theta[0]));
      converged = false;
      if (maxres <= fthr) {
        std::vector<double> Yc((size_t)me * k);
        for (int cc = 0; cc < k; ++cc)
          for (int l = 0; l < me; ++l) Yc[(size_t)cc * me + l] = Y[(size_t)l * me + cc];
        CU(cudaMemcpyAsync(c->Ydev, Yc.data(), sizeof(double) * Yc.size(), cudaMemcpyHostToDevice, c->st));
        {
          ProfScope ps(c, K_RITZ, (double)(me + k) * c->vb());
          launch_ritz(c->V, c->ldv, n, me, c->Ydev, k, c->X, c->st);
        }
        TRY(filter_check(c, k, &thA, &fres));
        L.applies += k;
        if (c->debug)
          fprintf(stderr, "[sfairsc] filter check: B-est %g (thr %g) L-resid %g target %g\n", maxres, fthr, fres,
                  tol_eff);
        if (fres <= tol_eff) converged = true;
        else fthr *= std::max(1e-3, std::min(0.1, 0.5 * tol_eff / fres));
      }
    }
    if (converged && filtering && !complete) break;  // X and thA from the check
    if (c->debug)
      fprintf(stderr, "[sfairsc] RR me=%d maxres=%g target=%g theta0=%.17g theta_k-1=%.17g\n", me, maxres, target,
              theta[0], theta[k - 1]);
    if (converged || L.restarts >= c->max_restarts) {
      // X = V[:, 0:me] Y[:, 0:k]
      std::vector<double> Yc((size_t)me * k);
      for (int cc = 0; cc < k; ++cc)
        for (int l = 0; l < me; ++l) Yc[(size_t)cc * me + l] = Y[(size_t)l * me + cc];
      CU(cudaMemcpyAsync(c->Ydev, Yc.data(), sizeof(double) * Yc.size(), cudaMemcpyHostToDevice, c->st));
      {
        ProfScope ps(c, K_RITZ, (double)(me + k) * c->vb());
        launch_ritz(c->V, c->ldv, n, me, c->Ydev, k, c->X, c->st);
      }
      CHECK_LAUNCH();
      break;
    }
    // ---- thick restart: keep the `keep` smallest Ritz pairs ----
    const int pk = std::min(L.keep, me - 1);
    std::vector<double> Yc((size_t)me * pk);
    for (int cc = 0; cc < pk; ++cc)
      for (int l = 0; l < me; ++l) Yc[(size_t)cc * me + l] = Y[(size_t)l * me + cc];
    CU(cudaMemcpyAsync(c->Ydev, Yc.data(), sizeof(double) * Yc.size(), cudaMemcpyHostToDevice, c->st));
    {
      ProfScope ps(c, K_RITZ, (double)(me + pk) * c->vb());
      launch_ritz(c->V, c->ldv, n, me, c->Ydev, pk, c->Vb, c->st);
    }
    CU(cudaMemcpyAsync(c->Vb + (long long)pk * c->ldv, c->V + (long long)me * c->ldv, sizeof(double) * c->ldv,
                       cudaMemcpyDeviceToDevice, c->st));
    CHECK_LAUNCH();
    std::swap(c->V, c->Vb);
    for (int i = 0; i < pk; ++i) {
      L.alpha[i] = theta[i];
      L.arrow[i] = bm * Y[(size_t)(me - 1) * me + i];
    }
    L.pk = pk;
    j = pk;
    jsync = pk;
    L.restarts++;
  }

  // ---- A11: true residuals with k fresh applies (filtered: the check's Rayleigh quotients and residuals) ----
  double max_resid = 0.0;
  if (filtering) {
    if (!converged || complete) {  // X from the final Ritz vectors: their Rayleigh quotients and residuals
      TRY(filter_check(c, k, &thA, &fres));
      L.applies += k;
    }
    // gap estimate: lambda of the (k+1)-th B Ritz value through p^{-1} where it lies below a (p >= 1)
    gap = std::numeric_limits<double>::quiet_NaN();
    if ((int)theta.size() > k && -theta[k] >= 1.0) {
      const double pc = 0.5 * (cut + c->sigma), pe = 0.5 * (c->sigma - cut);
      const double lam1 = pc - pe * std::cosh(std::acosh(-theta[k]) / c->filter_deg);
      gap = lam1 - thA[k - 1];
    }
    theta = thA;
    max_resid = fres;
  } else {
    TRY(true_residuals(c, theta.data(), k, &max_resid));
    L.applies += k;
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
  S.basis_size = L.m;
  S.kept = L.keep;
  S.filter_cut = filtering ? cut : 0.0;
  c->last = S;
  if (stats) *stats = S;
  if (!converged) return fail(SFAIRSC_E_NO_CONVERGENCE, "no convergence after %lld restarts", (long long)L.restarts);
  if (theta[k - 1] >= c->sigma * (1.0 - 1e-8))
    return fail(SFAIRSC_E_SHIFT_TOO_SMALL, "lambda_k=%g >= sigma(1-1e-8)=%g (Prop. 3.4)", theta[k - 1], c->sigma);
  return SFAIRSC_OK;
}

extern "C" sfairsc_status sfairsc_embed_kmeans(sfairsc_ctx* c, uint64_t seed, int32_t* labels_out, int32_t memspace,
                                               double* objective_out) {
  NvtxRange nv("sfairsc.kmeans");
  if (!c || !labels_out) return fail(SFAIRSC_E_INVALID_ARG, "null argument");
  if (!c->have_eigs) return fail(SFAIRSC_E_STATE, "sfairsc_eigs must succeed before sfairsc_embed_kmeans");
  if (memspace != SFAIRSC_MEM_HOST && memspace != SFAIRSC_MEM_DEVICE) return fail(SFAIRSC_E_INVALID_ARG, "memspace");
  if (c->dist) return dist_kmeans(c, seed, labels_out, memspace, objective_out);
  return kmeans_run(c, seed, labels_out, memspace, objective_out);
}

extern "C" int64_t sfairsc_launch_count(void) { return (int64_t)launch_count(); }

extern "C" int64_t sfairsc_struct_size(int32_t which) {
  switch (which) {
    case 0: return (int64_t)sizeof(sfairsc_csr);
    case 1: return (int64_t)sizeof(sfairsc_opts);
    case 2: return (int64_t)sizeof(sfairsc_stats);
    case 3: return (int64_t)sizeof(sfairsc_info);
    default: return -1;
  }
}

// host utility exported for tests of the Rayleigh-Ritz step
extern "C" int sfairsc_host_symeig(int32_t m, const double* A, double* evals, double* evecs) {
  if (m < 0 || (m > 0 && (!A || !evals))) return 1;
  std::vector<double> M(A, A + (size_t)m * m), ev;
  symeig(m, M, ev);
  for (int i = 0; i < m; ++i) evals[i] = ev[i];
  if (evecs)
    for (size_t i = 0; i < (size_t)m * m; ++i) evecs[i] = M[i];
  return 0;
}
extern "C" int sfairsc_host_symeig_sel(int32_t m, const double* A, double* evals, double* evecs, int32_t nvec) {
  if (m < 0 || nvec < 0 || nvec > m || (m > 0 && (!A || !evals))) return 1;
  std::vector<double> M(A, A + (size_t)m * m), ev;
  symeig(m, M, ev, nvec);
  for (int i = 0; i < m; ++i) evals[i] = ev[i];
  if (evecs)
    for (int l = 0; l < m; ++l)
      for (int c = 0; c < nvec; ++c) evecs[(size_t)l * m + c] = M[(size_t)l * m + c];
  return 0;
}
