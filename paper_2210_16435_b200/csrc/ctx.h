// Internal: the context behind the opaque sfairsc_ctx handle, shared by the
// library's host translation units (abi.cu, lanczos_block.cu).  Not part of the C ABI.
#pragma once
#include "sfairsc.h"
#include "kernels.cuh"

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <string>
#include <vector>

namespace sfz {
struct DistCtx;  // row-partitioned state (dist.cu)
}
using sfz::GraphDev;
using sfz::ProjDesc;
using sfz::kHB;

// --------------------------------------------------------------------------
// per-kernel event timing (sfairsc_profile_*)
// --------------------------------------------------------------------------
struct Prof {
  bool on = false;
  struct Pending {
    int kind;
    cudaEvent_t a, b;
    double bytes;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> pool;
  double total_ms[10] = {};
  int64_t launches[10] = {};
  double bytes[10] = {};
  cudaEvent_t get() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  void resolve() {
    for (auto& p : pending) {
      cudaEventSynchronize(p.b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, p.a, p.b);
      total_ms[p.kind] += ms;
      launches[p.kind] += 1;
      bytes[p.kind] += p.bytes;
      pool.push_back(p.a);
      pool.push_back(p.b);
    }
    pending.clear();
  }
  ~Prof() {
    for (auto& p : pending) {
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

enum { K_SPMV = 0, K_DOTS = 1, K_UPDDOT = 2, K_UPDNORM = 3, K_NORMALIZE = 4, K_RITZ = 5, K_PROJ = 6, K_FINISH = 7,
       K_KMEANS = 8, K_OTHER = 9 };

struct sfairsc_ctx {
  int device = 0, num_sms = 148;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  int n = 0, nnz = 0, h = 1, k_build = 1;
  bool normalized = false;
  long long ldv = 0;
  int vs = 8, spmv_grid = 1, sgrid = 1;
  double sigma = 0.0, tol_cap = 1e-10;
  uint64_t seed = 0x5F41C5EEDull;
  int m = 20, keep = 0, max_restarts = 100000;
  int check_symmetry = 1;
  int debug = 0;
  // device buffers
  int *rp = nullptr, *ci = nullptr, *row_split = nullptr;
  int2* tiles = nullptr;       // TMA SpMV tiles (spmv_tma.cu): (first row, first entry), ntiles + 1
  int* cta_tiles = nullptr;    // tile range per CTA, tma_grid + 1
  int tma_grid = 0;
  int *prp = nullptr, *pci = nullptr;  // padded CSR of the TMA SpMV (rows at multiples of 4 entries, pads col = -1)
  double* pvv = nullptr;               // its values, split block layout (nullptr: unit-weight pattern SpMV)
  int nnz_pad = 0;                     // padded entries (a multiple of 4)
  bool spmv_tma = false;               // the single-vector SpMV is the TMA-fed tile kernel
  sfz::SpmvTileShape spmv_shape;       // its tile shape and ring depth
  double *vv = nullptr, *dg = nullptr, *s = nullptr;
  uint8_t* grp = nullptr;
  double *isb = nullptr, *uh = nullptr;
  double* partials = nullptr;
  size_t partials_cnt = 0;
  unsigned* counters = nullptr;
  double *bs_w = nullptr, *bs_t = nullptr, *bs_v = nullptr, *nb = nullptr, *scal = nullptr;
  double *c1 = nullptr, *c2 = nullptr;
  double *vp = nullptr, *vt = nullptr, *vr = nullptr, *vy = nullptr;
  double *V = nullptr, *Vb = nullptr, *Ydev = nullptr, *X = nullptr;
  double *talpha = nullptr, *tbeta = nullptr;  // Lanczos T entries recorded on device
  int* flags = nullptr;
  double* hp = nullptr;  // pinned host staging (4 KB)
  // block Lanczos (lanczos_block.cu); bsz = 1: the single-vector path above
  int bsz = 1;
  double *bP = nullptr, *bT = nullptr, *bR = nullptr;  // interleaved ldv x bsz blocks
  double *Tdev = nullptr, *g2 = nullptr;                // projected matrix (ldT = m + bsz), CholQR Gram
  int ldT = 0;
  int* bflags = nullptr;                                // per-step breakdown flags
  // single-sweep (lagged) Lanczos (lanczos1.cu); uses ldT = m + 2 for H
  bool lagged = false;
  bool paired = false;     // lagged solver with two Lanczos steps per basis sweep (reorth 3, default where allowed)
  double* vrB = nullptr;   // paired steps: the second lagged vector of a pair
  double* lzp = nullptr;   // paired steps: epend | econv | cA | tr | pair dots (8 kMaxJ doubles)
  // Chebyshev-filtered Lanczos (§8(f) N2): degree (>= 2: on), cut a (<= 0: automatic),
  // two recurrence vectors, the Rayleigh quotients of the explicit check
  int filter_deg = 0;
  double filter_cut = 0.0;
  double* fbuf = nullptr;  // 2 ldv
  double* fth = nullptr;   // kMaxJ
  double *Hdev = nullptr, *sdev = nullptr, *lz = nullptr, *partials2 = nullptr, *dd = nullptr;
  // column-blocked CSR (the gathered vector exceeds L2, e.g. config 5): block-major copy of the CSR,
  // rpb[b*(n+1) + i] = start of row i in column block b; nblk = 1: plain CSR
  int nblk = 1, vs_blk = 2;
  bool skewed = false;  // max degree > 16 x mean degree (config 5's Pareto degrees)
  bool unit = false;    // unit-weight pattern: ctx_spmv streams column indices only (GraphDev::unit)
  double* vq = nullptr; // normalized unit-weight SpMV: gathered q = s o p
  double* vq_lz = nullptr; // the same for the lagged solver's p~, written by its normalisation kernel
  int* rpb = nullptr;
  double *pairP = nullptr, *pairT = nullptr, *pairY = nullptr;  // pair apply (lazily allocated)
  // dense constraint basis (§8(f) N4, sfairsc_build_operator_dense): Q n x qr row-major (ldq); nullptr: groups
  double* Qr = nullptr;
  int qr = 0, ldq = 0;
  int rank_in = 0;  // dense F: its column count (qr = the numerical rank of C)
  // row-partitioned contexts: all device state lives in dist
  sfz::DistCtx* dist = nullptr;
  // results
  bool have_eigs = false;
  int k_eigs = 0;
  std::vector<double> evals;
  std::vector<int32_t> groups_host;
  std::vector<int64_t> group_count;
  sfairsc_stats last{};
  double t_build = 0.0;
  Prof prof;
  // kmeans scratch (allocated lazily by kmeans.cu)
  void* km = nullptr;
  void (*km_free)(void*) = nullptr;

  GraphDev g() const {
    GraphDev G;
    G.n = n;
    G.nnz = nnz;
    G.rp = rp;
    G.ci = ci;
    G.vv = vv;
    G.dg = dg;
    G.s = s;
    G.grp = grp;
    G.normalized = normalized;
    G.Q = Qr;
    G.ldq = ldq;
    G.qr = qr;
    G.skewed = skewed;
    return G;
  }
  // the graph as ctx_spmv sees it (single-vector SpMV: the unit-weight kernels when the pattern allows)
  GraphDev gs() const {
    GraphDev G = g();
    G.unit = unit_spmv();
    return G;
  }
  // the dense-projector SpMV keeps its value-streaming kernel; normalized graphs take the pattern-only kernel
  // when column-blocked or TMA-fed (the LSU-fed round-1 kernel was gather-bound either way: config 4 720 vs 722 us)
  bool unit_spmv() const { return unit && !Qr && (!normalized || nblk > 1 || spmv_tma); }
  ProjDesc pd() const {
    ProjDesc P{Qr ? qr : h, isb, uh};
    P.Q = Qr;
    P.ldq = ldq;
    return P;
  }
  // algorithmic bytes: one read/write of each operand
  double vb() const { return 8.0 * n; }                      // one fp64 n-vector
  double sgb() const { return (normalized ? 8.0 * n : 0.0) + 1.0 * n; }  // s (normalized) + group ids
  // the CSR stream counts 12 B per entry even when the pattern-only SpMV leaves implied unit
  // values unread (the pattern-only kernel is a labelled variant, not a smaller workload)
  double csr_bytes() const { return 12.0 * nnz + 4.0 * (n + 1); }
  int gpasses() const { return (h + kHB - 1) / kHB; }
};


namespace sfz {
sfairsc_status fail(sfairsc_status st, const char* fmt, ...);
sfairsc_status apply_dev(sfairsc_ctx* c, const double* x, double* y);  // y = L^sigma x (device vectors)
sfairsc_status true_residuals(sfairsc_ctx* c, const double* theta, int k, double* max_out);  // over X
// t = L p (+ B^T t, p^T t into bs_t) through the plain or the column-blocked CSR
// t = L p (+ epilogue B^T t, p^T t); q_pre: s o p already formed (normalized unit-weight graphs), else nullptr
void ctx_spmv(sfairsc_ctx* c, const double* p, double* t, const double* q_pre = nullptr);
sfairsc_status apply_pair_dev(sfairsc_ctx* c, const double* x0, const double* x1, double* y0, double* y1);
double now_s();
}

// profiling scope: one event pair around a launch group (sfairsc_profile_*)
// NVTX range per library phase (SURVEY §5 tracing): sfairsc.build, sfairsc.eigs, sfairsc.restart_sync,
// sfairsc.rayleigh_ritz (host), sfairsc.true_residuals, sfairsc.kmeans, sfairsc.apply.  NVTX3 is header-only: the
// calls are no-ops unless a tool (Nsight Systems / Compute with --nvtx) injects itself.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct ProfScope {
  sfairsc_ctx* c;
  int kind;
  double bytes;
  cudaEvent_t a = nullptr;
  ProfScope(sfairsc_ctx* c_, int kind_, double bytes_ = 0.0) : c(c_), kind(kind_), bytes(bytes_) {
    if (c->prof.on) {
      a = c->prof.get();
      cudaEventRecord(a, c->st);
    }
  }
  ~ProfScope() {
    if (c->prof.on) {
      cudaEvent_t b = c->prof.get();
      cudaEventRecord(b, c->st);
      c->prof.pending.push_back({kind, a, b, bytes});
    }
  }
};

#define CU(expr)                                                                                        \
  do {                                                                                                  \
    cudaError_t e_ = (expr);                                                                            \
    if (e_ != cudaSuccess)                                                                              \
      return sfz::fail(e_ == cudaErrorMemoryAllocation ? SFAIRSC_E_OOM : SFAIRSC_E_CUDA, "%s: %s (%s:%d)", \
                       #expr, cudaGetErrorString(e_), __FILE__, __LINE__);                               \
  } while (0)

#define CHECK_LAUNCH() CU(cudaGetLastError())
#define TRY(expr)                              \
  do {                                         \
    sfairsc_status s_ = (expr);                \
    if (s_ != SFAIRSC_OK) return s_;           \
  } while (0)
