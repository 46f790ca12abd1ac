// libsfairsc — row-partitioned s-FairSC across GPUs.
//
// W and every n-vector are split into contiguous row blocks (cuts chosen by
// the caller; bench.py and lib.partition_rows use nnz-balanced cuts).  Part q
// holds rows [cut_q, cut_{q+1}): its CSR rows with column indices remapped to
// the padded gathered layout  col -> owner(col) * n_max + (col - cut_owner),
// its slice of d, s, group ids, of the Krylov basis and of X.  Per Lanczos
// step of the single-sweep method (lanczos1.cu) the exchanges are
//   * all-gather of the projected vector p~ (n_max doubles per part; NCCL
//     ncclAllGather in place) before the SpMV  (the x / halo exchange),
//   * all-reduce (sum) of [B^T t, p~^T t] (17 doubles) after the SpMV,
//   * all-reduce (sum) of [V^T w (J+1), |w|^2, B^T w (16)] after the sweep,
// and the small replicated state (projected matrix H, coefficients) is
// computed identically on every part, so thick restarts need no broadcast.
//
// Two transports implement the collectives: NCCL (one part per process and
// GPU, ranks joined by sfairsc_comm_init; NCCL is dlopen'ed so the library
// has no link-time NCCL dependency), and "virtual parts" (P parts in one
// process on one GPU; the gathered vector is shared and reductions are a
// fixed-order device sum) which tests the partitioned arithmetic on a single
// GPU.  Fixed partitions + fixed reduction order: bitwise reproducible for a
// fixed number of parts; results for different part counts agree to rounding.
#include "ctx.h"
#include "device_common.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <vector>

// ---------------------------------------------------------------------------
// NCCL via dlopen
// ---------------------------------------------------------------------------
namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) =
      nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
      api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
      api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
      api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
      api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.AllGather &&
               api.GetErrorString;
    }
  }
  return api;
}
}  // namespace

struct sfairsc_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1, device = 0;
};

#define NC(expr)                                                                                   \
  do {                                                                                             \
    ncclResult_t r_ = (expr);                                                                      \
    if (r_ != ncclSuccess) return sfz::fail(SFAIRSC_E_NCCL, "%s: %s", #expr, nccl().GetErrorString(r_)); \
  } while (0)

extern "C" sfairsc_status sfairsc_comm_unique_id(uint8_t id_out[128]) {
  if (!id_out) return sfz::fail(SFAIRSC_E_INVALID_ARG, "null id");
  if (!nccl().ok) return sfz::fail(SFAIRSC_E_NCCL, "libnccl.so.2 not loadable");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  NC(nccl().GetUniqueId(&id));
  std::memcpy(id_out, &id, 128);
  return SFAIRSC_OK;
}

extern "C" sfairsc_status sfairsc_comm_init(const uint8_t id[128], int32_t rank, int32_t nranks, int32_t device,
                                            sfairsc_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return sfz::fail(SFAIRSC_E_INVALID_ARG, "bad argument");
  if (!nccl().ok) return sfz::fail(SFAIRSC_E_NCCL, "libnccl.so.2 not loadable");
  *out = nullptr;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return sfz::fail(SFAIRSC_E_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  sfairsc_comm* c = new sfairsc_comm();
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return sfz::fail(SFAIRSC_E_NCCL, "ncclCommInitRank: %s", nccl().GetErrorString(r));
  }
  *out = c;
  return SFAIRSC_OK;
}

extern "C" void sfairsc_comm_destroy(sfairsc_comm* c) {
  if (!c) return;
  if (c->comm && nccl().ok) nccl().CommDestroy(c->comm);
  delete c;
}

namespace sfz {

void symeig(int m, std::vector<double>& A, std::vector<double>& evals);
void symeig(int m, std::vector<double>& A, std::vector<double>& evals, int nvec);
void bump_launch();
sfairsc_status kmeans_run(sfairsc_ctx* ctx, uint64_t seed, int32_t* labels_out, int32_t memspace, double* objective);


// ---------------------------------------------------------------------------
// kernels specific to the partitioned layout
// ---------------------------------------------------------------------------
namespace {
constexpr int kDT = 256;

// col -> owner * n_max + (col - cut_owner); flags: out of range / diagonal / unsorted / negative
// symmetry fingerprint of an entry (i, j, w): W = W^T  <=>  the multiset {(i, j, w)} equals {(j, i, w)},
// so sum_e [h(i, j, w) - h(j, i, w)] = 0 (mod 2^64) over all entries of all parts; an asymmetric W leaves
// a nonzero sum except with probability ~2^-64 (h asymmetric in (i, j), splitmix64 finaliser)
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ unsigned long long sym_hash(long long i, long long j, double w) {
  return mix64(mix64((unsigned long long)i) ^ ((unsigned long long)j * 0xD6E8FEB86659FD93ull)) ^
         mix64((unsigned long long)__double_as_longlong(w));
}

__global__ void k_remap_validate(const int* rp, int* ci, const double* vv, int n_loc, long long r0, long long n,
                                 const long long* cuts, int nparts, int n_max, int* flags,
                                 unsigned long long* symsum) {
  int f = 0, nonunit = 0;
  unsigned long long hs = 0ull;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_loc; i += gridDim.x * blockDim.x) {
    const int a = rp[i], b = rp[i + 1];
    if (b < a) {
      f |= 1;
      continue;
    }
    long long prev = -1;
    for (int e = a; e < b; ++e) {
      const long long j = ci[e];
      if (j < 0 || j >= n || j <= prev) f |= 1;
      if (j == r0 + i && vv[e] != 0.0) f |= 1;
      if (!(vv[e] >= 0.0)) f |= 2;
      if (vv[e] != 1.0 || j == r0 + i) nonunit = 1;
      if (j >= 0 && j < n) hs += sym_hash(r0 + i, j, vv[e]) - sym_hash(j, r0 + i, vv[e]);
      prev = j;
      int lo = 0, hi = nparts - 1;  // owner: cuts[o] <= j < cuts[o+1]
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (cuts[mid] <= j) lo = mid; else hi = mid - 1;
      }
      ci[e] = lo * n_max + (int)(j - cuts[lo]);
    }
  }
  if (f) atomicOr(flags, f);
  if (nonunit) atomicOr(flags + 1, 1);  // local, informational: this part's rows are not a unit-weight pattern
  if (hs) atomicAdd(symsum, hs);        // integer: order-independent
}

__global__ void k_degrees_d(const int* rp, const double* vv, int n_loc, double* d, int* flags) {
  int f = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_loc; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int e = rp[i]; e < rp[i + 1]; ++e) acc += vv[e];
    d[i] = acc;
    if (!(acc > 0.0)) f |= 8;
  }
  if (f) atomicOr(flags, f);
}

// s = d^{-1/2} into this part's segment of the gathered s (and the local copy)
__global__ void k_inv_sqrt_d(const double* d, int n_loc, double* s_loc, double* s_seg) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_loc; i += gridDim.x * blockDim.x) {
    const double v = 1.0 / sqrt(d[i]);
    s_loc[i] = v;
    s_seg[i] = v;
  }
}

// w_ij <- s_i w_ij s_j with s_j read from the gathered s (columns already remapped)
__global__ void k_scale_d(const int* rp, const int* ci, double* vv, const double* s_loc, const double* s_full,
                          int n_loc) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_loc; i += gridDim.x * blockDim.x) {
    const double si = s_loc[i];
    for (int e = rp[i]; e < rp[i + 1]; ++e) vv[e] = si * vv[e] * s_full[ci[e]];
  }
}

// local max of the column sums of |L| (sigma = ||L||_1): normalized 1 + sum_j w^_ij, unnormalized 2 d_i
__global__ void k_sigma_d(const int* rp, const double* vv, const double* d, int n_loc, bool normalized,
                          double* partials, unsigned* counter, double* out) {
  double mx = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_loc; i += gridDim.x * blockDim.x) {
    double v;
    if (normalized) {
      double acc = 0.0;
      for (int e = rp[i]; e < rp[i + 1]; ++e) acc += vv[e];
      v = 1.0 + acc;
    } else {
      v = 2.0 * d[i];
    }
    mx = fmax(mx, v);
  }
  __shared__ double red[kDT];
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int s = kDT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    double m = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) m = fmax(m, __ldcg(partials + b));
    *out = m;
    *counter = 0u;
  }
}

// virtual transport: out = fixed-order sum (or max) over the parts' buffers, written back to every part
__global__ void k_vreduce(double* const* bufs, int nparts, int count, int op_max) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < count; q += gridDim.x * blockDim.x) {
    double acc = bufs[0][q];
    for (int p = 1; p < nparts; ++p) acc = op_max ? fmax(acc, bufs[p][q]) : acc + bufs[p][q];
    for (int p = 0; p < nparts; ++p) bufs[p][q] = acc;
  }
}

// x_i = u - 1/2, u = Philox(key = seed, ctr = (global row, c1, stream, 0)): independent of the partition
__global__ void k_random_off(double* x, int n_loc, long long r0, uint64_t seed, unsigned c1, unsigned stream) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_loc; i += gridDim.x * blockDim.x)
    x[i] = philox_uniform(seed, (unsigned)(r0 + i), c1, stream, 0u) - 0.5;
}

int grid_for(int n) { return std::max(1, std::min((n + kDT - 1) / kDT, 148 * 8)); }
}  // namespace

// ---------------------------------------------------------------------------
// the partitioned context
// ---------------------------------------------------------------------------
struct DistPart {
  int q = 0;
  int n_loc = 0, nnz_loc = 0;
  long long r0 = 0, ldv = 0;
  int *rp = nullptr, *ci = nullptr, *row_split = nullptr;
  double *vv = nullptr, *dg = nullptr, *s = nullptr;
  uint8_t* grp = nullptr;
  double *isb = nullptr, *uh = nullptr;
  int spmv_grid = 1, vs = 8;
  // owner-segment column blocks (P_total > 1): block b = the columns owned by part b (n_max entries of the
  // gathered vector, L2-sized); rpb[b*(n_loc+1) + i] = start of row i in block b of the block-major CSR
  int nblk = 1, vs_blk = 2;
  int* rpb = nullptr;
  bool skewed = false;  // heavy-tailed local degrees: long rows get a whole warp in the SpMV
  bool unit = false;    // unnormalized unit-weight rows: the pattern-only SpMV (GraphDev::unit)
  double *vr = nullptr, *vy = nullptr, *vt = nullptr;  // v~ (lagged), w, t
  double* vrB = nullptr;  // paired steps: the pair's second lagged vector
  double *V = nullptr, *Vb = nullptr, *X = nullptr;
  double *partials = nullptr, *partials2 = nullptr;
  unsigned* counters = nullptr;
  double* small = nullptr;  // bs_t [0,64), bs_v [64,128), bs_w [128,192), nb [192,256), scal [256,320), dd [512, 1024),
                            // pair dots dd2 [1024, 2048)
  int* flags = nullptr;
  GraphDev g(bool normalized) const {
    GraphDev G;
    G.n = n_loc;
    G.nnz = nnz_loc;
    G.rp = rp;
    G.ci = ci;
    G.vv = vv;
    G.dg = dg;
    G.s = s;
    G.grp = grp;
    G.normalized = normalized;
    G.skewed = skewed;
    G.unit = unit && !normalized;
    return G;
  }
  double* bs_t() const { return small; }
  double* bs_v() const { return small + 64; }
  double* bs_w() const { return small + 128; }
  double* nb() const { return small + 192; }
  double* scal() const { return small + 256; }
  double* dd() const { return small + 512; }
  double* dd2() const { return small + 1024; }
};

struct DistCtx {
  sfairsc_comm* comm = nullptr;  // NCCL transport (one part) or nullptr (virtual parts)
  int P = 1;                      // parts held by this process
  int P_total = 1, part0 = 0;     // all parts, index of this process's first part
  long long n = 0;
  int n_max = 0;
  std::vector<long long> cuts;    // P_total + 1
  long long* cuts_dev = nullptr;
  double* p_full = nullptr;       // gathered projected vector, P_total * n_max
  double* s_full = nullptr;       // gathered s (normalized), P_total * n_max
  std::vector<DistPart> parts;
  double** ptr_tab = nullptr;     // device table of per-part buffer pointers (virtual reductions)
  cudaStream_t cst = nullptr;     // NCCL stream: the all-gather overlaps the own-block SpMV
  cudaEvent_t ev_ready = nullptr, ev_gathered = nullptr;
  // replicated Lanczos state (one copy per process)
  double *H = nullptr, *sv = nullptr, *lz = nullptr, *cs = nullptr, *cg = nullptr, *Ydev = nullptr;
  double* lzp = nullptr;  // paired steps: epend | econv | cA | tr (4 kMaxJ)
  int ldH = 0;
  int* bflags = nullptr;
  double* hp = nullptr;
  // the shadow single-GPU context used by k-means on the gathered H
  sfairsc_ctx* km = nullptr;
  double* X_full = nullptr;
  double* s_compact = nullptr;
};

// ---------------------------------------------------------------------------
// collectives
// ---------------------------------------------------------------------------
static sfairsc_status allreduce(DistCtx* D, cudaStream_t st, int count, double* (*sel)(const DistPart&), bool op_max = false) {
  if (D->comm) {
    double* b = sel(D->parts[0]);
    NC(nccl().AllReduce(b, b, count, ncclDouble, op_max ? ncclMax : ncclSum, D->comm->comm, st));
    return SFAIRSC_OK;
  }
  if (D->P == 1) return SFAIRSC_OK;
  std::vector<double*> ptrs(D->P);
  for (int q = 0; q < D->P; ++q) ptrs[q] = sel(D->parts[q]);
  CU(cudaMemcpyAsync(D->ptr_tab, ptrs.data(), sizeof(double*) * D->P, cudaMemcpyHostToDevice, st));
  bump_launch();
  k_vreduce<<<std::max(1, std::min((count + 255) / 256, 64)), 256, 0, st>>>(D->ptr_tab, D->P, count, op_max ? 1 : 0);
  CU(cudaGetLastError());
  // the pointer table is re-written by the next call: keep the copy ordered before it
  return SFAIRSC_OK;
}
static sfairsc_status allgather_full(DistCtx* D, cudaStream_t st, double* full) {
  if (D->comm)  // (one rank: an in-place no-op, still issued so the 1-rank tests run the NCCL path)
    NC(nccl().AllGather(full + (size_t)D->comm->rank * D->n_max, full, D->n_max, ncclDouble, D->comm->comm, st));
  return SFAIRSC_OK;  // virtual parts share `full`
}

// t = L p~ for every part with the halo exchange: the own column block first, overlapped with the NCCL
// all-gather of the other parts' segments on the communication stream, then the remote blocks (cmode:
// 1 first, 2 middle, 3 last incl. the B^T t / p^T t epilogue).  Without blocking (one part): the plain SpMV.
static sfairsc_status dist_spmv(DistCtx* D, sfairsc_ctx* c, cudaStream_t st) {
  const bool nccl_multi = D->comm != nullptr;
  if (nccl_multi) {  // p~ segment written on st; start the all-gather on cst
    CU(cudaEventRecord(D->ev_ready, st));
    CU(cudaStreamWaitEvent(D->cst, D->ev_ready, 0));
    NC(nccl().AllGather(D->p_full + (size_t)D->comm->rank * D->n_max, D->p_full, D->n_max, ncclDouble,
                        D->comm->comm, D->cst));
    CU(cudaEventRecord(D->ev_gathered, D->cst));
  }
  for (auto& p : D->parts) {
    const double* pself = D->p_full + (size_t)p.q * D->n_max;
    if (p.nblk <= 1) {
      if (nccl_multi) CU(cudaStreamWaitEvent(st, D->ev_gathered, 0));
      launch_spmm(p.g(c->normalized), 1, p.vs, p.row_split, p.spmv_grid, D->p_full, p.vt, p.partials,
                  p.counters + 1, p.bs_t(), st, pself);
      continue;
    }
    for (int idx = 0; idx < p.nblk; ++idx) {
      const int b = idx == 0 ? p.q : (idx <= p.q ? idx - 1 : idx);  // own block, then the others in order
      if (idx == 1 && nccl_multi) CU(cudaStreamWaitEvent(st, D->ev_gathered, 0));
      GraphDev g = p.g(c->normalized);
      g.rp = p.rpb + (size_t)b * (p.n_loc + 1);
      const int cmode = idx == 0 ? 1 : (idx + 1 < p.nblk ? 2 : 3);
      launch_spmv_colblock(g, p.vs_blk, p.row_split, p.spmv_grid, D->p_full, p.vt, p.partials, p.counters + 1,
                           p.bs_t(), cmode, st, pself);
    }
  }
  CU(cudaGetLastError());
  return SFAIRSC_OK;
}

void dist_free(DistCtx* D) {
  if (!D) return;
  for (auto& p : D->parts) {
    void* ptrs[] = {p.rp, p.ci, p.row_split, p.vv, p.dg, p.s, p.grp, p.isb, p.uh, p.vr, p.vy, p.vt, p.V, p.Vb, p.X,
                    p.partials, p.partials2, p.counters, p.small, p.flags, p.rpb, p.vrB};
    for (void* x : ptrs)
      if (x) cudaFree(x);
  }
  void* ptrs[] = {D->cuts_dev, D->p_full, D->s_full, D->ptr_tab, D->H, D->sv, D->lz, D->cs, D->cg, D->Ydev,
                  D->bflags, D->X_full, D->s_compact, D->lzp};
  for (void* x : ptrs)
    if (x) cudaFree(x);
  if (D->hp) cudaFreeHost(D->hp);
  if (D->cst) cudaStreamDestroy(D->cst);
  if (D->ev_ready) cudaEventDestroy(D->ev_ready);
  if (D->ev_gathered) cudaEventDestroy(D->ev_gathered);
  if (D->km) {
    // shadow context: owns nothing but its k-means scratch
    D->km->X = nullptr;
    D->km->s = nullptr;
    D->km->st = nullptr;
    D->km->own_stream = false;
    sfairsc_destroy(D->km);
  }
  delete D;
}

template <typename T>
static cudaError_t dal(T** p, size_t count) {
  return cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T));
}

// ---------------------------------------------------------------------------
// build-time agreement (advisor r1): every rank of a row-partitioned build takes part in exactly one
// max-all-reduce of its local validation status before any other collective, so a rank whose own checks
// fail (group ids, row block, CSR sizes) makes every rank return instead of leaving the others blocked in
// the first all-gather.  Ranks that pass their checks call it at the start of dist_build; a rank that
// fails calls it from sfairsc_build_operator_ex before returning.
// ---------------------------------------------------------------------------
sfairsc_status dist_agree(sfairsc_comm* comm, int local_status, cudaStream_t st) {
  if (!comm || !comm->comm || !nccl().ok) return SFAIRSC_OK;
  double* b = nullptr;
  if (cudaMalloc((void**)&b, sizeof(double)) != cudaSuccess) return fail(SFAIRSC_E_OOM, "agreement buffer");
  double v = (double)local_status, r = 0.0;
  cudaMemcpy(b, &v, sizeof(double), cudaMemcpyHostToDevice);
  const ncclResult_t nr = nccl().AllReduce(b, b, 1, ncclDouble, ncclMax, comm->comm, st);
  cudaError_t e = cudaMemcpyAsync(&r, b, sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(b);
  if (nr != ncclSuccess) return fail(SFAIRSC_E_NCCL, "build agreement: %s", nccl().GetErrorString(nr));
  if (e != cudaSuccess) return fail(SFAIRSC_E_CUDA, "build agreement: %s", cudaGetErrorString(e));
  return (sfairsc_status)(int)r;
}

// ---------------------------------------------------------------------------
// build (A0-A3, partitioned)
// ---------------------------------------------------------------------------
sfairsc_status dist_build(sfairsc_ctx* c, const sfairsc_csr* W, const int32_t* groups, int hh,
                          const std::vector<int64_t>& cnt_local, const sfairsc_opts& opts) {
  DistCtx* D = new DistCtx();
  c->dist = D;
  D->comm = opts.comm;
  const bool dev_in = W->memspace == SFAIRSC_MEM_DEVICE;
  const cudaMemcpyKind kind = dev_in ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  cudaStream_t st = c->st;
  D->n = W->n_cols;
  // ---- cuts ----
  std::vector<int32_t> hrp(W->n_rows + 1);
  CU(cudaMemcpy(hrp.data(), W->row_ptr, sizeof(int32_t) * (W->n_rows + 1),
                dev_in ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
  if (D->comm) {
    // local checks passed on this rank: agree with the others (a failed rank joins from the ABI)
    const sfairsc_status ag = dist_agree(D->comm, SFAIRSC_OK, st);
    if (ag != SFAIRSC_OK)
      return ag == SFAIRSC_E_NCCL || ag == SFAIRSC_E_CUDA || ag == SFAIRSC_E_OOM
                 ? ag : fail(ag, "another rank's build failed its input checks (status %d)", (int)ag);
    D->P = 1;
    D->P_total = D->comm->nranks;
    D->part0 = D->comm->rank;
    // every rank publishes (row_offset, n_rows); the row blocks must tile [0, n) in rank order
    double* tmp = nullptr;
    CU(dal(&tmp, 2 * D->P_total));
    std::vector<double> mine = {(double)W->row_offset, (double)W->n_rows};
    CU(cudaMemcpy(tmp + 2 * D->part0, mine.data(), 2 * sizeof(double), cudaMemcpyHostToDevice));
    NC(nccl().AllGather(tmp + 2 * D->part0, tmp, 2, ncclDouble, D->comm->comm, st));
    std::vector<double> all(2 * D->P_total);
    CU(cudaMemcpyAsync(all.data(), tmp, sizeof(double) * 2 * D->P_total, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    cudaFree(tmp);
    D->cuts.assign(D->P_total + 1, 0);
    for (int r = 0; r < D->P_total; ++r) {
      if ((long long)all[2 * r] != D->cuts[r]) return fail(SFAIRSC_E_DIM_MISMATCH, "row blocks do not tile [0, n) in rank order");
      D->cuts[r + 1] = D->cuts[r] + (long long)all[2 * r + 1];
    }
    if (D->cuts[D->P_total] != D->n) return fail(SFAIRSC_E_DIM_MISMATCH, "row blocks cover %lld of n = %lld rows",
                                                 D->cuts[D->P_total], D->n);
  } else {
    D->P = D->P_total = opts.virtual_parts;
    D->part0 = 0;
    // nnz-balanced cuts (weight nnz + 4 per row)
    const long long tot = (long long)hrp[W->n_rows] + 4LL * W->n_rows;
    D->cuts.assign(D->P + 1, 0);
    D->cuts[D->P] = W->n_rows;
    for (int q = 1; q < D->P; ++q) {
      const long long target = tot * q / D->P;
      long long lo = 0, hi = W->n_rows;
      while (lo < hi) {
        const long long mid = (lo + hi) / 2;
        if ((long long)hrp[mid] + 4 * mid < target) lo = mid + 1; else hi = mid;
      }
      D->cuts[q] = std::max(D->cuts[q - 1], lo);
    }
  }
  long long nmx = 1;
  for (int r = 0; r < D->P_total; ++r) nmx = std::max(nmx, D->cuts[r + 1] - D->cuts[r]);
  D->n_max = (int)((nmx + 255) / 256 * 256);
  CU(dal(&D->cuts_dev, D->P_total + 1));
  CU(cudaMemcpyAsync(D->cuts_dev, D->cuts.data(), sizeof(long long) * (D->P_total + 1), cudaMemcpyHostToDevice, st));
  CU(dal(&D->p_full, (size_t)D->P_total * D->n_max));
  CU(cudaMemsetAsync(D->p_full, 0, sizeof(double) * D->P_total * D->n_max, st));
  if (c->normalized) {
    CU(dal(&D->s_full, (size_t)D->P_total * D->n_max));
    CU(cudaMemsetAsync(D->s_full, 0, sizeof(double) * D->P_total * D->n_max, st));
  }
  CU(dal(&D->ptr_tab, 64));
  CU(cudaMallocHost((void**)&D->hp, 8192 * sizeof(double)));

  // ---- parts: local CSR, groups ----
  D->parts.resize(D->P);
  const int m = c->m;
  int hflags = 0;
  // per-part setup; a failure (e.g. OOM) on one rank must not leave the others blocked in the collectives
  // below, so the first local failure is recorded and agreed on (max over ranks) with the CSR flags
  unsigned long long symsum = 0ull;
  auto build_part = [&](int q) -> sfairsc_status {
    DistPart& p = D->parts[q];
    p.q = D->part0 + q;
    const long long a = D->comm ? 0 : D->cuts[q], b = D->comm ? W->n_rows : D->cuts[q + 1];  // rows in W
    p.r0 = D->cuts[p.q];
    p.n_loc = (int)(b - a);
    p.nnz_loc = hrp[b] - hrp[a];
    p.ldv = ((long long)std::max(p.n_loc, 1) + 255) / 256 * 256;
    CU(dal(&p.rp, p.n_loc + 1));
    CU(dal(&p.ci, p.nnz_loc));
    CU(dal(&p.vv, p.nnz_loc));
    std::vector<int32_t> lrp(p.n_loc + 1);
    for (long long i = 0; i <= p.n_loc; ++i) lrp[i] = hrp[a + i] - hrp[a];
    CU(cudaMemcpyAsync(p.rp, lrp.data(), sizeof(int32_t) * (p.n_loc + 1), cudaMemcpyHostToDevice, st));
    if (p.nnz_loc > 0) {
      CU(cudaMemcpyAsync(p.ci, W->col_idx + hrp[a], sizeof(int32_t) * p.nnz_loc, kind, st));
      CU(cudaMemcpyAsync(p.vv, W->values + hrp[a], sizeof(double) * p.nnz_loc, kind, st));
    }
    CU(dal(&p.dg, p.ldv));
    CU(cudaMemsetAsync(p.dg, 0, sizeof(double) * p.ldv, st));
    if (c->normalized) {
      CU(dal(&p.s, p.ldv));
      CU(cudaMemsetAsync(p.s, 0, sizeof(double) * p.ldv, st));
    }
    CU(dal(&p.grp, p.ldv));
    CU(cudaMemsetAsync(p.grp, 0, p.ldv, st));
    {
      std::vector<uint8_t> hg(p.n_loc);
      for (int i = 0; i < p.n_loc; ++i) hg[i] = (uint8_t)c->groups_host[a + i];
      CU(cudaMemcpyAsync(p.grp, hg.data(), p.n_loc, cudaMemcpyHostToDevice, st));
      CU(cudaStreamSynchronize(st));
    }
    CU(dal(&p.isb, 256));
    CU(dal(&p.uh, 256));
    CU(dal(&p.counters, 16));
    CU(cudaMemsetAsync(p.counters, 0, 16 * sizeof(unsigned), st));
    CU(dal(&p.flags, 8));
    CU(cudaMemsetAsync(p.flags, 0, 8 * sizeof(int), st));
    unsigned long long* psym = reinterpret_cast<unsigned long long*>(p.flags + 2);
    CU(dal(&p.small, 2048));
    CU(cudaMemsetAsync(p.small, 0, 2048 * sizeof(double), st));
    if (c->paired) {
      CU(dal(&p.vrB, p.ldv));
      CU(cudaMemsetAsync(p.vrB, 0, sizeof(double) * p.ldv, st));
    }
    for (double** v : {&p.vr, &p.vy, &p.vt}) {
      CU(dal(v, p.ldv));
      CU(cudaMemsetAsync(*v, 0, sizeof(double) * p.ldv, st));
    }
    CU(dal(&p.V, (size_t)(m + 1) * p.ldv));
    CU(dal(&p.Vb, (size_t)(m + 1) * p.ldv));
    CU(cudaMemsetAsync(p.V, 0, sizeof(double) * (m + 1) * p.ldv, st));
    CU(cudaMemsetAsync(p.Vb, 0, sizeof(double) * (m + 1) * p.ldv, st));
    CU(dal(&p.X, (size_t)c->k_build * p.ldv));
    CU(cudaMemsetAsync(p.X, 0, sizeof(double) * c->k_build * p.ldv, st));
    // A0: remap columns to the gathered layout + local validation
    bump_launch();
    k_remap_validate<<<grid_for(p.n_loc), kDT, 0, st>>>(p.rp, p.ci, p.vv, p.n_loc, p.r0, D->n, D->cuts_dev,
                                                        D->P_total, D->n_max, p.flags, psym);
    // A1: degrees
    bump_launch();
    k_degrees_d<<<grid_for(p.n_loc), kDT, 0, st>>>(p.rp, p.vv, p.n_loc, p.dg, p.flags);
    if (c->normalized) {
      bump_launch();
      k_inv_sqrt_d<<<grid_for(p.n_loc), kDT, 0, st>>>(p.dg, p.n_loc, p.s, D->s_full + (size_t)p.q * D->n_max);
    }
    CU(cudaGetLastError());
    // SpMV partition (nnz + 4 rows balanced)
    {
      const long long total = (long long)p.nnz_loc + 4LL * p.n_loc;
      const int G = std::max(1, std::min(c->num_sms * 8, (p.n_loc + 31) / 32));
      std::vector<int32_t> split(G + 1);
      split[0] = 0;
      split[G] = p.n_loc;
      for (int bb = 1; bb < G; ++bb) {
        const long long target = total * bb / G;
        int lo = 0, hi = p.n_loc;
        while (lo < hi) {
          const int mid = lo + ((hi - lo) >> 1);
          if ((long long)lrp[mid] + 4LL * mid < target) lo = mid + 1; else hi = mid;
        }
        split[bb] = std::max(split[bb - 1], lo);
      }
      p.spmv_grid = G;
      CU(dal(&p.row_split, G + 1));
      CU(cudaMemcpyAsync(p.row_split, split.data(), sizeof(int32_t) * (G + 1), cudaMemcpyHostToDevice, st));
    }
    p.vs = c->vs;
    {
      int maxdeg = 0;
      for (int i = 0; i < p.n_loc; ++i) maxdeg = std::max(maxdeg, lrp[i + 1] - lrp[i]);
      p.skewed = maxdeg > 16.0 * std::max(1.0, (double)p.nnz_loc / std::max(1, p.n_loc));
    }
    const size_t pc = std::max<size_t>((size_t)p.spmv_grid * 4 * kBT, (size_t)c->num_sms * 8 * (kMaxJ + 2));
    CU(dal(&p.partials, pc));
    CU(dal(&p.partials2, (size_t)c->num_sms * 8 * (kHB + 2)));
    int f2[4] = {0, 0, 0, 0};
    CU(cudaMemcpyAsync(f2, p.flags, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    hflags |= f2[0];
    unsigned long long ps_ = 0ull;
    std::memcpy(&ps_, f2 + 2, sizeof(ps_));
    symsum += ps_;
    // unit weights (unnormalized): each part decides for its own rows; the gathered p~ is used as is
    p.unit = !c->normalized && p.nnz_loc > 0 && f2[1] == 0 &&
             !(getenv("SFAIRSC_UNIT") && atoi(getenv("SFAIRSC_UNIT")) == 0);
      return SFAIRSC_OK;
  };
  sfairsc_status local_st = SFAIRSC_OK;
  std::string local_msg;
  for (int q = 0; q < D->P && local_st == SFAIRSC_OK; ++q) {
    local_st = build_part(q);
    if (local_st != SFAIRSC_OK) local_msg = sfairsc_last_error();
  }
  // symmetry: the fingerprint sums of all parts / ranks must cancel (mod 2^64).  Across NCCL ranks they
  // are summed as four 16-bit limbs in doubles (exact), recombined mod 2^64; every rank takes part even
  // after a local failure (its limbs are then 0 and its status is agreed on below).
  if (D->comm) {
    double limbs[4];
    for (int q = 0; q < 4; ++q) limbs[q] = local_st == SFAIRSC_OK ? (double)((symsum >> (16 * q)) & 0xFFFFull) : 0.0;
    double* t = D->parts[0].scal();
    CU(cudaMemcpyAsync(t, limbs, 4 * sizeof(double), cudaMemcpyHostToDevice, st));
    TRY(allreduce(D, st, 4, [](const DistPart& p) { return p.scal(); }));
    CU(cudaMemcpyAsync(limbs, t, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    symsum = 0ull;
    for (int q = 0; q < 4; ++q) symsum += (unsigned long long)limbs[q] << (16 * q);  // carries wrap mod 2^64
  }
  if (symsum != 0ull && c->check_symmetry) hflags |= 4;
  // flags and the local status: max over parts / ranks
  {
    double fl[2] = {(double)hflags, (double)local_st};
    double* t = D->parts[0].scal();
    CU(cudaMemcpyAsync(t, fl, 2 * sizeof(double), cudaMemcpyHostToDevice, st));
    TRY(allreduce(D, st, 2, [](const DistPart& p) { return p.scal(); }, true));
    CU(cudaMemcpyAsync(fl, t, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    hflags = (int)fl[0];
    if (local_st != SFAIRSC_OK) return fail(local_st, "%s", local_msg.c_str());
    if ((int)fl[1] != SFAIRSC_OK) return fail((sfairsc_status)(int)fl[1], "another rank failed its build (status %d)", (int)fl[1]);
  }
  if (hflags & 4) return fail(SFAIRSC_E_ASYMMETRIC, "W is not symmetric (distributed fingerprint of (i, j, w) vs (j, i, w))");
  if (hflags & 1) return fail(SFAIRSC_E_CSR_INVALID, "CSR invalid (row_ptr/col range, unsorted or duplicate columns, or nonzero diagonal)");
  if (hflags & 2) return fail(SFAIRSC_E_NEGATIVE_WEIGHT, "negative or NaN weight (P:121)");
  if (hflags & 8) return fail(SFAIRSC_E_ISOLATED_VERTEX, "isolated vertex: d_i = 0 (P:127-128)");
  // normalized: gather s, scale the stored values s_i w_ij s_j
  if (c->normalized) {
    TRY(allgather_full(D, st, D->s_full));
    for (auto& p : D->parts) {
      bump_launch();
      k_scale_d<<<grid_for(p.n_loc), kDT, 0, st>>>(p.rp, p.ci, p.vv, p.s, D->s_full, p.n_loc);
    }
  }
  // A2: sigma = ||L||_1 (max over parts)
  for (auto& p : D->parts) {
    bump_launch();
    k_sigma_d<<<std::max(1, std::min((p.n_loc + 4 * kDT - 1) / (4 * kDT), 296)), kDT, 0, st>>>(
        p.rp, p.vv, p.dg, p.n_loc, c->normalized, p.partials, p.counters + 0, p.scal());
  }
  TRY(allreduce(D, st, 1, [](const DistPart& p) { return p.scal(); }, true));
  double hsig = 0.0;
  CU(cudaMemcpyAsync(&hsig, D->parts[0].scal(), sizeof(double), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  c->sigma = opts.sigma_override > 0 ? opts.sigma_override : hsig;
  // owner-segment column blocking (P_total > 1 and a gathered vector beyond the ~48 MB that L2 keeps
  // across the CSR stream, e.g. config 5; env SFAIRSC_DIST_BLOCK=1 forces it, 0 disables): block-major
  // copy of each part's CSR.  Smaller problems gather first and run one SpMV (a 28 MB all-gather at
  // config 4 costs less than the extra column-block passes).
  bool blk = 8.0 * D->P_total * D->n_max > 48.0 * 1048576.0;
  if (getenv("SFAIRSC_DIST_BLOCK")) blk = atoi(getenv("SFAIRSC_DIST_BLOCK")) != 0;
  if (D->P_total > 1 && blk) {
    for (auto& p : D->parts) {
      if (p.nnz_loc == 0) continue;
      const int nb = D->P_total, nl = p.n_loc;
      int* cnt = nullptr;
      CU(dal(&cnt, (size_t)nb * nl));
      launch_colblk_starts(p.rp, p.ci, nl, nb, D->n_max, cnt, st);
      std::vector<int32_t> hc((size_t)nb * nl), hr((size_t)nb * (nl + 1));
      CU(cudaMemcpyAsync(hc.data(), cnt, sizeof(int32_t) * hc.size(), cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
      cudaFree(cnt);
      long long base = 0;
      for (int b = 0; b < nb; ++b) {
        int32_t* r = hr.data() + (size_t)b * (nl + 1);
        const int32_t* q = hc.data() + (size_t)b * nl;
        r[0] = (int32_t)base;
        for (int i = 0; i < nl; ++i) r[i + 1] = r[i] + q[i];
        base = r[nl];
      }
      if (base != p.nnz_loc) return fail(SFAIRSC_E_CUDA, "column blocking lost entries");
      CU(dal(&p.rpb, hr.size()));
      CU(cudaMemcpyAsync(p.rpb, hr.data(), sizeof(int32_t) * hr.size(), cudaMemcpyHostToDevice, st));
      int* ci2 = nullptr;
      double* vv2 = nullptr;
      CU(dal(&ci2, p.nnz_loc));
      CU(dal(&vv2, p.nnz_loc));
      launch_colblk_scatter(p.rp, p.ci, p.vv, nl, nb, p.rpb, ci2, vv2, st);
      CU(cudaGetLastError());
      CU(cudaStreamSynchronize(st));
      cudaFree(p.ci);
      cudaFree(p.vv);
      p.ci = ci2;
      p.vv = vv2;
      p.nblk = nb;
      const double mdb = (double)p.nnz_loc / std::max(1, nl) / nb;
      int vsb = 2;
      while (vsb < 32 && vsb * 4 < mdb) vsb *= 2;
      p.vs_blk = vsb;
    }
  }
  if (D->comm) {
    CU(cudaStreamCreateWithFlags(&D->cst, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&D->ev_ready, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&D->ev_gathered, cudaEventDisableTiming));
  }
  // A3: factored projector; group counts and beta_s = sum_{V_s} s_i^2 summed over parts
  std::vector<double> beta(hh), cntg(hh);
  {
    for (int s = 0; s < hh; ++s) cntg[s] = (double)cnt_local[s];
    if (D->comm) {  // the caller passed only this rank's groups
      double* t = D->parts[0].scal();
      CU(cudaMemcpyAsync(t, cntg.data(), sizeof(double) * hh, cudaMemcpyHostToDevice, st));
      TRY(allreduce(D, st, hh, [](const DistPart& p) { return p.scal(); }));
      CU(cudaMemcpyAsync(cntg.data(), t, sizeof(double) * hh, cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
    }
    for (int s = 0; s < hh; ++s)
      if (!(cntg[s] > 0)) return fail(SFAIRSC_E_EMPTY_GROUP, "group %d is empty (P:152)", s);
    if (c->normalized) {
      for (auto& p : D->parts)
        launch_gsum(p.g(true), p.s, 0, p.partials, p.counters + 3, p.bs_w(), st);
      TRY(allreduce(D, st, kHB, [](const DistPart& p) { return p.bs_w(); }));
      CU(cudaMemcpyAsync(beta.data(), D->parts[0].bs_w(), sizeof(double) * hh, cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
    } else {
      beta = cntg;
    }
  }
  std::vector<double> isb(hh), uh(hh);
  double un = 0.0;
  for (int s = 0; s < hh; ++s) {
    if (!(beta[s] > 0)) return fail(SFAIRSC_E_RANK_DEFICIENT, "group %d has zero weight", s);
    isb[s] = 1.0 / std::sqrt(beta[s]);
    uh[s] = cntg[s] * isb[s];
    un += uh[s] * uh[s];
  }
  un = std::sqrt(un);
  for (int s = 0; s < hh; ++s) uh[s] /= un;
  for (auto& p : D->parts) {
    CU(cudaMemcpyAsync(p.isb, isb.data(), sizeof(double) * hh, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(p.uh, uh.data(), sizeof(double) * hh, cudaMemcpyHostToDevice, st));
  }
  // replicated Lanczos state
  D->ldH = m + 2;
  CU(dal(&D->H, (size_t)D->ldH * D->ldH));
  CU(dal(&D->sv, m + 2));
  CU(dal(&D->lz, 16));
  CU(cudaMemsetAsync(D->lz, 0, 16 * sizeof(double), st));
  CU(dal(&D->cs, kMaxJ));
  CU(dal(&D->cg, kMaxJ));
  CU(dal(&D->Ydev, (size_t)(m + 1) * (m + 1)));
  CU(dal(&D->bflags, kMaxJ + 8));
  CU(cudaMemsetAsync(D->bflags, 0, sizeof(int) * (kMaxJ + 8), st));
  if (c->paired) {
    CU(dal(&D->lzp, 4 * kMaxJ));
    CU(cudaMemsetAsync(D->lzp, 0, sizeof(double) * 4 * kMaxJ, st));
  }
  CU(cudaStreamSynchronize(st));
  return SFAIRSC_OK;
}

}  // namespace sfz

// ---------------------------------------------------------------------------
// partitioned single-sweep Lanczos (the lanczos1.cu algorithm, one part per
// rank or P virtual parts; identical replicated coefficients everywhere)
// ---------------------------------------------------------------------------
#include "lanczos1.h"

namespace sfz {
namespace {

struct DistLanczos {
  sfairsc_ctx* c;
  DistCtx* D;
  int m, keep, k;
  int64_t applies = 0, steps = 0, restarts = 0, breakdowns = 0;
  unsigned inject = 0;
  double bd_tol = 0.0;

  cudaStream_t st() const { return c->st; }
  ProjDesc pd(const DistPart& p) const { return ProjDesc{c->h, p.isb, p.uh}; }
  double* pseg(const DistPart& p) const { return D->p_full + (size_t)p.q * D->n_max; }

  LzDev dev(const DistPart& p, int flag_idx) const {
    LzDev d{};
    d.H = D->H;
    d.ldH = D->ldH;
    d.s = D->sv;
    d.lz = D->lz;
    d.cs = D->cs;
    d.cg = D->cg;
    d.bs_t = p.bs_t();
    d.bs_v = p.bs_v();
    d.flag = D->bflags + flag_idx;
    d.sigma = c->sigma;
    d.bd_tol = bd_tol;
    d.epend = c->paired ? D->lzp : nullptr;
    d.econv = c->paired ? D->lzp + kMaxJ : nullptr;
    return d;
  }
  bool pend = false;  // host mirror of LZ_PEND >= 0
  sfairsc_status clear_pair_state() {
    pend = false;
    if (!c->paired) return SFAIRSC_OK;
    const double m1[5] = {-1.0, 1.0, -1.0, 1.0, 1.0};  // LZ_PEND, LZ_PRHO, LZ_CONV, LZ_CRHO, LZ_INVMU_A
    std::memcpy(D->hp + 2048, m1, sizeof(m1));
    CU(cudaMemcpyAsync(D->lz + LZ_PEND, D->hp + 2048, sizeof(m1), cudaMemcpyHostToDevice, st()));
    CU(cudaStreamSynchronize(st()));
    return SFAIRSC_OK;
  }

  // two Lanczos steps j, j+1 with one basis sweep per part (partitioned: the three-term
  // vector's |u|^2 / B^T u, the pair sweep's 2J + 3 dots and |w|^2 / B^T w / |v'|^2 are all-reduced)
  sfairsc_status pair(int j) {
    const bool rewrite = pend;
    {
      ProfScope ps(c, K_SPMV, 0.0);
      TRY(dist_spmv(D, c, st()));
      TRY(allreduce(D, st(), kBT, [](const DistPart& p) { return p.bs_t(); }));
    }
    launch_lz_coef(dev(D->parts[0], j), j, st());
    {
      ProfScope ps(c, K_NORMALIZE, 0.0);
      bool first = true;
      for (auto& p : D->parts) {
        const int G = std::max(1, std::min((p.n_loc + kThreads - 1) / kThreads, c->num_sms * 8));
        launch_lz_three(p.g(c->normalized), pd(p), p.vt, p.vr, p.V + (long long)(j - 1) * p.ldv, dev(p, j), j, p.vy,
                        p.dd(), D->lzp + 2 * kMaxJ, D->lzp + 3 * kMaxJ, p.partials, p.counters + 7, p.nb(), G, first,
                        st());
        first = false;
      }
      TRY(allreduce(D, st(), 1 + kHB, [](const DistPart& p) { return p.nb(); }));
      for (auto& p : D->parts)
        launch_lz_norm(p.g(c->normalized), pd(p), p.vy, p.nb(), p.dd(), j + 1, dev(p, j), j + 1, p.vrB, pseg(p),
                       p.bs_v(), st());
    }
    {
      ProfScope ps(c, K_SPMV, 0.0);
      TRY(dist_spmv(D, c, st()));
      TRY(allreduce(D, st(), kBT, [](const DistPart& p) { return p.bs_t(); }));
    }
    launch_lz_coef(dev(D->parts[0], j + 1), j + 1, st());
    {
      ProfScope ps(c, K_UPDDOT, 0.0);
      for (auto& p : D->parts) {
        LzPairArgs a{};
        a.V = p.V;
        a.ld = p.ldv;
        a.J = j;
        a.vtA = p.vr;
        a.vtB = p.vrB;
        a.t = p.vt;
        a.vj_out = p.V + (long long)j * p.ldv;
        a.vj1_out = p.V + (long long)(j + 1) * p.ldv;
        a.w_out = p.vy;
        a.conv_out = rewrite ? p.V + (long long)(j - 1) * p.ldv : nullptr;
        a.cA = D->lzp + 2 * kMaxJ;
        a.cB = D->cs;
        a.gB = D->cg;
        a.tr = D->lzp + 3 * kMaxJ;
        a.lz = D->lz;
        a.bs_t = p.bs_t();
        a.bs_v = p.bs_v();
        a.sigma = c->sigma;
        a.partials = p.partials;
        a.partials2 = p.partials2;
        a.counter = p.counters + 6;
        a.nb = p.nb();
        const int G = std::max(1, std::min((p.n_loc + 63) / 64, c->num_sms));
        launch_lz_pair(p.g(c->normalized), pd(p), a, G, st());
        launch_reduce_cols(p.partials, G, 2 * j + 3, p.dd2(), st());
      }
      // (one all-reduce each: 2 j + 3 dots, and |w|^2, B^T w, |v'|^2)
      TRY(allreduce(D, st(), 2 * j + 3, [](const DistPart& p) { return p.dd2(); }));
      TRY(allreduce(D, st(), 2 + kHB, [](const DistPart& p) { return p.nb(); }));
    }
    // the replicated bookkeeping once (part 0's reduced dots; every part then normalises with part 0's dd)
    launch_lz_pairpost(dev(D->parts[0], j + 1), j, D->parts[0].dd2(), D->parts[0].dd(), D->parts[0].nb(), D->bflags + j,
                       st());
    for (auto& p : D->parts)
      launch_lz_norm(p.g(c->normalized), pd(p), p.vy, p.nb(), D->parts[0].dd(), j + 2, dev(p, j + 1), j + 2, p.vr,
                     pseg(p), p.bs_v(), st());
    CHECK_LAUNCH();
    pend = true;
    applies += 2;
    steps += 2;
    return SFAIRSC_OK;
  }

  // v~ = P(w/|w|) on every part from the reduced nb (and dots)
  void norm_all(bool with_dots, int nd, int jrow, int flag_idx) {
    for (auto& p : D->parts)
      launch_lz_norm(p.g(c->normalized), pd(p), p.vy, p.nb(), with_dots ? p.dd() : nullptr, with_dots ? nd : 0,
                     dev(p, flag_idx), jrow, p.vr, pseg(p), p.bs_v(), st());
  }

  sfairsc_status step(int j) {
    {
      ProfScope ps(c, K_SPMV, 0.0);
      TRY(dist_spmv(D, c, st()));  // all-gather of p~ overlapped with the own-block SpMV
      TRY(allreduce(D, st(), kBT, [](const DistPart& p) { return p.bs_t(); }));
    }
    launch_lz_coef(dev(D->parts[0], j), j, st());
    {
      ProfScope ps(c, K_UPDDOT, 0.0);
      for (auto& p : D->parts) {
        LzSweepArgs a{};
        a.V = p.V;
        a.ld = p.ldv;
        a.J = j;
        a.vt = p.vr;
        a.t = p.vt;
        a.vj_out = p.V + (long long)j * p.ldv;
        a.w_out = p.vy;
        a.cs = D->cs;
        a.cg = D->cg;
        a.lz = D->lz;
        a.bs_t = p.bs_t();
        a.bs_v = p.bs_v();
        a.sigma = c->sigma;
        a.partials = p.partials;
        a.partials2 = p.partials2;
        a.counter = p.counters + 6;
        a.nb = p.nb();
        const int G = std::max(1, std::min((p.n_loc + 63) / 64, c->num_sms));
        launch_lz_update(p.g(c->normalized), pd(p), a, G, st());
        launch_reduce_cols(p.partials, G, j + 1, p.dd(), st());
      }
      TRY(allreduce(D, st(), j + 1, [](const DistPart& p) { return p.dd(); }));
      TRY(allreduce(D, st(), 1 + kHB, [](const DistPart& p) { return p.nb(); }));
    }
    norm_all(true, j + 1, j + 1, j);
    CHECK_LAUNCH();
    applies++;
    steps++;
    return SFAIRSC_OK;
  }

  // CGS2 (three sweeps, with reductions between them) of the vy blocks against V[:, 0:J]; |.|^2, B^T -> nb
  sfairsc_status cgs2_vy(int J) {
    for (auto& p : D->parts) {
      if (J > 0) {
        SweepArgs a{};
        a.V = p.V;
        a.ld = p.ldv;
        a.J = J;
        a.xin = p.vy;
        a.xout = p.vy;
        a.partials = p.partials;
        a.counter = p.counters + 2;
        a.norm_bsum = p.nb();
        const int G = sweep_grid(p.n_loc, c->num_sms);
        launch_sweep(3, p.g(c->normalized), pd(p), a, G, st());
        launch_reduce_cols(p.partials, G, J, p.dd(), st());
      }
    }
    if (J > 0) {
      TRY(allreduce(D, st(), J, [](const DistPart& p) { return p.dd(); }));
      for (auto& p : D->parts) {
        SweepArgs a{};
        a.V = p.V;
        a.ld = p.ldv;
        a.J = J;
        a.xin = p.vy;
        a.xout = p.vy;
        a.coef = p.dd();
        a.partials = p.partials;
        a.counter = p.counters + 2;
        a.norm_bsum = p.nb();
        const int G = sweep_grid(p.n_loc, c->num_sms);
        launch_sweep(1, p.g(c->normalized), pd(p), a, G, st());
        launch_reduce_cols(p.partials, G, J, p.dd() + 256, st());
      }
      TRY(allreduce(D, st(), J, [](const DistPart& p) { return p.dd() + 256; }));
    }
    for (auto& p : D->parts) {
      SweepArgs a{};
      a.V = p.V;
      a.ld = p.ldv;
      a.J = J;
      a.xin = p.vy;
      a.xout = p.vy;
      a.coef = p.dd() + 256;
      a.partials = p.partials;
      a.counter = p.counters + 2;
      a.norm_bsum = p.nb();
      launch_sweep(2, p.g(c->normalized), pd(p), a, sweep_grid(p.n_loc, c->num_sms), st());
    }
    TRY(allreduce(D, st(), 1 + kHB, [](const DistPart& p) { return p.nb(); }));
    CHECK_LAUNCH();
    return SFAIRSC_OK;
  }

  // v~_j = P(random) orthogonalised (CGS2 twice) against V[:, 0:j]; s = 0; H row j = 0
  sfairsc_status random_start(int j) {
    TRY(clear_pair_state());
    for (int attempt = 0; attempt < 5; ++attempt) {
      for (auto& p : D->parts) {
        bump_launch();
        k_random_off<<<grid_for(p.n_loc), kDT, 0, st()>>>(p.vt, p.n_loc, p.r0, c->seed, 4096u + inject, 7u);
        launch_gsum(p.g(c->normalized), p.vt, 0, p.partials, p.counters + 3, p.bs_w(), st());
      }
      inject++;
      TRY(allreduce(D, st(), kHB, [](const DistPart& p) { return p.bs_w(); }));
      for (auto& p : D->parts) launch_project(p.g(c->normalized), pd(p), p.vt, p.bs_w(), 1.0, p.vy, st());
      TRY(cgs2_vy(j));
      if (j > 0) TRY(cgs2_vy(j));
      CU(cudaMemsetAsync(D->bflags + kMaxJ, 0, sizeof(int), st()));
      norm_all(false, 0, -1, kMaxJ);
      CU(cudaMemsetAsync(D->sv, 0, sizeof(double) * (j + 1), st()));
      if (j > 0) {
        std::vector<double> zero(j, 0.0);
        CU(cudaMemcpy2DAsync(D->H + j, sizeof(double) * D->ldH, zero.data(), sizeof(double), sizeof(double), j,
                             cudaMemcpyHostToDevice, st()));
      }
      int flag = 0;
      CU(cudaMemcpyAsync(&flag, D->bflags + kMaxJ, sizeof(int), cudaMemcpyDeviceToHost, st()));
      CU(cudaStreamSynchronize(st()));
      if (!flag) return SFAIRSC_OK;
    }
    return fail(SFAIRSC_E_NO_CONVERGENCE, "could not generate a random vector outside the Krylov basis");
  }

  // y_i = L^sigma x_i - theta_i x_i norms for the k columns of X (A11), k distributed applies
  sfairsc_status true_residuals(const double* theta, double* max_out) {
    double mx = 0.0;
    for (int i = 0; i < k; ++i) {
      for (auto& p : D->parts)
        launch_gsum(p.g(c->normalized), p.X + (long long)i * p.ldv, 0, p.partials, p.counters + 3, p.bs_w(), st());
      TRY(allreduce(D, st(), kHB, [](const DistPart& p) { return p.bs_w(); }));
      for (auto& p : D->parts)
        launch_project(p.g(c->normalized), pd(p), p.X + (long long)i * p.ldv, p.bs_w(), 1.0, pseg(p), st());
      TRY(dist_spmv(D, c, st()));
      TRY(allreduce(D, st(), kBT, [](const DistPart& p) { return p.bs_t(); }));
      for (auto& p : D->parts) {
        launch_finish(p.g(c->normalized), pd(p), p.vt, p.bs_t(), p.bs_w(), c->sigma, p.vy, st());
        launch_resid(p.vy, p.X + (long long)i * p.ldv, theta[i], p.n_loc, p.partials, p.counters + 4, p.scal(), st());
      }
      TRY(allreduce(D, st(), 1, [](const DistPart& p) { return p.scal(); }));
      double r2 = 0.0;
      CU(cudaMemcpyAsync(&r2, D->parts[0].scal(), sizeof(double), cudaMemcpyDeviceToHost, st()));
      CU(cudaStreamSynchronize(st()));
      mx = std::max(mx, std::sqrt(r2) / c->sigma);
    }
    applies += k;
    *max_out = mx;
    return SFAIRSC_OK;
  }

  void ritz(int me, int pe, bool to_X) {
    for (auto& p : D->parts) launch_ritz(p.V, p.ldv, p.n_loc, me, D->Ydev, pe, to_X ? p.X : p.Vb, st());
  }
};

}  // namespace

sfairsc_status dist_eigs(sfairsc_ctx* c, int k, double tol, double* evals_out, double* evecs_out, int evecs_memspace,
                         sfairsc_stats* stats) {
  const double t0 = now_s();
  DistCtx* D = c->dist;
  c->have_eigs = false;
  DistLanczos L;
  L.c = c;
  L.D = D;
  L.m = c->m;
  L.keep = c->keep;
  L.k = k;
  const int m = L.m, keep = L.keep, ldH = D->ldH;
  const double tol_eff = std::min(tol, c->tol_cap);
  const double target = tol_eff * c->sigma;
  L.bd_tol = std::min(1e-12, 0.01 * tol_eff) * c->sigma;
  cudaStream_t st = c->st;
  CU(cudaMemsetAsync(D->H, 0, sizeof(double) * ldH * ldH, st));
  CU(cudaMemsetAsync(D->bflags, 0, sizeof(int) * (kMaxJ + 8), st));
  TRY(L.random_start(0));
  int j = 0, jsync = 0;
  bool converged = false;
  std::vector<double> theta, Y, Hh((size_t)ldH * ldH), sh(m + 2);
  double gap = std::numeric_limits<double>::quiet_NaN();
  double max_resid = std::numeric_limits<double>::infinity();
  for (;;) {
    {  // single first step(s) of a cycle, then pairs (paired builds), as in lanczos1.cu
      const int j0 = j;
      while (j < m) {
        if (!c->paired || j == j0 || (m - j) % 2 == 1) TRY(L.step(j++));
        else {
          TRY(L.pair(j));
          j += 2;
        }
      }
    }
    CU(cudaMemcpyAsync(Hh.data(), D->H, sizeof(double) * ldH * ldH, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(sh.data(), D->sv, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(D->hp, D->lz, sizeof(double) * 16, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(D->hp + 16, D->bflags, sizeof(int) * (m + 1), cudaMemcpyDeviceToHost, st));
    if (L.pend) CU(cudaMemcpyAsync(D->hp + 1024, D->lzp, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (c->prof.on) c->prof.resolve();
    int jb = -1;
    const int* fl = reinterpret_cast<const int*>(D->hp + 16);
    for (int q = jsync; q < m; ++q)
      if (fl[q]) {
        jb = q;
        break;
      }
    if (jb >= 0) {
      const int jn = (fl[jb] & 2) ? jb : jb + 1;
      L.breakdowns++;
      CU(cudaMemsetAsync(D->bflags, 0, sizeof(int) * (kMaxJ + 8), st));
      TRY(L.random_start(jn));
      j = jn;
      jsync = j;
      continue;
    }
    // paired steps: the last pair's odd column m-1 is still the stored v'
    const bool tconv = L.pend;
    const double prho = D->hp[LZ_PRHO];
    std::vector<double> pdef(tconv ? m - 1 : 0);
    if (tconv) {
      for (int l = 0; l < m - 1; ++l) pdef[l] = D->hp[1024 + l];
      pair_pending_to_orthonormal(m, ldH, Hh, sh, pdef.data(), prho);
    }
    auto to_stored = [&](double* x) {
      if (tconv) pair_coef_to_stored(m, x, pdef.data(), prho);
    };
    const double om = D->hp[LZ_OMEGA];
    double s2 = 0.0;
    for (int l = 0; l < m; ++l) s2 += sh[l] * sh[l];
    double mu = std::sqrt(std::max(om - s2, 0.0));
    if (!(mu > 0.0)) mu = 1.0;
    std::vector<double> bt(m), A((size_t)m * m);
    for (int l = 0; l < m; ++l) bt[l] = Hh[(size_t)l * ldH + m];
    for (int r = 0; r < m; ++r)
      for (int q = 0; q < m; ++q)
        A[(size_t)r * m + q] = 0.5 * ((Hh[(size_t)q * ldH + r] + sh[r] * bt[q]) + (Hh[(size_t)r * ldH + q] + sh[q] * bt[r]));
    Y = A;
    // only the kept (>= k) smallest Ritz vectors are used below: the selected-vector eigensolver
    const int nsel = std::min(m, std::max(keep, k));
    symeig(m, Y, theta, nsel);
    std::vector<double> bY(m, 0.0);
    double maxres = 0.0;
    for (int i = 0; i < nsel; ++i) {
      double acc = 0.0;
      for (int l = 0; l < m; ++l) acc += bt[l] * Y[(size_t)l * m + i];
      bY[i] = mu * acc;
    }
    for (int i = 0; i < k; ++i) maxres = std::max(maxres, std::fabs(bY[i]));
    if (k < m) gap = theta[k] - theta[k - 1];
    converged = maxres <= target;
    if (converged || L.restarts >= c->max_restarts) {
      std::vector<double> Yc((size_t)m * k);
      for (int cc = 0; cc < k; ++cc) {
        for (int l = 0; l < m; ++l) Yc[(size_t)cc * m + l] = Y[(size_t)l * m + cc];
        to_stored(Yc.data() + (size_t)cc * m);
      }
      CU(cudaMemcpyAsync(D->Ydev, Yc.data(), sizeof(double) * Yc.size(), cudaMemcpyHostToDevice, st));
      L.ritz(m, k, true);
      CHECK_LAUNCH();
      break;
    }
    for (auto& p : D->parts)
      CU(cudaMemcpyAsync(p.V + (long long)m * p.ldv, p.vr, sizeof(double) * p.ldv, cudaMemcpyDeviceToDevice, st));
    const int me = m + 1, pe = keep + 1;
    std::vector<double> Yc((size_t)me * pe, 0.0);
    for (int cc = 0; cc < keep; ++cc)
      for (int l = 0; l < m; ++l) Yc[(size_t)cc * me + l] = Y[(size_t)l * m + cc];
    for (int l = 0; l < m; ++l) Yc[(size_t)keep * me + l] = -sh[l] / mu;
    Yc[(size_t)keep * me + m] = 1.0 / mu;
    for (int cc = 0; cc <= keep; ++cc) to_stored(Yc.data() + (size_t)cc * me);
    CU(cudaMemcpyAsync(D->Ydev, Yc.data(), sizeof(double) * Yc.size(), cudaMemcpyHostToDevice, st));
    {
      ProfScope ps(c, K_RITZ, 0.0);
      L.ritz(me, pe, false);
    }
    for (auto& p : D->parts) std::swap(p.V, p.Vb);
    std::fill(Hh.begin(), Hh.end(), 0.0);
    for (int i = 0; i < keep; ++i) {
      Hh[(size_t)i * ldH + i] = theta[i];
      Hh[(size_t)i * ldH + keep] = bY[i];
    }
    CU(cudaMemcpyAsync(D->H, Hh.data(), sizeof(double) * ldH * ldH, cudaMemcpyHostToDevice, st));
    CU(cudaMemsetAsync(D->sv, 0, sizeof(double) * (m + 2), st));
    for (auto& p : D->parts) {  // v~ <- column keep (copy + |v|^2 + B^T v), then normalise
      SweepArgs a{};
      a.V = p.V;
      a.ld = p.ldv;
      a.J = 0;
      a.xin = p.V + (long long)keep * p.ldv;
      a.xout = p.vy;
      a.partials = p.partials;
      a.counter = p.counters + 2;
      a.norm_bsum = p.nb();
      launch_sweep(2, p.g(c->normalized), L.pd(p), a, sweep_grid(p.n_loc, c->num_sms), st);
    }
    TRY(allreduce(D, st, 1 + kHB, [](const DistPart& p) { return p.nb(); }));
    L.norm_all(false, 0, -1, kMaxJ);
    CHECK_LAUNCH();
    TRY(L.clear_pair_state());
    j = keep;
    jsync = keep;
    L.restarts++;
  }
  TRY(L.true_residuals(theta.data(), &max_resid));
  if (c->prof.on) c->prof.resolve();
  c->evals.assign(theta.begin(), theta.begin() + k);
  c->k_eigs = k;
  c->have_eigs = true;
  for (int i = 0; i < k; ++i) evals_out[i] = theta[i];
  if (evecs_out) {  // this process's rows: [sum of its parts' n_loc] x k, column-major
    const long long nl = D->cuts[D->part0 + D->P] - D->cuts[D->part0];
    const cudaMemcpyKind kind = evecs_memspace == SFAIRSC_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    long long off = 0;
    for (auto& p : D->parts) {
      CU(cudaMemcpy2DAsync(evecs_out + off, sizeof(double) * nl, p.X, sizeof(double) * p.ldv,
                           sizeof(double) * p.n_loc, k, kind, st));
      off += p.n_loc;
    }
    CU(cudaStreamSynchronize(st));
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
  S.basis_size = m;
  S.kept = keep;
  c->last = S;
  if (stats) *stats = S;
  if (!converged) return fail(SFAIRSC_E_NO_CONVERGENCE, "no convergence after %lld restarts", (long long)L.restarts);
  if (theta[k - 1] >= c->sigma * (1.0 - 1e-8))
    return fail(SFAIRSC_E_SHIFT_TOO_SMALL, "lambda_k=%g >= sigma(1-1e-8)=%g (Prop. 3.4)", theta[k - 1], c->sigma);
  return SFAIRSC_OK;
}

// y = L^sigma x for this process's rows (A4-A6, partitioned): x, y are [local rows] device vectors
sfairsc_status dist_apply(sfairsc_ctx* c, const double* x, double* y) {
  DistCtx* D = c->dist;
  cudaStream_t st = c->st;
  DistLanczos L;
  L.c = c;
  L.D = D;
  long long off = 0;
  for (auto& p : D->parts) {
    CU(cudaMemcpyAsync(p.vr, x + off, sizeof(double) * p.n_loc, cudaMemcpyDeviceToDevice, st));
    off += p.n_loc;
    launch_gsum(p.g(c->normalized), p.vr, 0, p.partials, p.counters + 3, p.bs_w(), st);
  }
  TRY(allreduce(D, st, kHB, [](const DistPart& p) { return p.bs_w(); }));
  for (auto& p : D->parts) launch_project(p.g(c->normalized), L.pd(p), p.vr, p.bs_w(), 1.0, L.pseg(p), st);
  TRY(dist_spmv(D, c, st));
  TRY(allreduce(D, st, kBT, [](const DistPart& p) { return p.bs_t(); }));
  off = 0;
  for (auto& p : D->parts) {
    launch_finish(p.g(c->normalized), L.pd(p), p.vt, p.bs_t(), p.bs_w(), c->sigma, y + off, st);
    off += p.n_loc;
  }
  CHECK_LAUNCH();
  return SFAIRSC_OK;
}

long long dist_local_rows(const sfairsc_ctx* c) {
  const DistCtx* D = c->dist;
  return D->cuts[D->part0 + D->P] - D->cuts[D->part0];
}

// k-means (Alg. 3 step 4) on the gathered H: every process runs the same
// deterministic k-means on all n rows and keeps the labels of its rows.
sfairsc_status dist_kmeans(sfairsc_ctx* c, uint64_t seed, int32_t* labels_out, int32_t memspace, double* objective) {
  DistCtx* D = c->dist;
  cudaStream_t st = c->st;
  const int k = c->k_eigs;
  const long long n = D->n, ldf = (n + 255) / 256 * 256;
  if (!D->X_full) {
    CU(dal(&D->X_full, (size_t)ldf * c->k_build));
    if (c->normalized) CU(dal(&D->s_compact, ldf));
  }
  // gather X (padded per part) then compact into X_full (n x k, ld = ldf)
  double* gath = nullptr;
  CU(dal(&gath, (size_t)D->P_total * D->n_max * k));
  for (int col = 0; col < k; ++col) {
    double* gc = gath + (size_t)col * D->P_total * D->n_max;
    for (auto& p : D->parts)
      CU(cudaMemcpyAsync(gc + (size_t)p.q * D->n_max, p.X + (long long)col * p.ldv, sizeof(double) * p.n_loc,
                         cudaMemcpyDeviceToDevice, st));
    if (D->comm)
      NC(nccl().AllGather(gc + (size_t)D->comm->rank * D->n_max, gc, D->n_max, ncclDouble, D->comm->comm, st));
  }
  for (int r = 0; r < D->P_total; ++r) {
    const long long nr = D->cuts[r + 1] - D->cuts[r];
    CU(cudaMemcpy2DAsync(D->X_full + D->cuts[r], sizeof(double) * ldf, gath + (size_t)r * D->n_max,
                         sizeof(double) * D->P_total * D->n_max, sizeof(double) * nr, k, cudaMemcpyDeviceToDevice, st));
    if (c->normalized)
      CU(cudaMemcpyAsync(D->s_compact + D->cuts[r], D->s_full + (size_t)r * D->n_max, sizeof(double) * nr,
                         cudaMemcpyDeviceToDevice, st));
  }
  CU(cudaStreamSynchronize(st));
  cudaFree(gath);
  if (!D->km) {
    D->km = new sfairsc_ctx();
    D->km->device = c->device;
    D->km->num_sms = c->num_sms;
  }
  sfairsc_ctx* S = D->km;
  S->st = st;
  S->n = (int)n;
  S->ldv = ldf;
  S->k_eigs = k;
  S->have_eigs = true;
  S->normalized = c->normalized;
  S->X = D->X_full;
  S->s = c->normalized ? D->s_compact : nullptr;
  int32_t* lab = nullptr;
  CU(dal(&lab, n));
  sfairsc_status rs = kmeans_run(S, seed, lab, SFAIRSC_MEM_DEVICE, objective);
  if (rs != SFAIRSC_OK) {
    cudaFree(lab);
    return rs;
  }
  const long long r0 = D->cuts[D->part0], nl = dist_local_rows(c);
  cudaError_t e = cudaMemcpyAsync(labels_out, lab + r0, sizeof(int32_t) * nl,
                                  memspace == SFAIRSC_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaFree(lab);
  if (e != cudaSuccess) return fail(SFAIRSC_E_CUDA, "labels copy: %s", cudaGetErrorString(e));
  return SFAIRSC_OK;
}

}  // namespace sfz
