// libsfairsc — k-means on the rows of H (Alg. 3 step 4), reading R16:
// k-means++ seeding with Philox4x32-10 draws (key = seed, counter (t, r, 8, 0)),
// Lloyd iterations (assignment ties -> lowest index; stop when no label
// changes or 300 iterations), an empty cluster is re-seeded at the point
// farthest from its assigned centroid, best of 10 restarts by WCSS.
// Rows h_i = s_i X[i, :] (normalized, H = D^{-1/2} X) or X[i, :], read in place
// from the column-major eigenvector block.  Squared distances are summed
// over dimensions in index order without FMA contraction (same arithmetic
// as the oracle's definition).  All reductions are fixed-order.
#include "sfairsc.h"
#include "device_common.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <limits>
#include <vector>

namespace sfz {

cudaStream_t ctx_stream(sfairsc_ctx* c);
int ctx_n(sfairsc_ctx* c);
int ctx_k(sfairsc_ctx* c);
const double* ctx_X(sfairsc_ctx* c, long long* ld);
const double* ctx_s(sfairsc_ctx* c);
int ctx_num_sms(sfairsc_ctx* c);
void** ctx_km(sfairsc_ctx* c, void (**freer)(void*));
void ctx_set_km_free(sfairsc_ctx* c, void (*f)(void*));
sfairsc_status ctx_fail(sfairsc_status st, const char* msg);
void ctx_prof_begin(sfairsc_ctx* c, cudaEvent_t* a);
void ctx_prof_end(sfairsc_ctx* c, int kind, cudaEvent_t a);
void bump_launch();

namespace {

constexpr int kBlk = 1024;     // D2 prefix blocks
int g_km_mma = 1;              // 1: tensor-core assignment with the exact guard; 0: direct (env SFAIRSC_KM_MMA)
int g_km_debug = 0;            // env SFAIRSC_DEBUG: per-iteration label changes on stderr
int g_km_incr = 1;             // 1: incremental cluster sums between full recomputations (env SFAIRSC_KM_INCR)
int g_km_prune = 0;            // 1: bound-pruned assignment (env SFAIRSC_KM_PRUNE)
constexpr int kKmRefresh = 16; // full recomputation at least every 16 Lloyd iterations (bounds the drift)
constexpr int kMaxDim = 64;    // k <= 64 handled in registers
constexpr int kKmStream = 8;   // Philox stream of the k-means draws

__device__ __forceinline__ double hval(const double* X, long long ld, const double* s, int i, int d) {
  const double x = X[(long long)d * ld + i];
  return s ? s[i] * x : x;
}

// squared distance, dimensions in order, no FMA contraction
template <int DP>
__device__ __forceinline__ double sqdist(const double (&h)[DP], const double* mu, int dim) {
  double acc = 0.0;
#pragma unroll
  for (int d = 0; d < DP; ++d)
    if (d < dim) {
      const double t = __dsub_rn(h[d], mu[d]);
      acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
  return acc;
}

template <int DP>
__device__ __forceinline__ void load_row(const double* X, long long ld, const double* s, int i, int dim, double (&h)[DP]) {
#pragma unroll
  for (int d = 0; d < DP; ++d) h[d] = d < dim ? hval(X, ld, s, i, d) : 0.0;
}

// D2_i = (init ? inf : D2_i) min |h_i - center|^2 ; per-block sums of D2 (fixed 1024-element blocks).
// Each thread carries kBlk/256 = 4 rows as independent accumulation chains (each
// still summed over d in index order) so the fp64 add latency is overlapped.
template <int DP>
__global__ void __launch_bounds__(256) k_d2(const double* X, long long ld, const double* s, int n, int dim,
                                            const double* center, int init, double* D2, double* blocksum) {
  constexpr int Q = kBlk / 256;
  __shared__ double red[256 / 32];
  __shared__ double cs[DP];
  for (int d = threadIdx.x; d < DP; d += blockDim.x) cs[d] = d < dim ? center[d] : 0.0;
  __syncthreads();
  const int b = blockIdx.x;
  int i[Q];
  double sc[Q], acc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    i[q] = b * kBlk + q * 256 + threadIdx.x;
    sc[q] = (s && i[q] < n) ? s[i[q]] : 1.0;
    acc[q] = 0.0;
  }
#pragma unroll
  for (int d = 0; d < DP; ++d)
    if (d < dim) {
#pragma unroll
      for (int q = 0; q < Q; ++q)
        if (i[q] < n) {
          const double x = X[(long long)d * ld + i[q]];
          const double t = __dsub_rn(s ? __dmul_rn(sc[q], x) : x, cs[d]);
          acc[q] = __dadd_rn(acc[q], __dmul_rn(t, t));
        }
    }
  double part = 0.0;
#pragma unroll
  for (int q = 0; q < Q; ++q)
    if (i[q] < n) {
      const double v = init ? acc[q] : fmin(acc[q], D2[i[q]]);
      D2[i[q]] = v;
      part += v;  // order irrelevant for the block sum's use (search), but fixed
    }
  part = warp_sum(part);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 256 / 32; ++w) t += red[w];
    blocksum[b] = t;
  }
}

// smallest i in block b with (running prefix from `base`) > target, sequential
__global__ void k_select_in_block(const double* D2, int b, int n, double base, double target, int* out) {
  if (threadIdx.x != 0) return;
  double cum = base;
  int last_pos = -1;
  const int i0 = b * kBlk, i1 = min(n, i0 + kBlk);
  for (int i = i0; i < i1; ++i) {
    const double v = D2[i];
    cum += v;
    if (v > 0) last_pos = i;
    if (cum > target) {
      *out = i;
      return;
    }
  }
  *out = last_pos >= 0 ? last_pos : i1 - 1;
}

__global__ void k_gather_row(const double* X, long long ld, const double* s, int i, int dim, double* out) {
  for (int d = threadIdx.x; d < dim; d += blockDim.x) out[d] = hval(X, ld, s, i, d);
}

__device__ __forceinline__ unsigned sptr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sptr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sptr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Assignment.  One CTA per SM, 8 warps; each warp owns 32 rows at a time (lane =
// row) and prefetches its next 32 rows into a private shared tile with cp.async
// while it computes the current ones from registers.  Centroids in shared memory
// as [K][dimp] (dimp = dim rounded up to even, so a pair of dimensions is one
// 16-byte load); four centroids are evaluated together (four independent chains,
// each summed over d in index order) and compared in increasing index order, so
// ties still go to the lowest index.
// 12 warps per CTA (3 per scheduler) while their row tiles fit in shared memory, else 8
template <int DP>
constexpr int asg_warps() { return DP <= 56 ? 12 : 8; }
inline size_t asg_smem(int K, int dim, int warps) {
  return sizeof(double) * ((size_t)K * ((dim + 1) & ~1) + (size_t)warps * (dim + 1) * 32);
}
template <int DP, int kAsgU, int kAsgWarps = asg_warps<DP>()>
__global__ void __launch_bounds__(kAsgWarps * 32) k_assign(const double* X, long long ld, const double* s, int n, int dim,
                                                           int K, const double* mu, const int* old_labels, int* labels,
                                                           double* dist, int* changes) {
  extern __shared__ __align__(16) double smu[];
  const int dimp = (dim + 1) & ~1;
  for (int e = threadIdx.x; e < K * dimp; e += blockDim.x) {
    const int c = e / dimp, d = e - c * dimp;
    smu[e] = d < dim ? mu[c * dim + d] : 0.0;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* tile = smu + (size_t)K * dimp + (size_t)w * (dim + 1) * 32;  // [dim][32], then s [32]
  const long long stride = (long long)gridDim.x * kAsgWarps * 32;
  long long base = ((long long)blockIdx.x * kAsgWarps + w) * 32;
  auto prefetch = [&](long long b0) {
    const long long i = b0 + lane;
    if (i < n) {
      for (int d = 0; d < dim; ++d) cp_async8(tile + d * 32 + lane, X + (long long)d * ld + i);
      if (s) cp_async8(tile + dim * 32 + lane, s + i);
    }
    cp_commit();
  };
  prefetch(base);
  __syncthreads();
  int ch = 0;
  for (; base < n; base += stride) {
    cp_wait<0>();
    __syncwarp();
    const long long i = base + lane;
    double h[DP];
    const double sc = s ? tile[dim * 32 + lane] : 1.0;
#pragma unroll
    for (int d = 0; d < DP; ++d) {
      const double x = d < dim ? tile[d * 32 + lane] : 0.0;
      h[d] = s ? __dmul_rn(sc, x) : x;
    }
    __syncwarp();
    prefetch(base + stride);
    if (i < n) {
      double best = 0.0;
      int bl = 0;
      for (int c0 = 0; c0 < K; c0 += kAsgU) {
        double a[kAsgU];
        const double* m[kAsgU];
#pragma unroll
        for (int j = 0; j < kAsgU; ++j) {
          a[j] = 0.0;
          m[j] = smu + min(c0 + j, K - 1) * dimp;
        }
#pragma unroll
        for (int d = 0; d < DP; d += 2)
          if (d < dim) {
#pragma unroll
            for (int j = 0; j < kAsgU; ++j) {
              const double2 q = *reinterpret_cast<const double2*>(m[j] + d);
              const double t0 = __dsub_rn(h[d], q.x);
              a[j] = __dadd_rn(a[j], __dmul_rn(t0, t0));
              if (d + 1 < dim) {
                const double t1 = __dsub_rn(h[d + 1], q.y);
                a[j] = __dadd_rn(a[j], __dmul_rn(t1, t1));
              }
            }
          }
#pragma unroll
        for (int j = 0; j < kAsgU; ++j)
          if (c0 + j < K && (c0 + j == 0 || a[j] < best)) {
            best = a[j];
            bl = c0 + j;
          }
      }
      if (old_labels && old_labels[i] != bl) ++ch;
      labels[i] = bl;
      dist[i] = best;
    }
  }
  cp_wait<0>();
  if (changes) {
    ch = __reduce_add_sync(0xffffffffu, ch);
    if (lane == 0 && ch) atomicAdd(changes, ch);  // integer: order-independent
  }
}

// Assignment on the fp64 tensor cores with an exact guard.  D~(i,c) = |h_i|^2 - 2 h_i.mu_c + |mu_c|^2
// from a DMMA (mma.sync m8n8k4 f64) product of a 128-row tile of H with M^T; |D~ - D| <= E_i with
// E_i = 4 (2 dim + 7) 2^-53 (|h_i| + max_c |mu_c|)^2 bounding the rounding of both D~ and the direct
// D (R16 arithmetic: index-order sum of (h_d - mu_d)^2, no FMA).  Every c with D~(i,c) <= min_c D~ + 2 E_i
// is a candidate; any other c has D(i,c) > D(i,c~) and cannot be (or tie) the minimum.  The candidates'
// D are then evaluated with the R16 arithmetic in increasing c (ties to the lowest index): the labels and
// dist are bit-identical to k_assign's.
constexpr int kMmaRows = 128, kMmaAS = 136, kMmaBS = 72;  // tile rows, smem strides (= 8 mod 16 doubles)
inline size_t asg_mma_smem(int dim) {
  const int dp4 = (dim + 3) & ~3;
  return sizeof(double) * ((size_t)dp4 * kMmaAS + (size_t)dp4 * kMmaBS + 64 + kMmaRows) +
         sizeof(unsigned long long) * kMmaRows;
}
__global__ void __launch_bounds__(256, 2) k_assign_mma(const double* X, long long ld, const double* s, int n,
                                                        int dim, int K, const double* mu, const int* old_labels,
                                                        int* labels, double* dist, int* changes) {
  extern __shared__ __align__(16) double sm[];
  const int dp4 = (dim + 3) & ~3;
  double* As = sm;                                  // [dp4][kMmaAS]  h (scaled rows), column d contiguous
  double* Bs = As + (size_t)dp4 * kMmaAS;           // [dp4][kMmaBS]  M^T, zero-padded to 64 columns
  double* musq = Bs + (size_t)dp4 * kMmaBS;         // [64]
  double* hn = musq + 64;                           // [128]
  unsigned long long* cmask = reinterpret_cast<unsigned long long*>(hn + kMmaRows);  // [128] candidate sets
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int KT = (K + 7) >> 3;  // 8-column DMMA tiles that hold centroids
  for (int e = tid; e < dp4 * kMmaBS; e += 256) {
    const int d = e / kMmaBS, c = e - d * kMmaBS;
    Bs[e] = (d < dim && c < K) ? mu[c * dim + d] : 0.0;
  }
  __syncthreads();
  if (tid < 64) {
    double a = 0.0;
    for (int d = 0; d < dim; ++d) a += Bs[d * kMmaBS + tid] * Bs[d * kMmaBS + tid];
    musq[tid] = a;
  }
  __syncthreads();
  double mumax = 0.0;
  for (int c = 0; c < K; ++c) mumax = fmax(mumax, musq[c]);
  mumax = sqrt(mumax);
  const double eunit = 4.0 * (2.0 * dim + 7.0) * 0x1p-53;
  int ch = 0;
  const int ntiles = (n + kMmaRows - 1) / kMmaRows;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long row0 = (long long)tile * kMmaRows;
    // stage the tile: As[d][r] = h_{row0+r, d} (R16 scaling s_i x, rounded like k_assign's load_row)
    {  // thread (r = tid & 127, d0 = tid >> 7) stages dims d0, d0 + 2, ...: 16 loads in flight per batch
      const int r = tid & (kMmaRows - 1), d0 = tid >> 7;
      const long long i = row0 + r;
      const bool rv = i < n;
      const double si = (s && rv) ? s[i] : 1.0;
      for (int dbase = 0; dbase < dp4; dbase += 32) {
        double v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int d = dbase + d0 + 2 * q;
          v[q] = (rv && d < dim) ? __ldg(X + (long long)d * ld + i) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int d = dbase + d0 + 2 * q;
          if (d < dp4) As[d * kMmaAS + r] = s ? __dmul_rn(si, v[q]) : v[q];
        }
      }
    }
    if (tid < kMmaRows) cmask[tid] = 0ull;
    __syncthreads();
    if (tid < kMmaRows) {
      double a = 0.0;
      for (int d = 0; d < dim; ++d) a += As[d * kMmaAS + tid] * As[d * kMmaAS + tid];
      hn[tid] = a;
    }
    // C = H_tile M^T: warp w owns rows 16 w .. 16 w + 15 (2 row tiles) and all KT column tiles
    double acc[2][8][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int ks = 0; ks < dp4; ks += 4) {
      double af[2], bf[8];
#pragma unroll
      for (int a = 0; a < 2; ++a) af[a] = As[(ks + tq) * kMmaAS + w * 16 + a * 8 + gq];
#pragma unroll
      for (int b = 0; b < 8; ++b) bf[b] = Bs[(ks + tq) * kMmaBS + b * 8 + gq];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b)
          if (b < KT)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[a][b][0]), "+d"(acc[a][b][1])
                         : "d"(af[a]), "d"(bf[b]));
    }
    __syncthreads();  // hn ready
    // approximate distances, row minima (lane: rows 16w + 8a + gq, columns 8b + 2tq + q)
    double dmin[2] = {INFINITY, INFINITY};
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int r = w * 16 + a * 8 + gq;
#pragma unroll
      for (int b = 0; b < 8; ++b)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int c = b * 8 + 2 * tq + q;
          if (b < KT && c < K) {
            acc[a][b][q] = hn[r] - 2.0 * acc[a][b][q] + musq[c];
            dmin[a] = fmin(dmin[a], acc[a][b][q]);
          }
        }
      dmin[a] = fmin(dmin[a], __shfl_xor_sync(0xffffffffu, dmin[a], 1));
      dmin[a] = fmin(dmin[a], __shfl_xor_sync(0xffffffffu, dmin[a], 2));
    }
    // candidates: D~ <= min D~ + 2 E_i
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int r = w * 16 + a * 8 + gq;
      const double nh = sqrt(hn[r]) + mumax;
      const double thr = dmin[a] + 2.0 * eunit * nh * nh;
      unsigned long long m = 0ull;
#pragma unroll
      for (int b = 0; b < 8; ++b)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int c = b * 8 + 2 * tq + q;
          if (b < KT && c < K && !(acc[a][b][q] > thr)) m |= 1ull << c;  // NaN-safe: NaN -> candidate
        }
      m |= __shfl_xor_sync(0xffffffffu, m, 1);
      m |= __shfl_xor_sync(0xffffffffu, m, 2);
      if (tq == 0) cmask[r] = m;
    }
    __syncthreads();
    // exact R16 distances of the candidates, increasing c
    if (tid < kMmaRows) {
      const long long i = row0 + tid;
      if (i < n) {
        unsigned long long m = cmask[tid];
        if (m == 0ull) m = (K >= 64) ? ~0ull : ((1ull << K) - 1ull);
        double best = 0.0;
        int bl = -1;
        while (m) {
          const int c = __ffsll((long long)m) - 1;
          m &= m - 1;
          double a = 0.0;
          for (int d = 0; d < dim; ++d) {
            const double t = __dsub_rn(As[d * kMmaAS + tid], Bs[d * kMmaBS + c]);
            a = __dadd_rn(a, __dmul_rn(t, t));
          }
          if (bl < 0 || a < best) {
            best = a;
            bl = c;
          }
        }
        if (old_labels && old_labels[i] != bl) ++ch;
        labels[i] = bl;
        dist[i] = best;
      }
    }
    __syncthreads();  // As / cmask reused by the next tile
  }
  if (changes) {
    ch = __reduce_add_sync(0xffffffffu, ch);
    if (lane == 0 && ch) atomicAdd(changes, ch);
  }
}

// dist_i = |h_i - mu_{label_i}|^2
template <int DP>
__global__ void __launch_bounds__(256) k_dist_own(const double* X, long long ld, const double* s, int n, int dim,
                                                  const double* mu, const int* labels, double* dist) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double h[DP];
    load_row<DP>(X, ld, s, i, dim, h);
    dist[i] = sqdist<DP>(h, mu + labels[i] * dim, dim);
  }
}

// per-CTA cluster sums and counts: partials[b][K*dim + K].  One CTA per SM over a
// contiguous row range, staged R rows at a time (cp.async, double-buffered;
// consecutive threads read consecutive rows of a column).  Thread t owns column
// c = t mod 64 (columns 0..dim-1 = coordinates, column dim = the count) of row
// quarter q = t / 64 and adds that quarter's rows of each tile, in row order, into
// the quarter's private accumulator; the four accumulators are combined in fixed
// order.  Every sum is therefore in a fixed order, independent of timing.
// Q row groups, 64 Q threads: thread (column c, group q).  Q = 4 with up to 128-row tiles (Q = 8 with
// 64-row tiles measured slower at config 4: 0.83 vs 0.71 ms).
inline size_t cp_smem_qr(int K, int dim, int Q, int R) {
  return sizeof(double) * ((size_t)Q * (K * dim + K) + 2 * (size_t)(dim + 1) * (R + 1)) + sizeof(int) * 2 * R;
}
inline void cp_config(int K, int dim, int* Q, int* R) {
  *Q = 4;
  *R = 128;
  while (*R > 32 && cp_smem_qr(K, dim, 4, *R) > 220 * 1024) *R /= 2;
}
template <int DP>
__global__ void __launch_bounds__(512) k_centroid_partials(const double* X, long long ld, const double* s, int n,
                                                           int dim, int K, int Q, int R, const int* labels,
                                                           double* partials) {
  extern __shared__ double acc[];  // [Q][W], tiles [2][dim + 1][R + 1] (row dim = s), labels [2][R]
  const int RP = R + 1;             // padded column stride: lanes on consecutive columns hit different banks
  const int W = K * dim + K;
  const int NT = blockDim.x;        // 64 Q
  double* tiles = acc + (size_t)Q * W;
  int* tl = reinterpret_cast<int*>(tiles + 2 * (size_t)(dim + 1) * RP);
  for (int e = threadIdx.x; e < Q * W; e += NT) acc[e] = 0.0;
  const long long i0 = (long long)n * blockIdx.x / gridDim.x, i1 = (long long)n * (blockIdx.x + 1) / gridDim.x;
  const int ntiles = (int)((i1 - i0 + R - 1) / R);
  auto prefetch = [&](int t) {
    if (t < ntiles) {
      double* tb = tiles + (size_t)(t & 1) * (dim + 1) * RP;
      int* lb = tl + (t & 1) * R;
      const long long r0 = i0 + (long long)t * R;
      const int ncol = dim + (s ? 1 : 0);
      const int r = threadIdx.x & (R - 1), dstep = NT / R;  // R: power of two <= NT
      if (r0 + r < i1)
        for (int d = threadIdx.x / R; d < ncol; d += dstep)
          cp_async8(tb + (size_t)d * RP + r, d < dim ? X + (long long)d * ld + r0 + r : s + r0 + r);
      for (int r = threadIdx.x; r < R; r += NT)
        if (r0 + r < i1) cp_async4(lb + r, labels + r0 + r);
    }
    cp_commit();
  };
  prefetch(0);
  const int c = threadIdx.x & 63, q = threadIdx.x >> 6, RQ = R / Q;
  double* a = acc + (size_t)q * W;
  for (int t = 0; t < ntiles; ++t) {
    prefetch(t + 1);
    cp_wait<1>();
    __syncthreads();
    const double* tb = tiles + (size_t)(t & 1) * (dim + 1) * RP;
    const int* lb = tl + (t & 1) * R;
    const int nr = (int)min((long long)R, i1 - (i0 + (long long)t * R));
    const int ra = q * RQ, rb = min(nr, ra + RQ);
    for (int cc = c; cc <= dim; cc += 64) {
      // column dim is the count: value 1, address K*dim + label
      const double* col = tb + (size_t)min(cc, dim - 1) * RP;
      const double* sv = tb + (size_t)dim * RP;
      const int mul = cc < dim ? dim : 1, off = cc < dim ? cc : K * dim;
      int r = ra;
      for (; r + 4 <= rb; r += 4) {  // operands loaded first; the four updates stay in row order
        double v[4];
        double* p[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          v[u] = cc < dim ? (s ? __dmul_rn(sv[r + u], col[r + u]) : col[r + u]) : 1.0;
          p[u] = a + lb[r + u] * mul + off;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) *p[u] += v[u];
      }
      for (; r < rb; ++r) a[lb[r] * mul + off] += cc < dim ? (s ? __dmul_rn(sv[r], col[r]) : col[r]) : 1.0;
    }
    __syncthreads();
  }
  cp_wait<0>();
  __syncthreads();
  for (int e = threadIdx.x; e < W; e += NT) {
    double v = acc[e];
    for (int g = 1; g < Q; ++g) v += acc[(size_t)g * W + e];  // fixed order
    partials[(size_t)blockIdx.x * W + e] = v;
  }
}

// ---- incremental centroid sums (Lloyd iterations where few labels change) ----
// Changed rows per 128-row tile, in row order: cnt[t], idx[128 t + j].
constexpr int kDT = 128;
__global__ void __launch_bounds__(kDT) k_changed_slots(const int* lab_old, const int* lab_new, int n, int* cnt,
                                                       int* idx) {
  __shared__ int wc[kDT / 32];
  const int t = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long i = (long long)t * kDT + threadIdx.x;
  const bool chg = i < n && lab_old[i] != lab_new[i];
  const unsigned m = __ballot_sync(0xffffffffu, chg);
  if (lane == 0) wc[w] = __popc(m);
  __syncthreads();
  int base = 0;
  for (int q = 0; q < w; ++q) base += wc[q];
  if (chg) idx[(size_t)t * kDT + base + __popc(m & ((1u << lane) - 1u))] = (int)i;
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int q = 0; q < kDT / 32; ++q) tot += wc[q];
    cnt[t] = tot;
  }
}
// Per-CTA delta of the cluster sums and counts over the changed rows of a contiguous tile range, in row
// order: sums[new] += [h_i, 1], sums[old] -= [h_i, 1] (column owners, fixed order).  partials[b][K dim + K].
constexpr int kDeltaThreads = 256, kDeltaTilesPerRound = 256, kDeltaSub = 64;
inline size_t delta_smem(int K, int dim) {
  return sizeof(double) * ((size_t)K * dim + K + (size_t)kDeltaSub * (dim + 1)) +
         sizeof(int) * ((size_t)kDeltaTilesPerRound * kDT + kDeltaTilesPerRound + 2 * kDeltaSub + 64);
}
__global__ void __launch_bounds__(kDeltaThreads) k_centroid_delta(const double* X, long long ld, const double* s, int n,
                                                                   int dim, int K, const int* lab_old,
                                                                   const int* lab_new, const int* cnt, const int* idx,
                                                                   double* partials) {
  extern __shared__ __align__(16) double dacc[];  // [K dim + K] | h [kDeltaSub][dim + 1] | ints
  const int W = K * dim + K;
  double* hb = dacc + W;
  int* list = reinterpret_cast<int*>(hb + (size_t)kDeltaSub * (dim + 1));
  int* tofs = list + kDeltaTilesPerRound * kDT;
  int* lo = tofs + kDeltaTilesPerRound;
  int* ln = lo + kDeltaSub;
  int* misc = ln + kDeltaSub;
  for (int e = threadIdx.x; e < W; e += blockDim.x) dacc[e] = 0.0;
  const int T = (n + kDT - 1) / kDT;
  const int t0 = (int)((long long)T * blockIdx.x / gridDim.x), t1 = (int)((long long)T * (blockIdx.x + 1) / gridDim.x);
  for (int r0 = t0; r0 < t1; r0 += kDeltaTilesPerRound) {
    const int nt = min(kDeltaTilesPerRound, t1 - r0);
    __syncthreads();
    if (threadIdx.x == 0) {  // exclusive offsets of the round's tiles (serial: <= 256 small adds)
      int acc = 0;
      for (int q = 0; q < nt; ++q) {
        tofs[q] = acc;
        acc += cnt[r0 + q];
      }
      misc[0] = acc;
    }
    __syncthreads();
    const int total = misc[0];
    for (int q = threadIdx.x; q < nt; q += blockDim.x) {
      const int c = cnt[r0 + q], o = tofs[q];
      for (int j = 0; j < c; ++j) list[o + j] = idx[(size_t)(r0 + q) * kDT + j];
    }
    __syncthreads();
    for (int b0 = 0; b0 < total; b0 += kDeltaSub) {
      const int nb = min(kDeltaSub, total - b0);
      for (int e = threadIdx.x; e < nb * dim; e += blockDim.x) {
        const int j = e / dim, d = e - j * dim;
        const int i = list[b0 + j];
        const double x = X[(long long)d * ld + i];
        hb[j * (dim + 1) + d] = s ? __dmul_rn(s[i], x) : x;
      }
      for (int j = threadIdx.x; j < nb; j += blockDim.x) {
        const int i = list[b0 + j];
        lo[j] = lab_old[i];
        ln[j] = lab_new[i];
      }
      __syncthreads();
      const int c = threadIdx.x;
      if (c < dim) {
        for (int j = 0; j < nb; ++j) {
          const double v = hb[j * (dim + 1) + c];
          dacc[ln[j] * dim + c] += v;
          dacc[lo[j] * dim + c] -= v;
        }
      } else if (c == dim) {
        for (int j = 0; j < nb; ++j) {
          dacc[K * dim + ln[j]] += 1.0;
          dacc[K * dim + lo[j]] -= 1.0;
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < W; e += blockDim.x) partials[(size_t)blockIdx.x * W + e] = dacc[e];
}
__global__ void k_add_sums(double* sums, const double* delta, int W) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < W; e += gridDim.x * blockDim.x) sums[e] += delta[e];
}

// ---- bound-pruned assignment (Hamerly's bounds, made exact) ----
// Per row: ub >= the true distance to the assigned centroid, lb <= the true distance to every other one
// (true = exact arithmetic on the stored centroids).  A centroid that moved by delta_c loosens them:
// ub += delta_a, lb -= max_{c != a} delta_c.  If ub (1 + eta) < lb (1 - eta), the assigned centroid is
// strictly nearest by a relative margin far above the rounding of the R16 distance sum, so the direct
// evaluation would return the same label: the row is skipped.  Other rows are evaluated directly over all
// centroids (R16 arithmetic, ties to the lowest index) and get fresh bounds.
constexpr double kEta = 1e-12;
__global__ void k_shift(const double* mu, const double* mu_old, int K, int dim, double* shift) {
  __shared__ double sh[64];
  const int c = threadIdx.x;
  if (c < K) {
    double a = 0.0;
    for (int d = 0; d < dim; ++d) {
      const double t = mu[c * dim + d] - mu_old[c * dim + d];
      a += t * t;
    }
    sh[c] = sqrt(a) * (1.0 + kEta) + 1e-300;  // >= the true shift
    shift[c] = sh[c];
  }
  __syncthreads();
  if (c == 0) {
    double m1 = 0.0, m2 = 0.0;
    int am = -1;
    for (int q = 0; q < K; ++q) {
      if (sh[q] > m1) {
        m2 = m1;
        m1 = sh[q];
        am = q;
      } else if (sh[q] > m2) {
        m2 = sh[q];
      }
    }
    shift[K] = m1;
    shift[K + 1] = m2;
    shift[K + 2] = (double)am;
  }
}
// prune test per row; rows that need an evaluation are listed per 128-row tile in row order (force: all)
__global__ void __launch_bounds__(kDT) k_prune_test(const int* lab_old, int* lab_new, double* ub, double* lb, int n,
                                                    int K, const double* shift, int force, int* cnt, int* idx) {
  __shared__ int wc[kDT / 32];
  const int t = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long i = (long long)t * kDT + threadIdx.x;
  bool need = false;
  if (i < n) {
    need = true;
    if (!force) {
      const int a = lab_old[i];
      const int am = (int)shift[K + 2];
      const double u = ub[i] + shift[a];
      const double l = lb[i] - (a == am ? shift[K + 1] : shift[K]);
      if (l > 0.0 && u * (1.0 + kEta) < l * (1.0 - kEta)) {
        need = false;
        lab_new[i] = a;
        ub[i] = u;
        lb[i] = l;
      }
    }
  }
  const unsigned m = __ballot_sync(0xffffffffu, need);
  if (lane == 0) wc[w] = __popc(m);
  __syncthreads();
  int base = 0;
  for (int q = 0; q < w; ++q) base += wc[q];
  if (need) idx[(size_t)t * kDT + base + __popc(m & ((1u << lane) - 1u))] = (int)i;
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int q = 0; q < kDT / 32; ++q) tot += wc[q];
    cnt[t] = tot;
  }
}
// direct R16 evaluation of the listed rows (all centroids): label, dist, fresh bounds
constexpr int kEvalTilesPerRound = 64;
inline size_t eval_smem(int K, int dim) {
  return sizeof(double) * (size_t)K * ((dim + 1) & ~1) + sizeof(int) * ((size_t)kEvalTilesPerRound * kDT + 64 + 8);
}
template <int DP>
__global__ void __launch_bounds__(256) k_eval_listed(const double* X, long long ld, const double* s, int n, int dim,
                                                     int K, const double* mu, const int* old_labels, int* labels,
                                                     double* dist, double* ub, double* lb, const int* cnt,
                                                     const int* idx, int* changes) {
  extern __shared__ __align__(16) double smu[];  // [K][dimp] | list | tile offsets
  const int dimp = (dim + 1) & ~1;
  int* list = reinterpret_cast<int*>(smu + (size_t)K * dimp);
  int* tofs = list + kEvalTilesPerRound * kDT;
  for (int e = threadIdx.x; e < K * dimp; e += blockDim.x) {
    const int c = e / dimp, d = e - c * dimp;
    smu[e] = d < dim ? mu[c * dim + d] : 0.0;
  }
  const int T = (n + kDT - 1) / kDT;
  const int t0 = (int)((long long)T * blockIdx.x / gridDim.x), t1 = (int)((long long)T * (blockIdx.x + 1) / gridDim.x);
  int ch = 0;
  for (int r0 = t0; r0 < t1; r0 += kEvalTilesPerRound) {
    const int nt = min(kEvalTilesPerRound, t1 - r0);
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int q = 0; q < nt; ++q) {
        tofs[q] = acc;
        acc += cnt[r0 + q];
      }
      tofs[64] = acc;
    }
    __syncthreads();
    const int total = tofs[64];
    for (int q = threadIdx.x; q < nt; q += blockDim.x) {
      const int c = cnt[r0 + q], o = tofs[q];
      for (int j = 0; j < c; ++j) list[o + j] = idx[(size_t)(r0 + q) * kDT + j];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < total; j += blockDim.x) {
      const int i = list[j];
      double h[DP];
      load_row<DP>(X, ld, s, i, dim, h);
      double best = 0.0, second = INFINITY;
      int bl = 0;
      for (int c0 = 0; c0 < K; c0 += 4) {
        double a[4];
        const double* m[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a[u] = 0.0;
          m[u] = smu + min(c0 + u, K - 1) * dimp;
        }
#pragma unroll
        for (int d = 0; d < DP; d += 2)
          if (d < dim) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double2 q = *reinterpret_cast<const double2*>(m[u] + d);
              const double e0 = __dsub_rn(h[d], q.x);
              a[u] = __dadd_rn(a[u], __dmul_rn(e0, e0));
              if (d + 1 < dim) {
                const double e1 = __dsub_rn(h[d + 1], q.y);
                a[u] = __dadd_rn(a[u], __dmul_rn(e1, e1));
              }
            }
          }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (c0 + u < K) {
            if (c0 + u == 0 || a[u] < best) {
              if (c0 + u > 0) second = fmin(second, best);
              best = a[u];
              bl = c0 + u;
            } else {
              second = fmin(second, a[u]);
            }
          }
      }
      if (old_labels && old_labels[i] != bl) ++ch;
      labels[i] = bl;
      dist[i] = best;
      ub[i] = sqrt(best) * (1.0 + kEta);
      lb[i] = K > 1 ? sqrt(second) * (1.0 - kEta) : INFINITY;
    }
  }
  if (changes) {
    ch = __reduce_add_sync(0xffffffffu, ch);
    if ((threadIdx.x & 31) == 0 && ch) atomicAdd(changes, ch);
  }
}

__global__ void k_means_div(const double* sums, int K, int dim, double* mu) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < K * dim; e += gridDim.x * blockDim.x) {
    const double cnt = sums[K * dim + e / dim];
    if (cnt > 0) mu[e] = sums[e] / cnt;
  }
}

// per-block (max value, lowest index) of dist excluding `used` indices
__global__ void k_argmax(const double* dist, int n, const int* used, int nused, double* bval, int* bidx) {
  __shared__ double sv[256];
  __shared__ int si[256];
  double best = -1.0;
  int bi = n;
  const int i0 = blockIdx.x * kBlk, i1 = min(n, i0 + kBlk);
  for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    bool ex = false;
    for (int u = 0; u < nused; ++u) ex |= (used[u] == i);
    const double v = ex ? -1.0 : dist[i];
    if (v > best || (v == best && i < bi)) {
      best = v;
      bi = i;
    }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      const double v = sv[threadIdx.x + st];
      const int ii = si[threadIdx.x + st];
      if (v > sv[threadIdx.x] || (v == sv[threadIdx.x] && ii < si[threadIdx.x])) {
        sv[threadIdx.x] = v;
        si[threadIdx.x] = ii;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bval[blockIdx.x] = sv[0];
    bidx[blockIdx.x] = si[0];
  }
}

__global__ void k_sum_blocks(const double* x, int n, double* blocksum) {
  __shared__ double red[8];
  double part = 0.0;
  const int i0 = blockIdx.x * kBlk, i1 = min(n, i0 + kBlk);
  for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) part += x[i];
  part = warp_sum(part);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    blocksum[blockIdx.x] = t;
  }
}

// Philox4x32-10 on the host (the library's own copy; the oracle has another)
inline void philox_host(unsigned c[4], unsigned k0, unsigned k1) {
  const unsigned M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const unsigned long long p0 = (unsigned long long)M0 * c[0], p1 = (unsigned long long)M1 * c[2];
    const unsigned hi0 = (unsigned)(p0 >> 32), lo0 = (unsigned)p0, hi1 = (unsigned)(p1 >> 32), lo1 = (unsigned)p1;
    const unsigned n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}
inline double uniform_host(uint64_t seed, unsigned c0, unsigned c1, unsigned c2) {
  unsigned c[4] = {c0, c1, c2, 0u};
  philox_host(c, (unsigned)seed, (unsigned)(seed >> 32));
  return ((double)(c[0] >> 5) * 67108864.0 + (double)(c[1] >> 6)) / 9007199254740992.0;
}

struct KmBuf {
  int n = 0, K = 0, G = 0, nblk = 0;
  double *D2 = nullptr, *bsum = nullptr, *mu = nullptr, *dist = nullptr, *partials = nullptr, *sums = nullptr;
  double* dsum = nullptr;               // delta of the sums (incremental iterations)
  double *ub = nullptr, *lb = nullptr, *mu_old = nullptr, *shift = nullptr;  // pruned assignment
  int *tcnt = nullptr, *tidx = nullptr;  // changed rows per 128-row tile
  double* bval = nullptr;
  int *lab = nullptr, *lab2 = nullptr, *best = nullptr, *idx = nullptr, *changes = nullptr, *bidx = nullptr,
      *used = nullptr;
};
void km_free(void* p) {
  KmBuf* b = static_cast<KmBuf*>(p);
  void* ptrs[] = {b->D2, b->bsum, b->mu, b->dist, b->partials, b->sums, b->bval, b->lab, b->lab2, b->best, b->idx,
                  b->changes, b->bidx, b->used, b->dsum, b->tcnt, b->tidx, b->ub, b->lb, b->mu_old, b->shift};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  delete b;
}

#define KCU(expr)                                                         \
  do {                                                                    \
    cudaError_t e_ = (expr);                                              \
    if (e_ != cudaSuccess)                                                \
      return ctx_fail(e_ == cudaErrorMemoryAllocation ? SFAIRSC_E_OOM : SFAIRSC_E_CUDA, cudaGetErrorString(e_)); \
  } while (0)

#define TRY_(e)                      \
  do {                               \
    sfairsc_status s_ = (e);         \
    if (s_ != SFAIRSC_OK) return s_; \
  } while (0)

template <int DP>
struct KM {
  const double* X;
  long long ld;
  const double* s;
  int n, dim, K, sms;
  cudaStream_t st;
  KmBuf* b;

  int grid_rows() const { return std::max(1, std::min((n + 255) / 256, sms * 8)); }
  void assign(const int* old_lab, int* new_lab, int* changes) {
    if (g_km_mma) {  // tensor-core distances with the exact guard (same labels)
      k_assign_mma<<<std::max(1, std::min((n + kMmaRows - 1) / kMmaRows, 2 * sms)), 256, asg_mma_smem(dim), st>>>(
          X, ld, s, n, dim, K, b->mu, old_lab, new_lab, b->dist, changes);
      return;
    }
    constexpr int NW = asg_warps<DP>();
    k_assign<DP, 4><<<grid_asg(), NW * 32, asg_smem(K, dim, NW), st>>>(X, ld, s, n, dim, K, b->mu, old_lab, new_lab,
                                                                     b->dist, changes);
  }
  // bound-pruned assignment: force = evaluate every row (bounds initialisation)
  void assign_pruned(const int* old_lab, int* new_lab, int* changes, bool force) {
    const int T = (n + kDT - 1) / kDT;
    if (!force) {
      bump_launch();
      k_shift<<<1, 64, 0, st>>>(b->mu, b->mu_old, K, dim, b->shift);
    }
    bump_launch();
    k_prune_test<<<T, kDT, 0, st>>>(old_lab ? old_lab : new_lab, new_lab, b->ub, b->lb, n, K, b->shift,
                                    force ? 1 : 0, b->tcnt, b->tidx);
    bump_launch();
    k_eval_listed<DP><<<std::max(1, std::min(T, sms)), 256, eval_smem(K, dim), st>>>(
        X, ld, s, n, dim, K, b->mu, old_lab, new_lab, b->dist, b->ub, b->lb, b->tcnt, b->tidx, changes);
  }
  int grid_asg() const { return std::max(1, std::min((n + 255) / 256, sms)); }

  sfairsc_status seed_centers(uint64_t seed, int r, std::vector<double>& hb) {
    const double u0 = uniform_host(seed, 0u, (unsigned)r, (unsigned)kKmStream);
    int idx = std::min((int)std::floor(u0 * n), n - 1);
    for (int t = 0; t < K; ++t) {
      if (t > 0) {
        KCU(cudaMemcpyAsync(hb.data(), b->bsum, sizeof(double) * b->nblk, cudaMemcpyDeviceToHost, st));
        KCU(cudaStreamSynchronize(st));
        double total = 0.0;
        for (int q = 0; q < b->nblk; ++q) total += hb[q];
        const double u = uniform_host(seed, (unsigned)t, (unsigned)r, (unsigned)kKmStream);
        if (total > 0) {
          const double target = u * total;
          double base = 0.0;
          int bsel = b->nblk - 1;
          for (int q = 0; q < b->nblk; ++q) {
            if (base + hb[q] > target) {
              bsel = q;
              break;
            }
            base += hb[q];
          }
          bump_launch();
          k_select_in_block<<<1, 32, 0, st>>>(b->D2, bsel, n, base, target, b->idx);
          int hidx = 0;
          KCU(cudaMemcpyAsync(&hidx, b->idx, sizeof(int), cudaMemcpyDeviceToHost, st));
          KCU(cudaStreamSynchronize(st));
          idx = hidx;
        } else {
          idx = std::min((int)std::floor(u * n), n - 1);
        }
      }
      bump_launch();
      k_gather_row<<<1, 64, 0, st>>>(X, ld, s, idx, dim, b->mu + (size_t)t * dim);
      bump_launch();
      k_d2<DP><<<b->nblk, 256, 0, st>>>(X, ld, s, n, dim, b->mu + (size_t)t * dim, t == 0, b->D2, b->bsum);
    }
    KCU(cudaGetLastError());
    return SFAIRSC_OK;
  }

  sfairsc_status means(const int* lab) {
    const int W = K * dim + K;
    bump_launch();
    int Q = 4, R = 128;
    cp_config(K, dim, &Q, &R);
    k_centroid_partials<DP><<<b->G, 64 * Q, cp_smem_qr(K, dim, Q, R), st>>>(X, ld, s, n, dim, K, Q, R, lab,
                                                                           b->partials);
    launch_reduce_cols(b->partials, b->G, W, b->sums, st);
    bump_launch();
    k_means_div<<<std::max(1, (K * dim + 255) / 256), 256, 0, st>>>(b->sums, K, dim, b->mu);
    KCU(cudaGetLastError());
    return SFAIRSC_OK;
  }

  // sums(lab) = sums(prev) + delta(prev -> lab), then mu (few changed labels: the changed rows only)
  sfairsc_status means_delta(const int* prev, const int* lab) {
    const int W = K * dim + K;
    const int T = (n + kDT - 1) / kDT;
    bump_launch();
    k_changed_slots<<<T, kDT, 0, st>>>(prev, lab, n, b->tcnt, b->tidx);
    bump_launch();
    k_centroid_delta<<<b->G, kDeltaThreads, delta_smem(K, dim), st>>>(X, ld, s, n, dim, K, prev, lab, b->tcnt,
                                                                      b->tidx, b->partials);
    launch_reduce_cols(b->partials, b->G, W, b->dsum, st);
    bump_launch();
    k_add_sums<<<std::max(1, (W + 255) / 256), 256, 0, st>>>(b->sums, b->dsum, W);
    bump_launch();
    k_means_div<<<std::max(1, (K * dim + 255) / 256), 256, 0, st>>>(b->sums, K, dim, b->mu);
    KCU(cudaGetLastError());
    return SFAIRSC_OK;
  }

  sfairsc_status run(uint64_t seed, int restarts, int max_iters, double* best_wcss) {
    std::vector<double> hb(std::max(b->nblk, K) + 8);
    std::vector<double> counts(K);
    std::vector<int> bidx(b->nblk);
    std::vector<double> bval(b->nblk);
    *best_wcss = std::numeric_limits<double>::infinity();
    for (int r = 0; r < restarts; ++r) {
      TRY_(seed_centers(seed, r, hb));
      bump_launch();
      if (g_km_prune) assign_pruned(nullptr, b->lab, nullptr, true);
      else assign(nullptr, b->lab, nullptr);
      int* lab = b->lab;
      int* lab_new = b->lab2;
      int last_ch = n, since_full = 0;
      for (int it = 0; it < max_iters; ++it) {
        // cluster sums: full recomputation on the first iteration, every kKmRefresh-th, and after many changes;
        // otherwise the previous sums plus the changed rows' contributions (lab_new holds the previous labels)
        if (g_km_prune) KCU(cudaMemcpyAsync(b->mu_old, b->mu, sizeof(double) * K * dim, cudaMemcpyDeviceToDevice, st));
        if (!g_km_incr || it == 0 || since_full + 1 >= kKmRefresh || (long long)last_ch * 16 > n) {
          TRY_(means(lab));
          since_full = 0;
        } else {
          TRY_(means_delta(lab_new, lab));
          ++since_full;
        }
        KCU(cudaMemcpyAsync(counts.data(), b->sums + (size_t)K * dim, sizeof(double) * K, cudaMemcpyDeviceToHost, st));
        KCU(cudaStreamSynchronize(st));
        bool any_empty = false;
        for (int c2 = 0; c2 < K; ++c2) any_empty |= counts[c2] == 0;
        if (any_empty) {  // re-seed empty clusters at the farthest points (increasing c)
          bump_launch();
          k_dist_own<DP><<<grid_rows(), 256, 0, st>>>(X, ld, s, n, dim, b->mu, lab, b->dist);
          std::vector<int> used;
          for (int c2 = 0; c2 < K; ++c2) {
            if (counts[c2] != 0) continue;
            if (!used.empty())
              KCU(cudaMemcpyAsync(b->used, used.data(), sizeof(int) * used.size(), cudaMemcpyHostToDevice, st));
            bump_launch();
            k_argmax<<<b->nblk, 256, 0, st>>>(b->dist, n, b->used, (int)used.size(), b->bval, b->bidx);
            KCU(cudaMemcpyAsync(bval.data(), b->bval, sizeof(double) * b->nblk, cudaMemcpyDeviceToHost, st));
            KCU(cudaMemcpyAsync(bidx.data(), b->bidx, sizeof(int) * b->nblk, cudaMemcpyDeviceToHost, st));
            KCU(cudaStreamSynchronize(st));
            double bv = -2.0;
            int bi = n;
            for (int q = 0; q < b->nblk; ++q)
              if (bval[q] > bv || (bval[q] == bv && bidx[q] < bi)) {
                bv = bval[q];
                bi = bidx[q];
              }
            used.push_back(bi);
            bump_launch();
            k_gather_row<<<1, 64, 0, st>>>(X, ld, s, bi, dim, b->mu + (size_t)c2 * dim);
          }
        }
        KCU(cudaMemsetAsync(b->changes, 0, sizeof(int), st));
        bump_launch();
        if (g_km_prune) assign_pruned(lab, lab_new, b->changes, false);
        else assign(lab, lab_new, b->changes);
        int ch = 0;
        KCU(cudaMemcpyAsync(&ch, b->changes, sizeof(int), cudaMemcpyDeviceToHost, st));
        KCU(cudaStreamSynchronize(st));
        if (g_km_debug && (it < 10 || it % 25 == 0))
          fprintf(stderr, "[sfairsc] kmeans restart %d iteration %d: %d labels changed\n", r, it, ch);
        if (ch == 0) break;
        last_ch = ch;
        std::swap(lab, lab_new);
      }
      // final centroids of the final labels, WCSS
      TRY_(means(lab));
      bump_launch();
      k_dist_own<DP><<<grid_rows(), 256, 0, st>>>(X, ld, s, n, dim, b->mu, lab, b->dist);
      bump_launch();
      k_sum_blocks<<<b->nblk, 256, 0, st>>>(b->dist, n, b->bsum);
      KCU(cudaMemcpyAsync(hb.data(), b->bsum, sizeof(double) * b->nblk, cudaMemcpyDeviceToHost, st));
      KCU(cudaStreamSynchronize(st));
      double wcss = 0.0;
      for (int q = 0; q < b->nblk; ++q) wcss += hb[q];
      if (wcss < *best_wcss) {
        *best_wcss = wcss;
        KCU(cudaMemcpyAsync(b->best, lab, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
      }
    }
    KCU(cudaStreamSynchronize(st));
    return SFAIRSC_OK;
  }
};

}  // namespace

sfairsc_status kmeans_run(sfairsc_ctx* ctx, uint64_t seed, int32_t* labels_out, int32_t memspace, double* objective) {
  if (getenv("SFAIRSC_KM_MMA")) g_km_mma = atoi(getenv("SFAIRSC_KM_MMA"));
  g_km_debug = getenv("SFAIRSC_DEBUG") ? atoi(getenv("SFAIRSC_DEBUG")) : 0;
  if (getenv("SFAIRSC_KM_INCR")) g_km_incr = atoi(getenv("SFAIRSC_KM_INCR"));
  if (getenv("SFAIRSC_KM_PRUNE")) g_km_prune = atoi(getenv("SFAIRSC_KM_PRUNE"));
  const int n = ctx_n(ctx), K = ctx_k(ctx);
  long long ld = 0;
  const double* X = ctx_X(ctx, &ld);
  const double* s = ctx_s(ctx);
  const int dim = K;
  if (dim > kMaxDim) return ctx_fail(SFAIRSC_E_INVALID_ARG, "embed_kmeans supports k <= 64");
  cudaStream_t st = ctx_stream(ctx);
  void (*fr)(void*) = nullptr;
  void** slot = ctx_km(ctx, &fr);
  KmBuf* b = static_cast<KmBuf*>(*slot);
  if (!b || b->n != n || b->K != K) {
    if (b) km_free(b);
    b = new KmBuf();
    *slot = b;
    ctx_set_km_free(ctx, km_free);
    b->n = -1;  // set to (n, K) only once every buffer below is allocated: a failed call is never reused
    b->K = -1;
    b->nblk = (n + kBlk - 1) / kBlk;
    b->G = std::max(1, std::min(ctx_num_sms(ctx), (n + 1023) / 1024));  // one CTA per SM (shared memory)
    const int W = K * dim + K;
    KCU(cudaMalloc(&b->D2, sizeof(double) * n));
    KCU(cudaMalloc(&b->bsum, sizeof(double) * b->nblk));
    KCU(cudaMalloc(&b->mu, sizeof(double) * K * dim));
    KCU(cudaMalloc(&b->dist, sizeof(double) * n));
    KCU(cudaMalloc(&b->partials, sizeof(double) * (size_t)b->G * W));
    KCU(cudaMalloc(&b->sums, sizeof(double) * W));
    KCU(cudaMalloc(&b->dsum, sizeof(double) * W));
    KCU(cudaMalloc(&b->ub, sizeof(double) * n));
    KCU(cudaMalloc(&b->lb, sizeof(double) * n));
    KCU(cudaMalloc(&b->mu_old, sizeof(double) * K * dim));
    KCU(cudaMalloc(&b->shift, sizeof(double) * (K + 4)));
    KCU(cudaMalloc(&b->tcnt, sizeof(int) * ((n + kDT - 1) / kDT)));
    KCU(cudaMalloc(&b->tidx, sizeof(int) * (size_t)((n + kDT - 1) / kDT) * kDT));
    KCU(cudaMalloc(&b->bval, sizeof(double) * b->nblk));
    KCU(cudaMalloc(&b->lab, sizeof(int) * n));
    KCU(cudaMalloc(&b->lab2, sizeof(int) * n));
    KCU(cudaMalloc(&b->best, sizeof(int) * n));
    KCU(cudaMalloc(&b->idx, sizeof(int) * 4));
    KCU(cudaMalloc(&b->changes, sizeof(int) * 4));
    KCU(cudaMalloc(&b->bidx, sizeof(int) * b->nblk));
    KCU(cudaMalloc(&b->used, sizeof(int) * (K + 1)));
    b->n = n;
    b->K = K;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_assign_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)asg_mma_smem(64));
      cudaFuncSetAttribute(k_centroid_delta, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)delta_smem(64, 64));
      auto big = [](const void* f) { cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024); };
      big((const void*)k_eval_listed<8>);
      big((const void*)k_eval_listed<16>);
      big((const void*)k_eval_listed<32>);
      big((const void*)k_eval_listed<48>);
      big((const void*)k_eval_listed<56>);
      big((const void*)k_eval_listed<64>);
      big((const void*)k_centroid_partials<8>);
      big((const void*)k_centroid_partials<16>);
      big((const void*)k_centroid_partials<32>);
      big((const void*)k_centroid_partials<48>);
      big((const void*)k_centroid_partials<56>);
      big((const void*)k_centroid_partials<64>);
      big((const void*)k_assign<8, 4>);
      big((const void*)k_assign<16, 4>);
      big((const void*)k_assign<32, 4>);
      big((const void*)k_assign<48, 4>);
      big((const void*)k_assign<56, 4>);
      big((const void*)k_assign<64, 4>);
      attr = true;
    }
  }
  cudaEvent_t ev;
  ctx_prof_begin(ctx, &ev);
  double wcss = 0.0;
  sfairsc_status stt;
  const int sms = ctx_num_sms(ctx);
  if (dim <= 8) stt = KM<8>{X, ld, s, n, dim, K, sms, st, b}.run(seed, 10, 300, &wcss);
  else if (dim <= 16) stt = KM<16>{X, ld, s, n, dim, K, sms, st, b}.run(seed, 10, 300, &wcss);
  else if (dim <= 32) stt = KM<32>{X, ld, s, n, dim, K, sms, st, b}.run(seed, 10, 300, &wcss);
  else if (dim <= 48) stt = KM<48>{X, ld, s, n, dim, K, sms, st, b}.run(seed, 10, 300, &wcss);
  else if (dim <= 56) stt = KM<56>{X, ld, s, n, dim, K, sms, st, b}.run(seed, 10, 300, &wcss);
  else stt = KM<64>{X, ld, s, n, dim, K, sms, st, b}.run(seed, 10, 300, &wcss);
  ctx_prof_end(ctx, 8, ev);
  if (stt != SFAIRSC_OK) return stt;
  KCU(cudaMemcpyAsync(labels_out, b->best, sizeof(int) * n,
                      memspace == SFAIRSC_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  KCU(cudaStreamSynchronize(st));
  if (objective) *objective = wcss;
  return SFAIRSC_OK;
}

}  // namespace sfz
