// libsfairsc — sm_100a fp64 kernels for the s-FairSC hot path.
//
// The path:
//   apply  y = L^sigma w = P(L(P w)) - sigma P w + sigma w
//     gsum      b_w = B^T w                                       (A4, factored Q)
//     project   p   = w - s o gam(b_w)_g          = P w            (A4)
//     spmv      t   = L p,  epilogue b_t = B^T t                   (A5)
//     finish    y   = t - s o (gam(b_t) - sigma gam(b_w))_g        (A6, Eq. asigma)
//   Lanczos step (A7-A9): sweep0 (finish + V^T y), sweep1 (update + V^T r'),
//   sweep2 (update + |r''|^2 + B^T r''), normalize (v, p of the next apply);
//   restart (A10): ritz  V Y.
//
// All reductions are two-stage with a fixed partition and fixed order (no
// floating-point atomics), so results are bitwise reproducible per GPU.
#include "kernels.cuh"
#include "device_common.cuh"

#include <algorithm>
#include <atomic>
#include <cstdio>

namespace sfz {

static std::atomic<long long> g_nlaunch{0};
static inline void bump() { g_nlaunch.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_nlaunch.load(); }
void bump_launch() { bump(); }

static inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// ----------------------------------------------------------------------------
// build-time kernels (A0-A3)
// ----------------------------------------------------------------------------
enum { F_CSR = 1, F_NEG = 2, F_ASYM = 4, F_ISO = 8, F_GRP = 16, F_NONUNIT = 32 };

__global__ void k_validate(GraphDev g, int check_sym, int* flags) {
  const int n = g.n;
  int f = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (g.rp[0] != 0 || g.rp[n] != g.nnz) f |= F_CSR;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int a = g.rp[i], b = g.rp[i + 1];
    if (b < a || a < 0 || b > g.nnz) {
      f |= F_CSR;
      continue;
    }
    int prev = -1;
    for (int e = a; e < b; ++e) {
      const int j = g.ci[e];
      const double w = g.vv[e];
      if (j < 0 || j >= n || j <= prev) f |= F_CSR;
      prev = j;
      if (!(w >= 0.0)) f |= F_NEG;  // also NaN
      if (j == i && w != 0.0) f |= F_CSR;
      if (w != 1.0 || j == i) f |= F_NONUNIT;  // not a unit-weight pattern (informational)
      if (check_sym && j >= 0 && j < n && j != i) {
        // partner row j is not validated by this thread: clamp its range into [0, nnz) (a malformed row_ptr
        // is flagged by j's own thread; the search must not read outside ci)
        int lo = max(0, g.rp[j]), hi = min(g.nnz, g.rp[j + 1]) - 1, found = -1;
        while (lo <= hi) {
          const int mid = lo + ((hi - lo) >> 1);  // rp values reach 1.6e9: no lo + hi overflow
          const int cm = g.ci[mid];
          if (cm == i) {
            found = mid;
            break;
          }
          if (cm < i) lo = mid + 1; else hi = mid - 1;
        }
        if (found < 0 || g.vv[found] != w) f |= F_ASYM;
      }
    }
  }
  if (f) atomicOr(flags, f);
}

__global__ void k_degrees(GraphDev g, double* d, int* flags) {
  int f = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int e = g.rp[i]; e < g.rp[i + 1]; ++e) acc += g.vv[e];
    d[i] = acc;
    if (!(acc > 0.0)) f |= F_ISO;
  }
  if (f) atomicOr(flags, f);
}

__global__ void k_inv_sqrt(const double* d, double* s, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) s[i] = 1.0 / sqrt(d[i]);
}

__global__ void k_scale_vec(const double* __restrict__ s, const double* __restrict__ p, double* __restrict__ q, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) q[i] = s[i] * p[i];
}

__global__ void k_scale_values(const int* rp, const int* ci, double* vv, const double* s, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double si = s[i];
    for (int e = rp[i]; e < rp[i + 1]; ++e) vv[e] = si * vv[e] * s[ci[e]];
  }
}

// sigma = ||L||_1 = max_j sum_i |L_ij|.  By symmetry column j = row j:
// normalized  1 + sum_i s_j w_ji s_i ; unnormalized  2 d_j.
__global__ void k_sigma(GraphDev g, double* partials, unsigned* counter, double* out) {
  double mx = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) {
    double v;
    if (g.normalized) {
      double acc = 0.0;
      for (int e = g.rp[i]; e < g.rp[i + 1]; ++e) acc += g.vv[e];
      v = 1.0 + acc;
    } else {
      v = 2.0 * g.dg[i];
    }
    mx = fmax(mx, v);
  }
  __shared__ double red[kThreads];
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
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

__global__ void k_group_check(const int32_t* groups, int n, int h, uint8_t* grp, int* flags) {
  int f = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int v = groups[i];
    if (v < 0 || v >= h) f |= F_GRP;
    grp[i] = (uint8_t)v;
  }
  if (f) atomicOr(flags, f);
}

// ----------------------------------------------------------------------------
// factored-projector kernels (A4, A6)
// ----------------------------------------------------------------------------
template <bool NORM, bool DQ = false>
__global__ void __launch_bounds__(kThreads) k_gsum(GraphDev g, const double* __restrict__ x, int g_base,
                                                   double* partials, unsigned* counter, double* bsum, int nout) {
  double acc[kHB];
#pragma unroll
  for (int q = 0; q < kHB; ++q) acc[q] = 0.0;
  const int n = g.n;
  const int i0 = (int)((long long)n * blockIdx.x / gridDim.x), i1 = (int)((long long)n * (blockIdx.x + 1) / gridDim.x);
  for (int i = i0 + threadIdx.x; i < i1; i += kThreads) {
    if constexpr (DQ) {
      accum_row<true, NORM>(g, i, x[i], acc);
    } else {
      const double v = NORM ? g.s[i] * x[i] : x[i];
      add_group(acc, (int)g.grp[i] - g_base, v);
    }
  }
  block_reduce_store<kHB>(acc, partials + (size_t)blockIdx.x * kHB);
  ticket_finalize<kHB>(partials, counter, bsum + g_base, nout);
}

template <bool NORM, bool DQ = false>
__global__ void __launch_bounds__(kThreads) k_project(GraphDev g, ProjDesc pd, const double* __restrict__ x,
                                                      const double* bsum, double scale, double* __restrict__ p) {
  __shared__ double gam[256];
  if (threadIdx.x == 0) gamma_serial(bsum, scale, pd, gam);
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) {
    if constexpr (DQ) {
      p[i] = x[i] - proj_row<true, NORM>(g, i, gam);
    } else {
      const double gi = gam[g.grp[i]];
      p[i] = NORM ? fma(-g.s[i], gi, x[i]) : x[i] - gi;
    }
  }
}

template <bool NORM, bool DQ = false>
__global__ void __launch_bounds__(kThreads) k_finish(GraphDev g, ProjDesc pd, const double* __restrict__ t,
                                                     const double* bsum_t, const double* bsum_w, double sigma,
                                                     double* __restrict__ y) {
  __shared__ double gt[256], gw[256];
  if (threadIdx.x == 0) {
    gamma_serial(bsum_t, 1.0, pd, gt);
    gamma_serial(bsum_w, 1.0, pd, gw);
    for (int s = 0; s < pd.h; ++s) gt[s] = gt[s] - sigma * gw[s];
  }
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) {
    if constexpr (DQ) {
      y[i] = t[i] - proj_row<true, NORM>(g, i, gt);
    } else {
      const double gi = gt[g.grp[i]];
      y[i] = NORM ? fma(-g.s[i], gi, t[i]) : t[i] - gi;
    }
  }
}

// Chebyshev three-term step (§8(f) N2) fused into the apply's finish:
// y_new = a (finish(t) - cc y_cur) + b y_prev, finish(t) = L^sigma y_cur as in k_finish (group projector).
// y_new may alias y_prev (each element is read before it is written by the same thread).
template <bool NORM>
__global__ void __launch_bounds__(kThreads) k_finish_cheb(GraphDev g, ProjDesc pd, const double* __restrict__ t,
                                                          const double* bsum_t, const double* bsum_w, double sigma,
                                                          const double* __restrict__ ycur, const double* yprev,
                                                          double a, double cc, double b, double* ynew) {
  __shared__ double gt[256], gw[256];
  if (threadIdx.x == 0) {
    gamma_serial(bsum_t, 1.0, pd, gt);
    gamma_serial(bsum_w, 1.0, pd, gw);
    for (int s = 0; s < pd.h; ++s) gt[s] = gt[s] - sigma * gw[s];
  }
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) {
    const double gi = gt[g.grp[i]];
    const double ay = NORM ? fma(-g.s[i], gi, t[i]) : t[i] - gi;  // (L^sigma y_cur)_i
    const double r = a * fma(-cc, ycur[i], ay);
    ynew[i] = b != 0.0 ? fma(b, yprev[i], r) : r;
  }
}

// ----------------------------------------------------------------------------
// Krylov sweeps (A7-A9)
// ----------------------------------------------------------------------------
template <int MODE, int MAXCW, bool NORM, bool DQ = false>
__global__ void __launch_bounds__(kThreads) k_sweep(GraphDev g, ProjDesc pd, SweepArgs a) {
  __shared__ double xs[kThreads];
  __shared__ double coef[kMaxJ];
  __shared__ double gam[256];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int n = g.n, J = a.J;
  if (MODE == 1 || MODE == 2)
    for (int l = tid; l < J; l += kThreads) coef[l] = a.coef[l];
  if (MODE == 0 && tid == 0) {
    __shared__ double gw[256];
    gamma_serial(a.bsum_t, 1.0, pd, gam);
    gamma_serial(a.bsum_w, 1.0, pd, gw);
    for (int s = 0; s < pd.h; ++s) gam[s] = gam[s] - a.sigma * gw[s];
  }
  __syncthreads();
  const int nchunks = (n + kThreads - 1) / kThreads;
  const int c0 = (int)((long long)nchunks * blockIdx.x / gridDim.x);
  const int c1 = (int)((long long)nchunks * (blockIdx.x + 1) / gridDim.x);
  double colacc[MAXCW];
#pragma unroll
  for (int cc = 0; cc < MAXCW; ++cc) colacc[cc] = 0.0;
  double gacc[kHB];
#pragma unroll
  for (int q = 0; q < kHB; ++q) gacc[q] = 0.0;
  double nrm = 0.0;
  const long long ld = a.ld;
  for (int c = c0; c < c1; ++c) {
    const int i = c * kThreads + tid;
    double x = 0.0;
    if (i < n) {
      if (MODE == 0) {
        if constexpr (DQ) x = a.xin[i] - proj_row<true, NORM>(g, i, gam);
        else x = NORM ? fma(-g.s[i], gam[g.grp[i]], a.xin[i]) : a.xin[i] - gam[g.grp[i]];
        a.xout[i] = x;
      } else if (MODE == 3) {
        x = a.xin[i];
      } else {
        double acc = a.xin[i];
        const double* __restrict__ vp = a.V + i;
        int l = 0;
        for (; l + 8 <= J; l += 8) {
          double v0 = vp[(l + 0) * ld], v1 = vp[(l + 1) * ld], v2 = vp[(l + 2) * ld], v3 = vp[(l + 3) * ld];
          double v4 = vp[(l + 4) * ld], v5 = vp[(l + 5) * ld], v6 = vp[(l + 6) * ld], v7 = vp[(l + 7) * ld];
          acc = fma(-v0, coef[l + 0], acc);
          acc = fma(-v1, coef[l + 1], acc);
          acc = fma(-v2, coef[l + 2], acc);
          acc = fma(-v3, coef[l + 3], acc);
          acc = fma(-v4, coef[l + 4], acc);
          acc = fma(-v5, coef[l + 5], acc);
          acc = fma(-v6, coef[l + 6], acc);
          acc = fma(-v7, coef[l + 7], acc);
        }
        for (; l < J; ++l) acc = fma(-vp[l * ld], coef[l], acc);
        x = acc;
        a.xout[i] = x;
        if (MODE == 2) {
          nrm = fma(x, x, nrm);
          accum_row<DQ, NORM>(g, i, x, gacc);
        }
      }
    }
    if (MODE != 2) {
      xs[tid] = x;
      __syncthreads();
      const long long base = (long long)c * kThreads + lane;
#pragma unroll
      for (int cc = 0; cc < MAXCW; ++cc) {
        const int l = w + cc * (kThreads / 32);
        if (l < J) {
          const double* __restrict__ vp = a.V + (long long)l * ld + base;
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < kThreads / 32; ++q) s = fma(vp[q * 32], xs[lane + 32 * q], s);
          colacc[cc] += s;
        }
      }
      __syncthreads();
    }
  }
  if (MODE != 2) {
#pragma unroll
    for (int cc = 0; cc < MAXCW; ++cc) {
      const int l = w + cc * (kThreads / 32);
      if (l < J) {
        const double s = warp_sum(colacc[cc]);
        if (lane == 0) a.partials[(size_t)blockIdx.x * J + l] = s;
      }
    }
  } else {
    double v[1 + kHB];
    v[0] = nrm;
#pragma unroll
    for (int q = 0; q < kHB; ++q) v[1 + q] = gacc[q];
    block_reduce_store<1 + kHB>(v, a.partials + (size_t)blockIdx.x * (1 + kHB));
    ticket_finalize<1 + kHB>(a.partials, a.counter, a.norm_bsum, 1 + min(pd.h, kHB));
  }
}

__global__ void k_reduce_cols(const double* __restrict__ partials, int G, int J, double* out) {
  const int l = blockIdx.x;
  double acc = 0.0;
  for (int b = threadIdx.x; b < G; b += blockDim.x) acc += partials[(size_t)b * J + l];
  __shared__ double red[32];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    out[l] = s;
  }
}

// v_{j+1} = r / beta, p = P v_{j+1} (factored), B^T v_{j+1} = B^T r / beta.
// beta = sqrt(|r|^2) is taken from device memory (no host round trip); block 0
// records T entries alpha_j = c1[j] + c2[j], beta_j and flags a breakdown
// (beta <= bd_tol: invariant subspace, handled by the host at the next sync).
template <bool NORM>
__global__ void __launch_bounds__(kThreads) k_normalize(GraphDev g, ProjDesc pd, const double* __restrict__ r,
                                                        NormArgs na, double* __restrict__ v, double* bsum_v,
                                                        double* __restrict__ p) {
  __shared__ double gam[256];
  __shared__ double s_inv;
  if (threadIdx.x == 0) {
    double beta = na.beta_host > 0 ? na.beta_host : sqrt(na.nb[0]);
    if (na.alpha_dev) {
      if (blockIdx.x == 0) {
        na.alpha_dev[na.j] = na.c1[na.j] + na.c2[na.j];
        na.beta_dev[na.j] = beta;
        if (!(beta > na.bd_tol)) atomicOr(na.flag, 1);
      }
    }
    if (!(beta > na.bd_tol)) beta = 1.0;  // breakdown: column is garbage, rolled back by the host
    s_inv = 1.0 / beta;
    gamma_serial(na.nb + 1, s_inv, pd, gam);
  }
  __syncthreads();
  const double inv = s_inv;
  if (blockIdx.x == 0)
    for (int s = threadIdx.x; s < pd.h; s += blockDim.x) bsum_v[s] = na.nb[1 + s] * inv;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) {
    const double vi = r[i] * inv;
    v[i] = vi;
    const double gi = gam[g.grp[i]];
    p[i] = NORM ? fma(-g.s[i], gi, vi) : vi - gi;
  }
}

__global__ void k_random(double* x, int n, uint64_t seed, unsigned c1, unsigned stream) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    x[i] = philox_uniform(seed, (unsigned)i, c1, stream, 0u) - 0.5;
}

__global__ void __launch_bounds__(kThreads) k_resid(const double* __restrict__ y, const double* __restrict__ x,
                                                    double theta, const double* theta_dev, int n, double* partials,
                                                    unsigned* counter, double* out) {
  if (theta_dev) theta = *theta_dev;
  double v[1] = {0.0};
  const int i0 = (int)((long long)n * blockIdx.x / gridDim.x), i1 = (int)((long long)n * (blockIdx.x + 1) / gridDim.x);
  for (int i = i0 + threadIdx.x; i < i1; i += kThreads) {
    const double r = fma(-theta, x[i], y[i]);
    v[0] = fma(r, r, v[0]);
  }
  block_reduce_store<1>(v, partials + blockIdx.x);
  ticket_finalize<1>(partials, counter, out, 1);
}

// out = x^T y (ticket reduced)
__global__ void __launch_bounds__(kThreads) k_dot(const double* __restrict__ x, const double* __restrict__ y, int n,
                                                  double* partials, unsigned* counter, double* out) {
  double v[1] = {0.0};
  const int i0 = (int)((long long)n * blockIdx.x / gridDim.x), i1 = (int)((long long)n * (blockIdx.x + 1) / gridDim.x);
  for (int i = i0 + threadIdx.x; i < i1; i += kThreads) v[0] = fma(x[i], y[i], v[0]);
  block_reduce_store<1>(v, partials + blockIdx.x);
  ticket_finalize<1>(partials, counter, out, 1);
}

// ----------------------------------------------------------------------------
// Dense constraint basis (§8(f) N4): Q = orth(C) by CholQR2 (Gram on the device, Cholesky on the host)
// element (i, a) of an n x r matrix at M[i * rs + a * cs]
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_gram_pairs(const double* __restrict__ M, long long rs, long long cs,
                                                         int n, int r, double* out) {
  const int a = blockIdx.x, b = blockIdx.y;
  if (a > b) return;
  double v[1] = {0.0};
  for (int i = threadIdx.x; i < n; i += kThreads) v[0] = fma(M[i * rs + a * cs], M[i * rs + b * cs], v[0]);
  block_reduce_store<1>(v, out + a * r + b);  // upper triangle; the host mirrors it
}
// rows scaled by s (C = D^{-1/2} F): F col-major (ld) in place
__global__ void k_scale_rows(double* M, long long ld, int n, int r, const double* s) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int a = 0; a < r; ++a) M[(long long)a * ld + i] *= s[i];
}
// Qout[i, :] = Min[i, :] T (T: r x rq row-major, r <= 64, rq <= 16), Qout row-major (ldq; columns rq..ldq zeroed)
__global__ void k_rows_times(const double* __restrict__ Min, long long rs, long long cs, int n, int r, int rq,
                             const double* __restrict__ T, double* __restrict__ Qout, int ldq) {
  __shared__ double Ts[64 * 16];
  for (int e = threadIdx.x; e < r * rq; e += blockDim.x) Ts[e] = T[e];
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.0;
    for (int a = 0; a < r; ++a) {
      const double m = Min[(long long)i * rs + (long long)a * cs];
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < rq) acc[j] = fma(m, Ts[a * rq + j], acc[j]);
    }
    for (int j = 0; j < ldq; ++j) Qout[(long long)i * ldq + j] = j < rq ? acc[j] : 0.0;
  }
}
void launch_gram_pairs(const double* M, long long rs, long long cs, int n, int r, double* out, cudaStream_t st);
void launch_scale_rows(double* M, long long ld, int n, int r, const double* s, cudaStream_t st);
void launch_rows_times(const double* Min, long long rs, long long cs, int n, int r, int rq, const double* T,
                       double* Qout, int ldq, cudaStream_t st);

// ----------------------------------------------------------------------------
// launch wrappers
// ----------------------------------------------------------------------------
static int num_sms_cached() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}
static int stream_grid(int n) { return std::max(1, std::min(cdiv(n, kThreads), num_sms_cached() * 8)); }
static int reduce_grid(int n) { return std::max(1, std::min(cdiv(n, 4 * kThreads), num_sms_cached() * 2)); }

void launch_validate_csr(const GraphDev& g, int check_sym, int* flags, cudaStream_t st) {
  bump();
  k_validate<<<stream_grid(g.n), kThreads, 0, st>>>(g, check_sym, flags);
}
void launch_degrees(const GraphDev& g, double* d, int* flags, cudaStream_t st) {
  bump();
  k_degrees<<<stream_grid(g.n), kThreads, 0, st>>>(g, d, flags);
}
void launch_inv_sqrt(const double* d, double* s, int n, cudaStream_t st) {
  bump();
  k_inv_sqrt<<<stream_grid(n), kThreads, 0, st>>>(d, s, n);
}
void launch_scale_vec(const double* s, const double* p, double* q, int n, cudaStream_t st) {
  bump();
  k_scale_vec<<<stream_grid(n), kThreads, 0, st>>>(s, p, q, n);
}
void launch_scale_values(const int* rp, const int* ci, double* vv, const double* s, int n, cudaStream_t st) {
  bump();
  k_scale_values<<<stream_grid(n), kThreads, 0, st>>>(rp, ci, vv, s, n);
}
void launch_sigma(const GraphDev& g, double* partials, unsigned* counter, double* out, cudaStream_t st) {
  bump();
  k_sigma<<<reduce_grid(g.n), kThreads, 0, st>>>(g, partials, counter, out);
}
void launch_group_check(const int32_t* groups, int n, int h, uint8_t* grp, int* flags, cudaStream_t st) {
  bump();
  k_group_check<<<stream_grid(n), kThreads, 0, st>>>(groups, n, h, grp, flags);
}

void launch_gsum(const GraphDev& g, const double* x, int g_base, double* partials, unsigned* counter, double* bsum,
                 cudaStream_t st) {
  bump();
  // bsum points at the h-array base; groups [g_base, g_base+16) are written
  const int G = reduce_grid(g.n);
  const int nout = kHB;  // caller guarantees room for kHB entries past g_base
  if (g.Q) {
    if (g.normalized) k_gsum<true, true><<<G, kThreads, 0, st>>>(g, x, 0, partials, counter, bsum, nout);
    else k_gsum<false, true><<<G, kThreads, 0, st>>>(g, x, 0, partials, counter, bsum, nout);
    return;
  }
  if (g.normalized)
    k_gsum<true><<<G, kThreads, 0, st>>>(g, x, g_base, partials, counter, bsum, nout);
  else
    k_gsum<false><<<G, kThreads, 0, st>>>(g, x, g_base, partials, counter, bsum, nout);
}
void launch_project(const GraphDev& g, const ProjDesc& pd, const double* x, const double* bsum, double scale,
                    double* p, cudaStream_t st) {
  bump();
  if (g.Q) {
    if (g.normalized) k_project<true, true><<<stream_grid(g.n), kThreads, 0, st>>>(g, pd, x, bsum, scale, p);
    else k_project<false, true><<<stream_grid(g.n), kThreads, 0, st>>>(g, pd, x, bsum, scale, p);
    return;
  }
  if (g.normalized)
    k_project<true><<<stream_grid(g.n), kThreads, 0, st>>>(g, pd, x, bsum, scale, p);
  else
    k_project<false><<<stream_grid(g.n), kThreads, 0, st>>>(g, pd, x, bsum, scale, p);
}

void launch_finish(const GraphDev& g, const ProjDesc& pd, const double* t, const double* bsum_t,
                   const double* bsum_w, double sigma, double* y, cudaStream_t st) {
  bump();
  if (g.Q) {
    if (g.normalized) k_finish<true, true><<<stream_grid(g.n), kThreads, 0, st>>>(g, pd, t, bsum_t, bsum_w, sigma, y);
    else k_finish<false, true><<<stream_grid(g.n), kThreads, 0, st>>>(g, pd, t, bsum_t, bsum_w, sigma, y);
    return;
  }
  if (g.normalized)
    k_finish<true><<<stream_grid(g.n), kThreads, 0, st>>>(g, pd, t, bsum_t, bsum_w, sigma, y);
  else
    k_finish<false><<<stream_grid(g.n), kThreads, 0, st>>>(g, pd, t, bsum_t, bsum_w, sigma, y);
}

// t = L p + epilogue B^T t, p^T t: the predicated multi-gather kernel (block.cu k_spmm<VS, 1>); the single-vector
// solvers call the TMA-fed tile kernel (spmv_tma.cu) instead where the graph allows
void launch_spmv(const GraphDev& g, int vs, const int* row_split, int grid, const double* p, double* t,
                 double* partials, unsigned* counter, double* bsum_t, cudaStream_t st) {
  launch_spmm(g, 1, vs, row_split, grid, p, t, partials, counter, bsum_t, st);
}

int sweep_grid(int n, int num_sms) { return std::max(1, std::min(cdiv(n, kThreads), num_sms * 4)); }

template <int MODE, bool NORM>
static void sweep_m(const GraphDev& g, const ProjDesc& pd, const SweepArgs& a, int grid, cudaStream_t st) {
  if (g.Q && (MODE == 0 || MODE == 2)) {  // dense projector: the modes that touch it
    if (a.J <= 64) k_sweep<MODE, 8, NORM, true><<<grid, kThreads, 0, st>>>(g, pd, a);
    else if (a.J <= 128) k_sweep<MODE, 16, NORM, true><<<grid, kThreads, 0, st>>>(g, pd, a);
    else if (a.J <= 256) k_sweep<MODE, 32, NORM, true><<<grid, kThreads, 0, st>>>(g, pd, a);
    else k_sweep<MODE, 64, NORM, true><<<grid, kThreads, 0, st>>>(g, pd, a);
    return;
  }
  if (a.J <= 64)
    k_sweep<MODE, 8, NORM><<<grid, kThreads, 0, st>>>(g, pd, a);
  else if (a.J <= 128)
    k_sweep<MODE, 16, NORM><<<grid, kThreads, 0, st>>>(g, pd, a);
  else if (a.J <= 256)
    k_sweep<MODE, 32, NORM><<<grid, kThreads, 0, st>>>(g, pd, a);
  else
    k_sweep<MODE, 64, NORM><<<grid, kThreads, 0, st>>>(g, pd, a);
}
template <int MODE>
static void sweep_n(const GraphDev& g, const ProjDesc& pd, const SweepArgs& a, int grid, cudaStream_t st) {
  if (g.normalized) sweep_m<MODE, true>(g, pd, a, grid, st);
  else sweep_m<MODE, false>(g, pd, a, grid, st);
}
void launch_sweep(int mode, const GraphDev& g, const ProjDesc& pd, const SweepArgs& a, int grid, cudaStream_t st) {
  bump();
  switch (mode) {
    case 0: sweep_n<0>(g, pd, a, grid, st); break;
    case 1: sweep_n<1>(g, pd, a, grid, st); break;
    case 2: sweep_n<2>(g, pd, a, grid, st); break;
    default: sweep_n<3>(g, pd, a, grid, st); break;
  }
}
void launch_reduce_cols(const double* partials, int G, int J, double* out, cudaStream_t st) {
  if (J <= 0) return;
  bump();
  k_reduce_cols<<<J, 128, 0, st>>>(partials, G, J, out);
}
void launch_normalize(const GraphDev& g, const ProjDesc& pd, const double* r, const NormArgs& na, double* vout,
                      double* bsum_v, double* p, cudaStream_t st) {
  bump();
  if (g.normalized)
    k_normalize<true><<<stream_grid(g.n), kThreads, 0, st>>>(g, pd, r, na, vout, bsum_v, p);
  else
    k_normalize<false><<<stream_grid(g.n), kThreads, 0, st>>>(g, pd, r, na, vout, bsum_v, p);
}
void launch_random(double* x, int n, uint64_t seed, unsigned c1, unsigned stream, cudaStream_t st) {
  bump();
  k_random<<<stream_grid(n), kThreads, 0, st>>>(x, n, seed, c1, stream);
}

void launch_ritz(const double* V, long long ld, int n, int m, const double* Y, int p, double* Vout, cudaStream_t st) {
  launch_ritz_rb(V, ld, n, m, Y, p, Vout, st);
}
void launch_resid(const double* y, const double* x, double theta, int n, double* partials, unsigned* counter,
                  double* out, cudaStream_t st) {
  bump();
  k_resid<<<reduce_grid(n), kThreads, 0, st>>>(y, x, theta, nullptr, n, partials, counter, out);
}
void launch_resid_dev(const double* y, const double* x, const double* theta_dev, int n, double* partials,
                      unsigned* counter, double* out, cudaStream_t st) {
  bump();
  k_resid<<<reduce_grid(n), kThreads, 0, st>>>(y, x, 0.0, theta_dev, n, partials, counter, out);
}
void launch_dot(const double* x, const double* y, int n, double* partials, unsigned* counter, double* out,
                cudaStream_t st) {
  bump();
  k_dot<<<reduce_grid(n), kThreads, 0, st>>>(x, y, n, partials, counter, out);
}
void launch_finish_cheb(const GraphDev& g, const ProjDesc& pd, const double* t, const double* bsum_t,
                        const double* bsum_w, double sigma, const double* ycur, const double* yprev, double a,
                        double cc, double b, double* ynew, cudaStream_t st) {
  bump();
  if (g.normalized)
    k_finish_cheb<true><<<stream_grid(g.n), kThreads, 0, st>>>(g, pd, t, bsum_t, bsum_w, sigma, ycur, yprev, a, cc, b,
                                                                ynew);
  else
    k_finish_cheb<false><<<stream_grid(g.n), kThreads, 0, st>>>(g, pd, t, bsum_t, bsum_w, sigma, ycur, yprev, a, cc,
                                                                 b, ynew);
}

}  // namespace sfz

namespace sfz {
void launch_gram_pairs(const double* M, long long rs, long long cs, int n, int r, double* out, cudaStream_t st) {
  bump();
  k_gram_pairs<<<dim3(r, r), kThreads, 0, st>>>(M, rs, cs, n, r, out);
}
void launch_scale_rows(double* M, long long ld, int n, int r, const double* s, cudaStream_t st) {
  bump();
  k_scale_rows<<<stream_grid(n), kThreads, 0, st>>>(M, ld, n, r, s);
}
void launch_rows_times(const double* Min, long long rs, long long cs, int n, int r, int rq, const double* T,
                       double* Qout, int ldq, cudaStream_t st) {
  bump();
  k_rows_times<<<stream_grid(n), kThreads, 0, st>>>(Min, rs, cs, n, r, rq, T, Qout, ldq);
}
}  // namespace sfz
