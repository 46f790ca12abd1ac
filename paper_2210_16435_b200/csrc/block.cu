// libsfairsc — block Krylov kernels (block thick-restart Lanczos).
//
// NB vectors travel together, stored interleaved (row-major n x NB), so one
// gather of row j of the projected block fetches NB contiguous doubles: a
// single 16/32-byte L2 request instead of NB random sector requests.  The
// single-vector SpMV is bound by random L2 requests, so the
// SpMM of NB = 2 vectors costs about one SpMV.  The CGS2 sweeps read the
// basis once per block instead of once per vector.
//
//   spmm    T = L P, epilogue B^T T                        (A5 for NB vectors)
//   bsweep  mode 0: R = finish(T), dots V^T R             (A6 + A8 pass 1)
//           mode 1: R -= V C1, dots V^T R                   (A8 pass 2)
//           mode 2: R -= V C2, Gram R^T R and B^T R         (A8 update + A9)
//           mode 3: dots V^T R (R unchanged)
//   bqr1    R <- R U1^{-1}, U1 = chol(R^T R); Gram of the result   (CholQR pass 1)
//   bqr2    Q = R U2^{-1} -> basis columns, P Q for the next SpMM,
//           T entries (C1 + C2 and U2 U1), B^T Q                     (CholQR pass 2)
//   bgsum / bproject / brandom: start and breakdown blocks.
//
// Reductions are two-stage with fixed partitions and fixed order (bitwise
// reproducible), as in kernels.cu.
#include "device_common.cuh"
#include "tma.cuh"

#include <algorithm>
#include <cstring>

namespace sfz {

void bump_launch();

namespace {
constexpr int kR = 64;  // rows per sweep chunk
constexpr int kMaxStages = 8;
constexpr size_t kRingBytes = 200 * 1024;
}  // namespace

template <int NB>
__host__ __device__ constexpr size_t bstage_doubles(int J) {
  return (size_t)(J + NB + 1) * kR + 16;
}

// NB doubles of row c of an interleaved block
template <int NB>
__device__ __forceinline__ void ld_row(const double* __restrict__ p, int c, double (&x)[NB]) {
  if constexpr (NB == 1) {
    x[0] = __ldg(p + c);
  } else {
    const double2* q = reinterpret_cast<const double2*>(p) + (size_t)c * (NB / 2);
#pragma unroll
    for (int h = 0; h < NB / 2; ++h) {
      const double2 u = __ldg(q + h);
      x[2 * h] = u.x;
      x[2 * h + 1] = u.y;
    }
  }
}

// ----------------------------------------------------------------------------
// SpMM  T = L P  (normalized: P - W^ P ; unnormalized: d o P - W P), VS lanes
// per row, nnz-balanced contiguous row ranges per CTA; each lane keeps up to
// 4 (col, val) pairs and 4 gathers in flight.  Epilogue: B^T T per vector.
// ----------------------------------------------------------------------------
// cmode (column-blocked SpMV for a gathered vector too large for L2, config 5):
//   0 whole matrix (write t, epilogue); 1 first column block (write t); 2 middle (t -= W_b p);
//   3 last (t -= W_b p, epilogue).  g.rp is then the block's row offsets into the block-major CSR.
// UNIT (unit-weight graphs): no value stream; p is then the gathered vector (normalized: q = s o p)
// and p_self the vector itself, the row sum scaled by s_i (normalized).
template <int VS, int NB, bool NORM, int cmode = 0, bool DQ = false, bool LONGR = false, bool UNIT = false>
__global__ void __launch_bounds__(kThreads) k_spmm(GraphDev g, const int* __restrict__ row_split,
                                                   const double* __restrict__ p, const double* __restrict__ p_self,
                                                   double* __restrict__ t, double* partials, unsigned* counter,
                                                   double* bsum_t) {
  constexpr int NG = kThreads / VS, U = 6;  // 6 (col, val) slots per lane: config 4 SpMV 733 -> 718 us (4: one extra pass for the ~45 % of rows above 32 entries; 8: 752 us)
  const int r0 = row_split[blockIdx.x], r1 = row_split[blockIdx.x + 1];
  const int lane = threadIdx.x % VS, gid = threadIdx.x / VS;
  const int* __restrict__ rp = g.rp;
  const int* __restrict__ ci = g.ci;
  const double* __restrict__ vv = g.vv;
  double ptacc[NB];  // p^T t (lane-0 rows)
#pragma unroll
  for (int c = 0; c < NB; ++c) ptacc[c] = 0.0;
  for (int base = r0; base < r1; base += NG) {
    const int row = base + gid;
    const bool valid = row < r1;
    double acc[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) acc[c] = 0.0;
    int a = 0, b = 0;
    if (valid) {
      a = __ldg(rp + row);
      b = __ldg(rp + row + 1);
    }
    // LONGR (skewed degrees, config 5): rows longer than kLong slots are left to the whole warp below
    constexpr int kLong = 32 * VS;
    if (valid && !(LONGR && b - a > kLong)) {
      for (int e0 = a + lane; e0 < b; e0 += U * VS) {
        int cix[U];
        double w[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int e = e0 + q * VS;
          const bool ok = e < b;
          cix[q] = ok ? ld_stream(ci + e) : row;
          w[q] = ok ? (UNIT ? 1.0 : ld_stream(vv + e)) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
          double x[NB];
          ld_row<NB>(p, cix[q], x);
#pragma unroll
          for (int c = 0; c < NB; ++c) acc[c] = fma(w[q], x[c], acc[c]);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < NB; ++c)
#pragma unroll
      for (int o = VS / 2; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
    if constexpr (LONGR && NB == 1) {  // warp-per-row for the long rows of this warp, one at a time
      const int wl = threadIdx.x & 31;
      const bool my_long = valid && lane == 0 && (b - a > kLong);
      unsigned m = __ballot_sync(0xffffffffu, my_long);
      double along = 0.0;
      while (m) {
        const int src = __ffs(m) - 1;
        const int la = __shfl_sync(0xffffffffu, a, src), lb = __shfl_sync(0xffffffffu, b, src);
        double sacc = 0.0;
        for (int e0 = la + wl; e0 < lb; e0 += 32 * U) {
          int cix[U];
          double w[U];
#pragma unroll
          for (int q = 0; q < U; ++q) {
            const int e = e0 + q * 32;
            const bool ok = e < lb;
            cix[q] = ok ? ld_stream(ci + e) : 0;
            w[q] = ok ? (UNIT ? 1.0 : ld_stream(vv + e)) : 0.0;
          }
#pragma unroll
          for (int q = 0; q < U; ++q) {
            double x[1];
            ld_row<1>(p, cix[q], x);
            sacc = fma(w[q], x[0], sacc);
          }
        }
        sacc = warp_sum(sacc);
        if (wl == src) along = sacc;
        m &= m - 1;
      }
      if (my_long) acc[0] = along;
    }
    if constexpr (UNIT && NORM) {
      if (valid && lane == 0) {
        const double si = g.s[row];
#pragma unroll
        for (int c = 0; c < NB; ++c) acc[c] *= si;
      }
    }
    if (valid && lane == 0) {
      double pi[NB];
      ld_row<NB>(p_self, row, pi);  // own rows (row-partitioned: this part's segment of the gathered p)
      const double di = NORM ? 1.0 : __ldg(g.dg + row);
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        double tc;
        if constexpr (cmode < 2) tc = fma(di, pi[c], -acc[c]);
        else tc = t[(size_t)row * NB + c] - acc[c];
        t[(size_t)row * NB + c] = tc;
        ptacc[c] = fma(pi[c], tc, ptacc[c]);
      }
    }
  }
  if constexpr (cmode == 1 || cmode == 2) return;  // partial column block: no epilogue
  // epilogue: B^T t and p^T t over this CTA's rows (fixed order), one vector at a time;
  // out layout: bsum_t[c * kBT + s] = (B^T t_c)_s (s < kHB), bsum_t[c * kBT + kHB] = p_c^T t_c
#pragma unroll 1
  for (int c = 0; c < NB; ++c) {
    __syncthreads();
    double gacc[kBT];
#pragma unroll
    for (int q = 0; q < kBT; ++q) gacc[q] = 0.0;
    for (int row = r0 + threadIdx.x; row < r1; row += kThreads) {
      const double ti = __ldcg(t + (size_t)row * NB + c);
      if constexpr (DQ) {  // dense projector: Q^T t
        const double* qr = g.Q + (size_t)row * g.ldq;
#pragma unroll
        for (int q = 0; q < kHB; ++q)
          if (q < g.qr) gacc[q] = fma(qr[q], ti, gacc[q]);
      } else {
        const double v = NORM ? g.s[row] * ti : ti;
        const int gg = g.grp[row];
#pragma unroll
        for (int q = 0; q < kHB; ++q)
          if (q == gg) gacc[q] += v;
      }
    }
#pragma unroll
    for (int cc = 0; cc < NB; ++cc)
      if (cc == c) gacc[kHB] = ptacc[cc];
    block_reduce_store<kBT>(gacc, partials + ((size_t)blockIdx.x * NB + c) * kBT);
  }
  ticket_finalize<NB * kBT>(partials, counter, bsum_t, NB * kBT);
}

// ----------------------------------------------------------------------------
// Block CGS2 sweeps, TMA-fed (same pipeline as k_sweep_tma): per 64-row chunk
// one 2-D tensor copy of the basis box (64 rows x J columns) and 1-D bulk
// copies of the block chunk (64 x NB interleaved), s and group ids.
// stage layout (doubles): [J][kR] basis | x[kR*NB] | s[kR] | grp[kR bytes + pad]
// ----------------------------------------------------------------------------
template <int NB>
__device__ __forceinline__ void issue_bchunk(const BlockSweepArgs& a, const GraphDev& g, bool need_sg,
                                             const CUtensorMap* tmap, int c, double* buf, unsigned long long* bar,
                                             int lane) {
  const int J = a.J;
  const long long row0 = (long long)c * kR;
  const bool with_s = need_sg && g.normalized;
  unsigned bytes = (unsigned)((J + NB) * kR * sizeof(double));
  if (need_sg) bytes += kR;
  if (with_s) bytes += kR * sizeof(double);
  if (lane == 0) mbar_arrive_expect_tx(bar, bytes);
  __syncwarp();
  if (lane == 0) {
    if (J > 0) tensor2d_g2s(buf, tmap, (int)row0, 0, bar);
    bulk_g2s(buf + (size_t)J * kR, a.xin + row0 * NB, kR * NB * sizeof(double), bar);
  } else if (lane == 1 && need_sg) {
    bulk_g2s(buf + (size_t)(J + NB + 1) * kR, g.grp + row0, kR, bar);
    if (with_s) bulk_g2s(buf + (size_t)(J + NB) * kR, g.s + row0, kR * sizeof(double), bar);
  }
}

template <int MODE, int MAXCW, int NB, bool NORM>
__global__ void __launch_bounds__(kThreads, 1) k_bsweep(GraphDev g, ProjDesc pd, BlockSweepArgs a, int kStages,
                                                         const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) double dsm[];
  __shared__ __align__(8) unsigned long long bars[kMaxStages];
  __shared__ double coef[kBMaxJ * NB];
  __shared__ double red[4][kR * NB];
  __shared__ double rs[kR * NB];
  __shared__ double gam[NB][kHB];
  constexpr int NV2 = NB + kHB;  // mode 2 outputs per vector: Gram row + group sums
  __shared__ double red2[kThreads / 32][NB][NV2];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int n = g.n, J = a.J;
  const int nchunks = (n + kR - 1) / kR;
  const size_t stage_elems = bstage_doubles<NB>(J);
  constexpr bool kNeedSG = (MODE == 0 || MODE == 2);

  if (MODE == 1 || MODE == 2)
    for (int e = tid; e < J * NB; e += kThreads) coef[e] = a.coef[e];
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (MODE == 0 && tid < NB) {  // thread c: gam_c = gamma(B^T t_c) - sigma gamma(B^T w_c)
    double gw[kHB];
    gamma_serial(a.bsum_t + tid * kBT, 1.0, pd, gam[tid]);
    gamma_serial(a.bsum_w + tid * kHB, 1.0, pd, gw);
    for (int s = 0; s < pd.h; ++s) gam[tid][s] -= a.sigma * gw[s];
  }
  __syncthreads();

  const int my_chunks = (nchunks - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  if (w == 0)
    for (int it = 0; it < kStages && it < my_chunks; ++it)
      issue_bchunk<NB>(a, g, kNeedSG, &tmap, blockIdx.x + it * gridDim.x, dsm + it * stage_elems, &bars[it], lane);

  double colacc[MAXCW][NB];
#pragma unroll
  for (int cc = 0; cc < MAXCW; ++cc)
#pragma unroll
    for (int c = 0; c < NB; ++c) colacc[cc][c] = 0.0;
  double v2[NV2];  // mode 2: this thread's vector c = tid % NB
#pragma unroll
  for (int q = 0; q < NV2; ++q) v2[q] = 0.0;

  for (int it = 0; it < my_chunks; ++it) {
    const int c = blockIdx.x + it * gridDim.x;
    const int st = it % kStages;
    const double* buf = dsm + st * stage_elems;
    mbar_wait(&bars[st], (unsigned)((it / kStages) & 1));
    const double* xs = buf + (size_t)J * kR;
    const double* ss = xs + kR * NB;
    const uint8_t* gs = reinterpret_cast<const uint8_t*>(ss + kR);
    const long long row0 = (long long)c * kR;

    // ---- phase 1: row-wise work on the block chunk ----
    if (MODE == 1 || MODE == 2) {
      const int i = tid % kR, cg = tid / kR;
      double part[NB];
#pragma unroll
      for (int q = 0; q < NB; ++q) part[q] = 0.0;
      for (int l = cg; l < J; l += 4) {
        const double v = buf[(size_t)l * kR + i];
#pragma unroll
        for (int q = 0; q < NB; ++q) part[q] = fma(v, coef[l * NB + q], part[q]);
      }
#pragma unroll
      for (int q = 0; q < NB; ++q) red[cg][i * NB + q] = part[q];
      __syncthreads();
      if (tid < kR * NB) {
        const long long gi = row0 + tid / NB;
        double x = 0.0;
        if (gi < n) {
          x = xs[tid] - (((red[0][tid] + red[1][tid]) + red[2][tid]) + red[3][tid]);
          a.xout[row0 * NB + tid] = x;
        }
        rs[tid] = x;
      }
    } else if (MODE == 0) {
      if (tid < kR * NB) {
        const int ii = tid / NB, q = tid % NB;
        double x = 0.0;
        if (row0 + ii < n) {
          const double gg = gam[q][gs[ii]];
          x = NORM ? fma(-ss[ii], gg, xs[tid]) : xs[tid] - gg;
          a.xout[row0 * NB + tid] = x;
        }
        rs[tid] = x;
      }
    } else {
      if (tid < kR * NB) rs[tid] = (row0 + tid / NB < n) ? xs[tid] : 0.0;
    }
    __syncthreads();

    if (MODE == 2) {
      if (tid < kR * NB) {
        const int ii = tid / NB;
        const double x = rs[tid];
#pragma unroll
        for (int q = 0; q < NB; ++q) v2[q] = fma(x, rs[ii * NB + q], v2[q]);
        if (row0 + ii < n) {
          const double sv = NORM ? ss[ii] * x : x;
          const int gg = gs[ii];
#pragma unroll
          for (int q = 0; q < kHB; ++q)
            if (q == gg) v2[NB + q] += sv;
        }
      }
    } else {
      // ---- phase 2: dots V[chunk, l]^T r_q ----
      double r0[NB], r1[NB];
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        r0[q] = rs[lane * NB + q];
        r1[q] = rs[(lane + 32) * NB + q];
      }
#pragma unroll
      for (int cc = 0; cc < MAXCW; ++cc) {
        const int l = w + cc * (kThreads / 32);
        if (l < J) {
          const double* col = buf + (size_t)l * kR;
          const double va = col[lane], vb = col[lane + 32];
#pragma unroll
          for (int q = 0; q < NB; ++q) colacc[cc][q] = fma(vb, r1[q], fma(va, r0[q], colacc[cc][q]));
        }
      }
    }
    __syncthreads();  // stage `st` fully consumed
    if (w == 0 && it + kStages < my_chunks) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_bchunk<NB>(a, g, kNeedSG, &tmap, blockIdx.x + (it + kStages) * gridDim.x, dsm + st * stage_elems,
                       &bars[st], lane);
    }
  }

  if (MODE != 2) {
#pragma unroll
    for (int cc = 0; cc < MAXCW; ++cc) {
      const int l = w + cc * (kThreads / 32);
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        const double s = warp_sum(colacc[cc][q]);
        if (lane == 0 && l < J) a.partials[(size_t)blockIdx.x * J * NB + l * NB + q] = s;
      }
    }
  } else {
    // reduce v2 over the threads that share vector q = tid % NB (NB divides 32)
#pragma unroll
    for (int j = 0; j < NV2; ++j) {
      double x = v2[j];
#pragma unroll
      for (int o = 16; o >= NB; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane < NB) red2[w][lane][j] = x;
    }
    __syncthreads();
    constexpr int NV = NB * NV2;
    for (int e = tid; e < NV; e += kThreads) {
      const int q = e / NV2, j = e % NV2;
      double acc = 0.0;
#pragma unroll
      for (int ww = 0; ww < kThreads / 32; ++ww) acc += red2[ww][q][j];
      a.partials[(size_t)blockIdx.x * NV + e] = acc;
    }
    ticket_finalize<NV>(a.partials, a.counter, a.out, NV);
  }
}

// ----------------------------------------------------------------------------
// CholQR2 normalisation of the block (A9 for NB vectors)
// ----------------------------------------------------------------------------
// U (upper, row-major) with G = U^T U; returns the smallest pivot (<= 0 or NaN: failure, U patched to stay finite)
template <int NB>
__device__ double chol_upper(const double* G, int ldg, double (&U)[NB][NB]) {
  double minpiv = 1e300;
  for (int i = 0; i < NB; ++i) {
    for (int j = 0; j < NB; ++j) U[i][j] = 0.0;
  }
  for (int j = 0; j < NB; ++j) {
    double d = G[j * ldg + j];
    for (int k = 0; k < j; ++k) d -= U[k][j] * U[k][j];
    double piv = d > 0.0 ? sqrt(d) : 0.0;
    minpiv = fmin(minpiv, piv);
    if (!(piv > 0.0)) piv = 1.0;
    U[j][j] = piv;
    for (int i = j + 1; i < NB; ++i) {
      double s = G[j * ldg + i];
      for (int k = 0; k < j; ++k) s -= U[k][j] * U[k][i];
      U[j][i] = s / piv;
    }
  }
  return minpiv;
}
template <int NB>
__device__ void inv_upper(const double (&U)[NB][NB], double (&Ui)[NB][NB]) {
  for (int i = 0; i < NB; ++i)
    for (int j = 0; j < NB; ++j) Ui[i][j] = 0.0;
  for (int j = 0; j < NB; ++j) {
    Ui[j][j] = 1.0 / U[j][j];
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1; k <= j; ++k) s += U[i][k] * Ui[k][j];
      Ui[i][j] = -s / U[i][i];
    }
  }
}

// pass 1: R <- R U1^{-1}; Gram of the result -> g2[NB*NB]
template <int NB>
__global__ void __launch_bounds__(kThreads) k_bqr1(int n, double* __restrict__ R, const double* nbo,
                                                   double* partials, unsigned* counter, double* g2) {
  __shared__ double Ui[NB][NB];
  if (threadIdx.x == 0) {
    double U[NB][NB], I[NB][NB];
    chol_upper<NB>(nbo, NB + kHB, U);
    inv_upper<NB>(U, I);
    for (int i = 0; i < NB; ++i)
      for (int j = 0; j < NB; ++j) Ui[i][j] = I[i][j];
  }
  __syncthreads();
  double gacc[NB * NB];
#pragma unroll
  for (int q = 0; q < NB * NB; ++q) gacc[q] = 0.0;
  const int i0 = (int)((long long)n * blockIdx.x / gridDim.x), i1 = (int)((long long)n * (blockIdx.x + 1) / gridDim.x);
  for (int i = i0 + threadIdx.x; i < i1; i += kThreads) {
    double r[NB], q[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) r[c] = R[(size_t)i * NB + c];
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      double s = 0.0;
#pragma unroll
      for (int c2 = 0; c2 <= c; ++c2) s = fma(r[c2], Ui[c2][c], s);
      q[c] = s;
      R[(size_t)i * NB + c] = s;
    }
#pragma unroll
    for (int c = 0; c < NB; ++c)
#pragma unroll
      for (int c2 = 0; c2 < NB; ++c2) gacc[c * NB + c2] = fma(q[c], q[c2], gacc[c * NB + c2]);
  }
  block_reduce_store<NB * NB>(gacc, partials + (size_t)blockIdx.x * NB * NB);
  ticket_finalize<NB * NB>(partials, counter, g2, NB * NB);
}

// pass 2 (or the only pass when g2 == nullptr): Q = R U2^{-1} into basis
// columns [J, J+NB); p = P Q interleaved; B^T Q -> bs_v; T entries; breakdown flag.
template <int NB, bool NORM>
__global__ void __launch_bounds__(kThreads) k_bqr2(GraphDev g, ProjDesc pd, const double* __restrict__ R,
                                                   BlockQRArgs qa, double* __restrict__ V, long long ld,
                                                   double* __restrict__ p) {
  __shared__ double Ui[NB][NB];
  __shared__ double gam[NB][kHB];
  const int tid = threadIdx.x;
  if (tid == 0) {
    double U1[NB][NB], U2[NB][NB], Ut[NB][NB], I1[NB][NB], I2[NB][NB], It[NB][NB];
    bool bad = false;
    double maxdiag = 0.0;
    for (int c = 0; c < NB; ++c) maxdiag = fmax(maxdiag, sqrt(fmax(qa.nbo[c * (NB + kHB) + c], 0.0)));
    double piv1 = chol_upper<NB>(qa.nbo, NB + kHB, U1);
    if (!(piv1 > qa.bd_tol) || !(piv1 > qa.rel_tol * maxdiag)) bad = true;
    if (qa.g2) {
      double piv2 = chol_upper<NB>(qa.g2, NB, U2);
      if (!(piv2 > 0.5)) bad = true;  // pass 1 left the block far from orthonormal
    } else {
      for (int i = 0; i < NB; ++i)
        for (int j = 0; j < NB; ++j) {
          U2[i][j] = U1[i][j];
          U1[i][j] = (i == j) ? 1.0 : 0.0;
        }
    }
    // Ut = U2 U1 (upper), inverses
    for (int i = 0; i < NB; ++i)
      for (int j = 0; j < NB; ++j) {
        double s = 0.0;
        for (int k = 0; k < NB; ++k) s += U2[i][k] * U1[k][j];
        Ut[i][j] = s;
      }
    inv_upper<NB>(U2, I2);
    inv_upper<NB>(Ut, It);
    (void)I1;
    for (int i = 0; i < NB; ++i)
      for (int j = 0; j < NB; ++j) Ui[i][j] = I2[i][j];
    // B^T Q = (B^T R_orig) Ut^{-1}, per vector c; gam_c = gamma(B^T q_c)
    double btq[NB][kHB];
    for (int c = 0; c < NB; ++c)
      for (int s = 0; s < kHB; ++s) {
        double acc = 0.0;
        for (int c2 = 0; c2 <= c; ++c2) acc += qa.nbo[c2 * (NB + kHB) + NB + s] * It[c2][c];
        btq[c][s] = acc;
      }
    for (int c = 0; c < NB; ++c) gamma_serial(btq[c], 1.0, pd, gam[c]);
    if (blockIdx.x == 0) {
      // the basis block is P q: B^T (P q) = B^T q - beta o gam (so that gamma(B^T w) = 0 in the next finish)
      for (int c = 0; c < NB; ++c)
        for (int s = 0; s < kHB; ++s)
          qa.bs_v[c * kHB + s] = s < pd.h ? btq[c][s] - gam[c][s] / (pd.isb[s] * pd.isb[s]) : 0.0;
      if (qa.T) {
        const int nv = qa.J;  // expanded block = columns [nv - NB, nv)
        for (int c = 0; c < NB; ++c)
          for (int r = 0; r < NB; ++r) qa.T[(size_t)(nv - NB + c) * qa.ldT + nv + r] = (r <= c) ? Ut[r][c] : 0.0;
      }
      *qa.flag = bad ? 1 : 0;
    }
  }
  if (blockIdx.x == 0 && qa.T) {  // T[0:nv, nv-NB+c] = C1 + C2 (projection coefficients)
    const int nv = qa.J;
    for (int e = tid; e < nv * NB; e += kThreads) {
      const int l = e / NB, c = e % NB;
      qa.T[(size_t)(nv - NB + c) * qa.ldT + l] = qa.c1[e] + (qa.c2 ? qa.c2[e] : 0.0);
    }
  }
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + tid; i < g.n; i += gridDim.x * blockDim.x) {
    double r[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) r[c] = R[(size_t)i * NB + c];
    const int gi = g.grp[i];
    const double si = NORM ? g.s[i] : 1.0;
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      double s = 0.0;
#pragma unroll
      for (int c2 = 0; c2 <= c; ++c2) s = fma(r[c2], Ui[c2][c], s);
      const double pc = fma(-si, gam[c][gi], s);  // P q: the basis stays in range(P) to rounding
      V[(long long)(qa.J + c) * ld + i] = pc;
      p[(size_t)i * NB + c] = pc;
    }
  }
}

// group sums of an interleaved block: out[c*kHB + s] = sum_{V_s} s_i x_ic
template <int NB, bool NORM>
__global__ void __launch_bounds__(kThreads) k_bgsum(GraphDev g, const double* __restrict__ x, double* partials,
                                                    unsigned* counter, double* out) {
  const int n = g.n;
  const int i0 = (int)((long long)n * blockIdx.x / gridDim.x), i1 = (int)((long long)n * (blockIdx.x + 1) / gridDim.x);
#pragma unroll 1
  for (int c = 0; c < NB; ++c) {
    __syncthreads();
    double acc[kHB];
#pragma unroll
    for (int q = 0; q < kHB; ++q) acc[q] = 0.0;
    for (int i = i0 + threadIdx.x; i < i1; i += kThreads) {
      const double v = x[(size_t)i * NB + c];
      add_group(acc, g.grp[i], NORM ? g.s[i] * v : v);
    }
    block_reduce_store<kHB>(acc, partials + ((size_t)blockIdx.x * NB + c) * kHB);
  }
  ticket_finalize<NB * kHB>(partials, counter, out, NB * kHB);
}

// y = P x for an interleaved block (factored projector); y may alias x
template <int NB, bool NORM>
__global__ void __launch_bounds__(kThreads) k_bproject(GraphDev g, ProjDesc pd, const double* x, const double* bsum,
                                                       double* y) {
  __shared__ double gam[NB][kHB];
  if (threadIdx.x < NB) gamma_serial(bsum + threadIdx.x * kHB, 1.0, pd, gam[threadIdx.x]);
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) {
    const int gi = g.grp[i];
    const double si = NORM ? g.s[i] : 1.0;
#pragma unroll
    for (int c = 0; c < NB; ++c) y[(size_t)i * NB + c] = fma(-si, gam[c][gi], x[(size_t)i * NB + c]);
  }
}

// ---------------------------------------------------------------------------
// Pair apply: L^sigma on two separate vectors through ONE SpMM of the
// interleaved pair (the SpMV is bound by random L2 requests, a 16-byte pair
// gather costs about one 8-byte gather).  Packing and unpacking are fused into
// the projection and finish passes, so no extra vector pass is added.
// ---------------------------------------------------------------------------
template <bool NORM>
__global__ void __launch_bounds__(kThreads) k_pair_gsum(GraphDev g, const double* __restrict__ x0,
                                                        const double* __restrict__ x1, double* partials,
                                                        unsigned* counter, double* out) {
  const int n = g.n;
  const int i0 = (int)((long long)n * blockIdx.x / gridDim.x), i1 = (int)((long long)n * (blockIdx.x + 1) / gridDim.x);
  double a0[kHB], a1[kHB];
#pragma unroll
  for (int q = 0; q < kHB; ++q) a0[q] = a1[q] = 0.0;
  for (int i = i0 + threadIdx.x; i < i1; i += kThreads) {
    const double si = NORM ? g.s[i] : 1.0;
    const int gg = g.grp[i];
    const double v0 = si * x0[i], v1 = si * x1[i];
#pragma unroll
    for (int q = 0; q < kHB; ++q)
      if (q == gg) {
        a0[q] += v0;
        a1[q] += v1;
      }
  }
  block_reduce_store<kHB>(a0, partials + ((size_t)blockIdx.x * 2 + 0) * kHB);
  __syncthreads();
  block_reduce_store<kHB>(a1, partials + ((size_t)blockIdx.x * 2 + 1) * kHB);
  ticket_finalize<2 * kHB>(partials, counter, out, 2 * kHB);
}
// p[i] = (P x0, P x1)_i interleaved
template <bool NORM>
__global__ void __launch_bounds__(kThreads) k_pair_project(GraphDev g, ProjDesc pd, const double* __restrict__ x0,
                                                           const double* __restrict__ x1, const double* bsum,
                                                           double* __restrict__ p) {
  __shared__ double gam[2][kHB];
  if (threadIdx.x < 2) gamma_serial(bsum + threadIdx.x * kHB, 1.0, pd, gam[threadIdx.x]);
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) {
    const int gi = g.grp[i];
    const double si = NORM ? g.s[i] : 1.0;
    double2 v;
    v.x = fma(-si, gam[0][gi], x0[i]);
    v.y = fma(-si, gam[1][gi], x1[i]);
    reinterpret_cast<double2*>(p)[i] = v;
  }
}
// y_c = t_c - s o (gam(B^T t_c) - sigma gam(B^T x_c))_g, unpacked to two vectors
template <bool NORM>
__global__ void __launch_bounds__(kThreads) k_pair_finish(GraphDev g, ProjDesc pd, const double* __restrict__ t,
                                                          const double* bsum_t, const double* bsum_x, double sigma,
                                                          double* __restrict__ y0, double* __restrict__ y1) {
  __shared__ double gam[2][kHB];
  if (threadIdx.x < 2) {
    double gw[kHB];
    gamma_serial(bsum_t + threadIdx.x * kBT, 1.0, pd, gam[threadIdx.x]);
    gamma_serial(bsum_x + threadIdx.x * kHB, 1.0, pd, gw);
    for (int s = 0; s < pd.h; ++s) gam[threadIdx.x][s] -= sigma * gw[s];
  }
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) {
    const int gi = g.grp[i];
    const double si = NORM ? g.s[i] : 1.0;
    const double2 v = reinterpret_cast<const double2*>(t)[i];
    y0[i] = fma(-si, gam[0][gi], v.x);
    y1[i] = fma(-si, gam[1][gi], v.y);
  }
}

// x[i*NB + c] = u - 1/2, u = Philox4x32-10(key = seed, ctr = (i, c1 + c, stream, 0))
__global__ void k_brandom(double* x, int n, int nb, uint64_t seed, unsigned c1, unsigned stream) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int c = 0; c < nb; ++c) x[(size_t)i * nb + c] = philox_uniform(seed, (unsigned)i, c1 + c, stream, 0u) - 0.5;
}

// ----------------------------------------------------------------------------
// launchers
// ----------------------------------------------------------------------------
static int n_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}
static int sgrid(int n) { return std::max(1, std::min((n + kThreads - 1) / kThreads, n_sms() * 8)); }
static int rgrid(int n) { return std::max(1, std::min((n + 4 * kThreads - 1) / (4 * kThreads), n_sms() * 2)); }

// instantiation map: the pattern-only, long-row (skewed degrees) and dense-projector variants exist for single
// vectors (NB = 1) only; column-blocked modes (cmode 1-3) likewise
template <int VS, int NB, int CM>
static void spmm_cm(const GraphDev& g, const int* split, int grid, const double* p, const double* ps, double* t,
                    double* partials, unsigned* counter, double* bsum_t, cudaStream_t st) {
  using K = void (*)(GraphDev, const int*, const double*, const double*, double*, double*, unsigned*, double*);
  auto go = [&](K kern) { kern<<<grid, kThreads, 0, st>>>(g, split, p, ps, t, partials, counter, bsum_t); };
  if constexpr (NB == 1) {
    const bool nm = g.normalized;
    if (g.Q) return go(nm ? k_spmm<VS, 1, true, CM, true> : k_spmm<VS, 1, false, CM, true>);
    if (g.unit && g.skewed)
      return go(nm ? k_spmm<VS, 1, true, CM, false, true, true> : k_spmm<VS, 1, false, CM, false, true, true>);
    if (g.unit) return go(nm ? k_spmm<VS, 1, true, CM, false, false, true> : k_spmm<VS, 1, false, CM, false, false, true>);
    if (g.skewed) return go(nm ? k_spmm<VS, 1, true, CM, false, true> : k_spmm<VS, 1, false, CM, false, true>);
  }
  go(g.normalized ? k_spmm<VS, NB, true, CM> : k_spmm<VS, NB, false, CM>);
}
template <int VS, int NB>
static void spmm_vs(const GraphDev& g, const int* split, int grid, const double* p, const double* ps, double* t,
                    double* partials, unsigned* counter, double* bsum_t, cudaStream_t st, int cmode = 0) {
  if constexpr (NB == 1) {
    switch (cmode) {
      case 0: return spmm_cm<VS, 1, 0>(g, split, grid, p, ps, t, partials, counter, bsum_t, st);
      case 1: return spmm_cm<VS, 1, 1>(g, split, grid, p, ps, t, partials, counter, bsum_t, st);
      case 2: return spmm_cm<VS, 1, 2>(g, split, grid, p, ps, t, partials, counter, bsum_t, st);
      default: return spmm_cm<VS, 1, 3>(g, split, grid, p, ps, t, partials, counter, bsum_t, st);
    }
  } else {
    spmm_cm<VS, NB, 0>(g, split, grid, p, ps, t, partials, counter, bsum_t, st);
  }
}
void launch_spmv_colblock(const GraphDev& g, int vs, const int* split, int grid, const double* p, double* t,
                          double* partials, unsigned* counter, double* bsum_t, int cmode, cudaStream_t st,
                          const double* p_self) {
  bump_launch();
  const double* ps = p_self ? p_self : p;
  switch (vs) {
    case 2: spmm_vs<2, 1>(g, split, grid, p, ps, t, partials, counter, bsum_t, st, cmode); break;
    case 4: spmm_vs<4, 1>(g, split, grid, p, ps, t, partials, counter, bsum_t, st, cmode); break;
    case 8: spmm_vs<8, 1>(g, split, grid, p, ps, t, partials, counter, bsum_t, st, cmode); break;
    case 16: spmm_vs<16, 1>(g, split, grid, p, ps, t, partials, counter, bsum_t, st, cmode); break;
    default: spmm_vs<32, 1>(g, split, grid, p, ps, t, partials, counter, bsum_t, st, cmode); break;
  }
}
// column blocking of the CSR (block-major copy): per row, the start of each column block (cols sorted)
__global__ void k_colblk_starts(const int* __restrict__ rp, const int* __restrict__ ci, int n, int nblk, int cb,
                                int* __restrict__ cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int a = rp[i], b = rp[i + 1];
    int prev = a;
    for (int q = 1; q <= nblk; ++q) {
      int pos = b;
      if (q < nblk) {  // first entry with col >= q * cb
        int lo = prev, hi = b;
        const long long bound = (long long)q * cb;
        while (lo < hi) {
          const int mid = lo + ((hi - lo) >> 1);
          if (ci[mid] < bound) lo = mid + 1; else hi = mid;
        }
        pos = lo;
      }
      cnt[(size_t)(q - 1) * n + i] = pos - prev;
      prev = pos;
    }
  }
}
__global__ void k_colblk_scatter(const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ vv,
                                 int n, int nblk, const int* __restrict__ rpb, int* __restrict__ ci2,
                                 double* __restrict__ vv2) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int src = rp[i];
    for (int q = 0; q < nblk; ++q) {
      const int d0 = rpb[(size_t)q * (n + 1) + i], d1 = rpb[(size_t)q * (n + 1) + i + 1];
      for (int e = d0; e < d1; ++e, ++src) {
        ci2[e] = ci[src];
        if (vv) vv2[e] = vv[src];  // vv == nullptr: pattern only (unit weights)
      }
    }
  }
}
void launch_colblk_starts(const int* rp, const int* ci, int n, int nblk, int cb, int* cnt, cudaStream_t st) {
  bump_launch();
  k_colblk_starts<<<sgrid(n), kThreads, 0, st>>>(rp, ci, n, nblk, cb, cnt);
}
void launch_colblk_scatter(const int* rp, const int* ci, const double* vv, int n, int nblk, const int* rpb, int* ci2,
                           double* vv2, cudaStream_t st) {
  bump_launch();
  k_colblk_scatter<<<sgrid(n), kThreads, 0, st>>>(rp, ci, vv, n, nblk, rpb, ci2, vv2);
}
template <int NB>
static void spmm_nb(const GraphDev& g, int vs, const int* split, int grid, const double* p, const double* ps,
                    double* t, double* partials, unsigned* counter, double* bsum_t, cudaStream_t st) {
  switch (vs) {
    case 2: spmm_vs<2, NB>(g, split, grid, p, ps, t, partials, counter, bsum_t, st); break;
    case 4: spmm_vs<4, NB>(g, split, grid, p, ps, t, partials, counter, bsum_t, st); break;
    case 8: spmm_vs<8, NB>(g, split, grid, p, ps, t, partials, counter, bsum_t, st); break;
    case 16: spmm_vs<16, NB>(g, split, grid, p, ps, t, partials, counter, bsum_t, st); break;
    default: spmm_vs<32, NB>(g, split, grid, p, ps, t, partials, counter, bsum_t, st); break;
  }
}
void launch_spmm(const GraphDev& g, int nb, int vs, const int* split, int grid, const double* p, double* t,
                 double* partials, unsigned* counter, double* bsum_t, cudaStream_t st, const double* p_self) {
  bump_launch();
  const double* ps = p_self ? p_self : p;
  switch (nb) {
    case 1: spmm_nb<1>(g, vs, split, grid, p, ps, t, partials, counter, bsum_t, st); break;
    case 2: spmm_nb<2>(g, vs, split, grid, p, ps, t, partials, counter, bsum_t, st); break;
    default: spmm_nb<4>(g, vs, split, grid, p, ps, t, partials, counter, bsum_t, st); break;
  }
}

template <int MODE, int MAXCW, int NB, bool NORM>
static void bsweep_launch(const GraphDev& g, const ProjDesc& pd, const BlockSweepArgs& a, int grid, cudaStream_t st) {
  const size_t stage = bstage_doubles<NB>(a.J) * sizeof(double);
  const int stages = (int)std::max<size_t>(2, std::min<size_t>(kMaxStages, kRingBytes / stage));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_bsweep<MODE, MAXCW, NB, NORM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)std::max(kRingBytes, 2 * bstage_doubles<NB>(kBMaxJ) * sizeof(double)));
    attr = true;
  }
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof(tmap));
  if (a.J > 0) encode_colmajor_map(a.V, a.ld, a.J, kR, &tmap);
  k_bsweep<MODE, MAXCW, NB, NORM><<<grid, kThreads, stages * stage, st>>>(g, pd, a, stages, tmap);
}
template <int MODE, int NB, bool NORM>
static void bsweep_m(const GraphDev& g, const ProjDesc& pd, const BlockSweepArgs& a, int grid, cudaStream_t st) {
  if constexpr (MODE == 2) {  // update + norm: no per-column dots
    bsweep_launch<MODE, 4, NB, NORM>(g, pd, a, grid, st);
    return;
  }
  if (a.J <= 32) bsweep_launch<MODE, 4, NB, NORM>(g, pd, a, grid, st);
  else if (a.J <= 64) bsweep_launch<MODE, 8, NB, NORM>(g, pd, a, grid, st);
  else if (a.J <= 128) bsweep_launch<MODE, 16, NB, NORM>(g, pd, a, grid, st);
  else bsweep_launch<MODE, 24, NB, NORM>(g, pd, a, grid, st);
}
template <int MODE, int NB>
static void bsweep_n(const GraphDev& g, const ProjDesc& pd, const BlockSweepArgs& a, int grid, cudaStream_t st) {
  if (g.normalized) bsweep_m<MODE, NB, true>(g, pd, a, grid, st);
  else bsweep_m<MODE, NB, false>(g, pd, a, grid, st);
}
template <int NB>
static void bsweep_nb(int mode, const GraphDev& g, const ProjDesc& pd, const BlockSweepArgs& a, int grid,
                      cudaStream_t st) {
  switch (mode) {
    case 0: bsweep_n<0, NB>(g, pd, a, grid, st); break;
    case 1: bsweep_n<1, NB>(g, pd, a, grid, st); break;
    case 2: bsweep_n<2, NB>(g, pd, a, grid, st); break;
    default: bsweep_n<3, NB>(g, pd, a, grid, st); break;
  }
}
int bsweep_grid(int n) { return std::max(1, std::min((n + kR - 1) / kR, n_sms())); }
void launch_bsweep(int mode, int nb, const GraphDev& g, const ProjDesc& pd, const BlockSweepArgs& a, int grid,
                   cudaStream_t st) {
  bump_launch();
  if (nb == 2) bsweep_nb<2>(mode, g, pd, a, grid, st);  // block Lanczos: block size 2 or 4
  else bsweep_nb<4>(mode, g, pd, a, grid, st);
}

void launch_bqr1(int nb, int n, double* R, const double* nbo, double* partials, unsigned* counter, double* g2,
                 cudaStream_t st) {
  bump_launch();
  const int G = rgrid(n);
  switch (nb) {
    case 1: k_bqr1<1><<<G, kThreads, 0, st>>>(n, R, nbo, partials, counter, g2); break;
    case 2: k_bqr1<2><<<G, kThreads, 0, st>>>(n, R, nbo, partials, counter, g2); break;
    default: k_bqr1<4><<<G, kThreads, 0, st>>>(n, R, nbo, partials, counter, g2); break;
  }
}
template <int NB>
static void bqr2_nb(const GraphDev& g, const ProjDesc& pd, const double* R, const BlockQRArgs& qa, double* V,
                    long long ld, double* p, cudaStream_t st) {
  if (g.normalized)
    k_bqr2<NB, true><<<sgrid(g.n), kThreads, 0, st>>>(g, pd, R, qa, V, ld, p);
  else
    k_bqr2<NB, false><<<sgrid(g.n), kThreads, 0, st>>>(g, pd, R, qa, V, ld, p);
}
void launch_bqr2(int nb, const GraphDev& g, const ProjDesc& pd, const double* R, const BlockQRArgs& qa, double* V,
                 long long ld, double* p, cudaStream_t st) {
  bump_launch();
  switch (nb) {
    case 1: bqr2_nb<1>(g, pd, R, qa, V, ld, p, st); break;
    case 2: bqr2_nb<2>(g, pd, R, qa, V, ld, p, st); break;
    default: bqr2_nb<4>(g, pd, R, qa, V, ld, p, st); break;
  }
}
void launch_bgsum(int nb, const GraphDev& g, const double* x, double* partials, unsigned* counter, double* out,
                  cudaStream_t st) {
  bump_launch();
  const int G = rgrid(g.n);
#define BG(NB_)                                                                   \
  if (g.normalized) k_bgsum<NB_, true><<<G, kThreads, 0, st>>>(g, x, partials, counter, out); \
  else k_bgsum<NB_, false><<<G, kThreads, 0, st>>>(g, x, partials, counter, out);
  switch (nb) {
    case 1: BG(1) break;
    case 2: BG(2) break;
    default: BG(4) break;
  }
#undef BG
}
void launch_bproject(int nb, const GraphDev& g, const ProjDesc& pd, const double* x, const double* bsum, double* y,
                     cudaStream_t st) {
  bump_launch();
  const int G = sgrid(g.n);
#define BP(NB_)                                                                      \
  if (g.normalized) k_bproject<NB_, true><<<G, kThreads, 0, st>>>(g, pd, x, bsum, y); \
  else k_bproject<NB_, false><<<G, kThreads, 0, st>>>(g, pd, x, bsum, y);
  switch (nb) {
    case 1: BP(1) break;
    case 2: BP(2) break;
    default: BP(4) break;
  }
#undef BP
}
void launch_pair_gsum(const GraphDev& g, const double* x0, const double* x1, double* partials, unsigned* counter,
                      double* out, cudaStream_t st) {
  bump_launch();
  const int G = std::max(1, std::min((g.n + kThreads - 1) / kThreads, n_sms() * 4));
  if (g.normalized) k_pair_gsum<true><<<G, kThreads, 0, st>>>(g, x0, x1, partials, counter, out);
  else k_pair_gsum<false><<<G, kThreads, 0, st>>>(g, x0, x1, partials, counter, out);
}
void launch_pair_project(const GraphDev& g, const ProjDesc& pd, const double* x0, const double* x1,
                         const double* bsum, double* p, cudaStream_t st) {
  bump_launch();
  if (g.normalized) k_pair_project<true><<<sgrid(g.n), kThreads, 0, st>>>(g, pd, x0, x1, bsum, p);
  else k_pair_project<false><<<sgrid(g.n), kThreads, 0, st>>>(g, pd, x0, x1, bsum, p);
}
void launch_pair_finish(const GraphDev& g, const ProjDesc& pd, const double* t, const double* bsum_t,
                        const double* bsum_x, double sigma, double* y0, double* y1, cudaStream_t st) {
  bump_launch();
  if (g.normalized) k_pair_finish<true><<<sgrid(g.n), kThreads, 0, st>>>(g, pd, t, bsum_t, bsum_x, sigma, y0, y1);
  else k_pair_finish<false><<<sgrid(g.n), kThreads, 0, st>>>(g, pd, t, bsum_t, bsum_x, sigma, y0, y1);
}
void launch_brandom(double* x, int n, int nb, uint64_t seed, unsigned c1, unsigned stream, cudaStream_t st) {
  bump_launch();
  k_brandom<<<sgrid(n), kThreads, 0, st>>>(x, n, nb, seed, c1, stream);
}

}  // namespace sfz
