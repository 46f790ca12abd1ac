// libsfairsc — single-sweep thick-restart Lanczos (A7-A11 with ONE pass over
// the Krylov basis per step).  Alg. 3 step 3 needs the k smallest
// eigenpairs of L^sigma; the paper uses eigs and names
// "orthonormalization of basis vectors" (O(nk^2)) as a main cost.
//
// Full reorthogonalisation is kept, but delayed by one step (the "lagged"
// vector of low-synchronisation Gram-Schmidt): step j works with v~_j whose
// projections s = V_j^T v~_j on the basis were measured by the previous pass.
//   coef   (1 CTA): mu = sqrt(|v~|^2 - |s|^2); the previous column of the
//                   projected matrix H absorbs the correction (H += s b~^T);
//                   from z = V_j^T A v~_j = H^T s + mu^2 b~ (no pass needed)
//                   and zeta = v~^T A v~ (SpMV epilogue) it forms the
//                   coefficients of the corrected v_j = (v~ - V s)/mu and of
//                   w = A v_j - V_j c - alpha v_j = y/mu - kappa v~ - V_j g.
//   spmv   t = L P v~ (epilogue B^T t, p~^T t)                          (A5)
//   update ONE TMA-fed sweep over V_j: writes v_j (basis column j) and w,
//          and accumulates the dots [V_j, v_j]^T w (next step's s), |w|^2,
//          B^T w                                                      (A6-A9)
//   norm   v~_{j+1} = p~ = P (w/|w|), s_{j+1} = dots/|w|               (A4, A9)
// The relation A V_j = V_j H_j + v_j b^T holds to rounding for the
// coefficients actually used, so the Rayleigh-Ritz matrix sym(H) is exact
// whatever way c was computed; v_j is orthogonal to V_j to O(eps) because
// v~_j's own loss is only O(eps sigma / beta) (it came out of a projected
// recurrence) and one measured projection removes it.  scripts/proto_lagged.py
// is the same algorithm in numpy.
#include "ctx.h"
#include "device_common.cuh"
#include "tma.cuh"
#include "lanczos1.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <vector>

namespace sfz {

void symeig(int m, std::vector<double>& A, std::vector<double>& evals);
void symeig(int m, std::vector<double>& A, std::vector<double>& evals, int nvec);
void bump_launch();

namespace {
constexpr int kR = 64;
constexpr int kMaxStages = 8;
constexpr size_t kRingBytes = 210 * 1024;
constexpr int kLMaxJ = 191;  // basis columns swept (+1 new column in the dots: <= 192)

}  // namespace



// ---------------------------------------------------------------------------
// coefficient step (one CTA)
// ---------------------------------------------------------------------------
// one CTA of kCoefT threads (the O(m^2) work is latency-bound: more threads, shorter chains)
constexpr int kCoefT = 1024;
// sum_{i0 <= i < i1} H[i * ld + row] x[i] in increasing i (one FMA chain), with the column loads issued eight at
// a time ahead of their FMAs (the chain waits on one L2 round trip per eight columns, not per column)
__device__ __forceinline__ double rowdot8(const double* __restrict__ H, int ld, int row, int i0, int i1,
                                          const double* x) {
  double acc = 0.0;
  int i = i0;
  for (; i + 8 <= i1; i += 8) {
    double h[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) h[q] = H[(size_t)(i + q) * ld + row];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc = fma(h[q], x[i + q], acc);
  }
  for (; i < i1; ++i) acc = fma(H[(size_t)i * ld + row], x[i], acc);
  return acc;
}
__global__ void __launch_bounds__(kCoefT) k_lz_coef(LzDev d, int j) {
  __shared__ double ss[kLMaxJ + 1], bt[kLMaxJ + 1], u[kLMaxJ + 1], v[kLMaxJ + 1], red[kCoefT / 32][3];
  __shared__ double upart[4][kLMaxJ + 2];
  __shared__ double sh_mu, sh_alpha, sh_kappa;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int ld = d.ldH;
  // ---- paired steps: the stored odd column p = j - 1 of the last pair is V'' T (T = I but column p =
  // [e; rho], e its measured defect): move the bookkeeping to the orthonormal basis V'' before anything
  // reads it — H <- T H T^-1 on the j x j block, the lagged row b~ <- T^-T b~, s <- T^-T s
  const int pcol = (d.epend && d.lz[LZ_PEND] == (double)(j - 1)) ? j - 1 : -1;
  if (pcol >= 0) {
    __shared__ double ee[kLMaxJ + 1], hle[kLMaxJ + 2];
    __shared__ double sh_es;
    const int p = pcol;  // == j - 1
    const double rho = d.lz[LZ_PRHO];
    for (int l = tid; l < p; l += kCoefT) ee[l] = d.epend[l];
    __syncthreads();
    {  // hle = H[rows 0..p and the lagged row j, cols 0..p-1] ee: thread per row (coalesced down the columns),
       // four column quarters, eight loads in flight per thread; quarters combined in order below
      const int l = tid & 255, qt = tid >> 8;
      if (l <= p + 1) {
        const int row = (l == p + 1) ? j : l;
        upart[qt][l] = rowdot8(d.H, ld, row, p * qt / 4, p * (qt + 1) / 4, ee);
      }
    }
    __syncthreads();
    for (int l = tid; l <= p + 1; l += kCoefT) hle[l] = ((upart[0][l] + upart[1][l]) + upart[2][l]) + upart[3][l];
    double es = 0.0;
    for (int l = tid; l < p; l += kCoefT) es = fma(ee[l], d.s[l], es);
    es = warp_sum(es);
    if (lane == 0) red[w][0] = es;
    __syncthreads();
    if (tid == 0) {
      double a = 0.0;
      for (int q = 0; q < (p + 31) / 32; ++q) a += red[q][0];  // (the other warps hold exact zeros)
      sh_es = a;
    }
    const double hpp = d.H[(size_t)p * ld + p];
    for (int l = tid; l < p; l += kCoefT)  // column p, rows < p
      d.H[(size_t)p * ld + l] = (d.H[(size_t)p * ld + l] + ee[l] * hpp - hle[l] - ee[l] * hle[p]) / rho;
    __syncthreads();
    if (tid == 0) {
      d.H[(size_t)p * ld + p] = hpp - hle[p];
      d.H[(size_t)p * ld + j] = (d.H[(size_t)p * ld + j] - hle[p + 1]) / rho;  // lagged row, column p
      d.s[p] = (d.s[p] - sh_es) / rho;
      d.lz[LZ_CONV] = p;  // the next sweep rewrites column p; coefficient vectors go out in the stored basis
      d.lz[LZ_CRHO] = rho;
      d.lz[LZ_PEND] = -1.0;
    }
    for (int c = w; c < p; c += kCoefT / 32) {  // columns c < p: rows < p += e H[p, c]; row p *= rho
      const double hpc = d.H[(size_t)c * ld + p];
      for (int l = lane; l < p; l += 32) d.H[(size_t)c * ld + l] = fma(ee[l], hpc, d.H[(size_t)c * ld + l]);
      __syncwarp();
      if (lane == 0) d.H[(size_t)c * ld + p] = rho * hpc;
    }
    for (int l = tid; l < p; l += kCoefT) d.econv[l] = ee[l];
    __syncthreads();
  }
  for (int l = tid; l < j; l += kCoefT) {
    ss[l] = d.s[l];
    bt[l] = d.H[(size_t)l * ld + j];  // row j: b~
  }
  __syncthreads();
  // |s|^2, b~ . s
  double a0 = 0.0, a1 = 0.0;
  for (int l = tid; l < j; l += kCoefT) {
    a0 = fma(ss[l], ss[l], a0);
    a1 = fma(bt[l], ss[l], a1);
  }
  a0 = warp_sum(a0);
  a1 = warp_sum(a1);
  if (lane == 0) {
    red[w][0] = a0;
    red[w][1] = a1;
  }
  __syncthreads();
  if (tid == 0) {
    double s2 = 0.0, bs = 0.0;
    for (int q = 0; q < (j + 31) / 32; ++q) {  // (warps beyond j / 32 hold exact zeros)
      s2 += red[q][0];
      bs += red[q][1];
    }
    const double omega = d.lz[LZ_OMEGA];
    double mu2 = omega - s2;
    int bad = 0;
    if (!(mu2 > 1e-12 * omega)) {  // v~ (numerically) inside span(V_j): breakdown
      bad = 2;
      mu2 = 1.0;
    }
    sh_mu = sqrt(mu2);
    red[0][2] = bs;
    *d.flag = bad;
  }
  __syncthreads();
  const double mu = sh_mu, bts = red[0][2];
  // H[:j,:j] += s b~^T ; H[j,:j] = mu b~   (column c of H gets s * b~_c)
  for (int c0 = 0; c0 < j; c0 += 32) {  // only the columns with b~_c != 0 (normally just c = j-1), found by ballot
    unsigned msk = __ballot_sync(0xffffffffu, c0 + lane < j && bt[c0 + lane] != 0.0);
    while (msk) {
      const int c = c0 + __ffs(msk) - 1;
      msk &= msk - 1;
      for (int r = tid; r < j; r += kCoefT) d.H[(size_t)c * ld + r] = fma(ss[r], bt[c], d.H[(size_t)c * ld + r]);
    }
  }
  __syncthreads();
  for (int l = tid; l < j; l += kCoefT) d.H[(size_t)l * ld + j] = mu * bt[l];
  // u = H_j s (thread per row, coalesced over columns), v = H_j^T s (warp per column, coalesced down it)
  {  // u: 4 partial sums per row over quarters of the columns, combined in order below
    const int l = tid & 255, qt = tid >> 8;
    if (l < j) upart[qt][l] = rowdot8(d.H, ld, l, j * qt / 4, j * (qt + 1) / 4, ss);
  }
  for (int l = w; l < j; l += kCoefT / 32) {  // v: warp per column, all its (<= 6 per lane) loads in flight
    double hv[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const int i = lane + 32 * q;
      hv[q] = i < j ? d.H[(size_t)l * ld + i] : 0.0;
    }
    double av = 0.0;
#pragma unroll
    for (int q = 0; q < 6; ++q)
      if (lane + 32 * q < j) av = fma(hv[q], ss[lane + 32 * q], av);
    av = warp_sum(av);
    if (lane == 0) v[l] = av;
  }
  __syncthreads();
  for (int l = tid; l < j; l += kCoefT) u[l] = ((upart[0][l] + upart[1][l]) + upart[2][l]) + upart[3][l];
  __syncthreads();
  // z = v + mu^2 b~ ; zeta = p~^T t + sigma (omega - |p~|^2)
  a0 = 0.0;
  a1 = 0.0;
  for (int l = tid; l < j; l += kCoefT) {
    const double z = fma(mu * mu, bt[l], v[l]);
    a0 = fma(ss[l], z, a0);      // s.z
    a1 = fma(ss[l], u[l], a1);   // s.H s
  }
  a0 = warp_sum(a0);
  a1 = warp_sum(a1);
  __syncthreads();
  if (lane == 0) {
    red[w][0] = a0;
    red[w][1] = a1;
  }
  __syncthreads();
  if (tid == 0) {
    double sz = 0.0, shs = 0.0;
    for (int q = 0; q < (j + 31) / 32; ++q) {  // (the other warps hold exact zeros)
      sz += red[q][0];
      shs += red[q][1];
    }
    const double omega = d.lz[LZ_OMEGA];
    const double zeta = d.bs_t[kHB] + d.sigma * (omega - d.lz[LZ_PNORM2]);
    const double alpha = (zeta - 2.0 * sz + shs) / (mu * mu);
    const double kappa = (alpha + bts) / mu;
    sh_alpha = alpha;
    sh_kappa = kappa;
    d.H[(size_t)j * ld + j] = alpha;
    d.lz[LZ_AY] = 1.0 / mu;
    d.lz[LZ_AV] = -kappa;
    d.lz[LZ_MU] = mu;
    d.lz[LZ_INVMU] = 1.0 / mu;
  }
  __syncthreads();
  const double kappa = sh_kappa;
  // the next sweep still holds the stored column q = LZ_CONV (not yet rewritten): coefficient vectors over
  // V'' = V' T^-1 go out as T^-1 x over the stored columns (x_q / rho at q, x_l - e_l x_q / rho below it)
  const int q = d.econv ? (int)d.lz[LZ_CONV] : -1;
  for (int l = tid; l < j; l += kCoefT) {
    const double z = fma(mu * mu, bt[l], v[l]);
    const double c = (z - u[l]) / mu;
    d.H[(size_t)j * ld + l] = c;                  // column j: c
    const double csl = ss[l] / mu;                // v_j = v~/mu - V (s/mu)
    const double cgl = u[l] / mu + c - kappa * ss[l];  // w = y/mu - kappa v~ - V g
    if (q < 0) {
      d.cs[l] = csl;
      d.cg[l] = cgl;
    } else {
      ss[l] = csl;  // (ss and u are free now)
      u[l] = cgl;
    }
  }
  if (q >= 0) {
    __syncthreads();
    const double ir = 1.0 / d.lz[LZ_CRHO], csq = ss[q] * ir, cgq = u[q] * ir;
    for (int l = tid; l < j; l += kCoefT) {
      const double el = l < q ? d.econv[l] : 0.0;
      d.cs[l] = l == q ? csq : fma(-el, csq, ss[l]);
      d.cg[l] = l == q ? cgq : fma(-el, cgq, u[l]);
    }
  }
}

// ---------------------------------------------------------------------------
// the one sweep: v_j, w, dots [V_j, v_j]^T w, |w|^2, B^T w
// stage (doubles): [J][kR] basis | v~[kR] | t[kR] | s[kR] | grp bytes (pad 128 B)
// ---------------------------------------------------------------------------


// stage layout (doubles): [J][kR] basis | v~[kR] | t[kR] | projector rows: group mode s[kR] + grp bytes,
// dense mode (§8(f) N4) Q[kR][ldq]; + 16 (128-byte pad)
__host__ __device__ constexpr size_t lz_stage_doubles(int J, int ldq = 0) {
  return (size_t)(J + 2) * kR + (size_t)kR * (ldq > 0 ? ldq : 1) + 16;
}

template <bool DQ>
__device__ __forceinline__ void lz_issue(const LzSweepArgs& a, const GraphDev& g, const CUtensorMap* tmap, int c,
                                         double* buf, unsigned long long* bar, int lane) {
  const int J = a.J;
  const long long row0 = (long long)c * kR;
  unsigned bytes = (unsigned)((J + 2) * kR * sizeof(double));
  if constexpr (DQ) bytes += (unsigned)(kR * g.ldq * sizeof(double));
  else bytes += kR + (g.normalized ? kR * sizeof(double) : 0);
  if (lane == 0) mbar_arrive_expect_tx(bar, bytes);
  __syncwarp();
  if (lane == 0) {
    if (J > 0) tensor2d_g2s(buf, tmap, (int)row0, 0, bar);
    bulk_g2s(buf + (size_t)J * kR, a.vt + row0, kR * sizeof(double), bar);
    bulk_g2s(buf + (size_t)(J + 1) * kR, a.t + row0, kR * sizeof(double), bar);
  } else if (lane == 1) {
    if constexpr (DQ) {
      bulk_g2s(buf + (size_t)(J + 2) * kR, g.Q + row0 * g.ldq, (unsigned)(kR * g.ldq * sizeof(double)), bar);
    } else {
      bulk_g2s(buf + (size_t)(J + 3) * kR, g.grp + row0, kR, bar);
      if (g.normalized) bulk_g2s(buf + (size_t)(J + 2) * kR, g.s + row0, kR * sizeof(double), bar);
    }
  }
}

template <int MAXCW, bool NORM, int NT, bool DQ = false>
__global__ void __launch_bounds__(NT, 1) k_lz_update(GraphDev g, ProjDesc pd, LzSweepArgs a, int kStages,
                                                      const __grid_constant__ CUtensorMap tmap) {
  constexpr int NCG = NT / kR;   // column groups of the update phase
  constexpr int NW = NT / 32;    // warps (column owners of the dots phase)
  extern __shared__ __align__(128) double dsm[];
  __shared__ __align__(8) unsigned long long bars[kMaxStages];
  __shared__ double cs[kLMaxJ + 1], cg[kLMaxJ + 1];
  __shared__ double red[2][NCG][kR];
  __shared__ double rw[kR], rv[kR];
  __shared__ double gam[kHB];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int n = g.n, J = a.J;
  const int nchunks = (n + kR - 1) / kR;
  const size_t stage_elems = lz_stage_doubles(J, DQ ? g.ldq : 0);
  for (int l = tid; l < J; l += NT) {
    cs[l] = a.cs[l];
    cg[l] = a.cg[l];
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    double gw[kHB];
    gamma_serial(a.bs_t, 1.0, pd, gam);  // y = t - s o (gam(B^T t) - sigma gam(B^T v~))_g
    gamma_serial(a.bs_v, 1.0, pd, gw);
    for (int s = 0; s < pd.h; ++s) gam[s] -= a.sigma * gw[s];
  }
  __syncthreads();
  const double ay = a.lz[LZ_AY], av = a.lz[LZ_AV], invmu = a.lz[LZ_INVMU];
  const int my_chunks = (nchunks - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  if (w == 0)
    for (int it = 0; it < kStages && it < my_chunks; ++it)
      lz_issue<DQ>(a, g, &tmap, blockIdx.x + it * gridDim.x, dsm + it * stage_elems, &bars[it], lane);

  double colacc[MAXCW];
#pragma unroll
  for (int cc = 0; cc < MAXCW; ++cc) colacc[cc] = 0.0;
  double v2[1 + kHB];
#pragma unroll
  for (int q = 0; q < 1 + kHB; ++q) v2[q] = 0.0;

  for (int it = 0; it < my_chunks; ++it) {
    const int c = blockIdx.x + it * gridDim.x;
    const int st = it % kStages;
    const double* buf = dsm + st * stage_elems;
    mbar_wait(&bars[st], (unsigned)((it / kStages) & 1));
    const double* vts = buf + (size_t)J * kR;
    const double* ts = vts + kR;
    const double* ssc = ts + kR;
    const uint8_t* gs = reinterpret_cast<const uint8_t*>(ssc + kR);
    const long long row0 = (long long)c * kR;
    {
      // four independent FMA chains per sum (the FP64 dependency latency, not bandwidth, bounded
      // the single-chain version: ncu "wait" stalls)
      const int i = tid % kR, cgp = tid / kR;
      double ps0 = 0.0, ps1 = 0.0, ps2 = 0.0, ps3 = 0.0, pg0 = 0.0, pg1 = 0.0, pg2 = 0.0, pg3 = 0.0;
      int l = cgp;
      for (; l + 3 * NCG < J; l += 4 * NCG) {
        const double v0 = buf[(size_t)l * kR + i], v1 = buf[(size_t)(l + NCG) * kR + i];
        const double v2_ = buf[(size_t)(l + 2 * NCG) * kR + i], v3 = buf[(size_t)(l + 3 * NCG) * kR + i];
        ps0 = fma(v0, cs[l], ps0);
        pg0 = fma(v0, cg[l], pg0);
        ps1 = fma(v1, cs[l + NCG], ps1);
        pg1 = fma(v1, cg[l + NCG], pg1);
        ps2 = fma(v2_, cs[l + 2 * NCG], ps2);
        pg2 = fma(v2_, cg[l + 2 * NCG], pg2);
        ps3 = fma(v3, cs[l + 3 * NCG], ps3);
        pg3 = fma(v3, cg[l + 3 * NCG], pg3);
      }
      for (; l < J; l += NCG) {
        const double vv = buf[(size_t)l * kR + i];
        ps0 = fma(vv, cs[l], ps0);
        pg0 = fma(vv, cg[l], pg0);
      }
      red[0][cgp][i] = (ps0 + ps1) + (ps2 + ps3);
      red[1][cgp][i] = (pg0 + pg1) + (pg2 + pg3);
    }
    __syncthreads();
    if (tid < kR) {
      const long long gi = row0 + tid;
      double wv = 0.0, vj = 0.0;
      if (gi < n) {
        double sumS = 0.0, sumG = 0.0;
#pragma unroll
        for (int q = 0; q < NCG; ++q) {
          sumS += red[0][q][tid];
          sumG += red[1][q][tid];
        }
        const double vti = vts[tid];
        vj = fma(vti, invmu, -sumS);
        if constexpr (DQ) {  // dense projector rows Q[i, :] staged after t
          const double* qr = ssc + (size_t)tid * g.ldq;
          double pr = 0.0;
#pragma unroll
          for (int q = 0; q < kHB; ++q)
            if (q < g.qr) pr = fma(qr[q], gam[q], pr);
          wv = fma(ay, ts[tid] - pr, fma(av, vti, -sumG));
          a.vj_out[gi] = vj;
          a.w_out[gi] = wv;
          v2[0] = fma(wv, wv, v2[0]);
#pragma unroll
          for (int q = 0; q < kHB; ++q)
            if (q < g.qr) v2[1 + q] = fma(qr[q], wv, v2[1 + q]);
        } else {
          const int gg = gs[tid];
          const double y = NORM ? fma(-ssc[tid], gam[gg], ts[tid]) : ts[tid] - gam[gg];
          wv = fma(ay, y, fma(av, vti, -sumG));
          a.vj_out[gi] = vj;
          a.w_out[gi] = wv;
          v2[0] = fma(wv, wv, v2[0]);
          const double sv = NORM ? ssc[tid] * wv : wv;
#pragma unroll
          for (int q = 0; q < kHB; ++q)
            if (q == gg) v2[1 + q] += sv;
        }
      }
      rw[tid] = wv;
      rv[tid] = vj;
    }
    __syncthreads();
    {
      const double r0 = rw[lane], r1 = rw[lane + 32];
#pragma unroll
      for (int cc = 0; cc < MAXCW; ++cc) {
        const int l = w + cc * NW;
        if (l <= J) {
          const double* col = (l < J) ? buf + (size_t)l * kR : rv;
          colacc[cc] = fma(col[lane + 32], r1, fma(col[lane], r0, colacc[cc]));
        }
      }
    }
    __syncthreads();
    if (w == 0 && it + kStages < my_chunks) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      lz_issue<DQ>(a, g, &tmap, blockIdx.x + (it + kStages) * gridDim.x, dsm + st * stage_elems, &bars[st], lane);
    }
  }
#pragma unroll
  for (int cc = 0; cc < MAXCW; ++cc) {
    const int l = w + cc * NW;
    const double s = warp_sum(colacc[cc]);
    if (lane == 0 && l <= J) a.partials[(size_t)blockIdx.x * (J + 1) + l] = s;
  }
  block_reduce_store<1 + kHB, NT>(v2, a.partials2 + (size_t)blockIdx.x * (1 + kHB));
  ticket_finalize<1 + kHB, NT>(a.partials2, a.counter, a.nb, 1 + min(pd.h, kHB));
}

// ---------------------------------------------------------------------------
// The single sweep with 64-row chunks and row PAIRS held in registers: thread
// (p, cg) = (lane, warp) owns rows 2p, 2p+1 of the chunk and columns cg + 8q.
// Its basis values are read from shared memory once (16-byte loads) and serve
// both the row combinations (phase 1, with {cs_l, cg_l} as one 16-byte broadcast)
// and the dots (phase 3); the dots stay per thread until one warp sum at the end.
// Same stage layout and TMA ring as k_lz_update.
// ---------------------------------------------------------------------------
template <int MAXQ, bool NORM>
__global__ void __launch_bounds__(kThreads, 1) k_lz_update_p(GraphDev g, ProjDesc pd, LzSweepArgs a, int kStages,
                                                              const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) double dsm[];
  __shared__ __align__(8) unsigned long long bars[kMaxStages];
  __shared__ __align__(16) double2 csg[kLMaxJ + 1];
  __shared__ __align__(16) double red[2][8][kR];
  __shared__ __align__(16) double rw[kR], rv[kR];
  __shared__ double gam[kHB];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int pr = lane, cgp = w;  // row pair (2 pr, 2 pr + 1), column group (columns cgp + 8 q)
  const int n = g.n, J = a.J;
  const int nchunks = (n + kR - 1) / kR;
  const size_t stage_elems = lz_stage_doubles(J);
  for (int l = tid; l < J; l += kThreads) csg[l] = make_double2(a.cs[l], a.cg[l]);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    double gw[kHB];
    gamma_serial(a.bs_t, 1.0, pd, gam);
    gamma_serial(a.bs_v, 1.0, pd, gw);
    for (int s = 0; s < pd.h; ++s) gam[s] -= a.sigma * gw[s];
  }
  __syncthreads();
  const double ay = a.lz[LZ_AY], av = a.lz[LZ_AV], invmu = a.lz[LZ_INVMU];
  const int my_chunks = (nchunks - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  if (w == 0)
    for (int it = 0; it < kStages && it < my_chunks; ++it)
      lz_issue<false>(a, g, &tmap, blockIdx.x + it * gridDim.x, dsm + it * stage_elems, &bars[it], lane);

  double colacc[MAXQ];
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) colacc[q] = 0.0;
  double accJ = 0.0;  // dots with the new column v_j (column J, group J % 8)
  double v2[1 + kHB];
#pragma unroll
  for (int q = 0; q < 1 + kHB; ++q) v2[q] = 0.0;

  for (int it = 0; it < my_chunks; ++it) {
    const int c = blockIdx.x + it * gridDim.x;
    const int st = it % kStages;
    const double* buf = dsm + st * stage_elems;
    mbar_wait(&bars[st], (unsigned)((it / kStages) & 1));
    const double* vts = buf + (size_t)J * kR;
    const double* ts = vts + kR;
    const double* ssc = ts + kR;
    const uint8_t* gs = reinterpret_cast<const uint8_t*>(ssc + kR);
    const long long row0 = (long long)c * kR;
    double2 vreg[MAXQ];
    double ps[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, pg[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // [q parity][row]
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      const int l = cgp + 8 * q;
      if (l < J) {
        vreg[q] = *reinterpret_cast<const double2*>(buf + (size_t)l * kR + 2 * pr);
        const double2 cc = csg[l];
        ps[q & 1][0] = fma(vreg[q].x, cc.x, ps[q & 1][0]);
        ps[q & 1][1] = fma(vreg[q].y, cc.x, ps[q & 1][1]);
        pg[q & 1][0] = fma(vreg[q].x, cc.y, pg[q & 1][0]);
        pg[q & 1][1] = fma(vreg[q].y, cc.y, pg[q & 1][1]);
      } else {
        vreg[q] = make_double2(0.0, 0.0);
      }
    }
    *reinterpret_cast<double2*>(&red[0][cgp][2 * pr]) = make_double2(ps[0][0] + ps[1][0], ps[0][1] + ps[1][1]);
    *reinterpret_cast<double2*>(&red[1][cgp][2 * pr]) = make_double2(pg[0][0] + pg[1][0], pg[0][1] + pg[1][1]);
    __syncthreads();
    if (tid < kR) {
      const long long gi = row0 + tid;
      double wv = 0.0, vj = 0.0;
      if (gi < n) {
        double sumS = 0.0, sumG = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          sumS += red[0][q][tid];
          sumG += red[1][q][tid];
        }
        const double vti = vts[tid];
        vj = fma(vti, invmu, -sumS);
        const int gg = gs[tid];
        const double y = NORM ? fma(-ssc[tid], gam[gg], ts[tid]) : ts[tid] - gam[gg];
        wv = fma(ay, y, fma(av, vti, -sumG));
        a.vj_out[gi] = vj;
        a.w_out[gi] = wv;
        v2[0] = fma(wv, wv, v2[0]);
        const double sv = NORM ? ssc[tid] * wv : wv;
#pragma unroll
        for (int q = 0; q < kHB; ++q)
          if (q == gg) v2[1 + q] += sv;
      }
      rw[tid] = wv;
      rv[tid] = vj;
    }
    __syncthreads();
    const double2 wp = *reinterpret_cast<const double2*>(&rw[2 * pr]);
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) colacc[q] = fma(vreg[q].y, wp.y, fma(vreg[q].x, wp.x, colacc[q]));
    if (cgp == (J & 7)) {
      const double2 vp = *reinterpret_cast<const double2*>(&rv[2 * pr]);
      accJ = fma(vp.y, wp.y, fma(vp.x, wp.x, accJ));
    }
    __syncthreads();  // stage `st` and rw/rv consumed
    if (w == 0 && it + kStages < my_chunks) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      lz_issue<false>(a, g, &tmap, blockIdx.x + (it + kStages) * gridDim.x, dsm + st * stage_elems, &bars[st], lane);
    }
  }
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) {
    const int l = cgp + 8 * q;
    const double sdot = warp_sum(colacc[q]);
    if (lane == 0 && l < J) a.partials[(size_t)blockIdx.x * (J + 1) + l] = sdot;
  }
  {
    const double sdot = warp_sum(accJ);
    if (lane == 0 && cgp == (J & 7)) a.partials[(size_t)blockIdx.x * (J + 1) + J] = sdot;
  }
  block_reduce_store<1 + kHB>(v2, a.partials2 + (size_t)blockIdx.x * (1 + kHB));
  ticket_finalize<1 + kHB>(a.partials2, a.counter, a.nb, 1 + min(pd.h, kHB));
}

// ---------------------------------------------------------------------------
// normalise: v~ = w/|w|, p~ = P v~, B^T v~, s = dots/|w|, |p~|^2, H row j+1
// ---------------------------------------------------------------------------
template <bool NORM, bool DQ = false>
__global__ void __launch_bounds__(kThreads) k_lz_norm(GraphDev g, ProjDesc pd, const double* __restrict__ w,
                                                      const double* nb, const double* dots, int nd, LzDev d, int jrow,
                                                      double* __restrict__ vt, double* __restrict__ p, double* bs_v,
                                                      double* __restrict__ q) {
  __shared__ double gam[kHB];
  __shared__ double s_inv;
  if (threadIdx.x == 0) {
    double beta = sqrt(nb[0]);
    if (!(beta > d.bd_tol)) {
      if (blockIdx.x == 0) atomicOr(d.flag, 1);
      beta = 1.0;
    }
    s_inv = 1.0 / beta;
    gamma_serial(nb + 1, s_inv, pd, gam);
    if (blockIdx.x == 0) {
      // v~ = P (w / |w|): the lagged vector is kept in range(P) (no drift out of null(C^T));
      // B^T v~ = B^T w/|w| - beta o gam,  |v~|^2 = |w|^2/|w|^2 - sum_s beta_s gam_s^2
      double q2 = 0.0;
      for (int s = 0; s < pd.h; ++s) {
        const double bet = DQ ? 1.0 : 1.0 / (pd.isb[s] * pd.isb[s]);  // dense: Q^T Q = I
        bs_v[s] = nb[1 + s] * s_inv - bet * gam[s];
        q2 += bet * gam[s] * gam[s];
      }
      const double omega = nb[0] * s_inv * s_inv - q2;
      d.lz[LZ_OMEGA] = omega;
      d.lz[LZ_PNORM2] = omega;
      d.lz[LZ_BETA] = beta;
    }
  }
  __syncthreads();
  const double inv = s_inv;
  if (blockIdx.x == 0) {
    for (int l = threadIdx.x; l < nd; l += blockDim.x) d.s[l] = dots[l] * inv;
    if (jrow >= 0)  // row jrow of H: b~ = beta e_{jrow-1}
      for (int l = threadIdx.x; l < jrow; l += blockDim.x)
        d.H[(size_t)l * d.ldH + jrow] = (l == jrow - 1) ? 1.0 / inv : 0.0;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) {
    const double vi = w[i] * inv;
    const double pi = vi - proj_row<DQ, NORM>(g, i, gam);
    vt[i] = pi;
    if (p) p[i] = pi;  // (null: the single-GPU solvers hand vt itself to the SpMV)
    if (NORM && q) q[i] = g.s[i] * pi;  // unit-weight SpMV input s o p~ (ctx_spmv's gathered vector)
  }
}

// ---------------------------------------------------------------------------
// Paired steps (two Lanczos steps per basis sweep, tests/tools/proto_pair.py).
//
// three-term vector of the pair's first step j (no basis pass): u = y/mu - kappa v~ - g_{j-1} v_{j-1}
// (y = t - s o gam, the operator apply assembled as in the sweep; g_{j-1} v_{j-1} the only large term
// of V_j g), |u|^2 and B^T u (last-CTA ticket) -> nb.  CTA 0 also records g_far = g with entries j-1
// and j zeroed as the analytic projections of v~_{j+1} (the `dots` of the normalisation that follows),
// subtracts g_far from column j of H (A v_j = V_j (c - g_far) + alpha v_j + |u| v~_{j+1}) and keeps
// 1/mu_j for the pair's sweep.
// ---------------------------------------------------------------------------
template <bool NORM>
__global__ void __launch_bounds__(kThreads, 4) k_lz_three(GraphDev g, ProjDesc pd, const double* __restrict__ t,
                                                       const double* __restrict__ vt, const double* __restrict__ vprev,
                                                       LzDev d, int j, double* __restrict__ u_out, double* dots,
                                                       double* cA, double* tr, double* partials, unsigned* counter,
                                                       double* nb, bool fix_h) {
  __shared__ double gam[kHB];
  if (threadIdx.x == 0) {
    double gw[kHB];
    gamma_serial(d.bs_t, 1.0, pd, gam);
    gamma_serial(d.bs_v, 1.0, pd, gw);
    for (int q = 0; q < pd.h; ++q) gam[q] -= d.sigma * gw[q];
  }
  __syncthreads();
  const double ay = d.lz[LZ_AY], av = d.lz[LZ_AV], gj = d.cg[j - 1];
  double acc[1 + kHB];
#pragma unroll
  for (int q = 0; q < 1 + kHB; ++q) acc[q] = 0.0;
  // (the 17 accumulators keep this kernel at 4 CTAs per SM: one wave of 4 x #SMs CTAs)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) {
    const int gg = g.grp[i];
    const double y = NORM ? fma(-g.s[i], gam[gg], t[i]) : t[i] - gam[gg];
    const double ui = fma(ay, y, fma(av, vt[i], -gj * vprev[i]));
    u_out[i] = ui;
    acc[0] = fma(ui, ui, acc[0]);
    const double su = NORM ? g.s[i] * ui : ui;
#pragma unroll
    for (int q = 0; q < kHB; ++q)
      if (q == gg) acc[1 + q] += su;
  }
  if (blockIdx.x == 0) {
    for (int l = threadIdx.x; l <= j; l += blockDim.x) {
      const double gf = (l >= j - 1) ? 0.0 : d.cg[l];
      dots[l] = gf;
      if (fix_h && l < j) d.H[(size_t)j * d.ldH + l] -= gf;  // (once per process: the replicated H)
    }
    // the pair's sweep needs step j's v_j coefficients after step j+1's coefficient step overwrote d.cs, and
    // the rewrite coefficients of the stored column LZ_CONV (v'' = (v' - V[:, :q] e) / rho)
    const int q = (int)d.lz[LZ_CONV];
    const double ir = q >= 0 ? 1.0 / d.lz[LZ_CRHO] : 0.0;
    for (int l = threadIdx.x; l < j; l += blockDim.x) {
      cA[l] = d.cs[l];
      tr[l] = l < q ? -d.econv[l] * ir : (l == q ? ir : 0.0);
    }
    if (threadIdx.x == 0 && fix_h) d.lz[LZ_INVMU_A] = d.lz[LZ_INVMU];
  }
  block_reduce_store<1 + kHB>(acc, partials + (size_t)blockIdx.x * (1 + kHB));
  ticket_finalize<1 + kHB>(partials, counter, nb, 1 + min(pd.h, kHB));
}

// the pair's one sweep over the stored V[:, 0:J] (J = j), per row:
//   v_j   = v~_j / mu_j - V cA                          (cA = s_j / mu_j, stored basis)
//   v'    = v~_{j+1} / mu_{j+1} - V cB - cB_J v_j        (analytic projections: the odd column)
//   w     = ay y + av v~_{j+1} - V gB - gB_J v_j         (y = t - s o gam of step j+1)
//   v''   = V tr  (rewrite of the stored column LZ_CONV of the previous pair, if any)
// writes V[:, j] = v_j, V[:, j+1] = v', w, V[:, conv] = v''; dots V^T w (J), V^T v' (J), v_j.w, v'.w,
// v_j.v' -> partials [grid][2J + 3]; |w|^2, B^T w, |v'|^2 (ticket) -> nb [0], [1..16], [1 + kHB].
// Stage (doubles): [J][kR] basis | v~_j | v~_{j+1} | t | s | grp bytes (the TMA ring of k_lz_update_p).

constexpr int kPairExtra = 3;  // vectors in a stage beside the basis and the s/grp rows: v~_j, v~_{j+1}, t
__host__ __device__ constexpr size_t lzp_stage_doubles(int J) { return (size_t)(J + kPairExtra) * kR + kR + 16; }

__device__ __forceinline__ void lzp_issue(const LzPairArgs& a, const GraphDev& g, const CUtensorMap* tmap, int c,
                                          double* buf, unsigned long long* bar, int lane) {
  const int J = a.J;
  const long long row0 = (long long)c * kR;
  unsigned bytes = (unsigned)((J + kPairExtra) * kR * sizeof(double)) + kR;
  if (g.normalized) bytes += kR * sizeof(double);
  if (lane == 0) mbar_arrive_expect_tx(bar, bytes);
  __syncwarp();
  if (lane == 0) {
    if (J > 0) tensor2d_g2s(buf, tmap, (int)row0, 0, bar);
    bulk_g2s(buf + (size_t)J * kR, a.vtA + row0, kR * sizeof(double), bar);
    bulk_g2s(buf + (size_t)(J + 1) * kR, a.vtB + row0, kR * sizeof(double), bar);
  } else if (lane == 1) {
    bulk_g2s(buf + (size_t)(J + 2) * kR, a.t + row0, kR * sizeof(double), bar);
    bulk_g2s(buf + (size_t)(J + 4) * kR, g.grp + row0, kR, bar);
    if (g.normalized) bulk_g2s(buf + (size_t)(J + 3) * kR, g.s + row0, kR * sizeof(double), bar);
  }
}

template <int MAXQ, bool NORM>
__global__ void __launch_bounds__(kThreads, 1) k_lz_pair(GraphDev g, ProjDesc pd, LzPairArgs a, int kStages,
                                                          const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) double dsm[];
  __shared__ __align__(8) unsigned long long bars[kMaxStages];
  __shared__ __align__(16) double2 cab[kLMaxJ + 1], cgt[kLMaxJ + 1];  // {cA, cB}, {gB, tr}
  __shared__ __align__(16) double red[4][8][kR];
  __shared__ __align__(16) double rw[kR], rv[kR], rv1[kR];
  __shared__ double gsum[kHB][kR];  // B^T w per row slot (thread (row, 2) adds its rows in chunk order)
  __shared__ double gam[kHB];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int pr = lane, cgp = w;
  const int n = g.n, J = a.J;
  const int nchunks = (n + kR - 1) / kR;
  const size_t stage_elems = lzp_stage_doubles(J);
  static_assert(kThreads == 4 * kR, "one thread per (row, combination) in the finishing phase");
  const bool conv = a.conv_out != nullptr;
  for (int e = tid; e < kHB * kR; e += kThreads) (&gsum[0][0])[e] = 0.0;
  for (int l = tid; l < 8 * MAXQ; l += kThreads) {  // zero coefficients pad the columns beyond J (no branch below)
    cab[l] = l < J ? make_double2(a.cA[l], a.cB[l]) : make_double2(0.0, 0.0);
    cgt[l] = l < J ? make_double2(a.gB[l], conv ? a.tr[l] : 0.0) : make_double2(0.0, 0.0);
  }
  if (tid == 0) {
    for (int st = 0; st < kStages; ++st) mbar_init(&bars[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    double gw[kHB];
    gamma_serial(a.bs_t, 1.0, pd, gam);
    gamma_serial(a.bs_v, 1.0, pd, gw);
    for (int q = 0; q < pd.h; ++q) gam[q] -= a.sigma * gw[q];
  }
  __syncthreads();
  const double invA = a.lz[LZ_INVMU_A], invB = a.lz[LZ_INVMU], ay = a.lz[LZ_AY], av = a.lz[LZ_AV];
  const double cBJ = a.cB[J], gBJ = a.gB[J];
  const int my_chunks = (nchunks - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  if (w == 0)
    for (int it = 0; it < kStages && it < my_chunks; ++it)
      lzp_issue(a, g, &tmap, blockIdx.x + it * gridDim.x, dsm + it * stage_elems, &bars[it], lane);

  double accW[MAXQ], accV[MAXQ];
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) accW[q] = accV[q] = 0.0;
  double dJw = 0.0, dJ1w = 0.0, dJv1 = 0.0;  // v_j.w, v'.w, v_j.v'
  double ww2 = 0.0, vv2 = 0.0;                // |w|^2, |v'|^2 (threads (row, 2) and (row, 1))

  for (int it = 0; it < my_chunks; ++it) {
    const int c = blockIdx.x + it * gridDim.x;
    const int st = it % kStages;
    const double* buf = dsm + st * stage_elems;
    mbar_wait(&bars[st], (unsigned)((it / kStages) & 1));
    const double* vAs = buf + (size_t)J * kR;
    const double* vBs = vAs + kR;
    const double* ts = vBs + kR;
    const double* ssc = ts + kR;
    const uint8_t* gs = reinterpret_cast<const uint8_t*>(ssc + kR);
    const long long row0 = (long long)c * kR;
    double2 vreg[MAXQ];
    double pa[2] = {0.0, 0.0}, pb[2] = {0.0, 0.0}, pg[2] = {0.0, 0.0}, pt[2] = {0.0, 0.0};
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {  // columns beyond J re-read column J - 1 (finite) with zero coefficients
      const int l = cgp + 8 * q;
      vreg[q] = *reinterpret_cast<const double2*>(buf + (size_t)min(l, J - 1) * kR + 2 * pr);
      const double2 ab = cab[l], gt = cgt[l];
      pa[0] = fma(vreg[q].x, ab.x, pa[0]);
      pa[1] = fma(vreg[q].y, ab.x, pa[1]);
      pb[0] = fma(vreg[q].x, ab.y, pb[0]);
      pb[1] = fma(vreg[q].y, ab.y, pb[1]);
      pg[0] = fma(vreg[q].x, gt.x, pg[0]);
      pg[1] = fma(vreg[q].y, gt.x, pg[1]);
      pt[0] = fma(vreg[q].x, gt.y, pt[0]);
      pt[1] = fma(vreg[q].y, gt.y, pt[1]);
    }
    *reinterpret_cast<double2*>(&red[0][cgp][2 * pr]) = make_double2(pa[0], pa[1]);
    *reinterpret_cast<double2*>(&red[1][cgp][2 * pr]) = make_double2(pb[0], pb[1]);
    *reinterpret_cast<double2*>(&red[2][cgp][2 * pr]) = make_double2(pg[0], pg[1]);
    *reinterpret_cast<double2*>(&red[3][cgp][2 * pr]) = make_double2(pt[0], pt[1]);
    __syncthreads();
    // thread (row rr, combination cc) sums the 8 column groups' partials of its combination and of v_j's
    // (every output needs v_j) and finishes output cc of row rr: 0 v_j, 1 v', 2 w, 3 v''
    const int rr = tid & (kR - 1), cc = tid >> 6;
    {
      // fixed-order pairwise sums of the 8 column groups (short dependency chains)
      const double sum = ((red[cc][0][rr] + red[cc][1][rr]) + (red[cc][2][rr] + red[cc][3][rr])) +
                         ((red[cc][4][rr] + red[cc][5][rr]) + (red[cc][6][rr] + red[cc][7][rr]));
      const double s0 = ((red[0][0][rr] + red[0][1][rr]) + (red[0][2][rr] + red[0][3][rr])) +
                        ((red[0][4][rr] + red[0][5][rr]) + (red[0][6][rr] + red[0][7][rr]));
      const long long gi = row0 + rr;
      const bool in = gi < n;
      const double vj = fma(vAs[rr], invA, -s0);
      double out = 0.0;
      if (cc == 0) {
        if (in) a.vj_out[gi] = vj;
        rv[rr] = in ? vj : 0.0;
      } else if (cc == 1) {
        out = fma(-cBJ, vj, fma(vBs[rr], invB, -sum));
        if (!in) out = 0.0;
        if (in) a.vj1_out[gi] = out;
        rv1[rr] = out;
        vv2 = fma(out, out, vv2);
      } else if (cc == 2) {
        if (in) {
          const int gg = gs[rr];
          const double y = NORM ? fma(-ssc[rr], gam[gg], ts[rr]) : ts[rr] - gam[gg];
          out = fma(-gBJ, vj, fma(ay, y, fma(av, vBs[rr], -sum)));
          a.w_out[gi] = out;
          ww2 = fma(out, out, ww2);
          if (gg < kHB) gsum[gg][rr] += NORM ? ssc[rr] * out : out;
        }
        rw[rr] = out;
      } else if (conv && in) {
        a.conv_out[gi] = sum;
      }
    }
    __syncthreads();  // rows finished; stage `st` (read only up to here) is free: refill it now
    if (w == 0 && it + kStages < my_chunks) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      lzp_issue(a, g, &tmap, blockIdx.x + (it + kStages) * gridDim.x, dsm + st * stage_elems, &bars[st], lane);
    }
    const double2 wp = *reinterpret_cast<const double2*>(&rw[2 * pr]);
    const double2 up = *reinterpret_cast<const double2*>(&rv1[2 * pr]);
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      accW[q] = fma(vreg[q].y, wp.y, fma(vreg[q].x, wp.x, accW[q]));
      accV[q] = fma(vreg[q].y, up.y, fma(vreg[q].x, up.x, accV[q]));
    }
    if (cgp == (J & 7)) {
      const double2 vp = *reinterpret_cast<const double2*>(&rv[2 * pr]);
      dJw = fma(vp.y, wp.y, fma(vp.x, wp.x, dJw));
      dJv1 = fma(vp.y, up.y, fma(vp.x, up.x, dJv1));
    }
    if (cgp == ((J + 1) & 7)) dJ1w = fma(up.y, wp.y, fma(up.x, wp.x, dJ1w));
    // (no barrier: red / rw / rv / rv1 are rewritten only after the next chunk's first barrier)
  }
  const size_t row = (size_t)blockIdx.x * (2 * J + 3);
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) {
    const int l = cgp + 8 * q;
    const double sw = warp_sum(accW[q]), sv = warp_sum(accV[q]);
    if (lane == 0 && l < J) {
      a.partials[row + l] = sw;
      a.partials[row + J + 2 + l] = sv;
    }
  }
  {
    const double x = warp_sum(dJw), y = warp_sum(dJv1), z = warp_sum(dJ1w);
    if (lane == 0 && cgp == (J & 7)) {
      a.partials[row + J] = x;
      a.partials[row + 2 * J + 2] = y;
    }
    if (lane == 0 && cgp == ((J + 1) & 7)) a.partials[row + J + 1] = z;
  }
  __syncthreads();  // gsum complete
  double v2[2 + kHB];
  v2[0] = ww2;
  v2[1 + kHB] = vv2;
#pragma unroll
  for (int q = 0; q < kHB; ++q) v2[1 + q] = tid < kR ? gsum[q][tid] : 0.0;
  block_reduce_store<2 + kHB>(v2, a.partials2 + (size_t)blockIdx.x * (2 + kHB));
  ticket_finalize<2 + kHB>(a.partials2, a.counter, a.nb, 2 + kHB);
}

// after the pair's sweep (one CTA): dd = [V_J, v_j, v']^T w (J + 2) and e = [V_J, v_j]^T v' (J + 1) in
// the stored basis; the column rewritten by this sweep (LZ_CONV) now holds v'' = V' T^-1 e_q: its dot
// entries move to the new column, x_q <- (x_q - e_old . x[:q]) / rho_old.  The odd column J + 1 becomes
// pending: epend = e, LZ_PRHO = sqrt(|v'|^2 - |e|^2), LZ_PEND = J + 1; the rewrite is done (LZ_CONV = -1).
__global__ void __launch_bounds__(kCoefT) k_lz_pairpost(LzDev d, int J, const double* __restrict__ dd2,
                                                        double* __restrict__ dd, const double* nb,
                                                        const int* __restrict__ flags) {
  __shared__ double r[2][kCoefT / 32];
  __shared__ double sh[2];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int q = (int)d.lz[LZ_CONV];
  double a0 = 0.0, a1 = 0.0;
  if (q >= 0)
    for (int l = tid; l < q; l += kCoefT) {
      a0 = fma(d.econv[l], dd2[l], a0);
      a1 = fma(d.econv[l], dd2[J + 2 + l], a1);
    }
  a0 = warp_sum(a0);
  a1 = warp_sum(a1);
  if (lane == 0) {
    r[0][w] = a0;
    r[1][w] = a1;
  }
  __syncthreads();
  if (tid == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int k = 0; k < (q + 31) / 32; ++k) {  // (warps beyond q / 32 hold exact zeros)
      s0 += r[0][k];
      s1 += r[1][k];
    }
    sh[0] = s0;
    sh[1] = s1;
  }
  __syncthreads();
  const double ir = q >= 0 ? 1.0 / d.lz[LZ_CRHO] : 1.0;
  double e2 = 0.0;
  for (int l = tid; l <= J + 1; l += kCoefT) {
    double x = dd2[l];
    if (l == q) x = (x - sh[0]) * ir;
    dd[l] = x;
    if (l <= J) {
      double e = dd2[J + 2 + l];
      if (l == q) e = (e - sh[1]) * ir;
      d.epend[l] = e;
      e2 = fma(e, e, e2);
    }
  }
  e2 = warp_sum(e2);
  __syncthreads();
  if (lane == 0) r[0][w] = e2;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int k = 0; k < (J + 2 + 31) / 32; ++k) s += r[0][k];  // (warps beyond (J + 2) / 32 hold exact zeros)
    const double nv = nb[1 + kHB];  // |v'|^2
    const double rho = sqrt(fmax(nv - s, 0.0));
    // a breakdown in the pair (flags of steps J, J+1 so far) leaves v' to the restart sync's roll-back: no basis
    // change from garbage (rho of a valid odd column is 1 to rounding)
    const bool ok = flags[0] == 0 && flags[1] == 0 && rho > 0.5 && rho < 2.0;
    d.lz[LZ_PRHO] = ok ? rho : 1.0;
    d.lz[LZ_PEND] = ok ? J + 1 : -1.0;
    d.lz[LZ_CONV] = -1.0;
  }
}
// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static int lz_sgrid(int n) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return std::max(1, std::min((n + kThreads - 1) / kThreads, sms * 8));
}

template <int MAXCW, bool NORM, int NT, bool DQ = false>
static void lz_update_launch(const GraphDev& g, const ProjDesc& pd, const LzSweepArgs& a, int grid, cudaStream_t st) {
  const size_t stage = lz_stage_doubles(a.J, DQ ? g.ldq : 0) * sizeof(double);
  const int stages = (int)std::max<size_t>(2, std::min<size_t>(kMaxStages, kRingBytes / stage));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_lz_update<MAXCW, NORM, NT, DQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)std::max(kRingBytes, 2 * lz_stage_doubles(kLMaxJ, DQ ? 16 : 0) * sizeof(double)));
    attr = true;
  }
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof(tmap));
  if (a.J > 0) encode_colmajor_map(a.V, a.ld, a.J, kR, &tmap);
  k_lz_update<MAXCW, NORM, NT, DQ><<<grid, NT, stages * stage, st>>>(g, pd, a, stages, tmap);
}
template <int MAXQ, bool NORM>
static void lz_update_p_launch(const GraphDev& g, const ProjDesc& pd, const LzSweepArgs& a, int grid,
                               cudaStream_t st) {
  const size_t stage = lz_stage_doubles(a.J) * sizeof(double);
  const int stages = (int)std::max<size_t>(2, std::min<size_t>(kMaxStages, kRingBytes / stage));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_lz_update_p<MAXQ, NORM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)std::max(kRingBytes, 2 * lz_stage_doubles(kLMaxJ) * sizeof(double)));
    attr = true;
  }
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof(tmap));
  if (a.J > 0) encode_colmajor_map(a.V, a.ld, a.J, kR, &tmap);
  k_lz_update_p<MAXQ, NORM><<<grid, kThreads, stages * stage, st>>>(g, pd, a, stages, tmap);
}
// group projector: 64-row chunks, register-held row pairs (config 4 sweep 768 -> 612 us against the
// shared-memory kernel); dense projector (§8(f) N4): the shared-memory kernel, whose stage carries the Q rows
template <bool NORM>
static void lz_update_m(const GraphDev& g, const ProjDesc& pd, const LzSweepArgs& a, int grid, cudaStream_t st) {
  if (!g.Q) {
    if (a.J <= 64) lz_update_p_launch<8, NORM>(g, pd, a, grid, st);
    else if (a.J <= 128) lz_update_p_launch<16, NORM>(g, pd, a, grid, st);
    else lz_update_p_launch<24, NORM>(g, pd, a, grid, st);
    return;
  }
  if (a.J + 1 <= 64) lz_update_launch<8, NORM, 256, true>(g, pd, a, grid, st);
  else if (a.J + 1 <= 128) lz_update_launch<16, NORM, 256, true>(g, pd, a, grid, st);
  else lz_update_launch<24, NORM, 256, true>(g, pd, a, grid, st);
}

template <int MAXQ, bool NORM>
static void lz_pair_launch(const GraphDev& g, const ProjDesc& pd, const LzPairArgs& a, int grid, cudaStream_t st) {
  // ring budget: 227 KB per CTA minus the kernel's 34 KB of static shared memory (2 stages up to J = 185)
  constexpr size_t kPairRing = 190 * 1024;
  const size_t stage = lzp_stage_doubles(a.J) * sizeof(double);
  const int stages = (int)std::max<size_t>(2, std::min<size_t>(kMaxStages, kPairRing / stage));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_lz_pair<MAXQ, NORM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPairRing);
    attr = true;
  }
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof(tmap));
  if (a.J > 0) encode_colmajor_map(a.V, a.ld, a.J, kR, &tmap);
  k_lz_pair<MAXQ, NORM><<<grid, kThreads, stages * stage, st>>>(g, pd, a, stages, tmap);
}
// one instantiation per column-group count MAXQ = ceil(J / 8): the sweep's time follows the padded column
// count 8 MAXQ, not J (ncu launch list, profiles/r2_final_launches.csv: 778 us at J = 127 with MAXQ = 16,
// 929 us at J = 129 with MAXQ = 24), so the padding stays below 8 columns
template <bool NORM, int Q = 1>
static void lz_pair_q(int maxq, const GraphDev& g, const ProjDesc& pd, const LzPairArgs& a, int grid,
                      cudaStream_t st) {
  if constexpr (Q < 24) {
    if (maxq > Q) {
      lz_pair_q<NORM, Q + 1>(maxq, g, pd, a, grid, st);
      return;
    }
  }
  lz_pair_launch<Q, NORM>(g, pd, a, grid, st);
}
template <bool NORM>
static void lz_pair_m(const GraphDev& g, const ProjDesc& pd, const LzPairArgs& a, int grid, cudaStream_t st) {
  lz_pair_q<NORM>(std::max(1, (a.J + 7) / 8), g, pd, a, grid, st);
}

void launch_lz_coef(const LzDev& d, int j, cudaStream_t st) {
  bump_launch();
  k_lz_coef<<<1, kCoefT, 0, st>>>(d, j);
}
void launch_lz_update(const GraphDev& g, const ProjDesc& pd, const LzSweepArgs& a, int grid, cudaStream_t st) {
  bump_launch();
  if (g.normalized) lz_update_m<true>(g, pd, a, grid, st);
  else lz_update_m<false>(g, pd, a, grid, st);
}
void launch_lz_norm(const GraphDev& g, const ProjDesc& pd, const double* w, const double* nb, const double* dots,
                    int nd, const LzDev& d, int jrow, double* vt, double* p, double* bs_v, cudaStream_t st,
                    double* q) {
  bump_launch();
  if (g.Q) {
    if (g.normalized) k_lz_norm<true, true><<<lz_sgrid(g.n), kThreads, 0, st>>>(g, pd, w, nb, dots, nd, d, jrow, vt, p, bs_v, q);
    else k_lz_norm<false, true><<<lz_sgrid(g.n), kThreads, 0, st>>>(g, pd, w, nb, dots, nd, d, jrow, vt, p, bs_v, q);
    return;
  }
  if (g.normalized)
    k_lz_norm<true><<<lz_sgrid(g.n), kThreads, 0, st>>>(g, pd, w, nb, dots, nd, d, jrow, vt, p, bs_v, q);
  else
    k_lz_norm<false><<<lz_sgrid(g.n), kThreads, 0, st>>>(g, pd, w, nb, dots, nd, d, jrow, vt, p, bs_v, q);
}

void launch_lz_three(const GraphDev& g, const ProjDesc& pd, const double* t, const double* vt, const double* vprev,
                     const LzDev& d, int j, double* u_out, double* dots, double* cA, double* tr, double* partials,
                     unsigned* counter, double* nb, int grid, bool fix_h, cudaStream_t st) {
  bump_launch();
  if (g.normalized)
    k_lz_three<true><<<grid, kThreads, 0, st>>>(g, pd, t, vt, vprev, d, j, u_out, dots, cA, tr, partials, counter, nb,
                                                fix_h);
  else
    k_lz_three<false><<<grid, kThreads, 0, st>>>(g, pd, t, vt, vprev, d, j, u_out, dots, cA, tr, partials, counter, nb,
                                                 fix_h);
}
void launch_lz_pair(const GraphDev& g, const ProjDesc& pd, const LzPairArgs& a, int grid, cudaStream_t st) {
  bump_launch();
  if (g.normalized) lz_pair_m<true>(g, pd, a, grid, st);
  else lz_pair_m<false>(g, pd, a, grid, st);
}
void launch_lz_pairpost(const LzDev& d, int J, const double* dd2, double* dd, const double* nb, const int* flags,
                        cudaStream_t st) {
  bump_launch();
  k_lz_pairpost<<<1, kCoefT, 0, st>>>(d, J, dd2, dd, nb, flags);
}

// host side of the paired steps' basis change at a restart sync (the coefficient kernel's prologue on the
// host copies): the stored odd column p = m - 1 is V'' T (column p of T = [e; rho])
void pair_pending_to_orthonormal(int m, int ldH, std::vector<double>& Hh, std::vector<double>& sh, const double* e,
                                 double rho) {
  const int pq = m - 1;
  auto H = [&](int r, int col) -> double& { return Hh[(size_t)col * ldH + r]; };
  std::vector<double> hle(pq + 2, 0.0);
  for (int l = 0; l <= pq + 1; ++l) {
    const int row = (l == pq + 1) ? m : l;
    double acc = 0.0;
    for (int cc = 0; cc < pq; ++cc) acc += H(row, cc) * e[cc];
    hle[l] = acc;
  }
  double es = 0.0;
  for (int l = 0; l < pq; ++l) es += e[l] * sh[l];
  const double hpp = H(pq, pq);
  for (int l = 0; l < pq; ++l) H(l, pq) = (H(l, pq) + e[l] * hpp - hle[l] - e[l] * hle[pq]) / rho;
  H(pq, pq) = hpp - hle[pq];
  H(m, pq) = (H(m, pq) - hle[pq + 1]) / rho;
  for (int cc = 0; cc < pq; ++cc) {
    const double hpc = H(pq, cc);
    for (int l = 0; l < pq; ++l) H(l, cc) += e[l] * hpc;
    H(pq, cc) = rho * hpc;
  }
  sh[pq] = (sh[pq] - es) / rho;
}
// coefficients x (m entries) over V'' -> T^-1 x over the stored columns
void pair_coef_to_stored(int m, double* x, const double* e, double rho) {
  const int pq = m - 1;
  const double xq = x[pq] / rho;
  for (int l = 0; l < pq; ++l) x[l] -= e[l] * xq;
  x[pq] = xq;
}

// ---------------------------------------------------------------------------
// driver
// ---------------------------------------------------------------------------
namespace {
struct Lagged {
  sfairsc_ctx* c;
  int m, keep, k;
  int64_t applies = 0, steps = 0, restarts = 0, breakdowns = 0;
  unsigned inject = 0;
  double bd_tol = 0.0;
  bool paired = false;  // two Lanczos steps per basis sweep (reorth 3)
  bool pend = false;    // host mirror of LZ_PEND >= 0: the last pair's odd column awaits its rewrite
  bool spmv_ready = false;  // the next step's SpMV (t = L p~) already ran (the restart prefetch)

  LzDev dev(int j) const {
    LzDev d{};
    d.H = c->Hdev;
    d.ldH = c->ldT;
    d.s = c->sdev;
    d.lz = c->lz;
    d.cs = c->c1;
    d.cg = c->c2;
    d.bs_t = c->bs_t;
    d.bs_v = c->bs_v;
    d.flag = c->bflags + j;
    d.sigma = c->sigma;
    d.bd_tol = bd_tol;
    d.epend = paired ? c->lzp : nullptr;
    d.econv = paired ? c->lzp + kMaxJ : nullptr;
    return d;
  }
  double* cA() const { return c->lzp + 2 * kMaxJ; }
  double* trc() const { return c->lzp + 3 * kMaxJ; }
  double* dd2() const { return c->lzp + 4 * kMaxJ; }  // 2 kMaxJ + 8
  // no pending / rewritten column (start, restart, breakdown)
  sfairsc_status clear_pair_state() {
    pend = false;
    if (!paired) return SFAIRSC_OK;
    const double m1[5] = {-1.0, 1.0, -1.0, 1.0, 1.0};  // LZ_PEND, LZ_PRHO, LZ_CONV, LZ_CRHO, LZ_INVMU_A
    std::memcpy(c->hp + 2048, m1, sizeof(m1));
    CU(cudaMemcpyAsync(c->lz + LZ_PEND, c->hp + 2048, sizeof(m1), cudaMemcpyHostToDevice, c->st));
    CU(cudaStreamSynchronize(c->st));
    return SFAIRSC_OK;
  }

  // two Lanczos steps j, j+1 with ONE basis sweep (tests/tools/proto_pair.py)
  sfairsc_status pair(int j) {
    const GraphDev g = c->g();
    const bool rewrite = pend;  // the previous pair's odd column j-1 is rewritten by this pair's sweep
    {
      ProfScope ps(c, K_SPMV, c->csr_bytes() + 3 * c->vb() + 1.0 * c->n);
      ctx_spmv(c, c->vr, c->vt, c->vq_lz);  // p~ = v~ (the normalisation writes it once, into vr)
    }
    {
      ProfScope ps(c, K_OTHER, 0.0);
      bump_launch();
      k_lz_coef<<<1, kCoefT, 0, c->st>>>(dev(j), j);  // (+ the pending column's basis change)
    }
    {
      ProfScope ps(c, K_NORMALIZE, 4 * c->vb() + c->sgb());
      bump_launch();
      // one wave of 4 CTAs per SM (partials: the SpMV's buffer, free again once its ticket is done)
      const int G = std::max(1, std::min((c->n + kThreads - 1) / kThreads, c->num_sms * 4));
      launch_lz_three(g, c->pd(), c->vt, c->vr, c->V + (long long)(j - 1) * c->ldv, dev(j), j, c->vy, c->dd, cA(),
                      trc(), c->partials, c->counters + 7, c->nb, G, true, c->st);
    }
    {
      ProfScope ps(c, K_NORMALIZE, 3 * c->vb() + c->sgb());
      launch_lz_norm(g, c->pd(), c->vy, c->nb, c->dd, j + 1, dev(j), j + 1, c->vrB, nullptr, c->bs_v, c->st,
                     c->unit_spmv() ? c->vq_lz : nullptr);
    }
    {
      ProfScope ps(c, K_SPMV, c->csr_bytes() + 3 * c->vb() + 1.0 * c->n);
      ctx_spmv(c, c->vrB, c->vt, c->vq_lz);
    }
    {
      ProfScope ps(c, K_OTHER, 0.0);
      bump_launch();
      k_lz_coef<<<1, kCoefT, 0, c->st>>>(dev(j + 1), j + 1);
    }
    {
      ProfScope ps(c, K_UPDDOT, (j + 6 + (rewrite ? 1 : 0)) * c->vb() + c->sgb());
      LzPairArgs a{};
      a.V = c->V;
      a.ld = c->ldv;
      a.J = j;
      a.vtA = c->vr;
      a.vtB = c->vrB;
      a.t = c->vt;
      a.vj_out = c->V + (long long)j * c->ldv;
      a.vj1_out = c->V + (long long)(j + 1) * c->ldv;
      a.w_out = c->vy;
      a.conv_out = rewrite ? c->V + (long long)(j - 1) * c->ldv : nullptr;
      a.cA = cA();
      a.cB = c->c1;
      a.gB = c->c2;
      a.tr = trc();
      a.lz = c->lz;
      a.bs_t = c->bs_t;
      a.bs_v = c->bs_v;
      a.sigma = c->sigma;
      a.partials = c->partials;
      a.partials2 = c->partials2;
      a.counter = c->counters + 6;
      a.nb = c->nb;
      const int G = sweep_tma_grid(c->n, c->num_sms);
      launch_lz_pair(g, c->pd(), a, G, c->st);
      launch_reduce_cols(c->partials, G, 2 * j + 3, dd2(), c->st);
    }
    {
      ProfScope ps(c, K_OTHER, 0.0);
      launch_lz_pairpost(dev(j + 1), j, dd2(), c->dd, c->nb, c->bflags + j, c->st);
    }
    norm(c->vy, c->dd, j + 2, j + 2, j + 1);
    CHECK_LAUNCH();
    pend = true;
    applies += 2;
    steps += 2;
    return SFAIRSC_OK;
  }


  void norm(const double* w, const double* dots, int nd, int jrow, int flag_idx) {
    ProfScope ps(c, K_NORMALIZE, 3 * c->vb() + c->sgb());
    launch_lz_norm(c->g(), c->pd(), w, c->nb, dots, nd, dev(flag_idx), jrow, c->vr, nullptr, c->bs_v, c->st,
                   c->unit_spmv() ? c->vq_lz : nullptr);
  }

  // one Lanczos step at column j (A5-A9)
  sfairsc_status step(int j) {
    if (spmv_ready) {
      spmv_ready = false;  // t = L p~ of the continuation vector ran beside the host Rayleigh-Ritz
    } else {
      ProfScope ps(c, K_SPMV, c->csr_bytes() + 3 * c->vb() + 1.0 * c->n);
      ctx_spmv(c, c->vr, c->vt, c->vq_lz);  // epilogue: B^T t and p~^T t (bs_t[kHB]); vq_lz = s o p~ (unit)
    }
    {
      ProfScope ps(c, K_OTHER, 0.0);
      bump_launch();
      k_lz_coef<<<1, kCoefT, 0, c->st>>>(dev(j), j);
    }
    {
      ProfScope ps(c, K_UPDDOT, (j + 4) * c->vb() + c->sgb());
      LzSweepArgs a{};
      a.V = c->V;
      a.ld = c->ldv;
      a.J = j;
      a.vt = c->vr;
      a.t = c->vt;
      a.vj_out = c->V + (long long)j * c->ldv;
      a.w_out = c->vy;
      a.cs = c->c1;
      a.cg = c->c2;
      a.lz = c->lz;
      a.bs_t = c->bs_t;
      a.bs_v = c->bs_v;
      a.sigma = c->sigma;
      a.partials = c->partials;
      a.partials2 = c->partials2;
      a.counter = c->counters + 6;
      a.nb = c->nb;
      const int G = sweep_tma_grid(c->n, c->num_sms);
      bump_launch();
      if (c->normalized) lz_update_m<true>(c->g(), c->pd(), a, G, c->st);
      else lz_update_m<false>(c->g(), c->pd(), a, G, c->st);
      launch_reduce_cols(c->partials, G, j + 1, c->dd, c->st);
    }
    norm(c->vy, c->dd, j + 1, j + 1, j);
    CHECK_LAUNCH();
    applies++;
    steps++;
    return SFAIRSC_OK;
  }

  // v~_j = random vector, projected, CGS2 (twice) against V[:, 0:j], normalised; s = 0, no coupling
  sfairsc_status random_start(int j) {
    TRY(clear_pair_state());
    const GraphDev g = c->g();
    for (int attempt = 0; attempt < 5; ++attempt) {
      launch_random(c->vt, c->n, c->seed, 4096u + inject++, 7u, c->st);
      for (int gb = 0; gb < c->h; gb += kHB) launch_gsum(g, c->vt, gb, c->partials, c->counters + 3, c->bs_w, c->st);
      launch_project(g, c->pd(), c->vt, c->bs_w, 1.0, c->vy, c->st);
      // CGS2 twice with the three-sweep kernels (mode 3 dots, mode 1 update+dots, mode 2 update+norm)
      for (int rep = 0; rep < (j > 0 ? 2 : 1); ++rep) {
        SweepArgs a{};
        a.V = c->V;
        a.ld = c->ldv;
        a.J = j;
        a.xin = c->vy;
        a.xout = c->vy;
        a.bsum_t = c->bs_t;
        a.bsum_w = c->bs_v;
        a.sigma = c->sigma;
        a.partials = c->partials;
        a.counter = c->counters + 2;
        a.norm_bsum = c->nb;
        if (j > 0) {
          launch_sweep(3, g, c->pd(), a, c->sgrid, c->st);
          launch_reduce_cols(c->partials, c->sgrid, j, c->c1, c->st);
          a.coef = c->c1;
          launch_sweep(1, g, c->pd(), a, c->sgrid, c->st);
          launch_reduce_cols(c->partials, c->sgrid, j, c->c2, c->st);
        }
        a.coef = c->c2;
        launch_sweep(2, g, c->pd(), a, c->sgrid, c->st);
        if (c->h > kHB)
          for (int gb = kHB; gb < c->h; gb += kHB)
            launch_gsum(g, c->vy, gb, c->partials, c->counters + 3, c->nb + 1, c->st);
      }
      CU(cudaMemsetAsync(c->bflags + kMaxJ, 0, sizeof(int), c->st));
      norm(c->vy, nullptr, 0, -1, kMaxJ);
      CU(cudaMemsetAsync(c->sdev, 0, sizeof(double) * (j + 1), c->st));
      // no coupling of the injected vector to the basis: H row j = 0
      std::vector<double> zero(std::max(j, 1), 0.0);
      if (j > 0)
        CU(cudaMemcpy2DAsync(c->Hdev + j, sizeof(double) * c->ldT, zero.data(), sizeof(double), sizeof(double), j,
                             cudaMemcpyHostToDevice, c->st));
      int flag = 0;
      CU(cudaMemcpyAsync(c->hp, c->bflags + kMaxJ, sizeof(int), cudaMemcpyDeviceToHost, c->st));
      CU(cudaStreamSynchronize(c->st));
      std::memcpy(&flag, c->hp, sizeof(int));
      if (!flag) return SFAIRSC_OK;
    }
    return fail(SFAIRSC_E_NO_CONVERGENCE, "could not generate a random vector outside the Krylov basis");
  }
};
}  // namespace

sfairsc_status eigs_lagged(sfairsc_ctx* c, int k, double tol, double* evals_out, double* evecs_out,
                           int evecs_memspace, sfairsc_stats* stats) {
  const double t0 = now_s();
  c->have_eigs = false;
  Lagged L;
  L.c = c;
  L.m = c->m;
  L.k = k;
  L.keep = c->keep;
  L.paired = c->paired;
  const int m = L.m, keep = L.keep, n = c->n, ldH = c->ldT;
  const double tol_eff = std::min(tol, c->tol_cap);
  const double target = tol_eff * c->sigma;
  L.bd_tol = std::min(1e-12, 0.01 * tol_eff) * c->sigma;
  CU(cudaMemsetAsync(c->Hdev, 0, sizeof(double) * ldH * ldH, c->st));
  CU(cudaMemsetAsync(c->bflags, 0, sizeof(int) * (kMaxJ + 8), c->st));
  TRY(L.random_start(0));
  int j = 0, jsync = 0;
  bool converged = false;
  std::vector<double> theta, Y, Hh((size_t)ldH * ldH), sh(m + 2);
  double gap = std::numeric_limits<double>::quiet_NaN();
  double max_resid = std::numeric_limits<double>::infinity();
  for (;;) {
    {  // the first step of a cycle is a single step (its g couples every kept Ritz vector), and one more if
       // the rest is odd; then pairs (paired builds) to m
      const int j0 = j;
      while (j < m) {
        if (!L.paired || j == j0 || (m - j) % 2 == 1) TRY(L.step(j++));
        else {
          TRY(L.pair(j));
          j += 2;
        }
      }
    }
    // ---- sync ----
    NvtxRange nv_sync("sfairsc.restart_sync");
    CU(cudaMemcpyAsync(Hh.data(), c->Hdev, sizeof(double) * ldH * ldH, cudaMemcpyDeviceToHost, c->st));
    CU(cudaMemcpyAsync(sh.data(), c->sdev, sizeof(double) * m, cudaMemcpyDeviceToHost, c->st));
    CU(cudaMemcpyAsync(c->hp, c->lz, sizeof(double) * 16, cudaMemcpyDeviceToHost, c->st));
    CU(cudaMemcpyAsync(c->hp + 16, c->bflags, sizeof(int) * (m + 1), cudaMemcpyDeviceToHost, c->st));
    if (L.pend) CU(cudaMemcpyAsync(c->hp + 1024, c->lzp, sizeof(double) * m, cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    if (c->prof.on) c->prof.resolve();
    int jb = -1;
    {
      const int* fl = reinterpret_cast<const int*>(c->hp + 16);
      for (int q = jsync; q < m; ++q)
        if (fl[q]) {
          jb = q;
          break;
        }
    }
    if (jb >= 0) {
      // flag 2 (coef): v~_jb numerically inside span(V_jb): columns 0..jb-1 valid, new v~_jb.
      // flag 1 (norm): |w| <= bd_tol, span(V_{jb+1}) invariant: columns 0..jb valid, new v~_{jb+1}.
      const int* fl = reinterpret_cast<const int*>(c->hp + 16);
      const int jn = (fl[jb] & 2) ? jb : jb + 1;
      if (c->debug) fprintf(stderr, "[sfairsc] lagged breakdown at step %d (flag %d)\n", jb, fl[jb]);
      L.breakdowns++;
      CU(cudaMemsetAsync(c->bflags, 0, sizeof(int) * (kMaxJ + 8), c->st));
      TRY(L.random_start(jn));
      j = jn;
      jsync = j;
      continue;
    }
    // ---- paired steps: the last pair's odd column m-1 is still the stored v' = V'' T: move H, the lagged row
    // and s to V'' (as the coefficient kernel does), and the Ritz coefficients back to the stored columns below
    const bool tconv = L.pend;
    const int pq = m - 1;
    const double prho = c->hp[LZ_PRHO];
    std::vector<double> pdef(tconv ? pq : 0);  // the pending column's defect e
    if (tconv) {
      for (int l = 0; l < pq; ++l) pdef[l] = c->hp[1024 + l];
      pair_pending_to_orthonormal(m, ldH, Hh, sh, pdef.data(), prho);
    }
    auto to_stored = [&](double* x) {
      if (tconv) pair_coef_to_stored(m, x, pdef.data(), prho);
    };
    // ---- Rayleigh-Ritz on sym(H_m + s b~^T) ----
    const double om = c->hp[LZ_OMEGA];
    double s2 = 0.0;
    for (int l = 0; l < m; ++l) s2 += sh[l] * sh[l];
    double mu = std::sqrt(std::max(om - s2, 0.0));
    if (!(mu > 0.0)) mu = 1.0;
    // ---- restart prefetch, enqueued before the host Rayleigh-Ritz below and run beside it: the continuation
    // vector v_m = (v~ - V s)/mu depends on s only, not on the Ritz vectors, so its pass over the basis
    // (x = v~ - V s in the stored basis, |x|^2, B^T x), its normalisation (v~, p~ of the next cycle's first step)
    // and that step's SpMV run on the GPU while the host solves the RR problem; the Ritz GEMM then forms only
    // the kept columns, and the first step's sweep writes column keep (v~/|v~|) without reading it.  Wasted
    // (one pass) at the final sync.
    {
      std::vector<double> x(m + 1, 0.0);
      for (int l = 0; l < m; ++l) x[l] = -sh[l] / mu;
      x[m] = 1.0 / mu;
      to_stored(x.data());
      double* hc = c->hp + 3072;  // pinned scratch (m <= 192)
      for (int l = 0; l < m; ++l) hc[l] = -x[l] * mu;  // x = v~ - V coef = mu v_m
      double* dcoef = c->Ydev + (size_t)(m + 1) * m;   // the last m + 1 entries: beyond every Ritz coefficient block
      CU(cudaMemcpyAsync(dcoef, hc, sizeof(double) * m, cudaMemcpyHostToDevice, c->st));
      {
        ProfScope ps(c, K_UPDDOT, (m + 2) * c->vb() + c->sgb());
        SweepArgs a{};
        a.V = c->V;
        a.ld = c->ldv;
        a.J = m;
        a.xin = c->vr;
        a.xout = c->vy;
        a.coef = dcoef;
        a.bsum_t = c->bs_t;
        a.bsum_w = c->bs_v;
        a.sigma = c->sigma;
        a.partials = c->partials;
        a.counter = c->counters + 2;
        a.norm_bsum = c->nb;
        launch_sweep(2, c->g(), c->pd(), a, c->sgrid, c->st);  // update + |x|^2 + B^T x
        if (c->h > kHB)
          for (int gb = kHB; gb < c->h; gb += kHB)
            launch_gsum(c->g(), c->vy, gb, c->partials, c->counters + 3, c->nb + 1, c->st);
      }
      L.norm(c->vy, nullptr, 0, -1, kMaxJ);
      {
        ProfScope ps(c, K_SPMV, c->csr_bytes() + 3 * c->vb() + 1.0 * c->n);
        ctx_spmv(c, c->vr, c->vt, c->vq_lz);
      }
      CHECK_LAUNCH();
    }
    std::vector<double> bt(m), A((size_t)m * m);
    for (int l = 0; l < m; ++l) bt[l] = Hh[(size_t)l * ldH + m];
    for (int r = 0; r < m; ++r)
      for (int q = 0; q < m; ++q) {
        const double hrq = Hh[(size_t)q * ldH + r] + sh[r] * bt[q];
        const double hqr = Hh[(size_t)r * ldH + q] + sh[q] * bt[r];
        A[(size_t)r * m + q] = 0.5 * (hrq + hqr);
      }
    Y = A;
    // only the kept (>= k) smallest Ritz vectors are used below: the selected-vector eigensolver
    const int nsel = std::min(m, std::max(keep, k));
    {
      NvtxRange nv_rr("sfairsc.rayleigh_ritz");
      symeig(m, Y, theta, nsel);
    }
    double maxres = 0.0;
    std::vector<double> bY(m, 0.0);
    for (int i = 0; i < nsel; ++i) {
      double acc = 0.0;
      for (int l = 0; l < m; ++l) acc += bt[l] * Y[(size_t)l * m + i];
      bY[i] = mu * acc;  // b = mu b~ : coupling of Ritz vector i to v_m
    }
    for (int i = 0; i < k; ++i) maxres = std::max(maxres, std::fabs(bY[i]));
    if (k < m) gap = theta[k] - theta[k - 1];
    converged = maxres <= target;
    if (c->debug)
      fprintf(stderr, "[sfairsc] lagged RR restarts=%lld steps=%lld maxres=%g target=%g theta_k=%.17g mu=%g\n",
              (long long)L.restarts, (long long)L.steps, maxres, target, theta[k - 1], mu);
    if (converged || L.restarts >= c->max_restarts) {
      std::vector<double> Yc((size_t)m * k);
      for (int cc = 0; cc < k; ++cc) {
        for (int l = 0; l < m; ++l) Yc[(size_t)cc * m + l] = Y[(size_t)l * m + cc];
        to_stored(Yc.data() + (size_t)cc * m);
      }
      CU(cudaMemcpyAsync(c->Ydev, Yc.data(), sizeof(double) * Yc.size(), cudaMemcpyHostToDevice, c->st));
      {
        ProfScope ps(c, K_RITZ, (double)(m + k) * c->vb());
        launch_ritz(c->V, c->ldv, n, m, c->Ydev, k, c->X, c->st);
      }
      CHECK_LAUNCH();
      break;
    }
    // ---- thick restart: V_m Y_keep (the continuation vector v_m is already normalised into v~, p~: prefetch) ----
    std::vector<double> Yc((size_t)m * keep, 0.0);
    for (int cc = 0; cc < keep; ++cc) {
      for (int l = 0; l < m; ++l) Yc[(size_t)cc * m + l] = Y[(size_t)l * m + cc];
      to_stored(Yc.data() + (size_t)cc * m);
    }
    CU(cudaMemcpyAsync(c->Ydev, Yc.data(), sizeof(double) * Yc.size(), cudaMemcpyHostToDevice, c->st));
    {
      ProfScope ps(c, K_RITZ, (double)(m + keep) * c->vb());
      launch_ritz(c->V, c->ldv, n, m, c->Ydev, keep, c->Vb, c->st);
    }
    CHECK_LAUNCH();
    std::swap(c->V, c->Vb);
    // state at j = keep: v~ = v_m (s = 0), coupling row b~ = (b Y)_i for the kept vectors
    std::fill(Hh.begin(), Hh.end(), 0.0);
    for (int i = 0; i < keep; ++i) {
      Hh[(size_t)i * ldH + i] = theta[i];
      Hh[(size_t)i * ldH + keep] = bY[i];
    }
    CU(cudaMemcpyAsync(c->Hdev, Hh.data(), sizeof(double) * ldH * ldH, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemsetAsync(c->sdev, 0, sizeof(double) * (m + 2), c->st));
    L.spmv_ready = true;
    TRY(L.clear_pair_state());
    j = keep;
    jsync = keep;
    L.restarts++;
  }

  TRY(true_residuals(c, theta.data(), k, &max_resid));
  L.applies += k;
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
  S.basis_size = m;
  S.kept = keep;
  c->last = S;
  if (stats) *stats = S;
  if (!converged) return fail(SFAIRSC_E_NO_CONVERGENCE, "no convergence after %lld restarts", (long long)L.restarts);
  if (theta[k - 1] >= c->sigma * (1.0 - 1e-8))
    return fail(SFAIRSC_E_SHIFT_TOO_SMALL, "lambda_k=%g >= sigma(1-1e-8)=%g (Prop. 3.4)", theta[k - 1], c->sigma);
  return SFAIRSC_OK;
}

}  // namespace sfz
