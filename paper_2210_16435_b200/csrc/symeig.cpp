// Dense symmetric eigensolver for the small Rayleigh-Ritz matrix T (m x m,
// m <= a few hundred) of the thick-restart Lanczos method.
// Householder reduction to tridiagonal form followed by the implicit QL
// iteration with Wilkinson-type shifts (the EISPACK tred2/tql2 pair, restated).
// Host code, fp64; runs once per restart.
#include <algorithm>
#include <cmath>
#include <vector>

namespace sfz {

namespace {
// sqrt(a^2 + b^2) without std::hypot's scaling (its libm call is ~0.5 ms of a 170 x 170 restart) when the
// squares can neither overflow nor underflow; std::hypot otherwise
inline double hyp(double a, double b) {
  const double m = std::max(std::fabs(a), std::fabs(b));
  if (m < 1e150 && m > 1e-150) return std::sqrt(a * a + b * b);
  return std::hypot(a, b);
}
struct Rot {
  int i;
  double c, s;
};
}  // namespace

// QL (tql2) on the symmetric tridiagonal (d[0..m-1], e[k] = coupling of k and k+1, e[m-1] = 0): eigenvalues
// into d (unsorted); the rotations Z <- Z G_t, G_t = [[c, s], [-s, c]] on columns (i, i+1), recorded in order
template <int kDummy>
static inline __attribute__((always_inline)) void ql_record(int m, std::vector<double>& d, std::vector<double>& e,
                                                             std::vector<Rot>& rots) {
  rots.reserve((size_t)m * 8);
  double f = 0.0, tst1 = 0.0;
  const double eps = std::ldexp(1.0, -52);
  for (int l = 0; l < m; ++l) {
    tst1 = std::max(tst1, std::fabs(d[l]) + std::fabs(e[l]));
    int mm = l;
    while (mm < m) {
      if (std::fabs(e[mm]) <= eps * tst1) break;
      ++mm;
    }
    if (mm == m) mm = m - 1;
    if (mm > l) {
      int iter = 0;
      do {
        ++iter;
        double g = d[l];
        double p = (d[l + 1] - g) / (2.0 * e[l]);
        double r = hyp(p, 1.0);
        if (p < 0) r = -r;
        d[l] = e[l] / (p + r);
        d[l + 1] = e[l] * (p + r);
        const double dl1 = d[l + 1];
        double h = g - d[l];
        for (int i = l + 2; i < m; ++i) d[i] -= h;
        f += h;
        p = d[mm];
        double c = 1.0, c2 = c, c3 = c;
        const double el1 = e[l + 1];
        double s = 0.0, s2 = 0.0;
        for (int i = mm - 1; i >= l; --i) {
          c3 = c2;
          c2 = c;
          s2 = s;
          g = c * e[i];
          h = c * p;
          r = hyp(p, e[i]);
          e[i + 1] = s * r;
          s = e[i] / r;
          c = p / r;
          p = c * d[i] - s * g;
          d[i + 1] = h + s * (c * g + s * d[i]);
          rots.push_back(Rot{i, c, s});
        }
        p = -s * s2 * c3 * el1 * e[l] / dl1;
        e[l] = s * p;
        d[l] = c * p;
      } while (std::fabs(e[l]) > eps * tst1 && iter < 200);
    }
    d[l] = d[l] + f;
    e[l] = 0.0;
  }
}

// The thick restart's selected-vector solver (nvec < m: only the nvec smallest Ritz pairs are kept).
// Householder tridiagonalisation on the full symmetric matrix with row-contiguous loops (LAPACK sytd2 order:
// H_k = I - beta_k v_k v_k^T acts on indices k+1 .. m-1 and zeroes A(k+2:, k); Q = H_0 ... H_{m-3}): the
// matrix-vector product as a sum of scaled rows and the rank-2 update are unit-stride loops that vectorise
// (m^3 multiply-adds, against EISPACK tred2's 2/3 m^3 in short strided loops); then QL with recorded
// rotations, which are applied in REVERSE order to the nvec selected unit vectors (rows of an m x nvec block:
// 6 nvec instead of 6 m flops per rotation), and the reflectors map that block back (2 m^2 nvec flops).
template <int kDummy>
static inline __attribute__((always_inline)) void symeig_select(int m, std::vector<double>& A,
                                                                 std::vector<double>& evals, int nvec) {
  std::vector<double> d(m, 0.0), e(m, 0.0), beta(m, 0.0), vbuf((size_t)m * m, 0.0), pv(m), wv(m);
  double* __restrict__ a = A.data();
  for (int k = 0; k + 2 < m; ++k) {
    const int n2 = m - k - 1;
    double* __restrict__ v = &vbuf[(size_t)k * m];  // v_k (length n2) = row k of A beyond the diagonal
    const double* __restrict__ rowk = a + (size_t)k * m + k + 1;
    double sig = 0.0;
    for (int q = 1; q < n2; ++q) sig += rowk[q] * rowk[q];
    const double alpha = rowk[0];
    d[k] = a[(size_t)k * m + k];
    if (sig == 0.0) {  // already tridiagonal in this column: H_k = I
      e[k] = alpha;
      beta[k] = 0.0;
      continue;
    }
    const double nrm = std::sqrt(alpha * alpha + sig);
    const double v0 = alpha >= 0.0 ? alpha + nrm : alpha - nrm;
    e[k] = alpha >= 0.0 ? -nrm : nrm;
    v[0] = v0;
    for (int q = 1; q < n2; ++q) v[q] = rowk[q];
    const double bk = 2.0 / (v0 * v0 + sig);
    beta[k] = bk;
    // p = beta B v (B = A(k+1:, k+1:), symmetric: a sum of its rows scaled by v)
    double* __restrict__ p = pv.data();
    for (int q = 0; q < n2; ++q) p[q] = 0.0;
    for (int r = 0; r < n2; ++r) {
      const double vr = bk * v[r];
      const double* __restrict__ br = a + (size_t)(k + 1 + r) * m + k + 1;
      for (int q = 0; q < n2; ++q) p[q] += vr * br[q];
    }
    double pvd = 0.0;
    for (int q = 0; q < n2; ++q) pvd += p[q] * v[q];
    const double K = 0.5 * bk * pvd;
    double* __restrict__ w = wv.data();
    for (int q = 0; q < n2; ++q) w[q] = p[q] - K * v[q];
    // B -= v w^T + w v^T
    for (int r = 0; r < n2; ++r) {
      double* __restrict__ br = a + (size_t)(k + 1 + r) * m + k + 1;
      const double vr = v[r], wr = w[r];
      for (int q = 0; q < n2; ++q) br[q] -= vr * w[q] + wr * v[q];
    }
  }
  if (m >= 2) {
    d[m - 2] = a[(size_t)(m - 2) * m + (m - 2)];
    e[m - 2] = a[(size_t)(m - 1) * m + (m - 2)];
  }
  d[m - 1] = a[(size_t)(m - 1) * m + (m - 1)];
  e[m - 1] = 0.0;
  std::vector<Rot> rots;
  ql_record<kDummy>(m, d, e, rots);
  std::vector<int> idx(m);
  for (int i = 0; i < m; ++i) idx[i] = i;
  std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return d[x] < d[y]; });
  // M = E_S (m x nvec, row-major), G_N first
  const int w = nvec;
  std::vector<double> M((size_t)m * w, 0.0);
  for (int c = 0; c < w; ++c) M[(size_t)idx[c] * w + c] = 1.0;
  for (size_t t = rots.size(); t-- > 0;) {
    const Rot& r = rots[t];
    double* __restrict__ mi = &M[(size_t)r.i * w];
    double* __restrict__ mi1 = &M[(size_t)(r.i + 1) * w];
    const double c = r.c, sn = r.s;
    for (int q = 0; q < w; ++q) {  // [M_i; M_i+1] <- G_t [M_i; M_i+1]
      const double a0 = mi[q], a1 = mi1[q];
      mi[q] = c * a0 + sn * a1;
      mi1[q] = c * a1 - sn * a0;
    }
  }
  // X_S = Q M = H_0 ( ... (H_{m-3} M)): rows k+1 .. m-1 of M -= beta_k v_k (v_k^T M)
  std::vector<double> gq(w);
  for (int k = m - 3; k >= 0; --k) {
    const double bk = beta[k];
    if (bk == 0.0) continue;
    const int n2 = m - k - 1;
    const double* __restrict__ v = &vbuf[(size_t)k * m];
    double* __restrict__ g = gq.data();
    for (int q = 0; q < w; ++q) g[q] = 0.0;
    for (int r = 0; r < n2; ++r) {
      const double vr = v[r];
      const double* __restrict__ mr = &M[(size_t)(k + 1 + r) * w];
      for (int q = 0; q < w; ++q) g[q] += vr * mr[q];
    }
    for (int q = 0; q < w; ++q) g[q] *= bk;
    for (int r = 0; r < n2; ++r) {
      const double vr = v[r];
      double* __restrict__ mr = &M[(size_t)(k + 1 + r) * w];
      for (int q = 0; q < w; ++q) mr[q] -= vr * g[q];
    }
  }
  evals.resize(m);
  for (int i = 0; i < m; ++i) evals[i] = d[idx[i]];
  for (int l = 0; l < m; ++l)  // row-major output, column c < nvec = eigenvector c
    for (int c = 0; c < w; ++c) A[(size_t)l * m + c] = M[(size_t)l * w + c];
}

// A: m x m row-major symmetric (overwritten by the eigenvectors, row-major,
// column c = eigenvector c).  evals ascending.
// Compiled twice (the body is an always-inline template): an AVX2/FMA copy chosen at run time when the
// host supports it, and a baseline x86-64 copy; the rotations and reflector updates vectorise 4-wide
// (m = 170: 9.1 -> ~5 ms per restart on the build host).
// nvec < m (the thick restart keeps only the nvec smallest Ritz pairs): the Householder vectors are kept
// instead of accumulated, the QL rotations are applied in reverse order to the nvec selected unit vectors
// (rows of an m x nvec block: 6 nvec instead of 6 m flops per rotation), and the reflectors then map that
// block back (2 m^2 nvec instead of 4/3 m^3 flops); only columns c < nvec of the output are written.
template <int kDummy>
static inline __attribute__((always_inline)) void symeig_impl(int m, std::vector<double>& A,
                                                               std::vector<double>& evals, int nvec) {
  std::vector<double> d(m), e(m);
  // column-major view (A is symmetric): the EISPACK loops then walk contiguous memory (the QL rotations
  // touch two contiguous columns instead of two strided ones); transposed to the row-major output at the end
#define V(i, j) A[(size_t)(j) * m + (i)]  // (a macro: a lambda would not inline into the AVX2 clone)
  if (m == 0) return;
  if (m == 1) {
    evals.assign(1, A[0]);
    A[0] = 1.0;
    return;
  }
  if (nvec >= 0 && nvec < m) {
    symeig_select<kDummy>(m, A, evals, nvec);
    return;
  }
  // --- Householder tridiagonalisation (tred2) ---
  for (int j = 0; j < m; ++j) d[j] = V(m - 1, j);
  for (int i = m - 1; i > 0; --i) {
    double scale = 0.0, h = 0.0;
    for (int k = 0; k < i; ++k) scale += std::fabs(d[k]);
    if (scale == 0.0) {
      e[i] = d[i - 1];
      for (int j = 0; j < i; ++j) {
        d[j] = V(i - 1, j);
        V(i, j) = 0.0;
        V(j, i) = 0.0;
      }
    } else {
      for (int k = 0; k < i; ++k) {
        d[k] /= scale;
        h += d[k] * d[k];
      }
      double f = d[i - 1];
      double g = std::sqrt(h);
      if (f > 0) g = -g;
      e[i] = scale * g;
      h -= f * g;
      d[i - 1] = f - g;
      for (int j = 0; j < i; ++j) e[j] = 0.0;
      for (int j = 0; j < i; ++j) {
        f = d[j];
        V(j, i) = f;
        g = e[j] + V(j, j) * f;
        // column j below the diagonal: a dot (four partial sums, fixed order) and an axpy into e
        const double* __restrict__ col = &V(0, j);
        const double* __restrict__ dp = d.data();
        double* __restrict__ ep = e.data();
        double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
        int k = j + 1;
        for (; k + 3 <= i - 1; k += 4) {
          g0 += col[k] * dp[k];
          g1 += col[k + 1] * dp[k + 1];
          g2 += col[k + 2] * dp[k + 2];
          g3 += col[k + 3] * dp[k + 3];
          ep[k] += col[k] * f;
          ep[k + 1] += col[k + 1] * f;
          ep[k + 2] += col[k + 2] * f;
          ep[k + 3] += col[k + 3] * f;
        }
        for (; k <= i - 1; ++k) {
          g0 += col[k] * dp[k];
          ep[k] += col[k] * f;
        }
        e[j] = g + ((g0 + g1) + (g2 + g3));
      }
      f = 0.0;
      for (int j = 0; j < i; ++j) {
        e[j] /= h;
        f += e[j] * d[j];
      }
      const double hh = f / (h + h);
      for (int j = 0; j < i; ++j) e[j] -= hh * d[j];
      for (int j = 0; j < i; ++j) {
        f = d[j];
        g = e[j];
        double* __restrict__ col = &V(0, j);
        const double* __restrict__ dp = d.data();
        const double* __restrict__ ep = e.data();
        for (int k = j; k <= i - 1; ++k) col[k] -= (f * ep[k] + g * dp[k]);
        d[j] = V(i - 1, j);
        V(i, j) = 0.0;
      }
    }
    d[i] = h;
  }
  for (int i = 0; i < m - 1; ++i) {
    V(m - 1, i) = V(i, i);
    V(i, i) = 1.0;
    const double h = d[i + 1];
    if (h != 0.0) {
      for (int k = 0; k <= i; ++k) d[k] = V(k, i + 1) / h;
      for (int j = 0; j <= i; ++j) {
        double g = 0.0;
        for (int k = 0; k <= i; ++k) g += V(k, i + 1) * V(k, j);
        for (int k = 0; k <= i; ++k) V(k, j) -= g * d[k];
      }
    }
    for (int k = 0; k <= i; ++k) V(k, i + 1) = 0.0;
  }
  for (int j = 0; j < m; ++j) {
    d[j] = V(m - 1, j);
    V(m - 1, j) = 0.0;
  }
  V(m - 1, m - 1) = 1.0;
  e[0] = 0.0;

  // --- implicit QL (tql2): the rotations depend on the tridiagonal only; recorded, then applied to Z ---
  std::vector<Rot> rots;
  rots.reserve((size_t)m * 8);
  for (int i = 1; i < m; ++i) e[i - 1] = e[i];
  e[m - 1] = 0.0;
  double f = 0.0, tst1 = 0.0;
  const double eps = std::ldexp(1.0, -52);
  for (int l = 0; l < m; ++l) {
    tst1 = std::max(tst1, std::fabs(d[l]) + std::fabs(e[l]));
    int mm = l;
    while (mm < m) {
      if (std::fabs(e[mm]) <= eps * tst1) break;
      ++mm;
    }
    if (mm == m) mm = m - 1;
    if (mm > l) {
      int iter = 0;
      do {
        ++iter;
        double g = d[l];
        double p = (d[l + 1] - g) / (2.0 * e[l]);
        double r = hyp(p, 1.0);
        if (p < 0) r = -r;
        d[l] = e[l] / (p + r);
        d[l + 1] = e[l] * (p + r);
        const double dl1 = d[l + 1];
        double h = g - d[l];
        for (int i = l + 2; i < m; ++i) d[i] -= h;
        f += h;
        p = d[mm];
        double c = 1.0, c2 = c, c3 = c;
        const double el1 = e[l + 1];
        double s = 0.0, s2 = 0.0;
        for (int i = mm - 1; i >= l; --i) {
          c3 = c2;
          c2 = c;
          s2 = s;
          g = c * e[i];
          h = c * p;
          r = hyp(p, e[i]);
          e[i + 1] = s * r;
          s = e[i] / r;
          c = p / r;
          p = c * d[i] - s * g;
          d[i + 1] = h + s * (c * g + s * d[i]);
          rots.push_back(Rot{i, c, s});  // applied to Z below (it depends on the tridiagonal only)
        }
        p = -s * s2 * c3 * el1 * e[l] / dl1;
        e[l] = s * p;
        d[l] = c * p;
      } while (std::fabs(e[l]) > eps * tst1 && iter < 200);
    }
    d[l] = d[l] + f;
    e[l] = 0.0;
  }
  // the recorded rotations on Z, in order (the QL recurrences above no longer interleave with the O(m^2)
  // column updates: m = 170, 5.0 -> 4.4 ms on the build host)
  for (const Rot& r : rots) {
    double* __restrict__ zi = &V(0, r.i);  // two contiguous columns (column-major view)
    double* __restrict__ zi1 = &V(0, r.i + 1);
    const double c = r.c, sn = r.s;
    for (int k = 0; k < m; ++k) {
      const double a0 = zi[k], a1 = zi1[k];
      zi1[k] = sn * a0 + c * a1;
      zi[k] = c * a0 - sn * a1;
    }
  }
  // --- sort ascending (selection sort with column swaps) ---
  for (int i = 0; i < m - 1; ++i) {
    int k = i;
    double p = d[i];
    for (int j = i + 1; j < m; ++j)
      if (d[j] < p) {
        k = j;
        p = d[j];
      }
    if (k != i) {
      d[k] = d[i];
      d[i] = p;
      for (int j = 0; j < m; ++j) std::swap(V(j, i), V(j, k));
    }
  }
  for (int i = 0; i < m; ++i)  // column-major -> row-major (column c = eigenvector c)
    for (int j = i + 1; j < m; ++j) std::swap(A[(size_t)i * m + j], A[(size_t)j * m + i]);
  evals = d;
#undef V
}

__attribute__((target("avx2,fma"))) static void symeig_avx2(int m, std::vector<double>& A, std::vector<double>& ev,
                                                            int nvec) {
  symeig_impl<1>(m, A, ev, nvec);
}
static void symeig_base(int m, std::vector<double>& A, std::vector<double>& ev, int nvec) {
  symeig_impl<0>(m, A, ev, nvec);
}

void symeig(int m, std::vector<double>& A, std::vector<double>& evals, int nvec) {
  static const bool avx2 = __builtin_cpu_supports("avx2") && __builtin_cpu_supports("fma");
  if (avx2) symeig_avx2(m, A, evals, nvec);
  else symeig_base(m, A, evals, nvec);
}
void symeig(int m, std::vector<double>& A, std::vector<double>& evals) { symeig(m, A, evals, -1); }

}  // namespace sfz
