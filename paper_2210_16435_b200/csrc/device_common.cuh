// Device helpers shared by the libsfairsc kernel files (warp/block reductions,
// last-CTA ticket finalisation, factored-projector coefficients, Philox).
#pragma once
#include "kernels.cuh"

namespace sfz {

// ----------------------------------------------------------------------------
// helpers
// ----------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// streaming (read-once) loads: bypass L1 allocation, read-only path
__device__ __forceinline__ int ld_stream(const int* p) {
  int v;
  asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// Block-wide fixed-order reduction of NV per-thread values; thread q < NV
// writes the CTA partial to out[q].
template <int NV, int NT = kThreads>
__device__ __forceinline__ void block_reduce_store(const double (&v)[NV], double* out) {
  __shared__ double red[NT / 32][NV];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const double x = warp_sum(v[q]);
    if (lane == 0) red[w][q] = x;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double acc = 0.0;
#pragma unroll
    for (int ww = 0; ww < NT / 32; ++ww) acc += red[ww][threadIdx.x];
    out[threadIdx.x] = acc;
  }
}

// Last-CTA-done finalisation: the CTA that takes the last ticket sums the
// grid's partial rows [gridDim.x][NV] in a fixed order and writes out[q]
// for q < nout.  Resets the ticket for the next launch.
template <int NV, int NT = kThreads>
__device__ __forceinline__ void ticket_finalize(const double* partials, unsigned* counter, double* out, int nout) {
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if constexpr (NV > 20) {  // wide rows (block Lanczos): a warp per output, four rows in flight per lane
    for (int q = w; q < nout; q += NT / 32) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int b = lane;
      for (; b + 96 < (int)gridDim.x; b += 128) {
        a0 += __ldcg(partials + (size_t)b * NV + q);
        a1 += __ldcg(partials + (size_t)(b + 32) * NV + q);
        a2 += __ldcg(partials + (size_t)(b + 64) * NV + q);
        a3 += __ldcg(partials + (size_t)(b + 96) * NV + q);
      }
      for (; b < (int)gridDim.x; b += 32) a0 += __ldcg(partials + (size_t)b * NV + q);
      const double acc = warp_sum((a0 + a1) + (a2 + a3));
      if (lane == 0) out[q] = acc;
    }
    if (threadIdx.x == 0) *counter = 0u;
    return;
  }
  // thread t sums the partial rows t, t + NT, ... (all NV entries of a row are independent loads, two rows in
  // flight: a few L2 round trips instead of one per 32 rows), then warp shuffles and the warps in order
  __shared__ double wsum[NT / 32][NV];
  double acc[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
  const int G = (int)gridDim.x;
  int b = threadIdx.x;
  for (; b + NT < G; b += 2 * NT) {
    double x0[NV], x1[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      x0[q] = q < nout ? __ldcg(partials + (size_t)b * NV + q) : 0.0;
      x1[q] = q < nout ? __ldcg(partials + (size_t)(b + NT) * NV + q) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] += x0[q] + x1[q];
  }
  if (b < G) {
#pragma unroll
    for (int q = 0; q < NV; ++q)
      if (q < nout) acc[q] += __ldcg(partials + (size_t)b * NV + q);
  }
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const double x = warp_sum(acc[q]);
    if (lane == 0) wsum[w][q] = x;
  }
  __syncthreads();
  if (threadIdx.x < nout) {
    double a = 0.0;
#pragma unroll
    for (int ww = 0; ww < NT / 32; ++ww) a += wsum[ww][threadIdx.x];
    out[threadIdx.x] = a;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// gam[s] for the factored projector; executed by thread 0, result in smem.
__device__ __forceinline__ void gamma_serial(const double* bsum, double scale, const ProjDesc& pd, double* gam) {
  if (pd.Q) {  // dense orthonormal Q: the coefficients of QQ^T x are Q^T x itself
    for (int s = 0; s < pd.h; ++s) gam[s] = scale * bsum[s];
    return;
  }
  double pi = 0.0;
  for (int s = 0; s < pd.h; ++s) {
    const double c = scale * bsum[s] * pd.isb[s];
    gam[s] = c;
    pi = fma(pd.uh[s], c, pi);
  }
  for (int s = 0; s < pd.h; ++s) gam[s] = (gam[s] - pd.uh[s] * pi) * pd.isb[s];
}

__device__ __forceinline__ void add_group(double (&acc)[kHB], int g, double v) {
#pragma unroll
  for (int q = 0; q < kHB; ++q)
    if (q == g) acc[q] += v;
}

// Projector rows.  Group mode: (QQ^T x)_i = s_i gam[g_i] and B^T x accumulates s_i x_i into group g_i.
// Dense mode (DQ): (QQ^T x)_i = Q[i, :] . gam and Q^T x accumulates Q[i, q] x_i.
template <bool DQ, bool NORM>
__device__ __forceinline__ double proj_row(const GraphDev& g, long long i, const double* gam) {
  if constexpr (DQ) {
    const double* q = g.Q + (size_t)i * g.ldq;
    double a = 0.0;
#pragma unroll
    for (int c = 0; c < kHB; ++c)
      if (c < g.qr) a = fma(q[c], gam[c], a);
    return a;
  } else {
    const double gv = gam[g.grp[i]];
    return NORM ? g.s[i] * gv : gv;
  }
}
template <bool DQ, bool NORM>
__device__ __forceinline__ void accum_row(const GraphDev& g, long long i, double x, double (&acc)[kHB]) {
  if constexpr (DQ) {
    const double* q = g.Q + (size_t)i * g.ldq;
#pragma unroll
    for (int c = 0; c < kHB; ++c)
      if (c < g.qr) acc[c] = fma(q[c], x, acc[c]);
  } else {
    add_group(acc, g.grp[i], NORM ? g.s[i] * x : x);
  }
}

// Philox4x32-10 (Salmon et al. SC'11), device implementation.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
  const unsigned M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k.x += W0;
      k.y += W1;
    }
    const unsigned hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const unsigned hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}
__device__ __forceinline__ double philox_uniform(uint64_t seed, unsigned c0, unsigned c1, unsigned c2, unsigned c3) {
  const uint4 x = philox4x32_10(make_uint4(c0, c1, c2, c3), make_uint2((unsigned)seed, (unsigned)(seed >> 32)));
  return ((double)(x.x >> 5) * 67108864.0 + (double)(x.y >> 6)) / 9007199254740992.0;
}


}  // namespace sfz
