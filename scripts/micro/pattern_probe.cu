// Pattern-only SpMV probe: unit-weight graphs need no value stream (t = W x
// streams 4 B/nnz of column indices instead of 12 B/nnz).  Derived from the
// SpMM probe for block Lanczos: Y = W X with X row-major
// n x b (b = 1, 2, 4, 8) on a cfg-4-sized random graph (n = 4M, 32 nnz/row,
// uniform random sorted columns, fp64 values).  Answers: how does the cost of
// one SpMM grow with b when the SpMV is bound by random L2 sector requests?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o spmm_probe spmm_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ int ld_s(const int* p) {
  int v;
  asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_s(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// variant A: VS lanes per row, each lane one nnz at a time, loads all B values of x row (vectorised)
template <int VS, int B>
__global__ void __launch_bounds__(256) spmm_a(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                              const double* __restrict__ vv, const double* __restrict__ X,
                                              double* __restrict__ Y) {
  const int lane = threadIdx.x % VS;
  const int row0 = (blockIdx.x * 256 + threadIdx.x) / VS;
  const int rstride = gridDim.x * 256 / VS;
  for (int row = row0; row < n; row += rstride) {
    double acc[B];
#pragma unroll
    for (int c = 0; c < B; ++c) acc[c] = 0.0;
    const int a = __ldg(rp + row), e1 = __ldg(rp + row + 1);
    int e = a + lane;
    for (; e + VS < e1; e += 2 * VS) {
      const int c0 = ld_s(ci + e), c1 = ld_s(ci + e + VS);
      const double w0 = ld_s(vv + e), w1 = ld_s(vv + e + VS);
      double x0[B], x1[B];
      if (B == 1) {
        x0[0] = __ldg(X + c0);
        x1[0] = __ldg(X + c1);
      } else {
#pragma unroll
        for (int c = 0; c < B; c += 2) {
          const double2 u = __ldg(reinterpret_cast<const double2*>(X + (size_t)c0 * B + c));
          const double2 v = __ldg(reinterpret_cast<const double2*>(X + (size_t)c1 * B + c));
          x0[c] = u.x; x0[c + 1] = u.y; x1[c] = v.x; x1[c + 1] = v.y;
        }
      }
#pragma unroll
      for (int c = 0; c < B; ++c) acc[c] = fma(w1, x1[c], fma(w0, x0[c], acc[c]));
    }
    if (e < e1) {
      const int c0 = ld_s(ci + e);
      const double w0 = ld_s(vv + e);
#pragma unroll
      for (int c = 0; c < B; ++c) acc[c] = fma(w0, __ldg(X + (size_t)c0 * B + c), acc[c]);
    }
#pragma unroll
    for (int c = 0; c < B; ++c)
#pragma unroll
      for (int o = VS / 2; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < B; ++c) Y[(size_t)row * B + c] = acc[c];
  }
}

// variant B: B lanes cooperate on one nnz (lane c loads x[col*B + c]); NZ nnz slots per row group
template <int B, int NZ>
__global__ void __launch_bounds__(256) spmm_b(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                              const double* __restrict__ vv, const double* __restrict__ X,
                                              double* __restrict__ Y) {
  constexpr int G = B * NZ;  // lanes per row
  const int lane = threadIdx.x % G, c = lane % B, z = lane / B;
  const int row0 = (blockIdx.x * 256 + threadIdx.x) / G;
  const int rstride = gridDim.x * 256 / G;
  for (int row = row0; row < n; row += rstride) {
    double acc = 0.0;
    const int a = __ldg(rp + row), e1 = __ldg(rp + row + 1);
    int e = a + z;
    for (; e + NZ < e1; e += 2 * NZ) {
      const int c0 = ld_s(ci + e), c1 = ld_s(ci + e + NZ);
      const double w0 = ld_s(vv + e), w1 = ld_s(vv + e + NZ);
      acc = fma(w0, __ldg(X + (size_t)c0 * B + c), acc);
      acc = fma(w1, __ldg(X + (size_t)c1 * B + c), acc);
    }
    if (e < e1) acc = fma(ld_s(vv + e), __ldg(X + (size_t)ld_s(ci + e) * B + c), acc);
#pragma unroll
    for (int o = G / 2; o >= B; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (z == 0) Y[(size_t)row * B + c] = acc;
  }
}


// variant P: pattern only (unit weights), U gathers in flight per lane
template <int VS, int U>
__global__ void __launch_bounds__(256) spmv_p(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                              const double* __restrict__ X, double* __restrict__ Y) {
  const int lane = threadIdx.x % VS;
  const int row0 = (blockIdx.x * 256 + threadIdx.x) / VS;
  const int rstride = gridDim.x * 256 / VS;
  for (int row = row0; row < n; row += rstride) {
    double acc = 0.0;
    const int a = __ldg(rp + row), e1 = __ldg(rp + row + 1);
    for (int e0 = a + lane; e0 < e1; e0 += U * VS) {
      int c[U];
#pragma unroll
      for (int q = 0; q < U; ++q) c[q] = e0 + q * VS < e1 ? ld_s(ci + e0 + q * VS) : -1;
#pragma unroll
      for (int q = 0; q < U; ++q) acc += c[q] >= 0 ? __ldg(X + c[q]) : 0.0;
    }
#pragma unroll
    for (int o = VS / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) Y[row] = acc;
  }
}
// variant V: values streamed, U gathers in flight per lane (the library's scheme)
template <int VS, int U>
__global__ void __launch_bounds__(256) spmv_v(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                              const double* __restrict__ vv, const double* __restrict__ X,
                                              double* __restrict__ Y) {
  const int lane = threadIdx.x % VS;
  const int row0 = (blockIdx.x * 256 + threadIdx.x) / VS;
  const int rstride = gridDim.x * 256 / VS;
  for (int row = row0; row < n; row += rstride) {
    double acc = 0.0;
    const int a = __ldg(rp + row), e1 = __ldg(rp + row + 1);
    for (int e0 = a + lane; e0 < e1; e0 += U * VS) {
      int c[U];
      double w[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const bool ok = e0 + q * VS < e1;
        c[q] = ok ? ld_s(ci + e0 + q * VS) : 0;
        w[q] = ok ? ld_s(vv + e0 + q * VS) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < U; ++q) acc = fma(w[q], __ldg(X + c[q]), acc);
    }
#pragma unroll
    for (int o = VS / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) Y[row] = acc;
  }
}

// variant V2: values streamed, each VS-lane group handles two rows per iteration (2U gathers in flight)
template <int VS, int U>
__global__ void __launch_bounds__(256) spmv_v2(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                               const double* __restrict__ vv, const double* __restrict__ X,
                                               double* __restrict__ Y) {
  const int lane = threadIdx.x % VS;
  const int g0 = (blockIdx.x * 256 + threadIdx.x) / VS;
  const int ng = gridDim.x * 256 / VS;
  for (int row = g0; row < n; row += 2 * ng) {
    const int rowb = row + ng;
    double acc = 0.0, accb = 0.0;
    const int a = __ldg(rp + row), e1 = __ldg(rp + row + 1);
    const int ab = rowb < n ? __ldg(rp + rowb) : 0, e1b = rowb < n ? __ldg(rp + rowb + 1) : 0;
    int e0 = a + lane, f0 = ab + lane;
    while (e0 < e1 || f0 < e1b) {
      int c[U], cb[U];
      double w[U], wb[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const bool ok = e0 + q * VS < e1, okb = f0 + q * VS < e1b;
        c[q] = ok ? ld_s(ci + e0 + q * VS) : 0;
        w[q] = ok ? ld_s(vv + e0 + q * VS) : 0.0;
        cb[q] = okb ? ld_s(ci + f0 + q * VS) : 0;
        wb[q] = okb ? ld_s(vv + f0 + q * VS) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        acc = fma(w[q], __ldg(X + c[q]), acc);
        accb = fma(wb[q], __ldg(X + cb[q]), accb);
      }
      e0 += U * VS;
      f0 += U * VS;
    }
#pragma unroll
    for (int o = VS / 2; o > 0; o >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      accb += __shfl_xor_sync(0xffffffffu, accb, o);
    }
    if (lane == 0) {
      Y[row] = acc;
      if (rowb < n) Y[rowb] = accb;
    }
  }
}
int main() {
  const int n = 4000000, deg = 32;
  const long long nnz = (long long)n * deg;
  std::vector<int> hrp(n + 1), hci(nnz);
  unsigned long long s = 88172645463325252ull;
  for (int i = 0; i <= n; ++i) hrp[i] = i * deg;
  for (int i = 0; i < n; ++i) {
    int* r = hci.data() + (size_t)i * deg;
    for (int q = 0; q < deg; ++q) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      r[q] = (int)(s % n);
    }
    std::sort(r, r + deg);
  }
  int *rp, *ci;
  double *vv, *X, *Y, *flush;
  cudaMalloc(&rp, sizeof(int) * (n + 1));
  cudaMalloc(&ci, sizeof(int) * nnz);
  cudaMalloc(&vv, sizeof(double) * nnz);
  cudaMalloc(&X, sizeof(double) * n);
  cudaMalloc(&Y, sizeof(double) * n);
  cudaMalloc(&flush, 512 << 20);
  cudaMemcpy(rp, hrp.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(ci, hci.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice);
  cudaMemset(vv, 0, sizeof(double) * nnz);
  cudaMemset(X, 0, sizeof(double) * n);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, bool vals, auto fn) {
    float tot = 0;
    for (int r = 0; r < 6; ++r) {
      cudaMemsetAsync(flush, r, 512 << 20);  // evict the CSR from L2
      cudaEventRecord(a);
      fn();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r) tot += ms;
    }
    const double ms = tot / 5;
    const double stream = (vals ? 12.0 : 4.0) * nnz + 4.0 * (n + 1) + 8.0 * n;
    printf("%-34s %9.1f us  stream %6.0f GB/s\n", name, ms * 1e3, stream / (ms * 1e-3) / 1e9);
  };
  for (int gm : {4, 8, 16}) {
    const int grid = sms * gm;
    printf("grid = %d x SMs\n", gm);
    run("values  VS=8 U=4", true, [&] { spmv_v<8, 4><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
    run("values2 VS=8 U=4 (2 rows/group)", true, [&] { spmv_v2<8, 4><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
    run("values2 VS=4 U=4 (2 rows/group)", true, [&] { spmv_v2<4, 4><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
    run("values  VS=8 U=8", true, [&] { spmv_v<8, 8><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
    run("pattern VS=8 U=4", false, [&] { spmv_p<8, 4><<<grid, 256>>>(n, rp, ci, X, Y); });
    run("pattern VS=8 U=2", false, [&] { spmv_p<8, 2><<<grid, 256>>>(n, rp, ci, X, Y); });
    run("pattern VS=4 U=4", false, [&] { spmv_p<4, 4><<<grid, 256>>>(n, rp, ci, X, Y); });
    run("pattern VS=16 U=2", false, [&] { spmv_p<16, 2><<<grid, 256>>>(n, rp, ci, X, Y); });
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
