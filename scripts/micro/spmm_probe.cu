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
  cudaMalloc(&X, sizeof(double) * n * 8);
  cudaMalloc(&Y, sizeof(double) * n * 8);
  cudaMalloc(&flush, 512 << 20);
  cudaMemcpy(rp, hrp.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(ci, hci.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice);
  cudaMemset(vv, 0, sizeof(double) * nnz);
  cudaMemset(X, 0, sizeof(double) * n * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, int B, auto fn) {
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
    const double alg = 12.0 * nnz + 4.0 * (n + 1) + 2.0 * 8 * n * B;
    printf("%-30s b=%d %9.1f us  %7.1f us/vector  alg %6.0f GB/s\n", name, B, ms * 1e3, ms * 1e3 / B,
           alg / (ms * 1e-3) / 1e9);
  };
  const int grid = sms * 8;
  run("A VS=8", 1, [&] { spmm_a<8, 1><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
  run("A VS=4", 1, [&] { spmm_a<4, 1><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
  run("A VS=8", 2, [&] { spmm_a<8, 2><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
  run("A VS=4", 2, [&] { spmm_a<4, 2><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
  run("A VS=8", 4, [&] { spmm_a<8, 4><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
  run("A VS=4", 4, [&] { spmm_a<4, 4><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
  run("A VS=8", 8, [&] { spmm_a<8, 8><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
  run("A VS=4", 8, [&] { spmm_a<4, 8><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
  run("B NZ=4", 2, [&] { spmm_b<2, 4><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
  run("B NZ=8", 2, [&] { spmm_b<2, 8><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
  run("B NZ=4", 4, [&] { spmm_b<4, 4><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
  run("B NZ=8", 4, [&] { spmm_b<4, 8><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
  run("B NZ=2", 8, [&] { spmm_b<8, 2><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
  run("B NZ=4", 8, [&] { spmm_b<8, 4><<<grid, 256>>>(n, rp, ci, vv, X, Y); });
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
