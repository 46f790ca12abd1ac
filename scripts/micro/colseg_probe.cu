// DRAM efficiency of the basis sweep access pattern on B200: a 4M x J fp64
// basis read per 64/128/256-row chunk (column-major: J separate segments of
// rows*8 bytes, 32 MB apart) vs a row-major chunk (one contiguous block).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o colseg_probe colseg_probe.cu
#include <cuda_runtime.h>
#include <cstdio>

template <int R>
__global__ void __launch_bounds__(256) colmajor(const double* __restrict__ V, long long ld, int n, int J, double* out) {
  double acc = 0.0;
  const int nch = n / R;
  for (int c = blockIdx.x; c < nch; c += gridDim.x) {
    const long long r0 = (long long)c * R;
    // J segments of R rows; 256 threads read double2
    for (int e = threadIdx.x; e < J * (R / 2); e += 256) {
      const int l = e / (R / 2), r2 = e % (R / 2);
      const double2 v = __ldcs(reinterpret_cast<const double2*>(V + (long long)l * ld + r0) + r2);
      acc += v.x + v.y;
    }
  }
  if (acc == 1.2345) out[0] = acc;
}
__global__ void __launch_bounds__(256) rowmajor(const double* __restrict__ V, int n, int J, double* out) {
  double acc = 0.0;
  const int R = 64, nch = n / R;
  for (int c = blockIdx.x; c < nch; c += gridDim.x) {
    const double2* base = reinterpret_cast<const double2*>(V + (long long)c * R * J);
    for (int e = threadIdx.x; e < R * J / 2; e += 256) {
      const double2 v = __ldcs(base + e);
      acc += v.x + v.y;
    }
  }
  if (acc == 1.2345) out[0] = acc;
}
int main() {
  const int n = 4000000, J = 150;
  double *V, *out;
  cudaMalloc(&V, sizeof(double) * (size_t)n * J);
  cudaMalloc(&out, 8);
  cudaMemset(V, 0, sizeof(double) * (size_t)n * J);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* nm, auto fn) {
    fn();
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) fn();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("%-32s %8.1f us  %7.0f GB/s\n", nm, ms * 1e3, 8.0 * n * J / (ms * 1e-3) / 1e9);
  };
  for (int occ : {1, 2, 4}) {
    char s[64];
    sprintf(s, "colmajor R=64  grid=%dxSM", occ); run(s, [&] { colmajor<64><<<sms * occ, 256>>>(V, n, n, J, out); });
    sprintf(s, "colmajor R=128 grid=%dxSM", occ); run(s, [&] { colmajor<128><<<sms * occ, 256>>>(V, n, n, J, out); });
    sprintf(s, "colmajor R=256 grid=%dxSM", occ); run(s, [&] { colmajor<256><<<sms * occ, 256>>>(V, n, n, J, out); });
    sprintf(s, "rowmajor R=64  grid=%dxSM", occ); run(s, [&] { rowmajor<<<sms * occ, 256>>>(V, n, J, out); });
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
