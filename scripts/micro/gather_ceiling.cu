// Random-gather ceiling on B200: G gathers of fp64 from an n-vector (L2-resident
// for n = 4M), int32 indices streamed, U independent gathers per thread.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
template <int U>
__global__ void gather(const int* __restrict__ idx, const double* __restrict__ x, double* out, long long G) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  double acc = 0;
  for (long long base = t * U; base < G; base += stride * U) {
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = __ldg(idx + base + u);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += __ldg(x + c[u]);
  }
  if (acc == 123.456) out[0] = acc;
}
__global__ void stream(const int* __restrict__ idx, const double* __restrict__ v, double* out, long long G) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  double acc = 0;
  for (long long i = t; i < G; i += stride) acc += v[i] * idx[i];
  if (acc == 123.456) out[0] = acc;
}
int main() {
  const int n = 4000000; const long long G = 128000000;
  int* idx; double *x, *out, *v;
  cudaMalloc(&idx, G * 4); cudaMalloc(&x, n * 8); cudaMalloc(&out, 8); cudaMalloc(&v, G * 8);
  int* h = (int*)malloc(G * 4); srand(1);
  for (long long i = 0; i < G; ++i) h[i] = (int)(((unsigned long long)rand() * 2654435761ull + i * 40503ull) % n);
  cudaMemcpy(idx, h, G * 4, cudaMemcpyHostToDevice);
  cudaMemset(x, 0, n * 8); cudaMemset(v, 0, G * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](const char* name, auto fn) {
    fn(); cudaEventRecord(a); for (int r = 0; r < 5; ++r) fn(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    printf("%-28s %8.1f us  %7.1f Ggather/s\n", name, ms * 1e3, G / (ms * 1e-3) / 1e9);
  };
  for (int occ : {4, 8, 16}) {
    char nm[64];
    sprintf(nm, "gather U=4 grid=%dxSM", occ); run(nm, [&] { gather<4><<<sms * occ, 256>>>(idx, x, out, G); });
    sprintf(nm, "gather U=8 grid=%dxSM", occ); run(nm, [&] { gather<8><<<sms * occ, 256>>>(idx, x, out, G); });
    sprintf(nm, "gather U=16 grid=%dxSM", occ); run(nm, [&] { gather<16><<<sms * occ, 256>>>(idx, x, out, G); });
  }
  run("stream idx+val (1.5GB)", [&] { stream<<<sms * 8, 256>>>(idx, v, out, G); });
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
