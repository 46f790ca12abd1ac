// Micro: fp64 tensor-core (mma.sync m8n8k4 f64 = DMMA) issue rate per SM, independent accumulators.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters) {
  double acc[8][2];
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1];
  if (s == 12345.678) out[0] = s;
}
int main() {
  double* o;
  cudaMalloc(&o, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  for (int warps : {4, 8, 16, 32}) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<sms, warps * 32>>>(o, 100);
    cudaEventRecord(e0);
    k<<<sms, warps * 32>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = (double)sms * warps * iters * 8 * 512;
    printf("warps/SM=%d: %.1f TFLOP/s fp64 DMMA\n", warps, flops / (ms * 1e-3) / 1e12);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
