// Micro: fp64 vector DADD/DMUL/DFMA issue rate per SM (independent chains).
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, int iters, double a, double b) {
  double x[8];
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) x[j] = __dadd_rn(x[j], a);
      else if (OP == 1) x[j] = __dmul_rn(x[j], b);
      else x[j] = __fma_rn(x[j], b, a);
    }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;
}
int main() {
  double* o;
  cudaMalloc(&o, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 20000;
  for (int op = 0; op < 3; ++op)
    for (int thr : {256, 512, 1024}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto launch = [&] {
        if (op == 0) k<0><<<sms * 2, thr>>>(o, iters, 1e-9, 1.0000001);
        else if (op == 1) k<1><<<sms * 2, thr>>>(o, iters, 1e-9, 1.0000001);
        else k<2><<<sms * 2, thr>>>(o, iters, 1e-9, 1.0000001);
      };
      launch();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)sms * 2 * thr * iters * 8;
      printf("op=%s threads/CTA=%d: %.2f Gop/s = %.1f ops/clk/SM (at %d MHz nominal)\n", op == 0 ? "DADD" : op == 1 ? "DMUL" : "DFMA",
             thr, ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  return 0;
}
