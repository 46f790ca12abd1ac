// Which path serves random fp64 gathers from an L2-resident vector fastest on B200?
//   A  LDG (L1tex, one request per sector)            -- the SpMV's current path
//   B  TMA tile::gather4 (4 rows of 16 B per op)      -- p viewed as [n/2][2] fp64, box {2, 1}
//   C  cp.async.bulk 1-D, 16 B per gather
//   D  A and B in the same CTA (warps 0..3 LDG, 4..7 TMA): do the paths add?
// G gathers of random indices (a hash of the gather number: no index stream), n = 4M (32 MB).
// Every wait is bounded (a lost completion exits the kernel instead of hanging).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gp gather_paths.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned hsh(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ void mb_init(unsigned long long* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void mb_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mb_wait(unsigned long long* b, unsigned par) {
  for (int it = 0; it < (1 << 24); ++it) {
    unsigned ok;
    asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                 : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
    if (ok) return true;
  }
  return false;
}

// A: LDG gathers, U in flight per thread
template <int U>
__global__ void gA(const double* __restrict__ x, int n, long long G, double* out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x, T = (long long)gridDim.x * blockDim.x;
  double acc = 0;
  for (long long b = t * U; b < G; b += T * U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(x + hsh((unsigned)(b + u)) % n);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 1.2345) out[0] = acc;
}

// B: TMA gather4.  Each lane issues one gather4 (4 rows x 16 B) per round into its warp's stage;
// S stages per warp in flight.  Warps [w_lo, 8) of each CTA use TMA; warps [0, w_lo) use LDG (mode D).
template <int S, int NW = 8>
__global__ void __launch_bounds__(NW * 32) gB(const __grid_constant__ CUtensorMap tm, const double* __restrict__ x, int n,
                                          long long G, int w_lo, double* out, int* err, int tma_pct = 50) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar[NW][S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
    for (int s = 0; s < S; ++s) mb_init(&bar[warp][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  double acc = 0;
  const int nw_tma = NW - w_lo;
  const long long Gt = w_lo > 0 ? G * tma_pct / 100 : G;
  if (warp >= w_lo) {
    // this warp's share of G: rounds of 128 gathers
    const long long gw = (long long)gridDim.x * nw_tma;
    const long long me = (long long)blockIdx.x * nw_tma + (warp - w_lo);
    const long long per = Gt / gw / 128;  // rounds for this warp
    unsigned char* base = sm + (size_t)(warp - w_lo) * S * 4096;
    for (long long r = 0; r < per + S; ++r) {
      const int s = (int)(r % S);
      if (r >= S) {  // consume round r - S
        if (!mb_wait(&bar[warp][s], (unsigned)(((r - S) / S) & 1))) { if (lane == 0) atomicAdd(err, 1); return; }
        const double2* d = reinterpret_cast<const double2*>(base + s * 4096);
#pragma unroll
        for (int q = 0; q < 4; ++q) acc += d[lane * 8 + q].x;
        __syncwarp();
      }
      if (r < per) {
        if (lane == 0) mb_expect(&bar[warp][s], 2048);
        __syncwarp();
        const unsigned g0 = (unsigned)((me * per + r) * 128 + lane * 4);
        const int r0 = (int)(hsh(g0) % n) >> 1, r1 = (int)(hsh(g0 + 1) % n) >> 1, r2 = (int)(hsh(g0 + 2) % n) >> 1,
                  r3 = (int)(hsh(g0 + 3) % n) >> 1;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4, %5, %6}], [%7];" ::"r"(sa(base + s * 4096 + lane * 128)),  // 128-B aligned destination
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sa(&bar[warp][s]))
            : "memory");
      }
    }
  } else {
    const long long T = (long long)gridDim.x * w_lo * 32, t = (long long)blockIdx.x * w_lo * 32 + threadIdx.x;
    const long long Gh = G - Gt;
    for (long long b = t * 8; b < Gh; b += T * 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(x + hsh((unsigned)(b + u + G)) % n);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
  }
  if (acc == 1.2345) out[0] = acc;
}

// C: cp.async.bulk 1-D, 16 B (aligned pair) per gather; each lane 4 gathers per round
template <int S>
__global__ void __launch_bounds__(256) gC(const double* __restrict__ x, int n, long long G, double* out, int* err) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar[8][S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
    for (int s = 0; s < S; ++s) mb_init(&bar[warp][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  double acc = 0;
  const long long gw = (long long)gridDim.x * 8, me = (long long)blockIdx.x * 8 + warp;
  const long long per = G / gw / 128;
  unsigned char* base = sm + (size_t)warp * S * 2048;
  for (long long r = 0; r < per + S; ++r) {
    const int s = (int)(r % S);
    if (r >= S) {
      if (!mb_wait(&bar[warp][s], (unsigned)(((r - S) / S) & 1))) { if (lane == 0) atomicAdd(err, 1); return; }
      const double2* d = reinterpret_cast<const double2*>(base + s * 2048);
#pragma unroll
      for (int q = 0; q < 4; ++q) acc += d[lane * 4 + q].x;
      __syncwarp();
    }
    if (r < per) {
      if (lane == 0) mb_expect(&bar[warp][s], 2048);
      __syncwarp();
      const unsigned g0 = (unsigned)((me * per + r) * 128 + lane * 4);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = (int)(hsh(g0 + q) % n) & ~1;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
                         sa(base + s * 2048 + lane * 64 + q * 16)),
                     "l"(x + c), "r"(sa(&bar[warp][s]))
                     : "memory");
      }
    }
  }
  if (acc == 1.2345) out[0] = acc;
}

int main(int argc, char** argv) {
  const char mode = argc > 1 ? argv[1][0] : 'A';
  const int n = 4000000;
  const long long G = 128LL << 20;  // 134M gathers
  double *x, *out;
  int* err;
  cudaMalloc(&x, (size_t)n * 8);
  cudaMalloc(&out, 8);
  cudaMalloc(&err, 4);
  cudaMemset(x, 0, (size_t)n * 8);
  cudaMemset(err, 0, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap tm;
  cuuint64_t gdim[2] = {2, (cuuint64_t)n / 2};
  cuuint64_t gstr[1] = {16};
  cuuint32_t box[2] = {2, 1}, es[2] = {1, 1};
  CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode gather map: %d\n", (int)cr);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto fn) {
    fn();
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%-34s error %s\n", name, cudaGetErrorString(e)); exit(1); }
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) fn();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    int he = 0;
    cudaMemcpy(&he, err, 4, cudaMemcpyDeviceToHost);
    printf("%-34s %8.1f us  %7.1f Ggather/s  (timeouts %d)\n", name, ms * 1e3, G / (ms * 1e-3) / 1e9, he);
  };
  if (mode == 'A')
  for (int occ : {4, 8})
    for (int U : {4, 8}) {
      char nm[64];
      sprintf(nm, "A LDG U=%d grid=%dxSM", U, occ);
      if (U == 4) run(nm, [&] { gA<4><<<sms * occ, 256>>>(x, n, G, out); });
      else run(nm, [&] { gA<8><<<sms * occ, 256>>>(x, n, G, out); });
    }
  for (int occ : {1, 2}) {
    char nm[64];
    const int smB = 8 * 3 * 4096, smC = 8 * 4 * 2048;
    cudaFuncSetAttribute(gB<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smB);
    cudaFuncSetAttribute(gC<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smC);
    if (mode == 'B') {
      sprintf(nm, "B TMA gather4 S=3 grid=%dxSM", occ);
      run(nm, [&] { gB<3><<<sms * occ, 256, smB>>>(tm, x, n, G, 0, out, err); });
    }
    if (mode == 'D') {
      cudaFuncSetAttribute(gB<3, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smB);
      for (int pct : {0, 20, 30, 40}) {
        sprintf(nm, "D 8 LDG + 8 gather4 warps, %d%% TMA, grid=%dxSM", pct, occ);
        run(nm, [&] { gB<3, 16><<<sms * occ, 512, smB>>>(tm, x, n, G, 8, out, err, pct); });
      }
    }
    if (mode == 'C') {
      sprintf(nm, "C bulk 16B S=4 grid=%dxSM", occ);
      run(nm, [&] { gC<4><<<sms * occ, 256, smC>>>(x, n, G, out, err); });
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
