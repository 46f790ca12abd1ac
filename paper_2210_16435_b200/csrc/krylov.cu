// libsfairsc — TMA-fed reorthogonalisation sweeps (CGS2 solver option) and the Ritz GEMM (sm_100a).
//
// Sweeps: a persistent CTA per SM walks 64-row chunks of the
// Krylov basis V (column-major, ld = ldv).  For each chunk, warp 0 issues one 2-D
// tensor copy (cp.async.bulk.tensor, the TMA engine) of the (64 rows x J columns)
// box plus 1-D bulk copies of the vector chunk into a shared-memory ring guarded by
// mbarriers (complete_tx), so the basis is streamed from HBM exactly once per sweep
// and both the update r' = r - V c and the dots V^T r' read it from shared memory.
// (One 1-D copy per column only when the driver lacks the tensor-map encoder.)
//
// Ritz GEMM (A10): Vout = V Y on the fp64 tensor cores (DMMA m8n8k4, k_ritz_dmma2);
// register-blocked fp64 FMA (k_ritz_rb) for a basis without 128-row padding.
#include "device_common.cuh"
#include "tma.cuh"

#include <algorithm>
#include <atomic>
#include <cstring>

namespace sfz {

namespace {

constexpr int kR = 64;       // rows per chunk
constexpr int kMaxStages = 8;                // smem ring depth (runtime: as many as fit)
constexpr int kTmaMaxJ = 192;
constexpr size_t kRingBytes = 200 * 1024;    // dynamic shared memory budget for the ring

// issue chunk `c` into stage buffer `buf` (warp 0): one 2-D tensor copy of the
// (64 rows x J columns) basis box + one 1-D copy of the vector chunk, or (use2d
// == 0) one 1-D copy per column.
// stage layout (doubles): [J][kR] basis | x[kR] | s[kR] | grp[kR bytes, padded to 128 B]
// (every stage starts 128-byte aligned: required by the 2-D tensor copy destination)
__host__ __device__ __forceinline__ size_t stage_doubles(int J) { return (size_t)(J + 2) * kR + 16; }

__device__ __forceinline__ void issue_chunk(const SweepArgs& a, const GraphDev& g, bool need_sg, const CUtensorMap* tmap,
                                            int use2d, int c, double* buf, unsigned long long* bar, int lane) {
  const int J = a.J;
  const long long row0 = (long long)c * kR;
  const bool with_s = need_sg && g.normalized;
  unsigned bytes = (unsigned)((J + 1) * kR * sizeof(double));
  if (need_sg) bytes += kR;                                   // group ids
  if (with_s) bytes += kR * sizeof(double);                   // s = d^{-1/2}
  if (lane == 0) mbar_arrive_expect_tx(bar, bytes);
  __syncwarp();
  if (lane == 1 && need_sg) {
    bulk_g2s(buf + (size_t)(J + 2) * kR, g.grp + row0, kR, bar);
    if (with_s) bulk_g2s(buf + (size_t)(J + 1) * kR, g.s + row0, kR * sizeof(double), bar);
  }
  if (use2d) {
    if (lane == 0) {
      tensor2d_g2s(buf, tmap, (int)row0, 0, bar);
      bulk_g2s(buf + (size_t)J * kR, a.xin + row0, kR * sizeof(double), bar);
    }
    return;
  }
  for (int l = lane; l <= J; l += 32) {
    const double* src = (l < J) ? a.V + (long long)l * a.ld + row0 : a.xin + row0;
    bulk_g2s(buf + (size_t)l * kR, src, kR * sizeof(double), bar);
  }
}

}  // namespace

// MODE 0: r = t - s o gam_g, dots V^T r ; 1: r' = r - V c, dots V^T r' ;
// 2: r'' = r - V c, |r''|^2 and B^T r'' (ticket) ; 3: dots V^T x.
template <int MODE, int MAXCW, bool NORM>
__global__ void __launch_bounds__(kThreads, 1) k_sweep_tma(GraphDev g, ProjDesc pd, SweepArgs a, int kStages,
                                                                 const __grid_constant__ CUtensorMap tmap, int use2d) {
  extern __shared__ __align__(128) double dsm[];  // [kStages][(J+1) * kR]
  __shared__ __align__(8) unsigned long long bars[kMaxStages];
  __shared__ double coef[kTmaMaxJ];
  __shared__ double red[4][kR];
  __shared__ double rs[kR];
  __shared__ double gam[256];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int n = g.n, J = a.J;
  const int nchunks = (n + kR - 1) / kR;
  const size_t stage_elems = stage_doubles(J);
  constexpr bool kNeedSG = (MODE == 0 || MODE == 2);

  if (MODE == 1 || MODE == 2)
    for (int l = tid; l < J; l += kThreads) coef[l] = a.coef[l];
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (MODE == 0) {
      __shared__ double gw[256];
      gamma_serial(a.bsum_t, 1.0, pd, gam);
      gamma_serial(a.bsum_w, 1.0, pd, gw);
      for (int s = 0; s < pd.h; ++s) gam[s] = gam[s] - a.sigma * gw[s];
    }
  }
  __syncthreads();

  // chunks of this CTA: c = blockIdx.x + it * gridDim.x
  const int my_chunks = (nchunks - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  if (w == 0) {
    for (int it = 0; it < kStages && it < my_chunks; ++it)
      issue_chunk(a, g, kNeedSG, &tmap, use2d, blockIdx.x + it * gridDim.x, dsm + it * stage_elems, &bars[it], lane);
  }

  double colacc[MAXCW];
#pragma unroll
  for (int cc = 0; cc < MAXCW; ++cc) colacc[cc] = 0.0;
  double gacc[kHB];
#pragma unroll
  for (int q = 0; q < kHB; ++q) gacc[q] = 0.0;
  double nrm = 0.0;

  for (int it = 0; it < my_chunks; ++it) {
    const int c = blockIdx.x + it * gridDim.x;
    const int st = it % kStages;
    const double* buf = dsm + st * stage_elems;
    mbar_wait(&bars[st], (unsigned)((it / kStages) & 1));
    const double* xs = buf + (size_t)J * kR;  // vector chunk
    const double* ss = xs + kR;                 // s chunk (normalized, modes 0/2)
    const uint8_t* gs = reinterpret_cast<const uint8_t*>(ss + kR);  // group ids (modes 0/2)
    const int row0 = c * kR;

    // ---- phase 1: row-wise work ----
    if (MODE == 1 || MODE == 2) {
      const int i = tid % kR, cg = tid / kR;  // 4 column groups
      double part = 0.0;
      for (int l = cg; l < J; l += 4) part = fma(buf[(size_t)l * kR + i], coef[l], part);
      red[cg][i] = part;
      __syncthreads();
      if (tid < kR) {
        const int gi = row0 + tid;
        double x = 0.0;
        if (gi < n) {
          x = xs[tid] - (((red[0][tid] + red[1][tid]) + red[2][tid]) + red[3][tid]);
          a.xout[gi] = x;
          if (MODE == 2) {
            nrm = fma(x, x, nrm);
            add_group(gacc, gs[tid], NORM ? ss[tid] * x : x);
          }
        }
        rs[tid] = x;
      }
    } else if (MODE == 0) {
      if (tid < kR) {
        const int gi = row0 + tid;
        double x = 0.0;
        if (gi < n) {
          x = NORM ? fma(-ss[tid], gam[gs[tid]], xs[tid]) : xs[tid] - gam[gs[tid]];
          a.xout[gi] = x;
        }
        rs[tid] = x;
      }
    } else {  // MODE 3
      if (tid < kR) rs[tid] = (row0 + tid < n) ? xs[tid] : 0.0;
    }
    __syncthreads();

    // ---- phase 2: dots V[chunk, l]^T r  (lane-level partials) ----
    if (MODE != 2) {
      const double r0 = rs[lane], r1 = rs[lane + 32];
#pragma unroll
      for (int cc = 0; cc < MAXCW; ++cc) {
        const int l = w + cc * (kThreads / 32);
        if (l < J) {
          const double* col = buf + (size_t)l * kR;
          colacc[cc] = fma(col[lane], r0, colacc[cc]);
          colacc[cc] = fma(col[lane + 32], r1, colacc[cc]);
        }
      }
    }
    __syncthreads();  // stage `st` fully consumed
    if (w == 0 && it + kStages < my_chunks) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_chunk(a, g, kNeedSG, &tmap, use2d, blockIdx.x + (it + kStages) * gridDim.x, dsm + st * stage_elems,
                  &bars[st], lane);
    }
  }

  if (MODE != 2) {
#pragma unroll
    for (int cc = 0; cc < MAXCW; ++cc) {
      const int l = w + cc * (kThreads / 32);
      if (l < J) {
        const double s = warp_sum(colacc[cc]);
        if (lane == 0) a.partials[(size_t)blockIdx.x * J + l] = s;
      }
    }
  } else {
    double v[1 + kHB];
    v[0] = nrm;
#pragma unroll
    for (int q = 0; q < kHB; ++q) v[1 + q] = gacc[q];
    block_reduce_store<1 + kHB>(v, a.partials + (size_t)blockIdx.x * (1 + kHB));
    ticket_finalize<1 + kHB>(a.partials, a.counter, a.norm_bsum, 1 + min(pd.h, kHB));
  }
}

// ---------------------------------------------------------------------------
// Ritz GEMM  Vout[:, c] = sum_l V[:, l] Y[l, c]
// ---------------------------------------------------------------------------
template <int TN>
__global__ void __launch_bounds__(kThreads) k_ritz_rb(const double* __restrict__ V, long long ld, int n, int m,
                                                      const double* __restrict__ Y, int p, double* __restrict__ Vout) {
  constexpr int TM = 128, KC = 16, CPT = TN / 16;
  __shared__ double As[KC][TM];
  __shared__ double Bs[KC][TN];
  const int ncol = (p + TN - 1) / TN;  // 1-D grid: row tile major, column tiles of a row tile adjacent (L2 reuse)
  const int col0 = (int)(blockIdx.x % ncol) * TN;
  const long long row0 = (long long)(blockIdx.x / ncol) * TM;
  const int tid = threadIdx.x;
  const int rg = tid % 16, cg = tid / 16;
  double acc[8][CPT];
#pragma unroll
  for (int q = 0; q < 8; ++q)
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[q][c] = 0.0;
  for (int k0 = 0; k0 < m; k0 += KC) {
    for (int e = tid; e < KC * TM; e += kThreads) {
      const int kk = e / TM, r = e % TM;
      const int l = k0 + kk;
      const long long i = row0 + r;
      As[kk][r] = (l < m && i < n) ? V[(long long)l * ld + i] : 0.0;
    }
    for (int e = tid; e < KC * TN; e += kThreads) {
      const int kk = e / TN, cc = e % TN;
      const int l = k0 + kk, c = col0 + cc;
      Bs[kk][cc] = (l < m && c < p) ? Y[(size_t)c * m + l] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      double av[8], bv[CPT];
#pragma unroll
      for (int q = 0; q < 8; ++q) av[q] = As[kk][rg + 16 * q];
#pragma unroll
      for (int c = 0; c < CPT; ++c) bv[c] = Bs[kk][cg * CPT + c];
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int c = 0; c < CPT; ++c) acc[q][c] = fma(av[q], bv[c], acc[q][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int col = col0 + cg * CPT + c;
    if (col >= p) continue;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const long long i = row0 + rg + 16 * q;
      if (i < n) Vout[(long long)col * ld + i] = acc[q][c];
    }
  }
}

// ---------------------------------------------------------------------------
// Ritz GEMM v2 (default): Vout = V Y on the fp64 tensor cores (DMMA
// m8n8k4), CTA tile 128 rows x GN columns (GN = 64 / 80 / 96 / 112 / 128: the smallest
// that covers p, so V is streamed once for p <= 128 with little padding), 8 warps
// as 4 (rows) x 2 (cols), each 32 x GN/2 = 4 x GN/16 DMMA tiles.  The V
// tile (16 columns x 128 rows) arrives by cp.async into a double-buffered
// shared-memory ring; the Y tile (column-major m x p, 16 k x 128 cols) is
// register-staged and stored transposed.  Shared-memory row stride 136
// doubles (= 8 mod 16): every fragment load is 2 wavefronts (conflict-free).
// ---------------------------------------------------------------------------
constexpr int kGM = 128, kGN = 128, kGK = 16, kGS = 136, kGStages = 4;

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}

template <int GN>  // CTA tile columns: 64, 80, 96, 112 or 128 (the smallest that covers p, else 128)
__global__ void __launch_bounds__(kThreads, 1) k_ritz_dmma2(const double* __restrict__ V, long long ld, int n, int m,
                                                            const double* __restrict__ Y, int p,
                                                            double* __restrict__ Vout) {
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                           // [kGStages][kGK][kGS]
  double* Bs = gsm + kGStages * kGK * kGS;    // [kGStages][kGK][kGS]
  constexpr int NBT = GN / 16;  // 8-column DMMA tiles per warp (2 warp columns)
  const int ncol = (p + GN - 1) / GN;
  const int col0 = (int)(blockIdx.x % ncol) * GN;
  const long long row0 = (long long)(blockIdx.x / ncol) * kGM;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wr = w & 3, wc = w >> 2;
  const int gq = lane >> 2, tq = lane & 3;
  const int nk = (m + kGK - 1) / kGK;
  // B staging: thread -> (col = tid / 2, 8 consecutive k starting at (tid & 1) * 8), 8-byte cp.async each (the
  // transpose of Y's column-major layout), zero-filled beyond p and m
  const int bcol = tid >> 1, bk0 = (tid & 1) * 8;
  // one k-tile (16 basis columns x 128 rows of V, 16 x GN of Y) into ring stage st as ONE cp.async group
  auto load_tile = [&](int st, int k0) {
    double* dst = As + st * kGK * kGS;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + q * kThreads;     // 16 columns x 64 pairs of rows
      const int kk = e >> 6, r2 = e & 63;
      const int l = k0 + kk;
      const double* src = V + (long long)min(l, m - 1) * ld + row0 + 2 * r2;
      cp_async16(dst + kk * kGS + 2 * r2, src, l < m ? 16 : 0);
    }
    if (bcol < GN) {
      double* bd = Bs + st * kGK * kGS;
      const int c = col0 + bcol;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int l = k0 + bk0 + q;
        const bool ok = c < p && l < m;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_addr(bd + (bk0 + q) * kGS + bcol)),
                     "l"(ok ? Y + (size_t)c * m + l : Y), "r"(ok ? 8 : 0)
                     : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[4][NBT][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < NBT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  // kGStages-deep ring: tiles kt+1 .. kt+kGStages-1 are in flight while tile kt is multiplied (a V tile arrives
  // from HBM in about one tile's DMMA time, so two stages left its latency exposed); one barrier per tile
#pragma unroll
  for (int s0 = 0; s0 < kGStages - 1; ++s0) {
    if (s0 < nk) load_tile(s0, s0 * kGK);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kGStages - 2) : "memory");
    __syncthreads();  // tile kt visible to all; stage (kt - 1) % kGStages free (everyone finished tile kt - 1)
    const int kn = kt + kGStages - 1;
    if (kn < nk) load_tile(kn % kGStages, kn * kGK);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    const double* A = As + (kt % kGStages) * kGK * kGS;
    const double* B = Bs + (kt % kGStages) * kGK * kGS;
#pragma unroll
    for (int ks = 0; ks < kGK; ks += 4) {
      double af[4], bf[NBT];
#pragma unroll
      for (int a = 0; a < 4; ++a) af[a] = A[(ks + tq) * kGS + wr * 32 + a * 8 + gq];
#pragma unroll
      for (int b = 0; b < NBT; ++b) bf[b] = B[(ks + tq) * kGS + wc * (GN / 2) + b * 8 + gq];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < NBT; ++b)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[a][b][0]), "+d"(acc[a][b][1])
                       : "d"(af[a]), "d"(bf[b]));
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const long long i = row0 + wr * 32 + a * 8 + gq;
    if (i >= n) continue;
#pragma unroll
    for (int b = 0; b < NBT; ++b)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int col = col0 + wc * (GN / 2) + b * 8 + 2 * tq + q;
        if (col < p) Vout[(long long)col * ld + i] = acc[a][b][q];
      }
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
void bump_launch();

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool encode_colmajor_map(const double* base, long long ld, int cols, int box_rows, CUtensorMap* m) {
  auto fn = get_encode();
  if (!fn || cols < 1 || cols > 256) return false;
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)cols};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// tensor map over V viewed as 2-D [J columns][ld rows] (fp64), box {64 rows, J columns}
static bool encode_basis_map(const SweepArgs& a, CUtensorMap* m) { return encode_colmajor_map(a.V, a.ld, a.J, kR, m); }

template <int MODE, int MAXCW, bool NORM>
static void tma_launch(const GraphDev& g, const ProjDesc& pd, const SweepArgs& a, int grid, cudaStream_t st) {
  const size_t stage = stage_doubles(a.J) * sizeof(double);
  const int stages = (int)std::max<size_t>(2, std::min<size_t>(kMaxStages, kRingBytes / stage));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sweep_tma<MODE, MAXCW, NORM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)std::max(kRingBytes, 2 * stage_doubles(kTmaMaxJ) * sizeof(double)));
    attr = true;
  }
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof(tmap));
  const int use2d = encode_basis_map(a, &tmap);  // 1-D copies per column only if the driver lacks the encoder
  k_sweep_tma<MODE, MAXCW, NORM><<<grid, kThreads, stages * stage, st>>>(g, pd, a, stages, tmap, use2d);
}

template <int MODE, bool NORM>
static void tma_m(const GraphDev& g, const ProjDesc& pd, const SweepArgs& a, int grid, cudaStream_t st) {
  if (a.J <= 64) tma_launch<MODE, 8, NORM>(g, pd, a, grid, st);
  else if (a.J <= 128) tma_launch<MODE, 16, NORM>(g, pd, a, grid, st);
  else tma_launch<MODE, 24, NORM>(g, pd, a, grid, st);
}
template <int MODE>
static void tma_n(const GraphDev& g, const ProjDesc& pd, const SweepArgs& a, int grid, cudaStream_t st) {
  if (g.normalized) tma_m<MODE, true>(g, pd, a, grid, st);
  else tma_m<MODE, false>(g, pd, a, grid, st);
}

bool sweep_tma_ok(int J) { return J >= 1 && J <= kTmaMaxJ; }
int sweep_tma_grid(int n, int num_sms) { return std::max(1, std::min((n + kR - 1) / kR, num_sms)); }

void launch_sweep_tma(int mode, const GraphDev& g, const ProjDesc& pd, const SweepArgs& a, int grid, cudaStream_t st) {
  bump_launch();
  switch (mode) {
    case 0: tma_n<0>(g, pd, a, grid, st); break;
    case 1: tma_n<1>(g, pd, a, grid, st); break;
    case 2: tma_n<2>(g, pd, a, grid, st); break;
    default: tma_n<3>(g, pd, a, grid, st); break;
  }
}

void launch_ritz_rb(const double* V, long long ld, int n, int m, const double* Y, int p, double* Vout,
                    cudaStream_t st) {
  if (p <= 0 || n <= 0) return;
  bump_launch();
  if (ld % 2 == 0 && ld >= (long long)((n + kGM - 1) / kGM) * kGM) {  // DMMA tiles (every library-owned basis)
    const int smem = 2 * kGStages * kGK * kGS * (int)sizeof(double);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_ritz_dmma2<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_ritz_dmma2<80>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_ritz_dmma2<96>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_ritz_dmma2<112>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_ritz_dmma2<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr = true;
    }
    const long long rows = (n + kGM - 1) / kGM;
    if (p <= 64) k_ritz_dmma2<64><<<rows, kThreads, smem, st>>>(V, ld, n, m, Y, p, Vout);
    else if (p <= 80) k_ritz_dmma2<80><<<rows, kThreads, smem, st>>>(V, ld, n, m, Y, p, Vout);
    else if (p <= 96) k_ritz_dmma2<96><<<rows, kThreads, smem, st>>>(V, ld, n, m, Y, p, Vout);
    else if (p <= 112) k_ritz_dmma2<112><<<rows, kThreads, smem, st>>>(V, ld, n, m, Y, p, Vout);
    else k_ritz_dmma2<128><<<rows * ((p + kGN - 1) / kGN), kThreads, smem, st>>>(V, ld, n, m, Y, p, Vout);
    return;
  }
  // fallback (a basis without 128-row padding): register-blocked FMA
  if (p <= 32) {
    const long long grid = (long long)((p + 31) / 32) * ((n + 127) / 128);
    k_ritz_rb<32><<<grid, kThreads, 0, st>>>(V, ld, n, m, Y, p, Vout);
  } else {
    const long long grid = (long long)((p + 63) / 64) * ((n + 127) / 128);
    k_ritz_rb<64><<<grid, kThreads, 0, st>>>(V, ld, n, m, Y, p, Vout);
  }
}

}  // namespace sfz
