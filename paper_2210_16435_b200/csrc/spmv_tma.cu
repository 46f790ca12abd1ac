// libsfairsc — the single-vector SpMV with a TMA-fed CSR stream (A5, §8(a); the
// dominant per-apply cost).
//
//   t = L p,  L p = p - W^ p (normalized, stored values s_i w_ij s_j)
//                 = d o p - W p (unnormalized, reading R1);  epilogue B^T t, p^T t.
//
// Why this layout.  The SpMV moves ~1.55 GB of CSR from HBM and does nnz
// random 8-byte gathers of p (L2-resident).  On B200 both kinds of access end in the same
// per-SM L1 data pipeline (about one wavefront per clock): a gather costs half a wavefront
// (two sectors per wavefront), and the round-1 kernel's unaligned per-row col/val loads cost
// ~0.6 more per entry and 1.3x the minimum L2 sectors.  Here:
//   * the build writes a PADDED copy of the CSR in which every row starts at a multiple of 4
//     entries (pad entries: col = -1, val = 0), its values split by 4-entry block into a "lo"
//     array (entries 0, 1 of every block) and a "hi" array (entries 2, 3), so a lane reads the 4
//     entries of a block with one 16-byte shared load of col and one of each value half —
//     consecutive lanes read consecutive 16 bytes: conflict-free, ~0.1 wavefront per entry;
//   * the CSR never passes through the LSU: a producer warp copies each row-aligned TILE
//     (<= S.tn padded entries, <= S.tr rows) — row_ptr, col, val and the per-row
//     epilogue operands (p_self, d or s, group ids) — into a shared-memory ring with
//     cp.async.bulk (TMA engine, mbarrier completion, L2 evict-first for the stream);
//   * consumer warps take VS lanes per row; lane l handles the row's 4-entry blocks
//     l, l + VS, ...: one 16-byte col load, two 16-byte val loads, 4 independent gathers
//     p[col] (none for a pad), fma in entry order, then a VS-lane shuffle tree; lane 0 writes
//     t_i and accumulates p^T t and B^T t in its row group's shared slots.  Stages are freed
//     per warp (an `empty` mbarrier), never by a CTA-wide barrier.
// A row longer than a tile (heavy-tailed degrees, config 5) is a tile of its own, read from
// global memory by all consumer warps.  Every reduction has a fixed order (bitwise
// reproducible): per-lane entry order, shuffle tree, per-group slots, fixed-order combine of the
// groups, last-CTA ticket over CTAs (kernels.cu).
#include "device_common.cuh"
#include "tma.cuh"

#include <algorithm>
#include <vector>

namespace sfz {

void bump_launch();

namespace {
constexpr int kPad = 4;          // rows start at multiples of kPad entries (16-byte col, 32-byte val)
constexpr int kConsumers = kThreads;           // 8 consumer warps
constexpr int kSpmvThreads = kConsumers + 32;  // + 1 producer warp
constexpr int kMaxStages = 4;
}  // namespace

// stage layout (bytes): [val lo | val hi] (tn f64, absent for unit weights) | col [tn] i32 |
//                       row_ptr [tr + 8] i32 | p_self [tr + 2] f64 | d or s [tr + 2] f64 | group ids [tr + 32] u8
SpmvTileShape spmv_tile_shape(int tn, int tr, int stages, bool unit) {
  SpmvTileShape S;
  S.tn = tn;
  S.tr = tr;
  S.stages = std::max(1, std::min(stages, kMaxStages));
  S.val_off = 0;
  S.col_off = unit ? 0 : tn * 8;
  S.rp_off = S.col_off + tn * 4;
  S.ps_off = (S.rp_off + (tr + 8) * 4 + 15) / 16 * 16;
  S.ds_off = S.ps_off + (tr + 2) * 8;
  S.gr_off = S.ds_off + (tr + 2) * 8;
  S.stage_bytes = ((S.gr_off + tr + 32) + 127) / 128 * 128;
  return S;
}

__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void consumers_sync() {  // named barrier 1 over the consumer warps only
  asm volatile("bar.sync 1, %0;" ::"r"(kConsumers) : "memory");
}

// tiles[t] = (first row, first padded entry) of tile t; tiles[ntiles] = (n, padded nnz).  CTA b
// owns tiles [cta_tiles[b], cta_tiles[b + 1]).  g.rp / g.ci / g.vv are the padded CSR.
template <bool NORM, bool UNIT>
__device__ __forceinline__ void spmv_issue(const GraphDev& g, const SpmvTileShape& S, const double* __restrict__ p_self,
                                           const int2* __restrict__ tiles, int tt, unsigned char* buf,
                                           unsigned long long* bar, uint64_t pol_stream, uint64_t pol_keep) {
  const int2 a = tiles[tt], b = tiles[tt + 1];
  const int ra = a.x, rb = b.x, ea = a.y, eb = b.y;  // ea, eb multiples of kPad
  const int r_al = ra & ~3, r_end = (rb + 1 + 3) & ~3;  // row_ptr[ra .. rb] inclusive
  const int d_al = ra & ~1, d_end = (rb + 1) & ~1;      // f64 per-row operands
  const int g_al = ra & ~15, g_end = (rb + 15) & ~15;   // u8 group ids
  const bool inl = eb - ea <= S.tn && eb > ea;          // a long row (one tile) is read from global memory
  unsigned bytes = (unsigned)(r_end - r_al) * 4u + 2u * (unsigned)(d_end - d_al) * 8u + (unsigned)(g_end - g_al);
  if (inl) bytes += (unsigned)(eb - ea) * (UNIT ? 4u : 12u);
  mbar_arrive_expect_tx(bar, bytes);
  bulk_g2s_hint(buf + S.rp_off, g.rp + r_al, (unsigned)(r_end - r_al) * 4u, bar, pol_stream);
  bulk_g2s_hint(buf + S.ps_off, p_self + d_al, (unsigned)(d_end - d_al) * 8u, bar, pol_keep);
  bulk_g2s_hint(buf + S.ds_off, (NORM ? g.s : g.dg) + d_al, (unsigned)(d_end - d_al) * 8u, bar, pol_stream);
  bulk_g2s_hint(buf + S.gr_off, g.grp + g_al, (unsigned)(g_end - g_al), bar, pol_stream);
  if (inl) {
    bulk_g2s_hint(buf + S.col_off, g.ci + ea, (unsigned)(eb - ea) * 4u, bar, pol_stream);
    if (!UNIT) {  // g.vv = [lo | hi], each half nnz_pad / 2 doubles (g.nnz = padded entries)
      bulk_g2s_hint(buf + S.val_off, g.vv + ea / 2, (unsigned)(eb - ea) * 4u, bar, pol_stream);
      bulk_g2s_hint(buf + S.val_off + S.tn * 4, g.vv + (size_t)g.nnz / 2 + ea / 2, (unsigned)(eb - ea) * 4u, bar,
                    pol_stream);
    }
  }
}

template <int VS, bool NORM, bool UNIT, int UB>
__global__ void __launch_bounds__(kSpmvThreads, 4) k_spmv_tma(GraphDev g, const SpmvTileShape S, const int2* __restrict__ tiles,
                                                               const int* __restrict__ cta_tiles,
                                                               const double* __restrict__ p,
                                                               const double* __restrict__ p_self,
                                                               double* __restrict__ t, double* partials,
                                                               unsigned* counter, double* bsum_t) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long full[kMaxStages], empty[kMaxStages];
  const int NS = S.stages;
  constexpr int NG = kConsumers / VS;
  __shared__ double gsm[NG][kBT];  // per row group: B^T t (kHB) and p^T t
  __shared__ double lred[kConsumers / 32];
  const int tid = threadIdx.x, lane = tid % VS, gid = tid / VS, warp = tid >> 5;
  const int t0 = cta_tiles[blockIdx.x], nt = cta_tiles[blockIdx.x + 1] - t0;
  for (int e = tid; e < NG * kBT; e += kSpmvThreads) (&gsm[0][0])[e] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumers / 32) {  // ---- producer ----
    if ((tid & 31) == 0) {
      uint64_t pol_stream, pol_keep;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
      for (int it = 0; it < nt; ++it) {
        const int st = it % NS;
        if (it >= NS) {
          mbar_wait(&empty[st], (unsigned)(((it / NS) - 1) & 1));
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before async writes
        }
        spmv_issue<NORM, UNIT>(g, S, p_self, tiles, t0 + it, sm + st * S.stage_bytes, &full[st], pol_stream, pol_keep);
      }
    }
  } else {  // ---- consumers ----
    for (int it = 0; it < nt; ++it) {
      const int st = it % NS;
      const unsigned char* buf = sm + st * S.stage_bytes;
      const int2 a = tiles[t0 + it], b = tiles[t0 + it + 1];
      const int ra = a.x, rb = b.x, ea = a.y, eb = b.y;
      mbar_wait(&full[st], (unsigned)((it / NS) & 1));
      const int* srp = reinterpret_cast<const int*>(buf + S.rp_off) + (ra & 3);  // srp[r - ra] = row_ptr[r]
      const double* sps = reinterpret_cast<const double*>(buf + S.ps_off) + (ra & 1);
      const double* sds = reinterpret_cast<const double*>(buf + S.ds_off) + (ra & 1);
      const uint8_t* sgr = reinterpret_cast<const uint8_t*>(buf + S.gr_off) + (ra & 15);
      if (eb - ea <= S.tn) {
        const int4* scol = reinterpret_cast<const int4*>(buf + S.col_off);       // block j: entries ea + 4j ..
        const double2* svlo = reinterpret_cast<const double2*>(buf + S.val_off);  // block j: entries 0, 1
        const double2* svhi = reinterpret_cast<const double2*>(buf + S.val_off + S.tn * 4);  // entries 2, 3
        for (int base = ra; base < rb; base += NG) {  // CTA-uniform trip count (the shuffles below)
          const int r = base + gid;
          const bool valid = r < rb;
          const int b0 = valid ? (srp[r - ra] - ea) / kPad : 0, b1 = valid ? (srp[r - ra + 1] - ea) / kPad : 0;
          double acc = 0.0;
          for (int j0 = b0 + lane; j0 < b1; j0 += UB * VS) {  // blocks j0 + u VS: 4 UB gathers in flight
            int4 cc[UB];
            double2 w01[UB], w23[UB];
            double x[UB][4];
#pragma unroll
            for (int u = 0; u < UB; ++u) {
              const int j = j0 + u * VS;
              cc[u] = j < b1 ? scol[j] : make_int4(-1, -1, -1, -1);
              w01[u] = w23[u] = make_double2(1.0, 1.0);
              if constexpr (!UNIT) {
                if (j < b1) {
                  w01[u] = svlo[j];
                  w23[u] = svhi[j];
                }
              }
            }
#pragma unroll
            for (int u = 0; u < UB; ++u) {
              x[u][0] = cc[u].x >= 0 ? __ldg(p + cc[u].x) : 0.0;
              x[u][1] = cc[u].y >= 0 ? __ldg(p + cc[u].y) : 0.0;
              x[u][2] = cc[u].z >= 0 ? __ldg(p + cc[u].z) : 0.0;
              x[u][3] = cc[u].w >= 0 ? __ldg(p + cc[u].w) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < UB; ++u) {
              if (cc[u].x >= 0) acc = fma(w01[u].x, x[u][0], acc);
              if (cc[u].y >= 0) acc = fma(w01[u].y, x[u][1], acc);
              if (cc[u].z >= 0) acc = fma(w23[u].x, x[u][2], acc);
              if (cc[u].w >= 0) acc = fma(w23[u].y, x[u][3], acc);
            }
          }
#pragma unroll
          for (int o = VS / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, VS);
          if (valid && lane == 0) {
            const double ds = sds[r - ra];
            if constexpr (UNIT && NORM) acc *= ds;
            const double pi = sps[r - ra];
            const double ti = NORM ? pi - acc : fma(ds, pi, -acc);
            t[r] = ti;
            gsm[gid][kHB] = fma(pi, ti, gsm[gid][kHB]);
            const int gg = sgr[r - ra];
            if (gg < kHB) gsm[gid][gg] += NORM ? ds * ti : ti;
          }
        }
      } else {
        // one long row (ra + 1 == rb), streamed from global memory by all consumer warps
        double acc = 0.0;
        for (int e = ea + tid; e < eb; e += kConsumers * 4) {
          int cc[4];
          double ww[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int ee = e + q * kConsumers;
            const bool ok = ee < eb;
            cc[q] = ok ? ld_stream(g.ci + ee) : -1;
            ww[q] = UNIT ? 1.0
                         : (ok && cc[q] >= 0 ? ld_stream(g.vv + ((ee & 2) ? (size_t)g.nnz / 2 : 0) + (ee >> 2) * 2 + (ee & 1))
                                             : 0.0);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (cc[q] >= 0) acc = fma(ww[q], __ldg(p + cc[q]), acc);
        }
        acc = warp_sum(acc);
        if ((tid & 31) == 0) lred[warp] = acc;
        consumers_sync();
        if (tid == 0) {
          double s = 0.0;
#pragma unroll
          for (int w = 0; w < kConsumers / 32; ++w) s += lred[w];
          const double ds = sds[0];
          if constexpr (UNIT && NORM) s *= ds;
          const double pi = sps[0];
          const double ti = NORM ? pi - s : fma(ds, pi, -s);
          t[ra] = ti;
          gsm[0][kHB] = fma(pi, ti, gsm[0][kHB]);
          const int gg = sgr[0];
          if (gg < kHB) gsm[0][gg] += NORM ? ds * ti : ti;
        }
        consumers_sync();  // lred reused by the next long row
      }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&empty[st]);  // this warp is done with stage `st`
    }
  }
  __syncthreads();
  // fixed-order combine of the row groups' slots, then the grid-wide ticket reduction
  if (tid < kBT) {
    double acc = 0.0;
    for (int q = 0; q < NG; ++q) acc += gsm[q][tid];
    partials[(size_t)blockIdx.x * kBT + tid] = acc;
  }
  ticket_finalize<kBT, kSpmvThreads>(partials, counter, bsum_t, kBT);
}

// padded CSR: prp[i] = sum_{r < i} ceil(deg_r / kPad) kPad; pad entries col = -1, val = 0.  Values in the
// split block layout: padded entry e -> pvv[(e & 2 ? npad / 2 : 0) + 2 (e / 4) + (e & 1)]
__device__ __forceinline__ size_t split_index(long long e, long long npad) {
  return (size_t)(((e & 2) ? npad / 2 : 0) + (e >> 2) * 2 + (e & 1));
}
__global__ void k_pad_csr(const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ vv, int n,
                          const int* __restrict__ prp, int* __restrict__ pci, double* __restrict__ pvv) {
  const long long npad = prp[n];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int a = rp[i], b = rp[i + 1], d = prp[i];
    for (int e = a; e < b; ++e) {
      pci[d + e - a] = ci[e];
      if (pvv) pvv[split_index(d + e - a, npad)] = vv[e];
    }
    for (int e = d + (b - a); e < prp[i + 1]; ++e) {
      pci[e] = -1;
      if (pvv) pvv[split_index(e, npad)] = 0.0;
    }
  }
}

// host: padded row offsets, row-aligned tiles (<= S.tn padded entries and <= S.tr rows; a
// longer row alone) and their split over G CTAs by cumulative (entries + 4 rows) weight.
void spmv_tma_layout(const int* hrp, int n, int G, const SpmvTileShape& S, std::vector<int>& prp,
                     std::vector<int2>& tiles, std::vector<int>& cta_tiles) {
  prp.assign(n + 1, 0);
  for (int i = 0; i < n; ++i) prp[i + 1] = prp[i] + (hrp[i + 1] - hrp[i] + kPad - 1) / kPad * kPad;
  tiles.clear();
  int r = 0;
  while (r < n) {
    const int ra = r, ea = prp[r];
    ++r;
    while (r < n && r - ra < S.tr && prp[r + 1] - ea <= S.tn) ++r;
    tiles.push_back(make_int2(ra, ea));
  }
  const int nt = (int)tiles.size();
  tiles.push_back(make_int2(n, prp[n]));
  G = std::max(1, std::min(G, nt));
  cta_tiles.assign(G + 1, nt);
  cta_tiles[0] = 0;
  const long long total = (long long)prp[n] + 4LL * n;
  int q = 0;
  for (int b = 1; b < G; ++b) {
    const long long target = total * b / G;
    while (q < nt && (long long)tiles[q].y + 4LL * tiles[q].x < target) ++q;
    cta_tiles[b] = std::max(cta_tiles[b - 1], q);
  }
}
void launch_pad_csr(const int* rp, const int* ci, const double* vv, int n, const int* prp, int* pci, double* pvv,
                    cudaStream_t st) {
  bump_launch();
  const int grid = std::max(1, std::min((n + kThreads - 1) / kThreads, 148 * 8));
  k_pad_csr<<<grid, kThreads, 0, st>>>(rp, ci, vv, n, prp, pci, pvv);
}
static int smem_bytes(const SpmvTileShape& S) { return S.stages * S.stage_bytes; }

template <int VS, bool NORM, bool UNIT, int UB>
static int spmv_tma_occ_ub(const SpmvTileShape& S) {
  cudaFuncSetAttribute(k_spmv_tma<VS, NORM, UNIT, UB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_spmv_tma<VS, NORM, UNIT, UB>, kSpmvThreads, smem_bytes(S)) !=
      cudaSuccess)
    nb = 1;
  return std::max(1, nb);
}
template <int VS, bool NORM, bool UNIT>
static int spmv_tma_occ(const SpmvTileShape& S) {
  return spmv_tma_occ_ub<VS, NORM, UNIT, 2>(S);
}
template <int VS>
static int spmv_tma_occ_vs(const SpmvTileShape& S, bool norm, bool unit) {
  if (unit) return norm ? spmv_tma_occ<VS, true, true>(S) : spmv_tma_occ<VS, false, true>(S);
  return norm ? spmv_tma_occ<VS, true, false>(S) : spmv_tma_occ<VS, false, false>(S);
}
// resident CTAs per SM of the instantiation a graph will use (the grid is one full wave)
int spmv_tma_ctas_per_sm(int vs, bool normalized, bool unit, const SpmvTileShape& S) {
  switch (vs) {
    case 2: return spmv_tma_occ_vs<2>(S, normalized, unit);
    case 4: return spmv_tma_occ_vs<4>(S, normalized, unit);
    case 8: return spmv_tma_occ_vs<8>(S, normalized, unit);
    case 16: return spmv_tma_occ_vs<16>(S, normalized, unit);
    default: return spmv_tma_occ_vs<32>(S, normalized, unit);
  }
}

template <int VS, bool NORM, bool UNIT, int UB>
static void spmv_tma_launch_ub(const GraphDev& g, const SpmvTileShape& S, const int2* tiles, const int* cta_tiles,
                               int grid, const double* p, const double* ps, double* t, double* partials,
                               unsigned* counter, double* bsum_t, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_spmv_tma<VS, NORM, UNIT, UB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  k_spmv_tma<VS, NORM, UNIT, UB><<<grid, kSpmvThreads, smem_bytes(S), st>>>(g, S, tiles, cta_tiles, p, ps, t, partials,
                                                                           counter, bsum_t);
}
template <int VS, bool NORM, bool UNIT>
static void spmv_tma_launch(const GraphDev& g, const SpmvTileShape& S, const int2* tiles, const int* cta_tiles,
                            int grid, const double* p, const double* ps, double* t, double* partials, unsigned* counter,
                            double* bsum_t, cudaStream_t st) {
  spmv_tma_launch_ub<VS, NORM, UNIT, 2>(g, S, tiles, cta_tiles, grid, p, ps, t, partials, counter, bsum_t, st);
}
template <int VS>
static void spmv_tma_vs(const GraphDev& g, const SpmvTileShape& S, const int2* tiles, const int* cta_tiles, int grid,
                        const double* p, const double* ps, double* t, double* partials, unsigned* counter,
                        double* bsum_t, cudaStream_t st) {
  if (g.unit) {
    if (g.normalized) spmv_tma_launch<VS, true, true>(g, S, tiles, cta_tiles, grid, p, ps, t, partials, counter, bsum_t, st);
    else spmv_tma_launch<VS, false, true>(g, S, tiles, cta_tiles, grid, p, ps, t, partials, counter, bsum_t, st);
  } else {
    if (g.normalized) spmv_tma_launch<VS, true, false>(g, S, tiles, cta_tiles, grid, p, ps, t, partials, counter, bsum_t, st);
    else spmv_tma_launch<VS, false, false>(g, S, tiles, cta_tiles, grid, p, ps, t, partials, counter, bsum_t, st);
  }
}
void launch_spmv_tma(const GraphDev& g, int vs, const SpmvTileShape& S, const int2* tiles, const int* cta_tiles,
                     int grid, const double* p, const double* p_self, double* t, double* partials, unsigned* counter,
                     double* bsum_t, cudaStream_t st) {
  bump_launch();
  const double* ps = p_self ? p_self : p;
  switch (vs) {
    case 2: spmv_tma_vs<2>(g, S, tiles, cta_tiles, grid, p, ps, t, partials, counter, bsum_t, st); break;
    case 4: spmv_tma_vs<4>(g, S, tiles, cta_tiles, grid, p, ps, t, partials, counter, bsum_t, st); break;
    case 8: spmv_tma_vs<8>(g, S, tiles, cta_tiles, grid, p, ps, t, partials, counter, bsum_t, st); break;
    case 16: spmv_tma_vs<16>(g, S, tiles, cta_tiles, grid, p, ps, t, partials, counter, bsum_t, st); break;
    default: spmv_tma_vs<32>(g, S, tiles, cta_tiles, grid, p, ps, t, partials, counter, bsum_t, st); break;
  }
}

}  // namespace sfz
