// CSR SpMM Y = A X on a tall-skinny row-major block (Alg. 1 S1/S3,
// Alg. 2 S2/S4; P:416 stores A as CSR).  A^T X uses the same kernels on the
// precomputed CSR(A^T) (built here by a stable counting sort), so the
// transposed product needs no atomics (north_star; P:460/P:498 note that
// cuSPARSE's implicitly transposed SpMM is the paper's bottleneck).
//
// Load balance for power-law rows:
//  * short rows (<= kLongRow nonzeros): a group of L lanes per row, each
//    lane owns VEC (2 when aligned) output columns; nonzeros in masked
//    batches of 8 so eight independent row gathers of X are in flight;
//  * long rows: split into segments of <= kSeg nonzeros, one CTA per segment
//    (256/L groups strided over the segment, fixed-order smem reduction);
//    rows with several segments write partials that a fix-up kernel sums in
//    segment order.  Deterministic: no floating-point atomics anywhere.
#include <algorithm>
#include <array>
#include <cstdlib>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "internal.h"
#include "ptx.cuh"

namespace tsvd {

constexpr int kLongRow = 64;   // rows up to this length: sub-warp groups (sorted)
constexpr int kMedRow = 512;   // rows up to this length: one warp each (sorted)
constexpr int kSeg = 2048;     // longer rows: CTA segments of this many nonzeros
constexpr int kPartW = 64;     // columns per partial slot of a split long row (w <= 64)

template <int VEC>
__device__ __forceinline__ void ldx_vec(const double* p, double (&x)[VEC]) {
  if constexpr (VEC == 2) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(p));
    x[0] = t.x;
    x[1] = t.y;
  } else {
    x[0] = __ldg(p);
  }
}

// Short rows: a group of L lanes per row, lane owns VEC consecutive output
// columns (double2 gathers when the block width and ld are even).  Nonzeros
// are consumed in batches of 8 with masked loads, so a row of <= 8 nonzeros
// costs one index-load + one gather round trip and 8 independent row
// gathers per lane are in flight.
template <int L, int VEC>
__device__ __forceinline__ void spmm_short_dev(
    const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colidx,
    const double* __restrict__ vals, const double* __restrict__ X, int64_t ldx,
    double* __restrict__ Y, int64_t ldy, const int32_t* __restrict__ perm, int64_t nrows,
    int w, int64_t bidx) {
  constexpr int RPW = 32 / L;  // rows per warp
  const int lane = threadIdx.x & 31;
  const int64_t warp = (bidx * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t pos = warp * RPW + lane / L;
  const int c = (lane % L) * VEC;
  if (pos >= nrows) return;
  // row-sorted layout: position pos holds output row perm[pos]; rows of
  // similar length share a warp and their nonzeros are adjacent in memory
  const int64_t row = __ldg(perm + pos);
  const int64_t beg = __ldg(rowptr + pos), end = __ldg(rowptr + pos + 1);
  const bool active = c < w;
  const double* Xc = X + c;
  double acc0[VEC], acc1[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc0[e] = acc1[e] = 0.0;
  for (int64_t k = beg; k < end; k += 8) {
    int32_t col[8];
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool ok = k + u < end;
      col[u] = ok ? __ldg(colidx + k + u) : 0;
      v[u] = ok ? __ldg(vals + k + u) : 0.0;
    }
    double x[8][VEC];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (active && k + u < end)
        ldx_vec<VEC>(Xc + (int64_t)col[u] * ldx, x[u]);
      else
#pragma unroll
        for (int e = 0; e < VEC; ++e) x[u][e] = 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; u += 2)
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        acc0[e] = fma(v[u], x[u][e], acc0[e]);
        acc1[e] = fma(v[u + 1], x[u + 1][e], acc1[e]);
      }
  }
  if (active) {
    if constexpr (VEC == 2) {
      *reinterpret_cast<double2*>(Y + row * ldy + c) = make_double2(acc0[0] + acc1[0], acc0[1] + acc1[1]);
    } else {
      Y[row * ldy + c] = acc0[0] + acc1[0];
    }
  }
}

// Medium rows (kLongRow < len <= kMedRow): one warp per row, 32/L lane groups
// strided over the row's nonzeros (batches of 8 per group), combined by
// xor-shuffles across groups (fixed order).
template <int L, int VEC>
__device__ __forceinline__ void spmm_medium_dev(
    const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colidx,
    const double* __restrict__ vals, const double* __restrict__ X, int64_t ldx,
    double* __restrict__ Y, int64_t ldy, const int32_t* __restrict__ perm, int64_t nrows,
    int w, int64_t bidx) {
  constexpr int G = 32 / L;
  const int lane = threadIdx.x & 31;
  const int64_t widx = (bidx * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (widx >= nrows) return;
  const int g = lane / L, c = (lane % L) * VEC;
  const bool active = c < w;
  const double* Xc = X + c;
  const int64_t row = __ldg(perm + widx);
  const int64_t beg = __ldg(rowptr + widx), end = __ldg(rowptr + widx + 1);
  double acc0[VEC], acc1[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc0[e] = acc1[e] = 0.0;
  for (int64_t k = beg + g; k < end; k += 8 * G) {
    int32_t col[8];
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool ok = k + u * G < end;
      col[u] = ok ? __ldg(colidx + k + u * G) : 0;
      v[u] = ok ? __ldg(vals + k + u * G) : 0.0;
    }
    double x[8][VEC];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (active && k + u * G < end)
        ldx_vec<VEC>(Xc + (int64_t)col[u] * ldx, x[u]);
      else
#pragma unroll
        for (int e = 0; e < VEC; ++e) x[u][e] = 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; u += 2)
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        acc0[e] = fma(v[u], x[u][e], acc0[e]);
        acc1[e] = fma(v[u + 1], x[u + 1][e], acc1[e]);
      }
  }
  double r[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    r[e] = acc0[e] + acc1[e];
#pragma unroll
    for (int o = L; o < 32; o <<= 1) r[e] += __shfl_xor_sync(0xffffffffu, r[e], o);
  }
  if (g == 0 && active) {
    if constexpr (VEC == 2) {
      *reinterpret_cast<double2*>(Y + row * ldy + c) = make_double2(r[0], r[1]);
    } else {
      Y[row * ldy + c] = r[0];
    }
  }
}

// Long rows: one CTA per segment of <= kSeg nonzeros; 256/L groups strided
// over the segment (adjacent groups read adjacent nonzeros), fixed-order
// shared-memory reduction of the groups; a row split into several segments
// writes one partial per segment, summed in segment order by the fix-up.
template <int L, int VEC>
__device__ __forceinline__ void spmm_long_dev(
    const int64_t* __restrict__ seg_row, const int64_t* __restrict__ seg_beg,
    const int64_t* __restrict__ seg_end, const int32_t* __restrict__ seg_slot,
    const int32_t* __restrict__ colidx, const double* __restrict__ vals,
    const double* __restrict__ X, int64_t ldx, double* __restrict__ Y, int64_t ldy, int w,
    double* __restrict__ part, int64_t bidx) {
  constexpr int G = 256 / L, CW = L * VEC;
  __shared__ double red[G][CW + 1];
  const int g = threadIdx.x / L, c = (threadIdx.x % L) * VEC;
  const int64_t s = bidx;
  const int64_t beg = seg_beg[s], end = seg_end[s];
  const bool active = c < w;
  const double* Xc = X + c;
  double acc0[VEC], acc1[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc0[e] = acc1[e] = 0.0;
  for (int64_t k = beg + g; k < end; k += 4 * G) {
    int32_t col[4];
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool ok = k + u * G < end;
      col[u] = ok ? __ldg(colidx + k + u * G) : 0;
      v[u] = ok ? __ldg(vals + k + u * G) : 0.0;
    }
    double x[4][VEC];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (active && k + u * G < end)
        ldx_vec<VEC>(Xc + (int64_t)col[u] * ldx, x[u]);
      else
#pragma unroll
        for (int e = 0; e < VEC; ++e) x[u][e] = 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; u += 2)
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        acc0[e] = fma(v[u], x[u][e], acc0[e]);
        acc1[e] = fma(v[u + 1], x[u + 1][e], acc1[e]);
      }
  }
#pragma unroll
  for (int e = 0; e < VEC; ++e)
    red[g][c + e] = acc0[e] + acc1[e];
  __syncthreads();
  if (threadIdx.x < w) {
    double sum = 0.0;
    for (int gg = 0; gg < G; ++gg) sum += red[gg][threadIdx.x];
    const int slot = seg_slot[s];
    if (slot < 0)
      Y[seg_row[s] * ldy + threadIdx.x] = sum;
    else
      part[(int64_t)slot * kPartW + threadIdx.x] = sum;
  }
}

// One launch for all three row classes so their tails overlap: the heaviest
// units (long-row segments) are scheduled first, then medium rows (one warp
// each), then short rows (sub-warp groups).
template <int L, int VEC>
__global__ void __launch_bounds__(256) spmm_kernel(Csr A, const double* __restrict__ X,
                                                   int64_t ldx, double* __restrict__ Y,
                                                   int64_t ldy, int w, double* __restrict__ part,
                                                   int64_t nb_long, int64_t nb_med,
                                                   int64_t nmed_run, int64_t nshort_run) {
  pdl_enter();
  const int64_t b = blockIdx.x;
  if (b < nb_long) {
    spmm_long_dev<L, VEC>(A.seg_row, A.seg_beg, A.seg_end, A.seg_slot, A.colidx, A.vals, X, ldx,
                          Y, ldy, w, part, b);
  } else if (b < nb_long + nb_med) {
    spmm_medium_dev<L, VEC>(A.rowptr + A.nshort, A.colidx, A.vals, X, ldx, Y, ldy,
                            A.perm + A.nshort, nmed_run, w, b - nb_long);
  } else {
    spmm_short_dev<L, VEC>(A.rowptr, A.colidx, A.vals, X, ldx, Y, ldy, A.perm, nshort_run, w,
                           b - nb_long - nb_med);
  }
}

__global__ void spmm_fixup_kernel(const int64_t* __restrict__ split_row,
                                  const int32_t* __restrict__ split_first,
                                  const int32_t* __restrict__ split_count,
                                  const double* __restrict__ part, double* __restrict__ Y,
                                  int64_t ldy, int w, int64_t nsplit) {
  pdl_enter();
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r = t / kPartW;
  const int c = (int)(t % kPartW);
  if (r >= nsplit || c >= w) return;
  const int first = split_first[r], cnt = split_count[r];
  double sum = 0.0;
  for (int j = 0; j < cnt; ++j) sum += part[(int64_t)(first + j) * kPartW + c];
  Y[split_row[r] * ldy + c] = sum;
}

// nmed_run / nshort_run: how many medium / short rows this launch covers
// (the first ones of each section; -1 = all).  With the staged kernel only
// the medium rows longer than its chunk go here.
template <int L, int VEC>
static void spmm_dispatch(const Csr& A, const double* X, int64_t ldx, double* Y, int64_t ldy,
                          int w, double* part, cudaStream_t st, int64_t nmed_run = -1,
                          int64_t nshort_run = -1, bool fixup = true) {
  constexpr int RPW = 32 / L;
  if (nmed_run < 0) nmed_run = A.nmed;
  if (nshort_run < 0) nshort_run = A.nshort;
  const int64_t rows_per_block = 8 * RPW;
  const int64_t nb_short = (nshort_run + rows_per_block - 1) / rows_per_block;
  const int64_t nb_med = (nmed_run + 7) / 8;
  const int64_t nb_long = A.nseg;
  const int64_t blocks = nb_short + nb_med + nb_long;
  if (blocks > 0) {
    launch_pdl(spmm_kernel<L, VEC>, (unsigned)blocks, 256, 0, st, A, X, ldx, Y, ldy, w, part, nb_long,
                                                           nb_med, nmed_run, nshort_run);
    TSVD_CHECK_LAUNCH();
  }
  if (fixup && A.nsplit > 0) {
    const int64_t thr = A.nsplit * kPartW;
    launch_pdl(spmm_fixup_kernel, (unsigned)((thr + 255) / 256), 256, 0, st, A.split_row, A.split_first, A.split_count, part, Y, ldy, w, A.nsplit);
    TSVD_CHECK_LAUNCH();
  }
}


// ------------------------------------------------------- staged SpMM ---
// Rows of length L <= NZC (nonzeros per chunk) go in chunks of R = NZC / L
// rows of one length bin (ELL-like: the row pointer is never read; a
// chunk's nonzeros are one contiguous range of the row-sorted arrays).
// Persistent CTAs = 8 consumer warps + 1 producer warp, two mbarrier rings
// in shared memory:
//   * index ring (NIS stages): a chunk's colidx, vals and output rows arrive
//     by three 1-D bulk copies (TMA engine, SASS UBLKCP), NIS - 1 chunks
//     ahead of the gathers that need them;
//   * gather ring (NXS stages): the producer warp gathers the X row of every
//     nonzero (2 LPR doubles) with TMA tile::gather4 (4 rows per
//     instruction, SASS UTMALDG), NXS - 1 chunks ahead of the consumers.
// So no register holds an in-flight gather, no gather waits behind an index
// load in the same thread, and the number of gathers in flight is bounded by
// shared memory (3 x 32 KB per SM).  Consumers multiply from shared memory:
// groups of LPR lanes own a row (or, for long rows, S = 2^k consecutive
// slices of it whose partials are summed in slice order).  Deterministic,
// no atomics.
template <int LPR>
struct StagedCfg {
  static constexpr int NZC = 2048 / LPR;          // nonzeros per chunk (256 / 128 / 64)
  static constexpr int G = 256 / LPR;             // lane groups of the 8 consumer warps
  static constexpr int NXS = 4;                   // gather stages
  static constexpr int NIS = 8;                   // index stages
  static constexpr int NPW = 4;                   // producer warps (gather4 issue is per
                                                  // lane-serialised: one warp per SMSP)
  static constexpr int NTHR = 256 + 32 * NPW;
  static constexpr int XROWS = NZC + 4;           // gather4 pads the last group of 4
  static constexpr int XD = XROWS * LPR * 2;      // doubles per gather stage (~32 KB)
  static constexpr int CI = NZC + 4, VI = NZC + 2, PI = NZC + 4;  // index stage sizes
  static constexpr int IDXB = ((CI * 4 + VI * 8 + PI * 4) + 15) / 16 * 16;
  static constexpr int MAXB = 260;                // bins with L <= NZC (L = 0..256)
  static constexpr size_t x_off = 0;
  static constexpr size_t i_off = x_off + (size_t)NXS * XD * 8;
  static constexpr size_t r_off = i_off + (size_t)NIS * IDXB;
  static constexpr size_t b_off = r_off + (size_t)G * LPR * 16;
  static constexpr size_t bar_off = b_off + (size_t)MAXB * 40;
  static constexpr size_t bytes = bar_off + (size_t)(2 * NIS + 2 * NXS) * 8 + 128;
};

struct ChunkGeo {
  int L, nr;          // row length, rows in this chunk
  int64_t pos, nz;    // first position, first nonzero
};

__device__ __forceinline__ ChunkGeo chunk_geo(int64_t c, int nb, int nzc, const int* sL,
                                              const int64_t* sCnt, const int64_t* sPos,
                                              const int64_t* sNz, const int64_t* sC0) {
  int lo = 0, hi = nb;  // last bin with sC0[bin] <= c
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (sC0[mid] <= c) lo = mid; else hi = mid;
  }
  ChunkGeo g;
  g.L = sL[lo];
  const int64_t R = g.L ? max(1, nzc / g.L) : nzc;
  const int64_t j = c - sC0[lo];
  g.pos = sPos[lo] + j * R;
  g.nr = (int)min(R, sCnt[lo] - j * R);
  g.nz = sNz[lo] + j * R * g.L;
  return g;
}

template <int LPR>
__global__ void __launch_bounds__(StagedCfg<LPR>::NTHR, 1) spmm_staged_kernel(
    const __grid_constant__ CUtensorMap xmap, const int32_t* __restrict__ colidx,
    const double* __restrict__ vals, const int32_t* __restrict__ perm,
    const int64_t* __restrict__ bins, const int64_t* __restrict__ chunk0, int nb,
    int64_t nchunks, double* __restrict__ Y, int64_t ldy, int w) {
  using C = StagedCfg<LPR>;
  constexpr int NZC = C::NZC, G = C::G, NXS = C::NXS, NIS = C::NIS, XW = 2 * LPR;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* xs = reinterpret_cast<double*>(smraw + C::x_off);
  unsigned char* idx = smraw + C::i_off;
  double2* red = reinterpret_cast<double2*>(smraw + C::r_off);
  int64_t* sCnt = reinterpret_cast<int64_t*>(smraw + C::b_off);
  int64_t* sPos = sCnt + C::MAXB;
  int64_t* sNz = sPos + C::MAXB;
  int64_t* sC0 = sNz + C::MAXB;
  int* sL = reinterpret_cast<int*>(sC0 + C::MAXB);
  uint64_t* ifull = reinterpret_cast<uint64_t*>(smraw + C::bar_off);
  uint64_t* iempty = ifull + NIS;
  uint64_t* xfull = iempty + NIS;
  uint64_t* xempty = xfull + NXS;
  // per index stage: offsets of colidx / vals / perm inside it, L, rows
  __shared__ int sMeta[NIS][5];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int b = tid; b < nb; b += C::NTHR) {
    sL[b] = (int)bins[4 * b];
    sCnt[b] = bins[4 * b + 1];
    sPos[b] = bins[4 * b + 2];
    sNz[b] = bins[4 * b + 3];
    sC0[b] = chunk0[b];
  }
  if (tid == 0) {
    for (int i = 0; i < NIS; ++i) {
      mbar_init(&ifull[i], 1);
      mbar_init(&iempty[i], 8);
    }
    for (int i = 0; i < NXS; ++i) {
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const int64_t c0 = blockIdx.x, cs = gridDim.x;
  const int64_t nmine = c0 < nchunks ? (nchunks - 1 - c0) / cs + 1 : 0;
  auto stage_ci = [&](int s) { return reinterpret_cast<int32_t*>(idx + (size_t)s * C::IDXB); };
  auto stage_va = [&](int s) {
    return reinterpret_cast<double*>(idx + (size_t)s * C::IDXB + C::CI * 4);
  };
  auto stage_pm = [&](int s) {
    return reinterpret_cast<int32_t*>(idx + (size_t)s * C::IDXB + C::CI * 4 + C::VI * 8);
  };

  if (warp >= 8) {
    // --------------------------------------------------------- producers --
    // warp 8 lane 0 also streams the index data; all producer warps split a
    // chunk's gather4s (the first expect_tx may trail some complete_tx: the
    // transaction count may go transiently negative, the phase cannot
    // complete before the arrival)
    const int pw = warp - 8;
    auto issue_idx = [&](int64_t i) {  // lane 0: bulk-copy chunk i's index data
      const int s = (int)(i % NIS);
      if (i >= NIS) mbar_wait(&iempty[s], (unsigned)((i / NIS - 1) & 1));
      const ChunkGeo cg = chunk_geo(c0 + i * cs, nb, NZC, sL, sCnt, sPos, sNz, sC0);
      const int64_t n = (int64_t)cg.nr * cg.L;
      const int64_t ca0 = cg.nz & ~3LL, ca1 = (cg.nz + n + 3) & ~3LL;
      const int64_t va0 = cg.nz & ~1LL, va1 = (cg.nz + n + 1) & ~1LL;
      const int64_t pa0 = cg.pos & ~3LL, pa1 = (cg.pos + cg.nr + 3) & ~3LL;
      const unsigned cb = n ? (unsigned)(ca1 - ca0) * 4 : 0;
      const unsigned vb = n ? (unsigned)(va1 - va0) * 8 : 0;
      const unsigned pb = (unsigned)(pa1 - pa0) * 4;
      sMeta[s][0] = (int)(cg.nz - ca0);
      sMeta[s][1] = (int)(cg.nz - va0);
      sMeta[s][2] = (int)(cg.pos - pa0);
      sMeta[s][3] = cg.L;
      sMeta[s][4] = cg.nr;
      mbar_expect_tx(&ifull[s], cb + vb + pb);  // release: sMeta visible to waiters
      if (cb) bulk_load(stage_ci(s), colidx + ca0, cb, &ifull[s]);
      if (vb) bulk_load(stage_va(s), vals + va0, vb, &ifull[s]);
      bulk_load(stage_pm(s), perm + pa0, pb, &ifull[s]);
    };
    if (pw == 0 && lane == 0)
      for (int64_t i = 0; i < NIS - 1 && i < nmine; ++i) issue_idx(i);
    for (int64_t i = 0; i < nmine; ++i) {
      if (pw == 0 && lane == 0 && i + NIS - 1 < nmine) issue_idx(i + NIS - 1);
      const int s = (int)(i % NIS), xsl = (int)(i % NXS);
      mbar_wait(&ifull[s], (unsigned)((i / NIS) & 1));
      if (i >= NXS) mbar_wait(&xempty[xsl], (unsigned)((i / NXS - 1) & 1));
      const int n = sMeta[s][3] * sMeta[s][4];
      const int n4 = (n + 3) >> 2;
      if (pw == 0 && lane == 0) mbar_expect_tx(&xfull[xsl], (unsigned)n4 * 4 * XW * 8);
      const int32_t* ci = stage_ci(s) + sMeta[s][0];
      double* xd = xs + (size_t)xsl * C::XD;
      for (int k4 = pw * 32 + lane; k4 < n4; k4 += 32 * C::NPW) {
        const int k = 4 * k4;
        const int r0 = ci[k];
        const int r1 = k + 1 < n ? ci[k + 1] : r0;
        const int r2 = k + 2 < n ? ci[k + 2] : r0;
        const int r3 = k + 3 < n ? ci[k + 3] : r0;
        tma_gather4(xd + (size_t)k * XW, &xmap, 0, r0, r1, r2, r3, &xfull[xsl]);
      }
    }
    return;
  }
  // ------------------------------------------------------------ consumers --
  const int g = tid / LPR, ln = tid % LPR;
  const bool lane_on = 2 * ln < w;
  for (int64_t i = 0; i < nmine; ++i) {
    const int s = (int)(i % NIS), xsl = (int)(i % NXS);
    mbar_wait(&xfull[xsl], (unsigned)((i / NXS) & 1));
    mbar_wait(&ifull[s], (unsigned)((i / NIS) & 1));  // long complete (gathers need it)
    const double* va = stage_va(s) + sMeta[s][1];
    const int32_t* pm = stage_pm(s) + sMeta[s][2];
    const double2* xd = reinterpret_cast<const double2*>(xs + (size_t)xsl * C::XD);
    const int L = sMeta[s][3], nr = sMeta[s][4];
    const int R = L ? max(1, NZC / L) : NZC;
    // slices per row: the largest power of two <= G / R (1 if R >= G)
    int lgS = 0;
    while (R < G && (2 << lgS) * R <= G) ++lgS;
    const int S = 1 << lgS;
    for (int task = g; task < (nr << lgS); task += G) {
      const int r = task >> lgS, sl = task & (S - 1);
      const int k0 = r * L + ((sl * L) >> lgS), k1 = r * L + (((sl + 1) * L) >> lgS);
      double a0 = 0.0, a1 = 0.0;
      for (int k = k0; k < k1; ++k) {
        const double v = va[k];
        const double2 x = xd[k * LPR + ln];
        a0 = fma(v, x.x, a0);
        a1 = fma(v, x.y, a1);
      }
      if (S == 1) {
        if (lane_on)
          *reinterpret_cast<double2*>(Y + (int64_t)pm[r] * ldy + 2 * ln) = make_double2(a0, a1);
      } else {
        red[task * LPR + ln] = make_double2(a0, a1);
      }
    }
    if (S > 1) {
      bar_consumers();
      for (int t = tid; t < nr * LPR; t += 256) {
        const int r = t / LPR, l2 = t % LPR;
        double a0 = 0.0, a1 = 0.0;
        for (int sl = 0; sl < S; ++sl) {
          const double2 p = red[((r << lgS) + sl) * LPR + l2];
          a0 += p.x;
          a1 += p.y;
        }
        if (2 * l2 < w)
          *reinterpret_cast<double2*>(Y + (int64_t)pm[r] * ldy + 2 * l2) = make_double2(a0, a1);
      }
      bar_consumers();  // red is reused by the next chunk
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&xempty[xsl]);
      mbar_arrive(&iempty[s]);
    }
  }
}

static bool g_spmm_staged = [] {
  const char* e = getenv("TSVD_SPMM_STAGED");
  return e && e[0] == '1';
}();

// X (rows x w, ld) as a 2-D tensor for tile::gather4: box = {2 LPR, 1}
// (columns >= w are zero-filled by the copy engine)
static bool gather_map(CUtensorMap* m, const double* X, int64_t rows, int w, int64_t ldx,
                       int box_cols) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || rows < 1 || rows > ((int64_t)1 << 31) || ((uintptr_t)X & 15) || (ldx & 1))
    return false;
  const cuuint64_t dims[2] = {(cuuint64_t)w, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ldx * 8};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, 1};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)X, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int LPR>
static bool staged_launch(const Csr& A, const double* X, int64_t ldx, double* Y, int64_t ldy,
                          int w, double* part, int v, cudaStream_t st) {
  using C = StagedCfg<LPR>;
  constexpr int VL = LPR == 8 ? 8 : LPR == 16 ? 16 : 32;  // spmm_kernel lane-group width
  CUtensorMap xmap;
  if (A.nchunks[v] > 0 && !gather_map(&xmap, X, A.cols, w, ldx, 2 * LPR)) return false;
  // medium rows longer than a chunk + long-row segments: warp / CTA path
  spmm_dispatch<VL, 2>(A, X, ldx, Y, ldy, w, part, st, A.med_gt[v], 0, false);
  if (A.nchunks[v] > 0) {
    static bool attr = false;
    if (!attr) {
      TSVD_CUDA(cudaFuncSetAttribute(spmm_staged_kernel<LPR>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::bytes));
      attr = true;
    }
    const unsigned grid = (unsigned)std::min<int64_t>(A.nchunks[v], 148);
    spmm_staged_kernel<LPR><<<grid, C::NTHR, C::bytes, st>>>(xmap, A.colidx, A.vals, A.perm, A.bins,
                                                         A.bin_chunk0[v], A.nbins_v[v],
                                                         A.nchunks[v], Y, ldy, w);
    TSVD_CHECK_LAUNCH();
  }
  if (A.nsplit > 0) {
    const int64_t thr = A.nsplit * kPartW;
    launch_pdl(spmm_fixup_kernel, (unsigned)((thr + 255) / 256), 256, 0, st, A.split_row, A.split_first, A.split_count, part, Y, ldy, w, A.nsplit);
    TSVD_CHECK_LAUNCH();
  }
  return true;
}

void launch_spmm(const Csr& A, const double* X, int64_t ldx, double* Y, int64_t ldy, int w,
                 double* part, cudaStream_t st) {
  const bool v2 = (w % 2 == 0) && (ldx % 2 == 0) && (ldy % 2 == 0) &&
                  ((uintptr_t)X % 16 == 0) && ((uintptr_t)Y % 16 == 0);
  if (v2 && g_spmm_staged && A.bins && w > 4) {
    if (w <= 16 ? staged_launch<8>(A, X, ldx, Y, ldy, w, part, 0, st)
                : w <= 32 ? staged_launch<16>(A, X, ldx, Y, ldy, w, part, 1, st)
                          : staged_launch<32>(A, X, ldx, Y, ldy, w, part, 2, st))
      return;
  }
  if (v2) {
    if (w <= 2)
      spmm_dispatch<1, 2>(A, X, ldx, Y, ldy, w, part, st);
    else if (w <= 4)
      spmm_dispatch<2, 2>(A, X, ldx, Y, ldy, w, part, st);
    else if (w <= 8)
      spmm_dispatch<4, 2>(A, X, ldx, Y, ldy, w, part, st);
    else if (w <= 16)
      spmm_dispatch<8, 2>(A, X, ldx, Y, ldy, w, part, st);
    else if (w <= 32)
      spmm_dispatch<16, 2>(A, X, ldx, Y, ldy, w, part, st);
    else  // 32 < w <= 64 (wide RandSVD blocks): a whole warp per short row
      spmm_dispatch<32, 2>(A, X, ldx, Y, ldy, w, part, st);
  } else {
    if (w > 32) throw Error{TSVD_EINVAL, "launch_spmm: w > 32 needs 16-byte aligned operands"};
    if (w <= 4)
      spmm_dispatch<4, 1>(A, X, ldx, Y, ldy, w, part, st);
    else if (w <= 8)
      spmm_dispatch<8, 1>(A, X, ldx, Y, ldy, w, part, st);
    else if (w <= 16)
      spmm_dispatch<16, 1>(A, X, ldx, Y, ldy, w, part, st);
    else
      spmm_dispatch<32, 1>(A, X, ldx, Y, ldy, w, part, st);
  }
}

void launch_spmm_wide(const Csr& A, const double* X, int64_t ldx, double* Y, int64_t ldy,
                      int w, double* part, cudaStream_t st) {
  // 64-column launches when the double2 path applies (A is read once per 64
  // columns of X instead of once per 32), else 32
  const bool v2 = (ldx % 2 == 0) && (ldy % 2 == 0) && ((uintptr_t)X % 16 == 0) &&
                  ((uintptr_t)Y % 16 == 0);
  const int cw = v2 ? 64 : 32;
  for (int c0 = 0; c0 < w; c0 += cw) {
    const int wc = w - c0 < cw ? w - c0 : cw;
    launch_spmm(A, X + c0, ldx, Y + c0, ldy, wc, part, st);
  }
}

// ------------------------------------------------------- plan / transpose --
// Copies the nonzeros of the rows in permuted order: position p of the new
// layout holds row perm[p] (one warp per row, lane-strided).
constexpr int64_t kPermWarpMax = 4096;  // > kMedRow: only long rows exceed it
__global__ void csr_permute_kernel(const int64_t* __restrict__ old_rp,
                                   const int32_t* __restrict__ old_ci,
                                   const double* __restrict__ old_va,
                                   const int32_t* __restrict__ perm,
                                   const int64_t* __restrict__ new_rp, int64_t rows,
                                   int32_t* __restrict__ new_ci, double* __restrict__ new_va,
                                   int64_t* __restrict__ long_rows, int* __restrict__ nlong) {
  const int lane = threadIdx.x & 31;
  for (int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; p < rows;
       p += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t ob = old_rp[perm[p]], nb = new_rp[p], len = new_rp[p + 1] - nb;
    if (len > kPermWarpMax) {  // listed for csr_permute_long_kernel
      if (lane == 0) long_rows[atomicAdd(nlong, 1)] = p;
      continue;
    }
    for (int64_t k = lane; k < len; k += 32) {
      new_ci[nb + k] = old_ci[ob + k];
      new_va[nb + k] = old_va[ob + k];
    }
  }
}

// the rows with more than kPermWarpMax nonzeros (listed by
// csr_permute_kernel, in any order -- each is a plain copy): every row's
// nonzeros spread over the whole grid instead of one warp (C2's
// 140 000-nonzero row took 0.75 ms per CSR)
__global__ void csr_permute_long_kernel(const int64_t* __restrict__ old_rp,
                                        const int32_t* __restrict__ old_ci,
                                        const double* __restrict__ old_va,
                                        const int32_t* __restrict__ perm,
                                        const int64_t* __restrict__ new_rp,
                                        const int64_t* __restrict__ long_rows,
                                        const int* __restrict__ nlong,
                                        int32_t* __restrict__ new_ci,
                                        double* __restrict__ new_va) {
  const int n = *nlong;
  for (int i = 0; i < n; ++i) {
    const int64_t p = long_rows[i];
    const int64_t nb = new_rp[p], len = new_rp[p + 1] - nb;
    const int64_t ob = old_rp[perm[p]];
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < len;
         k += (int64_t)gridDim.x * blockDim.x) {
      new_ci[nb + k] = old_ci[ob + k];
      new_va[nb + k] = old_va[ob + k];
    }
  }
}

// moves the nonzeros of A into the permuted row order (new_rp, A.perm)
static void csr_permute(const Csr& A, const int64_t* new_rp, int32_t* nci, double* nva,
                        cudaStream_t st) {
  int* nlong;
  int64_t* lrows;
  dmalloc_t(&nlong, 1, st);
  dmalloc_t(&lrows, A.nnz / kPermWarpMax + 2, st);
  TSVD_CUDA(cudaMemsetAsync(nlong, 0, sizeof(int), st));
  // one warp per row, up to 64 CTAs per SM in flight (latency-bound)
  const unsigned pg = (unsigned)std::min<int64_t>((A.rows + 7) / 8, 148 * 64);
  csr_permute_kernel<<<pg, 256, 0, st>>>(A.rowptr, A.colidx, A.vals, A.perm, new_rp, A.rows, nci,
                                         nva, lrows, nlong);
  TSVD_CHECK_LAUNCH();
  csr_permute_long_kernel<<<148 * 2, 256, 0, st>>>(A.rowptr, A.colidx, A.vals, A.perm, new_rp,
                                                   lrows, nlong, nci, nva);
  TSVD_CHECK_LAUNCH();
  dfree(lrows, st);
  dfree(nlong, st);
}

// Row-sorted layout + load-balancing plan (called once per CSR, after the
// transposition).  Rows are permuted to [short rows by decreasing length |
// medium rows by decreasing length | long rows] (stable), the nonzeros are
// moved to that order (A.rowptr becomes the permuted row pointer, A.perm the
// output row of each position), and long rows are cut into segments.  A warp
// of short rows then reads adjacent rows' nonzeros (one chain fewer than an
// order[] -> rowptr[row] indirection) and writes Y[perm[p]].
// ---------------------------------------------------- device-side plan ---
// The same plan as csr_build_plan, built on the device so handle creation
// does not walk the row pointer on the host (create time of C2: two host
// plans were ~30 ms of ~60 ms).  Rows get a sort key encoding their class
// and length -- short (<= kLongRow): kLongRow - len; medium: kLongRow + 1 +
// kMedRow - len; long: one key above -- and a stable radix sort of (key, row)
// yields exactly the host order (short / medium by decreasing length, ties
// and long rows in row order).  Only the long rows' positions come back to
// the host to cut them into segments.
constexpr uint32_t kKeyLong = kLongRow + 1 + kMedRow + 1;

__global__ void plan_keys_kernel(const int64_t* __restrict__ rowptr, int64_t rows,
                                 uint32_t* __restrict__ key, int32_t* __restrict__ idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t len = rowptr[i + 1] - rowptr[i];
    key[i] = len <= kLongRow ? (uint32_t)(kLongRow - len)
                             : len <= kMedRow ? (uint32_t)(kLongRow + 1 + kMedRow - len) : kKeyLong;
    idx[i] = (int32_t)i;
  }
}

__global__ void plan_lens_kernel(const int64_t* __restrict__ rowptr,
                                 const int32_t* __restrict__ perm, int64_t rows,
                                 int64_t* __restrict__ lens) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q <= rows;
       q += (int64_t)gridDim.x * blockDim.x)
    lens[q] = q < rows ? rowptr[perm[q] + 1] - rowptr[perm[q]] : 0;
}

// counts[0] = #keys <= kLongRow (short), counts[1] = #keys < kKeyLong, on sorted keys
__global__ void plan_counts_kernel(const uint32_t* __restrict__ key, int64_t rows,
                                   int64_t* __restrict__ counts) {
  const uint32_t bound = threadIdx.x == 0 ? (uint32_t)kLongRow + 1 : kKeyLong;
  if (threadIdx.x > 1) return;
  int64_t lo = 0, hi = rows;  // first position with key >= bound
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (key[mid] < bound) lo = mid + 1; else hi = mid;
  }
  counts[threadIdx.x] = lo;
}

static bool csr_build_plan_device(Csr& A, cudaStream_t st) {
  const int64_t rows = A.rows;
  if (rows <= 0 || rows >= (int64_t)INT32_MAX) return false;
  const unsigned grid = (unsigned)std::min<int64_t>((rows + 255) / 256, 148 * 16);
  uint32_t *k_in, *k_out;
  int32_t *i_in, *perm;
  int64_t *lens, *new_rp, *counts;
  dmalloc_t(&k_in, rows, st);
  dmalloc_t(&k_out, rows, st);
  dmalloc_t(&i_in, rows, st);
  dmalloc_t(&perm, rows + 4, st);  // + padding: bulk copies read whole 16-byte pieces
  TSVD_CUDA(cudaMemsetAsync(perm + rows, 0, 4 * sizeof(int32_t), st));
  dmalloc_t(&lens, rows + 1, st);
  dmalloc_t(&new_rp, rows + 1, st);
  dmalloc_t(&counts, 2, st);
  plan_keys_kernel<<<grid, 256, 0, st>>>(A.rowptr, rows, k_in, i_in);
  TSVD_CHECK_LAUNCH();
  int end_bit = 1;
  while ((1u << end_bit) <= kKeyLong) ++end_bit;
  size_t sort_b = 0, scan_b = 0;
  TSVD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_b, k_in, k_out, i_in, perm, (int)rows,
                                            0, end_bit, st));
  TSVD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_b, lens, new_rp, (int)(rows + 1), st));
  void* tmp = dmalloc(std::max(sort_b, scan_b), st);
  TSVD_CUDA(cub::DeviceRadixSort::SortPairs(tmp, sort_b, k_in, k_out, i_in, perm, (int)rows, 0,
                                            end_bit, st));
  plan_lens_kernel<<<grid, 256, 0, st>>>(A.rowptr, perm, rows, lens);
  plan_counts_kernel<<<1, 32, 0, st>>>(k_out, rows, counts);
  TSVD_CHECK_LAUNCH();
  TSVD_CUDA(cub::DeviceScan::ExclusiveSum(tmp, scan_b, lens, new_rp, (int)(rows + 1), st));
  int64_t hc[2] = {0, 0};
  TSVD_CUDA(cudaMemcpyAsync(hc, counts, sizeof(hc), cudaMemcpyDeviceToHost, st));
  TSVD_CUDA(cudaStreamSynchronize(st));
  const int64_t nshort = hc[0], nmed = hc[1] - hc[0], q0 = hc[1], nlong = rows - q0;
  // long rows: their rows and new row-pointer range back to the host
  std::vector<int32_t> lrow(nlong);
  std::vector<int64_t> lrp(nlong + 1);
  if (nlong > 0) {
    TSVD_CUDA(cudaMemcpyAsync(lrow.data(), perm + q0, nlong * sizeof(int32_t),
                              cudaMemcpyDeviceToHost, st));
    TSVD_CUDA(cudaMemcpyAsync(lrp.data(), new_rp + q0, (nlong + 1) * sizeof(int64_t),
                              cudaMemcpyDeviceToHost, st));
    TSVD_CUDA(cudaStreamSynchronize(st));
  }
  std::vector<int64_t> srow, sbeg, send, sprow;
  std::vector<int32_t> sslot, spfirst, spcnt;
  int32_t slots = 0;
  for (int64_t j = 0; j < nlong; ++j) {
    const int64_t i = lrow[j], b = lrp[j], len = lrp[j + 1] - lrp[j];
    const int64_t nseg = (len + kSeg - 1) / kSeg;
    if (nseg > 1) {
      sprow.push_back(i);
      spfirst.push_back(slots);
      spcnt.push_back((int32_t)nseg);
    }
    for (int64_t sg = 0; sg < nseg; ++sg) {
      srow.push_back(i);
      sbeg.push_back(b + sg * kSeg);
      send.push_back(std::min(b + len, b + (sg + 1) * kSeg));
      sslot.push_back(nseg > 1 ? slots++ : -1);
    }
  }
  A.nseg = (int64_t)srow.size();
  A.nsplit = (int64_t)sprow.size();
  A.nslots = slots;
  A.nshort = nshort;
  A.nmed = nmed;
  auto up64 = [&](std::vector<int64_t>& v, int64_t** d) {
    if (v.empty()) return;
    dmalloc_t(d, v.size(), st);
    TSVD_CUDA(cudaMemcpyAsync(*d, v.data(), v.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  };
  auto up32 = [&](std::vector<int32_t>& v, int32_t** d) {
    if (v.empty()) return;
    dmalloc_t(d, v.size(), st);
    TSVD_CUDA(cudaMemcpyAsync(*d, v.data(), v.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  };
  up64(srow, &A.seg_row);
  up64(sbeg, &A.seg_beg);
  up64(send, &A.seg_end);
  up32(sslot, &A.seg_slot);
  up64(sprow, &A.split_row);
  up32(spfirst, &A.split_first);
  up32(spcnt, &A.split_count);
  A.perm = perm;
  if (A.nnz > 0) {
    int32_t* nci;
    double* nva;
    dmalloc_t(&nci, A.nnz + 4, st);
    dmalloc_t(&nva, A.nnz + 2, st);
    csr_permute(A, new_rp, nci, nva, st);
    dfree(A.colidx, st);
    dfree(A.vals, st);
    A.colidx = nci;
    A.vals = nva;
  }
  dfree(A.rowptr, st);
  A.rowptr = new_rp;
  TSVD_CUDA(cudaStreamSynchronize(st));
  for (void* q : {(void*)k_in, (void*)k_out, (void*)i_in, (void*)lens, (void*)counts, tmp})
    dfree(q, st);
  return true;
}

void csr_plan(Csr& A, cudaStream_t st) {
  // the staged SpMM (TSVD_SPMM_STAGED=1) also needs the length bins: host plan
  if (!g_spmm_staged && csr_build_plan_device(A, st)) return;
  std::vector<int64_t> hrp(A.rows + 1);
  TSVD_CUDA(cudaMemcpy(hrp.data(), A.rowptr, (A.rows + 1) * sizeof(int64_t),
                       cudaMemcpyDeviceToHost));
  csr_build_plan(A, hrp.data(), st);
}

void csr_build_plan(Csr& A, const int64_t* hrp, cudaStream_t st) {
  auto len_of = [&](int64_t i) { return hrp[i + 1] - hrp[i]; };
  // short rows, counting-sorted by decreasing length (stable in the row index)
  std::vector<int64_t> cnt(kLongRow + 2, 0);
  for (int64_t i = 0; i < A.rows; ++i)
    if (len_of(i) <= kLongRow) ++cnt[kLongRow - len_of(i) + 1];
  for (int k = 1; k <= kLongRow + 1; ++k) cnt[k] += cnt[k - 1];
  const int64_t nshort = cnt[kLongRow + 1];
  std::vector<int32_t> perm(A.rows);
  for (int64_t i = 0; i < A.rows; ++i)
    if (len_of(i) <= kLongRow) perm[cnt[kLongRow - len_of(i)]++] = (int32_t)i;
  // medium rows by decreasing length, then long rows in row order
  std::vector<std::pair<int64_t, int32_t>> med;
  for (int64_t i = 0; i < A.rows; ++i)
    if (len_of(i) > kLongRow && len_of(i) <= kMedRow) med.push_back({-len_of(i), (int32_t)i});
  std::stable_sort(med.begin(), med.end(),
                   [](const auto& a, const auto& b) { return a.first < b.first; });
  int64_t p = nshort;
  for (auto& e : med) perm[p++] = e.second;
  const int64_t nmed = (int64_t)med.size();
  for (int64_t i = 0; i < A.rows; ++i)
    if (len_of(i) > kMedRow) perm[p++] = (int32_t)i;
  std::vector<int64_t> nrp(A.rows + 1);
  nrp[0] = 0;
  for (int64_t q = 0; q < A.rows; ++q) nrp[q + 1] = nrp[q] + len_of(perm[q]);
  // long rows: segments of <= kSeg nonzeros in the new layout
  std::vector<int64_t> srow, sbeg, send, sprow;
  std::vector<int32_t> sslot, spfirst, spcnt;
  int32_t slots = 0;
  for (int64_t q = nshort + nmed; q < A.rows; ++q) {
    const int64_t i = perm[q], len = len_of(i);
    const int64_t nseg = (len + kSeg - 1) / kSeg;
    if (nseg > 1) {
      sprow.push_back(i);
      spfirst.push_back(slots);
      spcnt.push_back((int32_t)nseg);
    }
    for (int64_t s = 0; s < nseg; ++s) {
      srow.push_back(i);
      sbeg.push_back(nrp[q] + s * kSeg);
      send.push_back(std::min(nrp[q + 1], nrp[q] + (s + 1) * kSeg));
      sslot.push_back(nseg > 1 ? slots++ : -1);
    }
  }
  A.nseg = (int64_t)srow.size();
  A.nsplit = (int64_t)sprow.size();
  A.nslots = slots;
  A.nshort = nshort;
  A.nmed = nmed;
  auto up64 = [&](std::vector<int64_t>& v, int64_t** d) {
    if (v.empty()) return;
    dmalloc_t(d, v.size(), st);
    TSVD_CUDA(cudaMemcpyAsync(*d, v.data(), v.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  };
  auto up32 = [&](std::vector<int32_t>& v, int32_t** d) {
    if (v.empty()) return;
    dmalloc_t(d, v.size(), st);
    TSVD_CUDA(cudaMemcpyAsync(*d, v.data(), v.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  };
  up64(srow, &A.seg_row);
  up64(sbeg, &A.seg_beg);
  up64(send, &A.seg_end);
  up32(sslot, &A.seg_slot);
  up64(sprow, &A.split_row);
  up32(spfirst, &A.split_first);
  up32(spcnt, &A.split_count);
  // staged SpMM bins: runs of equal length among the rows <= kMedRow (the
  // sorted sections make every length one contiguous run of positions)
  {
    std::vector<std::array<int64_t, 4>> bins;  // L, count, pos0, nz0
    for (int64_t q = 0; q < nshort + nmed;) {
      const int64_t L = len_of(perm[q]);
      int64_t e = q + 1;
      while (e < nshort + nmed && len_of(perm[e]) == L) ++e;
      bins.push_back({L, e - q, q, nrp[q]});
      q = e;
    }
    std::stable_sort(bins.begin(), bins.end(),
                     [](const auto& a, const auto& b) { return a[0] < b[0]; });
    A.nbins = (int)bins.size();
    std::vector<int64_t> flat;
    for (auto& b : bins) flat.insert(flat.end(), b.begin(), b.end());
    if (!flat.empty()) up64(flat, &A.bins);
    const int nzc[3] = {256, 128, 64};
    for (int v = 0; v < 3; ++v) {
      std::vector<int64_t> c0(1, 0);
      int nb = 0;
      for (auto& b : bins) {
        if (b[0] > nzc[v]) break;
        const int64_t R = b[0] ? std::max<int64_t>(1, nzc[v] / b[0]) : nzc[v];
        c0.push_back(c0.back() + (b[1] + R - 1) / R);
        ++nb;
      }
      A.nbins_v[v] = nb;
      A.nchunks[v] = c0.back();
      int64_t gt = 0;
      for (int64_t q = nshort; q < nshort + nmed; ++q)
        if (len_of(perm[q]) > nzc[v]) ++gt;
      A.med_gt[v] = gt;
      up64(c0, &A.bin_chunk0[v]);
    }
  }
  perm.resize(A.rows + 4, 0);  // bulk copies read whole 16-byte pieces
  up32(perm, &A.perm);
  // move the nonzeros into the permuted layout
  int64_t* new_rp = nullptr;
  up64(nrp, &new_rp);
  if (A.rows > 0 && A.nnz > 0) {
    int32_t* nci;
    double* nva;
    dmalloc_t(&nci, A.nnz + 4, st);  // +padding: bulk copies read whole 16-byte pieces
    dmalloc_t(&nva, A.nnz + 2, st);
    csr_permute(A, new_rp, nci, nva, st);
    dfree(A.colidx, st);
    dfree(A.vals, st);
    A.colidx = nci;
    A.vals = nva;
  }
  dfree(A.rowptr, st);
  A.rowptr = new_rp ? new_rp : A.rowptr;
  TSVD_CUDA(cudaStreamSynchronize(st));
}

__global__ void rebase_rowptr_kernel(const int64_t* __restrict__ src, int64_t n,
                                     int64_t* __restrict__ dst) {
  const int64_t base = src[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i] - base;
}

// Rows [r0, r1) of a canonical (not yet planned) CSR as a CSR of their own,
// with its own load-balancing plan (the row-range pieces of CSR(A_g^T) the
// pipelined reduce-scatter multiplies one n-shard at a time).
void csr_slice_rows(const Csr& A, int64_t r0, int64_t r1, Csr& P, cudaStream_t st) {
  P = Csr{};
  P.rows = r1 - r0;
  P.cols = A.cols;
  int64_t b[2] = {0, 0};
  TSVD_CUDA(cudaMemcpyAsync(&b[0], A.rowptr + r0, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  TSVD_CUDA(cudaMemcpyAsync(&b[1], A.rowptr + r1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  TSVD_CUDA(cudaStreamSynchronize(st));
  P.nnz = b[1] - b[0];
  dmalloc_t(&P.rowptr, P.rows + 1, st);
  dmalloc_t(&P.colidx, std::max<int64_t>(1, P.nnz), st);
  dmalloc_t(&P.vals, std::max<int64_t>(1, P.nnz), st);
  rebase_rowptr_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((P.rows + 256) / 256, 148 * 8)),
                         256, 0, st>>>(A.rowptr + r0, P.rows, P.rowptr);
  TSVD_CHECK_LAUNCH();
  if (P.nnz > 0) {
    TSVD_CUDA(cudaMemcpyAsync(P.colidx, A.colidx + b[0], P.nnz * sizeof(int32_t),
                              cudaMemcpyDeviceToDevice, st));
    TSVD_CUDA(cudaMemcpyAsync(P.vals, A.vals + b[0], P.nnz * sizeof(double),
                              cudaMemcpyDeviceToDevice, st));
  }
  csr_plan(P, st);
}

void csr_free(Csr& A, cudaStream_t st) {
  dfree(A.rowptr, st);
  dfree(A.colidx, st);
  dfree(A.vals, st);
  dfree(A.seg_row, st);
  dfree(A.seg_beg, st);
  dfree(A.seg_end, st);
  dfree(A.seg_slot, st);
  dfree(A.split_row, st);
  dfree(A.split_first, st);
  dfree(A.split_count, st);
  dfree(A.perm, st);
  dfree(A.bins, st);
  for (auto& p : A.bin_chunk0) dfree(p, st);
  A = Csr{};
}

__global__ void row_of_nz_kernel(const int64_t* __restrict__ rowptr, int64_t rows, int64_t nnz,
                                 int32_t* __restrict__ row_of) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = rows;  // largest i with rowptr[i] <= k
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (rowptr[mid] <= k) lo = mid; else hi = mid;
    }
    row_of[k] = (int32_t)lo;
  }
}

__global__ void iota_kernel(int32_t* p, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    p[k] = (int32_t)k;
}

__global__ void gather_t_kernel(const int32_t* __restrict__ perm,
                                const int32_t* __restrict__ row_of,
                                const double* __restrict__ vals, int32_t* __restrict__ tcol,
                                double* __restrict__ tval, int64_t nnz) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = perm[k];
    tcol[k] = row_of[p];
    tval[k] = vals[p];
  }
}

__global__ void t_rowptr_kernel(const int32_t* __restrict__ sorted_cols, int64_t nnz,
                                int64_t ncols, int64_t* __restrict__ trowptr) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= ncols;
       j += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nnz;  // first k with sorted_cols[k] >= j
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (sorted_cols[mid] < j) lo = mid + 1; else hi = mid;
    }
    trowptr[j] = lo;
  }
}

void csr_transpose(const Csr& A, Csr& T, cudaStream_t st) {
  T.rows = A.cols;
  T.cols = A.rows;
  T.nnz = A.nnz;
  if (A.nnz >= (int64_t)INT32_MAX) throw Error{TSVD_EINVAL, "nnz >= 2^31 per shard"};
  const int nnz = (int)A.nnz;
  dmalloc_t(&T.rowptr, T.rows + 1, st);
  dmalloc_t(&T.colidx, std::max<int64_t>(1, T.nnz), st);
  dmalloc_t(&T.vals, std::max<int64_t>(1, T.nnz), st);
  if (nnz == 0) {
    TSVD_CUDA(cudaMemsetAsync(T.rowptr, 0, (T.rows + 1) * sizeof(int64_t), st));
    TSVD_CUDA(cudaStreamSynchronize(st));
    return;
  }
  int32_t *row_of, *perm_in, *perm_out, *keys_out;
  dmalloc_t(&row_of, nnz, st);
  dmalloc_t(&perm_in, nnz, st);
  dmalloc_t(&perm_out, nnz, st);
  dmalloc_t(&keys_out, nnz, st);
  const unsigned grid = 148 * 8;
  row_of_nz_kernel<<<grid, 256, 0, st>>>(A.rowptr, A.rows, A.nnz, row_of);
  iota_kernel<<<grid, 256, 0, st>>>(perm_in, A.nnz);
  TSVD_CHECK_LAUNCH();
  int end_bit = 1;
  while (end_bit < 31 && (int64_t(1) << end_bit) < A.cols) ++end_bit;
  size_t tmp_bytes = 0;
  TSVD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, A.colidx, keys_out, perm_in,
                                            perm_out, nnz, 0, end_bit, st));
  void* tmp;
  tmp = dmalloc(tmp_bytes, st);
  TSVD_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, A.colidx, keys_out, perm_in,
                                            perm_out, nnz, 0, end_bit, st));
  gather_t_kernel<<<grid, 256, 0, st>>>(perm_out, row_of, A.vals, T.colidx, T.vals, A.nnz);
  t_rowptr_kernel<<<grid, 256, 0, st>>>(keys_out, A.nnz, T.rows, T.rowptr);
  TSVD_CHECK_LAUNCH();
  TSVD_CUDA(cudaStreamSynchronize(st));
  dfree(tmp, st);
  dfree(row_of, st);
  dfree(perm_in, st);
  dfree(perm_out, st);
  dfree(keys_out, st);
}

// Canonical-CSR check (include/tsvd.h) in two element-parallel passes, so a
// 140 000-nonzero row is not walked by one warp (that took 2.2 ms of C2's
// handle creation): (1) one thread per row checks the row pointer (bounds,
// monotone) and marks the first position of every nonempty row in a bitmap;
// (2) one thread per nonzero checks its column is in range and, unless it
// starts a row, larger than its predecessor's.  If (1) flags the row
// pointer, (2)'s row starts are meaningless, but the handle is rejected
// anyway.
__global__ void csr_validate_rows_kernel(const int64_t* __restrict__ rowptr, int64_t rows,
                                         int64_t nnz, unsigned* __restrict__ start_bits,
                                         int* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = rowptr[i], e = rowptr[i + 1];
    if (b > e || b < 0 || e > nnz) {
      atomicOr(bad, 1);
      continue;
    }
    if (b < e) atomicOr(start_bits + (b >> 5), 1u << (b & 31));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (rowptr[0] != 0 || rowptr[rows] != nnz) atomicOr(bad, 4);
  }
}

__global__ void csr_validate_cols_kernel(const int32_t* __restrict__ colidx, int64_t cols,
                                         int64_t nnz, const unsigned* __restrict__ start_bits,
                                         int* __restrict__ bad) {
  int flags = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = colidx[k];
    if (c < 0 || c >= cols) flags |= 8;
    else if (k > 0 && !((start_bits[k >> 5] >> (k & 31)) & 1u) && colidx[k - 1] >= c) flags |= 2;
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if (flags && (threadIdx.x & 31) == 0) atomicOr(bad, flags);
}

// ---------------------------------------------------------- canonicalise --
// unsorted column indices and duplicate entries are accepted and
// canonicalised on the device: a stable radix sort by (row, column) keeps the
// input order among duplicates, and each run of equal (row, column) is summed
// sequentially in that order by the thread owning its first entry, so the
// result does not depend on the launch configuration.
__global__ void csr_keys_kernel(const int32_t* __restrict__ row_of,
                                const int32_t* __restrict__ colidx, int64_t cols, int64_t nnz,
                                int64_t* __restrict__ key) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x)
    key[k] = (int64_t)row_of[k] * cols + colidx[k];
}

__global__ void csr_run_heads_kernel(const int64_t* __restrict__ key, int64_t nnz,
                                     int32_t* __restrict__ head) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x)
    head[k] = (k == 0 || key[k] != key[k - 1]) ? 1 : 0;
}

__global__ void csr_sum_runs_kernel(const int64_t* __restrict__ key,
                                    const int32_t* __restrict__ src,
                                    const double* __restrict__ vals,
                                    const int32_t* __restrict__ head,
                                    const int32_t* __restrict__ pos, int64_t cols, int64_t nnz,
                                    int32_t* __restrict__ out_row, int32_t* __restrict__ out_col,
                                    double* __restrict__ out_val) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (!head[k]) continue;
    double v = vals[src[k]];
    for (int64_t j = k + 1; j < nnz && key[j] == key[k]; ++j) v += vals[src[j]];
    const int32_t p = pos[k];
    out_row[p] = (int32_t)(key[k] / cols);
    out_col[p] = (int32_t)(key[k] % cols);
    out_val[p] = v;
  }
}

void csr_canonicalize(Csr& A, cudaStream_t st) {
  if (A.nnz >= (int64_t)INT32_MAX) throw Error{TSVD_EINVAL, "nnz >= 2^31 per shard"};
  const int nnz = (int)A.nnz;
  if (nnz == 0) return;
  const unsigned grid = 148 * 8;
  int32_t *row_of, *idx_in, *idx_out, *head, *pos;
  int64_t *key_in, *key_out;
  dmalloc_t(&row_of, nnz, st);
  dmalloc_t(&idx_in, nnz, st);
  dmalloc_t(&idx_out, nnz, st);
  dmalloc_t(&head, nnz, st);
  dmalloc_t(&pos, nnz, st);
  dmalloc_t(&key_in, nnz, st);
  dmalloc_t(&key_out, nnz, st);
  row_of_nz_kernel<<<grid, 256, 0, st>>>(A.rowptr, A.rows, A.nnz, row_of);
  iota_kernel<<<grid, 256, 0, st>>>(idx_in, A.nnz);
  csr_keys_kernel<<<grid, 256, 0, st>>>(row_of, A.colidx, A.cols, A.nnz, key_in);
  TSVD_CHECK_LAUNCH();
  int end_bit = 1;
  const unsigned long long kmax = (unsigned long long)A.rows * (unsigned long long)A.cols;
  while (end_bit < 63 && (1ULL << end_bit) < kmax) ++end_bit;
  size_t tmp_bytes = 0, scan_bytes = 0;
  TSVD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key_in, key_out, idx_in, idx_out,
                                            nnz, 0, end_bit, st));
  TSVD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, head, pos, nnz, st));
  void* tmp = dmalloc(std::max(tmp_bytes, scan_bytes), st);
  TSVD_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key_in, key_out, idx_in, idx_out, nnz,
                                            0, end_bit, st));
  csr_run_heads_kernel<<<grid, 256, 0, st>>>(key_out, A.nnz, head);
  TSVD_CHECK_LAUNCH();
  TSVD_CUDA(cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, head, pos, nnz, st));
  int last_pos = 0, last_head = 0;
  TSVD_CUDA(cudaMemcpyAsync(&last_pos, pos + nnz - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  TSVD_CUDA(cudaMemcpyAsync(&last_head, head + nnz - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  TSVD_CUDA(cudaStreamSynchronize(st));
  const int64_t nnz2 = (int64_t)last_pos + last_head;
  int32_t *new_row, *new_col;
  double* new_val;
  dmalloc_t(&new_row, nnz2, st);
  dmalloc_t(&new_col, nnz2, st);
  dmalloc_t(&new_val, nnz2, st);
  csr_sum_runs_kernel<<<grid, 256, 0, st>>>(key_out, idx_out, A.vals, head, pos, A.cols, A.nnz,
                                            new_row, new_col, new_val);
  TSVD_CHECK_LAUNCH();
  // row pointer: first position of each row in the sorted, deduplicated rows
  t_rowptr_kernel<<<grid, 256, 0, st>>>(new_row, nnz2, A.rows, A.rowptr);
  TSVD_CHECK_LAUNCH();
  TSVD_CUDA(cudaStreamSynchronize(st));
  for (void* p : {(void*)row_of, (void*)idx_in, (void*)idx_out, (void*)head, (void*)pos,
                  (void*)key_in, (void*)key_out, tmp, (void*)new_row})
    dfree(p, st);
  dfree(A.colidx, st);
  dfree(A.vals, st);
  A.colidx = new_col;
  A.vals = new_val;
  A.nnz = nnz2;
}

int csr_validate_device(const Csr& A, cudaStream_t st) {
  int* d;
  unsigned* bits;
  const int64_t nw = A.nnz / 32 + 1;
  dmalloc_t(&d, 1, st);
  dmalloc_t(&bits, nw, st);
  TSVD_CUDA(cudaMemsetAsync(d, 0, sizeof(int), st));
  TSVD_CUDA(cudaMemsetAsync(bits, 0, sizeof(unsigned) * nw, st));
  const unsigned rg = (unsigned)std::max<int64_t>(1, std::min<int64_t>((A.rows + 255) / 256, 148 * 16));
  csr_validate_rows_kernel<<<rg, 256, 0, st>>>(A.rowptr, A.rows, A.nnz, bits, d);
  TSVD_CHECK_LAUNCH();
  if (A.nnz > 0) {
    const unsigned cg = (unsigned)std::max<int64_t>(1, std::min<int64_t>((A.nnz + 255) / 256, 148 * 16));
    csr_validate_cols_kernel<<<cg, 256, 0, st>>>(A.colidx, A.cols, A.nnz, bits, d);
    TSVD_CHECK_LAUNCH();
  }
  int h = 0;
  TSVD_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, st));
  TSVD_CUDA(cudaStreamSynchronize(st));
  dfree(bits, st);
  dfree(d, st);
  return h;
}

}  // namespace tsvd
