// Tall-skinny FP64 products of the orthogonalisation passes on the FP64
// tensor-core path (DMMA = mma.sync.m8n8k4.f64; sm_100a has no f64 tcgen05
// kind and DMMA's measured peak equals DFMA's, 37 TF/s - it is used for the
// operand reuse, profiles/box_facts_r01.json):
//
//   gemm_tn : C (s x w) = X^T Y                Alg. 5 S1/S6 (H = P^T Q), dense A^T X
//   gemm_nn : Z (q x w) = alpha X H + beta Y T  Alg. 5 S2/S7 (Q -= P H), dense A X,
//             + per-CTA Gram Z^T Z                restart / outputs (Alg. 2 S7-S9),
//                                                 Alg. 4 S1/S4, Alg. 5 S3/S8 (Gram),
//                                                 Alg. 4 S3/S6, Alg. 5 S5/S10 (T = L^{-T})
//
// Both kernels stream the tall operand through shared memory with cp.async
// (LDGSTS) multi-stage pipelines so several tiles are in flight per SM, which
// is what an HBM-bound pass needs.  Split-K partial sums are
// reduced in a fixed order by a separate kernel; no floating-point atomics.
#include <cuda.h>

#include <climits>
#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace tsvd {

// D(8x8) += A(8x4) B(4x8); per lane: a = A[gid][tig], b = B[tig][gid],
// d0,d1 = D[gid][2 tig + {0,1}]  (gid = lane>>2, tig = lane&3)
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// rows [r0, r0+R) x cols [c0, c0+C) of a row-major (ld) matrix with nrows x
// ncols valid entries -> shared tile (row stride SP), zero-filled outside.
template <int R, int C, int SP, int VEC, int NTHR>
__device__ __forceinline__ void load_tile(double* s, const double* g, int64_t ld, int64_t r0,
                                          int64_t nrows, int c0, int ncols, const double* dummy) {
  constexpr int CV = C / VEC, NV = R * CV;
#pragma unroll 4
  for (int v = threadIdx.x; v < NV; v += NTHR) {
    const int r = v / CV, cv = (v % CV) * VEC;
    const int64_t row = r0 + r;
    const int col = c0 + cv;
    int nvalid = 0;
    if (row < nrows && g) nvalid = max(0, min(VEC, ncols - col));
    const double* src = nvalid ? g + row * ld + col : dummy;
    cp_async<VEC>(s + r * SP + cv, src, nvalid);
  }
}


// row-major rows x cols (ld) f64 matrix, box = 16 columns x box_rows, 128B swizzle
static bool make_map(CUtensorMap* m, const double* base, int64_t rows, int64_t cols, int64_t ld,
                     int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ------------------------------------------------------------------ TN ---
// CTA = (s-tile of TN_ST columns of X) x (contiguous range of row chunks).
// Each stage holds TN_RB rows of X's s-tile and of Y; each warp owns 4 rows
// (one DMMA k-step) of a stage and accumulates the full TN_ST x WP tile.
constexpr int TN_ST = 64;
constexpr int TN_RB = 32;
constexpr int TN_S = 4;

template <int WP>
struct TnCfg {
  static constexpr int XP = TN_ST + 4, YP = WP + 4, NT = WP / 8, MT = TN_ST / 8;
  static constexpr size_t stage = (size_t)TN_RB * (XP + YP);
  static constexpr size_t bytes = sizeof(double) * TN_S * stage;
};

struct TnGeom {
  int s_tiles, splits;
};

static TnGeom tn_geom(int64_t q, int s, int w) {
  TnGeom g;
  const int per_sm = (w > 16) ? 1 : 2;  // matches __launch_bounds__ of gemm_tn_kernel
  g.s_tiles = (s + TN_ST - 1) / TN_ST;
  if (g.s_tiles < 1) g.s_tiles = 1;
  const int64_t chunks = (q + TN_RB - 1) / TN_RB;
  // one wave: at most (CTAs per SM x 148) CTAs in total
  int64_t splits = (int64_t)(per_sm * 148) / g.s_tiles;
  const int64_t min_chunks = 8;  // keep the pipeline busy
  if (splits > chunks / min_chunks) splits = chunks / min_chunks;
  if (splits < 1) splits = 1;
  g.splits = (int)splits;
  return g;
}

constexpr int kTnMaxWaveSplit = 8;  // row splits of a many-s-tile product (tn_tma_go)

size_t tn_part_size(int64_t q, int s) {
  const TnGeom g = tn_geom(q, s, 1);  // the most splits any width uses
  return (size_t)(std::max(g.splits, kTnMaxWaveSplit) + 1) * (size_t)std::max(s, 1) * 32;
}

template <int WP, int VEC>
__global__ void __launch_bounds__(256, (WP == 32) ? 1 : 2) gemm_tn_kernel(const double* __restrict__ X, int64_t ldx,
                                                         const double* __restrict__ Y, int64_t ldy,
                                                         int64_t q, int s, int w,
                                                         double* __restrict__ C, int64_t ldc,
                                                         double* __restrict__ part) {
  pdl_enter();
  using CF = TnCfg<WP>;
  constexpr int XP = CF::XP, YP = CF::YP, NT = CF::NT, MT = CF::MT;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int s0 = blockIdx.x * TN_ST;
  const int split = blockIdx.y, nsplit = gridDim.y;
  const int64_t chunks = (q + TN_RB - 1) / TN_RB;
  const int64_t c_beg = chunks * split / nsplit, c_end = chunks * (split + 1) / nsplit;
  const int nsteps = (int)(c_end - c_beg);
  auto Xs = [&](int st) { return sm + (size_t)st * CF::stage; };
  auto Ys = [&](int st) { return sm + (size_t)st * CF::stage + TN_RB * XP; };
  auto issue = [&](int j) {
    if (j < nsteps) {
      const int st = j % TN_S;
      const int64_t r0 = (c_beg + j) * TN_RB;
      load_tile<TN_RB, TN_ST, XP, VEC, 256>(Xs(st), X, ldx, r0, q, s0, s, X);
      load_tile<TN_RB, WP, YP, VEC, 256>(Ys(st), Y, ldy, r0, q, 0, w, X);
    }
    cp_commit();
  };
  double acc[MT][NT][2];
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
#pragma unroll
  for (int j = 0; j < TN_S - 1; ++j) issue(j);
  for (int j = 0; j < nsteps; ++j) {
    issue(j + TN_S - 1);
    cp_wait<TN_S - 1>();
    __syncthreads();
    const double* xs = Xs(j % TN_S);
    const double* ys = Ys(j % TN_S);
    const int kr = warp * 4 + tig;
    double a[MT], b[NT];
#pragma unroll
    for (int mi = 0; mi < MT; ++mi) a[mi] = xs[kr * XP + mi * 8 + gid];
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) b[ni] = ys[kr * YP + ni * 8 + gid];
#pragma unroll
    for (int mi = 0; mi < MT; ++mi)
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    __syncthreads();
  }
  cp_wait<0>();
  __syncthreads();
  // fixed-order cross-warp reduction into Cs (reuses stage 0)
  double* Cs = sm;
  for (int wv = 0; wv < 8; ++wv) {
    if (warp == wv) {
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int i = mi * 8 + gid, j = ni * 8 + 2 * tig + e;
            if (wv == 0)
              Cs[i * WP + j] = acc[mi][ni][e];
            else
              Cs[i * WP + j] += acc[mi][ni][e];
          }
    }
    __syncthreads();
  }
  const int scols = min(TN_ST, s - s0);
  for (int idx = tid; idx < TN_ST * WP; idx += 256) {
    const int i = idx / WP, j = idx % WP;
    if (i < scols && j < w) {
      if (nsplit == 1)
        C[(int64_t)(s0 + i) * ldc + j] = Cs[idx];
      else
        part[((int64_t)split * s + s0 + i) * w + j] = Cs[idx];
    }
  }
}

// TMA variant of gemm_tn for 9 <= w <= 16 (the n- and m-side H = P^T Y
// passes): one producer warp loads 64-row x 16-column 128B-swizzled boxes of
// X (ST/16 of them) and Y into an mbarrier ring; consumer warp k takes rows
// 8k..8k+7 of a stage as two paired DMMA k-steps (lane tig: rows 2 tig + h),
// which makes both the X^T (A) and Y (B) fragment reads conflict-free under
// the swizzle.  ST adapts to s (16..64) so small-s passes do no zero work.
constexpr int TT_RB = 64;

template <int ST, int NYB = 1>  // NYB = 16-column boxes of Y (w <= 16 NYB)
struct TnTmaCfg {
  static constexpr int NB = ST / 16, MT = ST / 8;
  static constexpr int S = NYB == 2 ? (ST >= 32 ? 3 : 4) : (ST >= 48 ? 2 : 4);
  static constexpr size_t box = (size_t)TT_RB * 16 * 8;  // 8 KB
  static constexpr size_t stage = (NB + NYB) * box;
  static constexpr size_t bar_off = S * stage;
  static constexpr size_t bytes = bar_off + 2 * S * 8 + 1024;
  static constexpr unsigned tx = (unsigned)stage;
};

template <int ST, int NYB>
__global__ void __launch_bounds__(288, 2) gemm_tn_tma_kernel(
    const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap ymap,
    int64_t q, int s, int w, double* __restrict__ C, int64_t ldc, double* __restrict__ part) {
  pdl_enter();
  using CF = TnTmaCfg<ST, NYB>;
  constexpr int S = CF::S, MT = CF::MT, NT = 2 * NYB, WP = 16 * NYB;
  static_assert((size_t)ST * WP * 8 <= CF::stage * CF::S, "reduction tile must fit the ring");
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(sm + CF::bar_off);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int s0 = blockIdx.x * ST;
  const int split = blockIdx.y, nsplit = gridDim.y;
  const int64_t chunks = (q + TT_RB - 1) / TT_RB;
  const int64_t c_beg = chunks * split / nsplit, c_end = chunks * (split + 1) / nsplit;
  const int nsteps = (int)(c_end - c_beg);
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {
    if (lane == 0) {
      for (int j = 0; j < nsteps; ++j) {
        const int st = j % S;
        const unsigned u = (unsigned)(j / S);
        if (j >= S) mbar_wait(&empty[st], (u - 1) & 1);
        const int r0 = (int)((c_beg + j) * TT_RB);
        unsigned char* base = sm + (size_t)st * CF::stage;
        mbar_expect_tx(&full[st], CF::tx);
#pragma unroll
        for (int b = 0; b < CF::NB; ++b)
          tma_load_2d(base + b * CF::box, &xmap, s0 + b * 16, r0, &full[st]);
#pragma unroll
        for (int b = 0; b < NYB; ++b)
          tma_load_2d(base + (CF::NB + b) * CF::box, &ymap, b * 16, r0, &full[st]);
      }
    }
    return;
  }
  double acc[MT][NT][2];
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  for (int j = 0; j < nsteps; ++j) {
    const int st = j % S;
    mbar_wait(&full[st], (unsigned)(j / S) & 1);
    const unsigned char* base = sm + (size_t)st * CF::stage;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int kr = warp * 8 + 2 * tig + h, sw = kr & 7;
      double a[MT], b[NT];
#pragma unroll
      for (int mi = 0; mi < MT; ++mi) {
        const double* xb = (const double*)(base + (mi >> 1) * CF::box);
        const int c = (mi & 1) * 8 + gid;
        a[mi] = xb[kr * 16 + (((c >> 1) ^ sw) << 1) + (c & 1)];
      }
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) {
        const double* ys = (const double*)(base + (CF::NB + (ni >> 1)) * CF::box);
        const int c = (ni & 1) * 8 + gid;
        b[ni] = ys[kr * 16 + (((c >> 1) ^ sw) << 1) + (c & 1)];
      }
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  // fixed-order cross-warp reduction into stage memory (idle once every
  // consumer is past its last step; all loads were consumed)
  bar_consumers();
  double* Cs = (double*)sm;
  for (int wv = 0; wv < 8; ++wv) {
    if (warp == wv) {
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int i = mi * 8 + gid, jj = ni * 8 + 2 * tig + e;
            if (wv == 0)
              Cs[i * WP + jj] = acc[mi][ni][e];
            else
              Cs[i * WP + jj] += acc[mi][ni][e];
          }
    }
    bar_consumers();
  }
  const int scols = min(ST, s - s0);
  for (int idx = tid; idx < ST * WP; idx += 256) {
    const int i = idx / WP, jj = idx % WP;
    if (i < scols && jj < w) {
      if (nsplit == 1)
        C[(int64_t)(s0 + i) * ldc + jj] = Cs[idx];
      else
        part[((int64_t)split * s + s0 + i) * w + jj] = Cs[idx];
    }
  }
}

// Fixed-order split-K reduction: lanes own 32 consecutive outputs, warp k of
// the CTA sums partials k, k+8, k+16, ... (two interleaved accumulators), the
// 8 warp sums are added in warp order.  Deterministic for a given nparts.
__global__ void reduce_partials_kernel(const double* __restrict__ part, int nparts,
                                       int64_t count, double* __restrict__ out, int w,
                                       int64_t ldc) {
  pdl_enter();
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t base = (int64_t)blockIdx.x * 32; base < count; base += (int64_t)gridDim.x * 32) {
    const int64_t i = base + lane;
    double a0 = 0.0, a1 = 0.0;
    if (i < count) {
      int p = warp;
      for (; p + 8 < nparts; p += 16) {
        a0 += part[(int64_t)p * count + i];
        a1 += part[(int64_t)(p + 8) * count + i];
      }
      if (p < nparts) a0 += part[(int64_t)p * count + i];
    }
    red[warp][lane] = a0 + a1;
    __syncthreads();
    if (warp == 0 && i < count) {
      double sum = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) sum += red[k][lane];
      if (ldc)
        out[(i / w) * ldc + (i % w)] = sum;
      else
        out[i] = sum;
    }
    __syncthreads();
  }
}

static void reduce_launch(const double* part, int nparts, int64_t count, double* out, int w,
                          int64_t ldc, cudaStream_t st) {
  if (count <= 0) return;
  int64_t blocks = (count + 31) / 32;
  if (blocks > 148 * 8) blocks = 148 * 8;
  launch_pdl(reduce_partials_kernel, (unsigned)blocks, 256, 0, st, part, nparts, count, out, w, ldc);
  TSVD_CHECK_LAUNCH();
}

void reduce_partials(const double* part, int nparts, int64_t count, double* out,
                     cudaStream_t st) {
  reduce_launch(part, nparts, count, out, 1, 0, st);
}

static bool aligned16(const void* p, int64_t ld) {
  return (((uintptr_t)p) & 15) == 0 && (ld % 2) == 0;
}

template <int WP, int VEC>
static void tn_launch(dim3 grid, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                      int64_t q, int s, int w, double* C, int64_t ldc, double* part,
                      cudaStream_t st) {
  static bool attr = false;
  const size_t bytes = TnCfg<WP>::bytes;
  if (!attr) {
    TSVD_CUDA(cudaFuncSetAttribute(gemm_tn_kernel<WP, VEC>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    attr = true;
  }
  launch_pdl(gemm_tn_kernel<WP, VEC>, grid, 256, bytes, st, X, ldx, Y, ldy, q, s, w, C, ldc, part);
  TSVD_CHECK_LAUNCH();
}

bool g_tn_tma = getenv("TSVD_TN_TMA") ? atoi(getenv("TSVD_TN_TMA")) != 0 : true;

template <int ST, int NYB>
static void tn_tma_go(const CUtensorMap& xm, const CUtensorMap& ym, int64_t q, int s, int w,
                      double* C, int64_t ldc, double* part, cudaStream_t st) {
  using CF = TnTmaCfg<ST, NYB>;
  const int s_tiles = (s + ST - 1) / ST;
  const int64_t chunks = (q + TT_RB - 1) / TT_RB;
  int64_t splits = (int64_t)(2 * 148) / s_tiles;
  if (splits > chunks / 4) splits = chunks / 4;
  if (splits < 1) splits = 1;
  if (splits == 1 && s_tiles > 148) {
    // many s-tiles (dense A^T X, s = n): 625 tiles on 296 resident CTAs ran
    // 3 waves, the last 11 % full (0.70 of the DMMA peak at C4); a row split
    // ks makes the last wave nearly full -- the smallest ks reaching 95 %
    // (partials ks s w, within tn_part_size) -- summed by reduce_partials
    constexpr int R = 2 * 148;
    auto eff = [&](int64_t ks) {
      const int64_t u = (int64_t)s_tiles * ks;
      return (double)u / (double)(((u + R - 1) / R) * R);
    };
    for (int64_t ks = 2; ks <= kTnMaxWaveSplit && eff(splits) < 0.95; ++ks) {
      if (chunks / ks < 16) break;
      if (eff(ks) > eff(splits) + 0.02) splits = ks;
    }
  }
  static bool attr = false;
  if (!attr) {
    TSVD_CUDA(cudaFuncSetAttribute(gemm_tn_tma_kernel<ST, NYB>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::bytes));
    attr = true;
  }
  launch_pdl(gemm_tn_tma_kernel<ST, NYB>, dim3(s_tiles, (unsigned)splits), 288, CF::bytes, st, xm, ym, q, s, w, C, ldc, part);
  TSVD_CHECK_LAUNCH();
  if (splits > 1) reduce_launch(part, (int)splits, (int64_t)s * w, C, w, ldc == w ? 0 : ldc, st);
}

static bool tn_tma_launch(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t q,
                          int s, int w, double* C, int64_t ldc, double* part, cudaStream_t st) {
  CUtensorMap xm, ym;
  if (!make_map(&xm, X, q, s, ldx, TT_RB) || !make_map(&ym, Y, q, w, ldy, TT_RB)) return false;
  if (w > 16) {  // 16 < w <= 32: two Y boxes, s-tiles of at most 32 (registers)
    if (s <= 16) tn_tma_go<16, 2>(xm, ym, q, s, w, C, ldc, part, st);
    else tn_tma_go<32, 2>(xm, ym, q, s, w, C, ldc, part, st);
    return true;
  }
  // s-tile width: every s-tile gets the same rows, so a pass takes as long as
  // its widest tile; ST minimises s_tiles x (ST + w) -- each tile streams its
  // ST columns of X and all w of Y -- preferring the wider tile on ties (s =
  // 80: 48 + 32 instead of 64 + 16, which left half the CTAs idle for 60 %
  // of the pass)
  int best = 16;
  int64_t cost = INT64_MAX;
  for (int stv : {64, 48, 32, 16}) {
    const int64_t c = (int64_t)((s + stv - 1) / stv) * (stv + w);
    if (c < cost) cost = c, best = stv;
  }
  if (best == 16) tn_tma_go<16, 1>(xm, ym, q, s, w, C, ldc, part, st);
  else if (best == 32) tn_tma_go<32, 1>(xm, ym, q, s, w, C, ldc, part, st);
  else if (best == 48) tn_tma_go<48, 1>(xm, ym, q, s, w, C, ldc, part, st);
  else tn_tma_go<64, 1>(xm, ym, q, s, w, C, ldc, part, st);
  return true;
}

void gemm_tn(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t q, int s,
             int w, double* C, int64_t ldc, double* part, cudaStream_t st) {
  if (s <= 0 || w <= 0) return;
  if (w > 32) {
    for (int c0 = 0; c0 < w; c0 += 32)
      gemm_tn(X, ldx, Y + c0, ldy, q, s, std::min(32, w - c0), C + c0, ldc, part, st);
    return;
  }
  if (q <= 0) {  // empty reduction
    for (int i = 0; i < s; ++i)
      TSVD_CUDA(cudaMemsetAsync(C + (int64_t)i * ldc, 0, w * sizeof(double), st));
    return;
  }
  const bool v2 = aligned16(X, ldx) && aligned16(Y, ldy);
  if (w > 8 && w <= 32 && v2 && g_tn_tma && q < ((int64_t)1 << 31) &&
      tn_tma_launch(X, ldx, Y, ldy, q, s, w, C, ldc, part, st))
    return;
  const TnGeom g = tn_geom(q, s, w);
  dim3 grid(g.s_tiles, g.splits);
#define TN_CASE(WPV)                                                              \
  if (v2)                                                                         \
    tn_launch<WPV, 2>(grid, X, ldx, Y, ldy, q, s, w, C, ldc, part, st);          \
  else                                                                            \
    tn_launch<WPV, 1>(grid, X, ldx, Y, ldy, q, s, w, C, ldc, part, st);
  if (w <= 8) {
    TN_CASE(8)
  } else if (w <= 16) {
    TN_CASE(16)
  } else {
    TN_CASE(32)
  }
#undef TN_CASE
  if (g.splits > 1) reduce_launch(part, g.splits, (int64_t)s * w, C, w, ldc == w ? 0 : ldc, st);
}

// ------------------------------------------------------------------ NN ---
// Persistent CTAs over row tiles of NN_R rows; the K dimension (s) streams
// in chunks of NN_KC through an S-stage cp.async ring whose steps run across
// tile boundaries.  Each warp owns 16 rows (2 DMMA M-tiles) x WP columns and
// keeps two accumulator sets (even / odd k-steps) so 4*NT independent DMMA
// chains are in flight per warp.  The epilogue of a tile loads its Y rows
// straight into DMMA A-fragments (issued before the tile's last K chunk so
// the latency overlaps), forms beta*Y*T (T = L^{-T} upper triangular: the
// TRSM of Alg. 4/5 as a multiply; identity if T is null) + alpha*acc, stores
// Z through a shared out-tile (coalesced) and accumulates the Gram Z^T Z of
// the tile (DMMA).
constexpr int NN_R = 128;
constexpr int NN_KC = 32;

template <int WP>
struct NnCfg {
  static constexpr int KC = NN_KC;
  static constexpr int S = (WP == 32) ? 3 : 2;
  static constexpr int PER_SM = (WP >= 32) ? 1 : 2;
  static constexpr bool OS_ALIAS = false;  // out tile aliasing the consumed stage: slower
  static constexpr int NACC = (WP == 64) ? 1 : 2;  // even/odd accumulator sets
  static constexpr int XP = KC + 4, HP = WP + 4, OP = WP + 4, NT = WP / 8;
  static constexpr size_t stage = (size_t)NN_R * XP + (size_t)KC * HP;
  static constexpr size_t bytes =
      sizeof(double) * (S * stage + (OS_ALIAS ? 0 : (size_t)NN_R * OP) + (size_t)WP * WP);
  static_assert(!OS_ALIAS || (size_t)NN_R * OP <= (size_t)NN_R * XP, "out tile must fit a stage");
};

static int wp_of(int w) { return w <= 8 ? 8 : (w <= 16 ? 16 : (w <= 32 ? 32 : 64)); }

int nn_ctas(int64_t q, int w) {
  const int wp = wp_of(w);
  int64_t tiles = (q + NN_R - 1) / NN_R;
  const int64_t cap = 148 * (wp >= 32 ? 1 : 2);
  if (tiles > cap) tiles = cap;
  if (tiles < 1) tiles = 1;
  return (int)tiles;
}

template <int WP, int VEC>
__global__ void __launch_bounds__(256, NnCfg<WP>::PER_SM) gemm_nn_kernel(
    const double* __restrict__ X, int64_t ldx, const double* __restrict__ H, int64_t ldh,
    const double* Y, int64_t ldy, const double* __restrict__ T, double* Z, int64_t ldz,
    int64_t q, int s, int w, double alpha, double beta, double* __restrict__ gram) {
  pdl_enter();
  using CF = NnCfg<WP>;
  constexpr int S = CF::S, XP = CF::XP, HP = CF::HP, OP = CF::OP, NT = CF::NT;
  constexpr int NPAIR = NT * NT, PPW = (NPAIR + 7) / 8, KY = WP / 4, NACC = CF::NACC;
  // Gram schedule: with fewer 8x8 output pairs than warps, KSPLIT warps share a
  // pair and each takes a contiguous K (row) range; two accumulators per chain
  constexpr int KSPLIT = (NPAIR >= 8) ? 1 : 8 / NPAIR;
  constexpr int KSTEPS = NN_R / 4 / KSPLIT;
  constexpr bool kEpiY = WP != 64;  // the WP = 64 variant serves beta = 0 products only
  extern __shared__ __align__(16) double sm[];
  double* Os = sm + S * CF::stage;  // (OS_ALIAS: re-pointed at the consumed stage)
  double* Ts = CF::OS_ALIAS ? Os : Os + NN_R * OP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const double* dummy = X ? X : (H ? H : Y);
  for (int i = tid; i < WP * WP; i += 256) {
    const int r = i / WP, c = i % WP;
    Ts[i] = (r < w && c < w) ? (T ? T[r * w + c] : (r == c ? 1.0 : 0.0)) : 0.0;
  }
  const int64_t ntiles = (q + NN_R - 1) / NN_R;
  const int64_t my_tiles =
      (ntiles > (int64_t)blockIdx.x) ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  constexpr int KC = CF::KC;
  const int nk = s > 0 ? (s + KC - 1) / KC : 1;
  const int64_t nsteps = my_tiles * nk;
  auto Xs = [&](int st) { return sm + (size_t)st * CF::stage; };
  auto Hs = [&](int st) { return sm + (size_t)st * CF::stage + NN_R * XP; };
  auto issue = [&](int64_t j) {
    if (j < nsteps && s > 0) {
      const int st = (int)(j % S);
      const int64_t lt = j / nk;
      const int kc = (int)(j % nk);
      const int64_t r0 = (blockIdx.x + lt * gridDim.x) * NN_R;
      load_tile<NN_R, KC, XP, VEC, 256>(Xs(st), X, ldx, r0, q, kc * KC, s, dummy);
      load_tile<KC, WP, HP, VEC, 256>(Hs(st), H, ldh, kc * KC, s, 0, w, dummy);
    }
    cp_commit();
  };
  double g[PPW][2][2];
#pragma unroll
  for (int p = 0; p < PPW; ++p) g[p][0][0] = g[p][0][1] = g[p][1][0] = g[p][1][1] = 0.0;
  double acc[NACC][2][NT][2];
  double ya[kEpiY ? 2 : 1][kEpiY ? KY : 1], yn[kEpiY ? 2 : 1][kEpiY ? KY : 1];
#pragma unroll
  for (int j = 0; j < S - 1; ++j) issue(j);
  for (int64_t j = 0; j < nsteps; ++j) {
    issue(j + S - 1);
    const int st = (int)(j % S);
    const int kc = (int)(j % nk);
    const int64_t lt = j / nk;
    const int64_t r0 = (blockIdx.x + lt * gridDim.x) * NN_R;
    if (kc == 0) {
#pragma unroll
      for (int h = 0; h < NACC; ++h)
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) acc[h][mi][ni][0] = acc[h][mi][ni][1] = 0.0;
    }
    // this tile's Y rows as DMMA A-fragments: loaded before the tile's last K
    // chunk (nk > 1), or one tile ahead into yn when every step is a tile (nk == 1)
    auto load_ya = [&](double (&dst)[kEpiY ? 2 : 1][kEpiY ? KY : 1], int64_t rbase) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const int64_t row = rbase + warp * 16 + mi * 8 + gid;
#pragma unroll
        for (int kk = 0; kk < KY; ++kk) {
          const int col = kk * 4 + tig;
          if constexpr (kEpiY)
            dst[mi][kk] = (beta != 0.0 && Y && row < q && col < w) ? Y[row * ldy + col] : 0.0;
        }
      }
    };
    if (kEpiY && kc == nk - 1) {
      if (nk > 1) {
        load_ya(ya, r0);
      } else {
        if (j == 0) load_ya(ya, r0);
        else {
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int kk = 0; kk < KY; ++kk)
              if constexpr (kEpiY) ya[mi][kk] = yn[mi][kk];
        }
        if (j + 1 < nsteps) load_ya(yn, r0 + (int64_t)gridDim.x * NN_R);
      }
    }
    cp_wait<S - 1>();
    __syncthreads();
    if (s > 0) {
      const double* xs = Xs(st);
      const double* hs = Hs(st);
#pragma unroll
      for (int kk = 0; kk < KC / 4; ++kk) {
        const int h = (NACC == 2) ? (kk & 1) : 0;
        const double a0 = xs[(warp * 16 + gid) * XP + kk * 4 + tig];
        const double a1 = xs[(warp * 16 + 8 + gid) * XP + kk * 4 + tig];
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) {
          const double b = hs[(kk * 4 + tig) * HP + ni * 8 + gid];
          dmma884(acc[h][0][ni][0], acc[h][0][ni][1], a0, b);
          dmma884(acc[h][1][ni][0], acc[h][1][ni][1], a1, b);
        }
      }
    }
    if (kc == nk - 1) {
      // epilogue: Z = alpha*acc + beta*(Y T)
      if constexpr (CF::OS_ALIAS) {
        Os = Xs(st);
        __syncthreads();  // every warp is done reading stage st
      }
      double yt[kEpiY ? 2 : 1][kEpiY ? NT : 1][2];
#pragma unroll
      for (int mi = 0; mi < (kEpiY ? 2 : 1); ++mi)
#pragma unroll
        for (int ni = 0; ni < (kEpiY ? NT : 1); ++ni) yt[mi][ni][0] = yt[mi][ni][1] = 0.0;
      if constexpr (kEpiY) if (beta != 0.0) {
#pragma unroll
        for (int kk = 0; kk < KY; ++kk)
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) {
            const double b = Ts[(kk * 4 + tig) * WP + ni * 8 + gid];
            dmma884(yt[0][ni][0], yt[0][ni][1], ya[0][kk], b);
            dmma884(yt[1][ni][0], yt[1][ni][1], ya[1][kk], b);
          }
      }
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = warp * 16 + mi * 8 + gid, c = ni * 8 + 2 * tig + e;
            double z = alpha * (NACC == 2 ? acc[0][mi][ni][e] + acc[NACC - 1][mi][ni][e]
                                          : acc[0][mi][ni][e]);
            if constexpr (kEpiY) z += beta * yt[mi][ni][e];
            Os[r * OP + c] = (c < w && r0 + r < q) ? z : 0.0;
          }
      __syncthreads();
      if (Z) {
        for (int idx = tid; idx < NN_R * WP; idx += 256) {
          const int r = idx / WP, c = idx % WP;
          const int64_t row = r0 + r;
          if (row < q && c < w) Z[row * ldz + c] = Os[r * OP + c];
        }
      }
      if (gram) {
#pragma unroll
        for (int p = 0; p < PPW; ++p) {
          const int pair = (KSPLIT > 1) ? (warp % NPAIR) : (warp + 8 * p);
          const int k0 = (KSPLIT > 1) ? (warp / NPAIR) * KSTEPS : 0;
          if (pair < NPAIR) {
            const int mi = pair / NT, ni = pair % NT;
#pragma unroll 8
            for (int kk = 0; kk < KSTEPS; ++kk) {
              const int kr = (k0 + kk) * 4 + tig;
              const double a = Os[kr * OP + mi * 8 + gid];  // (Z^T)[i][k]
              const double b = Os[kr * OP + ni * 8 + gid];
              dmma884(g[p][kk & 1][0], g[p][kk & 1][1], a, b);
            }
          }
        }
      }
    }
    __syncthreads();
  }
  cp_wait<0>();
  if (gram) {
    if constexpr (KSPLIT == 1) {
#pragma unroll
      for (int p = 0; p < PPW; ++p) {
        const int pair = warp + 8 * p;
        if (pair < NPAIR) {
          const int mi = pair / NT, ni = pair % NT;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int i = mi * 8 + gid, j = ni * 8 + 2 * tig + e;
            if (i < w && j < w)
              gram[(int64_t)blockIdx.x * w * w + i * w + j] = g[p][0][e] + g[p][1][e];
          }
        }
      }
    } else {
      // the KSPLIT warps of a pair are summed in warp order (stage 0 is idle now)
      double* red = sm;
      __syncthreads();
#pragma unroll
      for (int e = 0; e < 2; ++e) red[warp * 64 + gid * 8 + 2 * tig + e] = g[0][0][e] + g[0][1][e];
      __syncthreads();
      for (int idx = tid; idx < NPAIR * 64; idx += 256) {
        const int pair = idx / 64, ii = (idx % 64) / 8, jj = idx % 8;
        double sum = 0.0;
        for (int k = 0; k < KSPLIT; ++k) sum += red[(k * NPAIR + pair) * 64 + ii * 8 + jj];
        const int mi = pair / NT, ni = pair % NT;
        const int i = mi * 8 + ii, j = ni * 8 + jj;
        if (i < w && j < w) gram[(int64_t)blockIdx.x * w * w + i * w + j] = sum;
      }
    }
  }
}

// s = 0 passes (Gram only, TRSM-as-multiply Y T, scaling): pure streaming.
// Warps are independent (no block barriers): each walks 8-row tiles, loads
// the rows straight into DMMA A-fragments (next tile prefetched), multiplies
// by T held in B-fragment registers, stores Z from the accumulator fragments
// and accumulates the tile's Gram by DMMA through an 8-row warp-private
// shared tile.  Per-CTA Gram partials are summed over warps in warp order.
#ifndef ROWT_PF
#define ROWT_PF 4
#endif
bool g_rowt32 = getenv("TSVD_ROWT32") ? atoi(getenv("TSVD_ROWT32")) != 0 : true;
template <int WP>
__global__ void __launch_bounds__(256) rowT_kernel(const double* Y, int64_t ldy,
                                                   const double* __restrict__ T, double* Z,
                                                   int64_t ldz, int64_t q, int w, double beta,
                                                   double* __restrict__ gram) {
  pdl_enter();
  // Gram: only the NPAIR upper-triangular 8 x 8 tile pairs (mi <= ni) are
  // accumulated (W is symmetric; mirrored when written)
  constexpr int NT = WP / 8, KY = WP / 4, NPAIR = NT * (NT + 1) / 2, ZP = WP + 4;
  constexpr int GCH = NPAIR < 4 ? NPAIR : 4;  // Gram tiles reduced per chunk (static smem)
  __shared__ double zs[8][8 * ZP];
  __shared__ double gred[8][GCH * 64];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  double tb[KY][NT];
#pragma unroll
  for (int kk = 0; kk < KY; ++kk)
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      const int r = kk * 4 + tig, c = ni * 8 + gid;
      tb[kk][ni] = (r < w && c < w) ? (T ? T[r * w + c] : (r == c ? 1.0 : 0.0)) : 0.0;
    }
  double g[NPAIR][2];
#pragma unroll
  for (int p = 0; p < NPAIR; ++p) g[p][0] = g[p][1] = 0.0;
  const int64_t ntiles = (q + 7) / 8;
  const int64_t gw = (int64_t)blockIdx.x * 8 + warp, nw = (int64_t)gridDim.x * 8;
  // PF tiles of Y in flight per warp (register ring)
  constexpr int PF = ROWT_PF;
  double yr[PF][KY];
  auto load = [&](double (&dst)[KY], int64_t t) {
    const int64_t row = t * 8 + gid;
#pragma unroll
    for (int kk = 0; kk < KY; ++kk) {
      const int col = kk * 4 + tig;
      dst[kk] = (t < ntiles && row < q && col < w) ? Y[row * ldy + col] : 0.0;
    }
  };
#pragma unroll
  for (int f = 0; f < PF - 1; ++f) load(yr[f], gw + f * nw);
  double* zw = zs[warp];
  int64_t it = 0;
  for (int64_t t = gw; t < ntiles; t += nw, ++it) {
    double ya[KY];
    // rotate the ring: yr[0] is this tile, yr[PF-1] <- tile t + (PF-1) nw
#pragma unroll
    for (int kk = 0; kk < KY; ++kk) ya[kk] = yr[0][kk];
#pragma unroll
    for (int f = 0; f < PF - 1; ++f)
#pragma unroll
      for (int kk = 0; kk < KY; ++kk) yr[f][kk] = yr[f + 1][kk];
    load(yr[PF - 2], t + (PF - 1) * nw);
    double acc[NT][2];
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) acc[ni][0] = acc[ni][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < KY; ++kk)
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) dmma884(acc[ni][0], acc[ni][1], ya[kk], tb[kk][ni]);
    const int64_t row = t * 8 + gid;
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      const int c = ni * 8 + 2 * tig;
      const double z0 = (row < q && c < w) ? beta * acc[ni][0] : 0.0;
      const double z1 = (row < q && c + 1 < w) ? beta * acc[ni][1] : 0.0;
      if (Z && row < q) {
        if (c + 1 < w && ((ldz | (uintptr_t)Z / 8 | c) & 1) == 0) {
          *reinterpret_cast<double2*>(Z + row * ldz + c) = make_double2(z0, z1);
        } else {
          if (c < w) Z[row * ldz + c] = z0;
          if (c + 1 < w) Z[row * ldz + c + 1] = z1;
        }
      }
      zw[gid * ZP + c] = z0;
      zw[gid * ZP + c + 1] = z1;
    }
    if (gram) {
      __syncwarp();
#pragma unroll
      for (int k2 = 0; k2 < 2; ++k2)
#pragma unroll
        for (int mi = 0, p = 0; mi < NT; ++mi) {
          const double a = zw[(k2 * 4 + tig) * ZP + mi * 8 + gid];
#pragma unroll
          for (int ni = mi; ni < NT; ++ni, ++p) {
            const double b = zw[(k2 * 4 + tig) * ZP + ni * 8 + gid];
            dmma884(g[p][0], g[p][1], a, b);
          }
        }
      __syncwarp();
    }
  }
  (void)it;
  if (gram) {
#pragma unroll
    for (int p0 = 0; p0 < NPAIR; p0 += GCH) {
      if (p0 > 0) __syncthreads();
#pragma unroll
      for (int p = 0; p < GCH; ++p)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (p0 + p < NPAIR) gred[warp][p * 64 + gid * 8 + 2 * tig + e] = g[p0 + p][e];
      __syncthreads();
      for (int idx = tid; idx < GCH * 64; idx += 256) {
        const int p = p0 + idx / 64, ii = (idx % 64) / 8, jj = idx % 8;
        if (p >= NPAIR) break;
        double sum = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) sum += gred[k][idx];
        int mi = 0, base = 0;
        while (p >= base + (NT - mi)) {
          base += NT - mi;
          ++mi;
        }
        const int ni = mi + (p - base);
        const int i = mi * 8 + ii, j = ni * 8 + jj;
        if (i < w && j < w) {
          gram[(int64_t)blockIdx.x * w * w + i * w + j] = sum;
          gram[(int64_t)blockIdx.x * w * w + j * w + i] = sum;
        }
      }
    }
  }
}

// ---------------------------------------------------------- NN (TMA) ---
// The w <= 16 main-pass variant of gemm_nn (the dominant kernel of C2):
// warp-specialised, one producer warp issuing TMA tile loads
// (cp.async.bulk.tensor, 128B-swizzled 16-column boxes, out-of-bounds rows /
// columns zero-filled by the copy engine) into an S-stage mbarrier ring, and
// eight consumer warps doing only LDS + DMMA.  The producer runs ahead across
// tile boundaries, so the X stream continues through the epilogue.  Bank
// conflicts of the swizzled layout are avoided by (i) pairing k-steps: lane
// (gid, tig) takes k = 8*kk2 + 2*tig + h for the two DMMAs h = 0, 1, so its two
// A values are one 16-byte LDS, and (ii) permuting the 8 rows of an M-tile,
// lane gid -> row prow = 4*(gid&1) + gid/2, so every quarter-warp reads 8
// distinct 16-byte chunks; the B (H) reads k = 8*kk2 + 2*tig + h are then
// conflict-free as well.  Output rows follow the same permutation.
constexpr int NT_R = 128;
bool g_nn_tma = getenv("TSVD_NN_TMA") ? atoi(getenv("TSVD_NN_TMA")) != 0 : true;
// w <= 16 with the producer folded into warp 0 (8 warps, 2 CTAs/SM): A/B knob
bool g_nn_fold16 = getenv("TSVD_NN_FOLD16") ? atoi(getenv("TSVD_NN_FOLD16")) != 0 : true;

template <int KC, int S, int NYB = 1>  // NYB = 16-column boxes of H / Y (w <= 16 NYB)
struct NnTmaCfg {
  static constexpr int NB = KC / 16;                       // 16-column boxes per stage
  static constexpr int WP = 16 * NYB;
  static constexpr size_t xbox = (size_t)NT_R * 16 * 8;    // 16 KB
  static constexpr size_t hbox = (size_t)KC * 16 * 8;
  static constexpr size_t stage = NB * xbox + NYB * hbox;  // multiple of 1024
  static constexpr size_t y_off = S * stage;               // Y tile (NYB boxes, own barriers)
  static constexpr int OP = WP + 4, TP = WP + 4;
  static constexpr size_t os_off = y_off + NYB * xbox;
  static constexpr size_t ts_off = os_off + (size_t)NT_R * OP * 8;
  static constexpr size_t bar_off = ts_off + WP * TP * 8;
  static constexpr size_t bytes = bar_off + (2 * S + 2) * 8 + 1024;  // + alignment slack
  static constexpr unsigned tx = (unsigned)stage;
};

template <int KC, int S, int NYB, bool FOLD>
__device__ __forceinline__ void nn_tma_body(
    const CUtensorMap& xmap, const CUtensorMap& hmap, const CUtensorMap& ymap, int use_y,
    const double* __restrict__ T, double* Z, int64_t ldz, int64_t q, int s, int w, double alpha,
    double beta, double* __restrict__ gram, int64_t zsplit) {
  // split-K (gridDim.y > 1, plain products only: no Y / T / Gram): CTA row y
  // takes K chunks [nk_all y / Y, nk_all (y+1) / Y) and writes its partial
  // product to Z + y zsplit; the caller sums the partials in a fixed order.
  using CF = NnTmaCfg<KC, S, NYB>;
  constexpr int WP = CF::WP, NT = 2 * NYB, OP = CF::OP, TP = CF::TP;
  // Gram: each warp accumulates W = Z^T Z over ITS OWN 16 rows of every tile
  // for the NGP upper-triangular 8 x 8 tile pairs (mi <= ni; W is symmetric),
  // so the tile epilogue needs no CTA barrier: Z is stored from the
  // fragments and a warp's out-tile rows are read back only by that warp
  constexpr int NGP = NT * (NT + 1) / 2;
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  const double* Ys = (const double*)(sm + CF::y_off);
  double* Os = (double*)(sm + CF::os_off);
  double* Ts = (double*)(sm + CF::ts_off);
  uint64_t* full = (uint64_t*)(sm + CF::bar_off);
  uint64_t* empty = full + S;
  uint64_t* yfull = empty + S;
  uint64_t* yempty = yfull + 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int prow = ((gid & 1) << 2) | (gid >> 1);
  for (int i = tid; i < WP * WP; i += blockDim.x) {
    const int r = i / WP, c = i % WP;
    Ts[r * TP + c] = (r < w && c < w) ? (T ? T[r * w + c] : (r == c ? 1.0 : 0.0)) : 0.0;
  }
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 8);
    }
    mbar_init(yfull, 1);
    mbar_init(yempty, 8);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t ntiles = (q + NT_R - 1) / NT_R;
  const int64_t my_tiles =
      (ntiles > (int64_t)blockIdx.x) ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int nk_all = (s + KC - 1) / KC;
  const int kb = (int)((int64_t)nk_all * blockIdx.y / gridDim.y);
  const int nk = (int)((int64_t)nk_all * (blockIdx.y + 1) / gridDim.y) - kb;
  const int64_t nsteps = my_tiles * nk;
  Z += (int64_t)blockIdx.y * zsplit;
  // producer: X/H chunks into the ring, the tile's Y rows into Ys.  Its ring
  // slot / phase and (tile, k-chunk) are running counters (no 64-bit
  // divisions by S and by the runtime nk per step).  FOLD = false: a 9th
  // warp; FOLD = true (w = 32): lane 0 of consumer warp 0 issues step
  // j + S - 1 at the top of its step j, so the CTA has 8 warps = 2 per SM
  // sub-partition and a thread may hold up to 255 registers (with 9 warps
  // one sub-partition hosts 3 and the cap is 168).
  int pst = 0, pkc = 0;
  unsigned pu = 0;
  int64_t plt = 0, pj = 0;
  auto produce = [&]() {  // issue step pj (lane 0 of the producing warp)
    if (pj > 0) {
      if (++pst == S) pst = 0, ++pu;
      if (++pkc == nk) pkc = 0, ++plt;
    }
    if (pj >= S) mbar_wait(&empty[pst], (pu - 1) & 1);
    const int r0 = (int)((blockIdx.x + plt * gridDim.x) * NT_R);
    unsigned char* base = sm + (size_t)pst * CF::stage;
    mbar_expect_tx(&full[pst], CF::tx);
#pragma unroll
    for (int b = 0; b < CF::NB; ++b)
      tma_load_2d(base + b * CF::xbox, &xmap, (kb + pkc) * KC + b * 16, r0, &full[pst]);
#pragma unroll
    for (int b = 0; b < NYB; ++b)
      tma_load_2d(base + CF::NB * CF::xbox + b * CF::hbox, &hmap, b * 16, (kb + pkc) * KC,
                  &full[pst]);
    if (!FOLD && use_y && pkc == nk - 1) {  // with the tile's last chunk: never stalls the X ring
      if (plt > 0) mbar_wait(yempty, (unsigned)(plt - 1) & 1);
      mbar_expect_tx(yfull, (unsigned)(NYB * CF::xbox));
#pragma unroll
      for (int b = 0; b < NYB; ++b)
        tma_load_2d(sm + CF::y_off + b * CF::xbox, &ymap, b * 16, r0, yfull);
    }
    ++pj;
  };
  if constexpr (!FOLD) {
    if (warp == 8) {
      if (lane == 0)
        while (pj < nsteps) produce();
      return;
    }
  } else {
    if (warp == 0 && lane == 0)
      while (pj < nsteps && pj < S - 1) produce();
  }
  double gw[NGP][2];
#pragma unroll
  for (int p = 0; p < NGP; ++p) gw[p][0] = gw[p][1] = 0.0;
  const bool zal = Z && ((((uintptr_t)Z) | (uintptr_t)(ldz * 8)) & 15) == 0;
  double* Ow = Os + warp * 16 * OP;  // this warp's rows of the out tile
  double acc[2][2][NT][2];
  int st = 0, kc = 0;
  unsigned u = 0;
  int64_t lt = 0;
  for (int64_t j = 0; j < nsteps; ++j) {
    if constexpr (FOLD) {
      if (warp == 0 && lane == 0 && pj < nsteps) produce();  // step j + S - 1
    }
    if (j > 0) {
      if (++st == S) st = 0, ++u;
      if (++kc == nk) kc = 0, ++lt;
    }
    const int64_t r0 = (blockIdx.x + lt * gridDim.x) * NT_R;
    if constexpr (FOLD) {
      // the tile's Y rows, issued when the tile starts: warp 0 has finished
      // the previous tile's epilogue itself (a wait inside produce() could
      // wait for warp 0's own arrival when a tile has fewer than S chunks)
      if (use_y && kc == 0 && warp == 0 && lane == 0) {
        if (lt > 0) mbar_wait(yempty, (unsigned)(lt - 1) & 1);
        mbar_expect_tx(yfull, (unsigned)(NYB * CF::xbox));
#pragma unroll
        for (int b = 0; b < NYB; ++b)
          tma_load_2d(sm + CF::y_off + b * CF::xbox, &ymap, b * 16, (int)r0, yfull);
      }
    }
    if (kc == 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) acc[h][mi][ni][0] = acc[h][mi][ni][1] = 0.0;
    }
    mbar_wait(&full[st], u & 1);
    {
      const unsigned char* base = sm + (size_t)st * CF::stage;
#pragma unroll
      for (int kk2 = 0; kk2 < KC / 8; ++kk2) {
        const double* xb = (const double*)(base + (kk2 >> 1) * CF::xbox);
        const int chunk = (((kk2 & 1) << 2) | tig) ^ prow;
        const double2 a0 =
            *reinterpret_cast<const double2*>(xb + (warp * 16 + prow) * 16 + chunk * 2);
        const double2 a1 =
            *reinterpret_cast<const double2*>(xb + (warp * 16 + 8 + prow) * 16 + chunk * 2);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int hr = kk2 * 8 + 2 * tig + h;
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) {
            const double* hs = (const double*)(base + CF::NB * CF::xbox + (ni >> 1) * CF::hbox);
            const int c = (ni & 1) * 8 + gid;
            const double b = hs[hr * 16 + (((c >> 1) ^ (hr & 7)) << 1) + (c & 1)];
            dmma884(acc[h][0][ni][0], acc[h][0][ni][1], h ? a0.y : a0.x, b);
            dmma884(acc[h][1][ni][0], acc[h][1][ni][1], h ? a1.y : a1.x, b);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (kc == nk - 1) {
      // epilogue: Z = alpha acc + beta (Y T); Y rows from the TMA-loaded tile
      // as paired-k A-fragments (same swizzle / row permutation as X)
      double yt[2][NT][2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) yt[mi][ni][0] = yt[mi][ni][1] = 0.0;
      if (use_y && !T) {
        // no T (Alg. 5 S2 / S7: Y - P H): the Y values in accumulator layout,
        // straight from the swizzled tile (row r = warp*16 + mi*8 + prow,
        // columns ni*8 + 2 tig + {0,1} = one 16-byte chunk) -- no identity DMMAs
        mbar_wait(yfull, (unsigned)lt & 1);
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) {
            const double2 yv = *reinterpret_cast<const double2*>(
                Ys + (ni >> 1) * (CF::xbox / 8) + (warp * 16 + mi * 8 + prow) * 16 +
                ((((ni & 1) << 2) | tig) ^ prow) * 2);
            yt[mi][ni][0] = yv.x;
            yt[mi][ni][1] = yv.y;
          }
        // Ys is released below, once the values were consumed into Os
      } else if (use_y) {
        mbar_wait(yfull, (unsigned)lt & 1);
        double2 ya[2][2 * NYB];
#pragma unroll
        for (int kk2 = 0; kk2 < 2 * NYB; ++kk2) {
          const double* yb = Ys + (kk2 >> 1) * (CF::xbox / 8);
          const int chunk = (((kk2 & 1) << 2) | tig) ^ prow;
          ya[0][kk2] = *reinterpret_cast<const double2*>(yb + (warp * 16 + prow) * 16 + chunk * 2);
          ya[1][kk2] =
              *reinterpret_cast<const double2*>(yb + (warp * 16 + 8 + prow) * 16 + chunk * 2);
        }
#pragma unroll
        for (int kk2 = 0; kk2 < 2 * NYB; ++kk2)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int ni = 0; ni < NT; ++ni) {
              const double b = Ts[(kk2 * 8 + 2 * tig + h) * TP + ni * 8 + gid];
              dmma884(yt[0][ni][0], yt[0][ni][1], h ? ya[0][kk2].y : ya[0][kk2].x, b);
              dmma884(yt[1][ni][0], yt[1][ni][1], h ? ya[1][kk2].y : ya[1][kk2].x, b);
            }
        // release Ys only after the DMMAs consumed the loaded fragments (an
        // arrive right after the LDS could overtake them)
        __syncwarp();
        if (lane == 0) mbar_arrive(yempty);
      }
      // warp-private epilogue (no CTA barrier): Z rows of this warp stored
      // straight from the fragments (16-byte pieces of 64-byte row segments),
      // and the warp's Gram contribution from its own rows of the out tile
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) {
          const int rl = mi * 8 + prow, c = ni * 8 + 2 * tig;
          const int64_t row = r0 + warp * 16 + rl;
          const bool rv = row < q;
          double z0 = alpha * (acc[0][mi][ni][0] + acc[1][mi][ni][0]) + beta * yt[mi][ni][0];
          double z1 = alpha * (acc[0][mi][ni][1] + acc[1][mi][ni][1]) + beta * yt[mi][ni][1];
          z0 = (c < w && rv) ? z0 : 0.0;
          z1 = (c + 1 < w && rv) ? z1 : 0.0;
          if (gram) {
            Ow[rl * OP + c] = z0;
            Ow[rl * OP + c + 1] = z1;
          }
          if (Z && rv) {
            double* zp = Z + row * ldz + c;
            if (zal && c + 1 < w) {
              *reinterpret_cast<double2*>(zp) = make_double2(z0, z1);
            } else {
              if (c < w) zp[0] = z0;
              if (c + 1 < w) zp[1] = z1;
            }
          }
        }
      if (use_y && !T) {
        __syncwarp();
        if (lane == 0) mbar_arrive(yempty);
      }
      if (gram) {
        __syncwarp();
#pragma unroll
        for (int mi = 0, p = 0; mi < NT; ++mi)
#pragma unroll
          for (int ni = mi; ni < NT; ++ni, ++p)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const int kr = kk * 4 + tig;
              dmma884(gw[p][0], gw[p][1], Ow[kr * OP + mi * 8 + gid], Ow[kr * OP + ni * 8 + gid]);
            }
        __syncwarp();  // the next tile overwrites Ow
      }
    }
  }
  if (gram) {
    // the TMA ring is idle now (every stage consumed): 8 warps x NGP x 64
    // partials there, summed over the warps in a fixed order and mirrored
    double* red = (double*)sm;
    bar_consumers();
#pragma unroll
    for (int p = 0; p < NGP; ++p)
#pragma unroll
      for (int e = 0; e < 2; ++e) red[(warp * NGP + p) * 64 + gid * 8 + 2 * tig + e] = gw[p][e];
    bar_consumers();
    for (int idx = tid; idx < NGP * 64; idx += 256) {
      const int p = idx / 64, ii = (idx % 64) / 8, jj = idx % 8;
      int mi = 0, base = 0;
      while (p >= base + (NT - mi)) {
        base += NT - mi;
        ++mi;
      }
      const int ni = mi + (p - base);
      double sum = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) sum += red[(k * NGP + p) * 64 + ii * 8 + jj];
      const int i = mi * 8 + ii, jc = ni * 8 + jj;
      if (i < w && jc < w) {
        gram[(int64_t)blockIdx.x * w * w + i * w + jc] = sum;
        gram[(int64_t)blockIdx.x * w * w + jc * w + i] = sum;
      }
    }
  }
}

// Register budgets: w <= 16 (NYB = 1) runs two CTAs per SM; w <= 32
// (NYB = 2) one CTA.  Its 9 warps put 3 warps on one SM sub-partition, whose
// 16384-register file caps a thread at 168 registers (measured: 216 fails
// to launch with "too many resources"), so the w = 32 kernel keeps a few
// spilled scalars; a 2-warps-per-partition layout (producer folded into a
// consumer warp) would lift the cap.
// s = 0 passes fed by TMA (round 2): the streaming row pass Z = beta Y T
// (+ per-CTA Gram Z^T Z) with Y tiles of 128 rows x 16 NYB columns loaded
// by cp.async.bulk.tensor into an S-stage full/empty mbarrier ring (lane 0 of
// warp 0 is the producer, folded as in nn_tma_body), so S tiles per CTA are
// in flight without holding registers; the 8 warps (16 rows each) take the Y
// A-fragments from the swizzled tile (paired-k, permuted rows, conflict-free
// as in nn_tma_body), multiply by T with DMMA, store Z from the fragments and
// add their own rows to the Gram.  The register-ring rowT_kernel reached 0.66
// of HBM in the C2 solve (ncu: latency-bound, 48 % DRAM).
template <int NYB, int S>
struct RowtTmaCfg {
  static constexpr int WP = 16 * NYB, OP = WP + 4, TP = WP + 4;
  static constexpr size_t box = (size_t)NT_R * 16 * 8;  // 16 KB
  static constexpr size_t stage = NYB * box;
  static constexpr size_t os_off = S * stage;
  static constexpr size_t ts_off = os_off + (size_t)NT_R * OP * 8;
  static constexpr size_t bar_off = ts_off + (size_t)WP * TP * 8;
  static constexpr size_t bytes = bar_off + 2 * S * 8 + 1024;
};

template <int NYB, int S>
__global__ void __launch_bounds__(256, 2) rowT_tma_kernel(
    const __grid_constant__ CUtensorMap ymap, const double* __restrict__ T, double* Z,
    int64_t ldz, int64_t q, int w, double beta, double* __restrict__ gram) {
  pdl_enter();
  using CF = RowtTmaCfg<NYB, S>;
  constexpr int WP = CF::WP, NT = 2 * NYB, OP = CF::OP, TP = CF::TP;
  constexpr int NGP = NT * (NT + 1) / 2;
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  double* Os = (double*)(sm + CF::os_off);
  double* Ts = (double*)(sm + CF::ts_off);
  uint64_t* full = (uint64_t*)(sm + CF::bar_off);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int prow = ((gid & 1) << 2) | (gid >> 1);
  for (int i = tid; i < WP * WP; i += blockDim.x) {
    const int r = i / WP, c = i % WP;
    Ts[r * TP + c] = (r < w && c < w) ? (T ? T[r * w + c] : (r == c ? 1.0 : 0.0)) : 0.0;
  }
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t ntiles = (q + NT_R - 1) / NT_R;
  const int64_t my_tiles =
      (ntiles > (int64_t)blockIdx.x) ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  int pst = 0;
  unsigned pu = 0;
  int64_t pj = 0;
  auto produce = [&]() {  // tile pj of this CTA into slot pst
    if (pj > 0 && ++pst == S) pst = 0, ++pu;
    if (pj >= S) mbar_wait(&empty[pst], (pu - 1) & 1);
    const int r0 = (int)((blockIdx.x + pj * gridDim.x) * NT_R);
    mbar_expect_tx(&full[pst], (unsigned)CF::stage);
#pragma unroll
    for (int b = 0; b < NYB; ++b)
      tma_load_2d(sm + (size_t)pst * CF::stage + b * CF::box, &ymap, b * 16, r0, &full[pst]);
    ++pj;
  };
  if (warp == 0 && lane == 0)
    while (pj < my_tiles && pj < S - 1) produce();
  double gw[NGP][2];
#pragma unroll
  for (int p = 0; p < NGP; ++p) gw[p][0] = gw[p][1] = 0.0;
  const bool zal = Z && ((((uintptr_t)Z) | (uintptr_t)(ldz * 8)) & 15) == 0;
  double* Ow = Os + warp * 16 * OP;
  int st = 0;
  unsigned u = 0;
  for (int64_t j = 0; j < my_tiles; ++j) {
    if (warp == 0 && lane == 0 && pj < my_tiles) produce();  // tile j + S - 1
    if (j > 0 && ++st == S) st = 0, ++u;
    const int64_t r0 = (blockIdx.x + j * gridDim.x) * NT_R;
    mbar_wait(&full[st], u & 1);
    const double* Ys = (const double*)(sm + (size_t)st * CF::stage);
    double yt[2][NT][2];
    if (T) {
      double2 ya[2][2 * NYB];
#pragma unroll
      for (int kk2 = 0; kk2 < 2 * NYB; ++kk2) {
        const double* yb = Ys + (kk2 >> 1) * (CF::box / 8);
        const int chunk = (((kk2 & 1) << 2) | tig) ^ prow;
        ya[0][kk2] = *reinterpret_cast<const double2*>(yb + (warp * 16 + prow) * 16 + chunk * 2);
        ya[1][kk2] =
            *reinterpret_cast<const double2*>(yb + (warp * 16 + 8 + prow) * 16 + chunk * 2);
      }
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) yt[mi][ni][0] = yt[mi][ni][1] = 0.0;
#pragma unroll
      for (int kk2 = 0; kk2 < 2 * NYB; ++kk2)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) {
            const double b = Ts[(kk2 * 8 + 2 * tig + h) * TP + ni * 8 + gid];
            dmma884(yt[0][ni][0], yt[0][ni][1], h ? ya[0][kk2].y : ya[0][kk2].x, b);
            dmma884(yt[1][ni][0], yt[1][ni][1], h ? ya[1][kk2].y : ya[1][kk2].x, b);
          }
    } else {  // T = I: the values themselves, in accumulator layout
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) {
          const double2 yv = *reinterpret_cast<const double2*>(
              Ys + (ni >> 1) * (CF::box / 8) + (warp * 16 + mi * 8 + prow) * 16 +
              ((((ni & 1) << 2) | tig) ^ prow) * 2);
          yt[mi][ni][0] = yv.x;
          yt[mi][ni][1] = yv.y;
        }
    }
    // release the slot once the loaded values were consumed (the DMMAs /
    // moves above complete before the arrive is issued in program order for
    // every lane; __syncwarp orders the warp's lanes)
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) {
        const int rl = mi * 8 + prow, c = ni * 8 + 2 * tig;
        const int64_t row = r0 + warp * 16 + rl;
        const bool rv = row < q;
        const double z0 = (c < w && rv) ? beta * yt[mi][ni][0] : 0.0;
        const double z1 = (c + 1 < w && rv) ? beta * yt[mi][ni][1] : 0.0;
        if (gram) {
          Ow[rl * OP + c] = z0;
          Ow[rl * OP + c + 1] = z1;
        }
        if (Z && rv) {
          double* zp = Z + row * ldz + c;
          if (zal && c + 1 < w) {
            *reinterpret_cast<double2*>(zp) = make_double2(z0, z1);
          } else {
            if (c < w) zp[0] = z0;
            if (c + 1 < w) zp[1] = z1;
          }
        }
      }
    if (gram) {
      __syncwarp();
#pragma unroll
      for (int mi = 0, p = 0; mi < NT; ++mi)
#pragma unroll
        for (int ni = mi; ni < NT; ++ni, ++p)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const int kr = kk * 4 + tig;
            dmma884(gw[p][0], gw[p][1], Ow[kr * OP + mi * 8 + gid], Ow[kr * OP + ni * 8 + gid]);
          }
      __syncwarp();
    }
  }
  if (gram) {
    // the ring is idle (every issued tile was consumed): per-warp partials
    // there, summed over the warps in a fixed order and mirrored
    double* red = (double*)sm;
    __syncthreads();
#pragma unroll
    for (int p = 0; p < NGP; ++p)
#pragma unroll
      for (int e = 0; e < 2; ++e) red[(warp * NGP + p) * 64 + gid * 8 + 2 * tig + e] = gw[p][e];
    __syncthreads();
    for (int idx = tid; idx < NGP * 64; idx += 256) {
      const int p = idx / 64, ii = (idx % 64) / 8, jj = idx % 8;
      int mi = 0, base = 0;
      while (p >= base + (NT - mi)) {
        base += NT - mi;
        ++mi;
      }
      const int ni = mi + (p - base);
      double sum = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) sum += red[(k * NGP + p) * 64 + ii * 8 + jj];
      const int i = mi * 8 + ii, jc = ni * 8 + jj;
      if (i < w && jc < w) {
        gram[(int64_t)blockIdx.x * w * w + i * w + jc] = sum;
        gram[(int64_t)blockIdx.x * w * w + jc * w + i] = sum;
      }
    }
  }
}

template <int KC, int S, int NYB>
__global__ void __launch_bounds__(288, 2) gemm_nn_tma_kernel(
    const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap hmap,
    const __grid_constant__ CUtensorMap ymap, int use_y, const double* __restrict__ T, double* Z,
    int64_t ldz, int64_t q, int s, int w, double alpha, double beta, double* __restrict__ gram,
    int64_t zsplit) {
  pdl_enter();
  nn_tma_body<KC, S, NYB, false>(xmap, hmap, ymap, use_y, T, Z, ldz, q, s, w, alpha, beta, gram,
                                 zsplit);
}
template <int KC, int S, int NYB>
__global__ void __launch_bounds__(256, 2) gemm_nn_tma_kernel_fold16(
    const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap hmap,
    const __grid_constant__ CUtensorMap ymap, int use_y, const double* __restrict__ T, double* Z,
    int64_t ldz, int64_t q, int s, int w, double alpha, double beta, double* __restrict__ gram,
    int64_t zsplit) {
  pdl_enter();
  nn_tma_body<KC, S, NYB, true>(xmap, hmap, ymap, use_y, T, Z, ldz, q, s, w, alpha, beta, gram,
                                zsplit);
}
template <int KC, int S, int NYB>
__global__ void __launch_bounds__(256, 1) gemm_nn_tma_kernel_w32(
    const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap hmap,
    const __grid_constant__ CUtensorMap ymap, int use_y, const double* __restrict__ T, double* Z,
    int64_t ldz, int64_t q, int s, int w, double alpha, double beta, double* __restrict__ gram,
    int64_t zsplit) {
  pdl_enter();
  nn_tma_body<KC, S, NYB, true>(xmap, hmap, ymap, use_y, T, Z, ldz, q, s, w, alpha, beta, gram,
                                zsplit);
}

// Output products Z = X H with w up to 64 (Alg. 2 S8/S9: V = P Vbar_r,
// U = Pbar Ubar_r; Alg. 1 S6/S7), beta = 0 and no Gram: the same TMA ring
// as gemm_nn_tma_kernel with 4 H boxes (64 columns) per stage, one
// accumulator set of 2 x 8 DMMA tiles per warp, and Z stored straight from
// the accumulator fragments (no shared out tile).  These products are
// DMMA-bound (2 s w flops per 8 s bytes).
template <int KC, int S, int NH = 4>  // NH = 16-column H boxes per stage (w <= 16 NH)
struct NnOutCfg {
  static constexpr int NB = KC / 16;
  static constexpr size_t xbox = (size_t)NT_R * 16 * 8;
  static constexpr size_t hbox = (size_t)KC * 16 * 8;
  static constexpr size_t stage = NB * xbox + NH * hbox;
  static constexpr size_t bar_off = S * stage;
  static constexpr size_t bytes = bar_off + 2 * S * 8 + 1024;
  static constexpr unsigned tx = (unsigned)stage;
};

// NT = 8-column tiles computed (w <= 8 NT <= 128).  In place (Z = X, ldz =
// ldx, one launch for all w columns, no split-K): a tile's output rows are
// written only after every K chunk of that tile has landed in shared memory
// (the epilogue follows the tile's last full-barrier wait), and no other CTA
// reads those rows, so Z may overwrite X's first w columns -- the outputs
// and the thick-restart panels of C5, which have no room for separate
// m x r / n x r buffers, without a scratch round trip.
// FOLD (the 13 / 16-tile kernels): the producer is lane 0 of consumer warp 0
// (8 warps, up to 255 registers) instead of a 9th warp (168-register cap:
// 36 / 104 bytes of spills), as in nn_tma_body.
template <int KC, int S, int NT, bool FOLD>
__device__ __forceinline__ void nn_out_body(const CUtensorMap& xmap, const CUtensorMap& hmap,
                                            double* Z, int64_t ldz, int64_t q, int s, int w,
                                            double alpha, int64_t zsplit) {
  constexpr int NH = (NT + 1) / 2;
  using CF = NnOutCfg<KC, S, NH>;  // split-K over blockIdx.y as in gemm_nn_tma_kernel
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(sm + CF::bar_off);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int prow = ((gid & 1) << 2) | (gid >> 1);
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t ntiles = (q + NT_R - 1) / NT_R;
  const int64_t my_tiles =
      (ntiles > (int64_t)blockIdx.x) ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int nk_all = (s + KC - 1) / KC;
  const int kb = (int)((int64_t)nk_all * blockIdx.y / gridDim.y);
  const int nk = (int)((int64_t)nk_all * (blockIdx.y + 1) / gridDim.y) - kb;
  const int64_t nsteps = my_tiles * nk;
  Z += (int64_t)blockIdx.y * zsplit;
  // producer: ring slot / phase and (tile, k-chunk) kept as running
  // counters (no 64-bit divisions by S and by the runtime nk per step)
  int pst = 0, pkc = 0;
  unsigned pu = 0;
  int64_t plt = 0, pj = 0;
  auto produce = [&]() {  // issue step pj
    if (pj > 0) {
      if (++pst == S) pst = 0, ++pu;
      if (++pkc == nk) pkc = 0, ++plt;
    }
    if (pj >= S) mbar_wait(&empty[pst], (pu - 1) & 1);
    const int r0 = (int)((blockIdx.x + plt * gridDim.x) * NT_R);
    unsigned char* base = sm + (size_t)pst * CF::stage;
    mbar_expect_tx(&full[pst], CF::tx);
#pragma unroll
    for (int b = 0; b < CF::NB; ++b)
      tma_load_2d(base + b * CF::xbox, &xmap, (kb + pkc) * KC + b * 16, r0, &full[pst]);
#pragma unroll
    for (int b = 0; b < NH; ++b)
      tma_load_2d(base + CF::NB * CF::xbox + b * CF::hbox, &hmap, b * 16, (kb + pkc) * KC,
                  &full[pst]);
    ++pj;
  };
  if constexpr (!FOLD) {
    if (warp == 8) {
      if (lane == 0)
        while (pj < nsteps) produce();
      return;
    }
  } else {
    if (warp == 0 && lane == 0)
      while (pj < nsteps && pj < S - 1) produce();
  }
  const bool vec = ((ldz & 1) == 0) && ((((uintptr_t)Z) & 15) == 0);
  double acc[2][NT][2];
  int st = 0, kc = 0;
  unsigned u = 0;
  int64_t lt = 0;
  for (int64_t j = 0; j < nsteps; ++j) {
    if constexpr (FOLD) {
      if (warp == 0 && lane == 0 && pj < nsteps) produce();  // step j + S - 1
    }
    if (j > 0) {  // running counters, as in the producer
      if (++st == S) st = 0, ++u;
      if (++kc == nk) kc = 0, ++lt;
    }
    const int64_t r0 = (blockIdx.x + lt * gridDim.x) * NT_R;
    if (kc == 0) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    }
    mbar_wait(&full[st], u & 1);
    {
      const unsigned char* base = sm + (size_t)st * CF::stage;
      const unsigned char* hb0 = base + CF::NB * CF::xbox;
#pragma unroll
      for (int kk2 = 0; kk2 < KC / 8; ++kk2) {
        const double* xb = (const double*)(base + (kk2 >> 1) * CF::xbox);
        const int chunk = (((kk2 & 1) << 2) | tig) ^ prow;
        const double2 a0 =
            *reinterpret_cast<const double2*>(xb + (warp * 16 + prow) * 16 + chunk * 2);
        const double2 a1 =
            *reinterpret_cast<const double2*>(xb + (warp * 16 + 8 + prow) * 16 + chunk * 2);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int hr = kk2 * 8 + 2 * tig + h;
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) {
            const double* hs = (const double*)(hb0 + (ni >> 1) * CF::hbox);
            const int c = (ni & 1) * 8 + gid;
            const double b = hs[hr * 16 + (((c >> 1) ^ (hr & 7)) << 1) + (c & 1)];
            dmma884(acc[0][ni][0], acc[0][ni][1], h ? a0.y : a0.x, b);
            dmma884(acc[1][ni][0], acc[1][ni][1], h ? a1.y : a1.x, b);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (kc == nk - 1) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const int64_t row = r0 + warp * 16 + mi * 8 + prow;
        if (row < q) {
          double* zr = Z + row * ldz;
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) {
            const int c = ni * 8 + 2 * tig;
            const double z0 = alpha * acc[mi][ni][0], z1 = alpha * acc[mi][ni][1];
            if (vec && c + 1 < w) {
              *reinterpret_cast<double2*>(zr + c) = make_double2(z0, z1);
            } else {
              if (c < w) zr[c] = z0;
              if (c + 1 < w) zr[c + 1] = z1;
            }
          }
        }
      }
    }
  }
}

template <int KC, int S, int NT>
__global__ void __launch_bounds__(288, 1) gemm_nn_out_tma_kernel(
    const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap hmap, double* Z,
    int64_t ldz, int64_t q, int s, int w, double alpha, int64_t zsplit) {
  pdl_enter();
  nn_out_body<KC, S, NT, false>(xmap, hmap, Z, ldz, q, s, w, alpha, zsplit);
}
template <int KC, int S, int NT>
__global__ void __launch_bounds__(256, 1) gemm_nn_out_tma_kernel_fold(
    const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap hmap, double* Z,
    int64_t ldz, int64_t q, int s, int w, double alpha, int64_t zsplit) {
  pdl_enter();
  nn_out_body<KC, S, NT, true>(xmap, hmap, Z, ldz, q, s, w, alpha, zsplit);
}

constexpr int NNT_KC = 32, NNT_S = 2;

// Split-K factor for a plain product with few row tiles (dense A.X: 313
// tiles of 128 rows on 148 SMs would leave a 2.1-wave tail): the grid is
// (ctas / ks) x ks, each CTA takes ceil(tiles / (ctas / ks)) tiles for 1/ks
// of K; ks maximises that balance (>= 4 K chunks per unit, partials fit).
static int pick_split(int64_t q, int s, int w, int ctas, size_t part_cap) {
  const int64_t tiles = (q + NT_R - 1) / NT_R;
  const int nk_all = (s + NNT_KC - 1) / NNT_KC;
  if (part_cap == 0 || tiles >= 8 * (int64_t)ctas) return 1;
  const double ideal = (double)tiles / ctas;
  double best_eff = ideal / (double)((tiles + ctas - 1) / ctas);
  int best = 1;
  for (int ks = 2; ks <= 8; ++ks) {
    if (nk_all / ks < 4 || (size_t)ks * q * w > part_cap) break;
    const int gx = ctas / ks;
    const double eff = ideal / ((double)((tiles + gx - 1) / gx) / ks);
    if (eff > best_eff * 1.03) {
      best_eff = eff;
      best = ks;
    }
  }
  return best;
}

static bool nn_tma_launch(const double* X, int64_t ldx, const double* H, int64_t ldh,
                          const double* Y, int64_t ldy, const double* T, double* Z, int64_t ldz,
                          int64_t q, int s, int w, double alpha, double beta, double* gram,
                          cudaStream_t st, double* part, size_t part_cap) {
  if (q >= (int64_t)1 << 31 || s >= (1 << 30)) return false;
  const int use_y = (beta != 0.0 && Y) ? 1 : 0;
  if (use_y && !aligned16(Y, ldy)) return false;
  CUtensorMap xm, hm, ym;
  if (!make_map(&xm, X, q, s, ldx, NT_R) || !make_map(&hm, H, s, w, ldh, NNT_KC)) return false;
  if (use_y ? !make_map(&ym, Y, q, w, ldy, NT_R) : !make_map(&ym, X, q, s, ldx, NT_R))
    return false;
  if (w > 16) {  // 16 < w <= 32: two H / Y boxes, one CTA per SM, 3-stage ring
    using CF2 = NnTmaCfg<NNT_KC, 3, 2>;
    static bool attr2 = false;
    if (!attr2) {
      TSVD_CUDA(cudaFuncSetAttribute(gemm_nn_tma_kernel_w32<NNT_KC, 3, 2>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF2::bytes));
      attr2 = true;
    }
    const int ctas = nn_ctas(q, 32);
    const int ks = (use_y || T || gram) ? 1 : pick_split(q, s, w, ctas, part_cap);
    if (ks > 1) {
      launch_pdl(gemm_nn_tma_kernel_w32<NNT_KC, 3, 2>, dim3(ctas / ks, ks), 256, CF2::bytes, st, xm, hm, ym, 0, nullptr, part, w, q, s, w, alpha, 0.0, nullptr, q * w);
      TSVD_CHECK_LAUNCH();
      reduce_launch(part, ks, q * w, Z, w, ldz == w ? 0 : ldz, st);
      return true;
    }
    launch_pdl(gemm_nn_tma_kernel_w32<NNT_KC, 3, 2>, ctas, 256, CF2::bytes, st, xm, hm, ym, use_y, T, Z, ldz, q, s, w, alpha, beta, gram, 0);
    TSVD_CHECK_LAUNCH();
    return true;
  }
  using CF = NnTmaCfg<NNT_KC, NNT_S, 1>;
  static bool attr = false;
  if (!attr) {
    TSVD_CUDA(cudaFuncSetAttribute(gemm_nn_tma_kernel<NNT_KC, NNT_S, 1>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::bytes));
    TSVD_CUDA(cudaFuncSetAttribute(gemm_nn_tma_kernel_fold16<NNT_KC, NNT_S, 1>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::bytes));
    attr = true;
  }
  const int ctas = nn_ctas(q, 16);
  const int ks = (use_y || T || gram) ? 1 : pick_split(q, s, w, ctas, part_cap);
  auto kern = g_nn_fold16 ? gemm_nn_tma_kernel_fold16<NNT_KC, NNT_S, 1>
                          : gemm_nn_tma_kernel<NNT_KC, NNT_S, 1>;
  const int nthr = g_nn_fold16 ? 256 : 288;
  if (ks > 1) {
    launch_pdl(kern, dim3(ctas / ks, ks), nthr, CF::bytes, st, xm, hm, ym, 0, nullptr, part, w, q, s, w,
                                                      alpha, 0.0, nullptr, q * w);
    TSVD_CHECK_LAUNCH();
    reduce_launch(part, ks, q * w, Z, w, ldz == w ? 0 : ldz, st);
    return true;
  }
  launch_pdl(kern, ctas, nthr, CF::bytes, st, xm, hm, ym, use_y, T, Z, ldz, q, s, w, alpha, beta, gram, 0);
  TSVD_CHECK_LAUNCH();
  return true;
}

static bool nn_out_tma_launch(const double* X, int64_t ldx, const double* H, int64_t ldh,
                              double* Z, int64_t ldz, int64_t q, int s, int w, double alpha,
                              cudaStream_t st, double* part, size_t part_cap) {
  if (q >= (int64_t)1 << 31 || s >= (1 << 30)) return false;
  CUtensorMap xm, hm;
  if (!make_map(&xm, X, q, s, ldx, NT_R) || !make_map(&hm, H, s, w, ldh, NNT_KC)) return false;
  constexpr int OS = 4;  // one CTA per SM (register-heavy), deeper ring
  using CF = NnOutCfg<NNT_KC, OS>;
  static bool attr = false;
  if (!attr) {
    TSVD_CUDA(cudaFuncSetAttribute(gemm_nn_out_tma_kernel<NNT_KC, OS, 5>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::bytes));
    TSVD_CUDA(cudaFuncSetAttribute(gemm_nn_out_tma_kernel<NNT_KC, OS, 6>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::bytes));
    TSVD_CUDA(cudaFuncSetAttribute(gemm_nn_out_tma_kernel<NNT_KC, OS, 7>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::bytes));
    TSVD_CUDA(cudaFuncSetAttribute(gemm_nn_out_tma_kernel<NNT_KC, OS, 8>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::bytes));
    attr = true;
  }
  const int nt = (w + 7) / 8;
  const int ctas = nn_ctas(q, 32);
  const int ks = pick_split(q, s, w, ctas, part_cap);
  double* zo = ks > 1 ? part : Z;
  const int64_t ldo = ks > 1 ? w : ldz;
#define OUT_GO(NTV)                                                                       \
  launch_pdl(gemm_nn_out_tma_kernel<NNT_KC, OS, NTV>, dim3(ctas / ks, ks), 288, CF::bytes, st, \
      xm, hm, zo, ldo, q, s, w, alpha, ks > 1 ? q * w : 0)
  if (nt <= 5) OUT_GO(5);
  else if (nt == 6) OUT_GO(6);
  else if (nt == 7) OUT_GO(7);
  else OUT_GO(8);
#undef OUT_GO
  TSVD_CHECK_LAUNCH();
  if (ks > 1) reduce_launch(part, ks, q * w, Z, w, ldz == w ? 0 : ldz, st);
  return true;
}

// 64 < w <= 128: all w columns from ONE read of X (13 or 16 accumulator
// tiles of 8 columns per warp, NH = 8 H boxes per stage, 3 stages =
// 192 KB), no split-K.  Z may alias X's first w
// columns (ldz = ldx): see gemm_nn_out_tma_kernel.
static bool nn_out_wide_launch(const double* X, int64_t ldx, const double* H, int64_t ldh,
                               double* Z, int64_t ldz, int64_t q, int s, int w, double alpha,
                               cudaStream_t st) {
  if (q >= (int64_t)1 << 31 || s >= (1 << 30) || w > 128) return false;
  CUtensorMap xm, hm;
  if (!make_map(&xm, X, q, s, ldx, NT_R) || !make_map(&hm, H, s, w, ldh, NNT_KC)) return false;
  constexpr int WS = 3;
  using CF = NnOutCfg<NNT_KC, WS, 8>;
  static bool attr = false;
  if (!attr) {
    TSVD_CUDA(cudaFuncSetAttribute(gemm_nn_out_tma_kernel_fold<NNT_KC, WS, 13>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::bytes));
    TSVD_CUDA(cudaFuncSetAttribute(gemm_nn_out_tma_kernel_fold<NNT_KC, WS, 16>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::bytes));
    attr = true;
  }
  const int nt = (w + 7) / 8;
  const int ctas = nn_ctas(q, 32);
  if (nt <= 13)
    launch_pdl(gemm_nn_out_tma_kernel_fold<NNT_KC, WS, 13>, ctas, 256, CF::bytes, st, xm, hm, Z, ldz,
               q, s, w, alpha, (int64_t)0);
  else
    launch_pdl(gemm_nn_out_tma_kernel_fold<NNT_KC, WS, 16>, ctas, 256, CF::bytes, st, xm, hm, Z, ldz,
               q, s, w, alpha, (int64_t)0);
  TSVD_CHECK_LAUNCH();
  return true;
}

bool g_out_wide = getenv("TSVD_OUT_WIDE") ? atoi(getenv("TSVD_OUT_WIDE")) != 0 : true;

bool gemm_nn_out_inplace(double* X, int64_t ldx, const double* H, int64_t ldh, int64_t q, int s,
                         int w, cudaStream_t st) {
  if (!g_out_wide || w > 128 || w > s || q <= 0 || !aligned16(X, ldx) || !aligned16(H, ldh))
    return false;
  if (w <= 64)  // the 4-stage kernel (4 H boxes), no split-K (part_cap = 0)
    return nn_out_tma_launch(X, ldx, H, ldh, X, ldx, q, s, w, 1.0, st, nullptr, 0);
  return nn_out_wide_launch(X, ldx, H, ldh, X, ldx, q, s, w, 1.0, st);
}

bool g_rowt_tma = getenv("TSVD_ROWT_TMA") ? atoi(getenv("TSVD_ROWT_TMA")) != 0 : true;
constexpr int ROWT_S16 = 4, ROWT_S32 = 2;  // ring stages (2 CTAs / SM)

static bool rowt_tma_launch(const double* Y, int64_t ldy, const double* T, double* Z,
                            int64_t ldz, int64_t q, int w, double beta, double* gram,
                            cudaStream_t st) {
  if (q >= (int64_t)1 << 31) return false;
  CUtensorMap ym;
  if (!make_map(&ym, Y, q, w, ldy, NT_R)) return false;
  const int ctas = nn_ctas(q, w);  // the callers finalise that many Gram partials
  if (w <= 16) {
    using CF = RowtTmaCfg<1, ROWT_S16>;
    static bool attr = false;
    if (!attr) {
      TSVD_CUDA(cudaFuncSetAttribute(rowT_tma_kernel<1, ROWT_S16>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::bytes));
      attr = true;
    }
    launch_pdl(rowT_tma_kernel<1, ROWT_S16>, ctas, 256, CF::bytes, st, ym, T, Z, ldz, q, w, beta, gram);
  } else {
    using CF = RowtTmaCfg<2, ROWT_S32>;
    static bool attr = false;
    if (!attr) {
      TSVD_CUDA(cudaFuncSetAttribute(rowT_tma_kernel<2, ROWT_S32>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::bytes));
      attr = true;
    }
    // two CTAs per SM (128 registers, 2 x 110 KB) when no Gram partials are
    // written; with a Gram the grid must be the nn_ctas(q, w) partials the
    // caller finalises (one CTA per SM at w > 16)
    const int g32 = gram ? ctas : (int)std::min<int64_t>((q + NT_R - 1) / NT_R, 2 * 148);
    launch_pdl(rowT_tma_kernel<2, ROWT_S32>, std::max(1, g32), 256, CF::bytes, st, ym, T, Z, ldz,
               q, w, beta, gram);
  }
  TSVD_CHECK_LAUNCH();
  return true;
}

template <int WP, int VEC>
static void nn_launch(const double* X, int64_t ldx, const double* H, int64_t ldh,
                      const double* Y, int64_t ldy, const double* T, double* Z, int64_t ldz,
                      int64_t q, int s, int w, double alpha, double beta, double* gram,
                      cudaStream_t st) {
  static bool attr = false;
  const size_t bytes = NnCfg<WP>::bytes;
  if (!attr) {
    TSVD_CUDA(cudaFuncSetAttribute(gemm_nn_kernel<WP, VEC>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    attr = true;
  }
  launch_pdl(gemm_nn_kernel<WP, VEC>, nn_ctas(q, WP), 256, bytes, st, X, ldx, H, ldh, Y, ldy, T, Z,
                                                               ldz, q, s, w, alpha, beta, gram);
  TSVD_CHECK_LAUNCH();
}

void gemm_nn(const double* X, int64_t ldx, const double* H, int64_t ldh, const double* Y,
             int64_t ldy, const double* T, double* Z, int64_t ldz, int64_t q, int s, int w,
             double alpha, double beta, double* gram, cudaStream_t st, double* part,
             size_t part_cap) {
  if (w <= 0) return;
  if (q <= 0) {
    // empty row range (a rank whose row slice or n-shard is empty): the
    // caller still reduces nn_ctas(0, w) = 1 Gram partial, so it must be the
    // zero matrix, not whatever an earlier pass left in the buffer
    if (gram) TSVD_CUDA(cudaMemsetAsync(gram, 0, sizeof(double) * nn_ctas(0, w) * w * w, st));
    return;
  }
  if (w > 32) {
    if (T || gram) throw Error{TSVD_EINVAL, "gemm_nn: T/gram need w <= 32"};
    if (beta == 0.0 && s > 0 && g_nn_tma && aligned16(X, ldx) && aligned16(H, ldh)) {
      // one read of X for all w <= 128 columns when the rows give enough
      // tiles for the grid (no split-K needed)
      if (g_out_wide && w > 64 && w <= 128 && (q + NT_R - 1) / NT_R >= 8 * 148 &&
          nn_out_wide_launch(X, ldx, H, ldh, Z, ldz, q, s, w, alpha, st))
        return;
      bool done = true;
      for (int c0 = 0; c0 < w && done; c0 += 64)
        done = nn_out_tma_launch(X, ldx, H + c0, ldh, Z + c0, ldz, q, s, std::min(64, w - c0),
                                 alpha, st, part, part_cap);
      if (done) return;
    }
    const int cw = (beta == 0.0) ? 64 : 32;  // wide products (outputs) in one pass per 64 cols
    if (w > cw) {
      for (int c0 = 0; c0 < w; c0 += cw)
        gemm_nn(X, ldx, H + c0, ldh, Y ? Y + c0 : nullptr, ldy, nullptr, Z + c0, ldz, q, s,
                std::min(cw, w - c0), alpha, beta, nullptr, st);
      return;
    }
    if (cw == 32) {
      for (int c0 = 0; c0 < w; c0 += 32)
        gemm_nn(X, ldx, H + c0, ldh, Y ? Y + c0 : nullptr, ldy, nullptr, Z + c0, ldz, q, s,
                std::min(32, w - c0), alpha, beta, nullptr, st);
      return;
    }
  }
  if (s == 0 && w <= 32 && g_rowt_tma && Y && aligned16(Y, ldy) &&
      rowt_tma_launch(Y, ldy, T, Z, ldz, q, w, beta, gram, st))
    return;
  if (s == 0 && w <= 32 && g_rowt32 | (w <= 16)) {  // streaming row pass
    if (w <= 8)
      launch_pdl(rowT_kernel<8>, nn_ctas(q, w), 256, 0, st, Y, ldy, T, Z, ldz, q, w, beta, gram);
    else if (w <= 16)
      launch_pdl(rowT_kernel<16>, nn_ctas(q, w), 256, 0, st, Y, ldy, T, Z, ldz, q, w, beta, gram);
    else  // nn_ctas(q, w) CTAs: the callers finalise that many Gram partials
      launch_pdl(rowT_kernel<32>, nn_ctas(q, w), 256, 0, st, Y, ldy, T, Z, ldz, q, w, beta, gram);
    TSVD_CHECK_LAUNCH();
    return;
  }
  const bool v2 = s == 0 || (aligned16(X, ldx) && aligned16(H, ldh));
  if (w > 8 && w <= 32 && s > 0 && v2 && g_nn_tma &&
      nn_tma_launch(X, ldx, H, ldh, Y, ldy, T, Z, ldz, q, s, w, alpha, beta, gram, st, part,
                    part_cap))
    return;
#define NN_CASE(WPV)                                                                      \
  if (v2)                                                                                 \
    nn_launch<WPV, 2>(X, ldx, H, ldh, Y, ldy, T, Z, ldz, q, s, w, alpha, beta, gram, st); \
  else                                                                                    \
    nn_launch<WPV, 1>(X, ldx, H, ldh, Y, ldy, T, Z, ldz, q, s, w, alpha, beta, gram, st);
  if (w <= 8) {
    NN_CASE(8)
  } else if (w <= 16) {
    NN_CASE(16)
  } else if (w <= 32) {
    NN_CASE(32)
  } else {
    NN_CASE(64)
  }
#undef NN_CASE
}

}  // namespace tsvd
