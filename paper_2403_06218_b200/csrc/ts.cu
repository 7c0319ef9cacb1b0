// Tall-skinny FP64 products of the orthogonalisation passes, on the FP64
// tensor-core path (DMMA, mma.sync.m8n8k4.f64 - sm_100a has no f64
// tcgen05 kind, and DMMA has the same peak as DFMA, so it is used for the
// operand reuse it gives):
//
//   gemm_tn : C (s x w) = X^T Y'            Alg. 5 S1/S6 (H = P^T Q), dense A^T.P
//             Y' = Y L^{-T} applied on load  (Alg. 5 S5 fused into S6)
//   gemm_nn : Z (q x w) = beta Y' + alpha X H   Alg. 5 S2/S7 (Q -= P H), dense A.Q,
//             + per-CTA Gram Z^T Z              restart / outputs (Alg. 2 S7-S9)
//                                               Alg. 4 S1/S4, Alg. 5 S3/S8 fused
//   finalisers: fixed-order partial sums, b x b Cholesky with breakdown flag
//               (P:275), R = Lbar^T L^T, H += Hbar L^T (readings R4/R5).
//
// Everything is deterministic: split-K partials are summed in a fixed order
// by a separate kernel; no floating-point atomics.
#include "internal.h"

namespace tsvd {

// D(8x8) += A(8x4) B(4x8); per lane: a = A[gid][tig], b = B[tig][gid],
// d0,d1 = D[gid][2 tig + {0,1}]  (gid = lane>>2, tig = lane&3)
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// In-register row trsm: y <- y L^{-T}  (solve x L^T = y; L lower, w x w,
// row-major in shared memory with leading dimension WP).
template <int WP>
__device__ __forceinline__ void row_trsm(double (&y)[WP], const double* __restrict__ Ls, int w) {
#pragma unroll
  for (int j = 0; j < WP; ++j) {
    if (j < w) {
      double s = y[j];
#pragma unroll
      for (int k = 0; k < j; ++k) s = fma(-y[k], Ls[j * WP + k], s);
      y[j] = s / Ls[j * WP + j];
    }
  }
}

// ------------------------------------------------------------------ TN ---
constexpr int TN_ST = 32;   // columns of X per CTA tile
constexpr int TN_RB = 64;   // rows per iteration

TnGeom tn_geom(int64_t q, int s) {
  TnGeom g;
  g.s_tiles = (s + TN_ST - 1) / TN_ST;
  if (g.s_tiles < 1) g.s_tiles = 1;
  const int64_t row_tiles = (q + TN_RB - 1) / TN_RB;
  int64_t splits = (2 * 148 + g.s_tiles - 1) / g.s_tiles;
  if (splits > row_tiles) splits = row_tiles;
  if (splits < 1) splits = 1;
  g.splits = (int)splits;
  return g;
}

template <int WP>
__global__ void __launch_bounds__(256) gemm_tn_kernel(const double* __restrict__ X, int64_t ldx,
                                                      const double* __restrict__ Y, int64_t ldy,
                                                      const double* __restrict__ L, int64_t q,
                                                      int s, int w, double* __restrict__ C,
                                                      int64_t ldc, double* __restrict__ part) {
  constexpr int XP = TN_ST + 4, YP = WP + 4, NT = WP / 8;
  __shared__ double Xs[TN_RB * XP];
  __shared__ double Ys[TN_RB * YP];
  __shared__ double Ls[WP * WP];
  double* Cs = Xs;  // reused after the main loop (TN_ST*WP <= TN_RB*XP)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int s0 = blockIdx.x * TN_ST;
  const int scols = min(TN_ST, s - s0);
  const int split = blockIdx.y, nsplit = gridDim.y;
  const int64_t row_tiles = (q + TN_RB - 1) / TN_RB;
  const int64_t t_beg = row_tiles * split / nsplit, t_end = row_tiles * (split + 1) / nsplit;
  if (L) {
    for (int i = tid; i < WP * WP; i += 256) {
      const int r = i / WP, c = i % WP;
      Ls[i] = (r < w && c < w) ? L[r * w + c] : 0.0;
    }
  }
  double acc[4][NT][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

  for (int64_t t = t_beg; t < t_end; ++t) {
    const int64_t r0 = t * TN_RB;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < (TN_RB * TN_ST) / 256; ++u) {
      const int idx = tid + 256 * u;
      const int r = idx / TN_ST, c = idx % TN_ST;
      const int64_t row = r0 + r;
      Xs[r * XP + c] = (row < q && c < scols) ? __ldg(X + row * ldx + s0 + c) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < (TN_RB * WP) / 256; ++u) {
      const int idx = tid + 256 * u;
      const int r = idx / WP, c = idx % WP;
      const int64_t row = r0 + r;
      Ys[r * YP + c] = (row < q && c < w) ? __ldg(Y + row * ldy + c) : 0.0;
    }
    if (L) {
      __syncthreads();
      if (tid < TN_RB) {
        double y[WP];
#pragma unroll
        for (int c = 0; c < WP; ++c) y[c] = Ys[tid * YP + c];
        row_trsm<WP>(y, Ls, w);
#pragma unroll
        for (int c = 0; c < WP; ++c) Ys[tid * YP + c] = y[c];
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const int kr = warp * 8 + kk * 4 + tig;
      double a[4], b[NT];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = Xs[kr * XP + mi * 8 + gid];
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) b[ni] = Ys[kr * YP + ni * 8 + gid];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
  }
  // fixed-order cross-warp reduction
  __syncthreads();
  for (int wv = 0; wv < 8; ++wv) {
    if (warp == wv) {
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
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

__global__ void reduce_partials_kernel(const double* __restrict__ part, int nparts,
                                       int64_t count, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < nparts; ++p) s += part[(int64_t)p * count + i];
    out[i] = s;
  }
}

__global__ void scatter_ld_kernel(const double* __restrict__ src, int s, int w,
                                  double* __restrict__ C, int64_t ldc) {
  const int64_t n = (int64_t)s * w;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    C[(i / w) * ldc + (i % w)] = src[i];
}

void reduce_partials(const double* part, int nparts, int64_t count, double* out,
                     cudaStream_t st) {
  if (count <= 0) return;
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  reduce_partials_kernel<<<(unsigned)blocks, 256, 0, st>>>(part, nparts, count, out);
  TSVD_CHECK_LAUNCH();
}

void gemm_tn(const double* X, int64_t ldx, const double* Y, int64_t ldy, const double* L,
             int64_t q, int s, int w, double* C, int64_t ldc, double* part, cudaStream_t st) {
  if (s <= 0 || w <= 0) return;
  if (w > 32) {
    for (int c0 = 0; c0 < w; c0 += 32) {
      if (L) throw Error{TSVD_EINVAL, "gemm_tn: trsm needs w <= 32"};
      gemm_tn(X, ldx, Y + c0, ldy, nullptr, q, s, std::min(32, w - c0), C + c0, ldc, part, st);
    }
    return;
  }
  if (q <= 0) {  // empty reduction
    for (int i = 0; i < s; ++i) TSVD_CUDA(cudaMemsetAsync(C + (int64_t)i * ldc, 0, w * sizeof(double), st));
    return;
  }
  const TnGeom g = tn_geom(q, s);
  dim3 grid(g.s_tiles, g.splits);
  if (w <= 8)
    gemm_tn_kernel<8><<<grid, 256, 0, st>>>(X, ldx, Y, ldy, L, q, s, w, C, ldc, part);
  else if (w <= 16)
    gemm_tn_kernel<16><<<grid, 256, 0, st>>>(X, ldx, Y, ldy, L, q, s, w, C, ldc, part);
  else
    gemm_tn_kernel<32><<<grid, 256, 0, st>>>(X, ldx, Y, ldy, L, q, s, w, C, ldc, part);
  TSVD_CHECK_LAUNCH();
  if (g.splits > 1) {
    if (ldc == w) {
      reduce_partials(part, g.splits, (int64_t)s * w, C, st);
    } else {
      double* tmp = part + (int64_t)g.splits * s * w;
      reduce_partials(part, g.splits, (int64_t)s * w, tmp, st);
      scatter_ld_kernel<<<148, 256, 0, st>>>(tmp, s, w, C, ldc);
      TSVD_CHECK_LAUNCH();
    }
  }
}

// ------------------------------------------------------------------ NN ---
constexpr int NN_RB = 64;  // rows per tile
constexpr int NN_KC = 32;  // K chunk

int nn_ctas(int64_t q) {
  int64_t tiles = (q + NN_RB - 1) / NN_RB;
  const int64_t cap = 148 * 4;
  if (tiles > cap) tiles = cap;
  if (tiles < 1) tiles = 1;
  return (int)tiles;
}

template <int WP>
struct NnSmem {
  static constexpr int XP = NN_KC + 4, HP = WP + 4, YP = WP + 4;
  static constexpr size_t bytes =
      sizeof(double) * (NN_RB * XP + NN_KC * HP + NN_RB * YP + WP * WP);
};

template <int WP>
__global__ void __launch_bounds__(256) gemm_nn_kernel(
    const double* __restrict__ X, int64_t ldx, const double* __restrict__ H, int64_t ldh,
    const double* __restrict__ Y, int64_t ldy, const double* __restrict__ L,
    double* __restrict__ Z, int64_t ldz, int64_t q, int s, int w, double alpha, double beta,
    double* __restrict__ gram) {
  using SM = NnSmem<WP>;
  constexpr int XP = SM::XP, HP = SM::HP, YP = SM::YP, NT = WP / 8;
  constexpr int NPAIR = NT * NT;
  constexpr int PPW = (NPAIR + 7) / 8;  // gram tile pairs per warp
  extern __shared__ double smem[];
  double* Xs = smem;
  double* Hs = Xs + NN_RB * XP;
  double* Ys = Hs + NN_KC * HP;
  double* Ls = Ys + NN_RB * YP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  if (L) {
    for (int i = tid; i < WP * WP; i += 256) {
      const int r = i / WP, c = i % WP;
      Ls[i] = (r < w && c < w) ? L[r * w + c] : 0.0;
    }
  }
  double g[PPW][2];
#pragma unroll
  for (int p = 0; p < PPW; ++p) g[p][0] = g[p][1] = 0.0;
  const int64_t ntiles = (q + NN_RB - 1) / NN_RB;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t r0 = t * NN_RB;
    __syncthreads();
    // Y tile (+ trsm)
#pragma unroll
    for (int u = 0; u < (NN_RB * WP) / 256; ++u) {
      const int idx = tid + 256 * u;
      const int r = idx / WP, c = idx % WP;
      const int64_t row = r0 + r;
      Ys[r * YP + c] = (beta != 0.0 && row < q && c < w) ? Y[row * ldy + c] : 0.0;
    }
    if (L && beta != 0.0) {
      __syncthreads();
      if (tid < NN_RB) {
        double y[WP];
#pragma unroll
        for (int c = 0; c < WP; ++c) y[c] = Ys[tid * YP + c];
        row_trsm<WP>(y, Ls, w);
#pragma unroll
        for (int c = 0; c < WP; ++c) Ys[tid * YP + c] = y[c];
      }
    }
    double acc[NT][2];
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) acc[ni][0] = acc[ni][1] = 0.0;
    for (int k0 = 0; k0 < s; k0 += NN_KC) {
      __syncthreads();
#pragma unroll
      for (int u = 0; u < (NN_RB * NN_KC) / 256; ++u) {
        const int idx = tid + 256 * u;
        const int r = idx / NN_KC, c = idx % NN_KC;
        const int64_t row = r0 + r;
        Xs[r * XP + c] = (row < q && k0 + c < s) ? __ldg(X + row * ldx + k0 + c) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < (NN_KC * WP) / 256; ++u) {
        const int idx = tid + 256 * u;
        const int r = idx / WP, c = idx % WP;
        Hs[r * HP + c] = (k0 + r < s && c < w) ? __ldg(H + (int64_t)(k0 + r) * ldh + c) : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < NN_KC / 4; ++kk) {
        const double a = Xs[(warp * 8 + gid) * XP + kk * 4 + tig];
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) {
          const double b = Hs[(kk * 4 + tig) * HP + ni * 8 + gid];
          dmma884(acc[ni][0], acc[ni][1], a, b);
        }
      }
    }
    __syncthreads();
    // epilogue: Z tile = beta*Y' + alpha*acc  (into Ys)
#pragma unroll
    for (int ni = 0; ni < NT; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = warp * 8 + gid, c = ni * 8 + 2 * tig + e;
        const double z = beta * Ys[r * YP + c] + alpha * acc[ni][e];
        Ys[r * YP + c] = (c < w && r0 + r < q) ? z : 0.0;
      }
    __syncthreads();
    if (Z) {
#pragma unroll
      for (int u = 0; u < (NN_RB * WP) / 256; ++u) {
        const int idx = tid + 256 * u;
        const int r = idx / WP, c = idx % WP;
        const int64_t row = r0 + r;
        if (row < q && c < w) Z[row * ldz + c] = Ys[r * YP + c];
      }
    }
    if (gram) {
#pragma unroll
      for (int p = 0; p < PPW; ++p) {
        const int pair = warp + 8 * p;
        if (pair < NPAIR) {
          const int mi = pair / NT, ni = pair % NT;
#pragma unroll
          for (int kk = 0; kk < NN_RB / 4; ++kk) {
            const double a = Ys[(kk * 4 + tig) * YP + mi * 8 + gid];  // (Z^T)[i][k] = Z[k][i]
            const double b = Ys[(kk * 4 + tig) * YP + ni * 8 + gid];
            dmma884(g[p][0], g[p][1], a, b);
          }
        }
      }
    }
  }
  if (gram) {
#pragma unroll
    for (int p = 0; p < PPW; ++p) {
      const int pair = warp + 8 * p;
      if (pair < NPAIR) {
        const int mi = pair / NT, ni = pair % NT;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = mi * 8 + gid, j = ni * 8 + 2 * tig + e;
          if (i < w && j < w) gram[(int64_t)blockIdx.x * w * w + i * w + j] = g[p][e];
        }
      }
    }
  }
}

template <int WP>
static void nn_launch(const double* X, int64_t ldx, const double* H, int64_t ldh,
                      const double* Y, int64_t ldy, const double* L, double* Z, int64_t ldz,
                      int64_t q, int s, int w, double alpha, double beta, double* gram,
                      cudaStream_t st) {
  static bool attr_set = false;
  const size_t bytes = NnSmem<WP>::bytes;
  if (!attr_set) {
    TSVD_CUDA(cudaFuncSetAttribute(gemm_nn_kernel<WP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)bytes));
    attr_set = true;
  }
  gemm_nn_kernel<WP><<<nn_ctas(q), 256, bytes, st>>>(X, ldx, H, ldh, Y, ldy, L, Z, ldz, q, s,
                                                      w, alpha, beta, gram);
  TSVD_CHECK_LAUNCH();
}

void gemm_nn(const double* X, int64_t ldx, const double* H, int64_t ldh, const double* Y,
             int64_t ldy, const double* L, double* Z, int64_t ldz, int64_t q, int s, int w,
             double alpha, double beta, double* gram, cudaStream_t st) {
  if (w <= 0 || q <= 0) return;
  if (w > 32) {
    if (L || gram) throw Error{TSVD_EINVAL, "gemm_nn: trsm/gram need w <= 32"};
    for (int c0 = 0; c0 < w; c0 += 32)
      gemm_nn(X, ldx, H + c0, ldh, Y ? Y + c0 : nullptr, ldy, nullptr, Z + c0, ldz, q, s,
              std::min(32, w - c0), alpha, beta, nullptr, st);
    return;
  }
  if (w <= 8)
    nn_launch<8>(X, ldx, H, ldh, Y, ldy, L, Z, ldz, q, s, w, alpha, beta, gram, st);
  else if (w <= 16)
    nn_launch<16>(X, ldx, H, ldh, Y, ldy, L, Z, ldz, q, s, w, alpha, beta, gram, st);
  else
    nn_launch<32>(X, ldx, H, ldh, Y, ldy, L, Z, ldz, q, s, w, alpha, beta, gram, st);
}

// ----------------------------------------------------------- finalisers ---
// One warp Cholesky of W (w x w, w <= 32) held in shared memory, row-major.
// Breakdown: a pivot <= 0 or non-finite -> *bad = 1; the pivot is
// then replaced by 1 so the (discarded) result stays finite.
__device__ void warp_cholesky(double* Ws, double* Lo, int w, int* bad) {
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < w; ++j) {
    double d = 0.0;
    if (lane == 0) {
      d = Ws[j * w + j];
      for (int k = 0; k < j; ++k) d = fma(-Lo[j * 32 + k], Lo[j * 32 + k], d);
      if (!(d > 0.0) || !isfinite(d)) {
        *bad = 1;
        d = 1.0;
      }
      Lo[j * 32 + j] = sqrt(d);
    }
    __syncwarp();
    const double ljj = Lo[j * 32 + j];
    for (int i = j + 1 + lane; i < w; i += 32) {
      double v = Ws[i * w + j];
      for (int k = 0; k < j; ++k) v = fma(-Lo[i * 32 + k], Lo[j * 32 + k], v);
      Lo[i * 32 + j] = v / ljj;
    }
    __syncwarp();
  }
}

__global__ void chol_finalize_kernel(const double* __restrict__ gram, int nparts, int w,
                                     double* __restrict__ L, int* __restrict__ flag) {
  __shared__ double Ws[32 * 32];
  __shared__ double Lo[32 * 32];
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int i = tid; i < w * w; i += blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < nparts; ++p) s += gram[(int64_t)p * w * w + i];
    Ws[i] = s;
  }
  for (int i = tid; i < 32 * 32; i += blockDim.x) Lo[i] = 0.0;
  __syncthreads();
  if (tid < 32) warp_cholesky(Ws, Lo, w, &bad);
  __syncthreads();
  for (int i = tid; i < w * w; i += blockDim.x) L[i] = Lo[(i / w) * 32 + (i % w)];
  if (tid == 0 && bad) *flag = 1;
}

void chol_finalize(const double* gram, int nparts, int w, double* L, int* flag,
                   cudaStream_t st) {
  chol_finalize_kernel<<<1, 256, 0, st>>>(gram, nparts, w, L, flag);
  TSVD_CHECK_LAUNCH();
}

// Second pass: Lbar = chol(Wbar); R = Lbar^T Lprev^T (Alg. 4 S7 / Alg. 5 S11,
// reading R4); H (s x w) += Hbar Lprev^T (Alg. 5 S12, reading R5).
__global__ void chol2_finalize_kernel(const double* __restrict__ gram, int nparts, int w,
                                      const double* __restrict__ Lprev, double* __restrict__ L2,
                                      double* __restrict__ R, double* __restrict__ H,
                                      const double* __restrict__ Hbar, int s,
                                      int* __restrict__ flag) {
  __shared__ double Ws[32 * 32];
  __shared__ double Lo[32 * 32];
  __shared__ double Lp[32 * 32];
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int i = tid; i < w * w; i += blockDim.x) {
    double sum = 0.0;
    for (int p = 0; p < nparts; ++p) sum += gram[(int64_t)p * w * w + i];
    Ws[i] = sum;
    Lp[i] = Lprev[i];
  }
  for (int i = tid; i < 32 * 32; i += blockDim.x) Lo[i] = 0.0;
  __syncthreads();
  if (tid < 32) warp_cholesky(Ws, Lo, w, &bad);
  __syncthreads();
  for (int i = tid; i < w * w; i += blockDim.x) {
    const int r = i / w, c = i % w;
    L2[i] = Lo[r * 32 + c];
    // R[r][c] = sum_k Lbar[k][r] * Lprev[c][k]
    double sum = 0.0;
    for (int k = 0; k < w; ++k) sum = fma(Lo[k * 32 + r], Lp[c * w + k], sum);
    R[i] = sum;
  }
  if (H) {
    for (int64_t i = tid; i < (int64_t)s * w; i += blockDim.x) {
      const int64_t r = i / w;
      const int c = (int)(i % w);
      double sum = 0.0;
      for (int k = 0; k < w; ++k) sum = fma(Hbar[r * w + k], Lp[c * w + k], sum);
      H[i] += sum;
    }
  }
  if (tid == 0 && bad) *flag = 1;
}

void chol2_finalize(const double* gram, int nparts, int w, const double* Lprev, double* L2,
                    double* R, double* H, const double* Hbar, int s, int* flag,
                    cudaStream_t st) {
  chol2_finalize_kernel<<<1, 256, 0, st>>>(gram, nparts, w, Lprev, L2, R, H, Hbar, s, flag);
  TSVD_CHECK_LAUNCH();
}

// --------------------------------------------------------------- helpers ---
__global__ void copy_block_kernel(const double* __restrict__ src, int64_t lds,
                                  double* __restrict__ dst, int64_t ldd, int64_t rows, int cols,
                                  int transpose) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols;
    const int c = (int)(i % cols);
    dst[r * ldd + c] = transpose ? src[(int64_t)c * lds + r] : src[r * lds + c];
  }
}

void copy_block(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
                int cols, bool transpose, cudaStream_t st) {
  const int64_t n = rows * cols;
  if (n <= 0) return;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  copy_block_kernel<<<(unsigned)blocks, 256, 0, st>>>(src, lds, dst, ldd, rows, cols,
                                                       transpose ? 1 : 0);
  TSVD_CHECK_LAUNCH();
}

void fill_zero(double* p, int64_t n, cudaStream_t st) {
  if (n > 0) TSVD_CUDA(cudaMemsetAsync(p, 0, n * sizeof(double), st));
}

// CGS2 per-column decision (P:275 fallback, reading R16):
// coef = c1 + c2 ; nrm = ||y''|| ; dependent = nrm <= tau ||y_orig||
__global__ void cgs2_col_finalize_kernel(const double* c1, const double* c2, int nb,
                                         const double* gram_y, const double* gram_orig,
                                         double tau, double* coef, double* nrm, int* dep) {
  for (int i = threadIdx.x; i < nb; i += blockDim.x) coef[i] = c1[i] + c2[i];
  if (threadIdx.x == 0) {
    const double ny = sqrt(gram_y[0]);
    const double no = sqrt(gram_orig[0]);
    nrm[0] = ny;
    dep[0] = (ny <= tau * no) ? 1 : 0;
  }
}

void cgs2_col_finalize(const double* c1, const double* c2, int nb, const double* gram_y,
                       const double* gram_orig, double tau, double* coef_out, double* nrm_out,
                       int* dependent, cudaStream_t st) {
  cgs2_col_finalize_kernel<<<1, 256, 0, st>>>(c1, c2, nb, gram_y, gram_orig, tau, coef_out,
                                              nrm_out, dependent);
  TSVD_CHECK_LAUNCH();
}

__global__ void scale_column_kernel(double* col, int64_t q, int64_t ld, const double* nrm) {
  const double inv = 1.0 / nrm[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < q;
       i += (int64_t)gridDim.x * blockDim.x)
    col[i * ld] = col[i * ld] * inv;
}

void scale_column(double* col, int64_t q, int64_t ld, const double* nrm, cudaStream_t st) {
  scale_column_kernel<<<148 * 4, 256, 0, st>>>(col, q, ld, nrm);
  TSVD_CHECK_LAUNCH();
}

// rho_i = ||Rbar Vb[(k-1)b : kb, i]||_2 / S[0]  (from Eq. 10; reading R12)
__global__ void lanczos_rho_kernel(const double* __restrict__ Rbar, int b,
                                   const double* __restrict__ Vb, int d,
                                   const double* __restrict__ S, int cnt,
                                   double* __restrict__ rho) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  double ss = 0.0;
  for (int j = 0; j < b; ++j) {
    double t = 0.0;
    for (int l = 0; l < b; ++l) t = fma(Rbar[j * b + l], Vb[(int64_t)(d - b + l) * d + i], t);
    ss = fma(t, t, ss);
  }
  rho[i] = sqrt(ss) / S[0];
}

void lanczos_rho(const double* Rbar, int b, const double* Vb, int d, const double* S, int cnt,
                 double* rho, cudaStream_t st) {
  lanczos_rho_kernel<<<(cnt + 127) / 128, 128, 0, st>>>(Rbar, b, Vb, d, S, cnt, rho);
  TSVD_CHECK_LAUNCH();
}

// sign normalisation (reading R28): per column i of V, the largest-|.| entry
// (lowest index on ties) is made positive; U's column flips with it.
__global__ void colmax_kernel(const double* __restrict__ V, int64_t n, int64_t ldv,
                              double* __restrict__ sgn) {
  __shared__ double bv[256];
  __shared__ int64_t bi[256];
  const int i = blockIdx.x;
  double best = -1.0;
  int64_t bidx = 0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const double a = fabs(V[j * ldv + i]);
    if (a > best) {  // strictly greater keeps the lowest index of this thread
      best = a;
      bidx = j;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = bidx;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      const double o = bv[threadIdx.x + off];
      const int64_t oi = bi[threadIdx.x + off];
      if (o > bv[threadIdx.x] || (o == bv[threadIdx.x] && oi < bi[threadIdx.x])) {
        bv[threadIdx.x] = o;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) sgn[i] = (V[bi[0] * ldv + i] < 0.0) ? -1.0 : 1.0;
}

__global__ void flip_kernel(double* __restrict__ M, int64_t rows, int64_t ld, int r,
                            const double* __restrict__ sgn) {
  const int64_t n = rows * r;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / r;
    const int i = (int)(t % r);
    if (sgn[i] < 0.0) M[j * ld + i] = -M[j * ld + i];
  }
}

void sign_normalize(double* U, int64_t m, int64_t ldu, double* V, int64_t n, int64_t ldv,
                    int r, double* work, cudaStream_t st) {
  if (r <= 0) return;
  colmax_kernel<<<r, 256, 0, st>>>(V, n, ldv, work);
  flip_kernel<<<148 * 4, 256, 0, st>>>(U, m, ldu, r, work);
  flip_kernel<<<148 * 4, 256, 0, st>>>(V, n, ldv, r, work);
  TSVD_CHECK_LAUNCH();
}

}  // namespace tsvd
