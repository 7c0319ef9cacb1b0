// Small single-CTA finalisers and helpers of the orthogonalisation passes:
// fixed-order partial sums, b x b Cholesky with the breakdown test of P:275,
// T = L^{-T} for the TRSM-as-multiply passes, R = Lbar^T L^T (reading R4),
// H += Hbar L^T (reading R5), block copies, CGS2 column bookkeeping, the
// Lanczos rho test and sign normalisation.
#include "internal.h"

namespace tsvd {

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

// T = L^{-T} (upper triangular) from the lower triangular L held in Lo (ld 32):
// lane j computes column j of L^{-1} by forward substitution into the shared
// scratch Xs (ld 33); T[j][i] = Linv[i][j].
__device__ void warp_tri_inverse_t(const double* Lo, double* Xs, double* Tout, int w) {
  const int j = threadIdx.x & 31;
  if (j < w) {
    for (int i = 0; i < w; ++i) {
      double v = 0.0;
      if (i >= j) {
        v = (i == j) ? 1.0 : 0.0;
        for (int k = j; k < i; ++k) v = fma(-Lo[i * 32 + k], Xs[k * 33 + j], v);
        v = v / Lo[i * 32 + i];
      }
      Xs[i * 33 + j] = v;
    }
  }
  __syncwarp();
  if (j < w)
    for (int i = 0; i < w; ++i) Tout[j * w + i] = Xs[i * 33 + j];  // T[j][i] = Linv[i][j]
}

__global__ void chol_finalize_kernel(const double* __restrict__ gram, int nparts, int w,
                                     double* __restrict__ L, double* __restrict__ T,
                                     int* __restrict__ flag) {
  __shared__ double Ws[32 * 33];
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
  if (tid < 32) warp_tri_inverse_t(Lo, Ws, T, w);
  if (tid == 0 && bad) *flag = 1;
}

void chol_from_w(const double* W, int w, double* L, double* T, int* flag, cudaStream_t st) {
  chol_finalize_kernel<<<1, 256, 0, st>>>(W, 1, w, L, T, flag);
  TSVD_CHECK_LAUNCH();
}

void chol_finalize(const double* gram, int nparts, int w, double* Wred, double* L, double* T,
                   int* flag, cudaStream_t st) {
  reduce_partials(gram, nparts, (int64_t)w * w, Wred, st);
  chol_finalize_kernel<<<1, 256, 0, st>>>(Wred, 1, w, L, T, flag);
  TSVD_CHECK_LAUNCH();
}

// Second pass: Lbar = chol(Wbar), Tbar = Lbar^{-T}; R = Lbar^T Lprev^T (Alg. 4 S7 /
// Alg. 5 S11, reading R4); H (s x w) += Hbar Lprev^T (Alg. 5 S12, reading R5).
__global__ void chol2_finalize_kernel(const double* __restrict__ gram, int nparts, int w,
                                      const double* __restrict__ Lprev, double* __restrict__ L2,
                                      double* __restrict__ T2, double* __restrict__ R,
                                      double* __restrict__ H, const double* __restrict__ Hbar,
                                      int s, int* __restrict__ flag) {
  __shared__ double Ws[32 * 33];
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
  if (tid < 32) warp_tri_inverse_t(Lo, Ws, T2, w);
  for (int i = tid; i < w * w; i += blockDim.x) {
    const int r = i / w, c = i % w;
    L2[i] = Lo[r * 32 + c];
    // R[r][c] = sum_k Lbar[k][r] * Lprev[c][k]
    double sum = 0.0;
    for (int k = 0; k < w; ++k) sum = fma(Lo[k * 32 + r], Lp[c * w + k], sum);
    R[i] = sum;
  }
  if (H) {
    // one H row per thread: its w Hbar entries are loaded together
    for (int r = tid; r < s; r += blockDim.x) {
      double hb[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) hb[k] = k < w ? Hbar[(int64_t)r * w + k] : 0.0;
      for (int c = 0; c < w; ++c) {
        double sum = 0.0;
#pragma unroll
        for (int k = 0; k < 32; ++k)
          if (k < w) sum = fma(hb[k], Lp[c * w + k], sum);
        H[(int64_t)r * w + c] += sum;
      }
    }
  }
  if (tid == 0 && bad) *flag = 1;
}

void chol2_from_w(const double* W, int w, const double* Lprev, double* L2, double* T2,
                  double* R, double* H, const double* Hbar, int s, int* flag, cudaStream_t st) {
  chol2_finalize_kernel<<<1, 256, 0, st>>>(W, 1, w, Lprev, L2, T2, R, H, Hbar, s, flag);
  TSVD_CHECK_LAUNCH();
}

void chol2_finalize(const double* gram, int nparts, int w, double* Wred, const double* Lprev,
                    double* L2, double* T2, double* R, double* H, const double* Hbar, int s,
                    int* flag, cudaStream_t st) {
  reduce_partials(gram, nparts, (int64_t)w * w, Wred, st);
  chol2_finalize_kernel<<<1, 256, 0, st>>>(Wred, 1, w, Lprev, L2, T2, R, H, Hbar, s, flag);
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
// (lowest index on ties) is made positive; the column of U flips with it.
// Pass 1: CTAs own row ranges, lanes own 32 consecutive columns (coalesced
// row reads), per-CTA (max, argmin-index) partials; pass 2: fixed-order scan
// of the partials per column -> sign.
constexpr int kSignCtas = 296;

__global__ void colmax_partial_kernel(const double* __restrict__ V, int64_t n, int64_t ldv,
                                      int r, double* __restrict__ pval,
                                      int64_t* __restrict__ pidx) {
  __shared__ double bv[8][32];
  __shared__ int64_t bi[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.y * 32 + lane;
  double best = -1.0;
  int64_t bidx = 0;
  if (c < r) {
    for (int64_t j = (int64_t)blockIdx.x * 8 + warp; j < n; j += (int64_t)gridDim.x * 8) {
      const double a = fabs(V[j * ldv + c]);
      if (a > best) {  // rows visited in increasing order: keeps the lowest index
        best = a;
        bidx = j;
      }
    }
  }
  bv[warp][lane] = best;
  bi[warp][lane] = bidx;
  __syncthreads();
  if (warp == 0 && c < r) {
    for (int k = 1; k < 8; ++k) {
      const double o = bv[k][lane];
      const int64_t oi = bi[k][lane];
      if (o > best || (o == best && oi < bidx)) {
        best = o;
        bidx = oi;
      }
    }
    pval[(int64_t)blockIdx.x * r + c] = best;
    pidx[(int64_t)blockIdx.x * r + c] = bidx;
  }
}

// per column: best (|v|, global row index, signed v) over the CTA partials
__global__ void colsign_local_kernel(const double* __restrict__ V, int64_t ldv, int r,
                                     const double* __restrict__ pval,
                                     const int64_t* __restrict__ pidx, int nparts, int64_t row0,
                                     double* __restrict__ loc) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= r) return;
  double best = -1.0;
  int64_t bidx = 0;
  for (int p = 0; p < nparts; ++p) {
    const double o = pval[(int64_t)p * r + c];
    const int64_t oi = pidx[(int64_t)p * r + c];
    if (o > best || (o == best && oi < bidx)) {
      best = o;
      bidx = oi;
    }
  }
  loc[3 * c] = best;
  loc[3 * c + 1] = (double)(bidx + row0);  // exact below 2^53
  loc[3 * c + 2] = best >= 0.0 ? V[bidx * ldv + c] : 1.0;
}

// winner over ranks (rank order; ties -> lower global index) -> sign
__global__ void colsign_final_kernel(const double* __restrict__ all, int world, int r,
                                     double* __restrict__ sgn) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= r) return;
  double best = -1.0, bidx = 0.0, bval = 1.0;
  for (int g = 0; g < world; ++g) {
    const double* e = all + ((size_t)g * r + c) * 3;
    if (e[0] > best || (e[0] == best && e[1] < bidx)) {
      best = e[0];
      bidx = e[1];
      bval = e[2];
    }
  }
  sgn[c] = bval < 0.0 ? -1.0 : 1.0;
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

size_t col_signs_work(int r, int world) {
  return (size_t)kSignCtas * r * 2 + (size_t)3 * r * (world + 1) + 8;
}

// Local pass: loc (3r doubles inside work) = per-column (|v|, global index,
// v) of this rank's rows.  Returns the pointer to loc (for the all-gather).
double* col_signs_local(const double* V, int64_t n, int64_t ldv, int r, int64_t row0,
                        double* work, cudaStream_t st) {
  double* pval = work;
  int64_t* pidx = (int64_t*)(work + (size_t)kSignCtas * r);
  double* loc = work + (size_t)kSignCtas * r * 2;
  dim3 grid(kSignCtas, (r + 31) / 32);
  colmax_partial_kernel<<<grid, 256, 0, st>>>(V, n, ldv, r, pval, pidx);
  TSVD_CHECK_LAUNCH();
  colsign_local_kernel<<<(r + 127) / 128, 128, 0, st>>>(V, ldv, r, pval, pidx, kSignCtas, row0,
                                                        loc);
  TSVD_CHECK_LAUNCH();
  return loc;
}

void col_signs_final(const double* all, int world, int r, double* sgn, cudaStream_t st) {
  colsign_final_kernel<<<(r + 127) / 128, 128, 0, st>>>(all, world, r, sgn);
  TSVD_CHECK_LAUNCH();
}

void flip_columns(double* M, int64_t rows, int64_t ld, int r, const double* sgn,
                  cudaStream_t st) {
  if (r <= 0 || rows <= 0) return;
  int64_t blocks = (rows * r + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  flip_kernel<<<(unsigned)blocks, 256, 0, st>>>(M, rows, ld, r, sgn);
  TSVD_CHECK_LAUNCH();
}

}  // namespace tsvd
