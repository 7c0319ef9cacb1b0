// Small single-CTA finalisers and helpers of the orthogonalisation passes:
// fixed-order partial sums, b x b Cholesky with the breakdown test of P:275,
// T = L^{-T} for the TRSM-as-multiply passes, R = Lbar^T L^T (reading R4),
// H += Hbar L^T (reading R5), block copies, CGS2 column bookkeeping, the
// Lanczos rho test and sign normalisation.
#include "internal.h"
#include "ptx.cuh"

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

// Fused Gram finaliser, one CTA of FIN_T threads:
//   1. W = sum of the np per-CTA Gram partials in a fixed order (thread t sums
//      partials g, g+G, g+2G, ... of entry e = t mod w^2, g = t div w^2,
//      G = FIN_T div w^2; the G group sums are added in g order).  np = 1
//      passes an already reduced W through bit for bit; for w >= 23 the
//      launcher first reduces the partials with gram_prereduce_kernel (one
//      CTA per 32 entries) and calls this kernel with np = 1.
//   2. mode >= 1: L = chol(W) with the breakdown test of P:275 and
//      T = L^{-T}; w <= 16 in registers (row i of W in lane i, right-looking
//      updates by shuffles; the column scaling multiplies by 1/l_jj =
//      rsqrt(pivot) as LAPACK's potf2 scales by a reciprocal, and the same
//      reciprocals serve the triangular inverse - no f64 divisions, which are
//      long dependent sequences on the GPU), else the shared-memory routines.
//   3. mode 2: R = Lbar^T Lprev^T (R4), H += Hbar Lprev^T (R5); Hbar is
//      staged into shared memory by all threads while step 2 runs.
// mode 0 only writes W (the multi-GPU path all-reduces it, then calls mode
// 1/2 with np = 1), so one and several ranks see identical arithmetic.
constexpr int FIN_T = 512;
constexpr int FIN_HB = 8192;  // doubles of Hbar staged per chunk (64 KB dynamic smem)

// 32 x 32 register Cholesky needs > 128 registers/thread: 256 threads then
constexpr int fin_threads(int wt) { return wt == 32 ? 256 : FIN_T; }

template <int WT>  // WT > 0: w == WT (all loops unrolled, no divergence); 0: any w <= 32
__global__ void __launch_bounds__(fin_threads(WT)) finalize_kernel(
    const double* __restrict__ gram, int np, int w_, int mode, double* __restrict__ Wout,
    const double* __restrict__ Lprev, double* __restrict__ L, double* __restrict__ T,
    double* __restrict__ R, double* __restrict__ H, const double* __restrict__ Hbar, int s,
    int* __restrict__ flag) {
  pdl_enter();
  constexpr int NTH = fin_threads(WT);
  __shared__ double red[NTH];
  __shared__ double Ws[32 * 33];
  __shared__ double Lo[32 * 32];
  __shared__ double Lp[32 * 32];
  __shared__ double Xs[32 * 33];
  __shared__ double rsd[32];
  __shared__ int bad;
  extern __shared__ double hbs[];
  const int w = WT > 0 ? WT : w_;
  const int tid = threadIdx.x, C = w * w, G = NTH / C;
  const int64_t nh = (mode == 2 && H) ? (int64_t)s * w : 0;
  if (tid == 0) bad = 0;
  if (tid < G * C) {
    const int e = tid % C, g = tid / C;
    double a = 0.0;
#pragma unroll 16
    for (int p = g; p < np; p += G) a += gram[(int64_t)p * C + e];
    red[tid] = a;
  }
  if (mode == 2)
    for (int i = tid; i < C; i += NTH) Lp[i] = Lprev[i];
  for (int i = tid; i < 32 * 32; i += NTH) Lo[i] = 0.0;
  // first Hbar chunk in flight during the Cholesky
  {
    const int n0 = (int)(nh < FIN_HB ? nh : FIN_HB);
    for (int i = tid; i < n0; i += NTH) hbs[i] = Hbar[i];
  }
  __syncthreads();
  if (G >= 1) {
    if (tid < C) {
      double a = red[tid];
      for (int g = 1; g < G; ++g) a += red[g * C + tid];
      Ws[tid] = a;
      if (mode == 0) Wout[tid] = a;
    }
  } else {
    // w^2 > NTH (w >= 23): each thread sums whole entries, partials in order;
    // its EPT entries advance side by side so their loads overlap (the order
    // of the additions of each entry is unchanged: p = 0, 1, ..., np - 1)
    constexpr int EPT = (32 * 32 + NTH - 1) / NTH;
    double a[EPT];
#pragma unroll
    for (int j = 0; j < EPT; ++j) a[j] = 0.0;
#pragma unroll 8
    for (int p = 0; p < np; ++p)
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        const int e = tid + j * NTH;
        if (e < C) a[j] += gram[(int64_t)p * C + e];
      }
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int e = tid + j * NTH;
      if (e < C) {
        Ws[e] = a[j];
        if (mode == 0) Wout[e] = a[j];
      }
    }
  }
  __syncthreads();
  if (mode == 0) return;
  if constexpr (WT > 0 && WT <= 16) {
    if (tid < 32) {
      const int lane = tid;
      double a[WT];
#pragma unroll
      for (int k = 0; k < WT; ++k) a[k] = (lane < WT && k <= lane) ? Ws[lane * WT + k] : 0.0;
      int bd = 0;
#pragma unroll
      for (int j = 0; j < WT; ++j) {
        double piv = __shfl_sync(~0u, a[j], j);
        if (!(piv > 0.0) || !isfinite(piv)) {
          bd = 1;
          piv = 1.0;
        }
        const double rj = rsqrt(piv);
        if (lane == 0) rsd[j] = rj;
        const double lij = lane > j ? a[j] * rj : (lane == j ? piv * rj : 0.0);
        a[j] = lij;
#pragma unroll
        for (int k = j + 1; k < WT; ++k) {
          const double lkj = __shfl_sync(~0u, lij, k);
          a[k] = (lane >= k) ? fma(-lij, lkj, a[k]) : a[k];
        }
      }
      if (lane == 0 && bd) bad = 1;
      if (lane < WT)
#pragma unroll
        for (int k = 0; k < WT; ++k) Lo[lane * 32 + k] = a[k];
      __syncwarp();
      // column `lane` of L^{-1} by forward substitution (x[m] kept in Xs);
      // 1/l_ii = rsd[i] from the factorisation
#pragma unroll
      for (int i = 0; i < WT; ++i) {
        double v = (i == lane) ? 1.0 : 0.0;
#pragma unroll
        for (int m = 0; m < i; ++m) v = fma(-__shfl_sync(~0u, a[m], i), Xs[m * 33 + lane], v);
        Xs[i * 33 + lane] = (i >= lane) ? v * rsd[i] : 0.0;
      }
    }
  } else if constexpr (WT == 32) {
    // Right-looking Cholesky + forward-substitution inverse in ROLLED loops
    // over shared memory (lane i owns row i; Lo = W's lower triangle, updated
    // in place).  The arithmetic and its order are those of the register
    // version above, but that version's ~19 000 straight-line instructions
    // for w = 32 ran from a cold instruction cache after every big pass
    // (58 us per call in ncu, 39 us rolled); for w <= 16 (5 900
    // instructions) the register version stays faster.
    if (tid < 32) {
      const int lane = tid;
      for (int k = 0; k < WT; ++k)
        Lo[lane * 32 + k] = (lane < WT && k <= lane) ? Ws[lane * WT + k] : 0.0;
      __syncwarp();
      int bd = 0;
#pragma unroll 1
      for (int j = 0; j < WT; ++j) {
        double piv = Lo[j * 32 + j];
        if (!(piv > 0.0) || !isfinite(piv)) {
          bd = 1;
          piv = 1.0;
        }
        const double rj = rsqrt(piv);
        if (lane == 0) rsd[j] = rj;
        const double aj = Lo[lane * 32 + j];
        const double lij = lane > j ? aj * rj : (lane == j ? piv * rj : 0.0);
        __syncwarp();
        if (lane < WT) Lo[lane * 32 + j] = lij;
        __syncwarp();
#pragma unroll 4
        for (int k = j + 1; k < WT; ++k) {
          const double lkj = Lo[k * 32 + j];
          if (lane >= k && lane < WT) Lo[lane * 32 + k] = fma(-lij, lkj, Lo[lane * 32 + k]);
        }
        __syncwarp();
      }
      if (lane == 0 && bd) bad = 1;
      // column `lane` of L^{-1} by forward substitution (x[m] kept in Xs);
      // 1/l_ii = rsd[i] from the factorisation
#pragma unroll 1
      for (int i = 0; i < WT; ++i) {
        double v = (i == lane) ? 1.0 : 0.0;
#pragma unroll 4
        for (int m = 0; m < i; ++m) v = fma(-Lo[i * 32 + m], Xs[m * 33 + lane], v);
        Xs[i * 33 + lane] = (i >= lane) ? v * rsd[i] : 0.0;
      }
    }
  } else if (tid < 32) {
    warp_cholesky(Ws, Lo, w, &bad);
    warp_tri_inverse_t(Lo, Ws, T, w);  // Ws is free now; writes T
  }
  __syncthreads();
  for (int i = tid; i < C; i += NTH) {
    const int r = i / w, c = i % w;
    L[i] = Lo[r * 32 + c];
    if constexpr (WT > 0) T[i] = Xs[c * 33 + r];  // T[r][c] = Linv[c][r]
    if (mode == 2) {
      double sum = 0.0;  // R[r][c] = sum_k Lbar[k][r] Lprev[c][k]
      if constexpr (WT > 0) {
#pragma unroll
        for (int k = 0; k < WT; ++k) sum = fma(Lo[k * 32 + r], Lp[c * WT + k], sum);
      } else {
        for (int k = 0; k < w; ++k) sum = fma(Lo[k * 32 + r], Lp[c * w + k], sum);
      }
      R[i] = sum;
    }
  }
  // H[r][c] += sum_k Hbar[r][k] Lprev[c][k], Hbar staged in chunks of whole rows
  const int rows_per = FIN_HB / w;
  for (int r0 = 0; (int64_t)r0 * w < nh; r0 += rows_per) {
    const int cnt = (rows_per < s - r0 ? rows_per : s - r0) * w;
    if (r0 > 0) {
      __syncthreads();
      for (int i = tid; i < cnt; i += NTH) hbs[i] = Hbar[(int64_t)r0 * w + i];
      __syncthreads();
    }
    for (int i = tid; i < cnt; i += NTH) {
      const int r = i / w, c = i % w;
      const double* hb = hbs + r * w;
      double sum = 0.0;
      if constexpr (WT > 0) {
#pragma unroll
        for (int k = 0; k < WT; ++k) sum = fma(hb[k], Lp[c * WT + k], sum);
      } else {
        for (int k = 0; k < w; ++k) sum = fma(hb[k], Lp[c * w + k], sum);
      }
      H[(int64_t)r0 * w + i] += sum;
    }
  }
  if (tid == 0 && bad) *flag = 1;
}

// Gram partial reduction for w >= 23 (w^2 entries > the finaliser's threads):
// CTA b sums entries [32 b, 32 b + 32) over the np partials -- 8 groups of 32
// threads take partials g, g + 8, g + 16, ... (all their loads in flight), the
// group sums are added in g order (fixed order, deterministic) -- and writes
// the total over partial slot 0 (only this CTA reads or writes those
// entries).  The single-CTA finaliser then runs with np = 1.
__global__ void __launch_bounds__(256) gram_prereduce_kernel(double* __restrict__ gram, int np,
                                                             int C) {
  pdl_enter();
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  double a = 0.0;
  if (e < C) {
#pragma unroll 4
    for (int p = g; p < np; p += 8) a += gram[(int64_t)p * C + e];
  }
  red[g][lane] = a;
  __syncthreads();
  if (g == 0 && e < C) {
    double t = red[0][lane];
#pragma unroll
    for (int k = 1; k < 8; ++k) t += red[k][lane];
    gram[e] = t;
  }
}

static void fin_launch(const double* gram, int np, int w, int mode, double* Wout,
                       const double* Lprev, double* L, double* T, double* R, double* H,
                       const double* Hbar, int s, int* flag, cudaStream_t st) {
  if (np > 1 && w * w > fin_threads(w == 32 ? 32 : 0)) {
    launch_pdl(gram_prereduce_kernel, (w * w + 31) / 32, 256, 0, st, const_cast<double*>(gram), np,
                                                             w * w);
    TSVD_CHECK_LAUNCH();
    np = 1;
  }
  static bool attr = false;
  const int dyn = FIN_HB * 8;
  if (!attr) {
    TSVD_CUDA(cudaFuncSetAttribute(finalize_kernel<0>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    TSVD_CUDA(cudaFuncSetAttribute(finalize_kernel<4>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    TSVD_CUDA(cudaFuncSetAttribute(finalize_kernel<8>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    TSVD_CUDA(cudaFuncSetAttribute(finalize_kernel<16>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    TSVD_CUDA(cudaFuncSetAttribute(finalize_kernel<32>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    attr = true;
  }
#define FIN_GO(WTV)                                                                           \
  launch_pdl(finalize_kernel<WTV>, 1, fin_threads(WTV), dyn, st, gram, np, w, mode, Wout, Lprev, L, T, R, H, Hbar, \
                                              s, flag)
  if (w == 32) FIN_GO(32);
  else if (w == 16) FIN_GO(16);
  else if (w == 8) FIN_GO(8);
  else if (w == 4) FIN_GO(4);
  else FIN_GO(0);
#undef FIN_GO
  TSVD_CHECK_LAUNCH();
}

void gram_reduce(const double* gram, int np, int w, double* Wred, cudaStream_t st) {
  fin_launch(gram, np, w, 0, Wred, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0,
             nullptr, st);
}

void chol_finalize(const double* gram, int np, int w, double* L, double* T, int* flag,
                   cudaStream_t st) {
  fin_launch(gram, np, w, 1, nullptr, nullptr, L, T, nullptr, nullptr, nullptr, 0, flag, st);
}

void chol2_finalize(const double* gram, int np, int w, const double* Lprev, double* L2,
                    double* T2, double* R, double* H, const double* Hbar, int s, int* flag,
                    cudaStream_t st) {
  fin_launch(gram, np, w, 2, nullptr, Lprev, L2, T2, R, H, Hbar, s, flag, st);
}

// ----------------------------------------------------- BCGS-PIP+ pass ---
// One CTA (256 threads, 8 warps) does the small work of one Pythagorean
// pass (reading R34; blocks.cu pip2): from C = [H; W] ((s + w) x w, the
// reduced [P Y]^T Y)
//   M = W - H^T H        (8 x 8 tiles by DMMA m8n8k4 over k = s, warp-strided)
//   L = chol(M) (P:275 breakdown test -> *flag), T = L^{-T}
//   Hp = H T             (s x w; DMMA tiles, K = w)
// and, for the second pass (L1 != null): R = L^T L1^T (= R2 R1) and, when
// Hout != null, Hout = H1 + H L1^T.  Every sum runs in a fixed order.
__device__ __forceinline__ void dmma884s(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) pip_finalize_kernel(
    const double* __restrict__ Cm, int s, int w, double* __restrict__ L,
    double* __restrict__ T, double* __restrict__ Hp, int* __restrict__ flag,
    const double* __restrict__ L1, double* __restrict__ R, const double* __restrict__ H1,
    double* __restrict__ Hout) {
  __shared__ double Ms[32 * 32];
  __shared__ double Lo[32 * 32];
  __shared__ double Xs[32 * 33];
  __shared__ double Ts[32 * 33];
  __shared__ double L1s[32 * 33];
  __shared__ int bad;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int nt = (w + 7) / 8;
  const double* H = Cm;
  const double* W = Cm + (size_t)s * w;
  if (tid == 0) bad = 0;
  for (int i = tid; i < 32 * 32; i += 256) Lo[i] = 0.0;
  if (L1)
    for (int i = tid; i < w * w; i += 256) L1s[(i / w) * 33 + i % w] = L1[i];
  // M = W - H^T H: tile (ti, tj), D[gid][2 tig + e] += sum_k H[k][ti 8 + gid] H[k][tj 8 + 2 tig + e]
  for (int t = warp; t < nt * nt; t += 8) {
    const int ti = t / nt, tj = t % nt;
    const int ci = ti * 8 + gid, cj = tj * 8 + gid;
    double d0 = 0.0, d1 = 0.0;
    for (int k0 = 0; k0 < s; k0 += 4) {
      const int k = k0 + tig;
      const double a = (k < s && ci < w) ? H[(size_t)k * w + ci] : 0.0;
      const double b = (k < s && cj < w) ? H[(size_t)k * w + cj] : 0.0;
      dmma884s(d0, d1, a, b);
    }
    const int r = ti * 8 + gid, c = tj * 8 + 2 * tig;
    if (r < w && c < w) Ms[r * w + c] = W[r * w + c] - d0;
    if (r < w && c + 1 < w) Ms[r * w + c + 1] = W[r * w + c + 1] - d1;
  }
  __syncthreads();
  if (warp == 0) {
    warp_cholesky(Ms, Lo, w, &bad);
    __syncwarp();
    // T = L^{-T} into Ts (ld 33): lane j forward-substitutes column j of L^{-1}
    const int j = lane;
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
      for (int i = 0; i < w; ++i) Ts[j * 33 + i] = Xs[i * 33 + j];  // T[j][i] = Linv[i][j]
  }
  __syncthreads();
  for (int i = tid; i < w * w; i += 256) {
    const int r = i / w, c = i % w;
    L[i] = Lo[r * 32 + c];
    T[i] = Ts[r * 33 + c];
    if (L1 && R) {  // R[r][c] = sum_k L[k][r] L1[c][k]  (= (L^T L1^T)[r][c])
      double a = 0.0;
      for (int k = 0; k < w; ++k) a = fma(Lo[k * 32 + r], L1s[c * 33 + k], a);
      R[i] = a;
    }
  }
  if (tid == 0 && bad) atomicOr(flag, 1);
  // Hp = H T and (pass 2) Hout = H1 + H L1^T: 8 x 8 row tiles, K = w
  const int nrt = (s + 7) / 8;
  for (int t = warp; t < nrt * nt; t += 8) {
    const int rt = t / nt, ct = t % nt;
    const int r = rt * 8 + gid, cb = ct * 8 + gid;
    double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
    for (int k0 = 0; k0 < w; k0 += 4) {
      const int k = k0 + tig;
      const double a = (r < s && k < w) ? H[(size_t)r * w + k] : 0.0;
      const double b = (k < w && cb < w) ? Ts[k * 33 + cb] : 0.0;
      dmma884s(d0, d1, a, b);
      if (Hout) {
        const double b2 = (k < w && cb < w) ? L1s[cb * 33 + k] : 0.0;  // L1^T[k][cb]
        dmma884s(e0, e1, a, b2);
      }
    }
    const int ro = rt * 8 + gid, c = ct * 8 + 2 * tig;
    if (ro < s) {
      if (c < w) Hp[(size_t)ro * w + c] = d0;
      if (c + 1 < w) Hp[(size_t)ro * w + c + 1] = d1;
      if (Hout) {
        if (c < w) Hout[(size_t)ro * w + c] = H1[(size_t)ro * w + c] + e0;
        if (c + 1 < w) Hout[(size_t)ro * w + c + 1] = H1[(size_t)ro * w + c + 1] + e1;
      }
    }
  }
}

void pip_finalize(const double* C, int s, int w, double* L, double* T, double* Hp, int* flag,
                  const double* L1, double* R, const double* H1, double* Hout,
                  cudaStream_t st) {
  pip_finalize_kernel<<<1, 256, 0, st>>>(C, s, w, L, T, Hp, flag, L1, R, H1, Hout);
  TSVD_CHECK_LAUNCH();
}

// ------------------------------------------------------------ small GEMM ---
// C (m x n, ldc) = alpha op(A) op(B) + beta C for the small matrices of
// BCGS-PIP+ (reading R34): W - H^T H, H T, L2^T L1^T, H1 + H2 L1^T.  One
// thread per entry, k summed in increasing order (deterministic); op(X) =
// X or X^T of a row-major X.
__global__ void small_gemm_kernel(const double* __restrict__ A, int lda, int ta,
                                  const double* __restrict__ B, int ldb, int tb,
                                  double* __restrict__ Cm, int ldc, int m, int n, int k,
                                  double alpha, double beta) {
  pdl_enter();
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)m * n) return;
  const int i = (int)(t / n), j = (int)(t % n);
  double a0 = 0.0, a1 = 0.0;
  int p = 0;
  for (; p + 1 < k; p += 2) {
    const double x0 = ta ? A[(int64_t)p * lda + i] : A[(int64_t)i * lda + p];
    const double y0 = tb ? B[(int64_t)j * ldb + p] : B[(int64_t)p * ldb + j];
    const double x1 = ta ? A[(int64_t)(p + 1) * lda + i] : A[(int64_t)i * lda + p + 1];
    const double y1 = tb ? B[(int64_t)j * ldb + p + 1] : B[(int64_t)(p + 1) * ldb + j];
    a0 = fma(x0, y0, a0);
    a1 = fma(x1, y1, a1);
  }
  if (p < k) {
    const double x0 = ta ? A[(int64_t)p * lda + i] : A[(int64_t)i * lda + p];
    const double y0 = tb ? B[(int64_t)j * ldb + p] : B[(int64_t)p * ldb + j];
    a0 = fma(x0, y0, a0);
  }
  const double v = alpha * (a0 + a1);
  Cm[(int64_t)i * ldc + j] = beta == 0.0 ? v : fma(beta, Cm[(int64_t)i * ldc + j], v);
}

void small_gemm(const double* A, int lda, bool ta, const double* B, int ldb, bool tb, double* C,
                int ldc, int m, int n, int k, double alpha, double beta, cudaStream_t st) {
  const int64_t e = (int64_t)m * n;
  if (e <= 0) return;
  launch_pdl(small_gemm_kernel, (unsigned)((e + 127) / 128), 128, 0, st, A, lda, ta ? 1 : 0, B, ldb,
                                                                  tb ? 1 : 0, C, ldc, m, n, k,
                                                                  alpha, beta);
  TSVD_CHECK_LAUNCH();
}

// --------------------------------------------------------------- helpers ---
__global__ void copy_block_kernel(const double* __restrict__ src, int64_t lds,
                                  double* __restrict__ dst, int64_t ldd, int64_t rows, int cols,
                                  int transpose) {
  pdl_enter();
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
  launch_pdl(copy_block_kernel, (unsigned)blocks, 256, 0, st, src, lds, dst, ldd, rows, cols,
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
  pdl_enter();
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
  launch_pdl(lanczos_rho_kernel, (cnt + 127) / 128, 128, 0, st, Rbar, b, Vb, d, S, cnt, rho);
  TSVD_CHECK_LAUNCH();
}

// Thick restart (oracle/lancsvd.py header): the first l
// columns/rows of the next cycle's projected matrix B' (d x d, row-major,
// zero elsewhere on entry):  B'[:l, :l] = diag(Sigma_l) and the "arrow" row
// block  B'[l:l+b, :l] = S = Rbar_k Vbar[d-b:d, :l]  (A P' = Pbar' Sigma_l +
// Qbar_{k+1} S).  One thread per column j < l.
__global__ void thick_arrow_kernel(const double* __restrict__ Rbar, int b,
                                   const double* __restrict__ Vb, int d,
                                   const double* __restrict__ S, int l,
                                   double* __restrict__ B) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= l) return;
  B[(int64_t)j * d + j] = S[j];
  for (int i = 0; i < b; ++i) {
    double t = 0.0;
    for (int c = 0; c < b; ++c) t = fma(Rbar[i * b + c], Vb[(int64_t)(d - b + c) * d + j], t);
    B[(int64_t)(l + i) * d + j] = t;
  }
}

void thick_arrow(const double* Rbar, int b, const double* Vb, int d, const double* S, int l,
                 double* B, cudaStream_t st) {
  thick_arrow_kernel<<<(l + 127) / 128, 128, 0, st>>>(Rbar, b, Vb, d, S, l, B);
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
