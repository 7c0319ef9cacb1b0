// Small projected SVD on the device: block one-sided (Hestenes) Jacobi.
// Alg. 1 S5 (SVD of R_p) and Alg. 2 (SVD of B_k, Eq. 9).  The paper runs
// LAPACK GESVD on the host (Table 1); any backward-stable SVD
// gives the same triplets up to signs (reading R20), and keeping it on the
// device removes the PCIe round trip (north_star (4)).
//
// G (initially B, column-major in global memory / L2) is orthogonalised by
// plane rotations applied from the right, V accumulates them; at convergence
// sigma_j = ||g_j||, ubar_j = g_j / sigma_j, vbar_j = v_j, sorted descending.
//
// Parallel block ordering (one cooperative launch, one CTA per block pair):
// the d columns are cut into nb blocks of JC columns; in each round of the
// round-robin tournament CTA p owns a disjoint pair of blocks (I, J) and
//   1. loads the 2*JC columns [G_I G_J] into shared memory,
//   2. runs one-sided Jacobi sweeps on those 2*JC columns in shared memory
//      (JC disjoint column pairs per inner round, one warp per pair), each
//      rotation computed from the current columns' dot products, and
//      accumulates the 2JC x 2JC orthogonal J of the applied rotations,
//   3. writes the rotated columns back and updates [V_I V_J] <- [V_I V_J] J,
// then all CTAs meet at a grid barrier.  A sweep = nb-1 rounds; sweeps repeat
// until no rotation with |g_p^T g_q| > tol ||g_p|| ||g_q|| (tol = d u) was needed.
// Rotation (Rutishauser): zeta = (M_qq - M_pp) / (2 M_pq),
//   t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), cs = 1/sqrt(1+t^2), sn = cs t,
//   [g_p g_q] <- [g_p g_q] [[cs, sn], [-sn, cs]].
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "internal.h"

namespace tsvd {

constexpr int JC = 8;        // columns per block
constexpr int JW = 2 * JC;   // columns per block pair
constexpr int JP = JW + 1;   // padded smem row
constexpr int kMaxSweeps = 60;  // Lanczos B_k: 12-19 sweeps; graded random B (tests): ~30
constexpr int kInnerSweeps = 1;
constexpr int kJacobiMaxD = kSmallSvdMaxD;

static int jac_nb(int d) {
  int nb = (d + JC - 1) / JC;
  if (nb < 2) nb = 2;
  if (nb & 1) ++nb;
  return nb;
}

static size_t jac_layout(size_t d, size_t dp) { return d * dp + dp * dp + dp; }

size_t small_svd_work(int d) {
  const size_t dp8 = (size_t)jac_nb(d) * JC;
  size_t n = jac_layout(d, dp8);
  const size_t dp4 = (size_t)(((d + 3) / 4 + 1) & ~1) * 4 + 8;
  n = std::max(n, jac_layout(d, dp4));
  const size_t dp2 = (size_t)(((d + 1) / 2 + 1) & ~1) * 2 + 8;
  n = std::max(n, jac_layout(d, dp2));
  return n + 64 + 1024;  // flags (1024 doubles), then control words (last 64 doubles)
}
static unsigned* jac_ctl(double* work, int d) {
  return (unsigned*)(work + small_svd_work(d) - 64);
}
// register path: per-sweep "rotated" words [0, kMaxSweeps) and per-block
// version counters [32, 32 + nb) (dataflow hand-off between CTAs)
static unsigned* jac_flags(double* work, int d) {
  return (unsigned*)(work + small_svd_work(d) - 64 - 1024);
}
constexpr int kJacFlagVer = 64;  // after the kMaxSweeps per-sweep words

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = bar + 1;
    const unsigned gen = *vgen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void circle_pair(int t, int round, int ne, int& p, int& q) {
  p = (t == 0) ? 0 : ((t - 1 + round) % (ne - 1)) + 1;
  q = ((ne - 2 - t + round) % (ne - 1)) + 1;
  if (p > q) {
    const int x = p;
    p = q;
    q = x;
  }
}

__global__ void jacobi_init_kernel(const double* __restrict__ B, int d, int dp,
                                   double* __restrict__ G, double* __restrict__ V,
                                   unsigned* __restrict__ ctl, unsigned* __restrict__ flags) {
  if (flags)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2048; i += gridDim.x * blockDim.x)
      flags[i] = 0u;
  const int64_t total = (int64_t)d * dp + (int64_t)dp * dp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < (int64_t)d * dp) {
      const int c = (int)(i / d), r = (int)(i % d);
      G[i] = c < d ? B[(int64_t)r * d + c] : 0.0;  // G column-major
    } else {
      const int64_t k = i - (int64_t)d * dp;
      const int c = (int)(k / dp), r = (int)(k % dp);
      V[k] = (r == c) ? 1.0 : 0.0;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < 8) ctl[threadIdx.x] = 0u;
}

// ||B||_F^2 into the control area (one CTA, fixed-order sums): the scale of
// the negligible-column test of the rotation loops.  A column pair whose
// smaller column has norm <= u ||B||_F is not rotated: such a column is
// rounding noise of size u ||B||, rotating it changes the SVD by less than
// the backward error already committed, and without the test a B with
// singular values below u sigma_1 (rank-deficient or graded B) keeps
// rotating noise until the sweep cap.
__global__ void __launch_bounds__(1024) jacobi_fro_kernel(const double* __restrict__ B, int d,
                                                          double* __restrict__ out) {
  __shared__ double red[1024];
  double a0 = 0.0, a1 = 0.0;
  const int64_t n = (int64_t)d * d;
  int64_t i = threadIdx.x;
  for (; i + 1024 < n; i += 2048) {
    a0 = fma(B[i], B[i], a0);
    a1 = fma(B[i + 1024], B[i + 1024], a1);
  }
  if (i < n) a0 = fma(B[i], B[i], a0);
  red[threadIdx.x] = a0 + a1;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

__global__ void __launch_bounds__(256) jacobi_block_kernel(double* __restrict__ G,
                                                           double* __restrict__ V, int d, int nb,
                                                           double* __restrict__ nrm,
                                                           double* __restrict__ Ub,
                                                           double* __restrict__ S,
                                                           double* __restrict__ Vb,
                                                           unsigned* __restrict__ ctl) {
  extern __shared__ double sm[];
  double* Gs = sm;                   // d x JP (row r, col k) ; reused for V chunks
  double* Js = Gs + (size_t)d * JP;  // JW x JP
  __shared__ int any_rot, inner_rot;
  unsigned* bar = ctl;          // [0] count, [1] generation
  unsigned* rot = ctl + 2;      // [2], [3] sweep flags (double-buffered)
  const int tid = threadIdx.x;
  const int dp = nb * JC;
  const unsigned nblk = gridDim.x;
  const double tol = (double)d * 0x1.0p-53;
  const double absmin = *reinterpret_cast<const double*>(ctl + 8) * 0x1.0p-106;  // (u ||B||_F)^2
  const int warp = tid >> 5, lane = tid & 31;

  int sweep = 0;
  for (; sweep < kMaxSweeps; ++sweep) {
    for (int round = 0; round < nb - 1; ++round) {
      int bi, bj;
      circle_pair(blockIdx.x, round, nb, bi, bj);
      // 1. load the pair's columns
      for (int base = 0; base < d * JW; base += 256 * 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int idx = base + tid + 256 * u;
          const int k = idx / d, r = idx % d;
          const int col = k < JC ? bi * JC + k : bj * JC + (k - JC);
          v[u] = idx < d * JW ? G[(size_t)col * d + r] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int idx = base + tid + 256 * u;
          if (idx < d * JW) Gs[(idx % d) * JP + idx / d] = v[u];
        }
      }
      if (tid == 0) any_rot = 0;
      __syncthreads();
      // 2. J = I
      {
        const int i = tid / JW, j = tid % JW;
        Js[i * JP + j] = (i == j) ? 1.0 : 0.0;
      }
      __syncthreads();
      // 3. one-sided Jacobi inside the pair: JC disjoint column pairs per
      //    inner round, one warp per pair, dot products from the current
      //    columns (no Gram matrix: keeps the relative accuracy of Hestenes
      //    rotations); J accumulates the rotations for V.
      for (int is = 0; is < kInnerSweeps; ++is) {
        if (tid == 0) inner_rot = 0;
        __syncthreads();
        for (int ir = 0; ir < JW - 1; ++ir) {
          int p, q;
          circle_pair(warp, ir, JW, p, q);
          double a = 0.0, b = 0.0, c = 0.0;
          for (int r = lane; r < d; r += 32) {
            const double x = Gs[r * JP + p], y = Gs[r * JP + q];
            a = fma(x, x, a);
            b = fma(y, y, b);
            c = fma(x, y, c);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
            c += __shfl_xor_sync(0xffffffffu, c, o);
          }
          if (a > absmin && b > absmin && c * c > (tol * tol) * (a * b)) {  // |c| > tol sqrt(ab)
            // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = h / c, h = (b - a)/2,
            // rewritten as sign(h) c / (|h| + sqrt(h^2 + c^2)) (one division)
            const double h = 0.5 * (b - a);
            const double t = (h >= 0.0 ? c : -c) / (fabs(h) + sqrt(fma(h, h, c * c)));
            const double cs = rsqrt(fma(t, t, 1.0));
            const double sn = cs * t;
            for (int r = lane; r < d; r += 32) {
              const double x = Gs[r * JP + p], y = Gs[r * JP + q];
              Gs[r * JP + p] = cs * x - sn * y;
              Gs[r * JP + q] = sn * x + cs * y;
            }
            if (lane < JW) {
              const double x = Js[lane * JP + p], y = Js[lane * JP + q];
              Js[lane * JP + p] = cs * x - sn * y;
              Js[lane * JP + q] = sn * x + cs * y;
            }
            if (lane == 0) inner_rot = 1;
          }
          __syncthreads();
        }
        const int ir_any = inner_rot;
        if (ir_any && tid == 0) any_rot = 1;
        __syncthreads();
        if (!ir_any) break;
      }
      // 4. write the rotated pair back; V pair <- V pair J
      if (any_rot) {
        for (int idx = tid; idx < d * JW; idx += 256) {
          const int k = idx / d, r = idx % d;
          const int col = k < JC ? bi * JC + k : bj * JC + (k - JC);
          G[(size_t)col * d + r] = Gs[r * JP + k];
        }
        const int chunk = min(256, d);  // Gs holds d rows
        for (int r0 = 0; r0 < dp; r0 += chunk) {
          const int rows = min(chunk, dp - r0);
          __syncthreads();
#pragma unroll 4
          for (int idx = tid; idx < rows * JW; idx += 256) {
            const int k = idx / rows, r = idx % rows;
            const int col = k < JC ? bi * JC + k : bj * JC + (k - JC);
            Gs[r * JP + k] = V[(size_t)col * dp + r0 + r];
          }
          __syncthreads();
          for (int idx = tid; idx < rows * JW; idx += 256) {
            const int k = idx / rows, r = idx % rows;
            double acc = 0.0;
#pragma unroll
            for (int l = 0; l < JW; ++l) acc = fma(Gs[r * JP + l], Js[l * JP + k], acc);
            const int col = k < JC ? bi * JC + k : bj * JC + (k - JC);
            V[(size_t)col * dp + r0 + r] = acc;
          }
        }
        if (tid == 0) atomicOr(rot + (sweep & 1), 1u);
      }
      grid_barrier(bar, nblk);
      if (round == 0 && blockIdx.x == 0 && tid == 0) atomicExch(rot + ((sweep + 1) & 1), 0u);
    }
    // every CTA passed the last barrier of the sweep: the flag is final
    const unsigned any = *((volatile unsigned*)(rot + (sweep & 1)));
    if (!any) break;
  }
  if (blockIdx.x == 0 && tid == 0) ctl[4] = (unsigned)sweep;
  // norms of the d genuine columns (padded columns are zero)
  for (int j = blockIdx.x * 8 + warp; j < dp; j += nblk * 8) {
    double a = 0.0;
    for (int i = lane; i < d; i += 32) {
      const double g = G[(size_t)j * d + i];
      a = fma(g, g, a);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) nrm[j] = sqrt(a);
  }
  grid_barrier(bar, nblk);
  // rank (descending, ties -> lower index) and outputs
  for (int j = blockIdx.x * 8 + warp; j < dp; j += nblk * 8) {
    const double sj = nrm[j];
    int cnt = 0;
    for (int k = lane; k < dp; k += 32) {
      const double sk = nrm[k];
      cnt += (sk > sj || (sk == sj && k < j)) ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (cnt >= d) continue;
    const double inv = sj > 0.0 ? 1.0 / sj : 0.0;
    if (lane == 0) S[cnt] = sj;
    for (int i = lane; i < d; i += 32) {
      Ub[(size_t)i * d + cnt] = __ldcg(G + (size_t)j * d + i) * inv;
      Vb[(size_t)i * d + cnt] = __ldcg(V + (size_t)j * dp + i);
    }
  }
}

// Register-resident variant (d <= 1024): during a round the pair's 2*JC
// columns of G are held in registers (rows tid + JR_T*k, k < RG), so a
// rotation touches no shared memory.  Per inner round every thread adds its
// rows' contributions to the 3*JC dot products, the CTA reduces them (warp
// recursive-halving butterfly, then a fixed-order sum over warps), JC
// threads form the rotations, every thread applies them to its rows and 128
// threads accumulate them into the 2JC x 2JC orthogonal J (shared memory).
// After the inner sweep the V rows are streamed through registers and
// multiplied by J.
__host__ __device__ constexpr int cpair_lo(int t, int r, int jw) {
  const int p = (t == 0) ? 0 : ((t - 1 + r) % (jw - 1)) + 1;
  const int q = ((jw - 2 - t + r) % (jw - 1)) + 1;
  return p < q ? p : q;
}
__host__ __device__ constexpr int cpair_hi(int t, int r, int jw) {
  const int p = (t == 0) ? 0 : ((t - 1 + r) % (jw - 1)) + 1;
  const int q = ((jw - 2 - t + r) % (jw - 1)) + 1;
  return p < q ? q : p;
}

// one recursive-halving level: M live values -> M/2 (lanes with bit o set
// keep the upper half)
template <int NVP, int M, int O>
__device__ __forceinline__ void rs_level(double (&v)[NVP], int lane) {
  if constexpr (O >= 1) {
    const bool up = (lane & O) != 0;
#pragma unroll
    for (int i = 0; i < M / 2; ++i) {
      const double send = up ? v[i] : v[i + M / 2], keep = up ? v[i + M / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, O);
    }
    rs_level<NVP, M / 2, O / 2>(v, lane);
  }
}

// warp reduce-scatter; afterwards NVP >= 32: v[j] = warp sum of value
// lane * (NVP/32) + j; NVP == 16: v[0] = warp sum of value lane % 16
template <int NVP>
__device__ __forceinline__ void warp_reduce_scatter(double (&v)[NVP], int lane) {
  if constexpr (NVP == 16) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], 16);
    rs_level<16, 16, 8>(v, lane);
  } else {
    rs_level<NVP, NVP, 16>(v, lane);
  }
}

// pair t of inner round ir: MODE 0 = circle over all 2 JB columns (2 JB - 1
// inner rounds), 1 = inside each of the two blocks (JB - 1), 2 = the JB x JB
// cross pairs (JB inner rounds)
template <int JB, int MODE>
__device__ __forceinline__ void jac_pair(int t, int ir, int& p, int& q) {
  if constexpr (MODE == 0) {
    p = cpair_lo(t, ir, 2 * JB);
    q = cpair_hi(t, ir, 2 * JB);
  } else if constexpr (MODE == 1) {
    const int h = JB / 2;
    const int off = t < h ? 0 : JB, tt = t < h ? t : t - h;
    p = off + cpair_lo(tt, ir, JB);
    q = off + cpair_hi(tt, ir, JB);
  } else {
    p = t;
    q = JB + (t + ir) % JB;
  }
}


// One inner round on the 2 JB columns held in registers (RG rows per
// thread, NTHR threads): dot products -> warp reduce-scatter -> one CTA
// barrier -> every warp sums the per-warp partials in warp order and computes
// the JB rotations (Rutishauser) redundantly (lane t: rotation t, broadcast by
// shuffles) -> apply to the columns; warp 0 also applies them to J.  red is
// double-buffered by inner-round parity, so one barrier per inner round
// suffices (a warp reads red[ir & 1] before it can reach barrier ir + 1).
template <int RG, int JB, int MODE, int NTHR, bool WV = true>
__device__ __forceinline__ void jac_inner(int ir, double (&x)[RG][2 * JB],
                                          double (&vv)[RG][2 * JB],
                                          double (*red)[3 * JB + 1], int* any_rot, double tol,
                                          double absmin) {
  constexpr int JW = 2 * JB, NV = 3 * JB;
  constexpr int NVP = NV <= 16 ? 16 : (NV <= 32 ? 32 : 64);
  constexpr int NW = NTHR / 32;
  static_assert(JB <= 32, "one lane per rotation");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double (*rb)[NV + 1] = red + (ir & 1) * NW;
  double v[NVP];
#pragma unroll
  for (int i = NV; i < NVP; ++i) v[i] = 0.0;
#pragma unroll
  for (int t = 0; t < JB; ++t) {
    int p, q;
    jac_pair<JB, MODE>(t, ir, p, q);
    double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
    for (int k = 0; k < RG; ++k) {
      a = fma(x[k][p], x[k][p], a);
      b = fma(x[k][q], x[k][q], b);
      c = fma(x[k][p], x[k][q], c);
    }
    v[3 * t] = a;
    v[3 * t + 1] = b;
    v[3 * t + 2] = c;
  }
  warp_reduce_scatter<NVP>(v, lane);
  if constexpr (NVP >= 32) {
#pragma unroll
    for (int j = 0; j < NVP / 32; ++j) {
      const int idx = lane * (NVP / 32) + j;
      if (idx < NV) rb[warp][idx] = v[j];
    }
  } else {
    if (lane < NV) rb[warp][lane] = v[0];
  }
  __syncthreads();
  double cs = 1.0, sn = 0.0;
  if (lane < JB) {
    double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
    for (int w2 = 0; w2 < NW; ++w2) {
      a += rb[w2][3 * lane];
      b += rb[w2][3 * lane + 1];
      c += rb[w2][3 * lane + 2];
    }
    if (a > absmin && b > absmin && c * c > (tol * tol) * (a * b)) {  // |c| > tol sqrt(ab)
      const double h = 0.5 * (b - a);
      const double t = (h >= 0.0 ? c : -c) / (fabs(h) + sqrt(fma(h, h, c * c)));
      cs = rsqrt(fma(t, t, 1.0));
      sn = cs * t;
      if (warp == 0) *any_rot = 1;
    }
  }
#pragma unroll
  for (int t = 0; t < JB; ++t) {
    int p, q;
    jac_pair<JB, MODE>(t, ir, p, q);
    const double ct = __shfl_sync(0xffffffffu, cs, t), st = __shfl_sync(0xffffffffu, sn, t);
#pragma unroll
    for (int k = 0; k < RG; ++k) {
      const double xp = x[k][p], xq = x[k][q];
      x[k][p] = ct * xp - st * xq;
      x[k][q] = st * xp + ct * xq;
      // the same rotation on this thread's rows of V (held in registers for
      // the round): no accumulated J, no serial J update on the step's path
      if constexpr (WV) {
        const double vp = vv[k][p], vq = vv[k][q];
        vv[k][p] = ct * vp - st * vq;
        vv[k][q] = st * vp + ct * vq;
      }
    }
  }
}


// Rounds hand blocks from CTA to CTA by dataflow instead of a grid barrier:
// every block b carries a version counter (the number of rounds it has been
// through); a CTA starts global round g on its pair (bi, bj) once both
// versions reach g, and publishes g + 1 after writing the blocks back
// (release / acquire through __threadfence + atomics; block data is read
// with L1-bypassing loads).  Each round visits every block exactly once, so
// a block's owner in round g is unique.  One grid barrier per sweep decides
// convergence from the per-sweep "rotated" word.
#ifdef JAC_TIMING
// development instrumentation (A/B build only): CTA 0 accumulates clock64
// cycles per round phase: [0] wait, [1] loads, [2] inner steps, [3] stores +
// fence + publish, [4] rounds
__device__ unsigned long long g_jac_t[8];
#define JT(k) do { if (blockIdx.x == 0 && threadIdx.x == 0) { const long long t_ = clock64(); g_jac_t[k] += t_ - jt0; jt0 = t_; } } while (0)
#else
#define JT(k) do { } while (0)
#endif

__device__ __forceinline__ void jac_wait_ver(unsigned* ver, int b, unsigned g) {
  volatile unsigned* v = ver + b;
  while (*v < g) __nanosleep(32);
}
__device__ __forceinline__ void jac_wait_acquire(const unsigned* p, unsigned g) {
  unsigned v;
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  } while (v < g);
}
__device__ __forceinline__ void st_relaxed_gpu(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// WV = false: the rotations are not applied to V (the caller forms the
// needed right vectors as B^T u_i / sigma_i afterwards, small_svd_top): half
// the rotation work and no V traffic per round.
template <int RG, int JC, bool CYC, int JR_T, bool WV = true>
__global__ void __launch_bounds__(JR_T, 1) jacobi_reg_kernel(double* __restrict__ G,
                                                            double* __restrict__ V, int d, int nb,
                                                            double* __restrict__ nrm,
                                                            double* __restrict__ Ub,
                                                            double* __restrict__ S,
                                                            double* __restrict__ Vb,
                                                            unsigned* __restrict__ ctl,
                                                            unsigned* __restrict__ flags,
                                                            int opt) {
  constexpr int JW = 2 * JC;   // columns of a block pair (shadows the file-scope JW)
  constexpr int NW = JR_T / 32;
  constexpr int NV = 3 * JC;  // partial sums per inner round
  __shared__ double red[2 * NW][NV + 1];
  __shared__ int any_rot;
  unsigned* bar = ctl;
  unsigned* rot = flags;                 // [sweep]
  unsigned* ver = flags + kJacFlagVer;   // [block]
  const int tid = threadIdx.x;
  const int dp = nb * JC;
  const unsigned nblk = gridDim.x;
  const double tol = (double)d * 0x1.0p-53;
  const double absmin = *reinterpret_cast<const double*>(ctl + 8) * 0x1.0p-106;  // (u ||B||_F)^2
  double x[RG][JW];
  // acquire / release hand-off (ld.acquire polling; fence.acq_rel + relaxed
  // version stores) instead of volatile polling + __threadfence + atomicExch:
  // d = 384 6.33 -> 5.71 ms, same results (TSVD_JACOBI_ACQREL = 0: the old one)
  const bool acqrel = opt != 0;
  int sweep = 0;
  // CYC: cyclic-by-blocks sweep (round 0 inside the home blocks 2k, 2k+1,
  // then nb-1 rounds of cross pairs: every pair once, ~d inner rounds);
  // else each round sweeps all pairs of the 2 JC columns (~2d inner rounds)
  const int nrounds = CYC ? nb : nb - 1;
  unsigned g = 0;  // global round counter
#ifdef JAC_TIMING
  long long jt0 = clock64();
#endif
  for (; sweep < kMaxSweeps; ++sweep) {
    for (int round = 0; round < nrounds; ++round, ++g) {
      JT(5);
      int bi, bj;
      if (CYC && round == 0) {
        bi = 2 * blockIdx.x;
        bj = 2 * blockIdx.x + 1;
      } else {
        circle_pair(blockIdx.x, CYC ? round - 1 : round, nb, bi, bj);
      }
      if (tid == 0) {
        if (acqrel) {
          jac_wait_acquire(ver + bi, g);
          jac_wait_acquire(ver + bj, g);
        } else {
          jac_wait_ver(ver, bi, g);
          jac_wait_ver(ver, bj, g);
          __threadfence();
        }
      }
      __syncthreads();
      JT(0);
#pragma unroll
      for (int k = 0; k < RG; ++k) {
        const int row = tid + JR_T * k;
#pragma unroll
        for (int c = 0; c < JW; ++c) {
          const int col = c < JC ? bi * JC + c : bj * JC + (c - JC);
          x[k][c] = row < d ? __ldcg(G + (size_t)col * d + row) : 0.0;
        }
      }
      // this round's V rows: in flight during the inner rounds (the pair's V
      // columns belong to this CTA until it publishes the new versions)
      double vv[RG][JW];
      if constexpr (WV) {
#pragma unroll
        for (int k = 0; k < RG; ++k) {
          const int row = tid + JR_T * k;
#pragma unroll
          for (int c = 0; c < JW; ++c) {
            const int col = c < JC ? bi * JC + c : bj * JC + (c - JC);
            vv[k][c] = row < dp ? __ldcg(V + (size_t)col * dp + row) : 0.0;
          }
        }
      }
      if (tid == 0) any_rot = 0;
#ifdef JAC_TIMING
      { double sink = 0.0;
#pragma unroll
        for (int k = 0; k < RG; ++k) sink += x[k][0];
        if (sink == 1.2345e300) any_rot = 2; }
      __syncthreads();
#endif
      JT(1);
      // any_rot initialised before warp 0 may set it (first inner barrier)
      if (!CYC) {
#pragma unroll
        for (int ir = 0; ir < JW - 1; ++ir)
          jac_inner<RG, JC, 0, JR_T, WV>(ir, x, vv, red, &any_rot, tol, absmin);
      } else if (round == 0) {
#pragma unroll
        for (int ir = 0; ir < JC - 1; ++ir)
          jac_inner<RG, JC, 1, JR_T, WV>(ir, x, vv, red, &any_rot, tol, absmin);
      } else {
#pragma unroll
        for (int ir = 0; ir < JC; ++ir)
          jac_inner<RG, JC, 2, JR_T, WV>(ir, x, vv, red, &any_rot, tol, absmin);
      }
      __syncthreads();
      JT(2);
      if (any_rot) {
#pragma unroll
        for (int k = 0; k < RG; ++k) {
          const int row = tid + JR_T * k;
          if (row < d) {
#pragma unroll
            for (int c = 0; c < JW; ++c) {
              const int col = c < JC ? bi * JC + c : bj * JC + (c - JC);
              __stcg(G + (size_t)col * d + row, x[k][c]);
            }
          }
        }
        // V pair rows, rotated in registers alongside G
        if constexpr (WV) {
#pragma unroll
          for (int k = 0; k < RG; ++k) {
            const int row = tid + JR_T * k;
            if (row < dp) {
#pragma unroll
              for (int c = 0; c < JW; ++c) {
                const int col = c < JC ? bi * JC + c : bj * JC + (c - JC);
                __stcg(V + (size_t)col * dp + row, vv[k][c]);
              }
            }
          }
        }
      }
      __syncthreads();
      if (tid == 0) {
        if (any_rot) atomicOr(rot + sweep, 1u);
        if (acqrel) {
          // release: the CTA's stores (ordered before this thread by the
          // barrier above) become visible before the new versions
          asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
          st_relaxed_gpu(ver + bi, g + 1);
          st_relaxed_gpu(ver + bj, g + 1);
        } else {
          __threadfence();
          atomicExch(ver + bi, g + 1);
          atomicExch(ver + bj, g + 1);
        }
      }
      JT(3);
#ifdef JAC_TIMING
      if (blockIdx.x == 0 && tid == 0) g_jac_t[4] += 1;
#endif
    }
    grid_barrier(bar, nblk);
    const unsigned any = *((volatile unsigned*)(rot + sweep));
    if (!any) break;
  }
  const int warp = tid >> 5, lane = tid & 31;
  if (blockIdx.x == 0 && tid == 0) ctl[4] = (unsigned)sweep;
  for (int j = blockIdx.x * NW + warp; j < dp; j += nblk * NW) {
    double a = 0.0;
    for (int i = lane; i < d; i += 32) {
      const double g = __ldcg(G + (size_t)j * d + i);
      a = fma(g, g, a);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) nrm[j] = sqrt(a);
  }
  grid_barrier(bar, nblk);
  for (int j = blockIdx.x * NW + warp; j < dp; j += nblk * NW) {
    const double sj = nrm[j];
    int cnt = 0;
    for (int k = lane; k < dp; k += 32) {
      const double sk = nrm[k];
      cnt += (sk > sj || (sk == sj && k < j)) ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (cnt >= d) continue;
    const double inv = sj > 0.0 ? 1.0 / sj : 0.0;
    if (lane == 0) S[cnt] = sj;
    for (int i = lane; i < d; i += 32) {
      Ub[(size_t)i * d + cnt] = __ldcg(G + (size_t)j * d + i) * inv;
      if constexpr (WV) Vb[(size_t)i * d + cnt] = __ldcg(V + (size_t)j * dp + i);
    }
  }
}

constexpr bool g_jacobi_cyc = true;  // the cyclic-by-blocks ordering (the only one built)

int g_jacobi_jc = getenv("TSVD_JACOBI_JC") ? atoi(getenv("TSVD_JACOBI_JC")) : 4;
// TSVD_JACOBI_NT = 64 | 128 | 256 forces the CTA size (0, default: by d)
int g_jacobi_nt = getenv("TSVD_JACOBI_NT") ? atoi(getenv("TSVD_JACOBI_NT")) : 0;
// acquire / release block hand-off between the CTAs (default on)
int g_jacobi_opt = getenv("TSVD_JACOBI_ACQREL") ? atoi(getenv("TSVD_JACOBI_ACQREL")) : 1;

template <int JCV, bool WV = true>
static bool reg_launch(const double* B, int d, double* Ub, double* S, double* Vb, double* work,
                       unsigned* ctl, cudaStream_t st, int hog_smem = 0) {
  int nbr = (d + JCV - 1) / JCV;
  if (nbr < 2) nbr = 2;
  if (nbr & 1) ++nbr;
  const int dpr = nbr * JCV;
  if (nbr / 2 > 148 || jac_layout(d, dpr) + 64 > small_svd_work(d)) return false;
  // threads per CTA: fewer warps make the per-step cross-warp reduction and
  // barrier cheaper (the step is latency-bound), too few leave the rows'
  // FMA chains exposed: 128 up to d = 768 (RG <= 6 rows per thread), else 256
  // (measured at d = 384: 64 threads 8.4 ms, 128 6.8 ms, 256 8.1 ms)
  const int nth = g_jacobi_nt ? g_jacobi_nt : (d <= 768 ? 128 : 256);
  const int RG = (d + nth - 1) / nth;
  void* fn = nullptr;
  // instantiated: the cyclic-by-blocks ordering (TSVD_JACOBI_CYC = 0, the
  // all-pairs-per-round ordering, was measured slower and is no longer built)
  // with 128 threads (d <= 768) or 256 threads (d <= 1024)
#define REG_FN(R, NT) fn = (void*)jacobi_reg_kernel<R, JCV, true, NT, WV>
  if (nth == 128) {
    if (RG <= 1) REG_FN(1, 128);
    else if (RG == 2) REG_FN(2, 128);
    else if (RG == 3) REG_FN(3, 128);
    else if (RG == 4) REG_FN(4, 128);
    else if (RG == 5) REG_FN(5, 128);
    else if (RG == 6) REG_FN(6, 128);
    else return false;
  } else if (nth == 256) {
    if (RG <= 1) REG_FN(1, 256);
    else if (RG == 2) REG_FN(2, 256);
    else if (RG == 3) REG_FN(3, 256);
    else if (RG == 4) REG_FN(4, 256);
    else return false;
  } else {
    return false;
  }
#undef REG_FN
  double* G = work;
  double* V = G + (size_t)d * dpr;
  double* nrm = V + (size_t)dpr * dpr;
  unsigned* flags = jac_flags(work, d);
  if (nbr + kJacFlagVer > 2048) return false;
  jacobi_init_kernel<<<148 * 4, 256, 0, st>>>(B, d, dpr, G, V, ctl, flags);
  jacobi_fro_kernel<<<1, 1024, 0, st>>>(B, d, reinterpret_cast<double*>(ctl + 8));
  TSVD_CHECK_LAUNCH();
  int nblocks = nbr / 2, nbv = nbr;
  int opt = g_jacobi_opt;
  void* args[] = {&G, &V, &d, &nbv, &nrm, &Ub, &S, &Vb, &ctl, &flags, &opt};
  if (hog_smem > 0) {
    // never more than the device grants a block beside the kernel's static
    // shared memory (B200: 227 KB); the reservation is only a placement hint
    int dev = 0, optin = 0;
    cudaFuncAttributes fa{};
    TSVD_CUDA(cudaGetDevice(&dev));
    TSVD_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    TSVD_CUDA(cudaFuncGetAttributes(&fa, fn));
    hog_smem = std::min(hog_smem, optin - (int)fa.sharedSizeBytes - 1024);
    if (hog_smem > 0)  // idempotent host call, no shared state between handles / threads
      TSVD_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, hog_smem));
    else
      hog_smem = 0;
  }
  TSVD_CUDA(cudaLaunchCooperativeKernel(fn, dim3(nblocks), dim3(nth), args,
                                        (size_t)std::max(0, hog_smem), st));
  TSVD_CHECK_LAUNCH();
  return true;
}

#ifdef JAC_TIMING
extern "C" int tsvd_dev_jacobi_timing(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_jac_t, sizeof(unsigned long long) * 8);
}
extern "C" int tsvd_dev_jacobi_timing_reset() {
  unsigned long long z[8] = {0};
  return (int)cudaMemcpyToSymbol(g_jac_t, z, sizeof(z));
}
#endif

const unsigned* small_svd_sweeps_dev(const double* work, int d) {
  return jac_ctl(const_cast<double*>(work), d) + 4;
}
int small_svd_max_sweeps() { return kMaxSweeps; }

int small_svd_sweeps(const double* work, int d) {
  const unsigned* ctl = jac_ctl(const_cast<double*>(work), d);
  unsigned h = 0;
  TSVD_CUDA(cudaMemcpy(&h, ctl + 4, sizeof(unsigned), cudaMemcpyDeviceToHost));
  return (int)h;
}

// Vbar[:, c] /= sigma_c for c < nv; ok = sigma_{nv-1} >= 1e-3 sigma_0 > 0
__global__ void vbar_scale_kernel(double* __restrict__ Vb, int d, int nv,
                                  const double* __restrict__ S, unsigned* __restrict__ ok) {
  const int64_t n = (int64_t)d * nv;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t / nv), c = (int)(t % nv);
    const double sc = S[c];
    Vb[(int64_t)i * d + c] = sc > 0.0 ? Vb[(int64_t)i * d + c] / sc : 0.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    *ok = (S[0] > 0.0 && S[nv - 1] >= 1e-3 * S[0]) ? 1u : 0u;
}

const unsigned* small_svd_top_ok_dev(const double* work, int d) {
  return jac_ctl(const_cast<double*>(work), d) + 12;
}

void small_svd_top(const double* B, int d, int nv, double* Ub, double* S, double* Vb,
                   double* work, double* part, cudaStream_t st, int hog_smem) {
  if (d > kJacobiMaxD) throw Error{TSVD_ESHAPE, "small_svd: d > 1536"};
  unsigned* ctl = jac_ctl(work, d);
  bool ok = false;
  if (g_jacobi_cyc) {
    if (g_jacobi_jc == 4) ok = reg_launch<4, false>(B, d, Ub, S, Vb, work, ctl, st, hog_smem);
    else if (g_jacobi_jc == 8) ok = reg_launch<8, false>(B, d, Ub, S, Vb, work, ctl, st, hog_smem);
  }
  if (!ok) {
    small_svd(B, d, Ub, S, Vb, work, st);  // no top-only path for this configuration
    TSVD_CUDA(cudaMemsetAsync(ctl + 12, 0xff, sizeof(unsigned), st));  // ok (V complete)
    return;
  }
  // Vbar[:, :nv] = B^T Ubar[:, :nv] diag(1 / sigma): the right singular
  // vectors from the left ones (B vbar_i = sigma_i ubar_i), forward error
  // O(u sigma_1 / sigma_i) -- the solver falls back to the rotated V when
  // sigma_nv < 1e-3 sigma_1 (flag ctl[12] = 0)
  gemm_tn(B, d, Ub, d, d, d, nv, Vb, d, part, st);
  const int64_t n = (int64_t)d * nv;
  vbar_scale_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 4), 256, 0, st>>>(
      Vb, d, nv, S, ctl + 12);
  TSVD_CHECK_LAUNCH();
}

void small_svd(const double* B, int d, double* Ub, double* S, double* Vb, double* work,
               cudaStream_t st) {
  if (d > kJacobiMaxD) throw Error{TSVD_ESHAPE, "small_svd: d > 1536"};
  const int nb = jac_nb(d), dp = nb * JC;
  double* G = work;
  double* V = G + (size_t)d * dp;
  double* nrm = V + (size_t)dp * dp;
  unsigned* ctl = jac_ctl(work, d);
  {
    // register path: blocks of JC columns, one CTA per block pair; the
    // cyclic-by-blocks sweep has ~d inner rounds whatever JC, so JC trades
    // per-round overheads (grid barrier, G / V traffic) against CTA count
    const int jc = g_jacobi_jc;
    if (jc == 4 && reg_launch<4>(B, d, Ub, S, Vb, work, ctl, st)) return;
    if (jc == 8 && reg_launch<8>(B, d, Ub, S, Vb, work, ctl, st)) return;
  }
  jacobi_init_kernel<<<148 * 4, 256, 0, st>>>(B, d, dp, G, V, ctl, nullptr);
  jacobi_fro_kernel<<<1, 1024, 0, st>>>(B, d, reinterpret_cast<double*>(ctl + 8));
  TSVD_CHECK_LAUNCH();
  const size_t smem = sizeof(double) * ((size_t)d * JP + 2 * JW * JP);
  static int attr_for = -1;
  if (attr_for < (int)smem) {
    TSVD_CUDA(cudaFuncSetAttribute(jacobi_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    attr_for = (int)smem;
  }
  int nblocks = nb / 2;
  int nbv = nb;
  void* args[] = {&G, &V, &d, &nbv, &nrm, &Ub, &S, &Vb, &ctl};
  TSVD_CUDA(cudaLaunchCooperativeKernel((void*)jacobi_block_kernel, dim3(nblocks), dim3(256), args,
                                        smem, st));
  TSVD_CHECK_LAUNCH();
}

}  // namespace tsvd
