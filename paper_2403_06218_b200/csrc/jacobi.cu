// Small projected SVD on the device: one-sided (Hestenes) Jacobi.
// Alg. 1 S5 (SVD of R_p) and Alg. 2 (SVD of B_k, Eq. 9).  The paper runs
// LAPACK GESVD on the host (Table 1); any backward-stable SVD
// gives the same triplets up to signs (reading R20), and keeping it on the
// device removes the PCIe round trip (north_star (4)).
//
// Columns g_p, g_q of G (initially B) are rotated until all pairs are
// orthogonal to |g_p^T g_q| <= sqrt(d) u ||g_p|| ||g_q||; V accumulates the
// rotations.  Then sigma_j = ||g_j||, ubar_j = g_j / sigma_j; sorted
// descending.  Parallel ordering: round-robin tournament, d/2 disjoint pairs
// per round, one warp per pair; rotation of Rutishauser form
//   zeta = (b - a) / (2c), t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)),
//   cs = 1/sqrt(1+t^2), sn = cs t,  [g_p g_q] <- [g_p g_q] [[cs, sn], [-sn, cs]].
#include "internal.h"

namespace tsvd {

size_t small_svd_work(int d) { return 2 * (size_t)d * d + 2 * (size_t)d + 64; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(1024) jacobi_svd_kernel(const double* __restrict__ B, int d,
                                                          double* __restrict__ Ub,
                                                          double* __restrict__ S,
                                                          double* __restrict__ Vb,
                                                          double* __restrict__ work) {
  double* G = work;                    // column-major d x d
  double* V = work + (size_t)d * d;    // column-major d x d
  double* nrm = V + (size_t)d * d;     // d
  __shared__ int rotated;
  __shared__ int sweeps_done;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  for (int64_t i = tid; i < (int64_t)d * d; i += blockDim.x) {
    const int r = (int)(i / d), c = (int)(i % d);
    G[(size_t)c * d + r] = B[i];
    V[(size_t)c * d + r] = (r == c) ? 1.0 : 0.0;
  }
  if (tid == 0) sweeps_done = 0;
  __syncthreads();
  const int ne = d + (d & 1);  // even number of players
  const double tol = sqrt((double)d) * 0x1.0p-53;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < ne - 1; ++round) {
      for (int t = warp; t < ne / 2; t += nw) {
        // circle method: position 0 fixed, others rotate
        int p = (t == 0) ? 0 : ((t - 1 + round) % (ne - 1)) + 1;
        int q = ((ne - 2 - t + round) % (ne - 1)) + 1;
        if (p >= d || q >= d) continue;
        if (p > q) {
          const int tmp = p;
          p = q;
          q = tmp;
        }
        double* gp = G + (size_t)p * d;
        double* gq = G + (size_t)q * d;
        double a = 0.0, b = 0.0, c = 0.0;
        for (int i = lane; i < d; i += 32) {
          const double x = gp[i], y = gq[i];
          a = fma(x, x, a);
          b = fma(y, y, b);
          c = fma(x, y, c);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        c = warp_sum(c);
        if (a == 0.0 || b == 0.0 || !(fabs(c) > tol * sqrt(a) * sqrt(b))) continue;
        const double zeta = (b - a) / (2.0 * c);
        const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + tt * tt);
        const double sn = cs * tt;
        for (int i = lane; i < d; i += 32) {
          const double x = gp[i], y = gq[i];
          gp[i] = cs * x - sn * y;
          gq[i] = sn * x + cs * y;
        }
        double* vp = V + (size_t)p * d;
        double* vq = V + (size_t)q * d;
        for (int i = lane; i < d; i += 32) {
          const double x = vp[i], y = vq[i];
          vp[i] = cs * x - sn * y;
          vq[i] = sn * x + cs * y;
        }
        if (lane == 0) rotated = 1;
      }
      __syncthreads();
    }
    const int any = rotated;
    __syncthreads();
    if (!any) break;
  }
  // norms
  for (int j = warp; j < d; j += nw) {
    const double* gj = G + (size_t)j * d;
    double a = 0.0;
    for (int i = lane; i < d; i += 32) a = fma(gj[i], gj[i], a);
    a = warp_sum(a);
    if (lane == 0) nrm[j] = sqrt(a);
  }
  __syncthreads();
  // rank = position in descending order (ties: lower index first)
  for (int j = warp; j < d; j += nw) {
    const double sj = nrm[j];
    int cnt = 0;
    for (int k = lane; k < d; k += 32) {
      const double sk = nrm[k];
      cnt += (sk > sj || (sk == sj && k < j)) ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    const int rank = cnt;
    const double inv = sj > 0.0 ? 1.0 / sj : 0.0;
    if (lane == 0) S[rank] = sj;
    const double* gj = G + (size_t)j * d;
    const double* vj = V + (size_t)j * d;
    for (int i = lane; i < d; i += 32) {
      Ub[(size_t)i * d + rank] = gj[i] * inv;
      Vb[(size_t)i * d + rank] = vj[i];
    }
  }
}

void small_svd(const double* B, int d, double* Ub, double* S, double* Vb, double* work,
               cudaStream_t st) {
  jacobi_svd_kernel<<<1, 1024, 0, st>>>(B, d, Ub, S, Vb, work);
  TSVD_CHECK_LAUNCH();
}

}  // namespace tsvd
