// Explicit residuals of the returned triplets: Eq. 14
// as corrected by reading R13,
//   e_i = ||A v_i - sigma_i u_i||_2 / sigma_1,   R_i = ||A v_i - sigma_i u_i||_2 / sigma_i,
// computed with the library's own products (apply: CSR SpMM or the dense
// gemm_nn, multi-GPU all-gather of V's n-shards included) and a column-norm
// kernel with a fixed-order reduction, so the acceptance numbers of bench.py
// and the tests come from the same kernels the solve uses.
//
// Columns go in chunks of <= 32 through the pass scratch buffer (m x 32,
// already sized by the solvers), so the check also runs when U, V were formed
// in place over the bases (C5 on one GPU).
#include <algorithm>
#include <cmath>

#include "ctx.h"

namespace tsvd {

constexpr int kResCtas = 148 * 2;

// part[cta * 32 + j] = sum over this CTA's rows of (Z[i, j] - s_j U[i, j])^2;
// 256 threads = 8 row lanes x 32 columns; rows strided by CTA, fixed order.
__global__ void __launch_bounds__(256) resid_colnorm_kernel(
    const double* __restrict__ Z, int64_t ldz, const double* __restrict__ U, int64_t ldu,
    const double* __restrict__ S, int64_t q, int w, double* __restrict__ part) {
  __shared__ double red[8][33];
  const int j = threadIdx.x & 31, rl = threadIdx.x >> 5;
  const int64_t per = (q + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(q, r0 + per);
  double a0 = 0.0, a1 = 0.0;
  if (j < w) {
    const double s = S[j];
    int64_t i = r0 + rl;
    for (; i + 8 < r1; i += 16) {
      const double d0 = Z[i * ldz + j] - s * U[i * ldu + j];
      const double d1 = Z[(i + 8) * ldz + j] - s * U[(i + 8) * ldu + j];
      a0 = fma(d0, d0, a0);
      a1 = fma(d1, d1, a1);
    }
    if (i < r1) {
      const double d0 = Z[i * ldz + j] - s * U[i * ldu + j];
      a0 = fma(d0, d0, a0);
    }
  }
  red[rl][j] = a0 + a1;
  __syncthreads();
  if (rl == 0) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][j];
    part[(int64_t)blockIdx.x * 32 + j] = t;
  }
}

void residuals(Ctx& c, double* e_host, double* rel_host) {
  if (!c.have) throw Error{TSVD_ESTATE, "tsvd_residuals: no results"};
  const int r = c.r;
  const int64_t m = c.m;
  double* Z = dbuf(c, "scratch", (size_t)std::max(c.m, c.n) * 32);
  double* part = dbuf(c, "resid_part", (size_t)kResCtas * 32);
  double* sums = dbuf(c, "resid_sums", (size_t)((r + 31) / 32) * 32);
  for (int c0 = 0; c0 < r; c0 += 32) {
    const int w = std::min(32, r - c0);
    apply(c, false, c.V + c0, c.ldV, Z, w, w);            // A v_i (this rank's rows)
    if (m > 0) {
      resid_colnorm_kernel<<<kResCtas, 256, 0, c.st>>>(Z, w, c.U + c0, c.ldU, c.S + c0, m, w,
                                                       part);
      TSVD_CHECK_LAUNCH();
      reduce_partials(part, kResCtas, 32, sums + c0, c.st);
    } else {
      fill_zero(sums + c0, 32, c.st);
    }
  }
  allreduce_sum(c, sums, (size_t)r);                       // row-sharded partial sums
  std::vector<double> hs(r), hS(r);
  TSVD_CUDA(cudaMemcpyAsync(hs.data(), sums, r * sizeof(double), cudaMemcpyDeviceToHost, c.st));
  TSVD_CUDA(cudaMemcpyAsync(hS.data(), c.S, r * sizeof(double), cudaMemcpyDeviceToHost, c.st));
  TSVD_CUDA(cudaStreamSynchronize(c.st));
  for (int i = 0; i < r; ++i) {
    const double nr = std::sqrt(hs[i]);
    if (e_host) e_host[i] = hS[0] > 0.0 ? nr / hS[0] : nr;
    if (rel_host) rel_host[i] = hS[i] > 0.0 ? nr / hS[i] : nr;
  }
}

}  // namespace tsvd
