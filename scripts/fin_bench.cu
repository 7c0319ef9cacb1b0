// Microbenchmark of the Gram finaliser (small.cu) - build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//        -Ipaper_2403_06218_b200/csrc scripts/fin_bench.cu -o scripts/fin_bench
#include "../paper_2403_06218_b200/csrc/small.cu"
#include <cstdio>
#include <vector>
namespace tsvd { std::atomic<long> g_launches{0}; }
template <int MODE>
__global__ void chol_var(const double* __restrict__ Wg, int w, double* L, double* T, int* flag) {
  __shared__ double Xs[32 * 33];
  const int lane = threadIdx.x;
  double a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = (lane < w && k <= lane) ? Wg[lane * w + k] : 0.0;
  int bd = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (j < w) {
      double piv = __shfl_sync(~0u, a[j], j);
      if (!(piv > 0.0) || !isfinite(piv)) { bd = 1; piv = 1.0; }
      double lij;
      if (MODE & 2) {
        const double rs = rsqrt(piv);
        const double ljj = piv * rs;
        lij = lane > j ? a[j] * rs : (lane == j ? ljj : 0.0);
      } else {
        const double ljj = sqrt(piv);
        lij = lane > j ? a[j] / ljj : (lane == j ? ljj : 0.0);
      }
      a[j] = lij;
#pragma unroll
      for (int k = j + 1; k < 16; ++k)
        if (k < w) {
          const double lkj = __shfl_sync(~0u, lij, k);
          if (lane >= k) a[k] = fma(-lij, lkj, a[k]);
        }
    }
  }
  if (MODE & 1) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < w) {
        double v = (i == lane) ? 1.0 : 0.0;
#pragma unroll
        for (int m = 0; m < i; ++m) v = fma(-__shfl_sync(~0u, a[m], i), Xs[m * 33 + lane], v);
        const double lii = __shfl_sync(~0u, a[i], i);
        Xs[i * 33 + lane] = (i >= lane) ? ((MODE & 2) ? v * (1.0 / lii) : v / lii) : 0.0;
      }
    }
    __syncwarp();
    if (lane < w) for (int i = 0; i < w; ++i) T[lane * w + i] = Xs[i * 33 + lane];
  }
  if (lane < w) for (int k = 0; k < w; ++k) L[lane * w + k] = a[k];
  if (lane == 0 && bd) *flag = 1;
}
template <int V>
__global__ void __launch_bounds__(1024) hupd_var(double* H, const double* __restrict__ Hbar, const double* __restrict__ Lprev, int s, int w) {
  __shared__ double Lp[32 * 32];
  extern __shared__ double hbs[];
  const int tid = threadIdx.x;
  const int64_t nh = (int64_t)s * w;
  for (int i = tid; i < w * w; i += 1024) Lp[i] = Lprev[i];
  if (V >= 1) for (int64_t i = tid; i < nh; i += 1024) hbs[i] = Hbar[i];
  __syncthreads();
  if (V == 0) {
    for (int i = tid; i < s * w; i += 1024) {
      const int r = i / w, c = i % w;
      const double* hb = Hbar + (int64_t)r * w;
      double sum = 0.0;
      for (int k = 0; k < w; ++k) sum = fma(hb[k], Lp[c * w + k], sum);
      H[i] += sum;
    }
  } else if (V == 1) {
    for (int64_t i = tid; i < nh; i += 1024) {
      const int r = (int)(i / w), c = (int)(i % w);
      const double* hb = hbs + (int64_t)r * w;
      double sum = 0.0;
      for (int k = 0; k < w; ++k) sum = fma(hb[k], Lp[c * w + k], sum);
      H[i] += sum;
    }
  } else {
    for (int i = tid; i < s * w; i += 1024) {
      const int r = i >> 4, c = i & 15;
      const double* hb = hbs + r * 16;
      double sum = 0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k) sum = fma(hb[k], Lp[c * 16 + k], sum);
      H[i] += sum;
    }
  }
}
__global__ void nop_kernel(int* f) { if (threadIdx.x == 1000) *f = 1; }
using namespace tsvd;
int main() {
  const int w = 16, np = 296, s = 384;
  std::vector<double> h(np * w * w);
  // SPD partials: each partial = I / np + small symmetric noise
  for (int p = 0; p < np; ++p)
    for (int i = 0; i < w; ++i)
      for (int j = 0; j < w; ++j) h[(p * w + i) * w + j] = (i == j ? 1.0 : 0.01 / (1 + i + j)) / np;
  double *g, *W, *L, *T, *L2, *T2, *R, *H, *Hb; int* flag;
  cudaMalloc(&g, h.size() * 8); cudaMemcpy(g, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&W, 1024 * 8); cudaMalloc(&L, 1024 * 8); cudaMalloc(&T, 1024 * 8);
  cudaMalloc(&L2, 1024 * 8); cudaMalloc(&T2, 1024 * 8); cudaMalloc(&R, 1024 * 8);
  cudaMalloc(&H, s * w * 8); cudaMalloc(&Hb, s * w * 8); cudaMalloc(&flag, 16);
  cudaMemset(H, 0, s * w * 8); cudaMemset(Hb, 0, s * w * 8); cudaMemset(flag, 0, 16);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto t = [&](const char* name, auto fn) {
    for (int i = 0; i < 10; ++i) fn();
    cudaEventRecord(a, st);
    for (int i = 0; i < 200; ++i) fn();
    cudaEventRecord(b, st); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %8.2f us\n", name, ms * 1000 / 200);
  };
  t("gram_reduce np=296", [&] { gram_reduce(g, np, w, W, st); });
  t("chol_finalize np=1", [&] { chol_finalize(W, 1, w, L, T, flag, st); });
  t("chol_finalize np=296", [&] { chol_finalize(g, np, w, L, T, flag, st); });
  t("chol2_finalize np=296 s=0", [&] { chol2_finalize(g, np, w, L, L2, T2, R, nullptr, nullptr, 0, flag, st); });
  t("chol2_finalize np=296 s=384", [&] { chol2_finalize(g, np, w, L, L2, T2, R, H, Hb, s, flag, st); });
  // t("chol_var<0> chol only, 32 thr", [&] { chol_var<0><<<1, 32, 0, st>>>(W, w, L, T, flag); });
  t("chol_var<1> chol+inv, 32 thr", [&] { chol_var<1><<<1, 32, 0, st>>>(W, w, L, T, flag); });
  t("chol_var<2> chol rsqrt", [&] { chol_var<2><<<1, 32, 0, st>>>(W, w, L, T, flag); });
  t("chol_var<3> chol+inv rsqrt/rcp", [&] { chol_var<3><<<1, 32, 0, st>>>(W, w, L, T, flag); });
  cudaFuncSetAttribute(hupd_var<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(hupd_var<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  t("hupd_var<0> global", [&] { hupd_var<0><<<1, 1024, 0, st>>>(H, Hb, L, s, w); });
  t("hupd_var<1> smem int64", [&] { hupd_var<1><<<1, 1024, 65536, st>>>(H, Hb, L, s, w); });
  t("hupd_var<2> smem w16 unrolled", [&] { hupd_var<2><<<1, 1024, 65536, st>>>(H, Hb, L, s, w); });
  t("nop 32 thr", [&] { nop_kernel<<<1, 32, 0, st>>>(flag); });
  t("nop 1024 thr", [&] { nop_kernel<<<1, 1024, 0, st>>>(flag); });
  t("empty-ish: copy_block 16x16", [&] { copy_block(L, w, T, w, w, w, 0, st); });
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
