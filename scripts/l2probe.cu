// L2 / gather bandwidth probe on the B200 (what bounds the SpMM gathers).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2probe scripts/l2probe.cu
// (a) coalesced 16-byte reads of an L2-resident buffer, (b) random 128- and
// 256-byte row gathers (one row per 8 / 16 lanes, double2 per lane) from an
// L2-resident table and (c) from a table far larger than L2.  Bytes moved /
// CUDA-event time, best of 5.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void read_kernel(const double2* __restrict__ p, size_t n, int reps, double* out) {
  double a = 0.0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
      const double2 v = __ldcg(p + i);
      a += v.x + v.y;
    }
  if (a == 12345.678) out[0] = a;
}

// LPR lanes per row (double2 each), U independent rows in flight per group
template <int LPR, int U>
__global__ void gather_kernel(const double2* __restrict__ tab, int64_t rows,
                              const int32_t* __restrict__ idx, int64_t nidx, double* out) {
  const int g = threadIdx.x / LPR, ln = threadIdx.x % LPR;
  const int64_t ng = (int64_t)gridDim.x * (blockDim.x / LPR);
  double a = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)(blockDim.x / LPR) + g; k < nidx; k += U * ng) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t kk = k + u * ng;
      v[u] = kk < nidx ? __ldg(tab + (int64_t)idx[kk] * LPR + ln) : make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) a += v[u].x + v[u].y;
  }
  if (a == 12345.678) out[0] = a;
}

template <class F>
static float best_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r > 0 && ms < best) best = ms;
  }
  return best;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  {  // (a) L2-resident coalesced reads
    for (size_t mb : {16, 48, 96}) {
      const size_t n = mb * (1 << 20) / 16;
      double2* p;
      cudaMalloc(&p, n * 16);
      cudaMemset(p, 0, n * 16);
      const int reps = 20;
      float ms = best_ms([&] { read_kernel<<<148 * 8, 512>>>(p, n, reps, out); });
      printf("coalesced read %zu MB x%d: %.1f GB/s\n", mb, reps, (double)n * 16 * reps / ms / 1e6);
      cudaFree(p);
    }
  }
  const int64_t nidx = 10'000'000;
  std::vector<int32_t> h(nidx);
  uint64_t x = 88172645463325252ULL;
  for (auto tab_mb : {32, 96, 2048}) {
    for (int rowb : {128, 256}) {
      const int64_t rows = (int64_t)tab_mb * (1 << 20) / rowb;
      for (auto& v : h) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        v = (int32_t)(x % rows);
      }
      int32_t* di;
      double2* tab;
      cudaMalloc(&di, nidx * 4);
      cudaMalloc(&tab, rows * rowb);
      cudaMemset(tab, 0, rows * rowb);
      cudaMemcpy(di, h.data(), nidx * 4, cudaMemcpyHostToDevice);
      float ms;
      if (rowb == 128)
        ms = best_ms([&] { gather_kernel<8, 8><<<148 * 8, 256>>>(tab, rows, di, nidx, out); });
      else
        ms = best_ms([&] { gather_kernel<16, 8><<<148 * 8, 256>>>(tab, rows, di, nidx, out); });
      printf("random %d-byte row gather, table %d MB: %.3f ms, %.1f GB/s of rows (+%.1f GB/s idx)\n",
             rowb, tab_mb, ms, (double)nidx * rowb / ms / 1e6, (double)nidx * 4 / ms / 1e6);
      cudaFree(di);
      cudaFree(tab);
    }
  }
  return 0;
}
