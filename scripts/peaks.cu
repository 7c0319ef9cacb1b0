// Box facts: FP64 DFMA and DMMA (mma.sync m8n8k4 f64)
// throughput per GPU, HBM read / copy bandwidth.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/peaks scripts/peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

__global__ void dfma_loop(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
         a6 = a0 + 6, a7 = a0 + 7;
  const double b = 1.0000001, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double d[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) d[k][0] = d[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[k][0]), "+d"(d[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// half the warps run DFMA chains, half DMMA chains: do the pipes add up?
__global__ void mixed_loop(double* out, int iters) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp & 1) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
           a6 = a0 + 6, a7 = a0 + 7;
    const double b = 1.0000001, c = 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
      }
    }
    s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  } else {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double d[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) d[k][0] = d[k][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(d[k][0]), "+d"(d[k][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void read_kernel(const double2* __restrict__ p, size_t n, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(p + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ p, double2* __restrict__ q, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(q + i, __ldcs(p + i));
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 1 << 26));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  // DFMA: blocks x 256 threads x iters x 64 FMA
  {
    const int iters = 20000, blocks = sms * 8;
    dfma_loop<<<blocks, 256>>>(out, 100);
    cudaEventRecord(a);
    dfma_loop<<<blocks, 256>>>(out, iters);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    const double fl = 2.0 * 64.0 * iters * 256.0 * blocks;
    printf("{\"dfma_tflops\": %.2f}\n", fl / (ms * 1e-3) / 1e12);
  }
  {
    const int iters = 20000, blocks = sms * 8;
    dmma_loop<<<blocks, 256>>>(out, 100);
    cudaEventRecord(a);
    dmma_loop<<<blocks, 256>>>(out, iters);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    const double fl = 2.0 * 256.0 * 8.0 * iters * (256.0 / 32.0) * blocks;
    printf("{\"dmma_tflops\": %.2f}\n", fl / (ms * 1e-3) / 1e12);
  }
  for (int bps : {1, 2, 4}) {  // DMMA throughput vs resident warps per SM
    const int iters = 20000, blocks = sms * bps;
    dmma_loop<<<blocks, 256>>>(out, 100);
    cudaEventRecord(a);
    dmma_loop<<<blocks, 256>>>(out, iters);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    const double fl = 2.0 * 256.0 * 8.0 * iters * (256.0 / 32.0) * blocks;
    printf("{\"dmma_tflops_warps_per_sm_%d\": %.2f}\n", 8 * bps, fl / (ms * 1e-3) / 1e12);
  }
  {
    const int iters = 20000, blocks = sms * 8;
    mixed_loop<<<blocks, 256>>>(out, 100);
    cudaEventRecord(a);
    mixed_loop<<<blocks, 256>>>(out, iters);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    // per iteration: DFMA warps 64 FMA x 32 lanes; DMMA warps 8 x 256 FMA
    const double fl = 2.0 * iters * blocks * 4.0 * (64.0 * 32.0 + 8.0 * 256.0);
    printf("{\"mixed_dfma_dmma_tflops\": %.2f}\n", fl / (ms * 1e-3) / 1e12);
  }
  {
    const size_t bytes = (size_t)8 << 30, n = bytes / 16;
    double2 *p, *q;
    CK(cudaMalloc(&p, bytes));
    CK(cudaMalloc(&q, bytes));
    cudaMemset(p, 0, bytes);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      read_kernel<<<sms * 8, 512>>>(p, n, out);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("{\"hbm_read_gbs\": %.1f}\n", bytes / (best * 1e-3) / 1e9);
    best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      copy_kernel<<<sms * 8, 512>>>(p, q, n / 2);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("{\"hbm_copy_gbs\": %.1f}\n", bytes / (best * 1e-3) / 1e9);
  }
  return 0;
}
