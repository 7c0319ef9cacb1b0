// Philox4x32-10 normal start blocks (reading R9).
//
// Independent re-implementation of the counter-based generator (Salmon et
// al., Random123): 10 rounds of
//   (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
//   c' = (hi1^c1^k0, lo1, hi0^c3^k1, lo0),  key += (W0, W1) between rounds.
// Element (i, j) of a q_total x w block, draw t, seed s:
//   key = (lo(s), hi(s)), e = i + j*q_total, ctr = (lo(e), hi(e), lo(t), hi(t))
//   u1 = (((x1:x0) >> 11) + 1) 2^-53, u2 = ((x3:x2) >> 11) 2^-53
//   z = sqrt(-2 ln u1) cos(2 pi u2)
// The index is global and column-major, so a row shard of a block is
// bit-identical to the same rows of the whole block.
#include "internal.h"

namespace tsvd {

__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += W0;
      k1 += W1;
    }
    const uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
    const uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

__global__ void philox_normal_kernel(double* __restrict__ out, int64_t q, int w, int64_t ld,
                                     uint64_t seed, uint64_t draw, int64_t row0,
                                     int64_t q_total) {
  const int64_t total = q * (int64_t)w;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / w;
    const int j = (int)(t - i * w);
    const uint64_t e = (uint64_t)(row0 + i) + (uint64_t)j * (uint64_t)q_total;
    uint32_t c[4] = {(uint32_t)e, (uint32_t)(e >> 32), (uint32_t)draw, (uint32_t)(draw >> 32)};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint64_t a = ((((uint64_t)c[1]) << 32) | c[0]) >> 11;
    const uint64_t b = ((((uint64_t)c[3]) << 32) | c[2]) >> 11;
    const double u1 = ((double)a + 1.0) * 0x1.0p-53;
    const double u2 = (double)b * 0x1.0p-53;
    out[i * ld + j] = sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
  }
}

__global__ void philox_words_kernel(const uint32_t* __restrict__ ctr,
                                    const uint32_t* __restrict__ key, uint32_t* __restrict__ out,
                                    int64_t count) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c[4] = {ctr[4 * t], ctr[4 * t + 1], ctr[4 * t + 2], ctr[4 * t + 3]};
    philox4x32_10(c, key[2 * t], key[2 * t + 1]);
    out[4 * t] = c[0];
    out[4 * t + 1] = c[1];
    out[4 * t + 2] = c[2];
    out[4 * t + 3] = c[3];
  }
}

void launch_philox_normal(double* out, int64_t q, int w, int64_t ld, uint64_t seed,
                          uint64_t draw, int64_t row0, int64_t q_total, cudaStream_t st) {
  const int64_t total = q * (int64_t)w;
  if (total <= 0) return;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  philox_normal_kernel<<<(unsigned)blocks, 256, 0, st>>>(out, q, w, ld, seed, draw, row0,
                                                          q_total);
  TSVD_CHECK_LAUNCH();
}

void launch_philox_words(const uint32_t* ctr, const uint32_t* key, uint32_t* out,
                         int64_t count, cudaStream_t st) {
  if (count <= 0) return;
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  philox_words_kernel<<<(unsigned)blocks, 256, 0, st>>>(ctr, key, out, count);
  TSVD_CHECK_LAUNCH();
}

}  // namespace tsvd
