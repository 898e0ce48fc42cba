// Per-rank normal streams for simulation (bg/rng.py:18-28, bg/distla/kernels.py:78-104).
//
// The reference draws N(0,1) deviates as ndtri(U) where U comes from numpy's
// Philox4x64-10 generator keyed by (seed << 64) + rank: one uint64 per double,
// U = (x >> 11) * 2^-53, an exact 0 replaced by 2^-54.  Each element here
// recomputes the Philox block holding its stream position, so a rank's
// stream is reproduced element-parallel and bit-for-bit up to the inverse
// CDF (normcdfinv vs scipy's ndtri: a few ulp).  Stream positions follow the
// reference's block order: blocks column-major over the API layout (padding
// included), elements column-major inside a block.
#include "bgp_common.cuh"
#include "bgp_internal.h"

namespace bgp {

__device__ __forceinline__ uint64_t philox_word(uint64_t pos, uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
  uint64_t c0 = pos / 4 + 1, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += W0;
      k1 += W1;
    }
    const uint64_t hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
    const uint64_t hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  const int w = (int)(pos & 3);
  return w == 0 ? c0 : (w == 1 ? c1 : (w == 2 ? c2 : c3));
}

__device__ __forceinline__ double stream_normal(uint64_t pos, uint64_t k0, uint64_t k1) {
  double u = (double)(philox_word(pos, k0, k1) >> 11) * (1.0 / 9007199254740992.0);
  if (u == 0.0) u = 5.551115123125783e-17;  // 2^-54, as bg/rng.py:15
  return normcdfinv(u);
}

// rectangular n x m object stored as transposed tiles (Tm tile rows);
// vector when m == 0
__global__ void rnorm_kernel(int64_t n, int64_t m, int64_t bs_r, int64_t bs_c, int64_t Br, uint64_t k0,
                             uint64_t k1, uint64_t offset, int b, int Tm, double* __restrict__ out) {
  const int64_t total = n * (m > 0 ? m : 1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (m == 0) {
      out[e] = stream_normal(offset + e, k0, k1);
      continue;
    }
    const int64_t i = e % n, j = e / n;  // element (i, j) of the n x m matrix
    const int64_t I = i / bs_r, r = i % bs_r, J = j / bs_c, c = j % bs_c;
    const uint64_t pos = offset + (uint64_t)((J * Br + I) * bs_r * bs_c + c * bs_r + r);
    const double z = stream_normal(pos, k0, k1);
    const int64_t tI = i / b, tA = j / b;
    out[(tI * Tm + tA) * (int64_t)b * b + (i % b) * b + (j % b)] = z;
  }
}

int launch_rnorm(Ctx* ctx, int64_t n, int64_t m, int64_t bs_r, int64_t bs_c, uint64_t seed, uint64_t rank,
                 uint64_t offset, int b, double* out, cudaStream_t s) {
  const int64_t total = n * (m > 0 ? m : 1);
  const int64_t Br = (n + bs_r - 1) / bs_r;
  const int Tm = m > 0 ? (int)((m + b - 1) / b) : 1;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  rnorm_kernel<<<(unsigned)blocks, 256, 0, s>>>(n, m, bs_r, bs_c, Br, rank, seed, offset, b, Tm, out);
  ctx->launches++;
  return check_launch(ctx, "rnorm");
}

}  // namespace bgp
