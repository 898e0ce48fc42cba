// K1: covariance-tile generation.
//
// Replaces distla.construct (bg/distla/kernels.py:35-75), pad_block
// (bg/distla/objects.py:60-80) and the entrywise generators of
// bg/gp/kernels.py:16-172.  One CTA writes one b x b tile; threads own tile
// rows (contiguous in the column-major tile), loop over tile columns, and keep
// the row point in registers and the tile's column points in shared memory, so
// every store is a fully coalesced 2 KB column segment.  The kernel is bound by
// the HBM write stream (8 B per entry) plus one FP64 exp per entry.
//
// Numerics follow numpy's evaluation order exactly (no FMA contraction:
// __dmul_rn/__dadd_rn/__ddiv_rn), so entries match the reference to the ulp
// of exp().
#include "bgp_common.cuh"
#include "bgp_internal.h"

namespace bgp {

constexpr int kMaxDim = 4;

__device__ __forceinline__ double matern_corr(double d, double rho, double sqrt2nu, int nucode) {
  // bg/gp/kernels.py:16-29: s = sqrt(2 nu) * d / rho
  double s = __ddiv_rn(__dmul_rn(sqrt2nu, d), rho);
  double e = exp(-s);
  if (nucode == 0) return e;
  if (nucode == 1) return __dmul_rn(__dadd_rn(1.0, s), e);
  return __dmul_rn(__dadd_rn(__dadd_rn(1.0, s), __ddiv_rn(__dmul_rn(s, s), 3.0)), e);
}

__device__ __forceinline__ double sqexp_corr(double d, double rho) {
  // bg/gp/kernels.py:32-34: exp(-0.5 * (d/rho)**2)
  double t = __ddiv_rn(d, rho);
  return exp(__dmul_rn(-0.5, __dmul_rn(t, t)));
}

// generator value at 0-based global indices (i, j); xi / xj point coordinates
__device__ __forceinline__ double gen_eval(const GenDev& g, const double* xi, const double* xj,
                                           int64_t i, int64_t j) {
  const bool same = (i == j);
  switch (g.family) {
    case BGP_GEN_ZERO:
      return 0.0;
    case BGP_GEN_DELTA:
      return same ? 1.0 : 0.0;
    case BGP_GEN_LINEAR_INDEX:  // i + n*(j-1.0) with 1-based i, j
      return __dadd_rn((double)(i + 1), __dmul_rn(g.p[0], (double)(j + 1) - 1.0));
    case BGP_GEN_WHITE:
      if (g.part == BGP_PART_CROSS) return 0.0;
      return same ? g.p[0] : 0.0;
    default:
      break;
  }
  double k;
  if (g.family == BGP_GEN_PRODUCT) {
    double d1 = fabs(xi[0] - xj[0]);
    double d2 = fabs(xi[1] - xj[1]);
    double c1 = matern_corr(d1, g.p[1], g.sqrt2nu, g.nucode);
    double c2 = matern_corr(d2, g.p[2], g.sqrt2nu2, g.nucode2);
    k = __dmul_rn(g.p[0], __dmul_rn(c1, c2));
  } else {
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < kMaxDim; ++d) {
      if (d < g.dim) {
        double df = xi[d] - xj[d];
        acc = (d == 0) ? __dmul_rn(df, df) : __dadd_rn(acc, __dmul_rn(df, df));
      }
    }
    double dist = __dsqrt_rn(acc);
    double corr = (g.family == BGP_GEN_SQEXP) ? sqexp_corr(dist, g.p[1])
                                              : matern_corr(dist, g.p[1], g.sqrt2nu, g.nucode);
    k = __dmul_rn(g.p[0], corr);
  }
  if (g.nugget && g.part == BGP_PART_COV && same) k = __dadd_rn(k, g.p[g.np - 1]);
  return k;
}

constexpr int kCovThreads = 256;

// triangular: one CTA per lower tile (flat packed index, or an explicit
// (I, J) list for a rank's share of a 2-D block-cyclic distribution)
template <bool kPts>
__global__ void __launch_bounds__(kCovThreads) cov_tri_kernel(GenDev g, const double* __restrict__ X,
                                                              int64_t n, int T, int b,
                                                              double* __restrict__ out,
                                                              const int32_t* __restrict__ tile_ij) {
  extern __shared__ double colpts[];  // b * dim
  int I, J;
  if (tile_ij) {
    I = tile_ij[2 * blockIdx.x];
    J = tile_ij[2 * blockIdx.x + 1];
  } else {
    tri_decode(blockIdx.x, T, I, J);
  }
  const int dim = g.dim;
  const int64_t j0 = (int64_t)J * b, i0 = (int64_t)I * b;
  for (int t = threadIdx.x; t < b * dim; t += blockDim.x) {
    int64_t jj = j0 + t / dim;
    colpts[t] = (kPts && jj < n) ? X[jj * dim + t % dim] : 0.0;
  }
  __syncthreads();
  double* tile = out + (int64_t)blockIdx.x * b * b;
  for (int r = threadIdx.x; r < b; r += blockDim.x) {
    const int64_t i = i0 + r;
    double xi[kMaxDim];
#pragma unroll
    for (int d = 0; d < kMaxDim; ++d) xi[d] = (kPts && d < dim && i < n) ? X[i * dim + d] : 0.0;
    const int cmax = (I == J) ? r : b - 1;
    for (int c = 0; c < b; ++c) {
      const int64_t j = j0 + c;
      double v;
      if (c > cmax) {
        v = 0.0;  // strict upper triangle of a diagonal tile
      } else if (i >= n || j >= n) {
        v = (i == j) ? 1.0 : 0.0;  // identity padding (objects.py:60-80)
      } else {
        v = gen_eval(g, xi, &colpts[c * dim], i, j);
      }
      tile[(int64_t)c * b + r] = v;
    }
  }
}

// rectangular, stored transposed: tile (A, I) of the m x n matrix V^T holds
// gen(i, a) for coords point i (column) and pred point a (row).
template <bool kPts>
__global__ void __launch_bounds__(kCovThreads) cov_rect_kernel(GenDev g, const double* __restrict__ X,
                                                               int64_t n, const double* __restrict__ Y,
                                                               int64_t m, int Tm, int b,
                                                               double* __restrict__ out) {
  extern __shared__ double colpts[];  // b * dim coords points of tile column I
  const int A = blockIdx.x % Tm, I = blockIdx.x / Tm;
  const int dim = g.dim;
  const int64_t i0 = (int64_t)I * b, a0 = (int64_t)A * b;
  for (int t = threadIdx.x; t < b * dim; t += blockDim.x) {
    int64_t ii = i0 + t / dim;
    colpts[t] = (kPts && ii < n) ? X[ii * dim + t % dim] : 0.0;
  }
  __syncthreads();
  double* tile = out + (int64_t)blockIdx.x * b * b;
  for (int r = threadIdx.x; r < b; r += blockDim.x) {
    const int64_t a = a0 + r;
    double ya[kMaxDim];
#pragma unroll
    for (int d = 0; d < kMaxDim; ++d) ya[d] = (kPts && d < dim && a < m) ? Y[a * dim + d] : 0.0;
    for (int c = 0; c < b; ++c) {
      const int64_t i = i0 + c;
      double v = 0.0;
      if (i < n && a < m) v = gen_eval(g, &colpts[c * dim], ya, i, a);
      tile[(int64_t)c * b + r] = v;
    }
  }
}

// vector generators (3-argument form, bg/distla/kernels.py:46-55)
__global__ void cov_vec_kernel(GenDev g, int64_t n, int64_t padded, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < padded;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    if (i < n) {
      if (g.part == BGP_PART_PREDVAR) v = g.p[0];
      else v = 0.0;  // gen.zero (mean functions)
    }
    out[i] = v;
  }
}

int construct(Ctx* ctx, int kind, const GenDev& g, const double* X, int64_t nx, const double* Y,
              int64_t ny, int b, double* out, cudaStream_t s) {
  const size_t smem = (size_t)b * (g.dim > 0 ? g.dim : 1) * sizeof(double);
  if (kind == BGP_TRI) {
    int T = (int)((nx + b - 1) / b);
    if (X)
      cov_tri_kernel<true><<<(unsigned)tri_count(T), kCovThreads, smem, s>>>(g, X, nx, T, b, out, nullptr);
    else
      cov_tri_kernel<false><<<(unsigned)tri_count(T), kCovThreads, smem, s>>>(g, X, nx, T, b, out, nullptr);
  } else if (kind == BGP_RECT) {
    int Tn = (int)((nx + b - 1) / b), Tm = (int)((ny + b - 1) / b);
    const unsigned grid = (unsigned)((int64_t)Tn * Tm);
    if (X && Y)
      cov_rect_kernel<true><<<grid, kCovThreads, smem, s>>>(g, X, nx, Y, ny, Tm, b, out);
    else
      cov_rect_kernel<false><<<grid, kCovThreads, smem, s>>>(g, X, nx, Y, ny, Tm, b, out);
  } else {
    int64_t padded = ((nx + b - 1) / b) * b;
    cov_vec_kernel<<<(unsigned)((padded + 255) / 256), 256, 0, s>>>(g, nx, padded, out);
  }
  ctx->launches++;
  return check_launch(ctx, "construct");
}

int construct_tiles(Ctx* ctx, const GenDev& g, const double* X, int64_t n, int b, const int32_t* tile_ij,
                    int64_t count, double* out, cudaStream_t s) {
  if (count <= 0) return BGP_OK;
  const size_t smem = (size_t)b * (g.dim > 0 ? g.dim : 1) * sizeof(double);
  const int T = (int)((n + b - 1) / b);
  if (X)
    cov_tri_kernel<true><<<(unsigned)count, kCovThreads, smem, s>>>(g, X, n, T, b, out, tile_ij);
  else
    cov_tri_kernel<false><<<(unsigned)count, kCovThreads, smem, s>>>(g, X, n, T, b, out, tile_ij);
  ctx->launches++;
  return check_launch(ctx, "construct_tiles");
}

}  // namespace bgp
