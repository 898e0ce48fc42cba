// K1: covariance-tile generation.
//
// Replaces distla.construct (bg/distla/kernels.py:35-75), pad_block
// (bg/distla/objects.py:60-80) and the entrywise generators of
// bg/gp/kernels.py:16-172.  One CTA writes one b x b tile (column-major).
//
// Interior tiles of the 2-D built-in kernels (all but the T diagonal /
// padded ones) take the fast path: a thread owns two adjacent rows, keeps
// their points in registers, reads each column point once from shared
// memory (16-byte loads) and writes both entries of a column with one
// 16-byte store -- a warp stores 512 contiguous bytes per column.  Per entry
// it spends ~17 FP64 instructions: difference and squared distance of
// points pre-scaled by sqrt(2 nu)/rho (so s = sqrt(q) directly), sqrt, and
// exp by a 256-entry table of sigma^2 2^(j/256) (so the variance costs
// nothing) with a one-step reduction, a degree-4 polynomial and
// magic-number rounding (no FP64<->int conversions, no branch).  The
// kernel is bound by the HBM write stream (8 B per entry) and the FP64 issue
// rate together.
//
// Numerics: the generic path (diagonal / padded tiles, other generators)
// follows numpy's evaluation order exactly (no FMA contraction); the fast
// path's entries differ from numpy's by a few ulp (<= 1e-15 absolute for
// entries <= sigma^2; the tests hold them to 1e-14, pkg/tests/test_distla.py:50).
#include "bgp_common.cuh"
#include "bgp_internal.h"

#include <cmath>

namespace bgp {

constexpr int kMaxDim = 4;
#ifndef COV_UNROLL
#define COV_UNROLL 4
#endif
constexpr int kCovUnroll = COV_UNROLL;  // columns per unrolled iteration of the fast path (2 entries each)
#ifndef COV_MIN_BLOCKS
#define COV_MIN_BLOCKS 1
#endif

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

// Fast path for the common generators in 2-D (KIND 1..3: Matern nu = 1/2,
// 3/2, 5/2; KIND 4: squared exponential); KIND 0 is the generic path.
constexpr int kExpTab = 256;
__device__ double kExp2Tab[kExpTab];  // 2^(j/256), host-computed (init_exp_table)

// sigma^2 exp(x) for x <= 0: x 256/ln2 = k + f by magic-number rounding
// (k in the low word of t), exp(x) = 2^(k>>8) 2^((k&255)/256) exp(r),
// r = x - k ln2/256 in one FMA (|r| <= ln2/512; the rounding of ln2/256
// costs |k| 2^-61 ~ |x| 1e-16 relative, i.e. under 4e-17 of the result),
// exp(r) by a degree-4 polynomial (truncation < 4e-17); the table holds
// sigma^2 2^(j/256).  Below 2^-1020 the result is 0 (the reference's exp
// underflows there as well, to within 1e-307).
// constant-bank operands of the fast path's FP64 instructions (an FP64
// immediate must have a zero low word; these do not)
__constant__ double kExpC[4] = {369.3299304675746, -0.0027076061740622863, 1.0 / 24.0, 1.0 / 6.0};
template <bool SAFE>
__device__ __forceinline__ double exp_scaled(double x, const double* __restrict__ tab) {
  const double magic = 6755399441055744.0;  // 1.5 * 2^52
  const double t = fma(x, kExpC[0], magic);  // x 256 / ln2
  const double kd = t - magic;
  const int k = __double2loint(t);
  const double r = fma(kd, kExpC[1], x);
  double p = fma(r, kExpC[2], kExpC[3]);
  p = fma(r, p, 0.5);
  p = fma(r, p, 1.0);
  p = fma(r, p, 1.0);
  const int n = k >> 8;  // k <= 0: arithmetic shift floors
  const double v = tab[k & (kExpTab - 1)] * p;
  const double w = __hiloint2double(__double2hiint(v) + (n << 20), __double2loint(v));
  return (SAFE || n >= -1020) ? w : 0.0;  // SAFE: the host's distance bound rules underflow out
}

// sqrt(q), q >= 0, to ~1 ulp without the library's special-case branch:
// hardware rsqrt seed y, d0 = q y, and one cubic correction of d0 itself,
// d0 (1 + e/2 + 3e^2/8) with e = 1 - d0 y (five FP64 instructions).  q below
// 2^-1022 (coincident points) is raised to 2^-1022 by one integer max on its
// high word: d = 2^-511, which every kernel maps to corr = 1, as for d = 0.
__device__ __forceinline__ double sqrt_fast(double q) {
  q = __hiloint2double(max(__double2hiint(q), 0x00100000), __double2loint(q));
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
  const double d0 = q * y;
  const double e = fma(-d0, y, 1.0);
  return fma(d0 * e, fma(e, 0.375, 0.5), d0);
}

// the fast path's coordinate scale (1 for the generic path, KIND 0)
template <int KIND>
__device__ __forceinline__ double cov_scale(const GenDev& g) {
  if constexpr ((KIND & 7) == 0) return 1.0;
  else return (KIND & 7) == 4 ? 1.0 / g.p[1] : g.sqrt2nu / g.p[1];
}

// sigma^2 * corr(d) for the fast path from q = (sc d)^2, the squared
// distance of points pre-scaled by sc = sqrt(2 nu) / rho (Matern) or 1 / rho
// (squared exponential).  KIND & 7: 1..3 Matern nu = 1/2, 3/2, 5/2, 4 squared
// exponential; KIND & 8: no underflow test (GenDev.safe_exp)
template <int KIND>
__device__ __forceinline__ double cov_fast(double q, const double* __restrict__ tab) {
  constexpr int K = KIND & 7;
  constexpr bool SAFE = (KIND & 8) != 0;
  if (K == 4) {  // bg/gp/kernels.py:32-34: exp(-0.5 (d/rho)^2)
    return exp_scaled<SAFE>(-0.5 * q, tab);
  }
  const double sv = sqrt_fast(q);  // bg/gp/kernels.py:16-29: s = sqrt(2 nu) d / rho
  const double e = exp_scaled<SAFE>(-sv, tab);
  if (K == 1) return e;
  if (K == 2) return fma(sv, e, e);
  return fma(fma(sv, 1.0 / 3.0, 1.0) * sv, e, e);
}

// Fast path of one tile: a thread owns rows r, r+1 (their points in
// registers) over a contiguous share of the columns, reads each column point
// once from shared memory and writes both entries with one 16-byte store.
// DIAG: strict upper triangle zero, nugget where i == j.  PAD: rows / columns
// past n are the identity padding (their point loads are clamped, the values
// masked).
template <int KIND, bool DIAG, bool PAD>
__device__ __forceinline__ void cov_tile_fast(const GenDev& g, const double* __restrict__ X, int64_t n, int b,
                                              int64_t i0, int64_t j0, const double* colpts,
                                              const double* __restrict__ tab, double* tile) {
  const int npairs = b / 2, nsplit = blockDim.x / npairs;
  const int pr = threadIdx.x % npairs, part = threadIdx.x / npairs;
  if (part >= nsplit) return;
  const int r = 2 * pr, cw = b / nsplit, c0 = part * cw;
  const int64_t ia = i0 + r, ib = ia + 1;
  // row points pre-scaled by sc like the column points in shared memory
  // (the scaled difference carries the same ~|x| sc 1e-16 absolute rounding
  // as the reference's unscaled one times sc)
  const double sc = cov_scale<KIND>(g);
  double2 x0 = *reinterpret_cast<const double2*>(X + 2 * (PAD ? min(ia, n - 1) : ia));
  double2 x1 = *reinterpret_cast<const double2*>(X + 2 * (PAD ? min(ib, n - 1) : ib));
  x0.x *= sc, x0.y *= sc, x1.x *= sc, x1.y *= sc;
  const double tau2 = (g.nugget && g.part == BGP_PART_COV) ? g.p[g.np - 1] : 0.0;
  const double2* cp = reinterpret_cast<const double2*>(colpts);
  double2* dst = reinterpret_cast<double2*>(tile + r);
#pragma unroll kCovUnroll
  for (int c = c0; c < c0 + cw; ++c) {
    const double2 pc = cp[c];
    const double ax = x0.x - pc.x, ay = x0.y - pc.y;
    const double bx = x1.x - pc.x, by = x1.y - pc.y;
    double2 v;
    v.x = cov_fast<KIND>(fma(ax, ax, ay * ay), tab);
    v.y = cov_fast<KIND>(fma(bx, bx, by * by), tab);
    if (DIAG) {  // rows r, r+1 of a diagonal tile: lower part, nugget where i == j
      v.x = c > r ? 0.0 : (c == r ? v.x + tau2 : v.x);
      v.y = c > r + 1 ? 0.0 : (c == r + 1 ? v.y + tau2 : v.y);
    }
    if (PAD) {  // identity padding (bg/distla/objects.py:60-80)
      const int64_t j = j0 + c;
      if (ia >= n || j >= n) v.x = (ia == j) ? 1.0 : 0.0;
      if (ib >= n || j >= n) v.y = (ib == j) ? 1.0 : 0.0;
    }
    __stcs(dst + (int64_t)c * (b / 2), v);
  }
}

// triangular: one CTA per lower tile (flat packed index, or an explicit
// (I, J) list for a rank's share of a 2-D block-cyclic distribution)
template <bool kPts, int KIND>
__global__ void __launch_bounds__(kCovThreads, COV_MIN_BLOCKS) cov_tri_kernel(GenDev g, const double* __restrict__ X,
                                                              int64_t n, int T, int b,
                                                              double* __restrict__ out,
                                                              const int32_t* __restrict__ tile_ij) {
  extern __shared__ __align__(16) double colpts[];  // b * dim (fast path: scaled by cov_scale)
  __shared__ double tab[kExpTab];     // fast path: sigma^2 2^(j/256)
  int I, J;
  if (tile_ij) {
    I = tile_ij[2 * blockIdx.x];
    J = tile_ij[2 * blockIdx.x + 1];
  } else {
    tri_decode(blockIdx.x, T, I, J);
  }
  BGP_CHECK(J >= 0 && J <= I && I < T && 2 * b >= blockDim.x);
  const int dim = g.dim;
  const int64_t j0 = (int64_t)J * b, i0 = (int64_t)I * b;
  const double sc = cov_scale<KIND>(g);  // 1 on the generic path
  for (int t = threadIdx.x; t < b * dim; t += blockDim.x) {
    int64_t jj = j0 + t / dim;
    colpts[t] = (kPts && jj < n) ? X[jj * dim + t % dim] * sc : 0.0;
  }
  // interior tiles (no padding, off the diagonal): no per-entry checks
  // every tile of a 2-D built-in kernel takes the fast path (cov_tile_fast);
  // diagonal tiles mask their strict upper triangle and add the nugget,
  // tiles of the last tile row mask the identity padding
  const bool fast = KIND != 0;
  if (fast)
    for (int t = threadIdx.x; t < kExpTab; t += blockDim.x) tab[t] = g.p[0] * kExp2Tab[t];
  __syncthreads();
  double* tile = out + (int64_t)blockIdx.x * b * b;
  if (fast) {
    const bool padded = i0 + b > n || j0 + b > n;
    if (I == J) {
      if (padded) cov_tile_fast<KIND, true, true>(g, X, n, b, i0, j0, colpts, tab, tile);
      else cov_tile_fast<KIND, true, false>(g, X, n, b, i0, j0, colpts, tab, tile);
    } else {
      if (padded) cov_tile_fast<KIND, false, true>(g, X, n, b, i0, j0, colpts, tab, tile);
      else cov_tile_fast<KIND, false, false>(g, X, n, b, i0, j0, colpts, tab, tile);
    }
    return;
  }
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

// fast-path variant for a generator (see cov_fast)
static int cov_kind(const GenDev& g) {
  if (g.dim != 2 || (g.part != BGP_PART_COV && g.part != BGP_PART_CROSS && g.part != BGP_PART_PRED)) return 0;
  if (g.family == BGP_GEN_MATERN && g.nucode >= 0 && g.nucode <= 2) return 1 + g.nucode;
  if (g.family == BGP_GEN_SQEXP) return 4;
  return 0;
}

static void init_exp_table() {
  static bool done = false;
  if (done) return;
  double tab[kExpTab];
  for (int j = 0; j < kExpTab; ++j) tab[j] = (double)exp2l((long double)j / (long double)kExpTab);
  cudaMemcpyToSymbol(kExp2Tab, tab, sizeof(tab));
  done = true;
}

template <bool kPts>
static void launch_cov_tri(const GenDev& g, unsigned grid, size_t smem, cudaStream_t s, const double* X, int64_t n,
                           int T, int b, double* out, const int32_t* tile_ij) {
  init_exp_table();
  const int kind = kPts ? cov_kind(g) : 0;
  switch (kind ? kind + (g.safe_exp ? 8 : 0) : 0) {
#define BGP_COV_CASE(K) \
  case K: cov_tri_kernel<kPts, K><<<grid, kCovThreads, smem, s>>>(g, X, n, T, b, out, tile_ij); break;
    BGP_COV_CASE(1) BGP_COV_CASE(2) BGP_COV_CASE(3) BGP_COV_CASE(4)
    BGP_COV_CASE(9) BGP_COV_CASE(10) BGP_COV_CASE(11) BGP_COV_CASE(12)
#undef BGP_COV_CASE
    default: cov_tri_kernel<kPts, 0><<<grid, kCovThreads, smem, s>>>(g, X, n, T, b, out, tile_ij); break;
  }
}

int construct(Ctx* ctx, int kind, const GenDev& g, const double* X, int64_t nx, const double* Y,
              int64_t ny, int b, double* out, cudaStream_t s) {
  const size_t smem = (size_t)b * (g.dim > 0 ? g.dim : 1) * sizeof(double);
  if (kind == BGP_TRI) {
    int T = (int)((nx + b - 1) / b);
    if (X)
      launch_cov_tri<true>(g, (unsigned)tri_count(T), smem, s, X, nx, T, b, out, nullptr);
    else
      launch_cov_tri<false>(g, (unsigned)tri_count(T), smem, s, X, nx, T, b, out, nullptr);
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
    launch_cov_tri<true>(g, (unsigned)count, smem, s, X, n, T, b, out, tile_ij);
  else
    launch_cov_tri<false>(g, (unsigned)count, smem, s, X, n, T, b, out, tile_ij);
  ctx->launches++;
  return check_launch(ctx, "construct_tiles");
}

}  // namespace bgp
