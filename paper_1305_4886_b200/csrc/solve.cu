// K3: triangular solves, crossproduct mat-vecs, reductions and data movement.
//
//   trsv (forward / back)   bg/distla/kernels.py:200-250  (solve_vector)
//   trsm_rect_back          bg/distla/kernels.py:253-307  (solve_rect, trans)
//   rowdot (V^T u, diag)    bg/distla/kernels.py:387-418, 461-487
//   logdet / sumsq          bg/distla/kernels.py:493-522
//   pack / unpack / diag    bg/distla/objects.py:83-123, __init__.py:126-151
//   sub                     bg/distla/kernels.py:550-564
// These are HBM-bandwidth or latency bound; the solves stream each L tile
// once with coalesced column reads and keep the solved block in shared memory.
#include "bgp_common.cuh"
#include "bgp_internal.h"

namespace bgp {

constexpr unsigned FULLM = 0xffffffffu;

// ---------------------------------------------------------------------------
// forward: solve L_JJ x_J = r_J in place (one CTA), zero diagonal -> info
__global__ void __launch_bounds__(256) trsv_diag_fwd_kernel(const double* __restrict__ tile, int b,
                                                            int64_t n, int64_t row0, double* __restrict__ xj,
                                                            unsigned long long* __restrict__ info) {
  __shared__ double xs[512];
  __shared__ int s_fail;
  if (*(volatile unsigned long long*)info != 0ull) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_fail = 0;
  for (int i = tid; i < b; i += blockDim.x) xs[i] = xj[i];
  __syncthreads();
  for (int c0 = 0; c0 < b; c0 += 32) {
    if (warp == 0) {
      // lane = row c0+lane; sequential over the 32 columns
      double r = xs[c0 + lane];
      const double dii = tile[(int64_t)(c0 + lane) * b + c0 + lane];
      const unsigned z = __ballot_sync(FULLM, dii == 0.0 && (row0 + c0 + lane) < n);
      if (z) {
        if (lane == 0) {
          set_info(info, row0 + c0 + __ffs(z));
          s_fail = 1;
        }
      } else {
        for (int j = 0; j < 32; ++j) {
          double xjv = 0.0;
          if (lane == j) xjv = r / dii;
          xjv = __shfl_sync(FULLM, xjv, j);
          if (lane == j) r = xjv;
          if (lane > j) r = fma(-tile[(int64_t)(c0 + j) * b + c0 + lane], xjv, r);
        }
        xs[c0 + lane] = r;
      }
    }
    __syncthreads();
    if (s_fail) return;
    for (int i = c0 + 32 + tid; i < b; i += blockDim.x) {
      double acc = xs[i];
#pragma unroll 8
      for (int k = 0; k < 32; ++k) acc = fma(-tile[(int64_t)(c0 + k) * b + i], xs[c0 + k], acc);
      xs[i] = acc;
    }
    __syncthreads();
  }
  for (int i = tid; i < b; i += blockDim.x) xj[i] = xs[i];
}

// forward update: r_I -= L_IJ x_J for I > J (one CTA per tile I)
__global__ void __launch_bounds__(256) trsv_update_fwd_kernel(const double* __restrict__ L, int T, int b,
                                                              int J, double* __restrict__ x,
                                                              const unsigned long long* __restrict__ info) {
  __shared__ double xs[512];
  if (*(volatile const unsigned long long*)info != 0ull) return;
  const int I = J + 1 + blockIdx.x;
  const double* tile = L + tri_index(I, J, T) * (int64_t)b * b;
  for (int i = threadIdx.x; i < b; i += blockDim.x) xs[i] = x[(int64_t)J * b + i];
  __syncthreads();
  for (int i = threadIdx.x; i < b; i += blockDim.x) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int k = 0; k < b; k += 4) {
      a0 = fma(tile[(int64_t)k * b + i], xs[k], a0);
      a1 = fma(tile[(int64_t)(k + 1) * b + i], xs[k + 1], a1);
      a2 = fma(tile[(int64_t)(k + 2) * b + i], xs[k + 2], a2);
      a3 = fma(tile[(int64_t)(k + 3) * b + i], xs[k + 3], a3);
    }
    x[(int64_t)I * b + i] -= (a0 + a1) + (a2 + a3);
  }
}

// back: solve L_JJ^T x_J = r_J in place (one CTA)
__global__ void __launch_bounds__(256) trsv_diag_back_kernel(const double* __restrict__ tile, int b,
                                                             int64_t n, int64_t row0, double* __restrict__ xj,
                                                             unsigned long long* __restrict__ info) {
  __shared__ double xs[512];
  __shared__ int s_fail;
  if (*(volatile unsigned long long*)info != 0ull) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_fail = 0;
  for (int i = tid; i < b; i += blockDim.x) xs[i] = xj[i];
  __syncthreads();
  for (int c0 = b - 32; c0 >= 0; c0 -= 32) {
    if (warp == 0) {
      double r = xs[c0 + lane];
      const double dii = tile[(int64_t)(c0 + lane) * b + c0 + lane];
      const unsigned z = __ballot_sync(FULLM, dii == 0.0 && (row0 + c0 + lane) < n);
      if (z) {
        if (lane == 0) {
          set_info(info, row0 + c0 + 32 - __clz(z));
          s_fail = 1;
        }
      } else {
        for (int j = 31; j >= 0; --j) {
          double xjv = 0.0;
          if (lane == j) xjv = r / dii;
          xjv = __shfl_sync(FULLM, xjv, j);
          if (lane == j) r = xjv;
          // (L^T)[lane][j] = L[j][lane], lane < j
          if (lane < j) r = fma(-tile[(int64_t)(c0 + lane) * b + c0 + j], xjv, r);
        }
        xs[c0 + lane] = r;
      }
    }
    __syncthreads();
    if (s_fail) return;
    for (int i = tid; i < c0; i += blockDim.x) {
      double acc = xs[i];
#pragma unroll 8
      for (int k = 0; k < 32; ++k) acc = fma(-tile[(int64_t)i * b + c0 + k], xs[c0 + k], acc);
      xs[i] = acc;
    }
    __syncthreads();
  }
  for (int i = tid; i < b; i += blockDim.x) xj[i] = xs[i];
}

// back update: r_K -= L_JK^T x_J for K < J (one CTA per tile K, warp per column)
__global__ void __launch_bounds__(256) trsv_update_back_kernel(const double* __restrict__ L, int T, int b,
                                                               int J, double* __restrict__ x,
                                                               const unsigned long long* __restrict__ info) {
  __shared__ double xs[512];
  if (*(volatile const unsigned long long*)info != 0ull) return;
  const int K = blockIdx.x;
  const double* tile = L + tri_index(J, K, T) * (int64_t)b * b;
  for (int i = threadIdx.x; i < b; i += blockDim.x) xs[i] = x[(int64_t)J * b + i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = warp; k < b; k += nw) {
    double acc = 0.0;
    for (int i = lane; i < b; i += 32) acc = fma(tile[(int64_t)k * b + i], xs[i], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULLM, acc, o);
    if (lane == 0) x[(int64_t)K * b + k] -= acc;
  }
}

int launch_trsv(Ctx* ctx, const double* L, int64_t n, int b, double* x, int trans, cudaStream_t s) {
  const int T = (int)((n + b - 1) / b);
  if (!trans) {
    return launch_trsv_fwd_persistent(ctx, L, n, b, x, s);
  } else {
    for (int J = T - 1; J >= 0; --J) {
      trsv_diag_back_kernel<<<1, 256, 0, s>>>(L + tri_index(J, J, T) * (int64_t)b * b, b, n, (int64_t)J * b,
                                              x + (int64_t)J * b, ctx->d_info);
      ctx->launches++;
      if (J > 0) {
        trsv_update_back_kernel<<<J, 256, 0, s>>>(L, T, b, J, x, ctx->d_info);
        ctx->launches++;
      }
    }
  }
  return check_launch(ctx, "trsv");
}

// ---------------------------------------------------------------------------
// y = L x (trans 0) / L^T x (trans 1) / C x for a symmetric C stored as its
// lower triangle (sym 1); one CTA per row block I, fixed J order, so the
// result is deterministic.  mult_vector (bg/distla/kernels.py:313-343) and
// the residual probes of the n = 131,072 checks.
__global__ void __launch_bounds__(256) tri_mv_kernel(const double* __restrict__ L, int T, int b,
                                                     const double* __restrict__ x, double* __restrict__ y,
                                                     int trans, int sym) {
  __shared__ double xs[512];
  __shared__ double red[8][512 / 8 + 1];
  const int I = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double acc0 = 0.0, acc1 = 0.0;  // rows tid, tid + 256
  // lower part: L_IJ x_J for J <= I (trans 0 / sym)
  if (!trans || sym) {
    for (int J = 0; J <= I; ++J) {
      __syncthreads();
      for (int i = tid; i < b; i += blockDim.x) xs[i] = x[(int64_t)J * b + i];
      __syncthreads();
      const double* tile = L + tri_index(I, J, T) * (int64_t)b * b;
      for (int i = tid; i < b; i += blockDim.x) {
        double a = 0.0;
        for (int k = 0; k < b; ++k) a = fma(tile[(int64_t)k * b + i], xs[k], a);
        if (i == tid) acc0 += a; else acc1 += a;
      }
    }
  }
  // transposed part: L_JI^T x_J for J >= I (trans) or J > I (sym, plus the
  // strict upper half of the diagonal tile)
  if (trans || sym) {
    for (int J = I; J < T; ++J) {
      __syncthreads();
      for (int i = tid; i < b; i += blockDim.x) xs[i] = x[(int64_t)J * b + i];
      __syncthreads();
      const double* tile = L + tri_index(J, I, T) * (int64_t)b * b;
      // column k of tile (J, I) dotted with x_J -> output row k of block I
      for (int k = warp; k < b; k += 8) {
        double a = 0.0;
        for (int i = lane; i < b; i += 32) {
          const bool use = (J > I) || (sym ? (i > k) : (i >= k));
          if (use) a = fma(tile[(int64_t)k * b + i], xs[i], a);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(FULLM, a, o);
        if (lane == 0) red[k & 7][k >> 3] = a;
      }
      __syncthreads();
      for (int i = tid; i < b; i += blockDim.x) {
        if (i == tid) acc0 += red[i & 7][i >> 3]; else acc1 += red[i & 7][i >> 3];
      }
    }
  }
  for (int i = tid; i < b; i += blockDim.x) y[(int64_t)I * b + i] = (i == tid) ? acc0 : acc1;
}

int launch_tri_mv(Ctx* ctx, const double* L, int64_t n, int b, const double* x, double* y, int trans, int sym,
                  cudaStream_t s) {
  const int T = (int)((n + b - 1) / b);
  tri_mv_kernel<<<T, 256, 0, s>>>(L, T, b, x, y, trans, sym);
  ctx->launches++;
  return check_launch(ctx, "tri_mv");
}

// ---------------------------------------------------------------------------
// L^T X = B for a transposed rectangular RHS (off the north-star path: one
// thread per RHS column, O(n^2) dot-product substitution, in place)
__global__ void trsm_rect_back_kernel(const double* __restrict__ L, int T, int b, int64_t n,
                                      double* __restrict__ Bt, int64_t m, int Tm,
                                      unsigned long long* __restrict__ info) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= m) return;
  const int A = (int)(a / b), alo = (int)(a % b);
  auto vt = [&](int64_t j) -> double& {
    const int I = (int)(j / b), ilo = (int)(j % b);
    return Bt[((int64_t)I * Tm + A) * b * b + (int64_t)ilo * b + alo];
  };
  auto Lel = [&](int64_t r, int64_t c) -> double {  // r >= c
    const int I = (int)(r / b), J = (int)(c / b);
    return L[tri_index(I, J, T) * (int64_t)b * b + (c % b) * b + (r % b)];
  };
  for (int64_t j = n - 1; j >= 0; --j) {
    double acc = vt(j);
    for (int64_t k = j + 1; k < n; ++k) acc = fma(-Lel(k, j), vt(k), acc);
    const double d = Lel(j, j);
    if (d == 0.0) {
      set_info(info, j + 1);
      return;
    }
    vt(j) = acc / d;
  }
}

int launch_trsm_rect_back(Ctx* ctx, const double* L, int64_t n, int b, double* Bt, int64_t m,
                          cudaStream_t s) {
  const int T = (int)((n + b - 1) / b), Tm = (int)((m + b - 1) / b);
  trsm_rect_back_kernel<<<(unsigned)((m + 127) / 128), 128, 0, s>>>(L, T, b, n, Bt, m, Tm, ctx->d_info);
  ctx->launches++;
  return check_launch(ctx, "trsm_rect_back");
}

// ---------------------------------------------------------------------------
// deterministic block reduction helpers
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLM, v, o);
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  v = 0.0;
  if (warp == 0) {
    v = (lane < NT / 32) ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLM, v, o);
  }
  return v;
}

// tile-list forms for the multi-GPU driver ------------------------------------
int launch_tile_trsv(Ctx* ctx, const double* Ljj, int b, int64_t row0, int64_t n, double* x, int trans,
                     cudaStream_t s) {
  if (!trans) trsv_diag_fwd_kernel<<<1, 256, 0, s>>>(Ljj, b, n, row0, x, ctx->d_info);
  else trsv_diag_back_kernel<<<1, 256, 0, s>>>(Ljj, b, n, row0, x, ctx->d_info);
  ctx->launches++;
  return check_launch(ctx, "tile_trsv");
}

// acc[target] += L_tile x (trans 0) or L_tile^T x (trans 1); items = (tile
// index, target block) pairs with distinct targets
__global__ void __launch_bounds__(256) tile_gemv_kernel(const double* __restrict__ base,
                                                        const int32_t* __restrict__ items, int b,
                                                        const double* __restrict__ xJ,
                                                        double* __restrict__ acc, int trans) {
  __shared__ double xs[512];
  const double* tile = base + (int64_t)items[2 * blockIdx.x] * b * b;
  double* out = acc + (int64_t)items[2 * blockIdx.x + 1] * b;
  for (int i = threadIdx.x; i < b; i += blockDim.x) xs[i] = xJ[i];
  __syncthreads();
  if (!trans) {
    for (int i = threadIdx.x; i < b; i += blockDim.x) {
      double a0 = 0.0, a1 = 0.0;
      for (int k = 0; k < b; k += 2) {
        a0 = fma(tile[(int64_t)k * b + i], xs[k], a0);
        a1 = fma(tile[(int64_t)(k + 1) * b + i], xs[k + 1], a1);
      }
      out[i] += a0 + a1;
    }
  } else {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int k = warp; k < b; k += nw) {
      double a = 0.0;
      for (int i = lane; i < b; i += 32) a = fma(tile[(int64_t)k * b + i], xs[i], a);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(FULLM, a, o);
      if (lane == 0) out[k] += a;
    }
  }
}

int launch_tile_gemv(Ctx* ctx, const double* base, const int32_t* items, int64_t count, int b, const double* xJ,
                     double* partial, int trans, cudaStream_t s) {
  if (count <= 0) return BGP_OK;
  tile_gemv_kernel<<<(unsigned)count, 256, 0, s>>>(base, items, b, xJ, partial, trans);
  ctx->launches++;
  return check_launch(ctx, "tile_gemv");
}

// 2 sum log L_ii over the live rows of listed diagonal tiles (tile index, J)
__global__ void __launch_bounds__(1024) tile_logdet_kernel(const double* __restrict__ base,
                                                           const int32_t* __restrict__ diag, int64_t count, int b,
                                                           int64_t n, double* __restrict__ out,
                                                           unsigned long long* __restrict__ info) {
  __shared__ double sh[32];
  double s = 0.0, c = 0.0;
  const int64_t total = count * b;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    const int64_t k = e / b;
    const int r = (int)(e % b);
    const int64_t row = (int64_t)diag[2 * k + 1] * b + r;
    if (row >= n) continue;
    const double d = base[(int64_t)diag[2 * k] * b * b + (int64_t)r * b + r];
    if (!(d > 0.0)) set_info(info, row + 1);
    const double y = log(d) - c;
    const double t = s + y;
    c = (t - s) - y;
    s = t;
  }
  const double tot = block_sum<1024>(s, sh);
  if (threadIdx.x == 0) out[0] = 2.0 * tot;
}

int launch_tile_logdet(Ctx* ctx, const double* base, const int32_t* diag, int64_t count, int b, int64_t n,
                       cudaStream_t s) {
  tile_logdet_kernel<<<1, 1024, 0, s>>>(base, diag, count, b, n, ctx->d_red, ctx->d_info);
  ctx->launches++;
  return check_launch(ctx, "tile_logdet");
}

// 2 * sum_{i<n} log L_ii; Kahan per thread, fixed-shape tree across threads
__global__ void __launch_bounds__(1024) logdet_kernel(const double* __restrict__ L, int64_t n, int T, int b,
                                                      double* __restrict__ out,
                                                      unsigned long long* __restrict__ info) {
  __shared__ double sh[32];
  double s = 0.0, c = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int I = (int)(i / b), r = (int)(i % b);
    const double d = L[tri_index(I, I, T) * (int64_t)b * b + (int64_t)r * b + r];
    if (!(d > 0.0)) set_info(info, i + 1);
    const double y = log(d) - c;
    const double t = s + y;
    c = (t - s) - y;
    s = t;
  }
  const double tot = block_sum<1024>(s, sh);
  if (threadIdx.x == 0) out[0] = 2.0 * tot;
}

__global__ void __launch_bounds__(1024) sumsq_kernel(const double* __restrict__ x, int64_t n,
                                                     double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0, c = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double y = x[i] * x[i] - c;
    const double t = s + y;
    c = (t - s) - y;
    s = t;
  }
  const double tot = block_sum<1024>(s, sh);
  if (threadIdx.x == 0) out[0] = tot;
}

int launch_logdet(Ctx* ctx, const double* L, int64_t n, int b, cudaStream_t s) {
  const int T = (int)((n + b - 1) / b);
  logdet_kernel<<<1, 1024, 0, s>>>(L, n, T, b, ctx->d_red, ctx->d_info);
  ctx->launches++;
  return check_launch(ctx, "logdet");
}

int launch_sumsq(Ctx* ctx, const double* x, int64_t n, cudaStream_t s) {
  sumsq_kernel<<<1, 1024, 0, s>>>(x, n, ctx->d_red);
  ctx->launches++;
  return check_launch(ctx, "sumsq");
}

// ---------------------------------------------------------------------------
// row dots of a transposed rectangular object (m x n tiles):
//   mode 0: w[a] = sum_i Vt[a][i] u[i]      (V^T u)
//   mode 1: d[a] = sum_i Vt[a][i]^2         (diag V^T V)
// stage 1: partial[I][a] per tile column I; stage 2: ordered sum over I.
__global__ void __launch_bounds__(256) rowdot_partial_kernel(const double* __restrict__ Vt, int Tm, int b,
                                                             const double* __restrict__ u, int mode,
                                                             double* __restrict__ part, int64_t mpad) {
  const int A = blockIdx.x % Tm, I = blockIdx.x / Tm;
  const double* tile = Vt + ((int64_t)I * Tm + A) * b * b;
  for (int r = threadIdx.x; r < b; r += blockDim.x) {
    double a0 = 0.0, a1 = 0.0;
    for (int c = 0; c < b; c += 2) {
      const double v0 = tile[(int64_t)c * b + r], v1 = tile[(int64_t)(c + 1) * b + r];
      if (mode == 0) {
        a0 = fma(v0, u[(int64_t)I * b + c], a0);
        a1 = fma(v1, u[(int64_t)I * b + c + 1], a1);
      } else {
        a0 = fma(v0, v0, a0);
        a1 = fma(v1, v1, a1);
      }
    }
    part[(int64_t)I * mpad + (int64_t)A * b + r] = a0 + a1;
  }
}

__global__ void rowdot_final_kernel(const double* __restrict__ part, int Tn, int64_t mpad,
                                    double* __restrict__ out) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= mpad) return;
  double s = 0.0;
  for (int I = 0; I < Tn; ++I) s += part[(int64_t)I * mpad + a];
  out[a] = s;
}

int launch_rowdot(Ctx* ctx, const double* Vt, int64_t n, int64_t m, int b, const double* u, double* w,
                  cudaStream_t s) {
  const int Tn = (int)((n + b - 1) / b), Tm = (int)((m + b - 1) / b);
  const int64_t mpad = (int64_t)Tm * b;
  int rc = ensure(ctx, (void**)&ctx->d_part, &ctx->part_cap, (size_t)Tn * mpad * sizeof(double));
  if (rc) return rc;
  rowdot_partial_kernel<<<Tn * Tm, 256, 0, s>>>(Vt, Tm, b, u, u ? 0 : 1, ctx->d_part, mpad);
  rowdot_final_kernel<<<(unsigned)((mpad + 255) / 256), 256, 0, s>>>(ctx->d_part, Tn, mpad, w);
  ctx->launches += 2;
  return check_launch(ctx, "rowdot");
}

// ---------------------------------------------------------------------------
// dense row-major <-> packed triangular tiles (32x32 smem transpose)
__global__ void pack_tri_kernel(const double* __restrict__ dense, int64_t n, int64_t ld, int T, int b,
                                double* __restrict__ tiles) {
  __shared__ double sh[32][33];
  int I, J;
  tri_decode(blockIdx.x, T, I, J);
  double* tile = tiles + (int64_t)blockIdx.x * b * b;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int rb = 0; rb < b; rb += 32) {
    for (int cb = 0; cb < b; cb += 32) {
      for (int yy = ty; yy < 32; yy += 8) {
        const int64_t i = (int64_t)I * b + rb + yy, j = (int64_t)J * b + cb + tx;
        double v;
        if (i >= n || j >= n) v = (i == j) ? 1.0 : 0.0;
        else v = (i >= j) ? dense[i * ld + j] : 0.0;
        sh[yy][tx] = v;
      }
      __syncthreads();
      for (int yy = ty; yy < 32; yy += 8) tile[(int64_t)(cb + yy) * b + rb + tx] = sh[tx][yy];
      __syncthreads();
    }
  }
}

__global__ void unpack_tri_kernel(const double* __restrict__ tiles, int64_t n, int T, int b,
                                  double* __restrict__ dense, int64_t ld) {
  __shared__ double sh[32][33];
  int I, J;
  tri_decode(blockIdx.x, T, I, J);
  const double* tile = tiles + (int64_t)blockIdx.x * b * b;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int rb = 0; rb < b; rb += 32) {
    for (int cb = 0; cb < b; cb += 32) {
      for (int yy = ty; yy < 32; yy += 8) sh[yy][tx] = tile[(int64_t)(cb + yy) * b + rb + tx];
      __syncthreads();
      for (int yy = ty; yy < 32; yy += 8) {
        const int64_t i = (int64_t)I * b + rb + yy, j = (int64_t)J * b + cb + tx;
        if (i < n && j < n) dense[i * ld + j] = (i >= j) ? sh[tx][yy] : 0.0;
      }
      __syncthreads();
    }
  }
}

// dense n x m row-major <-> transposed rect tiles (no transpose needed)
__global__ void pack_rect_kernel(const double* __restrict__ dense, int64_t n, int64_t m, int64_t ld, int Tm,
                                 int b, double* __restrict__ tiles) {
  const int A = blockIdx.x % Tm, I = blockIdx.x / Tm;
  double* tile = tiles + (int64_t)blockIdx.x * b * b;
  for (int64_t e = threadIdx.x; e < (int64_t)b * b; e += blockDim.x) {
    const int c = (int)(e / b), r = (int)(e % b);
    const int64_t i = (int64_t)I * b + c, a = (int64_t)A * b + r;
    tile[e] = (i < n && a < m) ? dense[i * ld + a] : 0.0;
  }
}

__global__ void unpack_rect_kernel(const double* __restrict__ tiles, int64_t n, int64_t m, int Tm, int b,
                                   double* __restrict__ dense, int64_t ld) {
  const int A = blockIdx.x % Tm, I = blockIdx.x / Tm;
  const double* tile = tiles + (int64_t)blockIdx.x * b * b;
  for (int64_t e = threadIdx.x; e < (int64_t)b * b; e += blockDim.x) {
    const int c = (int)(e / b), r = (int)(e % b);
    const int64_t i = (int64_t)I * b + c, a = (int64_t)A * b + r;
    if (i < n && a < m) dense[i * ld + a] = tile[e];
  }
}

__global__ void pack_vec_kernel(const double* __restrict__ in, int64_t n, int64_t padded, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < padded; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (i < n) ? in[i] : 0.0;
}

int launch_pack(Ctx* ctx, int kind, const double* dense, int64_t nrow, int64_t ncol, int64_t ld, int b,
                double* tiles, cudaStream_t s) {
  if (kind == BGP_TRI) {
    const int T = (int)((nrow + b - 1) / b);
    pack_tri_kernel<<<(unsigned)tri_count(T), dim3(32, 8), 0, s>>>(dense, nrow, ld, T, b, tiles);
  } else if (kind == BGP_RECT) {
    const int Tn = (int)((nrow + b - 1) / b), Tm = (int)((ncol + b - 1) / b);
    pack_rect_kernel<<<(unsigned)(Tn * Tm), 256, 0, s>>>(dense, nrow, ncol, ld, Tm, b, tiles);
  } else {
    const int64_t padded = ((nrow + b - 1) / b) * b;
    pack_vec_kernel<<<(unsigned)((padded + 255) / 256), 256, 0, s>>>(dense, nrow, padded, tiles);
  }
  ctx->launches++;
  return check_launch(ctx, "pack");
}

int launch_unpack(Ctx* ctx, int kind, const double* tiles, int64_t nrow, int64_t ncol, int b, double* dense,
                  int64_t ld, cudaStream_t s) {
  if (kind == BGP_TRI) {
    const int T = (int)((nrow + b - 1) / b);
    unpack_tri_kernel<<<(unsigned)tri_count(T), dim3(32, 8), 0, s>>>(tiles, nrow, T, b, dense, ld);
  } else if (kind == BGP_RECT) {
    const int Tn = (int)((nrow + b - 1) / b), Tm = (int)((ncol + b - 1) / b);
    unpack_rect_kernel<<<(unsigned)(Tn * Tm), 256, 0, s>>>(tiles, nrow, ncol, Tm, b, dense, ld);
  } else {
    pack_vec_kernel<<<(unsigned)((nrow + 255) / 256), 256, 0, s>>>(tiles, nrow, nrow, dense);
  }
  ctx->launches++;
  return check_launch(ctx, "unpack");
}

__global__ void tri_diag_kernel(const double* __restrict__ L, int64_t n, int T, int b, double* __restrict__ d) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int I = (int)(i / b), r = (int)(i % b);
  d[i] = L[tri_index(I, I, T) * (int64_t)b * b + (int64_t)r * b + r];
}

int launch_tri_diagonal(Ctx* ctx, const double* L, int64_t n, int b, double* d, cudaStream_t s) {
  const int T = (int)((n + b - 1) / b);
  tri_diag_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(L, n, T, b, d);
  ctx->launches++;
  return check_launch(ctx, "tri_diagonal");
}

__global__ void sub_kernel(const double* __restrict__ a, const double* __restrict__ bb, double* __restrict__ out,
                           int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] - bb[i];
}

int launch_sub(Ctx* ctx, const double* a, const double* bb, double* out, int64_t count, cudaStream_t s) {
  if (count <= 0) return BGP_OK;
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  sub_kernel<<<(unsigned)blocks, 256, 0, s>>>(a, bb, out, count);
  ctx->launches++;
  return check_launch(ctx, "sub");
}

// dst = src for `count` doubles (count even, 16-byte aligned): an SM copy,
// which is several times faster on the kriging solve's serial path than a
// device-to-device cudaMemcpyAsync of a few MB
__global__ void copy2_kernel(const double2* __restrict__ src, double2* __restrict__ dst, int64_t n2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __ldcs(src + i);
}

int launch_copy(Ctx* ctx, double* dst, const double* src, int64_t count, cudaStream_t s) {
  if (count <= 0) return BGP_OK;
  if ((count & 1) || ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15))
    return set_err(ctx, "copy: needs 16-byte aligned even counts", cudaErrorInvalidValue);
  const int64_t n2 = count / 2;
  int64_t blocks = (n2 + 255) / 256;
  if (blocks > (int64_t)ctx->num_sms * 8) blocks = (int64_t)ctx->num_sms * 8;
  copy2_kernel<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<const double2*>(src), reinterpret_cast<double2*>(dst),
                                                n2);
  ctx->launches++;
  return check_launch(ctx, "copy");
}

}  // namespace bgp
