// Probe: cycles of one warp's 32x32 Cholesky (+ inverse) variants on sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1305_4886_b200/csrc \
//        -o tools/probes/chol32_variants tools/probes/chol32_variants.cu
#include <cmath>
#include <cstdio>
#include <vector>

#include "bgp_common.cuh"
#include "bgp_internal.h"
#include "panel_device.cuh"

using namespace bgp;

// (measured variants, not in the product; in situ none beat the production
// warp_potrf32 + warp_trinv32 -- DESIGN.md section 9)
// branch-free 1 / sqrt(x), x > 0 normal: MUFU seed + one third-order Newton step
__device__ __forceinline__ double rsqrt_pos(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y * y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
}

// Factor the 32x32 diagonal block at Ab (element (r, c) at Ab[c * ld + r]) in
// registers, lane = row.  Every lane also carries the running diagonal d[c]
// (updated with the same FMA as lane c's own a[c], so bit-identical): the
// pivot of column j+1 needs no exchange, and the per-column chain is rsqrt ->
// scale -> one shared-memory broadcast -> FMA.  Column j of L goes to colm
// (colm[j * 33 + r] = L(r, j)), 1 / L_jj to rdiag, and *colcnt is raised to
// cbase + j + 1 after each column for the warp that inverts the block
// alongside (warp_trinv32_follow).  L is written back to Ab at the end unless
// a pivot was not positive; returns the failure bitmask (warp-uniform).  All
// columns are published even on failure, so the follower never waits forever.
__device__ __noinline__ unsigned warp_potrf32_pub(double* Ab, int64_t ld, double* colm, double* rdiag,
                                                  volatile int* colcnt, int cbase, int lane) {
  double a[NB], d[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    a[c] = (c <= lane) ? Ab[(int64_t)c * ld + lane] : 0.0;
    d[c] = Ab[(int64_t)c * ld + c];
  }
  unsigned fail = 0u;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const double piv = d[j];
    const bool ok = piv > 0.0;
    fail |= ok ? 0u : (1u << j);
    const double pv = ok ? piv : 1.0;
    const double r = rsqrt_pos(pv);
    const double l = (lane == j) ? pv * r : (lane > j ? a[j] * r : 0.0);
    colm[j * 33 + lane] = l;
    if (lane == 0) rdiag[j] = r;
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      *colcnt = cbase + j + 1;
    }
#pragma unroll
    for (int c = j + 1; c < NB; ++c) {
      const double lc = colm[j * 33 + c];
      if (lane >= c) a[c] = fma(-l, lc, a[c]);
      d[c] = fma(-lc, lc, d[c]);
    }
  }
  __syncwarp();
  if (!fail) {  // from colm: a[] dies column by column above
#pragma unroll
    for (int c = 0; c < NB; ++c)
      if (c <= lane) Ab[(int64_t)c * ld + lane] = colm[c * 33 + lane];
  }
  __syncwarp();
  return fail;
}

// Inverse of the block warp_potrf32_pub is factoring, one column behind it
// (right-looking: row j of the inverse is final once column j of L is, then
// its multiples leave the rows below), lane = column of the inverse.  Writes
// Dinv_s (row-major, ld 33) and, if given, gout (column-major 32x32).
__device__ __noinline__ void warp_trinv32_follow(const double* colm, const double* rdiag, const volatile int* colcnt,
                                                 int cbase, double* Dinv_s, double* gout, int lane) {
  double s[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) s[c] = (c == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    if (lane == 0)
      while (*colcnt < cbase + j + 1) {
      }
    __syncwarp();
    __threadfence_block();
    const double x = s[j] * rdiag[j];
    s[j] = x;
#pragma unroll
    for (int c = j + 1; c < NB; ++c) s[c] = fma(-colm[j * 33 + c], x, s[c]);
  }
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    Dinv_s[i * 33 + lane] = s[i];
    if (gout) gout[lane * NB + i] = s[i];
  }
}


// V1: warp_potrf32 with the branch-free rsqrt (pivot + column through smem)
__device__ __noinline__ unsigned potrf32_v1(double* A, int b, double* D, double* rdiag, double* col, int lane) {
  double a[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) a[j] = (j <= lane) ? A[(int64_t)j * b + lane] : 0.0;
  unsigned failmask = 0u;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    if (lane == j) col[j] = a[j];
    __syncwarp();
    const double piv = col[j];
    failmask |= (piv > 0.0) ? 0u : (1u << j);
    const double rinv = rsqrt_pos(piv > 0.0 ? piv : 1.0);
    const double ljj = (piv > 0.0 ? piv : 1.0) * rinv;
    if (lane == 0) rdiag[j] = rinv;
    a[j] = (lane == j) ? ljj : ((lane > j) ? a[j] * rinv : 0.0);
    __syncwarp();
    col[lane] = a[j];
    __syncwarp();
#pragma unroll
    for (int c = j + 1; c < NB; ++c)
      if (lane >= c) a[c] = fma(-a[j], col[c], a[c]);
    __syncwarp();
  }
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    D[lane * 33 + j] = (j <= lane) ? a[j] : 0.0;
    if (j <= lane) A[(int64_t)j * b + lane] = a[j];
  }
  __syncwarp();
  return failmask;
}

// V2: running diagonal in every lane (no pivot exchange), column through a
// 32x33 smem matrix, one __syncwarp per column, no publishing
__device__ __noinline__ unsigned potrf32_v2(double* Ab, int64_t ld, double* colm, double* rdiag, int lane) {
  double a[NB], d[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    a[c] = (c <= lane) ? Ab[(int64_t)c * ld + lane] : 0.0;
    d[c] = Ab[(int64_t)c * ld + c];
  }
  unsigned fail = 0u;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const double piv = d[j];
    const bool ok = piv > 0.0;
    fail |= ok ? 0u : (1u << j);
    const double pv = ok ? piv : 1.0;
    const double r = rsqrt_pos(pv);
    const double l = (lane == j) ? pv * r : (lane > j ? a[j] * r : 0.0);
    colm[j * 33 + lane] = l;
    if (lane == 0) rdiag[j] = r;
    __syncwarp();
#pragma unroll
    for (int c = j + 1; c < NB; ++c) {
      const double lc = colm[j * 33 + c];
      if (lane >= c) a[c] = fma(-l, lc, a[c]);
      d[c] = fma(-lc, lc, d[c]);
    }
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < NB; ++c)
    if (c <= lane) Ab[(int64_t)c * ld + lane] = colm[c * 33 + lane];
  __syncwarp();
  return fail;
}

__global__ void __launch_bounds__(64, 1) kern(double* A0, double* out, long long* cyc, int variant, int reps) {
  __shared__ double tile[32 * 32];
  __shared__ double D[32 * 33], Dinv[32 * 33], colm[32 * 33], rdiag[32], col[32];
  __shared__ int cc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long total = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) tile[i] = A0[i];
    if (threadIdx.x == 0) cc = 0;
    __syncthreads();
    long long t0 = clock64();
    if (variant == 0) {  // production: warp_potrf32 + warp_trinv32
      if (warp == 0) {
        warp_potrf32(tile, 32, 0, D, rdiag, col, lane);
        warp_trinv32(D, rdiag, Dinv, out + 2048, lane);
      }
    } else if (variant == 1) {  // V1 + trinv
      if (warp == 0) {
        potrf32_v1(tile, 32, D, rdiag, col, lane);
        warp_trinv32(D, rdiag, Dinv, out + 2048, lane);
      }
    } else if (variant == 2) {  // V2 only
      if (warp == 0) potrf32_v2(tile, 32, colm, rdiag, lane);
    } else if (variant == 3) {  // production potrf only
      if (warp == 0) warp_potrf32(tile, 32, 0, D, rdiag, col, lane);
    } else if (variant == 4) {  // V1 only
      if (warp == 0) potrf32_v1(tile, 32, D, rdiag, col, lane);
    } else if (variant == 5) {  // published V2 + follower inverse (the tile_potrf_device pair)
      if (warp == 0) warp_potrf32_pub(tile, 32, colm, rdiag, &cc, 0, lane);
      else warp_trinv32_follow(colm, rdiag, &cc, 0, Dinv, out + 2048, lane);
    } else if (variant == 6) {  // published V2, no follower
      if (warp == 0) warp_potrf32_pub(tile, 32, colm, rdiag, &cc, 0, lane);
    }
    __syncthreads();
    long long t1 = clock64();
    total += t1 - t0;
  }
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = tile[i];
  if (threadIdx.x == 0) *cyc = total / reps;
}

int main() {
  std::vector<double> h(1024);
  for (int c = 0; c < 32; ++c)
    for (int r = 0; r < 32; ++r) h[c * 32 + r] = (r == c) ? 32.0 : (r > c ? 1.0 / (1 + r - c) : 0.0);
  double *dA, *dO;
  long long* dc;
  cudaMalloc(&dA, 8192);
  cudaMalloc(&dO, 4096 * 8);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dA, h.data(), 8192, cudaMemcpyHostToDevice);
  const char* names[] = {"prod potrf32+trinv32", "v1 (rsqrt_pos)+trinv32", "v2 running diag", "prod potrf32 only",
                         "v1 only", "v2 published + follower inverse", "v2 published, no follower"};
  for (int v = 0; v < 7; ++v) {
    kern<<<1, 64>>>(dA, dO, dc, v, 20);
    long long cyc;
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    std::vector<double> L(1024);
    cudaMemcpy(L.data(), dO, 8192, cudaMemcpyDeviceToHost);
    double res = 0;
    for (int c = 0; c < 32; ++c)
      for (int r = c; r < 32; ++r) {
        double s = 0;
        for (int k = 0; k <= c; ++k) s += L[k * 32 + r] * L[k * 32 + c];
        res = fmax(res, fabs(s - h[c * 32 + r]));
      }
    printf("{\"variant\": %d, \"name\": \"%s\", \"cycles\": %lld, \"resid\": %.2e, \"err\": \"%s\"}\n", v, names[v], cyc,
           res, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
