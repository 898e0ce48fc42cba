// K2a tile POTRF, K2b panel TRSM and the 32x32 diagonal-block inverses.
//
// Replaces the LAPACK calls inside the reference's block sweep:
//   la.cholesky(A_JJ)                       bg/distla/kernels.py:146-148
//   solve_triangular(L_JJ, A_IJ^T)^T        bg/distla/kernels.py:163-164
// and the diagonal TRSM inside solve_rect (kernels.py:304-306).
//
// tile_potrf: one CTA factors a b x b diagonal tile held in global memory
// (it is L2-resident: the trailing update just wrote it).  Right-looking with
// 32-wide sub-panels: warp 0 factors the 32x32 diagonal block in registers
// (lane = row, shuffles), warp 1 inverts it, all threads apply the inverse to
// the sub-panel below, and the in-tile trailing update runs on FP64 DMMA with
// both operands in shared memory.  The first non-positive (or NaN) pivot
// records its 1-based global row in *info and stops the factorization.
//
// panel_trsm: X = A L^{-T} for a column of b x b tiles.  One CTA owns a
// 32-row slab of one tile in shared memory and sweeps the 32-wide column
// blocks: X_k = S_k Dinv_k^T, then S_{>k} -= X_k L_{>k,k}^T.
#include "bgp_common.cuh"
#include "bgp_internal.h"
#include "panel_device.cuh"

namespace bgp {

size_t potrf_smem_bytes(int b) { return (size_t)(2 * NB * 33 + (b - NB) * PLD + 2 * NB + 2) * sizeof(double); }

__global__ void __launch_bounds__(POTRF_THREADS, 1)
    tile_potrf_kernel(double* __restrict__ A, int b, int64_t row0, double* __restrict__ dinv,
                      unsigned long long* __restrict__ info, const int* __restrict__ gate, int gate_need) {
  extern __shared__ double sm[];
  __shared__ int s_skip;
  const int tid = threadIdx.x;
  if (info && *(volatile unsigned long long*)info != 0ull) return;  // an earlier step failed
  if (tid == 0) {
    s_skip = 0;
    // gate: a concurrently running trailing update signals when every block
    // of this tile has been reduced into L2 (release/acquire)
    if (gate) {
      unsigned ns = 64;
      long long spins = 0;
      while (ld_acquire_gpu(gate) < gate_need) {
        if (*(volatile unsigned long long*)info != 0ull) {
          s_skip = 1;
          break;
        }
        if (++spins > (1ll << 24)) {  // ~minutes: a broken dependency, not a slow GPU
          set_info(info, (long long)BGP_INFO_DATAFLOW_TIMEOUT);
          s_skip = 1;
          break;
        }
        __nanosleep(ns);
        if (ns < 2048) ns <<= 1;
      }
    }
  }
  __syncthreads();
  if (s_skip) return;
  tile_potrf_device(A, b, row0, dinv, info, sm, tid, 0);
}

// Full inverse of a factored diagonal tile, Linv = L^{-1} (column-major b x b,
// zero strict upper triangle), from its 32x32 diagonal-block inverses:
//   Linv[i][j] = -Dinv_i * sum_{m=j}^{i-1} L[i][m] Linv[m][j]     (i > j)
// One CTA per 32-wide column block j; it keeps its column of Linv blocks in
// shared memory.  Feeds the panel TRSM on the DMMA GEMM (X = A Linv^T).
__global__ void __launch_bounds__(256) tri_inv_kernel(const double* __restrict__ L,
                                                      const double* __restrict__ dinv, int b,
                                                      double* __restrict__ Linv, int* __restrict__ done) {
  extern __shared__ double xs[];  // Linv blocks (i, j), i >= j: [(i-j)*32 + r]*33 + c
  double* tmp = xs + (size_t)(b / NB) * NB * 33;  // 32 x 33
  const int j = blockIdx.x, nbk = b / NB;
  const int tid = threadIdx.x, r = tid & 31, c8 = tid >> 5;
  for (int idx = tid; idx < NB * NB; idx += blockDim.x) {
    const int c = idx >> 5, rr = idx & 31;
    xs[rr * 33 + c] = dinv[(int64_t)j * NB * NB + idx];
  }
  __syncthreads();
  for (int i = j + 1; i < nbk; ++i) {
    double sacc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int m = j; m < i; ++m) {
      const double* Xm = xs + (size_t)(m - j) * NB * 33;
#pragma unroll 8
      for (int q = 0; q < NB; ++q) {
        const double l = L[(int64_t)(m * NB + q) * b + i * NB + r];
#pragma unroll
        for (int u = 0; u < 4; ++u) sacc[u] = fma(l, Xm[q * 33 + c8 + 8 * u], sacc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) tmp[r * 33 + c8 + 8 * u] = sacc[u];
    __syncthreads();
    const double* Di = dinv + (int64_t)i * NB * NB;  // column-major: (r, q) at q*32 + r
    double* Xi = xs + (size_t)(i - j) * NB * 33;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c8 + 8 * u;
      double v = 0.0;
#pragma unroll 8
      for (int q = 0; q < NB; ++q) v = fma(Di[q * NB + r], tmp[q * 33 + c], v);
      Xi[r * 33 + c] = -v;
    }
    __syncthreads();
  }
  // column block j of Linv: rows < 32j are zero
  for (int idx = tid; idx < NB * b; idx += blockDim.x) {
    const int c = idx / b, row = idx % b;
    const int blk = row / NB;
    const double v = (blk < j) ? 0.0 : xs[((size_t)(blk - j) * NB + (row & 31)) * 33 + c];
    Linv[(int64_t)(j * NB + c) * b + row] = v;
  }
  if (done) {  // publish: the fused panel TRSM of the trailing update waits for all column blocks
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicAdd(done, 1);
  }
}

// Single-CTA inverse of a factored diagonal tile for the look-ahead stream
// (where only one SM is free): Linv = L^{-1} by block diagonals.  Diagonal
// d holds the blocks (j + d, j); each is
//   Linv[j+d][j] = -Dinv_{j+d} * sum_{m=j}^{j+d-1} L[j+d][m] Linv[m][j]
// and only needs diagonals < d, so all blocks of a diagonal are independent.
// Both products run on DMMA with fragments loaded from L2 (the tile was just
// factored); the partial sums of a diagonal are staged in shared memory.
size_t tri_inv_smem_bytes() { return (size_t)(TINV_THREADS / 32) * NB * 33 * sizeof(double); }

__global__ void __launch_bounds__(TINV_THREADS, 1)
    tri_inv_diag_kernel(const double* __restrict__ L, const double* __restrict__ dinv, int b,
                        double* __restrict__ Linv, int* __restrict__ done) {
  extern __shared__ double S[];
  tri_inv_diag_device(L, dinv, b, Linv, S, threadIdx.x, 0);
  if (done) {  // publish: the fused panel TRSM of the trailing update waits for this
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(done, b / NB);
  }
}

// inverses of the 32x32 diagonal sub-blocks of every diagonal tile of a packed
// triangle; zero diagonal -> info (SingularDiagonal, kernels.py:245-246)
__global__ void diag_inv_kernel(const double* __restrict__ L, int T, int b, int64_t n,
                                double* __restrict__ dinv, unsigned long long* __restrict__ info) {
  __shared__ double D[NB * 33];
  __shared__ double Dinv_s[NB * 33];
  const int nbk = b / NB;
  const int J = blockIdx.x / nbk, kb = blockIdx.x % nbk;
  const int lane = threadIdx.x;
  const double* tile = L + tri_index(J, J, T) * (int64_t)b * b;
  const int c0 = kb * NB;
#pragma unroll 4
  for (int j = 0; j < NB; ++j)
    D[lane * 33 + j] = (j <= lane) ? tile[(int64_t)(c0 + j) * b + c0 + lane] : 0.0;
  __syncwarp();
  const int64_t grow = (int64_t)J * b + c0 + lane;
  const bool zero = (D[lane * 33 + lane] == 0.0) && grow < n;
  const unsigned z = __ballot_sync(FULL, zero);
  if (z) {
    if (lane == 0) set_info(info, (int64_t)J * b + c0 + __ffs(z));
    return;
  }
  warp_trinv32(D, nullptr, Dinv_s, dinv + ((int64_t)J * nbk + kb) * NB * NB, lane);
}

// X = A L^{-T} (trans = 0) for `count` consecutive b x b tiles.
constexpr int TRSM_THREADS = 256;
constexpr int TRSM_R = 32;     // slab rows
constexpr int TRSM_CH = 64;    // staged L rows per update chunk

__global__ void __launch_bounds__(TRSM_THREADS, 2)
    panel_trsm_kernel(const double* __restrict__ Ld, const double* __restrict__ dinv,
                      double* __restrict__ Abase, int b, const unsigned long long* __restrict__ info) {
  extern __shared__ double sm[];
  double* S = sm;                       // b cols x TRSM_R rows, S[c*R + r]
  double* Lc = S + (int64_t)b * TRSM_R;   // TRSM_CH x 33
  double* Di = Lc + TRSM_CH * 33;       // 32 x 33
  if (info && *(volatile const unsigned long long*)info != 0ull) return;
  const int slabs = b / TRSM_R;
  const int64_t t = blockIdx.x / slabs;
  const int r0 = (blockIdx.x % slabs) * TRSM_R;
  double* A = Abase + t * (int64_t)b * b;
  const int tid = threadIdx.x, r = tid & 31, cw = tid >> 5;
  // load slab (coalesced: 32 consecutive rows per column)
  for (int idx = tid; idx < b * TRSM_R; idx += TRSM_THREADS) {
    const int c = idx / TRSM_R, rr = idx % TRSM_R;
    S[idx] = A[(int64_t)c * b + r0 + rr];
  }
  const int nbk = b / NB;
  for (int kb = 0; kb < nbk; ++kb) {
    const int c0 = kb * NB;
    // stage Dinv_k (column-major in global) as Di[j*33 + k] = Dinv[j][k]
    for (int idx = tid; idx < NB * NB; idx += TRSM_THREADS) {
      const int col = idx / NB, row = idx % NB;
      Di[row * 33 + col] = dinv[(int64_t)kb * NB * NB + idx];
    }
    __syncthreads();
    // X_k = S_k Dinv^T : thread (r, cw) computes columns j = cw + 8u
    double sv[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) sv[k] = S[(c0 + k) * TRSM_R + r];
    double xo[NB / 8];
#pragma unroll
    for (int u = 0; u < NB / 8; ++u) {
      const int j = cw + 8 * u;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < NB; ++k) s = (k <= j) ? fma(sv[k], Di[j * 33 + k], s) : s;
      xo[u] = s;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < NB / 8; ++u) S[(c0 + cw + 8 * u) * TRSM_R + r] = xo[u];
    __syncthreads();
    // X row r into registers
    double x[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) x[k] = S[(c0 + k) * TRSM_R + r];
    // update remaining columns in chunks of TRSM_CH staged L rows
    for (int cb = c0 + NB; cb < b; cb += TRSM_CH) {
      __syncthreads();
      for (int idx = tid; idx < TRSM_CH * NB; idx += TRSM_THREADS) {
        const int k = idx / TRSM_CH, cc = idx % TRSM_CH;  // coalesced over cc
        Lc[cc * 33 + k] = (cb + cc < b) ? Ld[(int64_t)(c0 + k) * b + cb + cc] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < TRSM_CH / 8; ++u) {
        const int cc = cw + 8 * u;
        const int c = cb + cc;
        if (c < b) {
          double s = S[c * TRSM_R + r];
#pragma unroll
          for (int k = 0; k < NB; ++k) s = fma(-x[k], Lc[cc * 33 + k], s);
          S[c * TRSM_R + r] = s;
        }
      }
    }
    __syncthreads();
  }
  for (int idx = tid; idx < b * TRSM_R; idx += TRSM_THREADS) {
    const int c = idx / TRSM_R, rr = idx % TRSM_R;
    A[(int64_t)c * b + r0 + rr] = S[idx];
  }
}

void potrf_prepare() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(tile_potrf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(panel_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(tri_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(tri_inv_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, diag_inv_kernel);
    done = true;
  }
}

int launch_tile_potrf(Ctx* ctx, double* tile, int b, int64_t row0, double* dinv, cudaStream_t s,
                      const int* gate, int gate_need) {
  const size_t smem = potrf_smem_bytes(b);
  potrf_prepare();
  tile_potrf_kernel<<<1, POTRF_THREADS, smem, s>>>(tile, b, row0, dinv, ctx->d_info, gate, gate_need);
  ctx->launches++;
  return check_launch(ctx, "tile_potrf");
}

int launch_tri_inv(Ctx* ctx, const double* Ltile, const double* dinv, int b, double* Linv, cudaStream_t s,
                   int* done, bool one_cta) {
  if (one_cta) {
    tri_inv_diag_kernel<<<1, TINV_THREADS, tri_inv_smem_bytes(), s>>>(Ltile, dinv, b, Linv, done);
    ctx->launches++;
    return check_launch(ctx, "tri_inv_diag");
  }
  const size_t smem = ((size_t)(b / NB) * NB * 33 + NB * 33) * sizeof(double);
  tri_inv_kernel<<<b / NB, 256, smem, s>>>(Ltile, dinv, b, Linv, done);
  ctx->launches++;
  return check_launch(ctx, "tri_inv");
}

int launch_diag_inv(Ctx* ctx, const double* L, int T, int b, int64_t n, double* dinv, cudaStream_t s) {
  diag_inv_kernel<<<T * (b / NB), 32, 0, s>>>(L, T, b, n, dinv, ctx->d_info);
  ctx->launches++;
  return check_launch(ctx, "diag_inv");
}

int launch_panel_trsm(Ctx* ctx, const double* Ld, const double* dinv, double* A, int64_t count, int b,
                      int trans, cudaStream_t s, bool check_info) {
  if (count <= 0) return BGP_OK;
  (void)trans;
  const size_t smem = ((size_t)b * TRSM_R + TRSM_CH * 33 + NB * 33) * sizeof(double);
  potrf_prepare();
  const int64_t grid = count * (b / TRSM_R);
  panel_trsm_kernel<<<(unsigned)grid, TRSM_THREADS, smem, s>>>(Ld, dinv, A, b,
                                                                      check_info ? ctx->d_info : nullptr);
  ctx->launches++;
  return check_launch(ctx, "panel_trsm");
}

}  // namespace bgp
