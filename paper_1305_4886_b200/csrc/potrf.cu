// K2a tile POTRF and tile inverse kernels, the 32x32 diagonal-block
// inverses of a factored triangle, and the FP64 substitution panel TRSM.
//
// Replaces the LAPACK calls inside the reference's block sweep:
//   la.cholesky(A_JJ)                       bg/distla/kernels.py:146-148
//   solve_triangular(L_JJ, A_IJ^T)^T        bg/distla/kernels.py:163-164
// and the diagonal TRSM inside solve_rect (kernels.py:304-306).
//
// tile_potrf_kernel / tri_inv_diag_kernel wrap the device code in
// panel_device.cuh (also run by the look-ahead CTA of the update launch).
// The Cholesky's panel solve itself runs on the DMMA GEMM with the tile
// inverse (gemm.cu); panel_trsm below (one CTA per 32-row slab of a tile,
// X_k = S_k Dinv_k^T, then S_{>k} -= X_k L_{>k,k}^T) serves the kriging
// multi-RHS solve and the multi-GPU tile API.
#include "bgp_common.cuh"
#include "bgp_internal.h"
#include "panel_device.cuh"

namespace bgp {

size_t potrf_smem_bytes(int b) { return (size_t)(2 * NB * 33 + (b - NB) * PLD + 2 * NB + 2) * sizeof(double); }
size_t tri_inv_smem_bytes() { return (size_t)(TINV_THREADS / 32) * NB * 33 * sizeof(double); }
size_t tile_potrf_inv_smem_bytes(int b, bool /*inv: the inverse is fused and needs no extra space*/) {
  return (b <= SMEM_TILE ? (size_t)b * b * sizeof(double) : 0) + potrf_smem_bytes(b);
}

__global__ void __launch_bounds__(POTRF_THREADS, 1)
    tile_potrf_kernel(double* __restrict__ A, int b, int64_t row0, double* __restrict__ dinv,
                      unsigned long long* __restrict__ info, const int* __restrict__ gate, int gate_need,
                      double* __restrict__ Linv) {
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
  tile_potrf_inv_device(A, b, row0, dinv, info, Linv, sm, tid, 0);
}


// Single-CTA inverse of a factored diagonal tile for the look-ahead stream
// (where only one SM is free): Linv = L^{-1} by block diagonals.  Diagonal
// d holds the blocks (j + d, j); each is
//   Linv[j+d][j] = -Dinv_{j+d} * sum_{m=j}^{j+d-1} L[j+d][m] Linv[m][j]
// and only needs diagonals < d, so all blocks of a diagonal are independent.
// Both products run on DMMA with fragments loaded from L2 (the tile was just
// factored); the partial sums of a diagonal are staged in shared memory.
__global__ void __launch_bounds__(TINV_THREADS, 1)
    tri_inv_diag_kernel(const double* __restrict__ L, const double* __restrict__ dinv, int b,
                        double* __restrict__ Linv, int* __restrict__ done) {
  extern __shared__ double S[];
  tri_inv_diag_device<false>(L, dinv, b, Linv, S, threadIdx.x, 0);
  if (done) {  // publish: the fused panel TRSM of the trailing update waits for this
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(done, b / NB);
  }
}

// Inverses of all T diagonal tiles of a factored packed triangle, one CTA
// per tile (the kriging solve's panel steps then run on the DMMA GEMM as
// X = B Linv^T instead of a substitution kernel on the serial path).
__global__ void __launch_bounds__(TINV_THREADS, 1)
    tri_inv_batch_kernel(const double* __restrict__ L, int T, const double* __restrict__ dinv, int b,
                         double* __restrict__ Linv, const unsigned long long* __restrict__ info) {
  extern __shared__ double S[];
  if (info && *(volatile const unsigned long long*)info != 0ull) return;  // singular diagonal found
  const int J = blockIdx.x;
  const int64_t tsz = (int64_t)b * b;
  tri_inv_diag_device<false>(L + tri_index(J, J, T) * tsz, dinv + (int64_t)J * (b / NB) * NB * NB, b,
                             Linv + (int64_t)J * tsz, S, threadIdx.x, 0);
}

int launch_tri_inv_batch(Ctx* ctx, const double* L, int T, const double* dinv, int b, double* Linv,
                         cudaStream_t s) {
  tri_inv_batch_kernel<<<T, TINV_THREADS, tri_inv_smem_bytes(), s>>>(L, T, dinv, b, Linv, ctx->d_info);
  ctx->launches++;
  return check_launch(ctx, "tri_inv_batch");
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
    cudaFuncSetAttribute(tri_inv_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(tri_inv_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, diag_inv_kernel);
    done = true;
  }
}

int launch_tile_potrf(Ctx* ctx, double* tile, int b, int64_t row0, double* dinv, cudaStream_t s,
                      const int* gate, int gate_need, double* Linv) {
  const size_t smem = tile_potrf_inv_smem_bytes(b, Linv != nullptr);
  potrf_prepare();
  tile_potrf_kernel<<<1, POTRF_THREADS, smem, s>>>(tile, b, row0, dinv, ctx->d_info, gate, gate_need, Linv);
  ctx->launches++;
  return check_launch(ctx, "tile_potrf");
}

int launch_tri_inv(Ctx* ctx, const double* Ltile, const double* dinv, int b, double* Linv, cudaStream_t s,
                   int* done) {
  tri_inv_diag_kernel<<<1, TINV_THREADS, tri_inv_smem_bytes(), s>>>(Ltile, dinv, b, Linv, done);
  ctx->launches++;
  return check_launch(ctx, "tri_inv_diag");
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
