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

namespace bgp {

constexpr unsigned FULL = 0xffffffffu;
constexpr int NB = 32;        // sub-panel width
constexpr int PLD = 36;       // smem leading dimension of the panel copy (conflict-free DMMA frags)
constexpr int POTRF_THREADS = 256;

// inverse of a lower-triangular 32x32 block held in smem D (ld 33);
// lane = column of the inverse.  rdiag (smem, optional) holds 1/D[i][i]; the
// dot products use four partial sums to shorten the dependent FMA chain.
// Writes Dinv_s (ld 33) and optionally global (column-major 32x32).
__device__ __forceinline__ void warp_trinv32(const double* D, const double* rdiag, double* Dinv_s, double* gout,
                                             int lane) {
  double x[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) {
      const double t = D[i * 33 + k] * x[k];
      if ((k & 3) == 0) s0 += t;
      else if ((k & 3) == 1) s1 += t;
      else if ((k & 3) == 2) s2 += t;
      else s3 += t;
    }
    const double r = rdiag ? rdiag[i] : 1.0 / D[i * 33 + i];
    x[i] = (i == lane) ? r : ((i > lane) ? -((s0 + s1) + (s2 + s3)) * r : 0.0);
  }
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    Dinv_s[i * 33 + lane] = x[i];
    if (gout) gout[lane * NB + i] = x[i];
  }
}

// Factor the 32x32 diagonal block at (c0, c0) of the tile in global memory
// (warp-wide; lane = row, column j exchanged through smem `col`), store L in
// A and D, 1/L_jj in rdiag.  Returns the failure bitmask (warp-uniform).
__device__ __forceinline__ unsigned warp_potrf32(double* A, int b, int c0, double* D, double* rdiag,
                                                 double* col, int lane) {
  double a[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) a[j] = (j <= lane) ? A[(int64_t)(c0 + j) * b + c0 + lane] : 0.0;
  unsigned failmask = 0u;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    if (lane == j) col[j] = a[j];
    __syncwarp();
    const double piv = col[j];
    failmask |= (piv > 0.0) ? 0u : (1u << j);
    const double rinv = rsqrt(piv > 0.0 ? piv : 1.0);
    const double ljj = (piv > 0.0 ? piv : 1.0) * rinv;
    if (lane == 0) rdiag[j] = rinv;
    a[j] = (lane == j) ? ljj : ((lane > j) ? a[j] * rinv : 0.0);
    __syncwarp();
    col[lane] = a[j];  // column j of L (rows < j hold 0)
    __syncwarp();
#pragma unroll
    for (int c = j + 1; c < NB; ++c)
      if (lane >= c) a[c] = fma(-a[j], col[c], a[c]);
    __syncwarp();
  }
  if (!failmask) {
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      D[lane * 33 + j] = (j <= lane) ? a[j] : 0.0;
      if (j <= lane) A[(int64_t)(c0 + j) * b + c0 + lane] = a[j];
    }
  }
  __syncwarp();
  return failmask;
}

// In-tile trailing update A[i][j] -= sum_k P[i][k] P[j][k] on 8x8 DMMA blocks
// blk in [first, last) of the lower triangle of the `rest` x `rest` trailing
// part (row-major block order), handed out round-robin over `nwarps` warps
// starting at `wid`, four blocks per iteration so the C loads overlap.
__device__ __forceinline__ void tile_trailing(double* A, int b, int base_rc, const double* P, int first,
                                              int last, int wid, int nwarps, int lane) {
  const int q = lane >> 2, s4 = lane & 3;
  constexpr int U = 4;
  for (int base = first + wid * U; base < last; base += nwarps * U) {
    int ibs[U], jbs[U];
    double cv[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int blk = base + u;
      int ib = 0, jb = 0;
      if (blk < last) {
        ib = (int)((sqrtf(8.0f * blk + 1.0f) - 1.0f) * 0.5f);
        while ((ib + 1) * (ib + 2) / 2 <= blk) ++ib;
        while (ib * (ib + 1) / 2 > blk) --ib;
        jb = blk - ib * (ib + 1) / 2;
      }
      ibs[u] = ib;
      jbs[u] = jb;
      const int64_t gr = base_rc + ib * 8 + q;
      const int64_t gc = base_rc + jb * 8 + 2 * s4;
      cv[u][0] = (blk < last) ? A[gc * b + gr] : 0.0;
      cv[u][1] = (blk < last) ? A[(gc + 1) * b + gr] : 0.0;
    }
#pragma unroll
    for (int kk = 0; kk < NB / 4; ++kk) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double av = -P[(ibs[u] * 8 + q) * PLD + kk * 4 + s4];
        const double bv = P[(jbs[u] * 8 + q) * PLD + kk * 4 + s4];
        dmma884(cv[u][0], cv[u][1], av, bv);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (base + u >= last) continue;
      const int64_t gr = base_rc + ibs[u] * 8 + q;
      const int64_t gc = base_rc + jbs[u] * 8 + 2 * s4;
      if (ibs[u] != jbs[u] || gr >= gc) A[gc * b + gr] = cv[u][0];
      if (ibs[u] != jbs[u] || gr >= gc + 1) A[(gc + 1) * b + gr] = cv[u][1];
    }
  }
}

// Right-looking blocked factorization of one b x b tile with 32-wide
// sub-panels and a one-block look-ahead inside the tile: while warps 1..7
// apply sub-panel k's trailing update, warp 0 updates, factors and inverts
// diagonal block k+1, so the serial 32x32 work overlaps the DMMA update.
__global__ void __launch_bounds__(POTRF_THREADS, 1)
    tile_potrf_kernel(double* __restrict__ A, int b, int64_t row0, double* __restrict__ dinv,
                      unsigned long long* __restrict__ info, const int* __restrict__ gate, int gate_need) {
  extern __shared__ double sm[];
  double* D = sm;                // 32 x 33
  double* Dinv_s = D + NB * 33;  // 32 x 33
  double* P = Dinv_s + NB * 33;  // (b - 32) x PLD
  __shared__ double rdiag[NB];
  __shared__ double col[NB];
  __shared__ int s_fail;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (info && *(volatile unsigned long long*)info != 0ull) return;  // an earlier step failed
  if (tid == 0) {
    s_fail = 0;
    // look-ahead gate: the concurrently running trailing update signals when
    // every block of this tile has been reduced into L2 (release/acquire)
    if (gate) {
      unsigned ns = 64;
      long long spins = 0;
      while (ld_acquire_gpu(gate) < gate_need) {
        if (*(volatile unsigned long long*)info != 0ull) {
          s_fail = 1;
          break;
        }
        if (++spins > (1ll << 24)) {  // ~minutes: a broken dependency, not a slow GPU
          set_info(info, (long long)BGP_INFO_DATAFLOW_TIMEOUT);
          s_fail = 1;
          break;
        }
        __nanosleep(ns);
        if (ns < 2048) ns <<= 1;
      }
    }
  }
  __syncthreads();
  if (s_fail) return;
  const int nbk = b / NB;
  // prologue: factor + invert diagonal block 0
  if (warp == 0) {
    const unsigned fm = warp_potrf32(A, b, 0, D, rdiag, col, lane);
    if (fm) {
      if (lane == 0) {
        if (info) set_info(info, row0 + __ffs(fm));
        s_fail = 1;
      }
    } else {
      warp_trinv32(D, rdiag, Dinv_s, dinv, lane);
    }
  }
  __syncthreads();
  if (s_fail) return;
  for (int kb = 0; kb + 1 < nbk; ++kb) {
    const int c0 = kb * NB;
    const int rest = b - c0 - NB;
    // (A) sub-panel X = A[c0+32:, c0:c0+32] Dinv_k^T (in place + smem copy);
    // Dinv is lower triangular with explicit zeros, so every dot is 32 long
    for (int r = tid; r < rest; r += POTRF_THREADS) {
      const int64_t gi = c0 + NB + r;
      double av[NB];
#pragma unroll
      for (int k = 0; k < NB; ++k) av[k] = A[(int64_t)(c0 + k) * b + gi];
#pragma unroll 2
      for (int j = 0; j < NB; ++j) {
        const double* dj = Dinv_s + j * 33;
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int k = 0; k < NB; k += 2) {
          s0 = fma(av[k], dj[k], s0);
          s1 = fma(av[k + 1], dj[k + 1], s1);
        }
        const double x = s0 + s1;
        A[(int64_t)(c0 + j) * b + gi] = x;
        P[r * PLD + j] = x;
      }
    }
    __syncthreads();
    // (B) trailing update; the first 10 blocks are diagonal block k+1
    const int nb8 = rest / 8;
    const int nblk = nb8 * (nb8 + 1) / 2;
    const int base_rc = c0 + NB;
    if (warp == 0) {
      tile_trailing(A, b, base_rc, P, 0, 10, 0, 1, lane);
      __syncwarp();
      __threadfence_block();
      const unsigned fm = warp_potrf32(A, b, base_rc, D, rdiag, col, lane);
      if (fm) {
        if (lane == 0) {
          if (info) set_info(info, row0 + base_rc + __ffs(fm));
          s_fail = 1;
        }
      } else {
        warp_trinv32(D, rdiag, Dinv_s, dinv ? dinv + (int64_t)(kb + 1) * NB * NB : nullptr, lane);
      }
    } else {
      tile_trailing(A, b, base_rc, P, 10, nblk, warp - 1, POTRF_THREADS / 32 - 1, lane);
    }
    __syncthreads();
    if (s_fail) return;
  }
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
constexpr int TINV_THREADS = 256;

// acc (32x32 block as 4x4 8x8 DMMA tiles) += A(32x32) B(32x32): A(r, k) at
// a[k * lda + r], B(k, c) at bm[c * ldb + k] (both column-major, from L2);
// all 64 fragments of a k range are loaded before the 128 DMMAs.
__device__ __forceinline__ void block_mma32(double (&acc)[4][4][2], const double* __restrict__ a, int64_t lda,
                                            const double* __restrict__ bm, int64_t ldb, int lane) {
  const int q = lane >> 2, s4 = lane & 3;
#pragma unroll
  for (int kh = 0; kh < 2; ++kh) {  // two halves of k (16 each) to bound registers
    double av[4][4], bv[4][4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int kk = kh * 16 + 4 * k + s4;
        av[k][t] = __ldcg(a + (int64_t)kk * lda + t * 8 + q);
        bv[k][t] = __ldcg(bm + (int64_t)(t * 8 + q) * ldb + kk);
      }
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int tr = 0; tr < 4; ++tr)
#pragma unroll
        for (int tc = 0; tc < 4; ++tc) dmma884(acc[tr][tc][0], acc[tr][tc][1], av[k][tr], bv[k][tc]);
  }
}

// Single-CTA inverse of a factored diagonal tile for the look-ahead stream
// (where only one SM is free): Linv = L^{-1} by block diagonals.  Diagonal
// d holds the blocks (j + d, j); each is
//   Linv[j+d][j] = -Dinv_{j+d} * sum_{m=j}^{j+d-1} L[j+d][m] Linv[m][j]
// and only needs diagonals < d, so all blocks of a diagonal are independent:
// one warp per 32x32 block, 4x4 DMMA tiles, 64 fragment loads (L2: the tile
// was just factored) in flight per 128 DMMAs.
__global__ void __launch_bounds__(TINV_THREADS, 1)
    tri_inv_diag_kernel(const double* __restrict__ L, const double* __restrict__ dinv, int b,
                        double* __restrict__ Linv, int* __restrict__ done) {
  extern __shared__ double S[];  // per warp: one 32x32 partial sum, [(w*32 + r)*33 + c]
  const int nbk = b / NB;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nw = TINV_THREADS / 32;
  const int q = lane >> 2, s4 = lane & 3;
  // block diagonal = Dinv, strictly upper blocks = 0 (below is written per diagonal)
  for (int idx = tid; idx < b * b; idx += TINV_THREADS) {
    const int c = idx / b, r = idx % b;
    const int bi = r / NB, bj = c / NB;
    if (bi < bj) Linv[idx] = 0.0;
    else if (bi == bj) Linv[idx] = dinv[(int64_t)bj * NB * NB + (c % NB) * NB + (r % NB)];
  }
  __syncthreads();
  double* Sw = S + (size_t)warp * NB * 33;
  for (int d = 1; d < nbk; ++d) {
    for (int j = warp; j < nbk - d; j += nw) {
      const int i = j + d;
      double acc[4][4][2];
#pragma unroll
      for (int tr = 0; tr < 4; ++tr)
#pragma unroll
        for (int tc = 0; tc < 4; ++tc) acc[tr][tc][0] = acc[tr][tc][1] = 0.0;
      // S = sum_m L[i][m] Linv[m][j]
      for (int m = j; m < i; ++m)
        block_mma32(acc, L + (int64_t)(m * NB) * b + i * NB, b, Linv + (int64_t)(j * NB) * b + m * NB, b, lane);
#pragma unroll
      for (int tr = 0; tr < 4; ++tr)
#pragma unroll
        for (int tc = 0; tc < 4; ++tc) {
          Sw[(tr * 8 + q) * 33 + tc * 8 + 2 * s4] = acc[tr][tc][0];
          Sw[(tr * 8 + q) * 33 + tc * 8 + 2 * s4 + 1] = acc[tr][tc][1];
          acc[tr][tc][0] = acc[tr][tc][1] = 0.0;
        }
      __syncwarp();
      // Linv[i][j] = -Dinv_i S   (Dinv column-major 32x32; S row-major, ld 33)
      const double* Di = dinv + (int64_t)i * NB * NB;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        double av[4], bv[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          av[t] = Di[(4 * k + s4) * NB + t * 8 + q];
          bv[t] = Sw[(4 * k + s4) * 33 + t * 8 + q];
        }
#pragma unroll
        for (int tr = 0; tr < 4; ++tr)
#pragma unroll
          for (int tc = 0; tc < 4; ++tc) dmma884(acc[tr][tc][0], acc[tr][tc][1], av[tr], bv[tc]);
      }
      __syncwarp();
#pragma unroll
      for (int tr = 0; tr < 4; ++tr)
#pragma unroll
        for (int tc = 0; tc < 4; ++tc) {
          const int row = i * NB + tr * 8 + q, col = j * NB + tc * 8 + 2 * s4;
          Linv[(int64_t)col * b + row] = -acc[tr][tc][0];
          Linv[(int64_t)(col + 1) * b + row] = -acc[tr][tc][1];
        }
    }
    __syncthreads();  // diagonal d complete before d + 1 reads it
  }
  if (done) {  // publish: the fused panel TRSM of the trailing update waits for this
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicAdd(done, nbk);
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
  const size_t smem = (size_t)(2 * NB * 33 + (b - NB) * PLD) * sizeof(double);
  potrf_prepare();
  tile_potrf_kernel<<<1, POTRF_THREADS, smem, s>>>(tile, b, row0, dinv, ctx->d_info, gate, gate_need);
  ctx->launches++;
  return check_launch(ctx, "tile_potrf");
}

int launch_tri_inv(Ctx* ctx, const double* Ltile, const double* dinv, int b, double* Linv, cudaStream_t s,
                   int* done, bool one_cta) {
  if (one_cta) {
    const size_t smem = (size_t)(TINV_THREADS / 32) * NB * 33 * sizeof(double);
    tri_inv_diag_kernel<<<1, TINV_THREADS, smem, s>>>(Ltile, dinv, b, Linv, done);
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
