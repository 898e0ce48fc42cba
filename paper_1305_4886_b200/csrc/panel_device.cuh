// Device code of the tile POTRF and the one-CTA tile inverse, shared by the
// standalone kernels (potrf.cu) and the look-ahead CTA of the trailing-update
// launch (gemm.cu).  See potrf.cu for the algorithms.
#pragma once

#include "bgp_common.cuh"
#include "bgp_internal.h"

namespace bgp {

constexpr unsigned FULL = 0xffffffffu;

// BGP_POTRF_TRACE (probe builds only, tools/probes/potrf_trace.cu): lane 0 of
// warps 0 and 1 stamp clock64() at the phase boundaries of tile_potrf_device
#ifdef BGP_POTRF_TRACE
__device__ long long g_ptrace[2][1024];
#define PTRACE()                                                                \
  do {                                                                          \
    if (lane == 0 && warp < 2 && pt_n < 1024) g_ptrace[warp][pt_n] = clock64(); \
    ++pt_n;                                                                     \
  } while (0)
#else
#define PTRACE() \
  do {           \
  } while (0)
#endif
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

// One 32x32 block (bi, bj), bi >= bj, of the in-tile trailing update
// A[i][j] -= sum_k P[i][k] P[j][k] (rows/cols relative to base_rc): all 32
// C values of a lane load at once (one L2 round trip per block instead of
// one per 8x8), then 8 k4-steps of 16 DMMAs with fragments from P in smem.
__device__ __forceinline__ void trail_block32(double* A, int b, int base_rc, const double* P, int bi, int bj,
                                              int lane) {
  const int q = lane >> 2, s4 = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int tr = 0; tr < 4; ++tr)
#pragma unroll
    for (int tc = 0; tc < 4; ++tc)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = bi * 32 + tr * 8 + q, n = bj * 32 + tc * 8 + 2 * s4 + e;
        acc[tr][tc][e] = A[(int64_t)(base_rc + n) * b + base_rc + m];
      }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    double av[4], bv[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      av[t] = -P[(bi * 32 + t * 8 + q) * PLD + 4 * k + s4];
      bv[t] = P[(bj * 32 + t * 8 + q) * PLD + 4 * k + s4];
    }
#pragma unroll
    for (int tr = 0; tr < 4; ++tr)
#pragma unroll
      for (int tc = 0; tc < 4; ++tc) dmma884(acc[tr][tc][0], acc[tr][tc][1], av[tr], bv[tc]);
  }
#pragma unroll
  for (int tr = 0; tr < 4; ++tr)
#pragma unroll
    for (int tc = 0; tc < 4; ++tc)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = bi * 32 + tr * 8 + q, n = bj * 32 + tc * 8 + 2 * s4 + e;
        if (bi != bj || m >= n) A[(int64_t)(base_rc + n) * b + base_rc + m] = acc[tr][tc][e];
      }
}

// acc (32x32 block as 4x4 8x8 DMMA tiles) += A(32x32) B(32x32): A(r, k) at
// a[k * lda + r], B(k, c) at bm[c * ldb + k] (both column-major, from L2);
// all 64 fragments of a k range are loaded before the 128 DMMAs.
template <bool ASMEM>
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
        av[k][t] = ASMEM ? a[(int64_t)kk * lda + t * 8 + q] : __ldcg(a + (int64_t)kk * lda + t * 8 + q);
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

// Right-looking blocked factorization of one b x b tile with 32-wide
// sub-panels and a one-block look-ahead inside the tile: while warps 1..7
// apply sub-panel k's trailing update, warp 0 updates, factors and inverts
// diagonal block k+1, so the serial 32x32 work overlaps the DMMA update.
// Run by 256 threads (tid 0..255) that synchronise on named barrier `bar`;
// `sm` is potrf_smem_bytes(b) of shared memory.  Returns false on a
// non-positive pivot (recorded in *info).  Used by tile_potrf_kernel and,
// for the look-ahead, by one CTA of the trailing-update launch.
// Linv[r][j] = -Dinv_r * S with S stored in Linv[r][j] (32x32 blocks of the
// column-major b x b Linv; Dinv_r column-major 32x32 in global memory): all
// fragments are loaded before the block is overwritten
__device__ __forceinline__ void linv_apply_block(const double* __restrict__ Dr, double* Lrj, int b, int lane) {
  const int q = lane >> 2, s4 = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int tr = 0; tr < 4; ++tr)
#pragma unroll
    for (int tc = 0; tc < 4; ++tc) acc[tr][tc][0] = acc[tr][tc][1] = 0.0;
  block_mma32<false>(acc, Dr, NB, Lrj, b, lane);
  __syncwarp();
#pragma unroll
  for (int tr = 0; tr < 4; ++tr)
#pragma unroll
    for (int tc = 0; tc < 4; ++tc) {
      const int row = tr * 8 + q, col = tc * 8 + 2 * s4;
      Lrj[(int64_t)col * b + row] = -acc[tr][tc][0];
      Lrj[(int64_t)(col + 1) * b + row] = -acc[tr][tc][1];
    }
}

// Row block r of the inverse: Linv[r][r] = Dinv_r (a copy), then
// Linv[r][j] = -Dinv_r S_rj for j < r, S_rj left in Linv[r][j] by
// linv_row_partial.  Blocks dealt to warps first .. first + nwarps - 1.
__device__ __forceinline__ void linv_row_apply(const double* __restrict__ dinv, double* Linv, int b, int r,
                                               int wid, int nwarps, int lane) {
  const double* Dr = dinv + (int64_t)r * NB * NB;
  for (int j = wid; j <= r; j += nwarps) {
    double* Lrj = Linv + (int64_t)(j * NB) * b + r * NB;
    if (j == r) {
      for (int c = 0; c < NB; ++c) Lrj[(int64_t)c * b + lane] = __ldcg(Dr + c * NB + lane);
    } else {
      linv_apply_block(Dr, Lrj, b, lane);
    }
  }
}

// S_rj = sum_{m=j}^{r-1} L[r][m] Linv[m][j] into Linv[r][j] for block j (rows
// < r of Linv final, L's rows up to r complete)
__device__ __forceinline__ void linv_row_partial(const double* __restrict__ L, bool l_smem, double* Linv, int b,
                                                 int r, int j, int lane) {
  const int q = lane >> 2, s4 = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int tr = 0; tr < 4; ++tr)
#pragma unroll
    for (int tc = 0; tc < 4; ++tc) acc[tr][tc][0] = acc[tr][tc][1] = 0.0;
  for (int m = j; m < r; ++m) {
    const double* a = L + (int64_t)(m * NB) * b + r * NB;
    const double* bm = Linv + (int64_t)(j * NB) * b + m * NB;
    if (l_smem) block_mma32<true>(acc, a, b, bm, b, lane);
    else block_mma32<false>(acc, a, b, bm, b, lane);
  }
  double* Lrj = Linv + (int64_t)(j * NB) * b + r * NB;
#pragma unroll
  for (int tr = 0; tr < 4; ++tr)
#pragma unroll
    for (int tc = 0; tc < 4; ++tc) {
      const int row = tr * 8 + q, col = tc * 8 + 2 * s4;
      Lrj[(int64_t)col * b + row] = acc[tr][tc][0];
      Lrj[(int64_t)(col + 1) * b + row] = acc[tr][tc][1];
    }
}

// With Linv (and dinv) given, the inverse L^{-1} is built during the
// factorization, row block by row block, in the warps' idle time: row r's
// partial sums S_rj = sum_m L[r][m] Linv[m][j] need only rows < r of Linv
// and L's rows up to r, so they run in step r-1's trailing phase next to
// the trailing blocks; Linv[r][j] = -Dinv_r S_rj follows in step r's
// sub-panel phase (Dinv_r is produced in step r-1's trailing phase).  (A
// right-looking order -- every step adding its term to all later rows --
// spreads the work more evenly but its read-modify-write of the partial
// sums measured slower.)
// l_smem: A is a shared-memory copy (see tile_potrf_inv_device).
// progress (A in global memory only): after diagonal block k's factor, its
// inverse Dinv_k and L's row block k (all columns < k) are final, the
// counter is raised to k + 1 (release; every thread fences first) -- the
// in-launch substitution panel solve (gemm.cu) consumes the factor that way
// while the factorization is still running.
__device__ __forceinline__ void potrf_publish(int* progress, int v, int tid, int bar) {
  __threadfence();
  named_bar_sync(bar, POTRF_THREADS);
  if (tid == 0) st_release_gpu(progress, v);
}

static __device__ __noinline__ bool tile_potrf_device(double* __restrict__ A, int b, int64_t row0, double* __restrict__ dinv,
                                  unsigned long long* __restrict__ info, double* sm, int tid, int bar,
                                  double* __restrict__ Linv = nullptr, bool l_smem = false,
                                  int* progress = nullptr) {
  double* D = sm;                // 32 x 33
  double* Dinv_s = D + NB * 33;  // 32 x 33
  double* P = Dinv_s + NB * 33;  // (b - 32) x PLD
  double* rdiag = P + (b - NB) * PLD;
  double* col = rdiag + NB;
  int* s_fail = reinterpret_cast<int*>(col + NB);
  const int lane = tid & 31, warp = tid >> 5;
  if (tid == 0) *s_fail = 0;
  const int nbk = b / NB;
#ifdef BGP_POTRF_TRACE
  int pt_n = 0;
#endif
  PTRACE();
  if (Linv) {  // strictly upper blocks of the inverse are zero: warp per column
    for (int c = warp; c < b; c += POTRF_THREADS / 32) {
      double2* colp = reinterpret_cast<double2*>(Linv + (int64_t)c * b);
      for (int r2 = lane; r2 < (c / NB) * NB / 2; r2 += 32) colp[r2] = make_double2(0.0, 0.0);
    }
  }
  named_bar_sync(bar, POTRF_THREADS);
  // prologue: factor + invert diagonal block 0
  if (warp == 0) {
    const unsigned fm = warp_potrf32(A, b, 0, D, rdiag, col, lane);
    if (fm) {
      if (lane == 0) {
        if (info) set_info(info, row0 + __ffs(fm));
        *s_fail = 1;
      }
    } else {
      warp_trinv32(D, rdiag, Dinv_s, dinv, lane);
    }
  }
  PTRACE();
  named_bar_sync(bar, POTRF_THREADS);
  if (*s_fail) return false;
  if (progress) potrf_publish(progress, 1, tid, bar);
  for (int kb = 0; kb + 1 < nbk; ++kb) {
    PTRACE();  // 2 + 6 kb
    const int c0 = kb * NB;
    const int rest = b - c0 - NB;
    // (A) sub-panel X = A[c0+32:, c0:c0+32] Dinv_k^T (in place + smem copy),
    // one 32-row block per warp on DMMA: the lane's 32 A values load at once
    // (one L2 round trip), Dinv (lower triangular, explicit zeros) from smem;
    // the inverse's row block kb is finished by the warps after the last
    // sub-panel block
    if (Linv) {
      const int nA = rest / NB;
      const int w0 = nA % (POTRF_THREADS / 32);  // first warp with no second sub-panel block
      linv_row_apply(dinv, Linv, b, kb, (warp - w0 + POTRF_THREADS / 32) % (POTRF_THREADS / 32),
                     POTRF_THREADS / 32, lane);
    }
    for (int t = warp; t < rest / NB; t += POTRF_THREADS / 32) {
      const int q = lane >> 2, s4 = lane & 3;
      const int r0 = t * NB;  // rows c0 + 32 + r0 .. of the tile
      double av[4][8];
#pragma unroll
      for (int tr = 0; tr < 4; ++tr)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) av[tr][kk] = A[(int64_t)(c0 + 4 * kk + s4) * b + c0 + NB + r0 + tr * 8 + q];
      double acc[4][4][2];
#pragma unroll
      for (int tr = 0; tr < 4; ++tr)
#pragma unroll
        for (int tc = 0; tc < 4; ++tc) acc[tr][tc][0] = acc[tr][tc][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        double bv[4];
#pragma unroll
        for (int tc = 0; tc < 4; ++tc) bv[tc] = Dinv_s[(tc * 8 + q) * 33 + 4 * kk + s4];
#pragma unroll
        for (int tr = 0; tr < 4; ++tr)
#pragma unroll
          for (int tc = 0; tc < 4; ++tc) dmma884(acc[tr][tc][0], acc[tr][tc][1], av[tr][kk], bv[tc]);
      }
#pragma unroll
      for (int tr = 0; tr < 4; ++tr)
#pragma unroll
        for (int tc = 0; tc < 4; ++tc)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = r0 + tr * 8 + q, j = tc * 8 + 2 * s4 + e;
            A[(int64_t)(c0 + j) * b + c0 + NB + r] = acc[tr][tc][e];
            P[r * PLD + j] = acc[tr][tc][e];
          }
    }
    if (Linv) __threadfence_block();  // inverse row kb before step kb's partial sums read it
    PTRACE();  // 3 + 6 kb: sub-panel phase done
    named_bar_sync(bar, POTRF_THREADS);
    PTRACE();  // 4 + 6 kb
    // (B) trailing update in 32x32 blocks; block (0, 0) is diagonal block k+1
    const int nb32 = rest / 32;
    const int nblk = nb32 * (nb32 + 1) / 2;
    const int base_rc = c0 + NB;
    if (warp == 0) {
      trail_block32(A, b, base_rc, P, 0, 0, lane);
      __syncwarp();
      __threadfence_block();
      PTRACE();  // 5 + 6 kb (warp 0): diagonal block updated
      const unsigned fm = warp_potrf32(A, b, base_rc, D, rdiag, col, lane);
      PTRACE();  // 6 + 6 kb (warp 0): factored
      if (fm) {
        if (lane == 0) {
          if (info) set_info(info, row0 + base_rc + __ffs(fm));
          *s_fail = 1;
        }
      } else {
        warp_trinv32(D, rdiag, Dinv_s, dinv ? dinv + (int64_t)(kb + 1) * NB * NB : nullptr, lane);
      }
    } else {
      // the inverse's partial sums of row block kb+1 (kb+1 blocks), then the
      // trailing blocks 1.. (row-major lower), dealt round-robin to warps 1..7
      const int nS = Linv ? kb + 1 : 0;
      for (int u = warp - 1; u < nS + nblk - 1; u += POTRF_THREADS / 32 - 1) {
        if (u < nS) {
          linv_row_partial(A, l_smem, Linv, b, kb + 1, u, lane);
          continue;
        }
        const int t = u - nS + 1;
        int bi = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
        while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
        while (bi * (bi + 1) / 2 > t) --bi;
        trail_block32(A, b, base_rc, P, bi, t - bi * (bi + 1) / 2, lane);
      }
      PTRACE();  // 5 + 6 kb (warp 1): trailing blocks done
      PTRACE();
    }
    PTRACE();  // 7 + 6 kb: warp 0 inverted / warp 1 done
    __threadfence_block();
    named_bar_sync(bar, POTRF_THREADS);
    if (*s_fail) return false;
    if (progress) potrf_publish(progress, kb + 2, tid, bar);
  }
  if (Linv) {  // the last row block of the inverse
    linv_row_apply(dinv, Linv, b, nbk - 1, warp, POTRF_THREADS / 32, lane);
    __threadfence_block();
    named_bar_sync(bar, POTRF_THREADS);
  }
  return true;
}

constexpr int TINV_THREADS = 256;

// Single-CTA inverse of a factored diagonal tile for the look-ahead stream
// (where only one SM is free): Linv = L^{-1} by block diagonals.  Diagonal
// d holds the blocks (j + d, j); each is
//   Linv[j+d][j] = -Dinv_{j+d} * sum_{m=j}^{j+d-1} L[j+d][m] Linv[m][j]
// and only needs diagonals < d, so all blocks of a diagonal are independent:
// one warp per 32x32 block, 4x4 DMMA tiles, 64 fragment loads (L2: the tile
// was just factored) in flight per 128 DMMAs.
// LSMEM: L is a shared-memory copy of the tile (ld b), see tile_potrf_inv_device.
template <bool LSMEM = false>
static __device__ __noinline__ void tri_inv_diag_device(const double* __restrict__ L, const double* __restrict__ dinv, int b,
                                    double* __restrict__ Linv, double* S, int tid, int bar) {
  // S: per warp one 32x32 partial sum, [(w*32 + r)*33 + c]
  const int nbk = b / NB;
  const int warp = tid >> 5, lane = tid & 31;
  const int nw = TINV_THREADS / 32;
  const int q = lane >> 2, s4 = lane & 3;
  // block diagonal = Dinv, strictly upper blocks = 0 (the blocks below are
  // written per diagonal): one warp per column, lanes on consecutive rows
  // (coalesced 16-byte stores, no per-element index arithmetic)
  for (int c = warp; c < b; c += nw) {
    const int bj = c / NB;
    double2* col = reinterpret_cast<double2*>(Linv + (int64_t)c * b);
    for (int r2 = lane; r2 < bj * NB / 2; r2 += 32) col[r2] = make_double2(0.0, 0.0);
    if (lane < NB / 2) {
      const double2* dsrc = reinterpret_cast<const double2*>(dinv + (int64_t)bj * NB * NB + (c % NB) * NB);
      col[bj * NB / 2 + lane] = __ldcg(dsrc + lane);
    }
  }
  __threadfence_block();
  named_bar_sync(bar, TINV_THREADS);
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
        block_mma32<LSMEM>(acc, L + (int64_t)(m * NB) * b + i * NB, b, Linv + (int64_t)(j * NB) * b + m * NB, b,
                           lane);
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
          av[t] = __ldcg(Di + (4 * k + s4) * NB + t * 8 + q);
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
    __threadfence_block();
    named_bar_sync(bar, TINV_THREADS);  // diagonal d complete before d + 1 reads it
  }
}


// Tiles up to SMEM_TILE: the whole b x b tile is copied into shared memory,
// factored there (no L2 round trip between the sub-panel steps) and, with
// Linv, inverted from the shared copy; L goes back once at the end.  The
// dependent chain of small steps is what bounds these tiles (tail steps,
// small problems).  Larger tiles run in place through L2.  `sm` holds
// tile_potrf_inv_smem_bytes(b).
constexpr int SMEM_TILE = 128;

static __device__ __noinline__ bool tile_potrf_inv_device(double* __restrict__ A, int b, int64_t row0,
                                                          double* __restrict__ dinv,
                                                          unsigned long long* __restrict__ info,
                                                          double* __restrict__ Linv, double* sm, int tid, int bar,
                                                          int* progress = nullptr) {
  static_assert(POTRF_THREADS == TINV_THREADS, "one thread set");
  // a published factor must be in global memory: with progress the tile is
  // factored in place whatever its size
  if (b > SMEM_TILE || progress) return tile_potrf_device(A, b, row0, dinv, info, sm, tid, bar, Linv, false, progress);
  double* T = sm;
  double* scratch = sm + (size_t)b * b;
  const int n2 = b * b / 2;
  const double2* src = reinterpret_cast<const double2*>(A);
  double2* dst = reinterpret_cast<double2*>(T);
  for (int i = tid; i < n2; i += POTRF_THREADS) dst[i] = __ldcg(src + i);
  named_bar_sync(bar, POTRF_THREADS);
  const bool ok = tile_potrf_device(T, b, row0, dinv, info, scratch, tid, bar, Linv, true);
  named_bar_sync(bar, POTRF_THREADS);
  double2* out = reinterpret_cast<double2*>(A);
  const double2* Ts = reinterpret_cast<const double2*>(T);
  for (int i = tid; i < n2; i += POTRF_THREADS) out[i] = Ts[i];
  __threadfence();
  named_bar_sync(bar, POTRF_THREADS);
  return ok;
}

}  // namespace bgp
