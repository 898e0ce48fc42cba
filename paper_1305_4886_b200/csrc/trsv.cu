// K3a: forward substitution L x = r over the packed tile triangle as ONE
// persistent, dataflow-ordered kernel.
//
// Replaces the reference's blocked forward solve (bg/distla/kernels.py:200-250,
// solve_vector with forward=True): x_J = L_JJ^{-1} (r_J - sum_{K<J} L_JK x_K).
//
// The old form launched two kernels per tile row (a latency-bound one-CTA
// diagonal solve, then the row updates), 2T launches in all.  Here each CTA
// takes 128-row blocks I in increasing order from an atomic counter and owns
// the whole block row: it streams blocks (I, 0..I-1) through a 3-stage
// shared-memory ring filled by TMA (2 CTAs per SM), subtracting L_IJ x_J as
// soon as x_J is published, then solves the diagonal tile with the inverses
// of its 32x32 diagonal blocks (from diag_inv_kernel) and publishes x_I with
// a release flag.  A row waits only on rows taken earlier by resident CTAs,
// so the schedule cannot deadlock, and every byte of L is read once: the
// kernel is bound by HBM bandwidth (8 B per stored entry), not by 2T launch
// latencies.  Sums run in a fixed order (K ascending, columns ascending), so
// the result is deterministic.
#include "bgp_common.cuh"
#include "bgp_internal.h"

namespace bgp {

// Rows are solved in blocks of TV_BS = 128 (sub-blocks of the storage
// tiles), so the serial chain x_{I-1} -> x_I that bounds the solve has 4x
// more, 16x cheaper links than with 512-row tiles, and more rows are in
// flight than there are SMs.
constexpr int TV_BS = 128;                  // solve block (rows of one CTA)
constexpr int TV_STAGES = 3;
constexpr int TV_CH = 32;                   // columns per stage
constexpr int TV_PAYLOAD = TV_BS * TV_CH * 8;  // 32 KB: a 128 x 32 box of L (or a 32x32 inverse)
constexpr int TV_XBYTES = 256;              // x_J entries of the stage's columns
constexpr int TV_STAGE_BYTES = TV_PAYLOAD + TV_XBYTES;
constexpr int TV_NB = 32;                   // diagonal block (one warp)
constexpr int TV_THREADS = TV_BS + 32;      // one thread per row + a producer warp

// Per block row I: the off-diagonal blocks stream through a 3-stage ring
// (for J < I, for c0 in [0, BS) step CH: L(I,J)[:, c0:c0+CH] by TMA, then
// x_J[c0:c0+CH] once x_J is published), while the diagonal block's data --
// the four 32x32 inverses and the six 32x32 sub-blocks below its diagonal
// blocks -- load into a separate area at row start, since they do not depend
// on x.  So the serial chain x_{I-1} -> x_I waits only for the x copies of
// block I-1 and the diagonal solve from shared memory.  L(I,J) is the
// 128 x 128 sub-block (I, J) of the packed b-tile triangle.
constexpr int TV_DIAG_BOXES = 6;                    // sub-blocks (kb, rb), kb < rb < 4
constexpr int TV_DIAG_BYTES = 4 * TV_NB * TV_NB * 8 + TV_DIAG_BOXES * TV_NB * TV_NB * 8;  // 80 KB

__device__ __forceinline__ int diag_box(int kb, int rb) {  // (0,1..3) (1,2..3) (2,3) -> 0..5
  return kb == 0 ? rb - 1 : (kb == 1 ? rb + 1 : 5);
}

__global__ void __launch_bounds__(TV_THREADS, 1)
    trsv_fwd_persistent_kernel(const __grid_constant__ CUtensorMap tmL, const __grid_constant__ CUtensorMap tmD,
                               const double* __restrict__ dinv, int T, int b, int Ts, double* __restrict__ x,
                               int* __restrict__ sync /* [0] row counter, [1+J] flags */) {
  extern __shared__ __align__(128) uint8_t tv_smem[];
  uint8_t* stages = tv_smem;
  uint8_t* dg = tv_smem + TV_STAGES * TV_STAGE_BYTES;                 // diagonal data
  const double* dg_inv = reinterpret_cast<const double*>(dg);         // 4 x (32x32 column-major)
  const double* dg_box = dg_inv + 4 * TV_NB * TV_NB;                  // 6 x (32 rows x 32 cols)
  double* r = reinterpret_cast<double*>(dg + TV_DIAG_BYTES);          // solved block values
  uint64_t* full = reinterpret_cast<uint64_t*>(r + TV_BS);
  uint64_t* empty = full + TV_STAGES;
  uint64_t* dfull = empty + TV_STAGES;
  uint64_t* dempty = dfull + 1;
  int* s_row = reinterpret_cast<int*>(dempty + 1);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps_c = TV_BS / 32;
  constexpr int nbk = TV_BS / TV_NB;
  const int sub = b / TV_BS;  // solve blocks per storage tile
  if (tid == 0) {
    for (int s = 0; s < TV_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwarps_c);
    }
    mbar_init(dfull, 1);
    mbar_init(dempty, nwarps_c);
    fence_barrier_init();
  }
  __syncthreads();

  int stage = 0;
  uint32_t phase = 0, dphase = 0;
  auto advance = [&]() {
    if (++stage == TV_STAGES) {
      stage = 0;
      phase ^= 1;
    }
  };

  if (tid >= TV_BS) {
    // ----------------------------- producer warp -----------------------------
    const uint64_t pol = l2_policy_evict_first();  // L is read once
    if (lane == 0) {
      prefetch_tmap(&tmL);
      prefetch_tmap(&tmD);
    }
    for (;;) {
      int row = 0;
      if (lane == 0) {
        row = atomicAdd(&sync[0], 1);
        *s_row = row;
      }
      named_bar_sync(0, TV_THREADS);  // publish the row (whole warp arrives)
      row = __shfl_sync(0xffffffffu, row, 0);
      if (row >= Ts) break;
      if (lane == 0) {
        const int I = row / sub, sr = (row % sub) * TV_BS;
        // diagonal data first (the previous row's diagonal solve has released it)
        mbar_wait(dempty, dphase ^ 1);
        mbar_arrive_expect_tx(dfull, TV_DIAG_BYTES);
        bulk_load(dg, dinv + (int64_t)row * nbk * TV_NB * TV_NB, 4 * TV_NB * TV_NB * 8, dfull);
        const int dtile = (int)tri_index(I, I, T);
        for (int kb = 0; kb + 1 < nbk; ++kb)
          for (int rb = kb + 1; rb < nbk; ++rb)
            tma_load_3d(dg + 4 * TV_NB * TV_NB * 8 + diag_box(kb, rb) * TV_NB * TV_NB * 8, &tmD, dfull,
                        sr + rb * TV_NB, sr + kb * TV_NB, dtile, pol);
        dphase ^= 1;
        // off-diagonal blocks through the ring
        for (int J = 0; J < row; ++J) {
          const int tile = (int)tri_index(I, J / sub, T);
          for (int c0 = 0; c0 < TV_BS; c0 += TV_CH) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* st = stages + stage * TV_STAGE_BYTES;
            mbar_arrive_expect_tx(&full[stage], (uint32_t)(TV_PAYLOAD + TV_CH * 8));
            tma_load_3d(st, &tmL, &full[stage], sr, (J % sub) * TV_BS + c0, tile, pol);  // no wait on x
            if (c0 == 0) {
              // x_J must be final before its entries are copied (release/acquire on flag J)
              unsigned ns = 32;
              while (ld_acquire_gpu(&sync[1 + J]) == 0) {
                __nanosleep(ns);
                if (ns < 256) ns <<= 1;
              }
              fence_proxy_async_global();
            }
            bulk_load(st + TV_PAYLOAD, x + (int64_t)J * TV_BS + c0, (uint32_t)(TV_CH * 8), &full[stage]);
            advance();
          }
        }
      }
      __syncwarp();
    }
    return;
  }

  // ------------------------------- consumers -------------------------------
  const int t = tid;  // row of this thread inside the block
  for (;;) {
    named_bar_sync(0, TV_THREADS);
    const int row = *s_row;
    if (row >= Ts) break;
    double acc = x[(int64_t)row * TV_BS + t];
    for (int J = 0; J < row; ++J) {
      for (int c0 = 0; c0 < TV_BS; c0 += TV_CH) {
        mbar_wait(&full[stage], phase);
        const double* S = reinterpret_cast<const double*>(stages + stage * TV_STAGE_BYTES);
        const double* xc = reinterpret_cast<const double*>(stages + stage * TV_STAGE_BYTES + TV_PAYLOAD);
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int c = 0; c < TV_CH; c += 4) {
          a0 = fma(S[c * TV_BS + t], xc[c], a0);
          a1 = fma(S[(c + 1) * TV_BS + t], xc[c + 1], a1);
          a2 = fma(S[(c + 2) * TV_BS + t], xc[c + 2], a2);
          a3 = fma(S[(c + 3) * TV_BS + t], xc[c + 3], a3);
        }
        acc -= (a0 + a1) + (a2 + a3);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        advance();
      }
    }
    // diagonal block from the diagonal area: 32-row block kb is warp kb
    mbar_wait(dfull, dphase);
    dphase ^= 1;
    for (int kb = 0; kb < nbk; ++kb) {
      if (warp == kb) {
        const double* Di = dg_inv + kb * TV_NB * TV_NB;
        double xi = 0.0;
#pragma unroll 8
        for (int j = 0; j < TV_NB; ++j) xi = fma(Di[j * TV_NB + lane], __shfl_sync(0xffffffffu, acc, j), xi);
        acc = xi;
        r[t] = xi;
      }
      if (kb + 1 == nbk) break;
      named_bar_sync(1, TV_BS);  // block kb of r is final
      if (warp > kb) {
        const double* S = dg_box + diag_box(kb, warp) * TV_NB * TV_NB;  // rows 32*warp.., cols 32*kb..
        double a0 = 0.0, a1 = 0.0;
#pragma unroll 8
        for (int c = 0; c < TV_NB; c += 2) {
          a0 = fma(S[c * TV_NB + lane], r[kb * TV_NB + c], a0);
          a1 = fma(S[(c + 1) * TV_NB + lane], r[kb * TV_NB + c + 1], a1);
        }
        acc -= a0 + a1;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(dempty);  // diagonal area free for the next row
    x[(int64_t)row * TV_BS + t] = acc;
    __threadfence();
    named_bar_sync(1, TV_BS);
    if (t == 0) st_release_gpu(&sync[1 + row], 1);
  }
}

int launch_trsv_fwd_persistent(Ctx* ctx, const double* L, int64_t n, int b, double* x, cudaStream_t s) {
  const int T = (int)((n + b - 1) / b);
  const int Ts = T * (b / TV_BS);  // solve blocks, padding included (identity rows solve to 0)
  const int nbk = b / TV_NB;
  int rc;
  if ((rc = ensure(ctx, (void**)&ctx->d_dinv, &ctx->dinv_cap, (size_t)T * nbk * TV_NB * TV_NB * sizeof(double))))
    return rc;
  if ((rc = ensure(ctx, (void**)&ctx->d_sync, &ctx->sync_cap, (size_t)(Ts + 1) * sizeof(int)))) return rc;
  if ((rc = launch_diag_inv(ctx, L, T, b, n, ctx->d_dinv, s))) return rc;
  cudaError_t e = cudaMemsetAsync(ctx->d_sync, 0, (size_t)(Ts + 1) * sizeof(int), s);
  if (e != cudaSuccess) return set_err(ctx, "trsv sync reset", e);
  CUtensorMap tm, td;
  if ((rc = make_tile_map(ctx, &tm, L, b, tri_count(T), TV_BS, TV_CH, false))) return rc;
  if ((rc = make_tile_map(ctx, &td, L, b, tri_count(T), TV_NB, TV_NB, false))) return rc;
  const size_t smem = (size_t)TV_STAGES * TV_STAGE_BYTES + TV_DIAG_BYTES + TV_BS * sizeof(double) +
                      (2 * TV_STAGES + 2) * 8 + 16;
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(trsv_fwd_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_done = true;
  }
  const int slots = ctx->num_sms;
  const int grid = Ts < slots ? Ts : slots;
  trsv_fwd_persistent_kernel<<<grid, TV_THREADS, smem, s>>>(tm, td, ctx->d_dinv, T, b, Ts, x, (int*)ctx->d_sync);
  ctx->launches++;
  return check_launch(ctx, "trsv_fwd_persistent");
}

}  // namespace bgp
