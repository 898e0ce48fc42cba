// K3a: forward substitution L x = r over the packed tile triangle as ONE
// persistent, dataflow-ordered kernel.
//
// Replaces the reference's blocked forward solve (bg/distla/kernels.py:200-250,
// solve_vector with forward=True): x_J = L_JJ^{-1} (r_J - sum_{K<J} L_JK x_K).
//
// The old form launched two kernels per tile row (a latency-bound one-CTA
// diagonal solve, then the row updates), 2T launches in all.  Here each CTA
// takes tile rows I in increasing order from an atomic counter and owns the
// whole row: it streams tiles (I, 0..I-1) through a 4-stage shared-memory
// ring filled by 1-D bulk copies (cp.async.bulk), subtracting L_IJ x_J as
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

constexpr int TV_STAGES = 4;
constexpr int TV_PAYLOAD = 32768;           // L columns (or a 32x32 inverse) per stage
constexpr int TV_XBYTES = 256;              // x_J entries of the stage's columns
constexpr int TV_STAGE_BYTES = TV_PAYLOAD + TV_XBYTES;
constexpr int TV_NB = 32;                   // diagonal block (one warp)

__host__ __device__ __forceinline__ int tv_cols_per_chunk(int b) {
  int ch = 32;
  while (ch * b * 8 > TV_PAYLOAD) ch >>= 1;
  return ch;  // 128: 32, 256: 16, 384: 8, 512: 8
}

// Chunk sequence of tile row I (producer and consumers walk it in lockstep):
//   off-diagonal: for J < I, for c0 in [0, b) step CH: L(I,J)[:, c0:c0+CH], x_J[c0:c0+CH]
//   diagonal:     for kb: Dinv_kb, then (kb < nbk-1) L(I,I)[:, 32kb + i*CH ...] (32/CH chunks)
__global__ void __launch_bounds__(512 + 32, 1)
    trsv_fwd_persistent_kernel(const double* __restrict__ L, const double* __restrict__ dinv, int T, int b,
                               double* __restrict__ x, int* __restrict__ sync /* [0] row counter, [1+J] flags */) {
  extern __shared__ __align__(128) uint8_t tv_smem[];
  uint8_t* stages = tv_smem;
  double* r = reinterpret_cast<double*>(tv_smem + TV_STAGES * TV_STAGE_BYTES);  // solved block values
  uint64_t* full = reinterpret_cast<uint64_t*>(r + 512);
  uint64_t* empty = full + TV_STAGES;
  int* s_row = reinterpret_cast<int*>(empty + TV_STAGES);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nconsumer = b;  // one thread per tile row
  const int nwarps_c = b / 32;
  const int CH = tv_cols_per_chunk(b);
  const int nbk = b / TV_NB;
  const int64_t tsz = (int64_t)b * b;
  if (tid == 0) {
    for (int s = 0; s < TV_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwarps_c);
    }
    fence_barrier_init();
  }
  __syncthreads();

  int stage = 0;
  uint32_t phase = 0;
  auto advance = [&]() {
    if (++stage == TV_STAGES) {
      stage = 0;
      phase ^= 1;
    }
  };

  auto produce_row = [&](int row) {
    for (int J = 0; J < row; ++J) {
      const double* tile = L + tri_index(row, J, T) * tsz;
      // x_J must be final before its entries are copied (release/acquire on flag J)
      unsigned ns = 32;
      while (ld_acquire_gpu(&sync[1 + J]) == 0) {
        __nanosleep(ns);
        if (ns < 1024) ns <<= 1;
      }
      fence_proxy_async_global();
      for (int c0 = 0; c0 < b; c0 += CH) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* st = stages + stage * TV_STAGE_BYTES;
        mbar_arrive_expect_tx(&full[stage], (uint32_t)(CH * b * 8 + CH * 8));
        bulk_load(st, tile + (int64_t)c0 * b, (uint32_t)(CH * b * 8), &full[stage]);
        bulk_load(st + TV_PAYLOAD, x + (int64_t)J * b + c0, (uint32_t)(CH * 8), &full[stage]);
        advance();
      }
    }
    const double* dt = L + tri_index(row, row, T) * tsz;
    for (int kb = 0; kb < nbk; ++kb) {
      mbar_wait(&empty[stage], phase ^ 1);
      uint8_t* st = stages + stage * TV_STAGE_BYTES;
      mbar_arrive_expect_tx(&full[stage], TV_NB * TV_NB * 8);
      bulk_load(st, dinv + ((int64_t)row * nbk + kb) * TV_NB * TV_NB, TV_NB * TV_NB * 8, &full[stage]);
      advance();
      if (kb + 1 == nbk) break;
      for (int c0 = kb * TV_NB; c0 < (kb + 1) * TV_NB; c0 += CH) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* st2 = stages + stage * TV_STAGE_BYTES;
        mbar_arrive_expect_tx(&full[stage], (uint32_t)(CH * b * 8));
        bulk_load(st2, dt + (int64_t)c0 * b, (uint32_t)(CH * b * 8), &full[stage]);
        advance();
      }
    }
  };

  if (tid >= nconsumer) {
    // ----------------------------- producer warp -----------------------------
    for (;;) {
      int row = 0;
      if (lane == 0) {
        row = atomicAdd(&sync[0], 1);
        *s_row = row;
      }
      named_bar_sync(0, nconsumer + 32);  // publish the row (whole warp arrives)
      row = __shfl_sync(0xffffffffu, row, 0);
      if (row >= T) break;
      if (lane == 0) produce_row(row);
      __syncwarp();
    }
    return;
  }

  // ------------------------------- consumers -------------------------------
  const int t = tid;  // tile row of this thread
  for (;;) {
    named_bar_sync(0, nconsumer + 32);
    const int row = *s_row;
    if (row >= T) break;
    double acc = x[(int64_t)row * b + t];
    for (int J = 0; J < row; ++J) {
      for (int c0 = 0; c0 < b; c0 += CH) {
        mbar_wait(&full[stage], phase);
        const double* S = reinterpret_cast<const double*>(stages + stage * TV_STAGE_BYTES);
        const double* xc = reinterpret_cast<const double*>(stages + stage * TV_STAGE_BYTES + TV_PAYLOAD);
        double a0 = 0.0, a1 = 0.0;
#pragma unroll 8
        for (int c = 0; c < CH; c += 2) {
          a0 = fma(S[c * b + t], xc[c], a0);
          a1 = fma(S[(c + 1) * b + t], xc[c + 1], a1);
        }
        acc -= a0 + a1;
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        advance();
      }
    }
    // diagonal tile: block kb is warp kb
    for (int kb = 0; kb < nbk; ++kb) {
      mbar_wait(&full[stage], phase);
      if (warp == kb) {
        const double* Di = reinterpret_cast<const double*>(stages + stage * TV_STAGE_BYTES);
        double xi = 0.0;
#pragma unroll 8
        for (int j = 0; j < TV_NB; ++j) xi = fma(Di[j * TV_NB + lane], __shfl_sync(0xffffffffu, acc, j), xi);
        acc = xi;
        r[t] = xi;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      advance();
      if (kb + 1 == nbk) break;
      named_bar_sync(1, nconsumer);  // block kb of r is final
      for (int c0 = kb * TV_NB; c0 < (kb + 1) * TV_NB; c0 += CH) {
        mbar_wait(&full[stage], phase);
        if (warp > kb) {
          const double* S = reinterpret_cast<const double*>(stages + stage * TV_STAGE_BYTES);
          double a0 = 0.0, a1 = 0.0;
          for (int c = 0; c < CH; c += 2) {
            a0 = fma(S[c * b + t], r[c0 + c], a0);
            a1 = fma(S[(c + 1) * b + t], r[c0 + c + 1], a1);
          }
          acc -= a0 + a1;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        advance();
      }
    }
    x[(int64_t)row * b + t] = acc;
    __threadfence();
    named_bar_sync(1, nconsumer);
    if (t == 0) st_release_gpu(&sync[1 + row], 1);
  }
}

int launch_trsv_fwd_persistent(Ctx* ctx, const double* L, int64_t n, int b, double* x, cudaStream_t s) {
  const int T = (int)((n + b - 1) / b);
  const int nbk = b / TV_NB;
  int rc;
  if ((rc = ensure(ctx, (void**)&ctx->d_dinv, &ctx->dinv_cap, (size_t)T * nbk * TV_NB * TV_NB * sizeof(double))))
    return rc;
  if ((rc = ensure(ctx, (void**)&ctx->d_sync, &ctx->sync_cap, (size_t)(T + 1) * sizeof(int)))) return rc;
  if ((rc = launch_diag_inv(ctx, L, T, b, n, ctx->d_dinv, s))) return rc;
  cudaError_t e = cudaMemsetAsync(ctx->d_sync, 0, (size_t)(T + 1) * sizeof(int), s);
  if (e != cudaSuccess) return set_err(ctx, "trsv sync reset", e);
  const size_t smem = (size_t)TV_STAGES * TV_STAGE_BYTES + 512 * sizeof(double) + 2 * TV_STAGES * 8 + 16;
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(trsv_fwd_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_done = true;
  }
  const int grid = T < ctx->num_sms ? T : ctx->num_sms;
  trsv_fwd_persistent_kernel<<<grid, b + 32, smem, s>>>(L, ctx->d_dinv, T, b, x, (int*)ctx->d_sync);
  ctx->launches++;
  return check_launch(ctx, "trsv_fwd_persistent");
}

}  // namespace bgp
