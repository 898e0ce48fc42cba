// K2c / K3b / K3c: persistent FP64 tensor-core GEMM on packed tiles.
//
// Computes, for a list of 128x128 output blocks of b x b column-major tiles,
//     D = beta * C + alpha * sum_k A(m, k) B(n, k)        (A, B "MN-major")
// which covers
//   * the Cholesky trailing SYRK/GEMM   A_RC -= L_RJ L_CJ^T
//     (bg/distla/kernels.py:188-192, ~all of the n^3/3 flops),
//   * the kriging multi-RHS update      B^T_I -= X^T_J L_IJ^T
//     (solve_rect partial GEMMs, kernels.py:287-291),
//   * the crossproduct                  S = V^T V   (xprod_self, kernels.py:448).
//
// sm_100a has no FP64 tcgen05 kind, so the MMA is mma.sync m8n8k4 f64
// (SASS DMMA.8x8x4, 128 flop/clk/SM).  Operands are staged by TMA
// (cp.async.bulk.tensor, 128B swizzle) into a 4-stage mbarrier ring filled by
// one producer warp; 8 MMA warps each own a 64x32 accumulator (64 FP64 regs).
// The C block is TMA-loaded into shared memory during the main loop and the
// result is TMA-stored from the same buffer, so the epilogue's HBM traffic
// overlaps the next block's main loop.  One CTA per SM, static round-robin
// over blocks (all blocks have equal cost).
//
// Bank conflicts: a 16-double-wide TMA box with 128B swizzle stores element
// (mn, k) at chunk ((mn&15)>>1) ^ (k&7).  Each MMA k4 step takes
// k = 2*(lane&3) + t (t = 0, 1) inside the 8-wide k stage, which makes the
// 16 lanes of each half-warp hit 16 distinct 8-byte slots.
#include "bgp_common.cuh"
#include "bgp_internal.h"

namespace bgp {

constexpr int BM = 128, BN = 128, BK = 8, STAGES = 4;
constexpr int MMA_WARPS = 8;
constexpr int THREADS = (MMA_WARPS + 1) * 32;
constexpr int WM = 64, WN = 32;
constexpr int STAGE_A_BYTES = BM * BK * 8;  // 8 KB
constexpr int STAGE_BYTES = 2 * STAGE_A_BYTES;
constexpr int CBUF_BYTES = BM * BN * 8;  // 128 KB
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + CBUF_BYTES + 1024 /*barriers*/ + 1024 /*align*/;

struct Item {
  int64_t cTile, aTile0, bTile0;
  int64_t aStride, bStride;  // tile-index stride per k tile
  int nkt;                   // number of k tiles
  int mrow0, nrow0;          // row offsets inside the A / B tiles (= C block offsets)
  int lower;                 // diagonal block of a diagonal tile: lower triangle only
  bool valid;
};

__device__ __forceinline__ int64_t gemm_num_items(const GemmProblem& p) {
  const int nbt = p.b / BM;
  switch (p.mode) {
    case GEMM_CHOL_TRAIL: {
      const int64_t k = p.T - p.J - 1;
      return k * (k + 1) / 2 * nbt * nbt;
    }
    case GEMM_RECT_TRAIL:
      return (int64_t)p.Tm * (p.T - p.J - 1) * nbt * nbt;
    case GEMM_SYRK_RECT:
      return (int64_t)p.Tm * (p.Tm + 1) / 2 * nbt * nbt;
    default:
      return p.count * nbt * nbt;
  }
}

__device__ __forceinline__ Item gemm_decode(const GemmProblem& p, int64_t item) {
  const int nbt = p.b / BM;
  const int nb2 = nbt * nbt;
  const int64_t t = item / nb2;
  const int blk = (int)(item % nb2);
  const int bi = blk / nbt, bj = blk % nbt;
  Item it;
  it.mrow0 = bi * BM;
  it.nrow0 = bj * BN;
  it.aStride = it.bStride = 0;
  it.nkt = 1;
  it.valid = true;
  it.lower = 0;
  switch (p.mode) {
    case GEMM_CHOL_TRAIL: {
      int rr, cc;
      tri_decode(t, p.T - p.J - 1, rr, cc);
      const int R = p.J + 1 + rr, C = p.J + 1 + cc;
      it.cTile = tri_index(R, C, p.T);
      it.aTile0 = tri_index(R, p.J, p.T);
      it.bTile0 = tri_index(C, p.J, p.T);
      if (R == C) {
        if (bi < bj) it.valid = false;
        it.lower = (bi == bj);
      }
      break;
    }
    case GEMM_RECT_TRAIL: {
      const int a = (int)(t % p.Tm);
      const int I = p.J + 1 + (int)(t / p.Tm);
      it.cTile = (int64_t)I * p.Tm + a;
      it.aTile0 = (int64_t)p.J * p.Tm + a;
      it.bTile0 = tri_index(I, p.J, p.T);
      break;
    }
    case GEMM_SYRK_RECT: {
      int rr, cc;
      tri_decode(t, p.Tm, rr, cc);
      it.cTile = tri_index(rr, cc, p.Tm);
      it.aTile0 = rr;
      it.bTile0 = cc;
      it.aStride = it.bStride = p.Tm;
      it.nkt = p.Tn;
      if (rr == cc) {
        if (bi < bj) it.valid = false;
        it.lower = (bi == bj);
      }
      break;
    }
    default: {  // GEMM_LIST: (C, A, B, lower) tile-index quadruples
      const int32_t* q = p.items + 4 * t;
      it.cTile = q[0];
      it.aTile0 = q[1];
      it.bTile0 = q[2];
      if (q[3]) {
        if (bi < bj) it.valid = false;
        it.lower = (bi == bj);
      }
      break;
    }
  }
  return it;
}

// byte offset of element (mn, k) inside one operand stage (8 boxes of 16x8)
__device__ __forceinline__ uint32_t op_off(int mn, int k) {
  return (uint32_t)((mn >> 4) * 1024 + k * 128 + ((((mn & 15) >> 1) ^ k) << 4) + ((mn & 1) << 3));
}
// byte offset of element (m, n) inside the C buffer (8 boxes of 16x128)
__device__ __forceinline__ uint32_t c_off(int m, int n) {
  return (uint32_t)((m >> 4) * 16384 + n * 128 + ((((m & 15) >> 1) ^ (n & 7)) << 4) + ((m & 1) << 3));
}

__global__ void __launch_bounds__(THREADS, 1)
    gemm_dmma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, const GemmProblem p,
                     const unsigned long long* __restrict__ info) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* stages = smem;
  uint8_t* cbuf = smem + STAGES * STAGE_BYTES;
  uint64_t* bars = (uint64_t*)(cbuf + CBUF_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* c_full = bars + 2 * STAGES;
  uint64_t* c_empty = c_full + 1;

  if (info && *(volatile const unsigned long long*)info != 0ull) return;  // factorization failed

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MMA_WARPS);
    }
    mbar_init(c_full, 1);
    mbar_init(c_empty, 1);
    fence_barrier_init();
  }
  __syncthreads();

  const int64_t nitems = gemm_num_items(p);
  const int kc_per_tile = p.b / BK;
  const bool load_c = (p.beta != 0.0);

  if (warp == MMA_WARPS) {
    // ------------------------------ producer ------------------------------
    if (lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      prefetch_tmap(&tmC);
      const uint64_t pol_keep = l2_policy_evict_last();
      const uint64_t pol_stream = l2_policy_evict_first();
      int stage = 0;
      uint32_t phase = 0, cphase = 0;
      for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
        const Item it = gemm_decode(p, item);
        if (!it.valid) continue;
        const int nk = it.nkt * kc_per_tile;
        for (int kc = 0; kc < nk; ++kc) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          const int kt = kc / kc_per_tile;
          const int kin = (kc % kc_per_tile) * BK;
          const int at = (int)(it.aTile0 + kt * it.aStride);
          const int bt = (int)(it.bTile0 + kt * it.bStride);
          uint8_t* sa = stages + stage * STAGE_BYTES;
          uint8_t* sb = sa + STAGE_A_BYTES;
#pragma unroll
          for (int i = 0; i < BM / 16; ++i)
            tma_load_3d(sa + i * 1024, &tmA, &full[stage], it.mrow0 + i * 16, kin, at, pol_keep);
#pragma unroll
          for (int i = 0; i < BN / 16; ++i)
            tma_load_3d(sb + i * 1024, &tmB, &full[stage], it.nrow0 + i * 16, kin, bt, pol_keep);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
          if (load_c && kc == (nk > 1 ? 1 : 0)) {
            mbar_wait(c_empty, cphase ^ 1);
            mbar_arrive_expect_tx(c_full, CBUF_BYTES);
#pragma unroll
            for (int i = 0; i < BM / 16; ++i)
              tma_load_3d(cbuf + i * 16384, &tmC, c_full, it.mrow0 + i * 16, it.nrow0, (int)it.cTile,
                          pol_stream);
            cphase ^= 1;
          }
        }
      }
    }
    return;
  }

  // -------------------------------- MMA warps --------------------------------
  const int wm = warp / (BN / WN), wn = warp % (BN / WN);
  const int q = lane >> 2, s4 = lane & 3;
  int stage = 0;
  uint32_t phase = 0, cphase = 0;
  bool store_pending = false;
  const uint32_t stages_u32 = smem_u32(stages);
  const uint32_t cbuf_u32 = smem_u32(cbuf);
  const uint64_t pol_stream = l2_policy_evict_first();

  for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
    const Item it = gemm_decode(p, item);
    if (!it.valid) continue;
    const int nk = it.nkt * kc_per_tile;
    double acc[WM / 8][WN / 8][2];
#pragma unroll
    for (int i = 0; i < WM / 8; ++i)
#pragma unroll
      for (int j = 0; j < WN / 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kc = 0; kc < nk; ++kc) {
      mbar_wait(&full[stage], phase);
      const uint32_t sa = stages_u32 + stage * STAGE_BYTES;
      const uint32_t sb = sa + STAGE_A_BYTES;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int k = 2 * s4 + t;
        double af[WM / 8], bf[WN / 8];
#pragma unroll
        for (int i = 0; i < WM / 8; ++i)
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(af[i]) : "r"(sa + op_off(wm * WM + i * 8 + q, k)));
#pragma unroll
        for (int j = 0; j < WN / 8; ++j)
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(bf[j]) : "r"(sb + op_off(wn * WN + j * 8 + q, k)));
#pragma unroll
        for (int i = 0; i < WM / 8; ++i)
#pragma unroll
          for (int j = 0; j < WN / 8; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
      if (kc == 0 && store_pending && threadIdx.x == 0) {
        // previous block's TMA store has to finish reading the C buffer
        // before the producer may overwrite it
        tma_store_wait_read0();
        mbar_arrive(c_empty);
      }
    }

    // ------------------------------- epilogue -------------------------------
    if (load_c) {
      mbar_wait(c_full, cphase);
    } else {
      if (store_pending && threadIdx.x == 0) tma_store_wait_read0();
      named_bar_sync(1, MMA_WARPS * 32);
    }
    cphase ^= 1;
#pragma unroll
    for (int i = 0; i < WM / 8; ++i) {
#pragma unroll
      for (int j = 0; j < WN / 8; ++j) {
        const int m = wm * WM + i * 8 + q;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = wn * WN + j * 8 + 2 * s4 + e;
          const uint32_t addr = cbuf_u32 + c_off(m, n);
          double cv = 0.0;
          if (load_c) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(cv) : "r"(addr));
          double d;
          if (it.lower && m < n) d = load_c ? cv : 0.0;  // keep the strict upper triangle
          else d = load_c ? fma(p.alpha, acc[i][j][e], p.beta * cv) : p.alpha * acc[i][j][e];
          asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(d) : "memory");
        }
      }
    }
    fence_proxy_async_smem();
    named_bar_sync(1, MMA_WARPS * 32);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int i = 0; i < BM / 16; ++i)
        tma_store_3d(&tmC, cbuf + i * 16384, it.mrow0 + i * 16, it.nrow0, (int)it.cTile, pol_stream);
      tma_store_commit();
    }
    store_pending = true;
  }
  if (threadIdx.x == 0 && store_pending) tma_store_wait_all0();
}

int launch_gemm(Ctx* ctx, const GemmProblem& p, double* Cbase, const double* Abase, int64_t nA,
                const double* Bbase, int64_t nB, int64_t nC, cudaStream_t s) {
  if (p.b % BM != 0) return set_err(ctx, "gemm: tile must be a multiple of 128", cudaErrorInvalidValue);
  int64_t items;
  {
    const int nbt = p.b / BM;
    switch (p.mode) {
      case GEMM_CHOL_TRAIL: {
        const int64_t k = p.T - p.J - 1;
        items = k * (k + 1) / 2 * nbt * nbt;
        break;
      }
      case GEMM_RECT_TRAIL:
        items = (int64_t)p.Tm * (p.T - p.J - 1) * nbt * nbt;
        break;
      case GEMM_SYRK_RECT:
        items = (int64_t)p.Tm * (p.Tm + 1) / 2 * nbt * nbt;
        break;
      default:
        items = p.count * nbt * nbt;
    }
  }
  if (items <= 0) return BGP_OK;
  CUtensorMap mA, mB, mC;
  int rc;
  if ((rc = make_tile_map(ctx, &mA, Abase, p.b, nA, 16, BK, true)) != BGP_OK) return rc;
  if ((rc = make_tile_map(ctx, &mB, Bbase, p.b, nB, 16, BK, true)) != BGP_OK) return rc;
  if ((rc = make_tile_map(ctx, &mC, Cbase, p.b, nC, 16, BN, true)) != BGP_OK) return rc;
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(gemm_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    attr_done = true;
  }
  const int64_t grid = items < ctx->num_sms ? items : ctx->num_sms;
  gemm_dmma_kernel<<<(unsigned)grid, THREADS, SMEM_BYTES, s>>>(mA, mB, mC, p, ctx->d_info);
  ctx->launches++;
  return check_launch(ctx, "gemm_dmma");
}

}  // namespace bgp
