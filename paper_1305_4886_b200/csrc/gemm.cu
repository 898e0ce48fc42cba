// K2c / K2b / K3b / K3c: persistent FP64 tensor-core GEMM on packed tiles.
//
// Computes, for a list of 128x64 output blocks of b x b column-major tiles,
//     D = beta * C + alpha * sum_k A(m, k) B(n, k)        (A, B "MN-major")
// which covers
//   * the Cholesky trailing SYRK/GEMM   A_RC -= L_RJ L_CJ^T
//     (bg/distla/kernels.py:188-192, ~all of the n^3/3 flops),
//   * the panel TRSM                    L_IJ = A_IJ L_JJ^-T = A_IJ Linv^T
//     (kernels.py:163-164), in place, 64 columns at a time right to left,
//   * the kriging multi-RHS update      B^T_I -= X^T_J L_IJ^T
//     (solve_rect partial GEMMs, kernels.py:287-291),
//   * the crossproduct                  S = V^T V   (xprod_self, kernels.py:448).
//
// sm_100a has no FP64 tcgen05 kind, so the MMA is mma.sync m8n8k4 f64
// (SASS DMMA.8x8x4, 128 flop/clk/SM).  Operands are staged by TMA
// (cp.async.bulk.tensor, 128B swizzle) into per-group mbarrier rings; results
// leave through shared memory by TMA store or TMA reduce-add (C += -acc in
// L2).  One CTA per SM.  Work is a queue of tasks claimed with an atomic
// counter by each group's producer warp, which hands the block id to its
// consumers through the ring (dynamic scheduling: no static imbalance).
// A trailing-update launch can append the TRSM of the next panel as tasks:
// their producer waits, per tile, until the update blocks of that tile have
// retired, and the launch's look-ahead CTA factors the next diagonal tile
// (publishing its inverse, or its progress for a substitution solve).  The
// chain-bound tail runs several steps per launch (nsteps > 1), ordered by
// per-tile counters.
//
// Bank conflicts: a 16-double-wide TMA box with 128B swizzle stores element
// (mn, k) at chunk ((mn&15)>>1) ^ (k&7).  Each MMA k4 step takes
// k = 2*(lane&3) + t (t = 0, 1) inside the 8-wide k stage, which makes the
// 16 lanes of each half-warp hit 16 distinct 8-byte slots.
#include "bgp_common.cuh"
#include "bgp_internal.h"
#include "panel_device.cuh"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

namespace bgp {
namespace dmma {

// Tile configuration.  One CTA per SM, three warpgroups:
//   WG0  producers: warp 0 feeds consumer group 0's ring, warp 1 group 1's
//        (setmaxnreg.dec to PRODUCER_REGS);
//   WG1, WG2  consumers: 4 MMA warps each (2 x 2 warps of 64x32), each group
//        owns a 128x64 output block at a time (setmaxnreg.inc to CONSUMER_REGS).
// Each group's producer claims blocks from the launch's task queue, and the
// two groups run concurrently (half a block apart), so one group's epilogue
// overlaps the other group's main loop and the DMMA pipe never drains.
// Two stages of BK = 32 per group at every tile size; the epilogue goes out
// in 16-row rounds (DESIGN.md section 5 records the alternatives measured).
constexpr int BM = 128, BN = 64, BK = 32, STAGES = 2, EPI_ROWS = 16;
constexpr int GROUPS = 2;
constexpr int WM = 64, WN = 32;
constexpr int PRODUCER_REGS = 56, CONSUMER_REGS = 224;
constexpr int WARPS_M = 2, WARPS_N = 2;       // per consumer group
constexpr int GROUP_WARPS = WARPS_M * WARPS_N;
constexpr int THREADS = 128 * (GROUPS + 1);
constexpr int MI = WM / 8, NJ = WN / 8;        // 8x8 DMMA tiles per warp
static_assert(BM == WARPS_M * WM && BN == WARPS_N * WN, "block = 2 x 2 warp tiles");
constexpr int BOX_BYTES = 16 * BK * 8;         // 2 KB: operand TMA box of 16 rows x BK k
constexpr int STAGE_A_BYTES = BM * BK * 8;     // 16 KB: 8 boxes
constexpr int STAGE_B_BYTES = BN * BK * 8;     // 8 KB: 4 boxes
constexpr int STAGE_BYTES = STAGE_A_BYTES + STAGE_B_BYTES;
constexpr int WBOX_BYTES = 16 * WN * 8;        // 4 KB: epilogue box of 16 rows x 32 cols
constexpr int EPI_BOXES = EPI_ROWS / 16;       // boxes per epilogue round
constexpr int EPI_ROUNDS = WM / EPI_ROWS;      // rounds per warp tile
constexpr int WSTAGE_BYTES = EPI_BOXES * WBOX_BYTES;  // a warp's epilogue slice (one round)
constexpr int HALVES = BK / 4;                 // k4 half-steps per stage
constexpr int CBUF_BYTES = GROUP_WARPS * WSTAGE_BYTES;
// When a warp's other epilogue rounds fit in its quarter of one operand stage,
// the epilogue stages them in the block's last stage (released to the
// producer only once the bulk reads are done, early in the next block) and
// the last round in the warp's own slice: no wait between rounds.
constexpr bool EPI_IN_STAGE = STAGE_BYTES >= GROUP_WARPS * (EPI_ROUNDS - 1) * WSTAGE_BYTES && EPI_ROUNDS > 1;
constexpr int GROUP_BYTES = STAGES * STAGE_BYTES + CBUF_BYTES;
constexpr int BAR_BYTES = 640;
constexpr int SMEM_BYTES = GROUPS * GROUP_BYTES + BAR_BYTES;
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
static_assert((GROUPS * 2 * STAGES + 1) * 8 <= 256 && 256 + GROUPS * STAGES * 48 <= BAR_BYTES, "barrier area");


struct Item {
  int cTile, aTile0, bTile0;  // tile indices (< 2^31: 1.4e5 tiles at n = 131,072, b = 256)
  int bTriRow;               // >= 0: B tile for k tile kt is L(bTriRow, triCol0 + kt) (TRMM, merged panels)
  int aTriRow;               // >= 0: A tile for k tile kt is L(aTriRow, triCol0 + kt) (merged panels)
  int triCol0;
  int aStride, bStride;      // tile-index stride per k tile
  int nkt;                   // number of k tiles
  int mrow0, nrow0;          // row offsets inside the A / B tiles (= C block offsets)
  int lower;                 // block straddles the diagonal of a diagonal tile
  int kstages;               // > 0: number of BK stages (triangular k range), else nkt * b / BK
  int store;                 // 1: TMA store of acc (beta = 0 / TRSM), 0: reduce-add of -acc
  int bLinv;                 // 1: B operand from the Linv map (fused TRSM block)
  int gate;                  // >= 0: column-gate index this block signals (update of column J+1)
  int slab, pass;            // trsm_par TRSM pass: slab index, pass (0 = rightmost); else slab = -1
  bool valid;
  bool pad;                  // skipped: every row lies in the identity padding (its gate still counts)
  bool subst;                // fused TRSM slab solved by substitution (no TMA stages)
};

__host__ __device__ __forceinline__ int64_t gemm_num_items(const GemmProblem& p) {
  const int nblk = (p.b / BM) * (p.b / BN);
  switch (p.mode) {
    case GEMM_CHOL_TRAIL: {
      const int64_t k = p.T - p.J - 1;
      if (k > 0 && p.pair_cols > 0) {  // columns J+1 .. J+m only
        const int64_t m = p.pair_cols < k ? p.pair_cols : k;
        return (m * k - m * (m - 1) / 2) * nblk;
      }
      return k > 0 ? k * (k + 1) / 2 * nblk : 0;
    }
    case GEMM_RECT_TRAIL:
      return (int64_t)p.Tm * (p.T - p.J - 1) * nblk;
    case GEMM_SYRK_RECT:
      return (int64_t)p.Tm * (p.Tm + 1) / 2 * nblk;
    case GEMM_TRMM_RECT:
      return (int64_t)p.Tm * p.T * nblk;
    default:  // GEMM_LIST, GEMM_TRSM_PANEL
      return p.count * nblk;
  }
}

// Tasks: a task is claimed by one consumer group and runs its blocks back to
// back.  Plain modes: one block per task.  TRSM (standalone, or appended to a
// trailing update for the next panel): a 128-row slab of a panel tile, its
// b/64 column blocks right to left, so the in-place solve never overwrites
// columns a later block still reads.
// Cholesky-type fused TRSM (the packed-triangle sweep, or a rank's tile list
// in the distributed sweep) whose column passes are independent tasks
__host__ __device__ __forceinline__ bool gemm_par_passes(const GemmProblem& p) {
  return (p.mode == GEMM_CHOL_TRAIL || p.mode == GEMM_LIST) && p.trsm_par;
}
__host__ __device__ __forceinline__ int64_t gemm_trsm_tasks(const GemmProblem& p) {
  if (p.mode == GEMM_TRSM_PANEL) return p.count * (p.b / BM) * (p.trsm_oop ? p.b / BN : 1);
  if (p.mode == GEMM_CHOL_TRAIL && p.trsm_next)
    return (int64_t)(p.T - p.J - 2) * (p.b / BM) * (p.trsm_par ? p.b / BN : 1);
  if (p.mode == GEMM_LIST && p.trsm_next) return p.trsm_count * (p.b / BM) * (p.trsm_par ? p.b / BN : 1);
  if (p.mode == GEMM_RECT_TRAIL && p.trsm_next) return (int64_t)p.Tm * (p.b / BM);
  return 0;
}
// a trailing update with the next panel's solve appended as gated tasks
__host__ __device__ __forceinline__ bool gemm_fused_trsm(const GemmProblem& p) {
  return (p.mode == GEMM_CHOL_TRAIL || p.mode == GEMM_RECT_TRAIL || p.mode == GEMM_LIST) && p.trsm_next;
}
// Queue position of the fused TRSM tasks in a trailing-update launch: after
// every block of tile column J+1 (their inputs) and early enough that the
// last ~trsm_tail update blocks, small and uniform, fill the launch's tail
// instead of the large TRSM tasks.
__host__ __device__ __forceinline__ int64_t gemm_trsm_pos(const GemmProblem& p) {
  const int64_t nupd = gemm_num_items(p);
  // blocks of the tiles the solve reads: tile column J+1 (Cholesky) or row
  // block J+1 of the transposed right-hand side (kriging solve)
  const int64_t col_tiles = p.mode == GEMM_RECT_TRAIL ? p.Tm : (p.mode == GEMM_LIST ? p.col_items : p.T - p.J - 1);
  const int64_t col = col_tiles * (p.b / BM) * (p.b / BN);
  const int64_t pos = nupd - p.trsm_tail;
  return pos > col ? pos : (col < nupd ? col : nupd);
}
// task -> (is TRSM, index among its kind)
__host__ __device__ __forceinline__ bool gemm_task_kind(const GemmProblem& p, int64_t task, int64_t& idx) {
  if (p.mode == GEMM_TRSM_PANEL) {
    idx = task;
    return true;
  }
  if (!gemm_fused_trsm(p)) {
    idx = task;
    return false;
  }
  const int64_t pos = gemm_trsm_pos(p), ntrsm = gemm_trsm_tasks(p);
  if (task < pos) {
    idx = task;
    return false;
  }
  if (task < pos + ntrsm) {
    idx = task - pos;
    return true;
  }
  idx = task - ntrsm;
  return false;
}

__host__ __device__ __forceinline__ int64_t gemm_step_tasks(const GemmProblem& p) {
  return p.mode == GEMM_TRSM_PANEL ? gemm_trsm_tasks(p) : gemm_num_items(p) + gemm_trsm_tasks(p);
}

// Multi-step launch (nsteps > 1): the view of step s as a one-step problem
// (its update by panel s, then the solve of panel s+1 unless s+1 is the last
// tile row); the TRSM tasks follow the step's column-(s+1) blocks directly
// (no tail filler: these steps are chain-bound).
__host__ __device__ __forceinline__ void multi_step_view(const GemmProblem& p, int s, GemmProblem& ps) {
  ps = p;
  ps.J = s;
  ps.nsteps = 1;
  ps.trsm_next = (s + 2 < p.T);
  ps.trsm_tail = 0;
}
// task -> step s and the task's index inside step s's list
__host__ __device__ __forceinline__ int multi_locate(const GemmProblem& p, int64_t task, GemmProblem& ps,
                                                     int64_t& local) {
  int s = p.J;
  for (;;) {
    multi_step_view(p, s, ps);
    const int64_t n = gemm_step_tasks(ps);
    if (task < n || s + 1 >= p.J + p.nsteps) break;
    task -= n;
    ++s;
  }
  local = task;
  return s;
}

__host__ __device__ __forceinline__ int64_t gemm_num_tasks(const GemmProblem& p) {
  if (p.mode == GEMM_CHOL_TRAIL && p.nsteps > 1) {
    int64_t n = 0;
    GemmProblem ps;
    for (int s = p.J; s < p.J + p.nsteps; ++s) {
      multi_step_view(p, s, ps);
      n += gemm_step_tasks(ps);
    }
    return n;
  }
  return gemm_step_tasks(p);
}

// diagonal-tile block (bi, bj): skip blocks strictly above the diagonal,
// mask the ones that straddle it
__device__ __forceinline__ void diag_block(Item& it, int bi, int bj) {
  if (bi * BM + BM - 1 < bj * BN) it.valid = false;
  it.lower = (bi * BM < bj * BN + BN - 1);
}

// TRSM block: slab task `task` (tile task / nbm, rows (task % nbm) * BM) of
// the panel starting at tile index panel0, column block pass-th from the right
__device__ __forceinline__ void trsm_block(Item& it, const GemmProblem& p, int64_t task, int pass,
                                           int64_t panel0) {
  const int nbn = p.b / BN, nbm = p.b / BM;
  const int bjj = nbn - 1 - pass;
  it.mrow0 = (int)(task % nbm) * BM;
  it.nrow0 = bjj * BN;
  it.cTile = it.aTile0 = (int)(panel0 + task / nbm);
  it.bTile0 = 0;                     // Linv (single tile)
  it.kstages = (bjj + 1) * BN / BK;  // Linv(n, k) = 0 for k > n
  it.store = 1;
  it.bLinv = 1;
}

// Order of the trailing triangle's k(k+1)/2 tiles in a Cholesky update
// launch: tile column J+1 first (the next panel: its blocks gate the
// look-ahead POTRF and solve), then super-columns of sw tile columns, each
// swept top to bottom, row by row.  A super-column's sw panel tiles (the B
// operands) stay in L2 while each row's panel tile (the A operand) is read
// from HBM once per super-column instead of once per tile column: the k-tile
// panel (233 MB at C4's first steps) exceeds L2, and a column-by-column sweep
// re-read it k/2 times (1.5x the algorithmic bytes per launch, round 1).
// The permutation changes no arithmetic: every C tile still receives one
// update per step.
__device__ __forceinline__ void trail_order(int64_t t, int k, int sw, int& rr, int& cc) {
  if (t < k) {
    rr = (int)t;
    cc = 0;
    return;
  }
  t -= k;
  for (int c0 = 1; c0 < k; c0 += sw) {
    const int w = min(sw, k - c0);
    const int64_t tri = (int64_t)w * (w + 1) / 2;  // rows c0 .. c0+w-1: row c0+i holds i+1 tiles
    const int64_t n = tri + (int64_t)(k - c0 - w) * w;
    if (t < n) {
      if (t < tri) {
        int i = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
        while ((int64_t)(i + 1) * (i + 2) / 2 <= t) ++i;
        while ((int64_t)i * (i + 1) / 2 > t) --i;
        rr = c0 + i;
        cc = c0 + (int)(t - (int64_t)i * (i + 1) / 2);
      } else {
        const int64_t u = t - tri;
        rr = c0 + w + (int)(u / w);
        cc = c0 + (int)(u % w);
      }
      return;
    }
    t -= n;
  }
  rr = cc = 0;  // unreachable for t < k(k+1)/2
}

// Block `pass` of task `task`.
__device__ __forceinline__ Item gemm_decode(const GemmProblem& p, int64_t task, int pass) {
  const int nbn = p.b / BN;
  const int nblk = (p.b / BM) * nbn;
  Item it;
  it.aStride = it.bStride = 0;
  it.nkt = 1;
  it.valid = true;
  it.pad = false;
  it.subst = false;
  it.lower = 0;
  it.bTriRow = -1;
  it.aTriRow = -1;
  it.triCol0 = 0;
  it.kstages = 0;
  it.store = (p.beta == 0.0);
  it.bLinv = 0;
  it.gate = -1;
  it.slab = -1;
  it.pass = 0;
  int64_t idx;
  if (gemm_task_kind(p, task, idx)) {
    // standalone panel, or the fused TRSM of panel J+1 (tiles J+2 .. T-1)
    if ((p.mode == GEMM_TRSM_PANEL && p.trsm_oop) || gemm_par_passes(p)) {
      pass = (int)(idx % nbn);  // one pass per task, right to left within a slab
      idx /= nbn;
      if (gemm_par_passes(p)) {
        it.slab = (int)idx;
        it.pass = pass;
      }
    }
    const int64_t panel0 = (p.mode == GEMM_TRSM_PANEL || p.mode == GEMM_LIST) ? p.panel0
                           : p.mode == GEMM_RECT_TRAIL                       ? (int64_t)(p.J + 1) * p.Tm
                                                                             : tri_index(p.J + 2, p.J + 1, p.T);
    trsm_block(it, p, idx, pass, panel0);
    it.subst = (p.mode == GEMM_CHOL_TRAIL || p.mode == GEMM_LIST || p.mode == GEMM_TRSM_PANEL) && p.trsm_subst;
    // Cholesky sweep: slabs of the last tile row that lie wholly in the
    // padding hold zeros and solve to zeros -- skipped
    if (p.mode == GEMM_CHOL_TRAIL && p.n_live > 0 &&
        (int64_t)(p.J + 2 + (int)(idx / (p.b / BM))) == p.T - 1 &&
        (int64_t)(p.T - 1) * p.b + it.mrow0 >= p.n_live)
      it.valid = false, it.pad = true;
    return it;
  }
  const int64_t t = idx / nblk;
  const int blk = (int)(idx % nblk);
  const int bi = blk / nbn, bj = blk % nbn;
  it.mrow0 = bi * BM;
  it.nrow0 = bj * BN;
  switch (p.mode) {
    case GEMM_CHOL_TRAIL: {
      int rr, cc;
      if (p.pair_cols > 0) {
        tri_decode(t, p.T - p.J - 1, rr, cc);  // the first columns, column by column
      } else {
        // super-column width: ~16 MB of panel tiles per merged panel depth
        // (8 .. 64 tiles; 2 .. 64 when several panels are merged)
        const int depth = p.pair_merge + 1;
        const int sw = max(depth > 1 ? 2 : 8, min(64, (int)((16ll << 20) / ((int64_t)depth * p.b * p.b * 8))));
        trail_order(t, p.T - p.J - 1, sw, rr, cc);
      }
      const int R = p.J + 1 + rr, C = p.J + 1 + cc;
      it.cTile = tri_index(R, C, p.T);
      if (p.pair_merge && cc >= 1) {
        // panels J-m .. J in one pass (k = (m+1) b); the k tile kt of a row
        // is its tile in panel J-m+kt (tri_index per k tile: the packed
        // triangle's column starts are not equally spaced)
        it.aTile0 = tri_index(R, p.J - p.pair_merge, p.T);
        it.bTile0 = tri_index(C, p.J - p.pair_merge, p.T);
        it.nkt = p.pair_merge + 1;
        it.aTriRow = R;
        it.bTriRow = C;
        it.triCol0 = p.J - p.pair_merge;
      } else {
        it.aTile0 = tri_index(R, p.J, p.T);
        it.bTile0 = tri_index(C, p.J, p.T);
      }
      if (R == C) diag_block(it, bi, bj);
      if (cc == 0 && p.col_gate) it.gate = rr;  // column J+1: POTRF / TRSM of the next panel wait on it
      // blocks of the last tile row wholly in the identity padding: their
      // panel rows are zero, so the update is exactly zero -- skipped (about
      // 1.4 % of the flops at C4, b = 512)
      if (p.n_live > 0 && R == p.T - 1 && (int64_t)R * p.b + it.mrow0 >= p.n_live && it.valid)
        it.valid = false, it.pad = true;
      break;
    }
    case GEMM_RECT_TRAIL: {
      const int a = (int)(t % p.Tm);
      const int I = p.J + 1 + (int)(t / p.Tm);
      it.cTile = I * p.Tm + a;
      it.aTile0 = p.J * p.Tm + a;
      it.bTile0 = tri_index(I, p.J, p.T);
      if (I == p.J + 1 && p.col_gate) it.gate = a;  // row block J+1: the fused solve waits on it
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
      if (rr == cc) diag_block(it, bi, bj);
      break;
    }
    case GEMM_TRMM_RECT: {  // Y^T(a, I) = sum_{J <= I} X^T(a, J) L(I, J)^T
      const int a = (int)(t % p.Tm);
      const int I = (int)(t / p.Tm);
      it.cTile = I * p.Tm + a;
      it.aTile0 = a;
      it.aStride = p.Tm;
      it.nkt = I + 1;
      it.bTile0 = 0;
      it.bTriRow = I;
      break;
    }
    default: {  // GEMM_LIST: (C, A, B, flags) tile-index quadruples
      // flags: bit 0 the C tile is a diagonal tile (lower part only); bits
      // 8.. gate + 1 (0: none): the column-(J+1) tiles of a distributed
      // sweep step, gate 0 the diagonal tile, 1.. the rank's panel tiles
      const int32_t* q = p.items + 4 * t;
      it.cTile = q[0];
      it.aTile0 = q[1];
      it.bTile0 = q[2];
      if (q[3] & 1) diag_block(it, bi, bj);
      if (p.col_gate) it.gate = (q[3] >> 8) - 1;
      break;
    }
  }
  return it;
}

__device__ __forceinline__ int gemm_task_passes(const GemmProblem& p, int64_t task) {
  int64_t idx;
  return (gemm_task_kind(p, task, idx) && !(p.mode == GEMM_TRSM_PANEL && p.trsm_oop) && !gemm_par_passes(p) &&
          !((p.mode == GEMM_CHOL_TRAIL || p.mode == GEMM_LIST || p.mode == GEMM_TRSM_PANEL) && p.trsm_subst))
             ? p.b / BN
             : 1;
}

// spin (acquire, exponential back-off, bounded) until *flag >= need or the
// factorization failed; returns false on failure / timeout.  A timeout is a
// dependency bug, not data: it is recorded in the status (host: an error).
__device__ __forceinline__ bool wait_count(const int* flag, int need, unsigned long long* info) {
  unsigned ns = 32;
  for (long long spins = 0; ld_acquire_gpu(flag) < need; ++spins) {
    if (info && *(volatile const unsigned long long*)info != 0ull) return false;
    if (spins > (1ll << 24)) {
      if (info) atomicCAS(info, 0ull, BGP_INFO_DATAFLOW_TIMEOUT);
      return false;
    }
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
  }
  return true;
}

// Per-lane byte offset of MMA fragment element (row p*8 + q of a 16-row TMA
// box, k = 2*s4 + t, t = 0, 1) inside a 128B-swizzled box whose 128-byte
// lines are k (operands) or n (C buffer):
//   line*128 + (((p<<2) ^ ((q>>1) ^ k)) << 4) + (q&1)*8.
// k-lines 8..15 of a BK = 16 box repeat the swizzle of lines 0..7, so the
// k4 half-steps t + 2 sit exactly 1024 bytes after half-steps t.
__device__ __forceinline__ uint32_t lane_off(int p, int t, int q, int s4) {
  const int k = 2 * s4 + t;
  return (uint32_t)(k * 128 + ((((p << 2) ^ ((q >> 1) ^ k)) & 7) << 4) + ((q & 1) << 3));
}

// tensor maps of the panel push destinations (GEMM_TRSM_PANEL, npush > 0)
struct PushMaps {
  CUtensorMap map[BGP_MAX_PUSH];
  double* ptr[BGP_MAX_PUSH];  // the same destinations as raw pointers (substitution panel solve)
};

// What the consumers need of a block, decoded once by the producer and
// handed over with the block's first stage (written before the `full` arrive)
struct BlockSlot {
  int valid;  // 0: no more work
  int cTile, mrow0, nrow0;
  int nk;     // BK stages
  int lower, store, gate;
  int slab, pass;  // trsm_par: slab index and pass (-1: not a parallel TRSM pass)
  int pad[2];
};
static_assert(sizeof(BlockSlot) == 48, "slot size");

struct GroupSmem {
  uint8_t* stages;
  uint8_t* cbuf;
  uint64_t* full;
  uint64_t* empty;
  BlockSlot* slot;  // per stage: the block starting there
};

__device__ __forceinline__ GroupSmem group_smem(uint8_t* smem, int g) {
  GroupSmem gs;
  gs.stages = smem + g * GROUP_BYTES;
  gs.cbuf = gs.stages + STAGES * STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + GROUPS * GROUP_BYTES) + g * (2 * STAGES);
  gs.full = bars;
  gs.empty = bars + STAGES;
  gs.slot = reinterpret_cast<BlockSlot*>(smem + GROUPS * GROUP_BYTES + 256) + g * STAGES;  // 16-byte aligned
  return gs;
}

__device__ __forceinline__ uint64_t* stagger_bar(uint8_t* smem) {
  return reinterpret_cast<uint64_t*>(smem + GROUPS * GROUP_BYTES) + GROUPS * 2 * STAGES;
}

// tmT: the C tiles with the operand box -- the A operand of an in-place TRSM
// block (the tile it solves), which differs from tmA when A / B are a panel
// buffer (the distributed sweep step)
// MULTI: the multi-step launch (nsteps > 1) -- a separate instantiation so
// the one-step path's code is unchanged by the per-task step lookup
template <bool MULTI>
__device__ __forceinline__ void producer_loop(const GroupSmem& gs, const CUtensorMap* tmA,
                                              const CUtensorMap* tmB, const CUtensorMap* tmL,
                                              const CUtensorMap* tmT, const GemmProblem& p,
                                              unsigned long long* info, uint64_t* stagger) {
  prefetch_tmap(tmA);
  prefetch_tmap(tmB);
  prefetch_tmap(tmL);
  prefetch_tmap(tmT);
  const uint64_t pol_keep = l2_policy_evict_last();
  const int kc_per_tile = p.b / BK;
  const int64_t ntasks = gemm_num_tasks(p);
  int stage = 0;
  uint32_t phase = 0;
  constexpr bool multi = MULTI;
  GemmProblem ps;  // multi: the claimed task's step as a one-step problem
  for (;;) {
    int64_t task = atomicAdd(reinterpret_cast<unsigned long long*>(p.queue), 1ull);
    if (task >= ntasks) break;
    int step = p.J;
    if constexpr (MULTI) step = multi_locate(p, task, ps, task);
    const GemmProblem& q = MULTI ? ps : p;
    int64_t idx;
    if (gemm_fused_trsm(q) && gemm_task_kind(q, task, idx)) {
      // fused TRSM of panel J+1: the tile's update blocks have retired and
      // (Cholesky) the look-ahead CTA published Linv(J+1); the kriging solve's
      // inverses are computed up front (no flag)
      const int per_tile = (p.b / BM) * (gemm_par_passes(q) ? p.b / BN : 1);
      const int tile = (int)(idx / per_tile);
      if (stagger) {  // group 0: release group 1 before blocking (see consumer_loop)
        mbar_arrive(stagger);
        stagger = nullptr;
      }
      if (multi) {  // tile (step+2+tile, step+1): the updates of steps J .. step retired
        const int64_t t = tri_index(step + 2 + tile, step + 1, p.T) - p.cnt_base;
        if (!wait_count(p.tile_cnt + t, (step + 1 - p.J) * p.tile_need, info)) break;
      } else {
        const int g0 = p.mode == GEMM_RECT_TRAIL ? 0 : 1;  // Cholesky gate 0 is the diagonal tile
        if (!wait_count(p.col_gate + g0 + tile, p.tile_need, info) ||
            (p.linv_flag && !p.trsm_subst && !wait_count(p.linv_flag, p.linv_need, info)))
          break;
      }
      fence_proxy_async_global();
    } else if (multi && step > p.J) {
      // update by panel `step`, solved inside this launch: wait for its two
      // panel tiles (generic stores of the substitution -> TMA reads)
      const Item i0 = gemm_decode(q, task, 0);
      if (i0.valid) {
        if (stagger) {
          mbar_arrive(stagger);
          stagger = nullptr;
        }
        if (!wait_count(p.solved + (i0.aTile0 - p.cnt_base), p.solved_need, info) ||
            !wait_count(p.solved + (i0.bTile0 - p.cnt_base), p.solved_need, info))
          break;
        fence_proxy_async_global();
      }
    }
    const int npass = gemm_task_passes(q, task);
    for (int pass = 0; pass < npass; ++pass) {
      Item it = gemm_decode(q, task, pass);
      // multi: every update block counts toward its C tile (solves and
      // factorizations of later steps wait on them)
      if (multi && !it.subst && !it.bLinv) it.gate = (int)(it.cTile - p.cnt_base);
      if (!it.valid) {
        // a padding block counts toward its tile's gate as if it had retired
        if (it.pad && it.gate >= 0) atomicAdd(p.col_gate + it.gate, GROUP_WARPS);
        // (multi) a padding slab counts as solved
        if (it.pad && multi && it.subst) atomicAdd(p.solved + (it.cTile - p.cnt_base), GROUP_WARPS);
        continue;
      }
      if (it.subst) {
        // substitution slab: no operand stages, the consumers read the tile,
        // the factor and Dinv themselves as the POTRF publishes them
        mbar_wait(&gs.empty[stage], phase ^ 1);
        BlockSlot& sl = gs.slot[stage];
        sl.valid = 1;
        sl.cTile = it.cTile;
        sl.mrow0 = it.mrow0;
        sl.nrow0 = 0;
        sl.nk = 0;
        sl.lower = sl.store = 0;
        sl.gate = -1;
        sl.slab = -1;
        sl.pass = 0;
        sl.pad[0] = 1;
        sl.pad[1] = step - p.J;  // multi: the step (its factor, Dinv and progress)
        mbar_arrive(&gs.full[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
        continue;
      }
      const CUtensorMap* tb = it.bLinv ? tmL : tmB;
      const CUtensorMap* ta = (it.bLinv && !p.trsm_oop) ? tmT : tmA;
      const int nk = it.kstages > 0 ? it.kstages : it.nkt * kc_per_tile;
      // k tiles outer (their tile indices computed once per k tile), BK
      // stages inner
      int kc = 0;
      for (int kt = 0; kc < nk; ++kt) {
        const int at = it.aTriRow >= 0 ? (int)tri_index(it.aTriRow, it.triCol0 + kt, q.T)
                                       : (int)(it.aTile0 + kt * it.aStride);
        const int bt = it.bTriRow >= 0 ? (int)tri_index(it.bTriRow, it.triCol0 + kt, q.T)
                                       : (int)(it.bTile0 + kt * it.bStride);
        BGP_CHECK(at >= 0 && at < (ta == tmT ? p.nC : p.nA));
        BGP_CHECK(bt >= 0 && bt < (it.bLinv ? 1 : p.nB));
        BGP_CHECK(it.mrow0 >= 0 && it.mrow0 + BM <= p.b && it.nrow0 >= 0 && it.nrow0 + BN <= p.b);
        for (int kin = 0; kin < p.b && kc < nk; kin += BK, ++kc) {
          mbar_wait(&gs.empty[stage], phase ^ 1);
          if (kc == 0) {  // read by the consumers after `full`
            BlockSlot& sl = gs.slot[stage];
            sl.valid = 1;
            sl.cTile = it.cTile;
            sl.mrow0 = it.mrow0;
            sl.nrow0 = it.nrow0;
            sl.nk = nk;
            sl.lower = it.lower;
            sl.store = it.store;
            sl.gate = it.gate;
            sl.slab = it.slab;
            sl.pass = it.pass;
            sl.pad[0] = 0;
          }
          mbar_arrive_expect_tx(&gs.full[stage], STAGE_BYTES);
          BGP_CHECK(kin + BK <= p.b);
          uint8_t* sa = gs.stages + stage * STAGE_BYTES;
          uint8_t* sb = sa + STAGE_A_BYTES;
#pragma unroll
          for (int i = 0; i < BM / 16; ++i)
            tma_load_3d(sa + i * BOX_BYTES, ta, &gs.full[stage], it.mrow0 + i * 16, kin, at, pol_keep);
#pragma unroll
          for (int i = 0; i < BN / 16; ++i)
            tma_load_3d(sb + i * BOX_BYTES, tb, &gs.full[stage], it.nrow0 + i * 16, kin, bt, pol_keep);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  }
  // no more work: hand the consumers a sentinel through the next stage
  mbar_wait(&gs.empty[stage], phase ^ 1);
  gs.slot[stage].valid = 0;
  mbar_arrive(&gs.full[stage]);
}

// ld.shared.f64 at a register base plus an immediate; volatile so it keeps
// its place between the (volatile) DMMAs of the software pipeline below
template <int OFF>
__device__ __forceinline__ double lds64(uint32_t base) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(base), "n"(OFF) : "memory");
  return v;
}

// one k4 half-step's fragments: A rows i*8.. of the warp tile (box i>>1,
// row-pair i&1), B columns j*8..
struct Frag {
  double a[MI], b[NJ];
};

template <int H2>  // k lines 8*H2 .. 8*H2 + 7 of the stage
__device__ __forceinline__ void load_frag(Frag& f, uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1) {
  constexpr int K = H2 * 1024;
  f.a[0] = lds64<K>(a0);
  f.a[1] = lds64<K>(a1);
  f.a[2] = lds64<K + BOX_BYTES>(a0);
  f.a[3] = lds64<K + BOX_BYTES>(a1);
  if constexpr (MI == 8) {
    f.a[4] = lds64<K + 2 * BOX_BYTES>(a0);
    f.a[5] = lds64<K + 2 * BOX_BYTES>(a1);
    f.a[6] = lds64<K + 3 * BOX_BYTES>(a0);
    f.a[7] = lds64<K + 3 * BOX_BYTES>(a1);
  }
  f.b[0] = lds64<K>(b0);
  f.b[1] = lds64<K>(b1);
  f.b[2] = lds64<K + BOX_BYTES>(b0);
  f.b[3] = lds64<K + BOX_BYTES>(b1);
}

__device__ __forceinline__ void mma_frag(double (&acc)[MI][NJ][2], const Frag& f) {
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) dmma884(acc[i][j][0], acc[i][j][1], f.a[i], f.b[j]);
}

template <int OFF>
__device__ __forceinline__ void sts64(uint32_t base, double v) {
  asm volatile("st.shared.f64 [%0+%1], %2;" ::"r"(base), "n"(OFF), "d"(v) : "memory");
}

// Stage the 8-row blocks i = R*NII + ii (ii < NII) of the warp's 64x32
// accumulator tile into its epilogue slice: NII/2 16x32 boxes, 128B swizzled
// like the operands (line = column n).  cb[p][e] are the lane's addresses of
// (row-pair p, column parity e) in box 0, column block j = 0.  NEG stages
// -acc (integer sign flip, no FP64 instruction); MASK zeroes the strict upper
// triangle of a diagonal tile (m < n).
template <int R, bool NEG, bool MASK, int II = 0, int J = 0>
__device__ __forceinline__ void stage_rows(const double (&acc)[MI][NJ][2], const uint32_t (&cb)[2][2], int m0,
                                           int n0) {
  constexpr int NII = EPI_ROWS / 8;
  if constexpr (II < NII && J < NJ) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double v = acc[R * NII + II][J][e];
      if (NEG) v = __longlong_as_double(__double_as_longlong(v) ^ (long long)0x8000000000000000ull);
      if (MASK && m0 + II * 8 < n0 + J * 8 + e) v = 0.0;
      // immediate offset: box (II >> 1), column block J
      sts64<(II >> 1) * WBOX_BYTES + J * 1024>(cb[II & 1][e], v);
    }
    stage_rows<R, NEG, MASK, II, J + 1>(acc, cb, m0, n0);
  } else if constexpr (II < NII) {
    stage_rows<R, NEG, MASK, II + 1, 0>(acc, cb, m0, n0);
  }
}

// epilogue round R: stage (NEG / MASK chosen per block) then TMA the boxes
template <int R>
__device__ __forceinline__ void stage_round(const double (&acc)[MI][NJ][2], const uint32_t (&cb)[2][2], int m0,
                                            int n0, bool store, bool lower) {
  if constexpr (R >= EPI_ROUNDS) return;
  else if (store) {
    if (lower) stage_rows<R, false, true>(acc, cb, m0, n0);
    else stage_rows<R, false, false>(acc, cb, m0, n0);
  } else {
    if (lower) stage_rows<R, true, true>(acc, cb, m0, n0);
    else stage_rows<R, true, false>(acc, cb, m0, n0);
  }
}

// half-steps H .. HALVES-2 of a stage: load the fragments of H+1, issue the
// DMMAs of H (compile-time recursion so every offset is an immediate)
template <int H, typename Hook>
__device__ __forceinline__ void stage_halves(Frag (&f)[2], double (&acc)[MI][NJ][2], const uint32_t (&offA)[2][2],
                                             const uint32_t (&offB)[2][2], uint32_t sb, Hook&& hook) {
  if constexpr (H + 1 < HALVES) {
    constexpr int N = H + 1;
    load_frag<(N >> 1)>(f[N & 1], offA[0][N & 1] + sb, offA[1][N & 1] + sb, offB[0][N & 1] + sb,
                        offB[1][N & 1] + sb);
    mma_frag(acc, f[H & 1]);
    if constexpr (H == 2) hook();  // a few k4 steps into the stage
    stage_halves<H + 1>(f, acc, offA, offB, sb, hook);
  }
}

// Panel solve by substitution for one warp: rows r0 .. r0+31 of the panel
// tile X (in place), X_k = (A_k - sum_{j<k} X_j L_kj^T) Dinv_k^T over the
// 32-column blocks k of the diagonal tile L = p.potrf_tile, each block as
// soon as the look-ahead POTRF has published it (p.potrf_progress > k), so
// the solve finishes about one block after the factorization instead of
// after a full tile inverse (bg/distla/kernels.py:163-164).  Fragments:
// DMMA 8x8x4, acc[tr][tc][e] = C(tr*8 + q, tc*8 + 2 s4 + e).
// With npush > 0 every solved block is also stored into tile `slot` of each
// destination panel buffer (the distributed sweep's exchange, plain stores
// to peer memory over NVLink).
__device__ __noinline__ void trsm_subst_rows(int b, const double* __restrict__ Ld, const double* __restrict__ Dv,
                                             const int* progress, double* __restrict__ X, int r0, int lane,
                                             unsigned long long* info, const PushMaps* pm, int npush,
                                             int64_t slot) {
  const int nbk = b / 32;
  const int q = lane >> 2, s4 = lane & 3;
  double* Xr = X + r0;
  for (int k = 0; k < nbk; ++k) {
    bool ok = true;
    if (lane == 0) ok = wait_count(progress, k + 1, info);
    if (!__shfl_sync(0xffffffffu, ok ? 1 : 0, 0)) return;  // factorization failed
    __syncwarp();  // lane 0's acquire orders every lane's reads below (all from L2)
    double acc[4][4][2];
#pragma unroll
    for (int tr = 0; tr < 4; ++tr)
#pragma unroll
      for (int tc = 0; tc < 4; ++tc)
#pragma unroll
        for (int e = 0; e < 2; ++e) acc[tr][tc][e] = __ldcg(Xr + (int64_t)(32 * k + tc * 8 + 2 * s4 + e) * b + tr * 8 + q);
    for (int j = 0; j < k; ++j) {  // acc -= X_j L_kj^T
#pragma unroll
      for (int kh = 0; kh < 2; ++kh) {
        double av[4][4], bv[4][4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const int kc = 32 * j + 16 * kh + 4 * kk + s4;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            av[kk][t] = -__ldcg(Xr + (int64_t)kc * b + t * 8 + q);
            bv[kk][t] = __ldcg(Ld + (int64_t)kc * b + 32 * k + t * 8 + q);
          }
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
          for (int tr = 0; tr < 4; ++tr)
#pragma unroll
            for (int tc = 0; tc < 4; ++tc) dmma884(acc[tr][tc][0], acc[tr][tc][1], av[kk][tr], bv[kk][tc]);
      }
    }
    // X_k = acc Dinv_k^T: acc to A fragments within each quad (A(row, c) for
    // c = 4 kk + s4 sits in lane ((kk & 1) * 2 + (s4 >> 1)) of the quad,
    // element s4 & 1 of column tile kk >> 1)
    double out[4][4][2];
#pragma unroll
    for (int tr = 0; tr < 4; ++tr)
#pragma unroll
      for (int tc = 0; tc < 4; ++tc) out[tr][tc][0] = out[tr][tc][1] = 0.0;
    const double* Dk = Dv + (int64_t)k * 1024;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int src = (lane & ~3) | ((kk & 1) * 2 + (s4 >> 1));
      double af[4], bd[4];
#pragma unroll
      for (int tr = 0; tr < 4; ++tr) {
        const double v0 = __shfl_sync(0xffffffffu, acc[tr][kk >> 1][0], src);
        const double v1 = __shfl_sync(0xffffffffu, acc[tr][kk >> 1][1], src);
        af[tr] = (s4 & 1) ? v1 : v0;
      }
#pragma unroll
      for (int tc = 0; tc < 4; ++tc) bd[tc] = __ldcg(Dk + (4 * kk + s4) * 32 + tc * 8 + q);  // Dinv_k^T
#pragma unroll
      for (int tr = 0; tr < 4; ++tr)
#pragma unroll
        for (int tc = 0; tc < 4; ++tc) dmma884(out[tr][tc][0], out[tr][tc][1], af[tr], bd[tc]);
    }
#pragma unroll
    for (int tr = 0; tr < 4; ++tr)
#pragma unroll
      for (int tc = 0; tc < 4; ++tc)
#pragma unroll
        for (int e = 0; e < 2; ++e) Xr[(int64_t)(32 * k + tc * 8 + 2 * s4 + e) * b + tr * 8 + q] = out[tr][tc][e];
    for (int d = 0; d < npush; ++d) {
      double* Pr = pm->ptr[d] + slot * b * b + r0;
#pragma unroll
      for (int tr = 0; tr < 4; ++tr)
#pragma unroll
        for (int tc = 0; tc < 4; ++tc)
#pragma unroll
          for (int e = 0; e < 2; ++e) Pr[(int64_t)(32 * k + tc * 8 + 2 * s4 + e) * b + tr * 8 + q] = out[tr][tc][e];
    }
    __syncwarp();  // X_k visible to the warp's lanes before the next blocks read it
  }
}

template <bool MULTI>
__device__ __forceinline__ void consumer_loop(const GroupSmem& gs, int g, int gwarp, int lane,
                                              const CUtensorMap* tmC, const GemmProblem& p,
                                              uint64_t* stagger, const PushMaps* pm,
                                              unsigned long long* info) {
  static_assert((MI == 8 || MI == 4) && NJ == 4 && WN / 16 == 2, "load_frag: 64x32 or 32x32 warp tiles");
  const int wm = gwarp % WARPS_M, wn = gwarp / WARPS_M;
  const int q = lane >> 2, s4 = lane & 3;
  // per-lane shared addresses of the fragments in stage 0 (t = k4 half-step)
  const uint32_t st0 = smem_u32(gs.stages);
  uint32_t offA[2][2], offB[2][2];
#pragma unroll
  for (int pp = 0; pp < 2; ++pp)
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      offA[pp][t] = st0 + (uint32_t)(wm * (WM / 16) * BOX_BYTES) + lane_off(pp, t, q, s4);
      offB[pp][t] = st0 + (uint32_t)(STAGE_A_BYTES + wn * (WN / 16) * BOX_BYTES) + lane_off(pp, t, q, s4);
    }
  uint8_t* cw = gs.cbuf + gwarp * WSTAGE_BYTES;
  uint32_t coff[2][2];
#pragma unroll
  for (int pp = 0; pp < 2; ++pp)
#pragma unroll
    for (int e = 0; e < 2; ++e) coff[pp][e] = lane_off(pp, e, q, s4);
  int stage = 0;
  uint32_t phase = 0;
  bool store_pending = false;
  int held = -1;  // EPI_IN_STAGE: stage still holding this warp's epilogue rows
  // release the held stage once its bulk reads are done (early in the next block)
  auto release_held = [&]() {
    if (EPI_IN_STAGE && held >= 0) {
      if (lane == 0) {
        tma_store_wait_read0();
        mbar_arrive(&gs.empty[held]);
      }
      __syncwarp();
      held = -1;
    }
  };
  const uint64_t pol_stream = l2_policy_evict_first();
  // Stagger: every block costs the same, so two groups that start together
  // would hit their epilogues together and leave the DMMA pipe idle.  Group 1
  // starts once group 0 is half-way through its first block.  The barrier
  // (count 1) also completes when group 0 has no block at all, and when group
  // 0's producer is about to wait on a gate, so group 1 never waits on a
  // group that itself waits (the gated work may be group 1's own).
  bool stagger_arrive = (g == 0 && gwarp == 0);
  if (g == 1) mbar_wait(stagger, 0);

  for (;;) {
    mbar_wait(&gs.full[stage], phase);  // first stage of the next block (or the sentinel)
    const BlockSlot it = gs.slot[stage];
    if (!it.valid) break;
    if (it.pad[0]) {  // fused TRSM slab by substitution: 32 rows per warp
      release_held();
      if (stagger_arrive) {
        __syncwarp();
        if (lane == 0) mbar_arrive(stagger);
        stagger_arrive = false;
      }
      // the step's factor, Dinv blocks and progress counter (multi: step J + pad[1])
      const int so = MULTI ? it.pad[1] : 0;
      const double* ptile = MULTI ? p.cbase + tri_index(p.J + so + 1, p.J + so + 1, p.T) * p.b * p.b : p.potrf_tile;
      trsm_subst_rows(p.b, ptile, p.dinv + (int64_t)so * p.b * 32, p.potrf_progress + so,
                      p.cbase + (int64_t)it.cTile * p.b * p.b, it.mrow0 + 32 * gwarp, lane, info, pm, p.npush,
                      (int64_t)it.cTile - p.panel0);
      __syncwarp();
      if (MULTI && lane == 0) {  // rows solved: later steps' update blocks read them by TMA
        __threadfence();
        atomicAdd(p.solved + (it.cTile - p.cnt_base), 1);
      }
      if (lane == 0) mbar_arrive(&gs.empty[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
      continue;
    }
    const int nk = it.nk;
    double acc[MI][NJ][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // Software pipeline over the stage ring.  A stage holds BK / 4 k4
    // half-steps; fragments alternate between two register sets, so the
    // loads of half-step h+1 issue in the DMMA gaps of half-step h.  The wait
    // for stage s+1 sits before the last half-step of stage s, and stage s
    // is released once its last DMMA issued (fragments in registers) -- except
    // the block's last stage under EPI_IN_STAGE, which holds epilogue rows
    // until release_held() early in the next block.
    Frag f[2];
    uint32_t sb = (uint32_t)stage * STAGE_BYTES;
    load_frag<0>(f[0], offA[0][0] + sb, offA[1][0] + sb, offB[0][0] + sb, offB[1][0] + sb);
    for (int kc = 0; kc + 1 < nk; ++kc) {
      const int cur = stage;
      if (stagger_arrive && kc == (nk >> 1)) {
        __syncwarp();
        if (lane == 0) mbar_arrive(stagger);
        stagger_arrive = false;
      }
      stage_halves<0>(f, acc, offA, offB, sb, release_held);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
      sb = (uint32_t)stage * STAGE_BYTES;
      mbar_wait(&gs.full[stage], phase);
      load_frag<0>(f[0], offA[0][0] + sb, offA[1][0] + sb, offB[0][0] + sb, offB[1][0] + sb);
      mma_frag(acc, f[(HALVES - 1) & 1]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&gs.empty[cur]);
    }
    stage_halves<0>(f, acc, offA, offB, sb, release_held);
    mma_frag(acc, f[(HALVES - 1) & 1]);
    const int last = stage;
    if constexpr (EPI_IN_STAGE) {
      // every warp of the group has read its fragments out of the last
      // stage before any warp overwrites it with epilogue rows
      named_bar_sync(3 + g, 32 * GROUP_WARPS);
    } else {
      __syncwarp();
      if (lane == 0) mbar_arrive(&gs.empty[stage]);
    }
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1;
    }

    // Parallel TRSM pass: this warp has read its operands; the block it
    // stores is read by the passes to its right (q < pass), so wait until
    // they have read theirs.  Those passes were queued earlier and never
    // wait on this one.
    if (it.slab >= 0) {
      int* pd = p.pass_done + (int64_t)it.slab * (p.b / BN);
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        atomicAdd(pd + it.pass, 1);
        for (int q = 0; q < it.pass; ++q)
          if (!wait_count(pd + q, GROUP_WARPS, info)) break;
      }
      __syncwarp();
    }

    // ------------------------------- epilogue -------------------------------
    // Per warp (no group barrier), in two rounds of 32 rows: stage the rows in
    // the warp's own 8 KB slice and issue two 16x32 TMA boxes.  Updates
    // (beta = 1): stage -acc and TMA reduce-add it into C in L2 -- no C load,
    // no read-modify-write on the critical path.  Stores (beta = 0, TRSM
    // blocks): TMA store of acc.  A round waits only until the previous
    // round's boxes were read out of shared memory.
#pragma unroll
    for (int r = 0; r < EPI_ROUNDS; ++r) {
      // rounds 0 .. EPI_ROUNDS-2 go to the warp's quarter of the last stage
      // (EPI_IN_STAGE), the last round to its own slice; otherwise every
      // round reuses the slice once the previous round's boxes were read
      const bool in_stage = EPI_IN_STAGE && r + 1 < EPI_ROUNDS;
      uint8_t* wbuf = in_stage ? gs.stages + last * STAGE_BYTES + (gwarp * (EPI_ROUNDS - 1) + r) * WSTAGE_BYTES
                               : cw;
      // (EPI_IN_STAGE: the previous block's reads were waited for when its
      // stage was released, so nothing is pending here)
      if (!EPI_IN_STAGE && lane == 0 && (store_pending || r > 0)) tma_store_wait_read0();  // slice free
      __syncwarp();
      uint32_t cb[2][2];
#pragma unroll
      for (int pp = 0; pp < 2; ++pp)
#pragma unroll
        for (int e = 0; e < 2; ++e) cb[pp][e] = smem_u32(wbuf) + coff[pp][e];
      // row m = m0 + ii*8 of the round, column n = n0 + j*8 + e (tile coordinates)
      const int m0 = it.mrow0 + wm * WM + r * EPI_ROWS + q, n0 = it.nrow0 + wn * WN + 2 * s4;
      switch (r) {
        case 0: stage_round<0>(acc, cb, m0, n0, it.store, it.lower); break;
        case 1: stage_round<1>(acc, cb, m0, n0, it.store, it.lower); break;
        case 2: stage_round<2>(acc, cb, m0, n0, it.store, it.lower); break;
        default: stage_round<3>(acc, cb, m0, n0, it.store, it.lower); break;
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        const int r0 = it.mrow0 + wm * WM + r * EPI_ROWS, c0 = it.nrow0 + wn * WN;
        BGP_CHECK(it.cTile >= 0 && it.cTile < p.nC);
        BGP_CHECK(p.npush == 0 || !it.store || (it.cTile - p.panel0 >= 0 && it.cTile - p.panel0 < p.push_tiles));
#pragma unroll
        for (int b2 = 0; b2 < EPI_BOXES; ++b2) {
          if (it.store) {
            tma_store_3d(tmC, wbuf + b2 * WBOX_BYTES, r0 + b2 * 16, c0, (int)it.cTile, pol_stream);
            // fused panel push: the same box into every destination panel
            // buffer (peer memory over NVLink), from the same staged rows
            for (int d = 0; d < p.npush; ++d)
              tma_store_3d(&pm->map[d], wbuf + b2 * WBOX_BYTES, r0 + b2 * 16, c0, (int)(it.cTile - p.panel0),
                           pol_stream);
          } else
            tma_reduce_add_3d(tmC, wbuf + b2 * WBOX_BYTES, r0 + b2 * 16, c0, (int)it.cTile, pol_stream);
        }
        tma_store_commit();
      }
    }
    store_pending = true;
    if constexpr (EPI_IN_STAGE) held = last;
    // Column-(J+1) gates: a warp signals a block once its bulk reduction has
    // retired (completion, proxy fence, release).  Not deferred: this group's
    // own producer may be the one waiting for the tile.
    if (it.gate >= 0) {
      if (lane == 0) {
        tma_store_wait_all0();
        fence_proxy_async_global();
        __threadfence();
        BGP_CHECK(it.gate < (MULTI ? tri_count(p.T - p.J - 1)
                                          : (p.mode == GEMM_LIST ? p.trsm_count + 1
                                                                 : (p.mode == GEMM_RECT_TRAIL ? p.Tm : p.T))));
        atomicAdd(p.col_gate + it.gate, 1);
      }
      __syncwarp();
    }
  }
  if (stagger_arrive && lane == 0) mbar_arrive(stagger);
  release_held();
  if (lane == 0 && store_pending) tma_store_wait_all0();
  if (p.npush > 0) __threadfence_system();  // pushed panel visible to the peers
}

// MULTI: the multi-step tail launch (nsteps > 1), its own instantiation
template <bool MULTI>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_dmma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmL, const __grid_constant__ CUtensorMap tmC,
                     const __grid_constant__ CUtensorMap tmT,
                     const GemmProblem p, unsigned long long* __restrict__ info,
                     const __grid_constant__ PushMaps pm) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ int s_go, s_role;
  if ((smem_u32(smem) & 1023u) != 0u) __trap();  // 128B swizzle needs 1 KB alignment
  if (info && *(volatile const unsigned long long*)info != 0ull) return;  // factorization failed

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wg = warp >> 2;
  if (threadIdx.x == 0) {
    for (int g = 0; g < GROUPS; ++g) {
      GroupSmem gs = group_smem(smem, g);
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&gs.full[s], 1);
        mbar_init(&gs.empty[s], GROUP_WARPS);
      }
    }
    mbar_init(stagger_bar(smem), 1);
    fence_barrier_init();
    // look-ahead role: the first CTA to start takes it (a CTA that is running
    // for sure -- a fixed block index might only be scheduled once others
    // exit, and those may be waiting for the inverse it publishes)
    s_role = p.potrf_tile != nullptr && atomicAdd(p.role_ticket, 1) == 0;
  }
  __syncthreads();
  // look-ahead CTA: factor (and invert) the next panel's diagonal tile first
  const bool lookahead_cta = s_role != 0;

  if (wg == 0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PRODUCER_REGS));
    if (lookahead_cta) named_bar_sync(1, THREADS);  // wait for the panel work below
    if (warp < GROUPS && lane == 0)
      producer_loop<MULTI>(group_smem(smem, warp), &tmA, &tmB, &tmL, &tmT, p, info,
                           warp == 0 ? stagger_bar(smem) : nullptr);
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CONSUMER_REGS));
    if (lookahead_cta) {
      // the first 256 consumer threads run the tile POTRF (and inverse) on
      // the ring memory once the update blocks of the diagonal tile retired;
      // other CTAs' TRSM tasks wait for the published inverse
      const int ctid = threadIdx.x - 128;
      if (MULTI && ctid < 256) {
        // multi-step launch: factor (K, K) for K = J+1 .. J+nsteps one after
        // another, each once the updates of steps J .. K-1 into it retired;
        // the substitution solves follow each through its progress counter
        double* psm = reinterpret_cast<double*>(smem);
        for (int K = p.J + 1; K <= p.J + p.nsteps && K < p.T; ++K) {
          const int64_t dt = tri_index(K, K, p.T);
          if (ctid == 0) s_go = wait_count(p.tile_cnt + (dt - p.cnt_base), (K - p.J) * p.diag_need, info) ? 1 : 0;
          named_bar_sync(2, 256);
          if (!s_go) break;
          const bool ok = tile_potrf_inv_device(p.cbase + dt * p.b * p.b, p.b, p.potrf_row0 + (int64_t)(K - p.J - 1) * p.b,
                                                p.dinv + (int64_t)(K - p.J - 1) * p.b * 32, info, nullptr, psm, ctid, 2,
                                                p.potrf_progress + (K - p.J - 1));
          named_bar_sync(2, 256);  // (shared memory and s_go reused by the next factorization)
          if (!ok) break;
        }
      } else if (ctid < 256) {
        double* psm = reinterpret_cast<double*>(smem);
        // (no gate: the first panel's POTRF, fused with its substitution solve)
        if (ctid == 0) s_go = p.col_gate ? (wait_count(p.col_gate, p.diag_need, info) ? 1 : 0) : 1;
        named_bar_sync(2, 256);
        const bool la_ok = s_go && tile_potrf_inv_device(p.potrf_tile, p.b, p.potrf_row0, p.dinv, info,
                                                        (p.trsm_next && !p.trsm_subst) ? p.linv : nullptr,
                                                        psm, ctid, 2, p.trsm_subst ? p.potrf_progress : nullptr);
        if (la_ok && p.trsm_next && !p.trsm_subst) {
          __threadfence();
          named_bar_sync(2, 256);
          if (ctid == 0) atomicAdd(p.linv_flag, p.b / 32);
        }
      }
      named_bar_sync(1, THREADS);  // release this CTA's producers
    }
    const int g = wg - 1;
    consumer_loop<MULTI>(group_smem(smem, g), g, warp & 3, lane, &tmC, p, stagger_bar(smem), &pm, info);
  }
}

// One-time function setup.  It also forces the module to load: with CUDA's
// lazy loading, the first launch of a kernel while a spin-waiting kernel runs
// on another stream (the look-ahead POTRF) could otherwise stall behind it.
// blocks of one b x b tile, and of a diagonal tile (the rest lie strictly
// above the diagonal), for the host's gate counts; warps per block
int tile_blocks(int b) { return (b / BM) * (b / BN); }
int diag_blocks(int b) {
  int c = 0;
  for (int bi = 0; bi < b / BM; ++bi)
    for (int bj = 0; bj < b / BN; ++bj) c += (bi * BM + BM - 1 >= bj * BN);
  return c;
}
int block_warps() { return GROUP_WARPS; }
int groups() { return GROUPS; }

void prepare() {
  static int occupancy = -1;
  if (occupancy < 0) {
    for (auto k : {gemm_dmma_kernel<false>, gemm_dmma_kernel<true>}) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
      cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occupancy, gemm_dmma_kernel<false>, THREADS, SMEM_BYTES);
    if (occupancy < 1) fprintf(stderr, "libbgp: gemm_dmma_kernel cannot be resident\n");
  }
}

int launch(Ctx* ctx, const GemmProblem& p_in, double* Cbase, const double* Abase, int64_t nA,
           const double* Bbase, int64_t nB, int64_t nC, cudaStream_t s, const double* Linv) {
  if (p_in.b % BM != 0) return set_err(ctx, "gemm: tile must be a multiple of 128", cudaErrorInvalidValue);
  GemmProblem p = p_in;
  p.cbase = Cbase;
  if (p.nsteps > 1) {
    if (p.mode != GEMM_CHOL_TRAIL || !p.trsm_subst || !p.tile_cnt || !p.solved || !p.potrf_progress ||
        !p.potrf_tile)
      return set_err(ctx, "gemm: bad multi-step launch", cudaErrorInvalidValue);
    p.col_gate = p.tile_cnt;
    p.solved_need = (p.b / BM) * GROUP_WARPS;
    p.cnt_base = tri_index(p.J + 1, p.J + 1, p.T);
  }
  p.nA = nA;
  p.nB = nB;
  p.nC = nC;
  const int64_t tasks = gemm_num_tasks(p);
  if (tasks <= 0) return BGP_OK;
  int rc;
  if (!p.queue || (p.potrf_tile && !p.role_ticket)) {
    // a zeroed task counter (+ look-ahead ticket) of this launch's own: slot
    // k of a ring, zeroed on the launch's stream.  Launches on one stream
    // are ordered; launches on different streams (the caller's overlap)
    // never share a slot unless QUEUE_RING launches are in flight at once.
    if ((rc = ensure(ctx, (void**)&ctx->d_queue_ring, &ctx->queue_ring_cap, Ctx::QUEUE_RING * 16))) return rc;
    int* slot = ctx->d_queue_ring + 4 * (ctx->queue_next++ % Ctx::QUEUE_RING);
    cudaError_t e = cudaMemsetAsync(slot, 0, 16, s);
    if (e != cudaSuccess) return set_err(ctx, "gemm queue reset", e);
    if (!p.queue) p.queue = slot;
    if (!p.role_ticket) p.role_ticket = slot + 2;
  }
  CUtensorMap mA, mB, mL, mC, mT;
  if ((rc = make_tile_map(ctx, &mA, Abase, p.b, nA, 16, BK, true)) != BGP_OK) return rc;
  if ((rc = make_tile_map(ctx, &mB, Bbase, p.b, nB, 16, BK, true)) != BGP_OK) return rc;
  if ((rc = make_tile_map(ctx, &mL, Linv ? Linv : Bbase, p.b, Linv ? 1 : nB, 16, BK, true)) != BGP_OK) return rc;
  if ((rc = make_tile_map(ctx, &mC, Cbase, p.b, nC, 16, WN, true)) != BGP_OK) return rc;
  if ((rc = make_tile_map(ctx, &mT, Cbase, p.b, nC, 16, BK, true)) != BGP_OK) return rc;
  PushMaps pm;
  memset(&pm, 0, sizeof(pm));
  if (p.npush < 0 || p.npush > BGP_MAX_PUSH || (p.npush > 0 && p.mode != GEMM_TRSM_PANEL && p.mode != GEMM_LIST))
    return set_err(ctx, "gemm: bad push destinations", cudaErrorInvalidValue);
  for (int d = 0; d < p.npush; ++d)
    if ((rc = make_tile_map(ctx, &pm.map[d], p.push_dst[d], p.b, p.push_tiles, 16, WN, true)) != BGP_OK) return rc;
  for (int d = 0; d < p.npush; ++d) pm.ptr[d] = p.push_dst[d];
  prepare();
  int64_t slots = (p.grid_limit > 0 && p.grid_limit < ctx->num_sms) ? p.grid_limit : ctx->num_sms;
  if (ctx->grid_cap > 0 && ctx->grid_cap < slots) slots = ctx->grid_cap;
  int64_t grid = (tasks + GROUPS - 1) / GROUPS < slots ? (tasks + GROUPS - 1) / GROUPS : slots;
  if (p.potrf_tile && grid < 2) grid = 2;  // the look-ahead CTA must not be the only one
  // the look-ahead CTA's device POTRF / inverse must fit the ring memory
  if (p.potrf_tile && tile_potrf_inv_smem_bytes(p.b, true) > (size_t)(GROUPS * GROUP_BYTES))
    return set_err(ctx, "gemm: look-ahead POTRF does not fit", cudaErrorInvalidValue);
  if (p.nsteps > 1)
    gemm_dmma_kernel<true><<<(unsigned)grid, THREADS, SMEM_BYTES, s>>>(mA, mB, mL, mC, mT, p,
                                                                        p.check_info ? ctx->d_info : nullptr, pm);
  else
    gemm_dmma_kernel<false><<<(unsigned)grid, THREADS, SMEM_BYTES, s>>>(mA, mB, mL, mC, mT, p,
                                                                         p.check_info ? ctx->d_info : nullptr, pm);
  ctx->launches++;
  return check_launch(ctx, "gemm_dmma");
}

}  // namespace dmma

void gemm_block_counts(int b, int* tile_need, int* diag_need, int* groups_per_cta) {
  *tile_need = dmma::tile_blocks(b) * dmma::block_warps();
  *diag_need = dmma::diag_blocks(b) * dmma::block_warps();
  *groups_per_cta = dmma::groups();
}

void gemm_prepare() { dmma::prepare(); }

int launch_gemm(Ctx* ctx, const GemmProblem& p, double* Cbase, const double* Abase, int64_t nA,
                const double* Bbase, int64_t nB, int64_t nC, cudaStream_t s, const double* Linv) {
  return dmma::launch(ctx, p, Cbase, Abase, nA, Bbase, nB, nC, s, Linv);
}
}  // namespace bgp
