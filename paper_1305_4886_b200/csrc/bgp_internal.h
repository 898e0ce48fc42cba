// Internal host-side declarations shared by the libbgp translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/bgp.h"

namespace bgp {

// device-side generator description (built from bgp_generator on the host)
struct GenDev {
  int family, part, nugget, np;
  double p[8];
  double sqrt2nu, sqrt2nu2;
  int nucode, nucode2;  // 0: nu=1/2, 1: 3/2, 2: 5/2
  int dim;
  int safe_exp;  // fast covariance path: no exp argument can underflow (span known)
};

struct Ctx {
  int device = 0;
  int num_sms = 148;
  std::string err;
  int64_t launches = 0;
  // device scratch owned by the context
  unsigned long long* d_info = nullptr;  // [0]: potrf / trsv status
  double* d_red = nullptr;               // reduction partials
  size_t red_cap = 0;
  double* d_dinv = nullptr;  // inverted 32x32 diagonal sub-blocks
  size_t dinv_cap = 0;
  double* d_part = nullptr;  // generic partial buffer (crossproducts)
  size_t part_cap = 0;
  int32_t* d_items = nullptr;
  size_t items_cap = 0;
  int* d_sync = nullptr;  // persistent-kernel row counter + ready flags
  size_t sync_cap = 0;
  int* d_gate = nullptr;  // per-step look-ahead counters of the Cholesky
  size_t gate_cap = 0;
  double* d_linv = nullptr;  // inverse of the current diagonal tile (panel TRSM on DMMA)
  size_t linv_cap = 0;
  int* d_pass = nullptr;  // per-step pass counters of the parallel fused TRSM
  size_t pass_cap = 0;
  int* d_multi = nullptr;  // counters of the multi-step tail launch (tiles, solves, progress, queue)
  size_t multi_cap = 0;
  double* d_linv_all = nullptr;  // inverses of every diagonal tile (kriging solve)
  size_t linv_all_cap = 0;
  // per-launch task counters (+ look-ahead tickets) of GEMM launches that do
  // not bring their own: a ring of 16-byte slots, one per launch
  static constexpr int QUEUE_RING = 1024;
  int* d_queue_ring = nullptr;
  size_t queue_ring_cap = 0;
  unsigned queue_next = 0;
  double* d_tail[2] = {nullptr, nullptr};  // re-tiled trailing triangles of the Cholesky tail
  size_t tail_cap[2] = {0, 0};
  int dist_T = 0, dist_b = 0;
  int grid_cap = 0;  // > 0: GEMM launches of this context use at most this many CTAs (bgp_set_grid_cap)  // bgp_dist_begin: tile rows and tile size of the current sweep
  int tail_tiles = 32;  // 512-tile rows finished on 256 tiles (half as many 256 rows on 128; bgp_set_tail)
  void* encode_fn = nullptr;  // cuTensorMapEncodeTiled
  // profiling (bgp_set_profiling / bgp_profile_read)
  bool profile = false;
  cudaEvent_t* events = nullptr;
  int events_cap = 0;
  double prof[BGP_PROFILE_SLOTS] = {};
  double step_ms[4096] = {};  // per-step update-launch time of the last profiled factorization
  int nsteps = 0;
};

int set_err(Ctx* ctx, const char* what, cudaError_t e);
int check_launch(Ctx* ctx, const char* what);
int ensure(Ctx* ctx, void** buf, size_t* cap, size_t bytes);

// encode a 3-D FP64 tensor map over `ntiles` b x b column-major tiles:
// dims (b rows, b cols, ntiles), box {box0 rows, box1 cols, 1}, 128B swizzle
int make_tile_map(Ctx* ctx, CUtensorMap* map, const double* base, int b, int64_t ntiles, int box0,
                  int box1, bool swizzle128);

int construct(Ctx* ctx, int kind, const GenDev& g, const double* X, int64_t nx, const double* Y,
              int64_t ny, int b, double* out, cudaStream_t s);

int construct_tiles(Ctx* ctx, const GenDev& g, const double* X, int64_t n, int b, const int32_t* tile_ij,
                    int64_t count, double* out, cudaStream_t s);
int launch_tile_trsv(Ctx* ctx, const double* Ljj, int b, int64_t row0, int64_t n, double* x, int trans,
                     cudaStream_t s);
int launch_tile_gemv(Ctx* ctx, const double* base, const int32_t* items, int64_t count, int b, const double* xJ,
                     double* partial, int trans, cudaStream_t s);
int launch_tile_logdet(Ctx* ctx, const double* base, const int32_t* diag, int64_t count, int b, int64_t n,
                       cudaStream_t s);

// one-time kernel attribute setup; also loads the modules eagerly (lazy
// loading must not happen while a look-ahead kernel spin-waits)
void gemm_prepare();
void potrf_prepare();
// retire counts of the update launch's gates for tile size b (warp-blocks of
// a full tile / of a diagonal tile) and consumer groups per CTA
void gemm_block_counts(int b, int* tile_need, int* diag_need, int* groups_per_cta);
size_t potrf_smem_bytes(int b);
size_t tri_inv_smem_bytes();
// tile POTRF (+ inverse) with the tile staged in shared memory for b <= 128
size_t tile_potrf_inv_smem_bytes(int b, bool inv);

// tile kernels
// info value reserved for a look-ahead wait that never completed (a bug, not data)
constexpr unsigned long long BGP_INFO_DATAFLOW_TIMEOUT = 1ull << 62;
// with Linv: the tile's inverse too, built during the factorization
int launch_tile_potrf(Ctx* ctx, double* tile, int b, int64_t row0, double* dinv, cudaStream_t s,
                      const int* gate = nullptr, int gate_need = 0, double* Linv = nullptr);
// one-CTA block-diagonal inverse of a factored tile (panel_device.cuh)
int launch_tri_inv(Ctx* ctx, const double* Ltile, const double* dinv, int b, double* Linv, cudaStream_t s,
                   int* done = nullptr);
int launch_diag_inv(Ctx* ctx, const double* L, int T, int b, int64_t n, double* dinv, cudaStream_t s);
// inverses of all T diagonal tiles of a factored packed triangle (dinv from launch_diag_inv)
int launch_tri_inv_batch(Ctx* ctx, const double* L, int T, const double* dinv, int b, double* Linv,
                         cudaStream_t s);
int launch_panel_trsm(Ctx* ctx, const double* Ld, const double* dinv, double* A, int64_t count, int b,
                      int trans, cudaStream_t s, bool check_info = true);

// DMMA/TMA GEMM problems
enum GemmMode {
  GEMM_CHOL_TRAIL = 0,  // tiles (R, C), J+1 <= C <= R < T, of the step-J trailing update
  GEMM_RECT_TRAIL = 1,
  GEMM_SYRK_RECT = 2,
  GEMM_LIST = 3,
  GEMM_TRMM_RECT = 4,
  GEMM_TRSM_PANEL = 6   // X = A Linv^T in place for `count` consecutive tiles from panel0
};
struct GemmProblem {
  int mode;
  int b;
  int T;    // tile rows of the packed triangle (L or S)
  int J;    // panel index (trailing modes)
  int Tm;   // tile rows of a transposed rectangular object
  int Tn;   // tile columns of a transposed rectangular object
  int64_t count;  // GEMM_LIST: number of (C, A, B, flags) tuples
  const int32_t* items;
  double alpha, beta;  // D = beta*C + alpha*sum(A B^T)
  bool check_info;     // skip the launch when ctx->d_info records a failure
  int grid_limit;      // > 0: at most this many CTAs (leaves SMs to a concurrent kernel)
  int64_t panel0;      // GEMM_TRSM_PANEL: tile index of the first panel tile
  int* queue;          // zeroed task counter (null: launch_gemm provides one)
  // GEMM_CHOL_TRAIL look-ahead: col_gate[r] counts retired warp-blocks of tile
  // (J+1+r, J+1); with trsm_next the launch also solves panel J+1 in place,
  // each tile once col_gate reaches tile_need and *linv_flag reaches linv_need
  int* col_gate;
  int trsm_next;
  int tile_need;
  int* linv_flag;
  int linv_need;
  int trsm_tail;       // update blocks queued after the fused TRSM tasks (tail filler)
  // look-ahead inside the launch: the first CTA to take role_ticket factors tile potrf_tile
  // (panel J+1's diagonal, once col_gate[0] reaches diag_need) into dinv, and
  // with trsm_next its inverse into linv (published through linv_flag), then
  // joins the queue
  double* potrf_tile;
  int64_t potrf_row0;
  double* dinv;
  double* linv;
  int diag_need;
  double* cbase;       // set by launch_gemm: C tiles (register epilogue variant)
  // GEMM_TRSM_PANEL push (multi-GPU): the epilogue also stores every solved
  // block into tile (cTile - panel0) of each of npush destination panel
  // buffers (this GPU's and its peers', IPC-mapped over NVLink); host-side
  // bases, each holding push_tiles tiles, turned into tensor maps at launch
  int npush;
  double* const* push_dst;
  int64_t push_tiles;
  // GEMM_TRSM_PANEL out of place: C (the launch's Cbase) is a separate
  // buffer, so the column passes of a slab read only A and are independent
  // tasks (in place they must run right to left in one task)
  int trsm_oop;
  // GEMM_CHOL_TRAIL fused TRSM with independent column passes: one task per
  // (slab, pass), right to left; pass p of a slab stores only after passes
  // 0 .. p-1 (the columns to its right, which read its block) finished
  // reading: pass_done[slab * (b / 64) + q] counts the warps of pass q done
  int trsm_par;
  int* pass_done;
  // GEMM_LIST as one step of the distributed sweep: the first col_items
  // tuples update tile column J+1 (their flags carry the gates); the fused
  // TRSM solves the rank's trsm_count panel tiles from local index panel0
  // (and pushes them when npush > 0)
  int64_t col_items;
  int64_t trsm_count;
  // zeroed int: the first CTA to take a ticket is the look-ahead CTA
  // (null: launch_gemm provides one)
  int* role_ticket;
  // GEMM_CHOL_TRAIL fused TRSM by substitution (tiles >= 256, chain-bound
  // steps): no tile inverse; each slab task solves its 128 rows column block
  // by column block as the look-ahead POTRF publishes them (potrf_progress)
  int trsm_subst;
  int* potrf_progress;
  // GEMM_CHOL_TRAIL: live rows of the triangle (rows >= n_live are identity
  // padding); blocks and TRSM slabs wholly in the padding are skipped (0: none)
  int64_t n_live;
  // tile counts behind the A / B / C tensor maps (set by launch_gemm; the
  // checked build asserts every tile index against them)
  int64_t nA, nB, nC;
  // GEMM_CHOL_TRAIL over nsteps > 1 consecutive steps J .. J+nsteps-1 in ONE
  // launch (the chain-bound tail, substitution solve): the steps' task lists
  // are queued one after another and ordered by counters instead of launch
  // boundaries.  tile_cnt[t] counts the retired warp-blocks of trailing tile
  // t (packed index minus cnt_base = tri_index(J+1, J+1, T); col_gate points
  // at it), solved[t] the warps that finished solving panel tile t by
  // substitution (solved_need per tile).  An update block of step s > J
  // waits until its two panel-s tiles are solved; the solve of tile
  // (R, s+1) waits for (s+1-J) steps of updates into it; the role CTA factors
  // (s+1, s+1) after (s+1-J) steps of updates, into dinv + (s-J) * b * 32
  // with progress counter potrf_progress[s-J].
  int nsteps;
  int* tile_cnt;
  int* solved;
  int solved_need;
  int64_t cnt_base;
  // GEMM_CHOL_TRAIL step groups (large steps, BGP_PAIR_STEPS; pairs by
  // default): pair_cols > 0 updates only tile columns J+1 .. J+pair_cols (the
  // thin launches of a group); pair_merge = m > 0 applies panels J-m .. J
  // together (k = (m+1) b) to columns >= J+2 and panel J alone to column J+1
  // (the group's last launch)
  int pair_cols;
  int pair_merge;
};
constexpr int BGP_MAX_PUSH = 8;
int launch_gemm(Ctx* ctx, const GemmProblem& p, double* Cbase, const double* Abase, int64_t nA,
                const double* Bbase, int64_t nB, int64_t nC, cudaStream_t s, const double* Linv = nullptr);

int launch_trsv_fwd_persistent(Ctx* ctx, const double* L, int64_t n, int b, double* x, cudaStream_t s);
int launch_trsv(Ctx* ctx, const double* L, int64_t n, int b, double* x, int trans, cudaStream_t s);
int launch_trsm_rect_back(Ctx* ctx, const double* L, int64_t n, int b, double* Bt, int64_t m,
                          cudaStream_t s);
int launch_rnorm(Ctx* ctx, int64_t n, int64_t m, int64_t bs_r, int64_t bs_c, uint64_t seed, uint64_t rank,
                 uint64_t offset, int b, double* out, cudaStream_t s);
int launch_tri_mv(Ctx* ctx, const double* L, int64_t n, int b, const double* x, double* y, int trans, int sym,
                  cudaStream_t s);
int launch_logdet(Ctx* ctx, const double* L, int64_t n, int b, cudaStream_t s);
int launch_sumsq(Ctx* ctx, const double* x, int64_t n, cudaStream_t s);
int launch_rowdot(Ctx* ctx, const double* Vt, int64_t n, int64_t m, int b, const double* u, double* w,
                  cudaStream_t s);
int launch_pack(Ctx* ctx, int kind, const double* dense, int64_t nrow, int64_t ncol, int64_t ld, int b,
                double* tiles, cudaStream_t s);
int launch_unpack(Ctx* ctx, int kind, const double* tiles, int64_t nrow, int64_t ncol, int b,
                  double* dense, int64_t ld, cudaStream_t s);
int launch_tri_diagonal(Ctx* ctx, const double* L, int64_t n, int b, double* d, cudaStream_t s);
int launch_sub(Ctx* ctx, const double* a, const double* bb, double* out, int64_t count, cudaStream_t s);
int launch_copy(Ctx* ctx, double* dst, const double* src, int64_t count, cudaStream_t s);

}  // namespace bgp

// the opaque C handle is the context itself
struct bgp_ctx : public bgp::Ctx {};
