/*
 * bgp.h -- C ABI of the B200-native bigGP likelihood path (libbgp.so).
 *
 * The reference (blockgp 0.1.0, pure Python) has no native library: its hot
 * path is a set of registered worker operations dispatched through
 * `Cluster.run(op_id, **kwargs)` (bg/transport/base.py:229-234) whose
 * arithmetic lives in numpy/scipy -> OpenBLAS/LAPACK.  Each entry point below
 * replaces one of those operations (or the BLAS/LAPACK calls inside it); the
 * citation after each declaration names the reference code it stands in
 * for.  `bg/` = /root/reference/pkg/src/blockgp/.
 *
 * Conventions
 *  - All matrices are FP64.  Every pointer marked (device) is a CUDA device
 *    pointer allocated and owned by the caller; the library never frees
 *    caller memory and only uses scratch it owns inside the context.
 *  - Triangular objects (n x n, lower) are stored as PACKED TILES: T = ceil(n/b)
 *    tile rows, tiles (I, J) with I >= J stored column-major over the tile
 *    grid at index  J*T - J*(J-1)/2 + (I-J)  (0-based), each tile b x b
 *    column-major.  The padded tail carries the identity on the diagonal and
 *    zeros elsewhere; the strict upper triangle of diagonal tiles is zero
 *    (bg/distla/objects.py:1-9, 60-80).
 *  - Rectangular objects (n x m) are stored TRANSPOSED as m x n tiles
 *    (Tm = ceil(m/b) tile rows, Tn = ceil(n/b) tile columns, tile (I, J) at
 *    index J*Tm + I, column-major inside), zero padded.  The transpose makes
 *    the left triangular solve L X = B a right solve X^T L^T = B^T, which runs
 *    on the same panel kernels as the Cholesky.
 *  - Vectors are dense, length T*b, zero padded.
 *  - `stream` is a cudaStream_t.  Calls are stream-ordered and asynchronous
 *    unless they return a host scalar or a status that depends on device
 *    data (bgp_potrf, bgp_logdet, bgp_sumsq, bgp_trsv, bgp_trsm_rect), which
 *    synchronize the stream before returning.
 *  - Return value: BGP_OK (0) or a negative BGP_E* code; device-data
 *    conditions are reported through `info` out-parameters.
 *  - A context is bound to one CUDA device and is not re-entrant
 *    (bg/transport/base.py:1-7: one master thread, one operation at a time).
 */
#ifndef BGP_H
#define BGP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BGP_OK 0
#define BGP_E_CUDA (-1)        /* CUDA runtime / driver failure           */
#define BGP_E_ARG (-2)         /* invalid argument or nonconforming shape  */
#define BGP_E_UNSUPPORTED (-3) /* generator / smoothness not built in      */

/* object kinds (bg/grid.py:198-234 "triangular" | "rectangular" | "vector") */
#define BGP_TRI 0
#define BGP_RECT 1
#define BGP_VEC 2

/* generator families (bg/gp/kernels.py:49-180) */
#define BGP_GEN_ZERO 0          /* gen.zero                         :49-53  */
#define BGP_GEN_DELTA 1         /* gen.delta                        :56-59  */
#define BGP_GEN_LINEAR_INDEX 2  /* gen.linear_index (params[0] = n) :62-65  */
#define BGP_GEN_MATERN 3        /* gen.matern[-nugget].*            :68-111 */
#define BGP_GEN_SQEXP 4         /* gen.sqexp[-nugget].*             :68-109 */
#define BGP_GEN_WHITE 5         /* gen.white.*                      :151-172 */
#define BGP_GEN_PRODUCT 6       /* gen.matern-product-nugget.*      :114-148 */

/* generator parts (bg/gp/kernels.py:77-93) */
#define BGP_PART_COV 0      /* coords x coords, nugget on i == j (if on) */
#define BGP_PART_CROSS 1    /* coords x pred_coords, no nugget           */
#define BGP_PART_PRED 2     /* pred_coords x pred_coords, no nugget      */
#define BGP_PART_PREDVAR 3  /* vector, params[0]                         */

typedef struct bgp_ctx* bgp_ctx_t;

/* Generator description.  Replaces the registry lookup of a generator id
 * (bg/registry.py:24-28) with a fixed device menu; unknown ids are rejected
 * on the host (no CPU fallback). */
typedef struct {
  int family;          /* BGP_GEN_*                                          */
  int part;            /* BGP_PART_*                                         */
  int nugget;          /* 1: add params[nparams-1] where global i == j (cov)  */
  int nparams;
  double params[8];    /* theta as in bg/gp/kernels.py:109-111, 174-180       */
  double nu;           /* Matern smoothness 0.5 / 1.5 / 2.5 (nu1 for product)  */
  double nu2;          /* second-axis smoothness (product kernel)             */
  double span;         /* upper bound on any point distance (0: unknown); lets
                          the covariance kernel skip its exp underflow test  */
} bgp_generator;

/* ---- context ------------------------------------------------------------ */
int bgp_init(int device, bgp_ctx_t* ctx);
int bgp_finalize(bgp_ctx_t ctx);
const char* bgp_last_error(bgp_ctx_t ctx);
/* library build string (arch, version) for provenance */
const char* bgp_version(void);
/* number of kernels this context has launched (evidence counter) */
int64_t bgp_launch_count(bgp_ctx_t ctx);

/* ---- K1 covariance construction ------------------------------------------
 * replaces distla.construct (bg/distla/kernels.py:35-75) + pad_block
 * (bg/distla/objects.py:60-80) + the gen.* generators (bg/gp/kernels.py).
 * X: (device) nx x dim row-major coordinates, Y: (device) ny x dim (may be
 * NULL unless part is CROSS/PRED).  kind BGP_TRI: out = packed tiles of the
 * nx x nx lower triangle; BGP_RECT: out = transposed tiles of nx x ny
 * (i.e. tiles of the ny x nx matrix); BGP_VEC: out = length ceil(nx/b)*b. */
int bgp_construct(bgp_ctx_t ctx, int kind, const bgp_generator* gen,
                  const double* X, int64_t nx, const double* Y, int64_t ny,
                  int dim, int tile, double* out, void* stream);

/* ---- K2 tiled Cholesky ----------------------------------------------------
 * replaces distla.cholesky / _cholesky_sweep (bg/distla/kernels.py:110-194),
 * in place on packed tiles.  info = 0 on success, else the 1-based global
 * row of the first non-positive pivot (LAPACK potrf convention); the caller
 * maps it to NotPositiveDefinite(block) with its layout (kernels.py:146-148).
 * The schedule has a one-panel look-ahead inside one launch per step: the
 * first CTA to take the look-ahead ticket factors the next panel's
 * diagonal tile (building its inverse during the factorization, or
 * publishing its progress per 32 columns for a substitution solve) once that
 * tile's update blocks have retired, and the next panel's solve runs as
 * gated tasks of the same launch; the chain-bound steps of
 * the last level run as ONE launch ordered by per-tile counters.  Every wait
 * is inside a launch, so the schedule also holds when kernels are serialised
 * (Nsight Compute).
 * BGP_LOOKAHEAD=0 in the environment runs POTRF, inverse, solve and update
 * as separate launches one after another on `stream` (diagnostics). */
int bgp_potrf(bgp_ctx_t ctx, double* tiles, int64_t n, int tile,
              int64_t* info, void* stream);
/* With 512 tiles and more than 2*tiles tile rows, bgp_potrf finishes the last
 * `tiles` tile rows on 256 tiles (the serial panel chain is ~4x shorter
 * there), and with 256 tiles the last tiles/2 rows on 128: the trailing
 * triangle is re-tiled into context scratch, factored, and copied back.
 * Default 32 (or BGP_TAIL in the environment); 0 disables. */
int bgp_set_tail(bgp_ctx_t ctx, int tiles);

/* ---- K3 solves -------------------------------------------------------------
 * bgp_trsv replaces distla.solve_vector (bg/distla/kernels.py:200-250):
 * x <- L^{-1} x (trans = 0, "forward") or L^{-T} x (trans = 1, "back").
 * bgp_trsm_rect replaces distla.solve_rect (kernels.py:253-307) on a
 * transposed rectangular object B^T (m x n tiles), in place.
 * info = 0, or the 1-based global row of the first zero diagonal entry
 * (SingularDiagonal, kernels.py:245-246, 302-303). */
/* Stream-ordered forms for pipelined evaluations (several factorizations in
 * flight, each on its own context and stream): no host synchronization.
 * bgp_potrf_async resets the context status and factors (a failing pivot
 * row stays in the status; later launches of the context skip);
 * bgp_trsv_async solves (a zero pivot goes to the status);
 * bgp_logdet_async / bgp_sumsq_async write their scalar to device memory;
 * bgp_info_copy copies the status (int64) to device memory. */
int bgp_potrf_async(bgp_ctx_t ctx, double* tiles, int64_t n, int tile, void* stream);
int bgp_trsv_async(bgp_ctx_t ctx, const double* L, int64_t n, int tile, double* x,
                   int trans, void* stream);
int bgp_logdet_async(bgp_ctx_t ctx, const double* L, int64_t n, int tile,
                     double* dev_out, void* stream);
int bgp_sumsq_async(bgp_ctx_t ctx, const double* x, int64_t n, double* dev_out,
                    void* stream);
int bgp_info_copy(bgp_ctx_t ctx, int64_t* dev_out, void* stream);
int bgp_trsv(bgp_ctx_t ctx, const double* L, int64_t n, int tile, double* x,
             int trans, int64_t* info, void* stream);
int bgp_trsm_rect(bgp_ctx_t ctx, const double* L, int64_t n, int tile,
                  double* Bt, int64_t m, int trans, int64_t* info, void* stream);

/* ---- K3 crossproducts (bg/distla/kernels.py:387-487) -----------------------
 * Vt: transposed rectangular object (m x n tiles). */
int bgp_xprod_mat_vec(bgp_ctx_t ctx, const double* Vt, int64_t n, int64_t m,
                      int tile, const double* u, double* w, void* stream);
int bgp_xprod_self_diag(bgp_ctx_t ctx, const double* Vt, int64_t n, int64_t m,
                        int tile, double* d, void* stream);
int bgp_xprod_self(bgp_ctx_t ctx, const double* Vt, int64_t n, int64_t m,
                   int tile, double* S, void* stream);

/* y = L x (mode 0, mult_vector, bg/distla/kernels.py:313-343), y = L^T x
 * (mode 1) or y = C x with C symmetric and stored as its lower triangle
 * (mode 2, residual probes).  x, y: (device) length ceil(n/b)*b, distinct. */
int bgp_tri_mv(bgp_ctx_t ctx, const double* L, int64_t n, int tile,
               const double* x, double* y, int mode, void* stream);

/* Y^T = X^T L^T for transposed rectangular X (m x n tiles): Y = L X, the
 * rectangular mult_chol of simulation (bg/distla/kernels.py:346-381), on the
 * DMMA GEMM (Yt must not alias Xt). */
int bgp_trmm_rect(bgp_ctx_t ctx, const double* L, int64_t n, int tile,
                  const double* Xt, int64_t m, double* Yt, void* stream);
/* N(0,1) fill from the rank stream of bg/rng.py:18-28 (Philox4x64-10 keyed by
 * (seed << 64) + rank, inverse normal CDF), starting `offset` draws into the
 * stream, in the reference's block order for API block sizes bs_r x bs_c
 * (bg/distla/kernels.py:78-104).  m = 0: vector of length n (dense); m > 0:
 * n x m object written as transposed tiles.  Padding entries are untouched
 * (zero-initialise `out`). */
int bgp_rnorm(bgp_ctx_t ctx, int64_t n, int64_t m, int64_t bs_r, int64_t bs_c,
              uint64_t seed, uint64_t rank, uint64_t offset, int tile,
              double* out, void* stream);

/* ---- K3d reductions (bg/distla/kernels.py:493-522, __init__.py:154-162) ----
 * logdet = 2 sum_{i<n} log L_ii (fixed-order tree sum); info = 1-based row
 * of the first non-positive diagonal (SingularDiagonal) or 0. */
int bgp_logdet(bgp_ctx_t ctx, const double* L, int64_t n, int tile,
               double* out, int64_t* info, void* stream);
int bgp_sumsq(bgp_ctx_t ctx, const double* x, int64_t n, double* out,
              void* stream);

/* ---- plumbing: distribute / collect / remote_apply("sub") -------------------
 * bgp_pack replaces distla.split (kernels.py:538-544, objects.py:83-105):
 * dense row-major (device) nrow x ncol array with leading dimension ld ->
 * tiles of `kind` (the lower triangle only for BGP_TRI; for BGP_RECT the
 * dense array is the n x m matrix and the tiles hold its transpose).
 * bgp_unpack is the inverse (bg/distla/objects.py:108-123, assemble);
 * triangular unpack writes the lower triangle and zeros above it.
 * bgp_tri_diagonal extracts diag (collect_diagonal, __init__.py:141-151).
 * bgp_sub: out = a - b elementwise over `count` doubles (kernels.py:564). */
int bgp_pack(bgp_ctx_t ctx, int kind, const double* dense, int64_t nrow,
             int64_t ncol, int64_t ld, int tile, double* tiles, void* stream);
int bgp_unpack(bgp_ctx_t ctx, int kind, const double* tiles, int64_t nrow,
               int64_t ncol, int tile, double* dense, int64_t ld, void* stream);
int bgp_tri_diagonal(bgp_ctx_t ctx, const double* L, int64_t n, int tile,
                     double* d, void* stream);
int bgp_sub(bgp_ctx_t ctx, const double* a, const double* b, double* out,
            int64_t count, void* stream);

/* ---- tile-level primitives (multi-GPU driver, look-ahead schedules) -------
 * bgp_tile_potrf: factor one b x b diagonal tile in place (info as above,
 *   `row0` = 0-based global row of the tile for the info value).
 * bgp_panel_trsm: X <- A L_d^{-T} for `count` b x b tiles at A (stride
 *   b*b doubles), L_d one factored diagonal tile (kernels.py:163-164).
 * bgp_tile_update: C -= A B^T over a list of `count` (C, A, B) tile index
 *   triples into three packed-tile bases (kernels.py:188-192); a triple with
 *   lower != 0 updates only the lower triangle (diagonal SYRK). */
/* Stream-ordered forms for the multi-GPU schedule (no host synchronization
 * per step): bgp_tile_potrf_async factors a diagonal tile and, when linv is
 * not null, writes its inverse (b x b column-major); a failing pivot is
 * recorded in the context's device status, which bgp_info_reset clears and
 * bgp_info_read returns (synchronizing).  bgp_panel_trsm_inv solves `count`
 * consecutive tiles in place, A <- A Linv^T, on the DMMA GEMM; it is skipped
 * once the status records a failure. */
int bgp_info_reset(bgp_ctx_t ctx, void* stream);
int bgp_info_read(bgp_ctx_t ctx, int64_t* info, void* stream);
int bgp_tile_potrf_async(bgp_ctx_t ctx, double* tile_ptr, int tile, int64_t row0,
                         double* linv, void* stream);
int bgp_panel_trsm_inv(bgp_ctx_t ctx, const double* linv, double* A, int64_t count,
                       int tile, void* stream);
/* bgp_tile_potrf_inv: bgp_tile_potrf (row0 = 0) followed by the one-CTA
 * inverse the look-ahead uses: linv (b x b column-major) = L^{-1}. */
int bgp_tile_potrf_inv(bgp_ctx_t ctx, double* tile_ptr, int tile, double* linv,
                       int64_t* info, void* stream);
int bgp_tile_potrf(bgp_ctx_t ctx, double* tile_ptr, int tile, int64_t row0,
                   int64_t* info, void* stream);
/* A rank's share of construct: lower tiles (I, J) listed in tile_ij (device,
 * 2 int32 per tile) written to consecutive b x b tiles of out
 * (bg/distla/kernels.py:45-75 over this rank's owned blocks). */
int bgp_construct_tiles(bgp_ctx_t ctx, const bgp_generator* gen, const double* X,
                        int64_t n, int dim, int tile, const int32_t* tile_ij,
                        int64_t count, double* out, void* stream);
/* Diagonal-tile solve of a distributed TRSV step: x (b doubles) <- L_jj^{-1} x
 * or L_jj^{-T} x; row0 = global row of the tile (kernels.py:244-249). */
/* bgp_tile_trsv with info == NULL: stream-ordered, the status stays in the
 * device (bgp_info_read). */
int bgp_tile_trsv(bgp_ctx_t ctx, const double* Ljj, int tile, int64_t row0,
                  int64_t n, double* x, int trans, int64_t* info, void* stream);
/* acc[target*b ...] += L_tile x_J (trans 0) or L_tile^T x_J (trans 1) for
 * (tile index, target block) pairs (device, distinct targets): the partial
 * products of solve_vector (kernels.py:219-235). */
int bgp_tile_gemv(bgp_ctx_t ctx, const double* base, const int32_t* items,
                  int64_t count, int tile, const double* xJ, double* acc,
                  int trans, void* stream);
/* Per-rank log-det partial over listed diagonal tiles (tile index, J)
 * (kernels.py:493-509). */
int bgp_tile_logdet(bgp_ctx_t ctx, const double* base, const int32_t* diag,
                    int64_t count, int tile, int64_t n, double* out,
                    int64_t* info, void* stream);
int bgp_panel_trsm(bgp_ctx_t ctx, const double* Ld, double* A, int64_t count,
                   int tile, void* stream);

/* Multi-GPU panel push (replaces the NCCL panel broadcast of the sweep,
 * kernels.py:165-187 send / 175-180 receive): panel buffers are allocated
 * here, exported as CUDA IPC handles (BGP_IPC_HANDLE_BYTES), and opened by
 * every peer process (NVLink P2P mappings).  bgp_panel_trsm_push is
 * bgp_panel_trsm_inv whose epilogue also stores every solved block into tile
 * slot0 + t of each of the ndst (<= 8) destination buffers dst[] (own and
 * peer panel buffers, each dst_tiles tiles) from the same staged rows: the
 * solve and the exchange are one kernel.  The caller orders the receivers'
 * reads after the kernel (a stream-ordered barrier) and the writes after the
 * receivers' last use of the buffer. */
#define BGP_IPC_HANDLE_BYTES 64
int bgp_ipc_alloc(bgp_ctx_t ctx, size_t bytes, void** ptr, void* handle);
int bgp_ipc_open(bgp_ctx_t ctx, const void* handle, void** ptr);
int bgp_ipc_close(bgp_ctx_t ctx, void* ptr);
int bgp_ipc_free(bgp_ctx_t ctx, void* ptr);
int bgp_panel_trsm_push(bgp_ctx_t ctx, const double* linv, double* A, int64_t count,
                        int tile, double* const* dst, int ndst, int64_t slot0,
                        int64_t dst_tiles, void* stream);
int bgp_tile_update(bgp_ctx_t ctx, double* Cbase, const double* Abase,
                    const double* Bbase, const int32_t* triples /*device, 4 per*/,
                    int64_t count, int tile, void* stream);

/* ---- one rank's share of the distributed block sweep ----------------------
 * Replaces the per-worker body of _cholesky_sweep (bg/distla/kernels.py:
 * 139-194) on a 2-D block-cyclic tile distribution; the host (parallel.py)
 * orders the steps with one stream-ordered barrier each.
 * bgp_dist_begin: zero the per-step counters of a T-step sweep, reset the
 *   status.
 * bgp_dist_step: step J as ONE launch.  items (device, 4 int32 per tuple):
 *   (C local tile, A panel slot, B panel slot, flags), flags bit 0 = C is a
 *   diagonal tile (lower part only), bits 8.. = gate + 1; the first
 *   col_items tuples update tile column J+1 (gate 0 the diagonal tile, 1..
 *   the rank's panel tiles in local order).  With diag != NULL the launch
 *   also factors that tile (row diag_row0 for the status) once its update
 *   retired (kernels.py:144-153 POTRF), inverts it, and solves the rank's
 *   trsm_count panel tiles local[trsm_first ..] in place (kernels.py:155-165
 *   TRSM) -- every solved block is also stored into tile slot0 + t of each of
 *   the ndst (<= 8) panel buffers dst[] (own and peers', IPC-mapped), which
 *   replaces the "col" sends of kernels.py:167-187.  Launches are skipped
 *   once the status records a failure. */
int bgp_dist_begin(bgp_ctx_t ctx, int T, int tile, void* stream);
int bgp_dist_step(bgp_ctx_t ctx, int J, double* local, int64_t nlocal,
                  const double* panel, int64_t npanel, const int32_t* items,
                  int64_t count, int64_t col_items, double* diag, int64_t diag_row0,
                  int64_t trsm_first, int64_t trsm_count, int trsm_par,
                  double* const* dst, int ndst, int64_t slot0, int64_t dst_tiles,
                  int tile, void* stream);

/* ---- measurement ----------------------------------------------------------
 * When profiling is on, bgp_potrf brackets every launch with CUDA events
 * (no extra synchronization: they are read at the status sync the call
 * already does).  bgp_profile_read returns and clears BGP_PROFILE_SLOTS values:
 *   out[0] potrf ms (look-ahead stream, overlaps the trailing update)
 *   out[1] trsm ms  out[2] gemm (trailing update, both parts) ms
 *   out[3] gemm launches  out[4] gemm algorithmic flops (b^3 k^2 per step)
 *   out[5] potrf launches  out[6] trsm launches  out[7] factorizations
 *   out[8] factorization ms (first to last launch on the caller's stream)
 *   out[9] potrf ms exposed on the critical path (caller's stream waiting)
 * (stands in for the reference's event log, bg/transport/base.py:121-123). */
#define BGP_PROFILE_SLOTS 10
int bgp_set_profiling(bgp_ctx_t ctx, int on);
/* GEMM launches of this context use at most max_ctas CTAs (0: all SMs) --
 * pipelined evaluations on several contexts leave SMs to each other's
 * latency-bound steps. */
int bgp_set_grid_cap(bgp_ctx_t ctx, int max_ctas);
int bgp_profile_read(bgp_ctx_t ctx, double* out);
/* per-step trailing-update launch times (ms) of the last profiled bgp_potrf;
 * returns the number written (<= max) */
int bgp_profile_steps(bgp_ctx_t ctx, double* out, int max);

#ifdef __cplusplus
}
#endif
#endif /* BGP_H */
