/*
 * pdhg_b200.h -- C ABI of the B200-native PDHG engine (libpdhg_b200.so).
 *
 * This is the drop-in boundary for the reference package's hot path,
 * `hybridlp.pdhg.run_pdhg` (/root/reference/pkg/src/hybridlp/pdhg.py:162-258).
 * The Python host (paper_2603_03150_b200/engine.py) keeps the reference's
 * Python signature and control flow and calls down through this ABI for all
 * arithmetic; a C/C++ caller can drive it the same way.
 *
 * Conventions
 *   - Every function returns 0 on success and a negative code on failure;
 *     pdhg_last_error() returns a thread-local message.  No C++ exception
 *     crosses this boundary.
 *   - The library never allocates device memory.  The caller owns every
 *     device buffer (the Python host allocates them as torch tensors) and
 *     passes raw device pointers; sizes come from pdhg_workspace_bytes().
 *   - All work is enqueued on the cudaStream_t given to pdhg_ctx_create;
 *     functions that return host scalars synchronise that stream.
 *   - fp64 values, int32 column indices and row offsets (nnz < 2^31).
 *   - Results are bitwise reproducible run to run for a fixed layout
 *     (fixed-order reductions, no floating-point atomics).
 */
#ifndef PDHG_B200_H
#define PDHG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDHG_ABI_VERSION 6

/* Error codes. */
#define PDHG_OK 0
#define PDHG_ERR_ARG (-1)
#define PDHG_ERR_CUDA (-2)
#define PDHG_ERR_STATE (-3)

/* Which iterate a call refers to. */
#define PDHG_PT_CUR 0  /* (x, y)            -- state.x / state.y      pdhg.py:55-56 */
#define PDHG_PT_AVG 1  /* (avg_x, avg_y)    -- state.avg_x / avg_y    pdhg.py:57-58 */
#define PDHG_PT_BEST 2 /* best point so far -- best_pt               pdhg.py:180,231-232 */

/* Number of doubles pdhg_check writes per scored point (see PDHG_Q_*). */
#define PDHG_NQ 8
#define PDHG_Q_RP2 0   /* sum r_p^2        -> ||r_p||_2^2   lp_core.py:436,458 */
#define PDHG_Q_RPMAX 1 /* max |r_p|        -> primal_inf    lp_core.py:476 */
#define PDHG_Q_BY 2    /* b'y              -> dual_obj      lp_core.py:442 */
#define PDHG_Q_RD2 3   /* sum r_d^2        -> ||r_d||_2^2   lp_core.py:437,459 */
#define PDHG_Q_RDMAX 4 /* max |r_d|        -> dual_inf      lp_core.py:477 */
#define PDHG_Q_CX 5    /* c'x              -> primal_obj    lp_core.py:441 */
#define PDHG_Q_XZ 6    /* x'z              -> comp          lp_core.py:443 */
#define PDHG_Q_RSV 7   /* reserved (0) */

/*
 * Problem on the device: the standard-form LP min c'x, Ax=b, x>=0 of
 * StandardLp (lp_core.py:106-142) in a dual layout -- A as CSR (rows i,
 * drives A@x) and A' as CSR (= CSC of A, drives A'y = StandardLp.at_y,
 * lp_core.py:140-142).  Rows longer than `heavy_threshold` are listed in
 * the heavy-row arrays and get a whole thread block each.
 */
/*
 * Panel-staged rows (PSR) layout of one operator (A or A'), built on the
 * device by pdhg_psr_plan + pdhg_psr_build (see csrc/psr.cuh for the
 * format).  Used by the step kernels when the host decides it pays
 * (enough entries in dense column panels); NULL = CSR-vector kernels.
 */
typedef struct pdhg_psr {
  int32_t rows, cols, R, W, nblk, ntiles, ngroups;
  int64_t nent;
  const int32_t* blk_tile_ptr;  /* nblk+1 */
  const int32_t* tile_bin;      /* ntiles, -1 = remote tile */
  const int32_t* gstart;        /* ntiles*(ngroups+1) */
  const uint16_t* rcnt;         /* ntiles*ngroups*32: entries of each row in each tile */
  const double* val;            /* nent */
  const uint16_t* col16;        /* nent: column inside the panel */
  const int32_t* col;           /* nent: global column */
  const uint8_t* heavy;         /* rows */
} pdhg_psr;

/* Sliced-ELL layout of one operator (csrc/sell_build.cu): slices of 32
 * consecutive rows, the k-th entry of a slice's rows stored contiguously at
 * sptr[slice] + 32*k + lane.  Light rows only (heavy rows stay on the
 * block-per-row CSR path); row lengths come from the operator's CSR ptr. */
typedef struct pdhg_sell {
  int32_t rows, nslices;
  const int64_t* sptr;   /* nslices+1 slot offsets */
  const int32_t* width;  /* nslices: longest light row of the slice */
  const int32_t* col;    /* slots */
  const double* val;     /* slots */
  const uint8_t* perm;   /* optional (rows rounded up to 32): lane -> row offset in its
                            slice, rows sorted by length inside each slice (NULL = identity) */
  int64_t nslots;        /* slots (sptr[nslices]); 0 = unknown (bounds-checked build only) */
} pdhg_sell;

typedef struct pdhg_problem {
  int32_t m, n;
  int64_t nnz;
  const int32_t* a_ptr;   /* m+1 */
  const int32_t* a_col;   /* nnz */
  const double* a_val;    /* nnz */
  const int32_t* at_ptr;  /* n+1 */
  const int32_t* at_col;  /* nnz */
  const double* at_val;   /* nnz */
  const double* b;        /* m */
  const double* c;        /* n */
  int32_t a_lanes;        /* lanes per row for A rows: 1,2,4,8,16,32 (0 = auto from mean row length) */
  int32_t at_lanes;       /* same for A' rows */
  int32_t heavy_threshold;/* rows with more entries are processed block-per-row */
  int32_t a_n_heavy, at_n_heavy;
  const int32_t* a_heavy;  /* device list of heavy rows of A */
  const int32_t* at_heavy; /* device list of heavy rows of A' */
  const pdhg_psr* a_psr;   /* optional PSR layout of A  (dual step)   */
  const pdhg_psr* at_psr;  /* optional PSR layout of A' (primal step) */
  int32_t l2_persist;      /* bit0/bit1: pin y (primal step) / xe (dual step) in L2 with a persisting access-policy window */
  /* Sharding (multi-GPU).  This context owns rows [of A] that
   * map to y-space slots [y_off, y_off+m) and rows [of A'] that map to
   * x-space slots [x_off, x_off+n) of full (padded) vectors of length m_full
   * and n_full; the column indices of A / A' are in x-space / y-space slots.
   * 0 / 0 / 0 / 0 = unsharded (m_full = m, n_full = n). */
  int32_t m_full, n_full, y_off, x_off;
  int64_t at_nnz;          /* entries of the A' block (0 = nnz; differs from nnz when sharded) */
  /* Optional split-K of the dual step over column chunks of A (see
   * pdhg_split_build): a_nsplit passes, a_split = (a_nsplit-1) arrays of m
   * split points.  1 / NULL = unsplit. */
  int32_t a_nsplit;
  const int32_t* a_split;
  /* Heavy-row threshold of A' rows when it differs from A's (0 = heavy_threshold). */
  int32_t at_heavy_threshold;
  /* Optional sliced-ELL layouts for the step kernels (NULL = CSR-vector). */
  const pdhg_sell* a_sell;   /* dual step (rows of A)    */
  const pdhg_sell* at_sell;  /* primal step (rows of A') */
  /* Period mode.  0: a CUDA graph of 2 kernels per iteration (captured once
   * per period length); 1: one cooperative (persistent) kernel with grid
   * barriers between half steps; 2: one single-block kernel (tiny models);
   * 3: direct stream launches, no graph.  1 and 2 need CSR layouts and an
   * unsharded context (ignored otherwise). */
  int32_t persistent;
  /* Medium rows (CSR step kernels only): rows of A / A' with light_max <
   * length <= heavy threshold, listed in a_medium / at_medium, run one warp
   * per row instead of sharing a warp-owns-32-rows pass.  0 = none. */
  int32_t a_light_max, at_light_max;
  int32_t a_n_medium, at_n_medium;
  const int32_t* a_medium;
  const int32_t* at_medium;
  /* Split primal step (rows of A'), as a_nsplit / a_split for the dual step:
   * at_nsplit passes over per-row entry ranges, at_split = (at_nsplit-1)
   * arrays of n split points.  Sharded contexts use 2 passes for both steps
   * (local-slot entries first) so that the all-gather of the other shards'
   * slices overlaps pass 0 (pdhg_half_step_pass). */
  int32_t at_nsplit;
  const int32_t* at_split;
  /* Optional sliced-ELL layouts of the two passes of a split step (with
   * a_nsplit / at_nsplit = 2): part 0 = each row's first segment (sharded:
   * its local-slot entries), part 1 = the rest, as two CSR matrices
   * (a_part_ptr[h] their row pointers) laid out by pdhg_sell_plan/fill.
   * Rows longer than the heavy threshold are left out of both parts (length
   * 0) and run whole, block per row, in pass 1.  NULL = the CSR-vector split
   * kernels over a_split / at_split. */
  const pdhg_sell* a_sell_part[2];
  const int32_t* a_part_ptr[2];
  const pdhg_sell* at_sell_part[2];
  const int32_t* at_part_ptr[2];
} pdhg_problem;

typedef struct pdhg_ctx pdhg_ctx;

/* ABI version and the thread-local message of the last failing call (the
 * reference raises Python exceptions instead; the Python host re-raises
 * them as InvalidModelError / ValueError where pdhg.py / lp_core.py do). */
int pdhg_abi_version(void);
const char* pdhg_last_error(void);

/* Device workspace the caller must provide (m, n: full vector lengths --
 * m_full, n_full when sharded): x, xe, x̄, x_best, z_best, y, ȳ, y_best
 * (PdhgState, pdhg.py:51-67) plus scratch, partials and step parameters. */
size_t pdhg_workspace_bytes(int32_t m, int32_t n);

/* Create / destroy an engine context bound to `stream` (a cudaStream_t):
 * the device side of one run_pdhg call on one StandardLp (pdhg.py:162-258;
 * the matrix layouts replace StandardLp.A / A_csc, lp_core.py:114-142). */
int pdhg_ctx_create(const pdhg_problem* prob, void* workspace, size_t workspace_bytes,
                    void* stream, pdhg_ctx** out);
int pdhg_ctx_destroy(pdhg_ctx* ctx);

/* out = A @ in (transpose=0) or A' @ in (transpose=1); device pointers.
 * Replaces scipy csr_matvec behind `p.A @ x` and `p.at_y(y)` (lp_core.py:140-142). */
int pdhg_spmv(pdhg_ctx* ctx, int transpose, const double* in, double* out);

/* Power iteration on A'A (estimate_opnorm, pdhg.py:80-109).  v0 (n doubles,
 * host or device memory) is the caller's normalised start vector (numpy
 * default_rng(seed), pdhg.py:89-91), in the context's column order. */
int pdhg_opnorm(pdhg_ctx* ctx, const double* v0_host, double tol, int32_t max_iters,
                double* lam_out, int32_t* iters_out);

/* x = y = avg_x = avg_y = 0 (initial_state, pdhg.py:120-127). */
int pdhg_reset(pdhg_ctx* ctx);

/* Run `iters` PDHG steps (pdhg_step, pdhg.py:140-151) starting at global
 * iteration `iter0` with steps tau/omega, sigma*omega and average weight w0
 * (integer-valued).  Steps after the first non-finite iterate are skipped
 * (pdhg.py:194-196); *fail_iter_out receives that iteration or -1. */
int pdhg_run_period(pdhg_ctx* ctx, int32_t iters, int64_t iter0, double tau_over_omega,
                    double sigma_omega, double w0, int64_t* fail_iter_out);
/* pdhg_run_period followed by pdhg_check of npts points (0..2) with a single
 * host synchronisation (one fewer round trip per period; the engine uses it
 * whenever a period ends on a check).  out_host as in pdhg_check. */
int pdhg_run_period_check(pdhg_ctx* ctx, int32_t iters, int64_t iter0, double tau_over_omega,
                          double sigma_omega, double w0, int32_t npts, const int32_t* specs,
                          int64_t* fail_iter_out, double* out_host);

/* Score points.  specs[k] selects point k's (x, y) source (PDHG_PT_*) and,
 * with PDHG_SPEC_BEST_Z, takes z from the stored best z instead of
 * z = max(0, c - A'y) (pdhg.py:112-114).  The stored-z form is how the
 * reference re-checks best_pt with the z it was scored with (pdhg.py:249).
 * Writes PDHG_NQ doubles per point, in spec order, to out_host. */
#define PDHG_SPEC_BEST_Z 16
int pdhg_check(pdhg_ctx* ctx, int32_t npts, const int32_t* specs, double* out_host);

/* Same as pdhg_check but leaves the PDHG_NQ*npts scalars in device memory
 * (pdhg_vector(ctx, PDHG_VEC_SCALARS)) without synchronising -- sharded
 * hosts all-gather them and combine per-shard partials in rank order. */
int pdhg_check_device(pdhg_ctx* ctx, int32_t npts, const int32_t* specs);

/* Check -> next step reuse.  With check_dot enabled (needs the sliced-ELL
 * layout of A' and one GPU, else PDHG_ERR_STATE), a two-point check also
 * leaves A'y of both checked points in the workspace.  The iterate the next
 * period starts from has one of those y's: the current point's when the
 * check does not restart or restarts to it, the average's after a restart to
 * the average (pdhg.py:234-240).  pdhg_use_check_dot(slot) (0 = first checked
 * point, 1 = second) makes the next period's first primal step
 * (pdhg.py:142-147) take that A'y instead of recomputing it -- the check's
 * dual side runs the primal step's own row loop, so the step's result is
 * bit for bit the same.  Valid only right after such a check (restart and
 * save_best in between are fine); any other call that moves the iterates
 * drops the dots.  Replaces the repeated `p.at_y(state.y)` of the first
 * pdhg_step after _score (pdhg.py:142, 201-204). */
int pdhg_check_dot_enable(pdhg_ctx* ctx, int32_t on);
int pdhg_use_check_dot(pdhg_ctx* ctx, int32_t slot);

/* Check fused into the steps.  With check_fuse enabled (needs the sliced-ELL
 * layouts of A and A' and one unsharded GPU, else PDHG_ERR_STATE), a
 * pdhg_run_period_check of >= 2 iterations whose points are exactly (CUR,
 * AVG) runs its last iteration with the check's A side inside it: the primal
 * step stores (xe, x, avg_x) per column as one 32-byte quad, the dual step
 * gathers the quads -- one pass over A for the step's A xe (pdhg.py:143) and
 * the check's A x, A avg_x (lp_core.py:436 for both points of pdhg.py:201-202)
 * -- and leaves each row's two primal residuals for the check, which
 * accumulates them in the separate A-side kernel's exact order: iterates and
 * check scalars are bit for bit those of the unfused path.  Since ABI 5 the
 * workspace holds the quads and residual pairs (32 bytes per column and 16
 * per row more than ABI 4's). */
int pdhg_check_fuse_enable(pdhg_ctx* ctx, int32_t on);

/* Restart at point `which` (CUR or AVG): x, y, avg_x, avg_y <- that point
 * (pdhg.py:235-238). */
int pdhg_restart(pdhg_ctx* ctx, int32_t which);

/* Best-point bookkeeping (pdhg.py:231-232).  With PDHG_BEST_Z the stored
 * best z <- max(0, c - A'y_which); with PDHG_BEST_XY best x,y <- point
 * `which`.  The split lets the host mirror the reference's aliasing: a
 * best point taken from the running average keeps its check-time z while
 * its x,y follow the average until the next restart (pdhg.py:147-148,237-238). */
#define PDHG_BEST_XY 1
#define PDHG_BEST_Z 2
int pdhg_save_best(pdhg_ctx* ctx, int32_t which, int32_t flags);

/* Copy point spec (as in pdhg_check) to host arrays (any may be NULL).
 * z is max(0, c - A'y) unless PDHG_SPEC_BEST_Z selects the stored best z. */
int pdhg_fetch(pdhg_ctx* ctx, int32_t spec, double* x_host, double* y_host, double* z_host);
/* Device-side form of pdhg_fetch (the KktPoint run_pdhg returns,
 * pdhg.py:249-258, with z = extract_reduced_costs, pdhg.py:112-114):
 * computes the point's z on the device (into scratch, unless spec carries
 * PDHG_SPEC_BEST_Z) and returns the device addresses of x, y, z (full padded
 * lengths), queued on the context's stream without synchronising -- for
 * callers with their own download path. */
int pdhg_point_device(pdhg_ctx* ctx, int32_t spec, const double** x_dev, const double** y_dev,
                      const double** z_dev);

/* Device vectors of the context (full, padded length), for host-driven
 * exchanges between shards (NCCL all-gather or device copies). */
#define PDHG_VEC_X 0
#define PDHG_VEC_XE 1
#define PDHG_VEC_XBAR 2
#define PDHG_VEC_XBEST 3
#define PDHG_VEC_ZBEST 4
#define PDHG_VEC_TN1 5
#define PDHG_VEC_TN2 6
#define PDHG_VEC_Y 7
#define PDHG_VEC_YBAR 8
#define PDHG_VEC_YBEST 9
#define PDHG_VEC_TM1 10
#define PDHG_VEC_SCALARS 11
#define PDHG_VEC_FAILWORD 12  /* the int64 first-failure iteration word of this context */
void* pdhg_vector(pdhg_ctx* ctx, int32_t which);

/* z = max(0, c - A'y) for this shard's rows of A' into z_slice (device):
 * extract_reduced_costs, pdhg.py:112-114. */
int pdhg_reduced_costs(pdhg_ctx* ctx, int32_t spec, double* z_slice);

/* Host-driven stepping (sharded execution exchanges vectors between the
 * half steps; pdhg_step, pdhg.py:140-151, split at the x+ / y+ boundary):
 * set the step parameters of the next steps (as
 * pdhg_run_period does), launch one primal (primal=1) or dual half step
 * number j, and read the first failing iteration (-1 = none, syncs). */
int pdhg_set_step(pdhg_ctx* ctx, int64_t iter0, double tau_over_omega, double sigma_omega,
                  double w0);
int pdhg_half_step(pdhg_ctx* ctx, int32_t primal, int32_t j);
/* One pass of a split half step (pass < 0: all passes).  An operator that is
 * not split runs whole at pass 0 and launches nothing at later passes, so a
 * host can always issue pass 0, (wait for the all-gather), pass 1. */
int pdhg_half_step_pass(pdhg_ctx* ctx, int32_t primal, int32_t j, int32_t pass);
/* Fused all-gather: from now on the primal (which = 0) / dual (which = 1)
 * step's epilogue also stores every new xe / y value into the full vector
 * of each of npeers peers, at this shard's slot (peers_dev: device array of
 * npeers pointers to the peers' full xe / y vectors -- other shards in this
 * process, or NVLink peer / symmetric-memory addresses).  npeers = 0 turns
 * it off.  The caller orders the next half step after every peer's writes
 * (stream order on one device; a cross-GPU barrier otherwise).
 * which = 2: peers_dev lists the other shards' fail words
 * (pdhg_vector(peer, PDHG_VEC_FAILWORD)); a non-finite iterate is then
 * recorded in all of them, so every shard stops at that iteration. */
int pdhg_set_peers(pdhg_ctx* ctx, int32_t which, const double* const* peers_dev, int32_t npeers);
int pdhg_fail_iter(pdhg_ctx* ctx, int64_t* fail_iter_out);

/* Power-iteration building blocks for sharded hosts: *out_dev = sum v^2
 * (fixed order) and v = w / s (IEEE division, pdhg.py:99). */
int pdhg_sumsq(pdhg_ctx* ctx, const double* v, int64_t len, double* out_dev);
int pdhg_div(pdhg_ctx* ctx, const double* w, double* v, int64_t len, double s);

/* Average device time (ms) of one launch of kernel `which` (0 = primal
 * step over A' rows, 1 = dual step over A rows, 2 = one whole iteration:
 * primal then dual) over `reps` launches, CUDA events on the context
 * stream.  The iterate is advanced. */
int pdhg_time_kernel(pdhg_ctx* ctx, int32_t which, int32_t reps, double tau_over_omega,
                     double sigma_omega, double* avg_ms_out);

/* Layout helper for the split dual step (A @ xe of pdhg.py:143 over column
 * chunks): split_out[(k-1)*m + i] = first
 * entry of row i whose column is >= k*chunk, k = 1..K-1.  Rows must have
 * sorted columns; *unsorted_out = 1 reports a row that has not (then do not
 * split).  flag_dev: 4 bytes of device scratch. */
int pdhg_split_build(int32_t m, const int32_t* ptr, const int32_t* col, int32_t K, int32_t chunk,
                     int32_t* split_out, int32_t* flag_dev, void* stream, int32_t* unsorted_out);

/* Layout helper: A' (CSR of the transpose, = CSC of A with rows ascending
 * in each column, as scipy's tocsc behind StandardLp.A_csc, lp_core.py:133-138)
 * from CSR A, all on the device.
 * tmp must hold pdhg_transpose_tmp_bytes(nnz, m, n) bytes. */
size_t pdhg_transpose_tmp_bytes(int64_t nnz, int32_t m, int32_t n);
int pdhg_transpose_csr(int32_t m, int32_t n, int64_t nnz, const int32_t* a_ptr,
                       const int32_t* a_col, const double* a_val, int32_t* at_ptr,
                       int32_t* at_col, double* at_val, void* tmp, size_t tmp_bytes,
                       void* stream);

/* PSR layout build (device; an optional step layout for the products of
 * pdhg.py:142-143).  pdhg_psr_plan fixes the row-block size R and
 * panel width W from the shape, counts entries per (row block, panel),
 * marks panels with >= min_staged entries as staged and returns the sizes
 * the caller must allocate: nblk, ntiles, and the number of entries that
 * land in staged panels (*staged_out) and in the layout (*nent_out; heavy
 * rows -- longer than heavy_threshold -- are left to the CSR heavy path).
 * tmp (pdhg_psr_tmp_bytes) carries the plan into pdhg_psr_build and must
 * not be touched in between. */
size_t pdhg_psr_tmp_bytes(int32_t rows, int32_t cols, int64_t nnz);
int pdhg_psr_plan(int32_t rows, int32_t cols, int64_t nnz, const int32_t* ptr, const int32_t* col,
                  int32_t heavy_threshold, int32_t min_staged, void* tmp, size_t tmp_bytes,
                  void* stream, int32_t* R_out, int32_t* W_out, int32_t* nblk_out,
                  int32_t* ngroups_out, int32_t* ntiles_out, int64_t* staged_out,
                  int64_t* nent_out);
int pdhg_psr_build(int32_t rows, int32_t cols, int64_t nnz, const int32_t* ptr, const int32_t* col,
                   const double* val, int32_t heavy_threshold, void* tmp, size_t tmp_bytes,
                   void* stream, int32_t* blk_tile_ptr, int32_t* tile_bin, int32_t* gstart,
                   uint16_t* rcnt, double* val_out, uint16_t* col16_out, int32_t* col_out,
                   uint8_t* heavy_out);

/* Ruiz equilibration on the device (hybridlp.transform.ruiz_equilibrate,
 * transform.py:35-77), bit-identical scales and scaled values: val (CSR of
 * A, nnz entries) is scaled in place; row_scale (m) and col_scale (n) are
 * written; lo/hi = 1/(1+tol), 1+tol; *applied_out = passes applied.  The
 * structural empty-row/column check (ScalingError) is the caller's. */
size_t pdhg_ruiz_tmp_bytes(int32_t m, int32_t n);
int pdhg_ruiz(int32_t m, int32_t n, int64_t nnz, const int32_t* ptr, const int32_t* col, double* val,
              double* row_scale, double* col_scale, int32_t max_iters, double lo, double hi,
              void* tmp, size_t tmp_bytes, void* stream, int32_t* applied_out);


/* Standard form of a general LP on the device (hybridlp.lp_core.to_standard_form,
 * lp_core.py:250-368).  Input: CSR of the general A
 * (m x n, sorted column indices, no duplicates), one sense code per row,
 * lower/upper bounds (+-inf allowed), rhs, c.  pdhg_stdform_plan sizes the
 * output (and flags non-finite matrix entries, GeneralLp.validate
 * lp_core.py:80-81); pdhg_stdform_build fills it: the standard-form CSR
 * (m_std+1 / nnz_std / nnz_std), b_std (m_std), c_std (n_std) and the
 * StandardFormMap arrays (lp_core.py:226-247): shifts, pos_col, neg_col (n),
 * slack_of_row, slack_coef, bound_var (m_std).  Bit-identical to the
 * reference's arrays.  obj_shift (a sequential sum over columns) is the
 * caller's.  tmp (pdhg_stdform_tmp_bytes) carries the plan into the build
 * and must not be touched in between. */
#define PDHG_SENSE_EQ 0
#define PDHG_SENSE_LE 1
#define PDHG_SENSE_GE 2
typedef struct pdhg_stdform_dims {
  int32_t m_std, n_std;
  int64_t nnz_std;
  int32_t n_struct;          /* structural columns (split variables count twice) */
  int32_t n_ineq;            /* slack/surplus columns of <= / >= rows */
  int32_t n_bound;           /* bound rows (finite upper bounds) */
  int32_t nonfinite_entries; /* 1 if A holds a NaN/inf entry */
} pdhg_stdform_dims;
size_t pdhg_stdform_tmp_bytes(int32_t m, int32_t n);
int pdhg_stdform_plan(int32_t m, int32_t n, int64_t nnz, const int32_t* ptr, const int32_t* col,
                      const double* val, const int8_t* sense, const double* lower,
                      const double* upper, void* tmp, size_t tmp_bytes, void* stream,
                      pdhg_stdform_dims* out);
int pdhg_stdform_build(int32_t m, int32_t n, int64_t nnz, const int32_t* ptr, const int32_t* col,
                       const double* val, const int8_t* sense, const double* rhs,
                       const double* lower, const double* upper, const double* c,
                       const pdhg_stdform_dims* dims, void* tmp, size_t tmp_bytes, void* stream,
                       int32_t* s_ptr, int32_t* s_col, double* s_val, double* b_std, double* c_std,
                       double* shifts, int32_t* pos_col, int32_t* neg_col, int32_t* slack_of_row,
                       double* slack_coef, int32_t* bound_var);


/* Finishing the PDHG point on the device: unscale_point
 * (transform.py:87-93), restrict_point (lp_core.py:371-385), lift_point
 * (lp_core.py:388-427), violation_summary (lp_core.py:468-485).
 * pdhg_spmv_seq: out[r] = sum over row r in stored order from 0.0 (scipy's
 * csr_matvec order, products rounded, no FMA) -- or base[r] - sum when base is
 * non-null; over the CSR of A' it reproduces scipy's A.T @ y.  All buffers are
 * device pointers; restrict/lift/unscale results are bit-identical to the
 * reference's.  pdhg_violation writes 5 host doubles: max|b - Ax|,
 * max|c - A'y - z|, c'x, b'y, x'z (dots in a fixed block-tree order). */
int pdhg_spmv_seq(int32_t rows, const int32_t* ptr, const int32_t* col, const double* val,
                  const double* v, const double* base, double* out, void* stream);
int pdhg_unscale_point(int32_t n, int32_t m, const double* row_scale, const double* col_scale,
                       const double* xs, const double* ys, const double* zs, double* x, double* y,
                       double* z, void* stream);
int pdhg_restrict_x(int32_t n_general, const int32_t* pos_col, const int32_t* neg_col,
                    const double* shifts, const double* x_std, double* x, void* stream);
int pdhg_lift_x(int32_t n_general, const double* x, const double* shifts, const int32_t* pos_col,
                const int32_t* neg_col, double* x_std, void* stream);
int pdhg_lift_slacks(int32_t m_std, const int32_t* slack_of_row, const double* slack_coef,
                     const double* r, double* x_std, void* stream);
int pdhg_lift_bound_duals(int32_t m_std, const int32_t* bound_var, const double* z_gen,
                          double* y_std, void* stream);
int pdhg_max0(int64_t len, const double* v, double* out, void* stream);
size_t pdhg_violation_tmp_bytes(int32_t m, int32_t n);
int pdhg_violation(int32_t m, int32_t n, const int32_t* a_ptr, const int32_t* a_col,
                   const double* a_val, const int32_t* at_ptr, const int32_t* at_col,
                   const double* at_val, const double* b, const double* c, const double* x,
                   const double* y, const double* z, void* tmp, size_t tmp_bytes, void* stream,
                   double* out_host);


/* Sliced-ELL build (device; the step / check / power-iteration layout of the
 * products at pdhg.py:89-109,142-143 for near-uniform rows): plan writes
 * width (nslices = ceil(rows/32)) and
 * sptr (nslices+1) and returns the slot count; optionally sort orders each
 * slice's rows by length (perm: lane -> row offset, inv: row offset -> lane,
 * both nslices*32 bytes); the caller allocates slots-sized col/val and calls
 * fill (inv NULL = unsorted).  Rows longer than heavy_threshold are left out. */
size_t pdhg_sell_tmp_bytes(int32_t rows);
int pdhg_sell_plan(int32_t rows, const int32_t* ptr, int32_t heavy_threshold, int32_t* width,
                   int64_t* sptr, void* tmp, size_t tmp_bytes, void* stream, int64_t* slots_out);
int pdhg_sell_sort(int32_t rows, const int32_t* ptr, int32_t heavy_threshold, uint8_t* perm, uint8_t* inv,
                   void* stream);
int pdhg_sell_fill(int32_t rows, const int32_t* ptr, const int32_t* col, const double* val,
                   int32_t heavy_threshold, const int64_t* sptr, const uint8_t* inv, int32_t* scol,
                   double* sval, void* stream);

/* Feature bits of the loaded build: 1 = the experiment layouts (PSR panels,
 * persistent period kernels, L2 persisting windows), compiled only with
 * -DPDHG_EXPERIMENTAL=1 (python -m paper_2603_03150_b200.build --experimental);
 * the product build rejects them in pdhg_ctx_create / pdhg_psr_*.
 * 2 = bounds-checked build (-DPDHG_BOUNDS_CHECK=1, --checked). */
int pdhg_features(void);
/* Bounds-checked build: out-of-bounds index count since the last call (and
 * the first index with its bound); resets the count.  Product build:
 * PDHG_ERR_STATE. */
int pdhg_debug_oob(int64_t* count, int64_t* first_index, int64_t* first_bound);

/* Row relabelling of a CSR matrix on the device (GpuOptions.row_order =
 * "length": the rows of A -- the y-space -- sorted by length inside windows so
 * the dual step's sliced-ELL slices hold rows of equal length).  New row r is
 * old row perm[r], entries keep their order; new_ptr (rows+1) holds the
 * scanned permuted lengths.  The LP is the same one with its constraints
 * renumbered: b is permuted alike and y is mapped back on every download. */
int pdhg_permute_rows(int32_t rows, const int32_t* perm, const int32_t* ptr, const int32_t* col,
                      const double* val, const int32_t* new_ptr, int32_t* new_col, double* new_val,
                      void* stream);


/* IPM hand-off (warmstart.py:62-107): center_toward_target
 * elementwise on the device with numpy's maximum / clip semantics (bit-identical
 * to the reference for the same mu), and a fixed-order dot product for
 * mu_target's x'z (OpenBLAS ddot in the reference; equal to rounding). */
int pdhg_center_toward_target(int64_t n, const double* x, const double* z, double mu, double alpha_min,
                              double delta_max, double* x_out, double* z_out, void* stream);
size_t pdhg_dot_tmp_bytes(void);
int pdhg_dot(int64_t n, const double* a, const double* b, void* tmp, size_t tmp_bytes, void* stream,
             double* out_host);

#ifdef __cplusplus
}
#endif
#endif /* PDHG_B200_H */
