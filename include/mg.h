/*
 * mg.h -- C ABI of libmgb200.so: the fp64 geometric-multigrid hot path of
 * arXiv 2405.05047 ("CUDA-Gascoigne 3d"), B200-native (sm_100a).
 *
 * Citation convention: P:n = line n of the paper's PAPER.md; S:n = SPEC.md;
 * Alg. `gmg` = the paper's Algorithm 1.  SURVEY.md §8(b) is the
 * design this header implements.
 *
 * What the library computes:
 *   - the V-cycle GMG(l, x_l, b_l) of Alg. `gmg`: Step 0 coarse
 *     solve A_0^{-1} b_0 or "several steps of the smoothing
 *     iteration"; Step 1 pre-smoothing; Step 2 residual + restriction
 *     d = R_{l-1}(b - A x) with R = P^T; Step 3 recursion from a
 *     zero guess; Step 4 x += P_{l-1} y; Step 5 post-smoothing;
 *   - the smoother x <- x + omega S (b - A x) with S the inverse n_c x n_c
 *     diagonal blocks (block Jacobi);
 *   - MG-preconditioned GMRES with modified Gram-Schmidt and Givens
 *     rotations, or MG as stand-alone iteration;
 *   - hanging-node interpolation y = H x.
 *
 * Data layout at the boundary (P:108, P:283 node-blocked unknowns):
 *   - block size bs = number of solution components n_c: 1, 2, 3, 4 or 6
 *     (6: the paper's first-order elasticity system (u, v));
 *   - vectors: fp64, node-major [n_rows * bs] (x_{i,c} at i*bs + c);
 *   - matrices: block-CSR (BSR), int64 row_ptr[n_rows+1] (row_ptr[0] == 0),
 *     int64 block column indices (strictly increasing within a row, in
 *     [0, n_cols)), fp64 values [nnzb * bs * bs], each block row-major;
 *   - transfers P_{l-1} (level l-1 -> level l, n_l x n_{l-1}) and H:
 *     CSR with int64 row_ptr / col and fp64 weights [nnz * weights_per_entry];
 *     weights_per_entry = 1 applies one scalar to every component,
 *     weights_per_entry = bs gives a per-component weight (component c of
 *     entry t at w[t*bs + c]).
 *
 * Levels: 0 is the coarsest, n_levels-1 the finest ("l = L ... 0").
 *
 * Ownership: every mg_set_* call COPIES its inputs (host or device memory, as
 * `mem` says) into context-owned device memory; the caller may free them on
 * return.  Vectors x, b, r, y passed to compute calls are caller-owned DEVICE
 * buffers of the level's rows x bs fp64 values; the library never keeps these
 * pointers past the call (graph caches key on the address only).  Outputs
 * must not alias inputs unless stated.  A rank that owns no rows of a level
 * may pass NULL vectors for it.
 *
 * Streams: all device work is ordered on the context's stream (the
 * cudaStream_t passed to mg_create, or an internal blocking stream if NULL,
 * which is ordered with the legacy default stream).  Compute calls are
 * asynchronous unless they return a host value (mg_dot, mg_solve).
 *
 * Errors: every call returns mg_status; nothing aborts or throws.
 * mg_last_error() returns a thread-local description of the last failure.
 * Invalid structure is rejected at mg_set_*; a singular diagonal block is
 * reported when the smoother is first built; non-convergence is
 * MG_NOT_CONVERGED with a valid x and info.
 */
#ifndef MGB200_MG_H
#define MGB200_MG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mg_ctx_s *mg_ctx;

typedef enum {
  MG_OK = 0,
  MG_NOT_CONVERGED = 1,     /* result valid, flagged in info */
  MG_ERR_INVALID_ARG = -1,  /* NULL pointer, bad level, bad option, aliasing */
  MG_ERR_DIMENSION = -2,    /* size mismatch between level / matrix / transfer */
  MG_ERR_STRUCTURE = -3,    /* row_ptr not monotone, cols unsorted / out of range, no diagonal block */
  MG_ERR_NONFINITE = -4,    /* NaN/Inf in matrix, weights, rhs or residual */
  MG_ERR_SINGULAR = -5,     /* singular diagonal block (D^-1) or singular coarse matrix */
  MG_ERR_STATE = -6,        /* call-order violation (e.g. vcycle before all levels are set) */
  MG_ERR_CUDA = -7,         /* CUDA runtime error; the context should be destroyed */
  MG_ERR_NCCL = -8,         /* NCCL error (multi-GPU) */
  MG_ERR_OOM = -9           /* device allocation failed */
} mg_status;

enum { MG_MEM_HOST = 0, MG_MEM_DEVICE = 1 };
enum { MG_TRANSPORT_NCCL = 0, MG_TRANSPORT_LOCAL = 1, MG_TRANSPORT_IPC = 2 };
enum { MG_COARSE_DIRECT = 0, MG_COARSE_SMOOTH = 1 };
enum { MG_GMRES = 0, MG_RICHARDSON = 1, MG_GMRES_DCGS2 = 2 };
enum { MG_PREC_FP64 = 0, MG_PREC_MIXED = 1 };

/* Global multigrid configuration (SPEC MgConfig; readings Z1-Z3).
 * omega: damping of the block-Jacobi smoother ("a damping factor");
 * nu_pre / nu_post: smoothing steps (Alg. gmg Steps 1 and 5);
 * coarse_mode: MG_COARSE_DIRECT = exact A_0^{-1} applied as a dense
 *   inverse, MG_COARSE_SMOOTH = coarse_sweeps smoothing steps from 0;
 * use_graphs: capture V-cycles into CUDA graphs (1) or launch eagerly (0);
 * precision: MG_PREC_FP64 (everything fp64), or MG_PREC_MIXED -- the
 *   V-cycle's operators A_l are stored rounded to fp32 (fp64 vectors, fp64
 *   accumulation, fp64 D^-1 / transfers / coarse inverse) while the finest
 *   level also keeps its fp64 A for the Krylov operator, residuals and
 *   mg_spmv / mg_residual ("single precision ... effectively
 *   doubles the arithmetic intensity").  MG iteration then runs as defect
 *   correction x += GMG(L, 0, b - A x) so both methods converge to the fp64
 *   solution. */
typedef struct {
  int n_levels;
  int block_size;
  int nu_pre;
  int nu_post;
  double omega;
  int coarse_mode;
  int coarse_sweeps;
  int use_graphs;
  int precision;
} mg_config;

/* Multi-GPU communicator description: NULL (or nranks == 1) => single GPU.
 * Row-partitioned solve, one rank per GPU (the paper is
 * single-GPU and names multi-GPU as future work).
 * transport = MG_TRANSPORT_NCCL: one process per GPU; all ranks pass the same
 *   128-byte NCCL unique id (mg_get_unique_id on rank 0, broadcast by the
 *   caller, e.g. via torch.distributed).  Halos: grouped ncclSend/ncclRecv;
 *   dots: ncclAllReduce; agglomeration: all-gather.
 * transport = MG_TRANSPORT_LOCAL: all ranks are host threads of ONE process
 *   sharing one device (a test transport: the full distributed algorithm on a
 *   single GPU); nccl_id is any 128-byte group key shared by the ranks.
 * transport = MG_TRANSPORT_IPC: one PROCESS per rank on one node, any mix of
 *   devices (several ranks may share one GPU, which NCCL refuses: "Duplicate
 *   GPU detected").  Device data moves through per-rank mailbox buffers
 *   exported with CUDA IPC memory handles (peer loads over NVLink between
 *   GPUs), ordered by inter-process CUDA events; the ranks meet at a host
 *   barrier in a POSIX shared-memory segment named after the first 16 bytes
 *   of nccl_id (any 128-byte key, e.g. random bytes from rank 0, broadcast
 *   by the caller).  Host barriers make it not graph-capturable: contexts on
 *   it run eagerly.  A rank that does not arrive within 300 s turns every
 *   barrier into MG_ERR_STATE instead of a hang.
 * With nranks > 1 every mg_* call below is collective: all ranks call it, in
 * the same order, with their own rows. */
typedef struct {
  int nranks;
  int rank;
  int transport;
  unsigned char nccl_id[128];
} mg_comm;

/* Solve options (SPEC GmresConfig S:410-413; reading Z5).
 * method: MG_GMRES (right-preconditioned GMRES(restart), MGS + Givens),
 *   MG_GMRES_DCGS2 (the same GMRES with the basis orthogonalised by classical
 *   Gram-Schmidt with one delayed reorthogonalisation: one multi-dot pass and
 *   one update pass per Arnoldi step, 2 all-reduces instead of j + 2; same
 *   Krylov space and minimal-residual iterate, an opt-in departure from the
 *   paper's MGS, reading Z29; restart <= 64) or
 *   MG_RICHARDSON (x <- GMG(L, x, b));
 * max_iter: maximum number of preconditioner applications (= V-cycles);
 * rtol: stop when ||b - A x||_2 <= rtol * ||b - A x0||_2 (GMRES: the Givens
 *   estimate |g_{j+1}|, re-checked with the true residual at every restart
 *   and at exit). */
typedef struct {
  int method;
  int restart;
  int max_iter;
  double rtol;
} mg_solve_opts;

/* iterations = number of preconditioner applications; rel_residual = true
 * ||b - A x||_2 / ||b - A x0||_2 at exit; converged = 1 iff rel_residual-based
 * test (or the GMRES estimate) met rtol. */
typedef struct {
  int iterations;
  double rel_residual;
  int converged;
} mg_solve_info;

/* -------------------------------------------------------------------------- */
/* Context and levels                                                          */
/* -------------------------------------------------------------------------- */

/* NCCL unique id for a multi-GPU context (call on one rank only).
 * MG_ERR_NCCL if libnccl.so.2 cannot be loaded. */
mg_status mg_get_unique_id(unsigned char out[128]);

/* Create a context on CUDA device `device`, ordering work on `cuda_stream`
 * (a cudaStream_t, or NULL for an internal blocking stream).  cfg is copied.
 * comm == NULL (or nranks == 1) => single GPU. */
mg_status mg_create(mg_ctx *out, const mg_config *cfg, int device, void *cuda_stream,
                    const mg_comm *comm);

/* Declare level `level` with n_rows_global block rows, of which this rank owns
 * rows [row_begin, row_end).  Single GPU: row_begin = 0, row_end = n_rows_global.
 * Multi-GPU: either the ranks' ranges tile [0, n_rows_global) in rank order
 * (a DISTRIBUTED level) or every rank passes [0, n_rows_global) (a
 * REPLICATED level, computed redundantly on every rank).  Levels below a
 * replicated level must be replicated; the restricted residual entering the
 * first replicated level is all-gathered (agglomeration).  With the direct
 * coarse solve, level 0 must be replicated. */
mg_status mg_create_level(mg_ctx ctx, int level, int64_t n_rows_global, int64_t row_begin,
                          int64_t row_end);

/* Set the (condensed, constrained) system matrix A_l of level `level` as BSR
 * (see layout above).  Rows are this rank's owned rows; columns are GLOBAL
 * block indices.  Every row must contain its diagonal block (global column
 * row_begin + i for local row i).  Multi-GPU: the library renumbers columns
 * into owned + ghost and builds the halo plan itself.  The matrix is
 * copied to the device once and is immutable afterwards; calling
 * again replaces it (the Newton re-upload of P:821). */
mg_status mg_set_matrix(mg_ctx ctx, int level, const int64_t *row_ptr, const int64_t *col,
                        const double *vals, int64_t nnzb, int mem);

/* Replace the VALUES of level `level`'s matrix, keeping the sparsity of the
 * last mg_set_matrix (the Newton / time-step re-upload of P:821): vals
 * [nnzb * bs * bs] in the same BSR entry order.  Scattered into the device
 * layout through a stored index map, D^-1 (unless user-supplied) and, on
 * level 0 with the direct coarse solve, the dense coarse inverse are rebuilt
 * on the device; halo plans and captured CUDA graphs stay valid.  Rank-local
 * (no communication).  Synchronises.  MG_ERR_NONFINITE / MG_ERR_SINGULAR as
 * for mg_set_matrix. */
mg_status mg_update_matrix(mg_ctx ctx, int level, const double *vals, int mem);

/* Set P_{fine_level-1}: level fine_level-1 -> level fine_level (n_fine x
 * n_coarse CSR).  The restriction R = P^T is built by the
 * library with a stable counting sort (columns of each R row ascending). */
mg_status mg_set_transfer(mg_ctx ctx, int fine_level, const int64_t *row_ptr, const int64_t *col,
                          const double *w, int64_t nnz, int weights_per_entry, int mem);

/* Override the smoother of one level: damping omega, nu_pre / nu_post (-1 keeps
 * the config values; omega <= 0 keeps the config value) and optionally the
 * inverse diagonal blocks dinv [n_rows * bs * bs] (row-major blocks; NULL =>
 * computed from the diagonal blocks of A by Gauss-Jordan with partial
 * pivoting, reading Z10). */
mg_status mg_set_smoother(mg_ctx ctx, int level, double omega, int nu_pre, int nu_post,
                          const double *dinv, int mem);

/* Vanka-type smoother on one level ("a Vanka smoother can be easily
 * implemented with custom kernels"): patch-wise additive Schwarz
 *   x <- x + omega sum_p R_p^T W_p A_pp^{-1} R_p (b - A x),
 * replacing the block-Jacobi sweep of that level in every smoothing step
 * (mg_smooth, mg_sweep, the V-cycle, the smoothing coarse solve).
 * patch_nodes [n_patches * nloc]: the level's rows (local ids, distinct within
 * a patch; e.g. the 2^d nodes of each mesh cell); every row must lie in at
 * least one patch; W = diag(1 / number of patches holding the row), so
 * overlapping patches average.  A_pp (nloc*bs square, blocks of A between the
 * patch's nodes, absent blocks 0; the V-cycle operator's values, i.e. fp32-
 * rounded in mixed precision) is inverted on the device by Gauss-Jordan with
 * partial pivoting at setup and after mg_update_matrix.  Constraints:
 * nloc * block_size <= 32, level not distributed, mg_set_matrix first.
 * n_patches = 0 switches the level back to block-Jacobi.  Errors:
 * MG_ERR_STRUCTURE (node out of range / repeated / uncovered row),
 * MG_ERR_SINGULAR (singular A_pp, reported at setup), MG_ERR_STATE. */
mg_status mg_set_vanka(mg_ctx ctx, int level, int64_t n_patches, int nloc, const int64_t *patch_nodes, int mem);

/* Hanging-node matrix H of the finest level (n x n CSR, weights_per_entry 1;
 * identity rows at regular nodes, master weights at hanging nodes). */
mg_status mg_set_constraints(mg_ctx ctx, const int64_t *H_row_ptr, const int64_t *H_col,
                             const double *H_w, int64_t nnz, int mem);

/* Global constraint w^T x = 0 on level `level` of a singular operator with
 * kernel span{k}: the normalisation int_Omega p = 0 "on each grid level" of
 * pure-Neumann problems (SPEC project_zero_mean S:452-460, S:474;
 * reading Z25).  w, k: [n_rows * bs] level-local rows (host or device per
 * `mem`, copied); w = lumped-mass weights (0 at identity rows), k = the kernel
 * vector (1 at free DOFs, 0 at identity rows).  Collective on distributed
 * levels; requires w^T k > 0 and k^T k > 0 (checked at setup, over all ranks).
 * Effect on the V-cycle: restricted right-hand sides become consistent,
 * d -= (k^T d / k^T k) k; after the coarse solve and after each level's
 * post-smoothing, x -= (w^T x / w^T k) k.  A direct coarse solve inverts
 * A_0 + alpha w w^T with alpha = max_i |(A_0)_ii| / max(w)^2 (nonsingular;
 * for consistent d its solution solves A_0 y = d with w^T y = 0).  mg_solve
 * makes b consistent (internal copy; b is not modified) and returns x with
 * w^T x = 0.  mg_vcycle / mg_vcycle_zero expect a consistent b.  w == NULL
 * removes the constraint.  MG_ERR_NONFINITE on non-finite entries. */
mg_status mg_set_mean_constraint(mg_ctx ctx, int level, const double *w, const double *k, int mem);

/* x <- x - (w^T x / w^T k) k on level `level` (zero weighted mean, SPEC
 * project_zero_mean S:452-460).  Async; MG_ERR_STATE without a constraint. */
mg_status mg_project_zero_mean(mg_ctx ctx, int level, double *x);

/* b <- b - (k^T b / k^T k) k on level `level` (the consistent right-hand side
 * of the singular system).  Async; MG_ERR_STATE without a constraint. */
mg_status mg_make_consistent(mg_ctx ctx, int level, double *b);

/* Finalise setup (R, D^-1, coarse inverse, work vectors).  Optional: the
 * first compute call finalises implicitly. */
mg_status mg_setup(mg_ctx ctx);

/* Release all device memory of the context.  ctx may be NULL. */
mg_status mg_destroy(mg_ctx ctx);

/* -------------------------------------------------------------------------- */
/* Solver                                                                      */
/* -------------------------------------------------------------------------- */

/* One V-cycle x <- GMG(L, x, b) on the finest level (Alg. gmg).
 * x: in/out device [n*bs]; b: device [n*bs]; must not alias.  Async. */
mg_status mg_vcycle(mg_ctx ctx, double *x, const double *b);

/* Preconditioner application z = GMG(L, 0, v): the V-cycle from a zero
 * guess, whose first pre-smoothing step is A-free (x = omega D^-1 v).
 * z: out device; v: device; must not alias.  Async. */
mg_status mg_vcycle_zero(mg_ctx ctx, double *z, const double *v);

/* Solve A x = b on the finest level from the initial guess in x (GMRES+MG or
 * MG iteration, see mg_solve_opts).  Synchronises; fills info if non-NULL.
 * Returns MG_OK, MG_NOT_CONVERGED, or an error. */
mg_status mg_solve(mg_ctx ctx, double *x, const double *b, const mg_solve_opts *opts,
                   mg_solve_info *info);

/* -------------------------------------------------------------------------- */
/* Per-operation entry points (parity tests, custom drivers).  All async,     */
/* device pointers, level-local rows.                                          */
/* -------------------------------------------------------------------------- */

/* y = alpha A_l x + beta y; beta == 0 => y is not read. */
mg_status mg_spmv(mg_ctx ctx, int level, double alpha, const double *x, double beta, double *y);

/* One damped block-Jacobi step out of place (the fused smoother kernel):
 * x_out = x + omega D^-1 (b - A_l x).  x_out must not alias x, b. */
mg_status mg_sweep(mg_ctx ctx, int level, const double *x, const double *b, double *x_out);

/* r = b - A_l x (Alg. gmg Step 2 residual). */
mg_status mg_residual(mg_ctx ctx, int level, const double *x, const double *b, double *r);

/* `sweeps` damped block-Jacobi steps x <- x + omega D^-1 (b - A x) in place
 * (P:321-325).  Uses one internal work vector (ping-pong). */
mg_status mg_smooth(mg_ctx ctx, int level, double *x, const double *b, int sweeps);

/* d_coarse = R_{fine_level-1} r_fine with R = P^T. */
mg_status mg_restrict(mg_ctx ctx, int fine_level, const double *r_fine, double *d_coarse);

/* x_fine += P_{fine_level-1} y_coarse. */
mg_status mg_prolong_add(mg_ctx ctx, int fine_level, const double *y_coarse, double *x_fine);

/* Coarse solve of Alg. gmg Step 0 on level 0: y = A_0^{-1} d (direct) or
 * coarse_sweeps smoothing steps from zero. */
mg_status mg_coarse_solve(mg_ctx ctx, const double *d, double *y);

/* x <- H x on the finest level.  In place (uses a work vector). */
mg_status mg_apply_constraints(mg_ctx ctx, double *x);

/* b_bar = H^T b on the finest level: condensation of an unconstrained load
 * vector onto the regular nodes (the "distributing" hanging-node operation of
 * P:338).  Hanging entries of b_bar come out 0 (hanging nodes are never
 * masters).  b_bar must not alias b. */
mg_status mg_condense_rhs(mg_ctx ctx, const double *b, double *b_bar);

/* *out_host = (a, b) over the level's rows (deterministic single-pass grid
 * reduction; all-reduced over ranks).  Synchronises. */
mg_status mg_dot(mg_ctx ctx, int level, const double *a, const double *b, double *out_host);

/* Description of the last error on this thread ("" if none). */
const char *mg_last_error(void);

/* Library version string. */
const char *mg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MGB200_MG_H */
