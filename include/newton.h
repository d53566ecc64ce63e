/* libmgb200 -- Newton's method around the GMRES + multigrid solver: the
 * paper's hybrid workflow in which "the Jacobian [is] assembled on the CPU"
 * and the linear systems are solved on the GPU (the Newton-Krylov
 * structure of P:343-347 with the V-cycle of Alg. gmg as preconditioner).
 * 2-3 Newton steps per time step, each re-uploading the
 * Jacobian of every level value-only (mg_update_matrix).
 *
 * One call of mg_newton runs, for k = 0, 1, ...:
 *   1. w_k (device, the caller's x) is copied to a pinned host buffer;
 *   2. assemble(user, w_k, F, NULL) fills the nonlinear residual F(w_k) (host,
 *      this rank's n_fine*bs entries);
 *   3. ||F_k||_2 (device dot over all ranks); stop when ||F_k|| <= ntol ||F_0||,
 *      ||F_k|| <= atol, or k = max_newton;
 *   4. unless the Jacobian is kept (below): assemble(user, w_k, NULL, vals)
 *      fills the BSR values of J(w_k) on every level -- vals[l] sized
 *      nnzb_l*bs*bs in the entry order the level's mg_set_matrix received
 *      (same sparsity pattern, constrained rows/columns already identity /
 *      eliminated), pinned host memory owned by the library -- and
 *      mg_update_matrix re-uploads every level (value-only; D^-1 and the
 *      coarse inverse rebuilt on the device);
 *      with reuse_rate > 0 the Jacobian is kept while ||F_k|| <=
 *      reuse_rate ||F_{k-1}||: "the usual inexact Newton algorithm, which
 *      only reassembles the Jacobian when the convergence rate deteriorates"
 *      (P:821);
 *   5. d = 0; mg_solve(d, -F_k) (GMRES or Richardson per opts->lin);
 *   6. w_{k+1} = H (w_k + d) on the device (H = mg_set_constraints' hanging
 *      matrix, skipped if none was set).
 * The context's matrices on entry must be a valid Jacobian (the one of the
 * initial iterate, say): with reuse_rate > 0 step 0 still rebuilds.
 *
 * Arguments: ctx fully set up (all levels, transfers, optional H); x device
 * pointer to this rank's fine-level rows (in/out); assemble must return
 * MG_OK or an error status, which aborts the iteration and is returned.
 * Synchronous (returns after the last host read).  Errors: MG_ERR_INVALID_ARG
 * (NULL ctx/x/assemble/opts, bad option values), any status of the calls
 * above; MG_NOT_CONVERGED when max_newton steps did not reach the tolerance
 * (x holds the last iterate, info is filled).  Multi-GPU: collective; the
 * callback sees this rank's rows only. */
#ifndef MGB200_NEWTON_H
#define MGB200_NEWTON_H

#include <stdint.h>

#include "mg.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef mg_status (*mg_newton_assemble_fn)(void *user, const double *w, double *F, double *const *vals);

typedef struct {
  int max_newton;     /* maximum Newton steps (linear solves), >= 0 */
  double ntol;        /* relative tolerance on ||F||_2 */
  double atol;        /* absolute tolerance on ||F||_2 */
  double reuse_rate;  /* keep the last Jacobian while ||F_k|| <= reuse_rate ||F_{k-1}|| (0: rebuild every step) */
  mg_solve_opts lin;  /* linear solver per Newton step */
} mg_newton_opts;

#define MG_NEWTON_MAX_HIST 32

typedef struct {
  int newton_its;                         /* linear solves performed */
  int gmres_its;                          /* total preconditioner applications */
  int jacobians;                          /* Jacobian assemblies + uploads performed */
  int converged;
  int lin_its[MG_NEWTON_MAX_HIST];        /* per Newton step */
  double res_norm[MG_NEWTON_MAX_HIST + 1];/* ||F_k||_2, k = 0 .. newton_its */
  double ms_assemble;                     /* host wall time: device->host copy of w + the callback */
  double ms_upload, ms_solve;             /* device time (CUDA events on the context's stream): every level's
                                             mg_update_matrix / mg_solve + the update w <- H(w + d) */
} mg_newton_info;

mg_status mg_newton(mg_ctx ctx, double *x, mg_newton_assemble_fn assemble, void *user, const mg_newton_opts *opts,
                    mg_newton_info *info);

/* y <- y + alpha x on this rank's rows of level `level` (n_l * bs doubles, device
 * pointers, caller-owned; x and y must not overlap partially).  Asynchronous on
 * the context's stream.  Errors: MG_ERR_INVALID_ARG (bad level, NULL vector with
 * rows), MG_ERR_NONFINITE (alpha not finite).  The Newton update w + d. */
mg_status mg_axpy(mg_ctx ctx, int level, double alpha, const double *x, double *y);

#ifdef __cplusplus
}
#endif
#endif /* MGB200_NEWTON_H */
