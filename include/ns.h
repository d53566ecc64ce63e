/* libmgb200 -- the explicit pressure-correction Navier-Stokes time step of
 * arXiv 2405.05047, Alg. 2 on the GPU.
 *
 * Discretisation (the caller assembles, SPEC NsOperators S:501-505):
 *   velocity V_h: Q1 on the midpoint refinement Omega_{h/2} (n_u nodes, three
 *     components, node-major (u_1, u_2, u_3) in user vectors);
 *   pressure Q_h = S_h: Q1 on Omega_h (n_p nodes);
 *   K_v[i,j] = int grad phi_j . grad phi_i, C_d[i,j] = int phi_j d_d phi_i
 *     (d = x, y, z), one pattern, 4 values per entry (K, C_x, C_y, C_z);
 *   Pi: nodal interpolation Q1(Omega_h) -> Q1(Omega_{h/2}) (n_u x n_p);
 *   G_c[i,j] = int psi_j d_c phi_i (n_u x n_p, 3 values per entry);
 *   m_u, m_p: lumped masses.
 *
 * One step (reading Z27; signs of the weak form P:610-613):
 *   Step 1:  u^m = u^{m-1} + dt/m_u [F - nu K_v u^{m-1}
 *            + sum_d C_d v^d + grad(p^{m-1} + q^{m-1})],  v^d_{i,c} = u_{i,d} u_{i,c}
 *            (Eqs. tp / multC), Dirichlet values re-imposed;
 *   Step 2:  d = sum_c G_c^T u^m_c, solve K_p q^m = -d/dt with the
 *            pressure solver (GMRES + MG, int q = 0 on every level, x0 = 0);
 *   Step 3:  p^m = p^{m-1} + q^m - nu d / m_p, then int p^m = 0.
 * The gradient grad(p)_c = G_c p is computed as C_c (Pi p): for the nested
 * Q1-iso-Q2 / Q1 pair psi_j = sum_k Pi_kj phi_k, so G_c = C_c Pi exactly (up to
 * rounding); the library relies on this identity.
 *
 * Memory: operators are copied at ns_set_* (host or device input per `mem`);
 * the state (u, p, q) lives in the context (ns_set_state / ns_get_state).
 * All calls run on the pressure solver's stream; ns_step synchronises (the
 * GMRES iterations do).  Errors: mg_status codes, message in mg_last_error().
 * Single GPU (the pressure context must not be distributed). */
#ifndef MGB200_NS_H
#define MGB200_NS_H

#include <stdint.h>

#include "mg.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ns_ctx_s *ns_ctx;

typedef struct {
  int iterations;      /* GMRES iterations of the pressure solve */
  double rel_residual; /* its final relative residual */
  int converged;
  double ms[4];        /* if timing: Step 1 (mom), d and rhs (pres-rhs), solve (pres-solve), Step 3 (pres-up) */
} ns_step_info;

/* pressure: an mg_ctx whose finest level is the pressure-Poisson system on
 * Omega_h (n_p rows, block size 1, mean constraint set; not owned, must
 * outlive the ns_ctx). */
mg_status ns_create(ns_ctx *out, mg_ctx pressure, int64_t n_u, int64_t n_p);
mg_status ns_destroy(ns_ctx ctx);

/* Velocity operators on one pattern: CSR (n_u x n_u), vals[nnz*4] = per
 * entry (K_v, C_x, C_y, C_z). */
mg_status ns_set_momentum(ns_ctx ctx, const int64_t *row_ptr, const int64_t *col, const double *vals,
                          int64_t nnz, int mem);

/* Pi (n_u x n_p, one weight per entry) and G (n_u x n_p, vals[nnz*3] = per
 * entry (G_x, G_y, G_z)); the divergence operator G^T is built by the library. */
mg_status ns_set_coupling(ns_ctx ctx, const int64_t *pi_row_ptr, const int64_t *pi_col, const double *pi_w,
                          int64_t pi_nnz, const int64_t *g_row_ptr, const int64_t *g_col, const double *g_vals,
                          int64_t g_nnz, int mem);

/* Lumped masses m_u[n_u], m_p[n_p] (positive). */
mg_status ns_set_mass(ns_ctx ctx, const double *m_u, const double *m_p, int mem);

/* Dirichlet velocity nodes rows[n] (ascending, distinct) with values vals[n*3]. */
mg_status ns_set_dirichlet(ns_ctx ctx, const int64_t *rows, const double *vals, int64_t n, int mem);

/* Lumped load F = M_v^l f [n_u*3] (NULL: f = 0). */
mg_status ns_set_force(ns_ctx ctx, const double *F, int mem);

/* nu = 1/Re, time step dt, pressure solve: GMRES(restart) to rtol, at most
 * max_iter iterations; timing != 0 fills ns_step_info.ms (CUDA events). */
mg_status ns_set_params(ns_ctx ctx, double nu, double dt, double rtol, int restart, int max_iter, int timing);

/* State (u[n_u*3] node-major, p[n_p], q[n_p]); host or device per `mem`. */
mg_status ns_set_state(ns_ctx ctx, const double *u, const double *p, const double *q, int mem);
mg_status ns_get_state(ns_ctx ctx, double *u, double *p, double *q, int mem);

/* One time step of Alg. 2 (Steps 1-3), advancing the state.  Returns MG_OK,
 * MG_NOT_CONVERGED (pressure solve; the step is still completed), or an error. */
mg_status ns_step(ns_ctx ctx, ns_step_info *info);

/* Step 1 alone from the current state (the state is not advanced): u_new
 * [n_u*3], host or device per `mem`. */
mg_status ns_momentum(ns_ctx ctx, double *u_new, int mem);

/* d = sum_c G_c^T u_c of the last ns_step ([n_p]; the Step-2 rhs is -d/dt). */
mg_status ns_get_divergence(ns_ctx ctx, double *d, int mem);

/* Kernels launched by the context so far. */
int64_t ns_launch_count(ns_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif /* MGB200_NS_H */
