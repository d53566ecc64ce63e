"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The explicit pressure-correction Navier-Stokes time step of Alg. 2
with the mass-lumped interpolated convection of Eqs. `conv_mass_lumping`,
`tp`, `multC`, written out in the paper's order with the signs of
the weak form Eq. `weaknstokes1` (SPEC ns_momentum_step S:535-545,
ns_pressure_step S:546-553, ns_pressure_update S:554-561; reading Z27).
Sparse products use scipy's CSR matvec (a library primitive); no fusion, no
reordering: every term is formed on its own, then summed.

Operators (all assembled by the caller, SPEC NsOperators S:501-505):
  K_v[i, j] = int grad phi_j . grad phi_i          (velocity stiffness, without nu)
  C_d[i, j] = int phi_j d_d phi_i                  (d = x, y, z)
  G_c[i, j] = int psi_j d_c phi_i                  (velocity rows, pressure columns)
  m_u, m_p                                         (lumped masses)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .mg import gmres, project_zero_mean


@dataclass
class NsOperators:
    K: sp.csr_matrix
    C: tuple          # (C_x, C_y, C_z)
    G: tuple          # (G_x, G_y, G_z), n_u x n_p
    m_u: np.ndarray
    m_p: np.ndarray
    dir_rows: np.ndarray
    dir_vals: np.ndarray
    nu: float
    dt: float

    @classmethod
    def from_arrays(cls, n_u, n_p, mom_rp, mom_col, mom_val, G, m_u, m_p, dir_rows, dir_vals, nu, dt):
        """mom_val (nnz, 4) = (K_v, C_x, C_y, C_z) on one pattern; G = (rp, col, vals (nnz, 3))."""
        mat = lambda rp, col, v, nc: sp.csr_matrix((v, col, rp), shape=(len(rp) - 1, nc))  # noqa: E731
        K = mat(mom_rp, mom_col, mom_val[:, 0], n_u)
        C = tuple(mat(mom_rp, mom_col, mom_val[:, 1 + d], n_u) for d in range(3))
        grp, gcol, gval = G
        Gs = tuple(mat(grp, gcol, gval[:, c], n_p) for c in range(3))
        return cls(K, C, Gs, np.asarray(m_u, np.float64), np.asarray(m_p, np.float64),
                   np.asarray(dir_rows), np.asarray(dir_vals, np.float64), float(nu), float(dt))


def nodewise_products(u):
    """v^d_{i,c} = u_{i,d} u_{i,c} (Eq. `tp`).
    Returns v with v[d][i, c]."""
    u = np.asarray(u, np.float64)
    return np.stack([u[:, d:d + 1] * u for d in range(3)])


def convection(ops: NsOperators, u):
    """conv(u)_{., c} = sum_d C_d v^d_{., c} (Eq. `multC`, P:686-689 with the sign of
    -n(u (x) u, chi) moved to the right-hand side)."""
    v = nodewise_products(u)
    out = np.zeros_like(u)
    for c in range(3):
        for d in range(3):
            out[:, c] += ops.C[d] @ v[d][:, c]
    return out


def gradient(ops: NsOperators, p):
    """(p, div chi) tested with chi = phi_i e_c: (G_c p)_i."""
    return np.stack([ops.G[c] @ p for c in range(3)], axis=1)


def divergence(ops: NsOperators, u):
    """d_j = (div u_h, psi_j) = sum_c (G_c^T u_{., c})_j (Alg. 2 Steps 2-3)."""
    return sum(ops.G[c].T @ u[:, c] for c in range(3))


def momentum(ops: NsOperators, u, p, q, F=None):
    """Alg. 2 Step 1: the explicit lumped-mass update
    u^m = u^{m-1} + dt (M_v^l)^{-1} [F - nu K_v u^{m-1} + conv(u^{m-1}) + grad(p^{m-1} + q^{m-1})],
    F = M_v^l f (lumped load, default 0), then the Dirichlet values re-imposed
    (SPEC S:538).  Returns u^m (n_u, 3)."""
    u = np.asarray(u, np.float64)
    visc = np.stack([ops.K @ u[:, c] for c in range(3)], axis=1)
    rhs = -ops.nu * visc + convection(ops, u) + gradient(ops, np.asarray(p) + np.asarray(q))
    if F is not None:
        rhs = rhs + F
    un = u + ops.dt * rhs / ops.m_u[:, None]
    un[ops.dir_rows] = ops.dir_vals
    return un


def pressure_rhs(ops: NsOperators, d):
    """Alg. 2 Step 2 right-hand side: -(1/k) (div u^m, phi)."""
    return -d / ops.dt


def pressure_update(ops: NsOperators, p, q, d):
    """Alg. 2 Step 3 with the lumped pressure mass:
    p^m = p^{m-1} + q^m - nu (M_p^l)^{-1} d, then int p^m = 0."""
    pn = np.asarray(p) + np.asarray(q) - ops.nu * d / ops.m_p
    return project_zero_mean(pn, ops.m_p)


def step(ops: NsOperators, h, u, p, q, F=None, rtol=1e-6, restart=30, max_iter=200):
    """One time step of Alg. 2: Step 1, Step 2 (GMRES+MG with int q = 0 on every
    level, x0 = 0), Step 3.  h: pressure-Poisson MgHierarchy with the mean
    constraints.  Returns (u^m, p^m, q^m, d, gmres_iterations)."""
    un = momentum(ops, u, p, q, F)
    d = divergence(ops, un)
    qn, its, _, rel = gmres(h, pressure_rhs(ops, d), rtol=rtol, restart=restart, max_iter=max_iter)
    pn = pressure_update(ops, p, qn, d)
    return un, pn, qn, d, its
