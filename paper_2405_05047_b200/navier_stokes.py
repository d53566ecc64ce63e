"""Convenience wrapper owning one ns_ctx (argument marshalling only; every
operation is a call into libmgb200.so, include/ns.h)."""
from __future__ import annotations

from . import (MG_COARSE_DIRECT, ns_create, ns_destroy, ns_get_divergence, ns_get_state, ns_momentum,
               ns_set_coupling, ns_set_dirichlet, ns_set_force, ns_set_mass, ns_set_momentum, ns_set_params,
               ns_set_state, ns_step)
from .solver import Multigrid


class NavierStokes:
    """The explicit pressure-correction step of Alg. 2 for a
    problem carrying: pres_levels (pressure-Poisson hierarchy, coarse -> fine,
    with mean_w / mean_k), omega, n_u, n_p, mom_rp / mom_col / mom_val (nnz, 4),
    Pi, G, m_u, m_p, dir_rows, dir_vals, nu, dt (e.g. problems.ns.NsProblem)."""

    def __init__(self, P, *, rtol=1e-6, restart=30, max_iter=200, timing=False, precision=0, use_graphs=True,
                 device=0, vanka=False, omega=None):
        """vanka: the pressure levels' cell patches (pres_levels[l].patches) smooth
        with the Vanka-type patch smoother (mg_set_vanka) instead of Jacobi."""
        self.pressure = Multigrid(P.pres_levels, 1, omega=omega if omega else P.omega, coarse_mode=MG_COARSE_DIRECT,
                                  precision=precision, use_graphs=use_graphs, device=device, vanka=vanka)
        self.n_u, self.n_p = P.n_u, P.n_p
        self.ctx = ns_create(self.pressure.ctx, P.n_u, P.n_p)
        try:
            ns_set_momentum(self.ctx, P.mom_rp, P.mom_col, P.mom_val.reshape(-1))
            grp, gcol, gval = P.G
            ns_set_coupling(self.ctx, P.Pi, (grp, gcol, gval.reshape(-1)))
            ns_set_mass(self.ctx, P.m_u, P.m_p)
            ns_set_dirichlet(self.ctx, P.dir_rows, P.dir_vals.reshape(-1))
            ns_set_params(self.ctx, P.nu, P.dt, rtol=rtol, restart=restart, max_iter=max_iter, timing=timing)
        except Exception:
            self.close()
            raise

    def set_force(self, F):
        ns_set_force(self.ctx, F)

    def set_state(self, u, p, q):
        ns_set_state(self.ctx, u.reshape(-1), p, q)

    def get_state(self):
        import numpy as np
        u = np.zeros(3 * self.n_u)
        p = np.zeros(self.n_p)
        q = np.zeros(self.n_p)
        ns_get_state(self.ctx, u, p, q)
        return u.reshape(-1, 3), p, q

    def step(self):
        return ns_step(self.ctx)

    def momentum(self):
        import numpy as np
        u = np.zeros(3 * self.n_u)
        ns_momentum(self.ctx, u)
        return u.reshape(-1, 3)

    def divergence(self):
        import numpy as np
        d = np.zeros(self.n_p)
        ns_get_divergence(self.ctx, d)
        return d

    def close(self):
        if getattr(self, "ctx", None) is not None:
            ns_destroy(self.ctx)
            self.ctx = None
        if getattr(self, "pressure", None) is not None:
            self.pressure.close()
            self.pressure = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
