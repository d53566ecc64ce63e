"""Convenience wrapper owning one mg_ctx (argument marshalling only; every
operation is a call into libmgb200.so)."""
from __future__ import annotations

from . import (MG_COARSE_DIRECT, MG_GMRES, level_info, mg_apply_constraints, mg_create, mg_create_level, mg_destroy,
               mg_newton,
               mg_set_constraints, mg_set_matrix, mg_set_vanka, mg_set_mean_constraint, mg_set_smoother, mg_set_transfer, mg_setup, mg_solve,
               mg_vcycle, mg_vcycle_zero)


class Multigrid:
    """levels: coarse -> fine sequence of objects with attributes
    n, row_ptr, col, val (BSR, val shaped (nnzb, bs, bs) or flat), and for
    l >= 1 P = (row_ptr, col, w) (n_l x n_{l-1}) and wpe.  H (optional):
    (row_ptr, col, w) hanging matrix of the finest level.  Levels with
    attributes mean_w / mean_k (not None) carry the global constraint
    w^T x = 0 of a pure-Neumann operator.
    Multi-GPU: comm = (nranks, rank, id_bytes, transport) and levels carrying
    n_global, row_begin, row_end (this rank's rows; columns global), e.g. from
    problems.partition.
    vanka: levels carrying `patches` ((n_patches, nloc) rows, e.g. mesh cells)
    use the Vanka-type patch smoother (mg_set_vanka) instead of
    block-Jacobi."""

    def __init__(self, levels, bs, *, omega=0.8, nu_pre=2, nu_post=2, coarse_mode=MG_COARSE_DIRECT,
                 coarse_sweeps=20, use_graphs=True, device=0, stream=None, H=None, omegas=None, comm=None,
                 precision=0, vanka=False):
        self.bs = bs
        self.n = [int(L.n) for L in levels]
        self.ctx = mg_create(len(levels), bs, nu_pre=nu_pre, nu_post=nu_post, omega=omega,
                             coarse_mode=coarse_mode, coarse_sweeps=coarse_sweeps, use_graphs=use_graphs,
                             device=device, stream=stream, comm=comm, precision=precision)
        try:
            for l, L in enumerate(levels):
                ng = int(getattr(L, "n_global", L.n))
                rb = int(getattr(L, "row_begin", 0))
                mg_create_level(self.ctx, l, ng, rb, rb + int(L.n))
            for l, L in enumerate(levels):
                val = L.val.reshape(-1) if hasattr(L.val, "reshape") else L.val
                mg_set_matrix(self.ctx, l, L.row_ptr, L.col, val)
                if l > 0:
                    rp, col, w = L.P
                    mg_set_transfer(self.ctx, l, rp, col, w, getattr(L, "wpe", 1))
                if omegas is not None:
                    mg_set_smoother(self.ctx, l, omegas[l])
                if vanka and getattr(L, "patches", None) is not None:
                    mg_set_vanka(self.ctx, l, L.patches)
                if getattr(L, "mean_w", None) is not None:
                    mg_set_mean_constraint(self.ctx, l, L.mean_w, L.mean_k)
            if H is not None:
                mg_set_constraints(self.ctx, *H)
            mg_setup(self.ctx)
        except Exception:
            mg_destroy(self.ctx)
            self.ctx = None
            raise

    @property
    def n_dof(self) -> int:
        return self.n[-1] * self.bs

    def vcycle(self, x, b):
        mg_vcycle(self.ctx, x, b)

    def precondition(self, z, v):
        mg_vcycle_zero(self.ctx, z, v)

    def solve(self, x, b, method=MG_GMRES, restart=30, max_iter=200, rtol=1e-10):
        return mg_solve(self.ctx, x, b, method=method, restart=restart, max_iter=max_iter, rtol=rtol)

    def newton(self, x, assemble, *, max_newton=3, ntol=1e-8, atol=0.0, reuse_rate=0.0, restart=30, max_iter=200,
               rtol=1e-10):
        """Newton's method with the caller's CPU assembly (include/newton.h):
        assemble(w, F, vals) fills F(w) unless F is None and every level's
        Jacobian values unless vals is None.  Returns (status, info)."""
        sizes = [level_info(self.ctx, l)["nnzb"] * self.bs * self.bs for l in range(len(self.n))]
        return mg_newton(self.ctx, x, assemble, self.n_dof, sizes, max_newton=max_newton, ntol=ntol, atol=atol,
                         reuse_rate=reuse_rate, restart=restart, max_iter=max_iter, rtol=rtol)

    def apply_constraints(self, x):
        mg_apply_constraints(self.ctx, x)

    def close(self):
        if self.ctx is not None:
            mg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
