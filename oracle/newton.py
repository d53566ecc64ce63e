"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Newton's method for one backward-Euler time step of the C4 Navier-Stokes
system (the paper's hybrid workflow P:821: the Jacobian is
rebuilt on the CPU and the linear systems are solved by GMRES preconditioned
with the multigrid V-cycle).  Written out in the textbook order:

    for k = 0, 1, ...:
        F_k = F(w_k);            stop if ||F_k|| <= ntol ||F_0||  (or k = max_newton)
        J_k = J(w_k) on every level (rediscretised) -- or, with
              reuse_rate > 0 and ||F_k|| <= reuse_rate ||F_{k-1}||, J_{k-1} kept
              ("inexact Newton ... only reassembles the Jacobian when the
              convergence rate deteriorates")
        solve J_k d = -F_k       (right-preconditioned GMRES(m) + GMG(L, 0, .), x0 = 0)
        w_{k+1} = H (w_k + d)    (hanging values re-interpolated)

`residual(w)` and `jacobians(w)` are the caller's CPU assembly (problems/
channel.py); this module only sequences them.
"""
from __future__ import annotations

import numpy as np

from .mg import MgHierarchy, apply_H, gmres


def newton_step(levels_of, residual, jacobians, H, w, *, omega, rtol=1e-10, ntol=1e-8, max_newton=3,
                restart=30, max_iter=200, reuse_rate=0.0):
    """levels_of(vals) -> LevelData list with those values; residual(w) -> F (flat);
    jacobians(w) -> per-level values; H: finest hanging matrix (rp, col, w).
    Returns (w, history) with history = [(||F_k||, gmres iterations)]."""
    bs = w.shape[1]
    w = np.array(w, np.float64)
    hist = []
    F0 = None
    h = None
    for k in range(max_newton + 1):
        Fk = residual(w)
        nF = float(np.linalg.norm(Fk))
        if F0 is None:
            F0 = nF
        if k == max_newton or nF <= ntol * F0 or nF == 0.0:
            hist.append((nF, 0))
            break
        if h is None or not (reuse_rate > 0.0 and nF <= reuse_rate * hist[-1][0]):
            h = MgHierarchy.from_arrays(levels_of(jacobians(w)), omega=omega)
        d, its, _, _ = gmres(h, -Fk, rtol=rtol, restart=restart, max_iter=max_iter)
        hist.append((nF, its))
        w = apply_H(H, (w.reshape(-1) + d), bs).reshape(-1, bs)
    return w, hist
