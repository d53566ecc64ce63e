"""Oracle multigrid: Alg. `gmg`, MG as stand-alone solver
and MG-preconditioned GMRES.  TEST INFRASTRUCTURE ONLY.

Written step by step in the paper's order and notation; every heavy operation
is one of the plain per-op C definitions in oracle/__init__.py.
Readings: Z3 coarse solve exact (LU) by default, "several steps of
the smoothing iteration" as option; Z5 right preconditioning, MGS,
restart m, a cycle ends at |g_{j+1}| <= rtol * beta_0 and the solve stops when
the true residual ||b - A x|| <= rtol * beta_0 (else it restarts) or on a happy
breakdown; Z6 Euclidean norm over all
DOFs; Z21 the coarse solve ignores the incoming x; iteration count = number of
preconditioner applications.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import (block_diag_inverse, bsr_to_dense, csr_transpose, dot, jacobi_sweep, lu_factor,
               lu_solve, nrm2, residual, spmv, transfer)


@dataclass
class MgLevel:
    n: int
    bs: int
    rp: np.ndarray
    col: np.ndarray
    val: np.ndarray
    P: tuple | None = None        # (rp, col, w) n x n_{l-1}: prolongation from level l-1
    wpe: int = 1
    dinv: np.ndarray | None = None
    R: tuple | None = None        # R_{l-1} = P_{l-1}^T (built here)
    vanka: tuple | None = None    # (patches, A_pp^{-1}, W) of the Vanka smoother, or None


@dataclass
class MgHierarchy:
    levels: list                  # coarse -> fine
    omega: float = 0.8
    nu_pre: int = 2
    nu_post: int = 2
    coarse: str = "direct"        # "direct" | "smooth"
    coarse_sweeps: int = 20
    H: tuple | None = None        # fine-level hanging matrix
    lu: tuple | None = field(default=None, repr=False)
    mean: list | None = None      # per level: (w, k) of the global constraint w^T x = 0, or None

    @classmethod
    def from_arrays(cls, levels, omega=0.8, nu_pre=2, nu_post=2, coarse="direct", coarse_sweeps=20, H=None,
                    mean=None, vanka=False):
        """levels: list (coarse -> fine) of objects with n, bs, row_ptr, col, val,
        P (or None), wpe.  mean: per level (w, k) or None -- the global
        constraint int_Omega p = w^T x = 0 imposed on every level of a
        singular operator with kernel span{k} (pure-Neumann scalar problems:
        k = 1 on free DOFs, 0 on identity rows; w = lumped-mass weights)."""
        out = []
        for l, L in enumerate(levels):
            lv = MgLevel(L.n, L.bs, np.asarray(L.row_ptr, np.int64), np.asarray(L.col, np.int64),
                         np.asarray(L.val, np.float64), L.P if l > 0 else None, getattr(L, "wpe", 1))
            lv.dinv = block_diag_inverse(lv.n, lv.bs, lv.rp, lv.col, lv.val)
            if vanka and getattr(L, "patches", None) is not None:
                lv.vanka = vanka_setup(lv, L.patches)
            if l > 0:
                prp, pcol, pw = lv.P
                lv.R = csr_transpose(lv.n, out[-1].n, prp, pcol, pw, lv.wpe)
            out.append(lv)
        h = cls(out, omega, nu_pre, nu_post, coarse, coarse_sweeps, H)
        if mean is not None:
            h.mean = [None if c is None else (np.asarray(c[0], np.float64), np.asarray(c[1], np.float64))
                      for c in mean]
        if coarse == "direct":
            c = out[0]
            A0 = bsr_to_dense(c.n, c.bs, c.rp, c.col, c.val)
            if h.mean is not None and h.mean[0] is not None:
                A0 = A0 + coarse_regularisation(A0, h.mean[0][0])
            h.lu = lu_factor(A0)
        return h

    # --- the operations of Alg. gmg on level l -------------------------------
    def A(self, l, x):
        L = self.levels[l]
        return spmv(L.n, L.bs, L.rp, L.col, L.val, x)

    def smooth(self, l, x, b):
        """S_l(x, b): one damped block-Jacobi step x + omega D^{-1}(b - A x),
        or a Vanka patch step on levels with patches."""
        L = self.levels[l]
        if getattr(L, "vanka", None) is not None:
            return vanka_sweep(L, L.vanka, self.omega, x, b)
        return jacobi_sweep(L.n, L.bs, L.rp, L.col, L.val, L.dinv, self.omega, x, b)

    def restrict(self, l, r):
        """R_{l-1} r with R = P^T."""
        L = self.levels[l]
        rrp, rcol, rw = L.R
        return transfer(self.levels[l - 1].n, L.bs, rrp, rcol, rw, L.wpe, r)

    def prolongate_add(self, l, x, y):
        """x + P_{l-1} y."""
        L = self.levels[l]
        prp, pcol, pw = L.P
        return transfer(L.n, L.bs, prp, pcol, pw, L.wpe, y, x)

    def coarse_solve(self, b):
        """Step 0: A_0^{-1} b_0, or coarse_sweeps smoothing steps from 0."""
        if self.coarse == "direct":
            return lu_solve(self.lu[0], self.lu[1], b)
        x = np.zeros_like(b)
        for _ in range(self.coarse_sweeps):
            x = self.smooth(0, x, b)
        return x


def vanka_setup(L, patches):
    """Vanka-type smoother data: for every patch p (rows patches[p]) the
    dense inverse of A_pp -- the blocks of A between the patch's nodes, absent
    blocks zero -- by LAPACK (numpy.linalg.inv, a library primitive), and the
    weights W = 1 / (number of patches holding the row)."""
    patches = np.asarray(patches, np.int64)
    npch, nl = patches.shape
    bs, n = L.bs, L.n
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(L.rp))
    keys = rows * n + L.col                                   # ascending (CSR, sorted columns)
    q = (patches[:, :, None] * n + patches[:, None, :]).ravel()
    pos = np.minimum(np.searchsorted(keys, q), len(keys) - 1)
    hit = keys[pos] == q
    blk = np.where(hit[:, None, None], L.val.reshape(-1, bs, bs)[pos], 0.0).reshape(npch, nl, nl, bs, bs)
    A_pp = blk.transpose(0, 1, 3, 2, 4).reshape(npch, nl * bs, nl * bs)
    mult = np.bincount(patches.ravel(), minlength=n)
    if np.any(mult == 0):
        raise ValueError("row in no patch")
    return patches, np.linalg.inv(A_pp), 1.0 / mult


def vanka_sweep(L, vk, omega, x, b):
    """One Vanka step x + omega sum_p R_p^T W A_pp^{-1} R_p (b - A x)."""
    patches, inv, w = vk
    bs = L.bs
    r = residual(L.n, bs, L.rp, L.col, L.val, x, b).reshape(-1, bs)
    rp = r[patches].reshape(len(patches), -1)                  # R_p r
    c = np.einsum("pij,pj->pi", inv, rp).reshape(len(patches), -1, bs)
    acc = np.zeros_like(r)
    np.add.at(acc, patches.ravel(), c.reshape(-1, bs))
    return np.asarray(x, np.float64) + omega * (w[:, None] * acc).reshape(-1)


def project_zero_mean(x, w, k=None):
    """x - (w^T x / w^T k) k: zero weighted mean, i.e. int x_h = 0 with lumped-mass
    weights w (SPEC project_zero_mean S:452-460); k = 1 by default, the
    kernel vector (1 on free DOFs, 0 on identity rows) otherwise."""
    x = np.asarray(x, np.float64)
    k = np.ones_like(x) if k is None else np.asarray(k, np.float64)
    return x - dot(w, x) / dot(w, k) * k


def consistent(b, k=None):
    """b - (k^T b / k^T k) k: the Euclidean projection onto range(A) = k-perp of a
    symmetric operator with kernel span{k} (solvability of the Neumann problem)."""
    b = np.asarray(b, np.float64)
    k = np.ones_like(b) if k is None else np.asarray(k, np.float64)
    return b - dot(k, b) / dot(k, k) * k


def coarse_regularisation(A0, w):
    """alpha w w^T with alpha = max|diag A0| / max(w)^2: A0 + alpha w w^T is
    nonsingular for a kernel span{1} (w > 0), and for consistent b its solution
    is the solution of A0 x = b with w^T x = 0 (reading DESIGN.md Z25)."""
    alpha = np.max(np.abs(np.diag(A0))) / np.max(w) ** 2
    return alpha * np.outer(w, w)


def vcycle(h: MgHierarchy, l: int, x: np.ndarray, b: np.ndarray) -> np.ndarray:
    """GMG(l, x_l, b_l) of Alg. `gmg`.  With a global constraint on
    level l: the restricted right-hand side is made consistent, and the
    corrections are shifted to zero weighted mean after the coarse solve and
    after post-smoothing (reading Z25)."""
    mc = h.mean[l] if h.mean is not None else None
    if l == 0:                                           # Step 0
        y = h.coarse_solve(consistent(b, mc[1]) if mc is not None else b)
        return project_zero_mean(y, *mc) if mc is not None else y
    for _ in range(h.nu_pre):                            # Step 1: pre-smooth
        x = h.smooth(l, x, b)
    L = h.levels[l]
    d = h.restrict(l, residual(L.n, L.bs, L.rp, L.col, L.val, x, b))   # Step 2
    if h.mean is not None and h.mean[l - 1] is not None:
        d = consistent(d, h.mean[l - 1][1])
    y = vcycle(h, l - 1, np.zeros(h.levels[l - 1].n * L.bs), d)         # Step 3
    x = h.prolongate_add(l, x, y)                        # Step 4
    for _ in range(h.nu_post):                           # Step 5: post-smooth
        x = h.smooth(l, x, b)
    return project_zero_mean(x, *mc) if mc is not None else x


def richardson(h: MgHierarchy, b, x0=None, rtol=1e-10, max_iter=100):
    """x^{(n)} = GMG(L, x^{(n-1)}, b) until ||b - A x|| <= rtol ||b - A x0||.
    Returns x, iterations, residual history."""
    Lf = len(h.levels) - 1
    F = h.levels[-1]
    if h.mean is not None and h.mean[-1] is not None:
        b = consistent(b, h.mean[-1][1])                 # solvable pure-Neumann rhs
    x = np.zeros(F.n * F.bs) if x0 is None else np.array(x0, np.float64)
    r0 = nrm2(residual(F.n, F.bs, F.rp, F.col, F.val, x, b))
    hist = [r0]
    if r0 == 0.0:
        return x, 0, hist
    for it in range(1, max_iter + 1):
        x = vcycle(h, Lf, x, b)
        hist.append(nrm2(residual(F.n, F.bs, F.rp, F.col, F.val, x, b)))
        if hist[-1] <= rtol * r0:
            return x, it, hist
    return x, max_iter, hist


def gmres(h: MgHierarchy, b, x0=None, rtol=1e-10, restart=30, max_iter=200, precondition=True, op=None):
    """Right-preconditioned GMRES(m) with modified Gram-Schmidt and Givens
    rotations (Saad §6.5.3 as cited at P:346; stored-Z form, reading O8/Z5).
    The iteration count is the number of preconditioner applications.
    op: optional outer operator (an MgLevel-like object with n, bs, rp, col,
    val) when the preconditioning hierarchy h approximates it (mixed-precision
    V-cycle); default the finest level of h.
    Returns x, iterations, history of |g_{j+1}| / beta_0 estimates, true rel. residual."""
    Lf = len(h.levels) - 1
    F = h.levels[-1] if op is None else op
    N = F.n * F.bs
    mc = h.mean[-1] if h.mean is not None else None
    if mc is not None:
        b = consistent(b, mc[1])                         # solvable pure-Neumann rhs
    x = np.zeros(N) if x0 is None else np.array(x0, np.float64)
    r = residual(F.n, F.bs, F.rp, F.col, F.val, x, b)
    beta0 = nrm2(r)
    hist = [1.0]
    if beta0 == 0.0:
        return x, 0, hist, 0.0
    its = 0
    beta = beta0
    while its < max_iter:
        m = min(restart, max_iter - its)
        V = np.zeros((m + 1, N))
        Z = np.zeros((m, N))
        Hh = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        V[0] = r / beta
        g[0] = beta
        k = 0
        happy = False                                    # happy breakdown h_{j+1,j} = 0
        for j in range(m):
            Z[j] = vcycle(h, Lf, np.zeros(N), V[j]) if precondition else V[j]
            its += 1
            w = spmv(F.n, F.bs, F.rp, F.col, F.val, Z[j])
            for i in range(j + 1):                       # modified Gram-Schmidt
                Hh[i, j] = dot(w, V[i])
                w = w - Hh[i, j] * V[i]
            hn = nrm2(w)
            Hh[j + 1, j] = hn
            for i in range(j):                           # previous rotations
                t = cs[i] * Hh[i, j] + sn[i] * Hh[i + 1, j]
                Hh[i + 1, j] = -sn[i] * Hh[i, j] + cs[i] * Hh[i + 1, j]
                Hh[i, j] = t
            rho = np.hypot(Hh[j, j], Hh[j + 1, j])
            cs[j] = Hh[j, j] / rho
            sn[j] = Hh[j + 1, j] / rho
            breakdown = hn == 0.0
            Hh[j, j] = rho
            Hh[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            hist.append(abs(g[j + 1]) / beta0)
            k = j + 1
            if abs(g[j + 1]) <= rtol * beta0 or breakdown:
                happy = breakdown
                break
            V[j + 1] = w / hn
        y = np.zeros(k)                                  # back substitution H y = g
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - Hh[i, i + 1:k] @ y[i + 1:k]) / Hh[i, i]
        for i in range(k):
            x = x + y[i] * Z[i]
        r = residual(F.n, F.bs, F.rp, F.col, F.val, x, b)
        beta = nrm2(r)
        if happy or beta <= rtol * beta0:               # converged on the TRUE residual; an estimate
            break                                        # below rtol with a true residual above it restarts
    if mc is not None:
        x = project_zero_mean(x, *mc)                    # the normalised solution int p = 0
    return x, its, hist, beta / beta0


def gmres_dcgs2(h: MgHierarchy, b, x0=None, rtol=1e-10, restart=30, max_iter=200, op=None):
    """Right-preconditioned GMRES(m) whose Arnoldi basis is orthogonalised by
    classical Gram-Schmidt with ONE delayed reorthogonalisation (DCGS2; reading
    Z29 in DESIGN.md -- an opt-in alternative to the paper's MGS, with
    the same Krylov space and the same minimal-residual iterate in exact
    arithmetic).  Step j, with Q_{j-1} = [q_0 .. q_{j-1}] final and u_j the
    once-projected (not normalised) new direction:
      1. z_j = B u_j (V-cycle), w^ = A z_j;
      2. one reduction: a = Q_{j-1}^T u_j, nu = u_j^T u_j, bb = Q_{j-1}^T w^,
         mu = u_j^T w^;
      3. beta = sqrt(nu - a^T a); q_j = (u_j - Q_{j-1} a) / beta; column j-1 of
         the Hessenberg matrix becomes final: [s_{j-1} + a ; beta];
      4. w_j = A B q_j = (w^ - Q_j t) / beta with t = Hbar_{j-1} a (Arnoldi
         relation A B Q_{j-1} = Q_j Hbar_{j-1}); its first projection
         s_j = Q_j^T w_j = [(bb - t_{0:j}) / beta ; ((mu - a^T bb)/beta - t_j)/beta];
      5. u_{j+1} = w_j - Q_j s_j = w^/beta - Q_j (t/beta + s_j);
      6. the tentative column j = [s_j ; ||u_{j+1}||] gives the Givens estimate
         |g_{j+1}| that ends the cycle (its reorthogonalisation correction is
         O(eps) and is folded in at step j+1 by redoing rotation j).
    Since z_j = B u_j and U = Q R (R upper triangular: R[:j, j] = a, R[j, j] =
    beta), the update is x += Z (R^{-1} y) with y from H y = g.
    Returns x, iterations, history of estimates, true relative residual (as gmres)."""
    Lf = len(h.levels) - 1
    F = h.levels[-1] if op is None else op
    N = F.n * F.bs
    mc = h.mean[-1] if h.mean is not None else None
    if mc is not None:
        b = consistent(b, mc[1])
    x = np.zeros(N) if x0 is None else np.array(x0, np.float64)
    r = residual(F.n, F.bs, F.rp, F.col, F.val, x, b)
    beta0 = nrm2(r)
    hist = [1.0]
    if beta0 == 0.0:
        return x, 0, hist, 0.0
    its = 0
    beta_true = beta0
    while its < max_iter:
        m = min(restart, max_iter - its)
        Q = np.zeros((m + 1, N))       # slot j: u_j until step j turns it into q_j
        Z = np.zeros((m, N))           # z_j = B u_j
        Hraw = np.zeros((m + 1, m))    # unrotated Hessenberg columns (final or tentative)
        R = np.zeros((m, m))
        cs, sn = np.zeros(m), np.zeros(m)
        g = np.zeros(m + 1)
        gpre = np.zeros(m + 1)         # g_j before rotation j (rotation j is redone at step j+1)
        Q[0] = r
        k = 0
        happy = False

        def rotate(j):                  # rotations 0..j-1 applied to raw column j, then rotation j
            col = Hraw[:j + 2, j].copy()
            for i in range(j):
                t = cs[i] * col[i] + sn[i] * col[i + 1]
                col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1]
                col[i] = t
            rho = np.hypot(col[j], col[j + 1])
            cs[j] = col[j] / rho
            sn[j] = col[j + 1] / rho
            g[j + 1] = -sn[j] * gpre[j]
            g[j] = cs[j] * gpre[j]

        for j in range(m):
            u = Q[j]
            Z[j] = vcycle(h, Lf, np.zeros(N), u)
            its += 1
            wh = spmv(F.n, F.bs, F.rp, F.col, F.val, Z[j])
            a = np.array([dot(Q[i], u) for i in range(j)])
            bb = np.array([dot(Q[i], wh) for i in range(j)])
            nu = dot(u, u)
            mu = dot(u, wh)
            beta = np.sqrt(max(nu - float(a @ a) if j else nu, 0.0))
            R[:j, j] = a
            R[j, j] = beta
            if j == 0:
                g[0] = beta                            # = ||r0|| of this cycle
            else:
                Hraw[:j, j - 1] += a                   # column j-1 final: [s_{j-1} + a ; beta]
                Hraw[j, j - 1] = beta
                rotate(j - 1)
            if beta == 0.0:                            # u_j in span(Q_{j-1}): breakdown at j-1
                happy = True
                break
            t = Hraw[:j + 1, :j] @ a if j else np.zeros(1)
            s = np.empty(j + 1)
            s[:j] = (bb - t[:j]) / beta
            s[j] = ((mu - float(a @ bb) if j else mu) / beta - t[j]) / beta
            c = t / beta + s
            q = u.copy()
            for i in range(j):
                q = q - a[i] * Q[i]
            q = q / beta
            un = wh / beta
            for i in range(j):
                un = un - c[i] * Q[i]
            un = un - c[j] * q
            Q[j] = q
            Q[j + 1] = un
            hn = nrm2(un)
            Hraw[:j + 1, j] = s                         # tentative column j
            Hraw[j + 1, j] = hn
            gpre[j] = g[j]
            rotate(j)
            hist.append(abs(g[j + 1]) / beta0)
            k = j + 1
            if abs(g[j + 1]) <= rtol * beta0 or hn == 0.0:
                happy = hn == 0.0
                break
        if k:
            Hr = np.zeros((k, k))                      # rotated H (upper triangular)
            for jj in range(k):
                col = Hraw[:jj + 2, jj].copy()
                for i in range(jj + 1):
                    t = cs[i] * col[i] + sn[i] * col[i + 1]
                    col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1]
                    col[i] = t
                Hr[:jj + 1, jj] = col[:jj + 1]
            y = np.zeros(k)                            # back substitution H y = g
            for i in range(k - 1, -1, -1):
                y[i] = (g[i] - Hr[i, i + 1:k] @ y[i + 1:k]) / Hr[i, i]
            yp = np.zeros(k)                           # R y' = y
            for i in range(k - 1, -1, -1):
                yp[i] = (y[i] - R[i, i + 1:k] @ yp[i + 1:k]) / R[i, i]
            for i in range(k):
                x = x + yp[i] * Z[i]
        r = residual(F.n, F.bs, F.rp, F.col, F.val, x, b)
        beta_true = nrm2(r)
        if happy or beta_true <= rtol * beta0:
            break
    if mc is not None:
        x = project_zero_mean(x, *mc)
    return x, its, hist, beta_true / beta0


def apply_H(H, x, bs):
    """x <- H x after the solve (reading Z7)."""
    rp, col, w = H
    n = len(rp) - 1
    return transfer(n, bs, rp, col, w, 1, x)
