"""Seeded input generator for the paper's explicit pressure-correction
Navier-Stokes step (Alg. 2): the 3D driven cavity on
the graded tensor-product mesh of P:706-718.

SEEDED INPUT GENERATOR (test/bench infrastructure; no solve arithmetic):
meshes, assembled matrices and initial states only.

Discretisation (SPEC ns_assemble S:527-533):
  * pressure / pressure-Poisson space S_h = Q_h: Q1 on the graded mesh Omega_h
    of (Nx, Ny, Nz) cells;
  * velocity space V_h: Q1 on its equidistant (midpoint) refinement
    Omega_{h/2} (the Q1-iso-Q2 / Q1 pair), three components, node-major
    (u_1, u_2, u_3) per node;
  * node numbering lexicographic, x fastest: n(i, j, k) = (k ny + j) nx + i.
Every cell is an axis-aligned box, so every Q1 matrix is a Kronecker
product of exact 1D integrals of piecewise-linear hats (2-point Gauss per
cell, exact for these degree <= 2 integrands):
  M = Mz (x) My (x) Mx,  K = Mz (x) My (x) Kx + Mz (x) Ky (x) Mx + Kz (x) My (x) Mx,
  C_x[i, j] = int phi_j d_x phi_i = Mz (x) My (x) Dx,  Dx[i, j] = int phi_j phi_i',
  G_c[i, j] = int psi_j d_c phi_i  (psi: pressure hats on Omega_h) from 1D
  fine x coarse quadrature (independent of the nesting identity G_c = C_c Pi).
Lumped masses m_i = sum_j (phi_j, phi_i) are Kronecker products of
1D row sums.
Mesh (reading Z26): x_i = (1 - cos(i pi / Nx)) / 2, same for y;
z_k = 1 + sin((2k - Nz) pi / (2 Nz)) on [0, 2] (the printed formula maps to
[0, 1], inconsistent with Omega = (0,1)^2 x (0,2)).
Boundary data: u = (0, 1, 0) on x = 1 (lid, including its edges),
u = 0 on the rest of the boundary.  Re = 1e3 (nu = 1e-3), dt = 1e-4.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from types import SimpleNamespace

import numpy as np
import scipy.sparse as sp

from .configs import SEED_BASE

GAUSS = np.array([0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0)])


# ---------------------------------------------------------------------------
# 1D pieces
# ---------------------------------------------------------------------------

def graded(N: int, axis: str) -> np.ndarray:
    """Node coordinates of the graded mesh (reading Z26), ascending."""
    i = np.arange(N + 1, dtype=np.float64)
    if axis in ("x", "y"):
        return 0.5 * (1.0 - np.cos(i * np.pi / N))
    return 1.0 + np.sin((2.0 * i - N) * np.pi / (2.0 * N))


def midpoint_refine(x: np.ndarray) -> np.ndarray:
    out = np.empty(2 * len(x) - 1)
    out[0::2] = x
    out[1::2] = 0.5 * (x[:-1] + x[1:])
    return out


def hat(xc: np.ndarray, j: int, t: float) -> float:
    """Value of the coarse hat psi_j (nodes xc) at the point t."""
    if t == xc[j]:
        return 1.0
    if t < xc[j]:
        if j == 0 or t <= xc[j - 1]:
            return 0.0
        return (t - xc[j - 1]) / (xc[j] - xc[j - 1])
    if j == len(xc) - 1 or t >= xc[j + 1]:
        return 0.0
    return (xc[j + 1] - t) / (xc[j + 1] - xc[j])


def fe1d(x: np.ndarray):
    """Mass M, stiffness K, convection D[i, j] = int phi_j phi_i' on nodes x,
    by 2-point Gauss on every cell (exact)."""
    n = len(x)
    rows, cols, m, k, d = [], [], [], [], []
    for a in range(n - 1):
        h = x[a + 1] - x[a]
        for q in GAUSS:
            w = 0.5 * h
            phi = np.array([1.0 - q, q])
            dphi = np.array([-1.0 / h, 1.0 / h])
            for il in range(2):
                for jl in range(2):
                    rows.append(a + il)
                    cols.append(a + jl)
                    m.append(w * (phi[il] * phi[jl]))
                    k.append(w * (dphi[il] * dphi[jl]))
                    d.append(w * phi[jl] * dphi[il])
    mk = lambda v: sp.csr_matrix((np.array(v), (rows, cols)), shape=(n, n))  # noqa: E731  (duplicates summed)
    return mk(m), mk(k), mk(d)


def cross1d(xf: np.ndarray, xc: np.ndarray):
    """Fine x coarse integrals on the fine cells: Mfc[i, j] = int phi_i psi_j,
    Gfc[i, j] = int psi_j phi_i' (phi: hats on xf, psi: hats on xc; xf refines
    xc), by 2-point Gauss per fine cell with psi evaluated from its own formula."""
    nf, nc = len(xf), len(xc)
    rows, cols, m, g = [], [], [], []
    for a in range(nf - 1):
        h = xf[a + 1] - xf[a]
        c = int(np.searchsorted(xc, 0.5 * (xf[a] + xf[a + 1]))) - 1   # coarse cell containing it
        for q in GAUSS:
            t = xf[a] + q * h
            w = 0.5 * h
            phi = np.array([1.0 - q, q])
            dphi = np.array([-1.0 / h, 1.0 / h])
            for jc in (c, c + 1):
                psi = hat(xc, jc, t)
                for il in range(2):
                    rows.append(a + il)
                    cols.append(jc)
                    m.append(w * phi[il] * psi)
                    g.append(w * psi * dphi[il])
    mk = lambda v: sp.csr_matrix((np.array(v), (rows, cols)), shape=(nf, nc))  # noqa: E731
    return mk(m), mk(g)


def interp1d(xf: np.ndarray, xc: np.ndarray) -> sp.csr_matrix:
    """P[i, j] = psi_j(xf_i): nodal interpolation of coarse Q1 into fine Q1
    (nested meshes; Eq. `prolongation`)."""
    rows, cols, w = [], [], []
    for i, t in enumerate(xf):
        c = int(np.searchsorted(xc, t))
        for j in (c - 1, c):
            if 0 <= j < len(xc):
                v = hat(xc, j, t)
                if v != 0.0:
                    rows.append(i)
                    cols.append(j)
                    w.append(v)
    return sp.csr_matrix((np.array(w), (rows, cols)), shape=(len(xf), len(xc)))


def kron3(az, ay, ax) -> sp.csr_matrix:
    return sp.kron(az, sp.kron(ay, ax, format="csr"), format="csr")


def lumped1d(M) -> np.ndarray:
    return np.asarray(M.sum(axis=1)).ravel()


def _csr(A: sp.csr_matrix):
    A = A.tocsr()
    A.sort_indices()
    return A.indptr.astype(np.int64), A.indices.astype(np.int64), A.data.astype(np.float64)


def tensor_csr(S, terms):
    """CSR of sum_t A^z_t (x) A^y_t (x) A^x_t for several matrices at once on the
    structural pattern S = (Sz, Sy, Sx) (dense boolean 1D patterns).
    terms: per output matrix a list of (az, ay, ax) dense 1D factors.
    Returns rp, col, vals (nnz, len(terms))."""
    Sz, Sy, Sx = S
    pat = kron3(sp.csr_matrix(Sz.astype(float)), sp.csr_matrix(Sy.astype(float)), sp.csr_matrix(Sx.astype(float)))
    pat.sort_indices()
    rp, col = pat.indptr.astype(np.int64), pat.indices.astype(np.int64)
    rows = np.repeat(np.arange(pat.shape[0], dtype=np.int64), np.diff(rp))
    nxr, nyr = Sx.shape[0], Sy.shape[0]
    nxc, nyc = Sx.shape[1], Sy.shape[1]
    ir, jr, kr = rows % nxr, (rows // nxr) % nyr, rows // (nxr * nyr)
    ic, jc, kc = col % nxc, (col // nxc) % nyc, col // (nxc * nyc)
    del rows
    vals = np.zeros((len(col), len(terms)))
    for m, tl in enumerate(terms):
        for az, ay, ax in tl:
            vals[:, m] += az[kr, kc] * (ay[jr, jc] * ax[ir, ic])
    return rp, col, vals


# ---------------------------------------------------------------------------
# The NS problem
# ---------------------------------------------------------------------------

@dataclass
class NsProblem:
    name: str
    cells: tuple                 # pressure mesh (Nx, Ny, Nz)
    xp: tuple                    # pressure-mesh coordinates per axis
    xu: tuple                    # velocity-mesh coordinates per axis
    n_u: int
    n_p: int
    mom_rp: np.ndarray           # (n_u+1,) velocity pattern (27-point)
    mom_col: np.ndarray
    mom_val: np.ndarray          # (nnz, 4): K_v, C_x, C_y, C_z  (K_v without the factor nu)
    Pi: tuple                    # (rp, col, w): Q1(Omega_h) -> Q1(Omega_h/2) interpolation, n_u x n_p
    G: tuple                     # (rp, col, vals (nnz, 3)): G_c[i, j] = int psi_j d_c phi_i, n_u x n_p
    m_u: np.ndarray              # (n_u,) lumped velocity mass
    m_p: np.ndarray              # (n_p,) lumped pressure mass
    dir_rows: np.ndarray         # (n_dir,) Dirichlet velocity nodes
    dir_vals: np.ndarray         # (n_dir, 3)
    pres_levels: list            # pressure-Poisson hierarchy (coarse -> fine), LevelData-like
    nu: float = 1e-3
    dt: float = 1e-4
    omega: float = 0.4           # Jacobi damping of the pressure MG: lambda_max(D^-1 A) = 4.42 on the graded mesh (Z27)
    meta: dict = field(default_factory=dict)

    @property
    def pres_fine(self):
        return self.pres_levels[-1]


def _pressure_level(xs, prev_xs):
    Ms, Ks = [], []
    for x in xs[::-1]:                       # z, y, x order for kron3
        M, K, _ = fe1d(x)
        Ms.append(M)
        Ks.append(K)
    Mz, My, Mx = Ms
    Kz, Ky, Kx = Ks
    A = kron3(Mz, My, Kx) + kron3(Mz, Ky, Mx) + kron3(Kz, My, Mx)
    rp, col, val = _csr(A)
    n = len(rp) - 1
    L = SimpleNamespace(n=n, bs=1, row_ptr=rp, col=col, val=val.reshape(-1, 1, 1), wpe=1, P=None)
    L.mean_w = np.kron(lumped1d(Mz), np.kron(lumped1d(My), lumped1d(Mx)))
    L.mean_k = np.ones(n)
    L.coords = xs
    # cells of the tensor-product mesh (Vanka patches): 8 nodes, lexicographic ids
    nx, ny, nz = (len(x) for x in xs)
    I, J, K = np.meshgrid(np.arange(nx - 1), np.arange(ny - 1), np.arange(nz - 1), indexing="ij")
    base = ((K * ny + J) * nx + I).ravel()
    L.patches = np.stack([base + o for o in (0, 1, nx, nx + 1, nx * ny, nx * ny + 1, nx * ny + nx,
                                             nx * ny + nx + 1)], axis=1).astype(np.int64)
    if prev_xs is not None:
        Pz, Py, Px = (interp1d(xs[a], prev_xs[a]) for a in (2, 1, 0))
        L.P = _csr(kron3(Pz, Py, Px))
    return L


def make_ns(name, cells, *, nu=1e-3, dt=1e-4, omega=0.4, coarse_cells=None) -> NsProblem:
    Nx, Ny, Nz = cells
    xp = (graded(Nx, "x"), graded(Ny, "y"), graded(Nz, "z"))
    xu = tuple(midpoint_refine(x) for x in xp)
    # pressure-Poisson hierarchy: subsample the graded coordinates (global coarsening
    # of the uniformly refined graded mesh) down to coarse_cells
    cc = coarse_cells or tuple(max(1, c // 8) for c in cells)
    hier = [xp]
    while all(len(x) - 1 > c for x, c in zip(hier[-1], cc)) and all((len(x) - 1) % 2 == 0 for x in hier[-1]):
        hier.append(tuple(x[::2] for x in hier[-1]))
    hier = hier[::-1]
    levels = []
    prev = None
    for xs in hier:
        levels.append(_pressure_level(xs, prev))
        prev = xs
    # velocity operators on the common 27-point pattern: K_v, C_x, C_y, C_z
    fe = [tuple(A.toarray() for A in fe1d(x)) for x in xu]   # per axis x, y, z: dense (M, K, D)
    (Mx, Kx, Dx), (My, Ky, Dy), (Mz, Kz, Dz) = fe
    S = tuple(M != 0.0 for M in (Mz, My, Mx))
    mom_rp, mom_col, mom_val = tensor_csr(S, [
        [(Mz, My, Kx), (Mz, Ky, Mx), (Kz, My, Mx)],       # K_v = int grad phi_j . grad phi_i
        [(Mz, My, Dx)],                                   # C_x[i, j] = int phi_j d_x phi_i
        [(Mz, Dy, Mx)],
        [(Dz, My, Mx)]])
    # cross-space operators G_c[i, j] = int psi_j d_c phi_i (fine rows, coarse columns)
    cr = [tuple(A.toarray() for A in cross1d(xu[a], xp[a])) for a in range(3)]
    (Mfx, Gfx), (Mfy, Gfy), (Mfz, Gfz) = cr
    S = tuple(M != 0.0 for M in (Mfz, Mfy, Mfx))
    G = tensor_csr(S, [[(Mfz, Mfy, Gfx)], [(Mfz, Gfy, Mfx)], [(Gfz, Mfy, Mfx)]])
    Pi = _csr(kron3(interp1d(xu[2], xp[2]), interp1d(xu[1], xp[1]), interp1d(xu[0], xp[0])))
    m_u = np.kron(Mz.sum(axis=1), np.kron(My.sum(axis=1), Mx.sum(axis=1)))
    m_p = levels[-1].mean_w.copy()
    # Dirichlet: the whole boundary; lid x = 1 carries (0, 1, 0)
    nx, ny, nz = (len(x) for x in xu)
    I, J, K = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    idx = ((K * ny + J) * nx + I).ravel()
    bnd = ((I == 0) | (I == nx - 1) | (J == 0) | (J == ny - 1) | (K == 0) | (K == nz - 1)).ravel()
    lid = (I == nx - 1).ravel()
    order = np.argsort(idx[bnd])
    dir_rows = idx[bnd][order].astype(np.int64)
    dir_vals = np.zeros((len(dir_rows), 3))
    dir_vals[:, 1] = lid[bnd][order].astype(float)
    return NsProblem(name, tuple(cells), xp, xu, nx * ny * nz, levels[-1].n, mom_rp, mom_col, mom_val, Pi, G,
                     m_u, m_p, dir_rows, dir_vals, levels, nu=nu, dt=dt, omega=omega,
                     meta={"coarse_cells": tuple(len(x) - 1 for x in hier[0]), "levels": len(levels)})


NS_CONFIGS = {
    # name: (pressure cells, seed index)
    "ns": ((32, 32, 64), 20),          # the paper's cavity: 70,785 pressure / 545,025 velocity nodes
    "ns_mid": ((8, 8, 16), 21),
    "ns_small": ((4, 4, 8), 22),
}


def build_ns(name: str, **kw) -> NsProblem:
    cells, si = NS_CONFIGS[name]
    P = make_ns(name, cells, **kw)
    P.meta["seed"] = SEED_BASE + si
    return P


def initial_state(P: NsProblem):
    """The paper's start (Alg. 2): u_0 = 0 with the boundary data, p^0 = q^0 = 0."""
    u = np.zeros((P.n_u, 3))
    u[P.dir_rows] = P.dir_vals
    return u, np.zeros(P.n_p), np.zeros(P.n_p)


def random_state(P: NsProblem, scale=1.0):
    """Seeded random state for parity tests: interior velocity N(0, scale^2),
    boundary data imposed; p, q N(0, 1)."""
    g = np.random.Generator(np.random.PCG64(P.meta["seed"]))
    u = scale * g.standard_normal((P.n_u, 3))
    u[P.dir_rows] = P.dir_vals
    p = g.standard_normal(P.n_p)
    q = g.standard_normal(P.n_p)
    return u, p, q
