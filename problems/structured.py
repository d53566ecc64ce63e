"""Per-rank generator of the C5 workload for weak scaling (SURVEY §8(d) C5,
§8(e); VERDICT r1 "next" 4).

SEEDED INPUT GENERATOR (test/bench infrastructure; no solve arithmetic).

C5 is a uniform box mesh: (0,1)x(0,1)x(0,2) cut into root * 2^R equal cubic
cells, equal-order Q1 generalised Stokes with 4x4 blocks (p, u, v, w; PSPG +
eps M_p, reading Z23), velocity Dirichlet on the boundary with the cavity lid
u_1 = 1 on z = 0.  Every cell has the same element matrix, so any rank can
assemble ITS OWN rows of every level directly (problems/csrc/assemble.c
`asm_structured`, `tr_structured`) without the global octree machinery of
problems/configs.py -- the only way to reach the 135M-DOF P = 8 size, which
no single host process can generate and ship.

Numbering: lexicographic, id = i + (nx+1) (j + (ny+1) k) (on a structured grid
a 32-row slice then gathers 32 consecutive x entries per neighbour offset).
Partition: contiguous z-plane ranges; the fine level's plane splitters apply
on every level (a coarse node lives with its coincident fine node), levels
with fewer than `min_rows_per_rank` rows per rank and level 0 are replicated
(agglomerated), as in problems/partition.py.
Right-hand side: standard normal per node, drawn plane by plane from
PCG64(SeedSequence([240505047 + 4, k])) so every rank draws the same values
for its planes whatever the partition; constrained entries then take their
boundary value (reading G8).

Weak-scaling sizes: P = 1 (4,4,8) * 2^5 = 128^2 x 256 cells
(17.1M DOFs), P = 2 (5,5,10) * 2^5, P = 4 (3,3,6) * 2^6, P = 8 (4,4,8) * 2^6
= 256^2 x 512 (135.5M DOFs, 16.9M per GPU).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import fem as F
from ._native import lib, ptr
from .configs import SEED_BASE, STOKES3

BOX = (1.0, 1.0, 2.0)
C5_WEAK = {1: ((4, 4, 8), 5), 2: ((5, 5, 10), 5), 4: ((3, 3, 6), 6), 8: ((4, 4, 8), 6)}
OMEGA = 0.6
SEED_INDEX = 4
BMASK = np.array([0, 1, 1, 1], np.uint8)   # velocity components Dirichlet on the boundary, pressure free
LID_COMP = 1                               # u_1 = 1 on the lid z = 0 (configs.lid)


@dataclass
class RankLevel:
    """One level of one rank: rows [row_begin, row_end) of n_global (global column ids)."""
    n: int
    bs: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray               # (nnzb, bs, bs)
    n_global: int
    row_begin: int
    row_end: int
    P: tuple | None = None        # (rp, col, w) rows = this rank's rows, cols = global coarse ids
    wpe: int = 4
    nx: int = 0
    ny: int = 0
    nz: int = 0

    @property
    def nnzb(self) -> int:
        return int(self.row_ptr[-1])


def grid(root, l):
    return tuple(int(r) << l for r in root)


def n_nodes(g):
    return (g[0] + 1) * (g[1] + 1) * (g[2] + 1)


def element_matrix(op: F.Operator, g) -> np.ndarray:
    """The single element matrix of the uniform grid g: A_e = sum_t S_t T_t
    (problems/fem.py element_terms), summed in term order."""
    h = np.array([[BOX[a] / g[a] for a in range(3)]])
    T, S = F.element_terms(op, 3, h)
    Ae = np.zeros(T.shape[1:])
    for t in range(T.shape[0]):
        Ae = Ae + S[0, t] * T[t]
    return np.ascontiguousarray(Ae)


def plane_ranges(root, R, P, min_rows_per_rank=16384):
    """Per level l (coarse -> fine) the [row_begin, row_end) of every rank."""
    gf = grid(root, R)
    npl = gf[2] + 1
    K = [(r * npl) // P for r in range(P)] + [npl]
    out = []
    for l in range(R + 1):
        g = grid(root, l)
        n = n_nodes(g)
        pl = (g[0] + 1) * (g[1] + 1)
        if P == 1 or l == 0 or n // P < min_rows_per_rank:
            out.append([(0, n)] * P)
            continue
        s = 1 << (R - l)
        ks = [-(-K[r] // s) for r in range(P)] + [g[2] + 1]
        out.append([(ks[r] * pl, ks[r + 1] * pl) for r in range(P)])
    return out


def _rows(g, bs, Ae, r0, r1, b):
    L = lib()
    rp = np.zeros(r1 - r0 + 1, np.int64)
    L.asm_structured(g[0], g[1], g[2], bs, ptr(Ae), ptr(BMASK), LID_COMP, r0, r1, 0, ptr(rp), None, None, None)
    nnzb = int(rp[-1])
    col = np.empty(nnzb, np.int64)
    val = np.empty((nnzb, bs, bs))
    L.asm_structured(g[0], g[1], g[2], bs, ptr(Ae), ptr(BMASK), LID_COMP, r0, r1, 1, ptr(rp), ptr(col), ptr(val),
                     ptr(b) if b is not None else None)
    return rp, col, val


def _transfer(gf, bs, r0, r1):
    L = lib()
    rp = np.zeros(r1 - r0 + 1, np.int64)
    L.tr_structured(gf[0], gf[1], gf[2], bs, ptr(BMASK), r0, r1, 0, ptr(rp), None, None)
    nnz = int(rp[-1])
    col = np.empty(nnz, np.int64)
    w = np.empty(nnz * bs)
    L.tr_structured(gf[0], gf[1], gf[2], bs, ptr(BMASK), r0, r1, 1, ptr(rp), ptr(col), ptr(w))
    return rp, col, w


def raw_rhs(g, bs, r0, r1, seed_index=SEED_INDEX):
    """Standard normal right-hand side of rows [r0, r1), drawn per z-plane."""
    pl = (g[0] + 1) * (g[1] + 1)
    k0, k1 = r0 // pl, -(-r1 // pl)
    out = np.empty(((k1 - k0) * pl, bs))
    for k in range(k0, k1):
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED_BASE + seed_index, k])))
        out[(k - k0) * pl:(k - k0 + 1) * pl] = rng.standard_normal((pl, bs))
    return np.ascontiguousarray(out[r0 - k0 * pl:r1 - k0 * pl])


def build_rank(P=1, rank=0, *, root=None, R=None, min_rows_per_rank=16384, raw_b=None, seed_index=SEED_INDEX):
    """This rank's levels (coarse -> fine, RankLevel) and its rows of the fine
    right-hand side.  root/R default to the weak-scaling size of P.
    raw_b: optional (n_fine_rows_of_rank, bs) raw rhs replacing the seeded one."""
    if root is None:
        root, R = C5_WEAK[P]
    op = F.Operator("stokes", 4, False, STOKES3)
    bs = op.bs
    ranges = plane_ranges(root, R, P, min_rows_per_rank)
    levels = []
    b = None
    for l in range(R + 1):
        g = grid(root, l)
        n = n_nodes(g)
        r0, r1 = ranges[l][rank]
        Ae = element_matrix(op, g)
        bl = None
        if l == R:
            bl = raw_rhs(g, bs, r0, r1, seed_index) if raw_b is None else np.array(raw_b, np.float64).reshape(-1, bs)
        rp, col, val = _rows(g, bs, Ae, r0, r1, bl)
        lv = RankLevel(r1 - r0, bs, rp, col, val, n, r0, r1, nx=g[0], ny=g[1], nz=g[2])
        if l > 0:
            lv.P = _transfer(g, bs, r0, r1)
            lv.wpe = bs
        levels.append(lv)
        if l == R:
            b = bl.reshape(-1)
    return levels, b, ranges


def n_dof(P=1, root=None, R=None):
    if root is None:
        root, R = C5_WEAK[P]
    return n_nodes(grid(root, R)) * 4
