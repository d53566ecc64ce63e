"""Named synthetic workloads (SURVEY §8(d) C1-C3 plus small test cases) and the
seeded problem builder:  mesh -> hierarchy -> per-level condensed BSR systems,
hanging matrices, transfers, right-hand sides.

SEEDED INPUT GENERATOR (test/bench infrastructure; no solve arithmetic).
Recipe: seeds numpy PCG64(240505047 + config index);
throughput right-hand sides are standard normal with constrained entries set
to their boundary value (0), x0 = 0.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import fem as F
from . import mesh as M

SEED_BASE = 240505047


@dataclass
class LevelData:
    n: int
    bs: int
    row_ptr: np.ndarray          # (n+1,) int64
    col: np.ndarray              # (nnzb,) int64
    val: np.ndarray              # (nnzb, bs, bs) float64
    cmask: np.ndarray            # (n, bs) bool  constrained (hanging or Dirichlet)
    H: tuple                     # (rp, col, w) hanging matrix, n x n
    P: tuple | None = None       # (rp, col, w) prolongation from level-1, n x n_{l-1}
    wpe: int = 1                 # weights per P entry (1 or bs)
    keys: np.ndarray | None = None  # (n,) sorted Morton keys at the finest lattice level (partitioning)
    mean_w: np.ndarray | None = None  # (n,) pure Neumann: lumped-mass weights H^T m of int p = 0
    mean_k: np.ndarray | None = None  # (n,) pure Neumann: kernel vector (1 free, 0 hanging)
    mesh: M.Mesh | None = None
    nodes: M.NodeSet | None = None
    patches: np.ndarray | None = None  # (n_cells, 2^d) node ids of each mesh cell (Vanka patches)

    @property
    def nnzb(self) -> int:
        return int(self.row_ptr[-1])


@dataclass
class Problem:
    name: str
    dim: int
    bs: int
    box: tuple
    op: F.Operator
    levels: list                 # coarse -> fine
    b: np.ndarray                # (n_fine*bs,) rhs on the finest level
    g: np.ndarray                # (n_fine, bs) Dirichlet values on the finest level
    omega: float = 0.8
    nu_pre: int = 2
    nu_post: int = 2
    meta: dict = field(default_factory=dict)

    @property
    def fine(self) -> LevelData:
        return self.levels[-1]

    @property
    def n_dof(self) -> int:
        return self.fine.n * self.bs


# --------------------------------------------------------------------------


def build_mesh(root, steps) -> M.Mesh:
    """steps: list of ("uniform",) or ("band", axes, K)."""
    m = M.uniform(root)
    for st in steps:
        if st[0] == "uniform":
            m = M.refine(m, np.ones(m.n_cells, bool))
        elif st[0] == "band":
            m = M.refine(m, M.band_mark(m, st[1], st[2]))
        else:
            raise ValueError(st)
    return m


def node_xyz(nodes: M.NodeSet, root, box) -> np.ndarray:
    h = np.array([box[a] / (root[a] * (1 << nodes.R)) for a in range(len(root))])
    return nodes.coords * h[None, :]


def load_vector(mesh: M.Mesh, nodes: M.NodeSet, box, f, bs: int) -> np.ndarray:
    """f_i = ∫ f φ_i by the 2-point Gauss rule on every leaf (unconstrained)."""
    dim = mesh.dim
    xq, wq = F.gauss2(dim)
    phi, _ = F.q1_basis(dim, xq)
    h = F.cell_sizes(mesh, box)
    x0 = mesh.ijk * h
    vol = np.prod(h, axis=1)
    out = np.zeros((len(nodes.keys), bs))
    for q in range(len(wq)):
        xp = x0 + xq[q][None, :] * h
        fv = np.asarray(f(xp)).reshape(len(xp), bs)
        for a in range(1 << dim):
            np.add.at(out, nodes.conn[:, a], (wq[q] * vol * phi[q, a])[:, None] * fv)
    return out


def apply_HT(H, v: np.ndarray) -> np.ndarray:
    """Condensation of a load vector: H^T v, hanging entries then zeroed
    by the caller via the constraint mask."""
    rp, col, w = H
    rows = F.row_of(rp)
    out = np.zeros_like(v)
    np.add.at(out, col, w[:, None] * v[rows])
    return out


def make_problem(name, root, box, steps, op: F.Operator, *, seed_index=0, omega=0.8,
                 nu=(2, 2), f=None, g_fun=None, keep_geometry=True, neumann=False) -> Problem:
    """neumann: no Dirichlet boundary (the pressure Poisson problem of the
    projection step); every level then carries the kernel vector
    and lumped-mass weights of the constraint int p = 0."""
    fine_mesh = build_mesh(root, steps)
    meshes = M.hierarchy(fine_mesh)
    R = fine_mesh.max_level
    bs = op.bs
    vel_only = op.name == "stokes"      # Dirichlet on velocity only (reading Z23)
    levels = []
    prev = None
    for lm in meshes:
        nodes = M.build_nodes(lm, R)
        H = F.hanging_matrix(nodes)
        n = len(nodes.keys)
        bnd = M.boundary_nodes(lm, nodes)
        cmask = np.repeat(((nodes.hanging | bnd) if not neumann else nodes.hanging)[:, None], bs, axis=1)
        if vel_only:
            cmask[:, 0] = nodes.hanging
        rp, col, val = F.assemble(lm, nodes, op, box, H)
        lvl = LevelData(n, bs, rp, col, val, cmask, H, keys=nodes.keys, mesh=lm if keep_geometry else None,
                        nodes=nodes if keep_geometry else None, patches=np.ascontiguousarray(nodes.conn, np.int64))
        if neumann:
            lvl.mean_k = (~nodes.hanging).astype(np.float64)
            m = apply_HT(H, load_vector(lm, nodes, box, lambda xp: np.ones(len(xp)), 1))[:, 0]
            lvl.mean_w = np.where(nodes.hanging, 0.0, m)
            bnd = np.zeros_like(bnd)
        lvl._bnd = bnd
        lvl._nodes = nodes
        lvl._mesh = lm
        if prev is not None and not vel_only:
            lvl.P = F.prolongation(prev._mesh, prev._nodes, prev.H, ~prev.cmask[:, 0],
                                   lm, nodes, ~cmask[:, 0])
        elif prev is not None:
            # per-component Pi: weights_per_entry = bs (pressure free at the boundary)
            prp, pcol, pw = F.prolongation(prev._mesh, prev._nodes, prev.H, ~prev._nodes.hanging,
                                           lm, nodes, ~nodes.hanging)
            rows = F.row_of(prp)
            wc = pw[:, None] * (~cmask[rows]) * (~prev.cmask[pcol])
            keep = np.any(wc != 0.0, axis=1)
            rp2 = np.zeros(n + 1, np.int64)
            np.add.at(rp2, rows[keep] + 1, 1)
            lvl.P = (np.cumsum(rp2), pcol[keep], np.ascontiguousarray(wc[keep]).reshape(-1))
            lvl.wpe = bs
        levels.append(lvl)
        prev = lvl
    # constraints on every level: identity rows at hanging/Dirichlet DOFs
    fine = levels[-1]
    xyz = node_xyz(fine._nodes, root, box)
    g = np.zeros((fine.n, bs))
    if g_fun is not None:
        g[fine._bnd] = np.asarray(g_fun(xyz[fine._bnd])).reshape(-1, bs)
    g[fine._nodes.hanging] = 0.0
    rng = np.random.Generator(np.random.PCG64(SEED_BASE + seed_index))
    if f is None:
        b = rng.standard_normal((fine.n, bs))
    else:
        b = apply_HT(fine.H, load_vector(fine._mesh, fine._nodes, box, f, bs))
    for lvl in levels:
        gl = g if lvl is fine else np.zeros((lvl.n, bs))
        F.apply_constraints(lvl.row_ptr, lvl.col, lvl.val, lvl.cmask, gl, b if lvl is fine else None)
        if not keep_geometry:
            lvl.mesh = None
            lvl.nodes = None
        for attr in ("_bnd", "_nodes", "_mesh"):
            if not keep_geometry:
                delattr(lvl, attr)
    if f is None:
        b[fine.cmask] = g[fine.cmask]
    return Problem(name, fine_mesh.dim, bs, tuple(box), op, levels, b.reshape(-1).copy(), g,
                   omega=omega, nu_pre=nu[0], nu_post=nu[1],
                   meta={"root": tuple(root), "steps": list(steps), "R": R, "seed": SEED_BASE + seed_index})


# --------------------------------------------------------------------------
# Named configs
# --------------------------------------------------------------------------

TD = dict(lam=0.01, b=(0.0, -1.0), dt=0.02)
STOKES2 = dict(nu=1e-3, dt=1e-2, eps=1e-2, alpha=1.0)          # reading Z23 (C4)
STOKES3 = dict(nu=1e-3, dt=1e-4, eps=1e-2, alpha=1.0)          # P:595, reading Z23 (C5)


def lid(dim, bs):
    """Cavity velocity Dirichlet data: u_1 = 1 on the moving lid x_{d-1} = 0
    (the face the band rule refines toward), 0 elsewhere; pressure free."""
    def g(xyz):
        out = np.zeros((len(xyz), bs))
        out[:, 1] = (xyz[:, dim - 1] == 0.0).astype(float)
        return out
    return g
ELAST = dict(lam=8e4, mu=2e4, dt=0.025)


def theta_ex(t, x, y):
    """Exact transport-diffusion solution."""
    m = lambda z: 0.5 + 0.25 * np.cos(0.5 * np.pi * t) - z  # noqa: E731
    return np.exp(-0.25 * (m(x) ** 2 + m(y) ** 2))


CONFIGS = {
    # name: (root, box, steps, operator, omega, seed index)
    "c1": ((4, 4), (1.0, 1.0), [("uniform",)] * 3, F.Operator("td", 1, False, TD), 0.8, 0),
    "c1_poisson": ((4, 4), (1.0, 1.0), [("uniform",)] * 3, F.Operator("poisson", 1, True), 0.8, 0),
    # the paper's transport-diffusion table: uniform Q1 meshes L7..L10 of the unit
    # square, (2^L + 1)^2 nodes; td_l10 = 1,050,625 DOFs (the "about 34x" case)
    "td_l7": ((4, 4), (1.0, 1.0), [("uniform",)] * 5, F.Operator("td", 1, False, TD), 0.8, 8),
    "td_l10": ((4, 4), (1.0, 1.0), [("uniform",)] * 8, F.Operator("td", 1, False, TD), 0.8, 8),
    "c2": ((32, 32), (1.0, 1.0), [("band", [1], 20)] * 7, F.Operator("td", 1, False, TD), 0.8, 1),
    "c3": ((9, 9, 9), (1.0, 1.0, 1.0), [("band", [0], 1)] * 6,
           F.Operator("elasticity", 3, True, ELAST), 0.5, 2),
    # small cases with the same structure (parity tests: several tiles + ragged tails)
    "c2_small": ((8, 8), (1.0, 1.0), [("band", [1], 2)] * 3, F.Operator("td", 1, False, TD), 0.8, 1),
    "c3_small": ((4, 4, 4), (1.0, 1.0, 1.0), [("band", [0], 1)] * 2,
                 F.Operator("elasticity", 3, True, ELAST), 0.5, 2),
    "c3_mid": ((6, 6, 6), (1.0, 1.0, 1.0), [("band", [0], 1)] * 3,
               F.Operator("elasticity", 3, True, ELAST), 0.5, 2),
    "face_poisson": ((8, 8, 8), (1.0, 1.0, 1.0), [("band", [0], 1)] * 2, F.Operator("poisson", 1, True), 0.8, 3),
}


CONFIGS.update({
    # N4: the paper's 6-component (u, v) elasticity system on Table `ndofs` face meshes (8^3 root,
    # K = 1 band toward x = 0): L2 = 2,925 nodes = 17,550 DOFs ... L5 = 172,505 nodes = 1,035,030 DOFs
    #
    "e6_face_l2": ((8, 8, 8), (1.0, 1.0, 1.0), [("band", [0], 1)] * 1,
                   F.Operator("elasticity6", 6, False, ELAST), 0.5, 5),
    "e6_face_l3": ((8, 8, 8), (1.0, 1.0, 1.0), [("band", [0], 1)] * 2,
                   F.Operator("elasticity6", 6, False, ELAST), 0.5, 5),
    "e6_face_l5": ((8, 8, 8), (1.0, 1.0, 1.0), [("band", [0], 1)] * 4,
                   F.Operator("elasticity6", 6, False, ELAST), 0.5, 5),
    # Table `ndofs` edge and vertex patterns, L6: band toward the edge x = y = 0 /
    # the vertex 0 (reading Z16): 34,985 / 3,749 nodes = 209,910 / 22,494 DOFs
    "e6_edge_l6": ((8, 8, 8), (1.0, 1.0, 1.0), [("band", [0, 1], 1)] * 5,
                   F.Operator("elasticity6", 6, False, ELAST), 0.5, 5),
    "e6_vertex_l6": ((8, 8, 8), (1.0, 1.0, 1.0), [("band", [0, 1, 2], 1)] * 5,
                     F.Operator("elasticity6", 6, False, ELAST), 0.5, 5),
    # C4: 2D NS-shaped generalised Stokes, 3x3 blocks (p, u, v), lid cavity, band toward the lid
    "c4": ((32, 32), (1.0, 1.0), [("band", [1], 20)] * 6, F.Operator("stokes", 3, False, STOKES2), 0.8, 3),
    "c4_small": ((8, 8), (1.0, 1.0), [("band", [1], 2)] * 3, F.Operator("stokes", 3, False, STOKES2), 0.8, 3),
    # C5: 3D NS-shaped, 4x4 blocks (p, u, v, w) on (0,1)x(0,1)x(0,2), root (4,4,8), uniform refinement
    # omega: 0.8 diverges on the adaptive 3D case (rho ~ 1.2); 0.6 gives h-independent
    # GMRES counts (25-27 at 1.4k..70.8k nodes), tests/test_oracle_stokes.py
    "c5": ((4, 4, 8), (1.0, 1.0, 2.0), [("uniform",)] * 5, F.Operator("stokes", 4, False, STOKES3), 0.6, 4),
    "c5_small": ((2, 2, 4), (1.0, 1.0, 2.0), [("uniform",)] * 2, F.Operator("stokes", 4, False, STOKES3), 0.6, 4),
    "c5_mid": ((2, 2, 4), (1.0, 1.0, 2.0), [("band", [2], 1)] * 2 + [("uniform",)],
               F.Operator("stokes", 4, False, STOKES3), 0.6, 4),
})

# Pure-Neumann pressure Poisson of the projection step (Alg. 2 Step 2, P:618-636;
# Table `ns` pres-solve) on the NS cavity domain (0,1)x(0,1)x(0,2), root
# (4,4,8): "pres" = 3 uniform steps = 70,785 nodes (the paper's 32x32x64 mesh,
# P:706), "pres_l5" = 5 steps = 4,293,249 nodes (bench size), "pres_mid" adds
# hanging nodes (band refinement), "pres_small" for parity.
NEUMANN = {"pres", "pres_small", "pres_mid", "pres_l5"}
CONFIGS.update({
    "pres": ((4, 4, 8), (1.0, 1.0, 2.0), [("uniform",)] * 3, F.Operator("poisson", 1, True), 0.8, 6),
    "pres_l5": ((4, 4, 8), (1.0, 1.0, 2.0), [("uniform",)] * 5, F.Operator("poisson", 1, True), 0.8, 6),
    "pres_small": ((2, 2, 4), (1.0, 1.0, 2.0), [("uniform",)] * 2, F.Operator("poisson", 1, True), 0.8, 6),
    "pres_mid": ((2, 2, 4), (1.0, 1.0, 2.0), [("band", [2], 1)] * 2 + [("uniform",)],
                 F.Operator("poisson", 1, True), 0.8, 6),
})


def build(name: str, **kw) -> Problem:
    root, box, steps, op, omega, si = CONFIGS[name]
    if op.name == "stokes" and "g_fun" not in kw:
        kw["g_fun"] = lid(len(root), op.bs)
    if name in NEUMANN:
        kw.setdefault("neumann", True)
    return make_problem(name, root, box, steps, op, seed_index=si, omega=omega, **kw)
