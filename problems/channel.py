"""Config C4 as SURVEY §8(d) states it: 2D instationary Navier-Stokes flow around a
cylinder, equal-order Q1 stabilised, 3x3 blocks (p, u, v), backward Euler with
Newton's method per time step and the Jacobian of every level re-uploaded
value-only before each GMRES+MG solve (the paper's hybrid: assembly on the CPU,
the linear solver on the GPU).

SEEDED INPUT GENERATOR (test/bench infrastructure; no solve arithmetic): meshes,
the CPU assembly of the nonlinear residual F(w) and of the Newton Jacobian
J(w) on every level.  The Newton iteration itself (solve J d = -F, w += d) is
the caller's: paper_2405_05047_b200.newton (GPU) and oracle.newton (CPU).

Geometry (DFG benchmark 2D-2, not in the paper): channel
(0, 2.2) x (0, 0.41), cylinder of radius 0.05 centred at (0.2, 0.2), root 44 x 8
box cells, u uniform refinements then band steps toward the circle (finest
leaves whose centre lies within 4 K h of the circle, h the finest cell width).
The obstacle is the Brinkman limit (reading Z28): velocity nodes in the closed
disk are Dirichlet u = 0 and pressure nodes strictly inside it are removed
(p = 0), so the mesh stays a conforming quadtree with hanging nodes.  Parabolic inflow u = 4 U_m y (H - y) / H^2, U_m = 1.5 (mean 1), no-slip
walls and disk, do-nothing outflow at x = 2.2, pressure free in the fluid.

Operator (reading Z23/Z28; unknowns (p, u_1, u_2) node-major):
  velocity row (i, c):  (w_c/dt, phi_i) + nu (grad w_c, grad phi_i)
                        + ((w . grad) w_c, phi_i) - (p, d_c phi_i)
  pressure row i:       (div w, phi_i) + sum_T delta_T (grad p, grad phi_i)_T
                        + eps (p, phi_i),  delta_T = (1/dt + nu/h_T^2)^-1,
with w the Q1 field; the convection integrals are exact for Q1 (2-point Gauss).
Residual F(w) = A(w) w - M u_old / dt (condensed, constrained rows 0); Newton
Jacobian J(w) = A(w) + N(w), N(w)[(i,c),(j,b)] = int phi_j d_b w_c phi_i.
Coarse levels are rediscretised with w injected (coarse nodes are fine nodes).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import fem as F
from . import mesh as M
from .configs import SEED_BASE, LevelData

BOX = (2.2, 0.41)
ROOT = (44, 8)
CYL = (0.2, 0.2, 0.05)
U_MAX = 1.5
NS2 = dict(nu=1e-3, dt=1e-2, eps=1e-2, alpha=1.0)


def circle_band_mark(mesh: M.Mesh, box, K: int) -> np.ndarray:
    """Finest leaves whose centre is within 4 K h of the circle (h = finest cell width in x)."""
    L = mesh.max_level
    h = np.array([box[a] / (mesh.root[a] << L) for a in range(2)])
    m = mesh.lev == L
    ctr = (mesh.ijk + 0.5) * h[None, :]
    d = np.abs(np.hypot(ctr[:, 0] - CYL[0], ctr[:, 1] - CYL[1]) - CYL[2])
    return m & (d < 4 * K * h[0])


def channel_mesh(uniform: int, band: int, K: int) -> M.Mesh:
    m = M.uniform(ROOT)
    for _ in range(uniform):
        m = M.refine(m, np.ones(m.n_cells, bool))
    for _ in range(band):
        m = M.refine(m, circle_band_mark(m, BOX, K))
    return m


def conv_tensor():
    """C3[a, k, i, j] = int_ref phi_k phi_i d_a phi_j on the unit square (2-point Gauss, exact)."""
    xq, wq = F.gauss2(2)
    phi, grad = F.q1_basis(2, xq)
    return np.einsum("q,qk,qi,qja->akij", wq, phi, phi, grad)


def _blk(A, r, c, bs=3, nloc=4):
    Tb = np.zeros((nloc, bs, nloc, bs))
    Tb[:, r, :, c] = A
    return Tb.reshape(nloc * bs, nloc * bs)


@dataclass
class ChannelLevel:
    data: LevelData
    conn: np.ndarray
    hsz: np.ndarray              # (n_e, 2) cell sizes
    T_static: np.ndarray
    S_static: np.ndarray
    T_mass: np.ndarray
    S_mass: np.ndarray
    inject: np.ndarray | None    # (n,) index of each node in the finest level
    mesh: M.Mesh = None
    nodes: M.NodeSet = None
    plan: tuple = None           # cached constraint plan of the level's pattern
    static_val: np.ndarray = None  # cached values of the w-independent Stokes part
    mass_val: np.ndarray = None    # finest level: cached velocity mass / dt


@dataclass
class ChannelProblem:
    name: str
    levels: list                 # ChannelLevel, coarse -> fine
    g: np.ndarray                # (n_fine, 3) Dirichlet data at the finest level (velocity comps)
    xyz: np.ndarray              # (n_fine, 2)
    nu: float
    dt: float
    omega: float = 0.8
    bs: int = 3
    meta: dict = field(default_factory=dict)
    T_conv: np.ndarray = None    # (8, 12, 12): terms (a, k) of the Picard convection
    T_newt: np.ndarray = None    # (16, 12, 12): terms (b, c, k) of the Newton term
    T_sd: np.ndarray = None      # (4, 12, 12): terms (a, b) of the streamline diffusion
    sd: float = 1.0              # streamline-diffusion factor alpha_sd (0: Galerkin convection)

    @property
    def fine(self) -> LevelData:
        return self.levels[-1].data

    @property
    def n_dof(self) -> int:
        return self.fine.n * 3

    @property
    def lev_data(self):
        return [L.data for L in self.levels]


def build_channel(name: str, uniform: int, band: int, K: int, *, omega=0.6, seed_index=7, params=NS2):
    """omega: block-Jacobi damping of the V-cycle on the Newton Jacobians (reading
    Z28): 0.8 stalls once the flow develops (34-150 GMRES iterations per Newton
    step on c4ns_mid), 0.6 gives 14-17 (tests/test_oracle_channel.py)."""
    fine_mesh = channel_mesh(uniform, band, K)
    meshes = M.hierarchy(fine_mesh)
    R = fine_mesh.max_level
    op = F.Operator("stokes", 3, False, params)
    C3 = conv_tensor()
    T_conv = np.stack([sum(_blk(C3[a, k], 1 + c, 1 + c) for c in range(2)) for a in range(2) for k in range(4)])
    # Newton term: row (i, 1+c), col (j, 1+b): sum_k w_{k,c} vol/h_b int phi_j phi_i d_b phi_k
    # C3[b][j, i, k] = int phi_j phi_i d_b phi_k; the block entry [i, j] is C3[b][j, i, k]
    T_newt = np.stack([_blk(np.transpose(C3[b], (1, 0, 2))[:, :, k], 1 + c, 1 + b)
                       for b in range(2) for c in range(2) for k in range(4)])
    Mref, G, _ = F.reference_tensors(2)
    T_sd = np.stack([sum(_blk(G[a, b], 1 + c, 1 + c) for c in range(2)) for a in range(2) for b in range(2)])
    T_mass = np.stack([sum(_blk(Mref, c, c) for c in range(1, 3))])
    levels = []
    prev = None
    scale = np.array([BOX[a] / (ROOT[a] << R) for a in range(2)])
    for lm in meshes:
        nodes = M.build_nodes(lm, R)
        H = F.hanging_matrix(nodes)
        n = len(nodes.keys)
        xyz = nodes.coords * scale[None, :]
        mx = np.array([ROOT[a] << R for a in range(2)])
        c = nodes.coords
        dirich = (c[:, 0] == 0) | (c[:, 1] == 0) | (c[:, 1] == mx[1]) | \
                 (np.hypot(xyz[:, 0] - CYL[0], xyz[:, 1] - CYL[1]) <= CYL[2])
        cmask = np.zeros((n, 3), bool)
        cmask[:, 0] = nodes.hanging
        # the obstacle is not part of the fluid: pressure nodes strictly inside the disk are
        # removed (identity rows, p = 0) -- left free they form a PSPG-only sub-problem the
        # rediscretised coarse levels misrepresent (GMRES 100+ its at 0.5M DOFs vs 23)
        cmask[:, 0] |= np.hypot(xyz[:, 0] - CYL[0], xyz[:, 1] - CYL[1]) < CYL[2]
        cmask[:, 1:] = (nodes.hanging | dirich)[:, None]
        hsz = F.cell_sizes(lm, BOX)
        T, S = F.element_terms(op, 2, hsz)
        vol = np.prod(hsz, axis=1)
        S_mass = (vol / params["dt"])[:, None]
        rp, col, _ = F.assemble_terms(lm, nodes, T_mass, S_mass, 3, True, H)
        lvl = LevelData(n, 3, rp, col, None, cmask, H, keys=nodes.keys)
        if prev is not None:
            prp, pcol, pw = F.prolongation(prev.mesh, prev.nodes, prev.data.H, ~prev.nodes.hanging,
                                           lm, nodes, ~nodes.hanging)
            rows = F.row_of(prp)
            wc = pw[:, None] * (~cmask[rows]) * (~prev.data.cmask[pcol])
            keep = np.any(wc != 0.0, axis=1)
            rp2 = np.zeros(n + 1, np.int64)
            np.add.at(rp2, rows[keep] + 1, 1)
            lvl.P = (np.cumsum(rp2), pcol[keep], np.ascontiguousarray(wc[keep]).reshape(-1))
            lvl.wpe = 3
        CL = ChannelLevel(lvl, np.ascontiguousarray(nodes.conn, np.int64), hsz, T, S, T_mass, S_mass, None,
                          mesh=lm, nodes=nodes)
        levels.append(CL)
        prev = CL
    fine = levels[-1]
    for CL in levels:
        found, idx = M.lookup(fine.nodes.keys, CL.nodes.keys)
        assert found.all()
        CL.inject = idx
    xyz = fine.nodes.coords * scale[None, :]
    g = np.zeros((fine.data.n, 3))
    inflow = fine.nodes.coords[:, 0] == 0
    y = xyz[:, 1]
    g[inflow, 1] = 4.0 * U_MAX * y[inflow] * (BOX[1] - y[inflow]) / BOX[1] ** 2
    g[fine.nodes.hanging] = 0.0
    g[:, 0] = 0.0
    P = ChannelProblem(name, levels, g, xyz, params["nu"], params["dt"], omega=omega,
                       meta={"uniform": uniform, "band": band, "K": K, "R": R, "seed": SEED_BASE + seed_index})
    P.T_conv, P.T_newt, P.T_sd = T_conv, T_newt, T_sd
    return P


# --------------------------------------------------------------------------
# CPU assembly of F(w) and J(w) (the paper's CPU side of the hybrid)
# --------------------------------------------------------------------------


def _field_terms(P: ChannelProblem, CL: ChannelLevel, w_nodes: np.ndarray, newton: bool, lag_nodes=None,
                 static: bool = True, convection: bool = True):
    """Element terms (T, S) of the level operator for the nodal velocity field
    w_nodes (n, 2): the static Stokes part (static), the Galerkin convection
    (convection), streamline diffusion with the lagged (previous time step)
    field lag_nodes -- linear in w, so J stays the exact derivative of F -- and
    the Newton term (newton)."""
    vol = np.prod(CL.hsz, axis=1)
    we = w_nodes[CL.conn]                     # (n_e, 4, 2)
    T, S = [], []
    if static:
        T.append(CL.T_static)
        S.append(CL.S_static)
    if convection:
        T.append(P.T_conv)
        S.append(np.concatenate([we[:, :, a] * (vol / CL.hsz[:, a])[:, None] for a in range(2)], axis=1))
    if P.sd > 0.0 and lag_nodes is not None:
        wb, delta = _sd_delta(P, CL, lag_nodes)
        Ss = np.stack([delta * wb[:, a] * wb[:, b] * vol / (CL.hsz[:, a] * CL.hsz[:, b])
                       for a in range(2) for b in range(2)], axis=1)
        T.append(P.T_sd)
        S.append(Ss)
    if newton:
        Sn = np.concatenate([we[:, :, c] * (vol / CL.hsz[:, b])[:, None] for b in range(2) for c in range(2)],
                            axis=1)
        T.append(P.T_newt)
        S.append(Sn)
    return np.concatenate(T), np.concatenate(S, axis=1)


def _assemble(CL: ChannelLevel, T, S):
    d = CL.data
    rp, col, val = F.assemble_terms(CL.mesh, CL.nodes, T, S, 3, False, d.H, row_ptr=d.row_ptr)
    return val


def _bsr_mv(d: LevelData, val, x):
    A = sp.bsr_matrix((val, d.col, d.row_ptr), shape=(d.n * 3, d.n * 3))
    return A @ x.reshape(-1)


def full_field(P: ChannelProblem, w: np.ndarray) -> np.ndarray:
    """Hanging values interpolated: (H w) of the finest level, (n, 3)."""
    rp, col, wt = P.fine.H
    rows = F.row_of(rp)
    out = np.zeros_like(w)
    np.add.at(out, rows, wt[:, None] * w[col])
    return out


def step_cache(P: ChannelProblem, u_old: np.ndarray) -> dict:
    """What stays fixed within one time step: the w-independent Stokes part of
    every level (assembled once per problem) and M u_old / dt on the finest level."""
    for CL in P.levels:
        if CL.static_val is None:
            CL.static_val = _assemble(CL, CL.T_static, CL.S_static)
            if CL is P.levels[-1]:
                CL.mass_val = _assemble(CL, CL.T_mass, CL.S_mass)
    CL = P.levels[-1]
    return {"Mu": _bsr_mv(CL.data, CL.mass_val, u_old), "u_old": u_old}


def _sd_delta(P: ChannelProblem, CL: ChannelLevel, lag_nodes: np.ndarray):
    wb = lag_nodes[CL.conn].mean(axis=1)      # (n_e, 2) element mean of the lagged field
    hT = CL.hsz.max(axis=1)
    return wb, P.sd / (1.0 / P.dt + np.hypot(wb[:, 0], wb[:, 1]) / hT + P.nu / hT ** 2)


def _field_vector(P: ChannelProblem, w: np.ndarray, u_old: np.ndarray) -> np.ndarray:
    """H^T [c(w; w, .) + sd(u_old; w, .)] on the finest level, element by element:
    ((w . grad) w_c, phi_i) and sum_T delta_T (wb . grad w_c, wb . grad phi_i)_T with
    the same integrals as the T_conv / T_sd terms."""
    CL = P.levels[-1]
    vol = np.prod(CL.hsz, axis=1)
    we = w[CL.conn][:, :, 1:]                                      # (n_e, 4, 2)
    ne = len(we)
    C3 = conv_tensor()                                             # [a, k, i, j]
    coef = we * (vol[:, None, None] / CL.hsz[:, None, :])          # w_{k,a} vol / h_a
    Me = (coef.transpose(0, 2, 1).reshape(ne, 8) @ C3.reshape(8, 16)).reshape(ne, 4, 4)
    if P.sd > 0.0:
        _, G, _ = F.reference_tensors(2)
        wb, delta = _sd_delta(P, CL, u_old[:, 1:])
        cs = np.stack([delta * wb[:, a] * wb[:, b] * vol / (CL.hsz[:, a] * CL.hsz[:, b])
                       for a in range(2) for b in range(2)], axis=1)
        Me = Me + (cs @ G.reshape(4, 16)).reshape(ne, 4, 4)
    loc = Me @ we                                                  # (n_e, 4, 2)
    n = CL.data.n
    full = np.stack([np.bincount(CL.conn.ravel(), loc[:, :, c].ravel(), minlength=n) for c in range(2)], 1)
    rp, col, wt = CL.data.H
    rows = F.row_of(rp)
    cond = np.stack([np.bincount(col, wt * full[rows, c], minlength=n) for c in range(2)], 1)
    out = np.zeros((n, 3))
    out[:, 1:] = cond
    return out


def residual(P: ChannelProblem, w: np.ndarray, u_old: np.ndarray, cache: dict | None = None) -> np.ndarray:
    """F(w) = A(w) w - M u_old/dt on the finest level (condensed), constrained rows 0:
    the cached Stokes part times w plus the element-wise convection and
    streamline-diffusion vector.
    w, u_old: (n, 3) full fields (hanging values interpolated, Dirichlet data imposed)."""
    cache = cache if cache is not None else step_cache(P, u_old)
    CL = P.levels[-1]
    Fv = _bsr_mv(CL.data, CL.static_val, w) + _field_vector(P, w, u_old).reshape(-1) - cache["Mu"]
    Fv = Fv.reshape(-1, 3)
    Fv[CL.data.cmask] = 0.0
    return Fv.reshape(-1)


def jacobians(P: ChannelProblem, w: np.ndarray, u_old: np.ndarray, newton: bool = True, cache: dict | None = None):
    """Per level (coarse -> fine) the BSR values (nnzb, 3, 3) of J(w_l) (Newton) or
    A(w_l) (Picard), w_l = w injected, constraints applied (identity rows and
    eliminated columns, homogeneous: the Newton correction vanishes there)."""
    cache = cache if cache is not None else step_cache(P, u_old)
    out = []
    for l, CL in enumerate(P.levels):
        T, S = _field_terms(P, CL, w[CL.inject, 1:], newton, lag_nodes=u_old[CL.inject, 1:], static=False)
        val = _assemble(CL, T, S) + CL.static_val
        if CL.plan is None:
            d = CL.data
            CL.plan = F.constraint_plan(d.row_ptr, d.col, d.cmask)
        F.apply_constraint_plan(val, CL.plan)
        out.append(val)
    return out


def initial_state(P: ChannelProblem) -> np.ndarray:
    """Impulsive start: u = 0 with the boundary data (hanging values interpolated), p = 0."""
    return full_field(P, P.g)


def assemble_callback(P: ChannelProblem, u_old: np.ndarray):
    """The CPU side of one time step for the library's Newton driver
    (include/newton.h): fills F(w) and every level's Jacobian values."""
    cache = step_cache(P, u_old)

    def asm(w, F, vals):
        W = np.asarray(w).reshape(-1, 3)
        if F is not None:
            F[:] = residual(P, W, u_old, cache)
        if vals is not None:
            for l, v in enumerate(jacobians(P, W, u_old, cache=cache)):
                vals[l][:] = v.reshape(-1)
    return asm


def with_values(P: ChannelProblem, vals) -> list:
    """LevelData list with the given per-level values (for building solvers / oracle hierarchies)."""
    out = []
    for CL, v in zip(P.levels, vals):
        d = CL.data
        out.append(LevelData(d.n, 3, d.row_ptr, d.col, v, d.cmask, d.H, P=d.P, wpe=d.wpe, keys=d.keys,
                             patches=CL.conn))
    return out


CHANNEL_CONFIGS = {
    # name: (uniform, band steps, K, seed index)
    "c4ns": (2, 6, 9, 7),          # 348,562 nodes = 1,045,686 DOFs
    "c4ns_small": (0, 2, 1, 7),
    "c4ns_mid": (1, 3, 2, 7),
}


def build(name: str, **kw) -> ChannelProblem:
    u, b, K, si = CHANNEL_CONFIGS[name]
    return build_channel(name, u, b, K, seed_index=si, **kw)
