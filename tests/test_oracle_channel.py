"""Pins of config C4 as SURVEY §8(d) states it -- 2D instationary Navier-Stokes
flow around a cylinder, equal-order Q1 stabilised, 3x3 blocks, Newton + GMRES
with the MG preconditioner per time step (problems/channel.py, oracle/newton.py).

What pins it (no paper numbers exist for this configuration, BASELINE config 4):
  * the Jacobian is the exact derivative of the residual: F is quadratic in w,
    so central differences reproduce J v up to rounding, at every step size;
  * closed forms of the Galerkin convection integral c(w; u, phi) =
    int (w . grad u) phi: rows annihilate constants (sum_j grad phi_j = 0), and
    for a constant field w the operator is skew-symmetric away from the
    boundary (c(w; u, v) + c(w; v, u) = int_dOmega (w.n) u v);
  * Newton converges quadratically with exact (sparse direct) linear solves;
  * GMRES + V(2,2) iteration counts stay bounded from the small to the mid
    mesh over several time steps (h-independent preconditioner);
  * mesh invariants: 2:1 balance, Dirichlet disk nodes on every level, root
    mesh 45 x 9 nodes as level 0."""
import functools

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spl

from oracle import newton as ON
from problems import channel as C
from problems import mesh as M


@functools.lru_cache(maxsize=None)
def prob(name):
    return C.build(name)


def perturbed_state(P, scale=0.3, seed=0):
    rng = np.random.default_rng(seed)
    u = C.initial_state(P)
    w = u + scale * rng.standard_normal(u.shape) * (~P.fine.cmask)
    return u, C.full_field(P, w)


def bsr(d, val):
    return sp.bsr_matrix((val, d.col, d.row_ptr), shape=(d.n * 3, d.n * 3)).tocsr()


@pytest.mark.parametrize("name", ["c4ns_small", "c4ns_mid"])
def test_jacobian_is_exact_derivative(name):
    P = prob(name)
    u, w = perturbed_state(P)
    J = bsr(P.fine, C.jacobians(P, w, u)[-1])
    rng = np.random.default_rng(1)
    v = rng.standard_normal(w.shape) * (~P.fine.cmask)
    Jv = J @ v.reshape(-1)
    for eps in (1e-2, 1e-4):
        fd = (C.residual(P, C.full_field(P, w + eps * v), u) - C.residual(P, C.full_field(P, w - eps * v), u)) / (2 * eps)
        assert np.linalg.norm(fd - Jv) <= 1e-9 * np.linalg.norm(fd)
    # dropping the Newton term (Picard) must fail the same check
    Jp = bsr(P.fine, C.jacobians(P, w, u, newton=False)[-1])
    assert np.linalg.norm(fd - Jp @ v.reshape(-1)) > 1e-3 * np.linalg.norm(fd)


def _raw_convection(P, CL, wfield):
    """Galerkin convection alone, condensed, no constraints: A(w) - A(0) with sd off."""
    sd = P.sd
    P.sd = 0.0
    try:
        T1, S1 = C._field_terms(P, CL, wfield, newton=False)
        T0, S0 = C._field_terms(P, CL, np.zeros_like(wfield), newton=False)
    finally:
        P.sd = sd
    return bsr(CL.data, C._assemble(CL, T1, S1)) - bsr(CL.data, C._assemble(CL, T0, S0))


def test_convection_closed_forms():
    P = prob("c4ns_mid")
    CL = P.levels[-1]
    n = CL.data.n
    Cw = _raw_convection(P, CL, np.tile([0.7, -0.3], (n, 1)))
    # velocity rows only, no pressure coupling from convection
    assert abs(Cw[0::3, :]).max() == 0.0 and abs(Cw[:, 0::3]).max() == 0.0
    # c(w; 1, phi_i) = 0 for each velocity component
    for c in (1, 2):
        one = np.zeros((n, 3))
        one[:, c] = 1.0
        assert np.abs(Cw @ one.reshape(-1)).max() <= 1e-15 * abs(Cw).max() * 10
    # constant w: skew-symmetric on nodes off the rectangle's boundary (regular nodes)
    coords = CL.nodes.coords
    mx = np.array([C.ROOT[a] << P.meta["R"] for a in range(2)])
    inner = ~np.any((coords == 0) | (coords == mx[None, :]), axis=1) & ~CL.nodes.hanging
    sel = np.repeat(inner, 3)
    Ci = Cw[sel][:, sel]
    assert abs(Ci + Ci.T).max() <= 1e-14 * abs(Ci).max()
    assert abs(Ci).max() > 0
    # ... and not symmetric part-free on the boundary (the (w.n) u v term)
    assert abs(Cw + Cw.T).max() > 1e-6 * abs(Cw).max()


def test_newton_quadratic_with_exact_solves():
    P = prob("c4ns_small")
    u_old = C.initial_state(P)
    w = u_old.copy()
    norms = []
    for k in range(7):
        F = C.residual(P, w, u_old)
        norms.append(np.linalg.norm(F))
        if norms[-1] <= 1e-12 * norms[0]:
            break
        J = bsr(P.fine, C.jacobians(P, w, u_old)[-1])
        d = spl.spsolve(J.tocsc(), -F)
        w = C.full_field(P, (w.reshape(-1) + d).reshape(-1, 3))
    assert norms[-1] <= 1e-12 * norms[0]
    # quadratic: ||F_{k+1}|| <= K ||F_k||^2 with a bounded K once in the basin
    ratios = [norms[k + 1] / norms[k] ** 2 for k in range(1, len(norms) - 1) if norms[k + 1] > 1e-12 * norms[0]]
    assert ratios and max(ratios) < 50.0, (norms, ratios)


def test_gmres_mg_counts_bounded_over_time_steps():
    its = {}
    for name in ("c4ns_small", "c4ns_mid"):
        P = prob(name)
        u = C.initial_state(P)
        counts = []
        for _ in range(3):
            u_old = u.copy()
            u, hist = ON.newton_step(lambda v: C.with_values(P, v), lambda w: C.residual(P, w, u_old),
                                     lambda w: C.jacobians(P, w, u_old), P.fine.H, u, omega=P.omega, max_newton=4)
            assert hist[-1][0] <= 1e-8 * hist[0][0], hist
            counts += [k for _, k in hist[:-1]]
        its[name] = counts
    assert max(its["c4ns_small"]) <= 25 and max(its["c4ns_mid"]) <= 25, its
    assert abs(max(its["c4ns_mid"]) - max(its["c4ns_small"])) <= 6, its


def test_mesh_invariants():
    P = prob("c4ns_mid")
    fine_mesh = C.channel_mesh(*C.CHANNEL_CONFIGS["c4ns_mid"][:3])
    assert M.balance_violations(fine_mesh).size == 0 or not M.balance_violations(fine_mesh).any()
    assert P.levels[0].data.n == (C.ROOT[0] + 1) * (C.ROOT[1] + 1)
    R = P.meta["R"]
    scale = np.array([C.BOX[a] / (C.ROOT[a] << R) for a in range(2)])
    for CL in P.levels:
        xyz = CL.nodes.coords * scale[None, :]
        disk = np.hypot(xyz[:, 0] - C.CYL[0], xyz[:, 1] - C.CYL[1]) <= C.CYL[2]
        assert disk.any() and CL.data.cmask[disk, 1:].all()
        outflow = CL.nodes.coords[:, 0] == (C.ROOT[0] << R)
        inner_out = outflow & (CL.nodes.coords[:, 1] > 0) & (CL.nodes.coords[:, 1] < (C.ROOT[1] << R))
        assert not CL.data.cmask[inner_out & ~CL.nodes.hanging, 1:].any()   # do-nothing outflow
        inside = np.hypot(xyz[:, 0] - C.CYL[0], xyz[:, 1] - C.CYL[1]) < C.CYL[2]
        assert np.array_equal(CL.data.cmask[:, 0], CL.nodes.hanging | inside)   # pressure free in the fluid
    # inflow profile: parabola with maximum U_m at mid-height
    g = P.g
    inflow = P.xyz[:, 0] == 0.0
    assert np.isclose(g[inflow, 1].max(), C.U_MAX * (1 - (2 * np.min(np.abs(P.xyz[inflow, 1] - C.BOX[1] / 2)) / C.BOX[1]) ** 2))


def test_elementwise_field_vector_equals_assembled_operator():
    """The residual's element-wise vector H^T [c(w; w, .) + sd(u_old; w, .)] equals
    the assembled convection + streamline-diffusion terms (condensed) times w."""
    P = prob("c4ns_mid")
    u_old, _ = perturbed_state(P, seed=4)
    _, w = perturbed_state(P, seed=3)
    CL = P.levels[-1]
    T1, S1 = C._field_terms(P, CL, w[:, 1:], newton=False, lag_nodes=u_old[:, 1:], static=False)
    A1 = bsr(CL.data, C._assemble(CL, T1, S1))
    got = C._field_vector(P, w, u_old).reshape(-1)
    exp = A1 @ w.reshape(-1)
    assert np.abs(got - exp).max() <= 1e-13 * np.abs(exp).max()


def test_inexact_newton_reaches_the_same_solution():
    """Jacobian reuse changes the path, not the fixed point F(w) = 0:
    with reuse_rate 0.3 at least one Jacobian is kept, more Newton steps are
    taken, and both iterations end at the same w."""
    P = prob("c4ns_small")
    u = C.initial_state(P)
    built = []

    def jac(w):
        built.append(1)
        return C.jacobians(P, w, u)
    run = lambda r: ON.newton_step(lambda v: C.with_values(P, v), lambda w: C.residual(P, w, u), jac,  # noqa: E731
                                   P.fine.H, u, omega=P.omega, max_newton=12, reuse_rate=r, ntol=1e-10)
    w0, h0 = run(0.0)
    n0 = len(built)
    w1, h1 = run(0.3)
    n1 = len(built) - n0
    assert h0[-1][0] <= 1e-10 * h0[0][0] and h1[-1][0] <= 1e-10 * h1[0][0]
    assert n1 < len(h1) - 1 and len(h1) >= len(h0)
    assert np.linalg.norm(w1 - w0) <= 1e-8 * np.linalg.norm(w0)
