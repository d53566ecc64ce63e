"""GPU parity of the explicit pressure-correction NS step (Alg. 2, P:618-636;
SURVEY N2) through include/ns.h against oracle/ns.py on the same seeded
inputs: Step 1 (the fused momentum kernel: node-wise products, C_d products,
viscous term, pressure gradient via C_c Pi, lumped-mass inverse, Dirichlet
values), Step 2 (divergence G^T u and the pure-Neumann pressure solve) and
Step 3 (pressure update with int p = 0), single steps and a short run from
rest, plus the paper's full-size cavity (70,785 / 545,025 nodes).

Tolerances (reading Z11): per-op 1e-12 scaled by the magnitude of the terms
(|u| + dt/m (nu|K||u| + sum_d |C_d||v^d| + |G||p + q|)); pressure solves at
rtol 1e-10 agree to 1e-8 relative with iteration counts +-1."""
import functools

import numpy as np
import pytest

from gpu_util import TOL_OP

import oracle
from oracle import ns as ons
from problems import ns

pytestmark = pytest.mark.gpu


@functools.lru_cache(maxsize=None)
def prob(name):
    return ns.build_ns(name)


def ops_of(P):
    return ons.NsOperators.from_arrays(P.n_u, P.n_p, P.mom_rp, P.mom_col, P.mom_val, P.G, P.m_u, P.m_p,
                                       P.dir_rows, P.dir_vals, P.nu, P.dt)


def abs_ops(P):
    return ons.NsOperators.from_arrays(P.n_u, P.n_p, P.mom_rp, P.mom_col, np.abs(P.mom_val),
                                       (P.G[0], P.G[1], np.abs(P.G[2])), P.m_u, P.m_p, P.dir_rows,
                                       np.abs(P.dir_vals), P.nu, P.dt)


def momentum_scale(P, u, p, q):
    """Per-entry magnitude of the Step-1 computation."""
    A = abs_ops(P)
    au = np.abs(u)
    visc = np.stack([A.K @ au[:, c] for c in range(3)], 1)
    conv = ons.convection(A, au)
    grad = ons.gradient(A, np.abs(p) + np.abs(q))
    return au + P.dt / P.m_u[:, None] * (P.nu * visc + conv + grad)


def pres_h(P):
    return oracle.MgHierarchy.from_arrays(P.pres_levels, omega=P.omega,
                                          mean=[(L.mean_w, L.mean_k) for L in P.pres_levels])


def gpu_ns(P, **kw):
    from paper_2405_05047_b200 import NavierStokes
    return NavierStokes(P, **kw)


@pytest.mark.parametrize("name", ["ns_small", "ns_mid"])
def test_momentum_matches_oracle(name):
    P = prob(name)
    g = gpu_ns(P)
    u, p, q = ns.random_state(P)
    g.set_state(u, p, q)
    got = g.momentum()
    exp = ons.momentum(ops_of(P), u, p, q)
    sc = momentum_scale(P, u, p, q)
    err = np.abs(got - exp)
    assert np.max(err) <= TOL_OP * np.max(sc), np.max(err) / np.max(sc)
    assert np.array_equal(got[P.dir_rows], P.dir_vals)
    # the state is not advanced by ns_momentum
    u2, p2, q2 = g.get_state()
    assert np.array_equal(u2, u) and np.array_equal(p2, p) and np.array_equal(q2, q)
    g.close()


@pytest.mark.parametrize("name", ["ns_small", "ns_mid"])
def test_step_matches_oracle(name):
    P = prob(name)
    ops = ops_of(P)
    g = gpu_ns(P, rtol=1e-10)
    u, p, q = ns.random_state(P, scale=0.5)
    g.set_state(u, p, q)
    st, its, rel, conv, ms = g.step()
    un, pn, qn = g.get_state()
    d = g.divergence()
    # Step 1
    exp_u = ons.momentum(ops, u, p, q)
    assert np.max(np.abs(un - exp_u)) <= TOL_OP * np.max(momentum_scale(P, u, p, q))
    # Step 2: divergence of the GPU's u^m, then the pressure solve
    exp_d = ons.divergence(ops, un)
    A = abs_ops(P)
    dsc = sum(A.G[c].T @ np.abs(un[:, c]) for c in range(3))
    assert np.max(np.abs(d - exp_d)) <= TOL_OP * np.max(dsc)
    h = pres_h(P)
    qe, ite, _, _ = oracle.gmres(h, ons.pressure_rhs(ops, d), rtol=1e-10)
    assert conv and abs(its - ite) <= 1, (its, ite)
    assert np.linalg.norm(qn - qe) <= 1e-8 * np.linalg.norm(qe)
    # Step 3 from the GPU's q and d
    exp_p = ons.pressure_update(ops, p, qn, d)
    psc = np.abs(p) + np.abs(qn) + P.nu * np.abs(d) / P.m_p
    assert np.max(np.abs(pn - exp_p)) <= TOL_OP * np.max(psc)
    for v in (pn, qn):
        assert abs(P.m_p @ v) <= 1e-13 * np.abs(P.m_p * v).sum()
    g.close()


def test_run_from_rest_matches_oracle():
    """20 steps of the driven cavity from rest: GPU and oracle fields
    agree to the solver tolerance; the lid drives a flow (kinetic energy > 0)."""
    P = prob("ns_mid")
    ops = ops_of(P)
    h = pres_h(P)
    g = gpu_ns(P, rtol=1e-10)
    u, p, q = ns.initial_state(P)
    g.set_state(u, p, q)
    for k in range(20):
        st, its, rel, conv, ms = g.step()
        assert conv
        u, p, q, d, ite = ons.step(ops, h, u, p, q, rtol=1e-10)
    ug, pg, qg = g.get_state()
    assert np.linalg.norm(ug - u) <= 1e-9 * np.linalg.norm(u)
    assert np.linalg.norm(pg - p) <= 1e-7 * np.linalg.norm(p)
    ke = 0.5 * np.sum(P.m_u[:, None] * ug ** 2)
    assert ke > 0.0 and np.all(np.isfinite(ug))
    g.close()


def test_errors():
    import paper_2405_05047_b200 as m
    P = prob("ns_small")
    g = gpu_ns(P)
    with pytest.raises(m.MgError) as e:
        g.step()                                        # no state yet
    assert e.value.status == m.MG_ERR_STATE
    with pytest.raises(m.MgError) as e:
        g.divergence()
    assert e.value.status == m.MG_ERR_STATE
    with pytest.raises(m.MgError) as e:
        m.ns_set_mass(g.ctx, -P.m_u, P.m_p)
    assert e.value.status == m.MG_ERR_INVALID_ARG
    rows = P.dir_rows[::-1].copy()
    with pytest.raises(m.MgError) as e:
        m.ns_set_dirichlet(g.ctx, rows, P.dir_vals.reshape(-1))
    assert e.value.status == m.MG_ERR_INVALID_ARG
    with pytest.raises(m.MgError) as e:
        m.ns_create(g.pressure.ctx, P.n_u, P.n_p + 1)
    assert e.value.status == m.MG_ERR_DIMENSION
    g.close()


@pytest.mark.slow
def test_paper_cavity_full_size_step():
    """The paper's mesh (32 x 32 x 64 pressure cells): one step from a
    random state, Step 1 on every row and the pressure solve at rtol 1e-6
    (GMRES(30) + V(2,2), omega = 0.4, reading Z27) against the oracle."""
    P = prob("ns")
    ops = ops_of(P)
    g = gpu_ns(P, rtol=1e-6)
    u, p, q = ns.random_state(P, scale=0.5)
    g.set_state(u, p, q)
    st, its, rel, conv, ms = g.step()
    un, pn, qn = g.get_state()
    exp_u = ons.momentum(ops, u, p, q)
    assert np.max(np.abs(un - exp_u)) <= TOL_OP * np.max(momentum_scale(P, u, p, q))
    d = g.divergence()
    qe, ite, _, rele = oracle.gmres(pres_h(P), ons.pressure_rhs(ops, d), rtol=1e-6)
    assert conv and abs(its - ite) <= 1, (its, ite)
    assert np.linalg.norm(qn - qe) <= 1e-5 * np.linalg.norm(qe)
    g.close()


@pytest.mark.parametrize("name", ["ns_mid", "ns"])
def test_step_with_vanka_pressure_smoother(name):
    """The pressure MG with the Vanka-type cell-patch smoother (mg_set_vanka,
    P:822; omega = 0.8): same step as the oracle with the same smoother, far
    fewer GMRES iterations than point Jacobi on the graded (anisotropic) mesh."""
    P = prob(name)
    ops = ops_of(P)
    g = gpu_ns(P, rtol=1e-6, vanka=True, omega=0.8)
    u, p, q = ns.random_state(P, scale=0.5)
    g.set_state(u, p, q)
    st, its, rel, conv, ms = g.step()
    _, _, qn = g.get_state()
    d = g.divergence()
    h = oracle.MgHierarchy.from_arrays(P.pres_levels, omega=0.8, mean=[(L.mean_w, L.mean_k) for L in P.pres_levels],
                                       vanka=True)
    qe, ite, _, rele = oracle.gmres(h, ons.pressure_rhs(ops, d), rtol=1e-6)
    assert conv and abs(its - ite) <= 1, (its, ite)
    assert np.linalg.norm(qn - qe) <= 1e-5 * np.linalg.norm(qe)
    _, ite_j, _, _ = oracle.gmres(pres_h(P), ons.pressure_rhs(ops, d), rtol=1e-6)
    assert ite < ite_j, (ite, ite_j)
    g.close()
