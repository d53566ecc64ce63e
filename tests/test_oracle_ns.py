"""Pins of the NS generator (problems/ns.py) and of the oracle's explicit
pressure-correction step (oracle/ns.py; Alg. 2) against
closed forms and identities of the mathematics: exact 1D element integrals,
partition of unity, the divergence theorem, exact reproduction of linear
fields by Q1, the nesting identity G_c = C_c Pi of the Q1-iso-Q2 pair, the
SPEC's worked examples and a bordered dense solve."""
import functools

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from oracle import ns as ons
from problems import ns


@functools.lru_cache(maxsize=None)
def prob(name):
    return ns.build_ns(name)


def ops_of(P, nu=None):
    return ons.NsOperators.from_arrays(P.n_u, P.n_p, P.mom_rp, P.mom_col, P.mom_val, P.G, P.m_u, P.m_p,
                                       P.dir_rows, P.dir_vals, P.nu if nu is None else nu, P.dt)


def grid(xs):
    """Node coordinates (n, 3), x fastest."""
    X, Y, Z = np.meshgrid(*xs, indexing="ij")
    return np.stack([X.transpose(2, 1, 0).ravel(), Y.transpose(2, 1, 0).ravel(), Z.transpose(2, 1, 0).ravel()], 1)


def interior(xs):
    xyz = grid(xs)
    lo = np.array([x[0] for x in xs])
    hi = np.array([x[-1] for x in xs])
    return np.all((xyz > lo) & (xyz < hi), axis=1)


def test_1d_element_integrals():
    h = 0.3
    M, K, D = (A.toarray() for A in ns.fe1d(np.array([0.0, h])))
    assert np.allclose(M, [[h / 3, h / 6], [h / 6, h / 3]], rtol=1e-15, atol=0)
    assert np.allclose(K, [[1 / h, -1 / h], [-1 / h, 1 / h]], rtol=1e-15, atol=0)
    assert np.allclose(D, [[-0.5, -0.5], [0.5, 0.5]], rtol=1e-15, atol=1e-16)


def test_graded_mesh_and_counts():
    x = ns.graded(32, "x")
    z = ns.graded(64, "z")
    assert x[0] == 0.0 and abs(x[-1] - 1.0) < 1e-15 and np.all(np.diff(x) > 0)
    assert np.allclose(x + x[::-1], 1.0, atol=1e-15)                 # cos grading symmetric
    assert abs(z[0]) < 1e-15 and abs(z[-1] - 2.0) < 1e-15 and np.all(np.diff(z) > 0)   # reading Z26
    P = ns.make_ns("t", (2, 2, 2))
    assert (P.n_u, P.n_p) == (125, 27)
    Pp = prob("ns")
    assert (Pp.n_u, Pp.n_p) == (545025, 70785)                       # (32, 32, 64) cells


@pytest.mark.parametrize("name", ["ns_small", "ns_mid"])
def test_operator_identities(name):
    P = prob(name)
    ops = ops_of(P)
    one_u, one_p = np.ones(P.n_u), np.ones(P.n_p)
    # K_v 1 = 0 and symmetry; K_p 1 = 0 on every level (pure Neumann)
    assert np.max(np.abs(ops.K @ one_u)) < 1e-13 * abs(ops.K).max()
    assert abs(ops.K - ops.K.T).max() == 0.0
    for L in P.pres_levels:
        A = sp.csr_matrix((L.val.reshape(-1), L.col, L.row_ptr), shape=(L.n, L.n))
        assert np.max(np.abs(A @ np.ones(L.n))) < 1e-13 * abs(A).max()
    # lumped masses: sum = |Omega| = 2, exact on linear functions
    xyz_u, xyz_p = grid(P.xu), grid(P.xp)
    for m, xyz in ((P.m_u, xyz_u), (P.m_p, xyz_p)):
        assert abs(m.sum() - 2.0) < 1e-13
        assert abs(m @ (xyz @ [1.0, 2.0, 3.0]) - 2.0 * (0.5 + 1.0 + 3.0)) < 1e-12
    inn = interior(P.xu)
    # C_d row sums: int d_d phi_i = 0 inside; = +- face integral on the x-faces (divergence theorem)
    for d in range(3):
        assert np.max(np.abs((ops.C[d] @ one_u)[inn])) < 1e-14
    rs = ops.C[0] @ one_u
    My, Mz = (A.toarray().sum(1) for A in (ns.fe1d(P.xu[1])[0], ns.fe1d(P.xu[2])[0]))
    face = np.kron(Mz, My)                                           # int_{x=1} phi_i dS, (y, z) order
    on_x1 = np.isclose(xyz_u[:, 0], 1.0)
    on_x0 = xyz_u[:, 0] == 0.0
    assert np.allclose(rs[on_x1], face, rtol=1e-13, atol=1e-16)
    assert np.allclose(rs[on_x0], -face, rtol=1e-13, atol=1e-16)
    # K_v reproduces linear fields: (grad phi_i, grad u) = 0 inside for linear u
    lin = xyz_u @ [0.3, -1.1, 0.7]
    assert np.max(np.abs((ops.K @ lin)[inn])) < 1e-12


@pytest.mark.parametrize("name", ["ns_small", "ns_mid"])
def test_gradient_coupling_nesting_and_identities(name):
    P = prob(name)
    ops = ops_of(P)
    Pi = sp.csr_matrix((P.Pi[2], P.Pi[1], P.Pi[0]), shape=(P.n_u, P.n_p))
    assert abs(Pi @ np.ones(P.n_p) - 1.0).max() < 1e-15               # partition of unity
    xyz_u, xyz_p = grid(P.xu), grid(P.xp)
    assert np.max(np.abs(Pi @ (xyz_p @ [1.0, 2.0, 3.0]) - xyz_u @ [1.0, 2.0, 3.0])) < 1e-14
    # Q1(Omega_h) in Q1(Omega_h/2): psi_j = sum_k Pi_kj phi_k, so G_c = C_c Pi (G from its own quadrature)
    for c in range(3):
        diff = abs(ops.G[c] - ops.C[c] @ Pi).max()
        assert diff < 1e-15 * 1e2 * abs(ops.G[c]).max(), (c, diff)
    inn = interior(P.xu)
    for c in range(3):
        assert np.max(np.abs((ops.G[c] @ np.ones(P.n_p))[inn])) < 1e-14
        assert np.max(np.abs(ops.G[c].T @ np.ones(P.n_u))) < 1e-14           # D_c const = 0
    # linear pressure p = z: (p, div phi_i e_c) = -int phi_i dp/dx_c = -m_u delta_cz inside
    gz = ons.gradient(ops, xyz_p[:, 2])
    assert np.allclose(gz[inn, 2], -P.m_u[inn], rtol=1e-12, atol=0)
    assert np.max(np.abs(gz[inn, :2])) < 1e-14
    # divergence of linear velocity fields: (div u, psi_j) exactly
    u = np.zeros((P.n_u, 3))
    u[:, 0] = xyz_u[:, 0]
    assert np.allclose(ons.divergence(ops, u), P.m_p, rtol=1e-12, atol=1e-16)
    u = np.stack([xyz_u[:, 0], xyz_u[:, 1], -2.0 * xyz_u[:, 2]], 1)
    assert np.max(np.abs(ons.divergence(ops, u))) < 1e-14


def test_nodewise_products():
    g = np.random.default_rng(0)
    u = g.standard_normal((50, 3))
    v = ons.nodewise_products(u)
    for d in range(3):
        for c in range(3):
            assert np.array_equal(v[d][:, c], u[:, d] * u[:, c])      # I_h(u x u)(x_k) = u(x_k) x u(x_k)
            assert np.array_equal(v[d][:, c], v[c][:, d])             # S:118 symmetry


def test_momentum_spec_examples():
    P = prob("ns_mid")
    ops = ops_of(P)
    inn = interior(P.xu)
    z_u, z_p = np.zeros((P.n_u, 3)), np.zeros(P.n_p)
    un = ons.momentum(ops, z_u, z_p, z_p)
    assert np.all(un[inn] == 0.0) and np.array_equal(un[P.dir_rows], P.dir_vals)
    assert np.all(P.dir_vals[:, 1][np.isclose(grid(P.xu)[P.dir_rows, 0], 1.0)] == 1.0)
    # constant velocity, nu = 0: the interpolated convection vanishes inside
    ops0 = ops_of(P, nu=0.0)
    uc = np.tile([0.3, -0.7, 1.1], (P.n_u, 1))
    un = ons.momentum(ops0, uc, z_p, z_p)
    assert np.max(np.abs(un[inn] - uc[inn])) < 1e-14
    # linear pressure p + q = z pushes -dt e_z inside: du/dt = -grad p
    xyz_p = grid(P.xp)
    un = ons.momentum(ops, z_u, 0.5 * xyz_p[:, 2], 0.5 * xyz_p[:, 2])
    assert np.allclose(un[inn], np.tile([0.0, 0.0, -P.dt], (inn.sum(), 1)), rtol=0, atol=1e-15)


def pres_h(P):
    return oracle.MgHierarchy.from_arrays(P.pres_levels, omega=P.omega,
                                          mean=[(L.mean_w, L.mean_k) for L in P.pres_levels])


def test_pressure_steps_spec_examples():
    P = prob("ns_small")
    ops = ops_of(P)
    h = pres_h(P)
    # u^m = 0 -> q = 0
    d = ons.divergence(ops, np.zeros((P.n_u, 3)))
    q, its, _, _ = oracle.gmres(h, ons.pressure_rhs(ops, d), rtol=1e-10)
    assert np.all(q == 0.0) and its == 0
    # discretely divergence-free u -> d = 0 -> p^m = P(p + q)
    xyz_u = grid(P.xu)
    u = np.stack([xyz_u[:, 0], xyz_u[:, 1], -2.0 * xyz_u[:, 2]], 1)
    d = ons.divergence(ops, u)
    assert np.max(np.abs(d)) < 1e-14
    g = np.random.default_rng(1)
    p, qq = g.standard_normal(P.n_p), g.standard_normal(P.n_p)
    pn = ons.pressure_update(ops, p, qq, d)
    assert np.allclose(pn, oracle.project_zero_mean(p + qq, P.m_p), atol=1e-13)
    assert abs(P.m_p @ pn) < 1e-13 * np.abs(P.m_p * pn).sum()


def test_pressure_solve_matches_bordered_dense():
    P = prob("ns_small")
    ops = ops_of(P)
    F = P.pres_fine
    u, p, q = ns.random_state(P)
    d = ons.divergence(ops, u)
    rhs = ons.pressure_rhs(ops, d)
    q1, its, _, rel = oracle.gmres(pres_h(P), rhs, rtol=1e-12)
    A = oracle.bsr_to_dense(F.n, 1, F.row_ptr, F.col, F.val)
    K = np.zeros((F.n + 1, F.n + 1))
    K[:F.n, :F.n] = A
    K[:F.n, F.n] = P.m_p
    K[F.n, :F.n] = P.m_p
    rc = rhs - rhs.mean()
    sol = np.linalg.solve(K, np.concatenate([rc, [0.0]]))
    assert np.linalg.norm(q1 - sol[:F.n]) <= 1e-9 * np.linalg.norm(sol[:F.n])


def test_pressure_mg_omega_reading():
    """Z27: lambda_max(D^-1 K_p) on the graded paper mesh is 4.42, so Jacobi
    damping must stay below 2 / 4.42 = 0.45; omega = 0.4 converges (45 GMRES
    iterations to 1e-6), omega = 0.6 stagnates."""
    import scipy.sparse.linalg as spl
    P = prob("ns")
    F = P.pres_fine
    A = sp.csr_matrix((F.val.reshape(-1), F.col, F.row_ptr), shape=(F.n, F.n))
    Dh = sp.diags(1.0 / np.sqrt(A.diagonal()))
    lam = spl.eigsh(Dh @ A @ Dh, k=1, which="LA", tol=1e-6)[0][0]
    assert 4.3 < lam < 4.5 and P.omega * lam < 2.0
    b = np.random.default_rng(0).standard_normal(P.n_p)
    _, its, _, rel = oracle.gmres(pres_h(P), b, rtol=1e-6)
    assert rel <= 1e-6 and its <= 60


def test_step_invariants():
    P = prob("ns_mid")
    ops = ops_of(P)
    u, p, q = ns.random_state(P, scale=0.1)
    un, pn, qn, d, its = ons.step(ops, pres_h(P), u, p, q, rtol=1e-10)
    assert np.array_equal(un[P.dir_rows], P.dir_vals)
    for v in (pn, qn):
        assert abs(P.m_p @ v) < 1e-13 * np.abs(P.m_p * v).sum()
    F = P.pres_fine
    rhs = ons.pressure_rhs(ops, d)
    r = oracle.residual(F.n, 1, F.row_ptr, F.col, F.val, qn, rhs - rhs.mean())
    assert np.linalg.norm(r) <= 2e-10 * np.linalg.norm(rhs - rhs.mean())
    assert np.allclose(d, ons.divergence(ops, un), rtol=0, atol=0)
