"""Oracle pins for the global constraint int_Omega p = 0 on every level (
SPEC project_zero_mean S:452-460, invariants S:466-467, design S:474) and the
pure-Neumann pressure Poisson generator (Alg. 2 Step 2).

Pinned against things other than the oracle itself: the SPEC's worked
examples, a closed-form 1D Neumann solve, the exact lumped-mass quadrature of
linear functions, the kernel of the Neumann operator, and the solution of the
bordered saddle system [[A, w], [w^T, 0]] by a dense library solve."""
import numpy as np
import pytest

import oracle
from problems import configs

NEU = ["pres_small", "pres_mid"]


def test_project_zero_mean_spec_examples():
    w = np.array([1.0, 1.0])
    assert np.array_equal(oracle.project_zero_mean(np.array([1.0, 3.0]), w), [-1.0, 1.0])
    c = np.full(5, 3.25)
    assert np.array_equal(oracle.project_zero_mean(c, np.arange(1.0, 6.0)), np.zeros(5))
    g = np.random.default_rng(0)
    x, wr = g.standard_normal(40), g.random(40) + 0.1
    p = oracle.project_zero_mean(x, wr)
    assert abs(wr @ p) < 1e-13 * np.abs(wr * x).sum()
    assert np.allclose(oracle.project_zero_mean(p, wr), p, atol=1e-14)                     # idempotent
    assert np.allclose(oracle.project_zero_mean(x + 7.5, wr), p, atol=1e-13)               # P(x + c1) = P(x)
    # kernel-vector form: entries with k = 0 (identity rows) are never touched
    k = (g.random(40) > 0.2).astype(float)
    q = oracle.project_zero_mean(x, wr * k, k)
    assert np.array_equal(q[k == 0], x[k == 0]) and abs((wr * k) @ q) < 1e-13 * np.abs(wr * x).sum()


def test_consistent_projection():
    g = np.random.default_rng(1)
    k = (g.random(30) > 0.25).astype(float)
    b = g.standard_normal(30)
    c = oracle.consistent(b, k)
    assert abs(k @ c) < 1e-13 * np.abs(b).sum()
    assert np.array_equal(c[k == 0], b[k == 0])
    assert np.allclose(oracle.consistent(c, k), c, atol=1e-15)


def test_coarse_regularisation_closed_form():
    """1D Neumann Laplacian (3 nodes, h = 1), lumped mass w = (1/2, 1, 1/2),
    b = (1, 0, -1): A x = b with w^T x = 0 has the solution x = (1, 0, -1)
    (x2 = x1 - 1, x3 = x1 - 2, 2 x1 - 2 = 0)."""
    A = np.array([[1.0, -1.0, 0.0], [-1.0, 2.0, -1.0], [0.0, -1.0, 1.0]])
    w = np.array([0.5, 1.0, 0.5])
    x = np.linalg.solve(A + oracle.mg.coarse_regularisation(A, w), np.array([1.0, 0.0, -1.0]))
    assert np.allclose(x, [1.0, 0.0, -1.0], atol=1e-14)


@pytest.mark.parametrize("name", NEU + ["pres"])
def test_neumann_generator_weights_and_kernel(name):
    P = configs.build(name)
    root, box = P.meta["root"], P.box
    vol = float(np.prod(box))
    for L in P.levels:
        # A_l k_l = 0: the condensed Neumann operator annihilates constants
        Ak = oracle.spmv(L.n, 1, L.row_ptr, L.col, L.val, L.mean_k)
        assert np.max(np.abs(Ak)) < 1e-12 * np.max(np.abs(L.val))
        # lumped-mass weights integrate every linear function exactly (Q1 with
        # conforming hanging-node interpolation reproduces it): int 1 = |Omega|,
        # int (x + 2y + 3z) = |Omega| (0.5 + 2*0.5 + 3*1)
        assert abs(L.mean_w.sum() - vol) < 1e-13 * vol
        xyz = configs.node_xyz(L.nodes, root, box)
        f = xyz @ np.array([1.0, 2.0, 3.0])
        assert abs(L.mean_w @ f - vol * 4.5) < 1e-12 * vol * 4.5
        assert np.all(L.mean_w[L.mean_k == 1] > 0) and np.all(L.mean_w[L.mean_k == 0] == 0)
    if name == "pres":
        assert P.fine.n == 70785          # the paper's 32 x 32 x 64 pressure mesh


def bordered_solution(L, w, b):
    A = oracle.bsr_to_dense(L.n, 1, L.row_ptr, L.col, L.val)
    n = L.n
    K = np.zeros((n + 1, n + 1))
    K[:n, :n] = A
    K[:n, n] = w
    K[n, :n] = w
    sol = np.linalg.solve(K, np.concatenate([b, [0.0]]))
    return sol[:n], sol[n]


@pytest.mark.parametrize("name", NEU)
def test_neumann_gmres_matches_bordered_solve(name):
    P = configs.build(name)
    F = P.fine
    h = oracle.MgHierarchy.from_arrays(P.levels, omega=P.omega, mean=[(L.mean_w, L.mean_k) for L in P.levels])
    x, its, hist, rel = oracle.gmres(h, P.b, rtol=1e-12)
    bc = oracle.consistent(P.b, F.mean_k)
    xe, lam = bordered_solution(F, F.mean_w, bc)
    assert abs(lam) < 1e-10 * np.abs(bc).max()          # consistent rhs: the multiplier vanishes
    assert np.linalg.norm(x - xe) <= 1e-9 * np.linalg.norm(xe)
    assert abs(F.mean_w @ x) <= 1e-13 * np.abs(F.mean_w * x).sum()
    assert its <= 10                                    # P:159 "a maximum of n_G <= 10"
    xr, itr, hr = oracle.richardson(h, P.b, rtol=1e-10, max_iter=60)
    assert np.linalg.norm(xr - xe) <= 1e-8 * np.linalg.norm(xe)
    assert (hr[-1] / hr[0]) ** (1.0 / itr) < 0.2          # h-independent contraction of the V-cycle


def test_neumann_vcycle_linear_and_zero_mean():
    """V-cycle from zero is linear in b and its output has zero weighted
    mean on the finest level; constants added to b are projected away."""
    P = configs.build("pres_mid")
    F = P.fine
    h = oracle.MgHierarchy.from_arrays(P.levels, omega=P.omega, mean=[(L.mean_w, L.mean_k) for L in P.levels])
    Lf = len(P.levels) - 1
    g = np.random.default_rng(3)
    b1 = oracle.consistent(g.standard_normal(F.n), F.mean_k)
    b2 = oracle.consistent(g.standard_normal(F.n), F.mean_k)
    z = np.zeros(F.n)
    v1, v2 = oracle.vcycle(h, Lf, z, b1), oracle.vcycle(h, Lf, z, b2)
    v12 = oracle.vcycle(h, Lf, z, 2.0 * b1 - 3.0 * b2)
    assert np.linalg.norm(v12 - (2.0 * v1 - 3.0 * v2)) <= 1e-12 * np.linalg.norm(v12)
    assert abs(F.mean_w @ v1) <= 1e-13 * np.abs(F.mean_w * v1).sum()


def test_neumann_iterations_h_independent():
    its = []
    for name in NEU + ["pres"]:
        P = configs.build(name, keep_geometry=False)
        h = oracle.MgHierarchy.from_arrays(P.levels, omega=P.omega, mean=[(L.mean_w, L.mean_k) for L in P.levels])
        its.append(oracle.gmres(h, P.b, rtol=1e-10)[1])
    assert max(its) - min(its) <= 2 and max(its) <= 10, its
