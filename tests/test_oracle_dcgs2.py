"""Pins of the oracle's GMRES with delayed classical Gram-Schmidt
reorthogonalisation (`oracle.gmres_dcgs2`, reading Z29 in DESIGN.md; an
opt-in alternative to the paper's MGS) against the property that
defines GMRES whatever the orthogonalisation: one restart cycle of k steps
from x0 returns the minimiser of ||b - A x|| over x0 + B K_k(A B, r0), built
here with a Householder-QR basis and LAPACK least squares
(`_min_res_cycle` of tests/test_oracle_pins_r2.py), and convergence against a
sparse LU solve with the error bound ||x - x*|| <= ||b - A x|| / lambda_min."""
import numpy as np
import pytest

import oracle as O
from mgtest_util import problem
from test_oracle_pins_r2 import _lu_solve_and_lambda_min, _min_res_cycle, _sparse, weak_hierarchy


@pytest.mark.parametrize("k", [1, 2, 4, 7])
def test_dcgs2_truncation_is_min_residual(k):
    p = problem("c3_small")
    h = O.MgHierarchy.from_arrays(p.levels, omega=p.omega)
    A = _sparse(h.levels[-1])
    x0 = np.random.default_rng(5).standard_normal(A.shape[0]) * 0.1
    x, its, hist, rel = O.gmres_dcgs2(h, p.b, x0=x0, rtol=1e-14, restart=30, max_iter=k)
    assert its == k
    exp = _min_res_cycle(h, A, p.b, x0, k)
    assert np.linalg.norm(x - exp) <= 1e-9 * np.linalg.norm(exp)
    r_exp = np.linalg.norm(p.b - A @ exp) / np.linalg.norm(p.b - A @ x0)
    # the estimate uses the tentative last column (reorthogonalisation folded in one step later)
    assert abs(hist[-1] - r_exp) <= 1e-7 * r_exp + 1e-15
    assert abs(rel - r_exp) <= 1e-8 * r_exp + 1e-15


@pytest.mark.parametrize("restart,max_iter", [(3, 6), (3, 7), (2, 5), (1, 3)])
def test_dcgs2_restart_is_repeated_min_residual(restart, max_iter):
    p = problem("c3_small")
    h = O.MgHierarchy.from_arrays(p.levels, omega=p.omega)
    A = _sparse(h.levels[-1])
    x, its, hist, rel = O.gmres_dcgs2(h, p.b, rtol=1e-15, restart=restart, max_iter=max_iter)
    assert its == max_iter
    exp = np.zeros(A.shape[0])
    left = max_iter
    while left:
        kk = min(restart, left)
        exp = _min_res_cycle(h, A, p.b, exp, kk)
        left -= kk
    assert np.linalg.norm(x - exp) <= 1e-9 * np.linalg.norm(exp)


def test_dcgs2_converges_to_lu_restart3():
    p = problem("c3_small")
    h = O.MgHierarchy.from_arrays(p.levels, omega=p.omega)
    A = _sparse(h.levels[-1])
    xe, lmin = _lu_solve_and_lambda_min(A, p.b)
    x, its, hist, rel = O.gmres_dcgs2(h, p.b, rtol=1e-10, restart=3, max_iter=300)
    assert rel <= 1e-10 and its < 300
    rn = np.linalg.norm(p.b - A @ x)
    assert np.linalg.norm(x - xe) <= 1.01 * rn / lmin + 1e-13 * np.linalg.norm(xe)


def test_dcgs2_beyond_one_restart_cycle():
    """A weak preconditioner: more than 30 steps, the basis grows to m = 30
    vectors (where classical Gram-Schmidt without reorthogonalisation would
    lose orthogonality first)."""
    p, h = weak_hierarchy()
    A = _sparse(h.levels[-1])
    x, its, hist, rel = O.gmres_dcgs2(h, p.b, rtol=1e-10, restart=30, max_iter=400)
    x_m, its_m, _, _ = O.gmres(h, p.b, rtol=1e-10, restart=30, max_iter=400)
    assert 30 < its < 400 and rel <= 1e-10 and abs(its - its_m) <= 1
    xe, lmin = _lu_solve_and_lambda_min(A, p.b)
    rn = np.linalg.norm(p.b - A @ x)
    assert np.linalg.norm(x - xe) <= 1.01 * rn / lmin + 1e-13 * np.linalg.norm(xe)
    x30, its30, _, _ = O.gmres_dcgs2(h, p.b, rtol=1e-15, restart=30, max_iter=30)
    exp = _min_res_cycle(h, A, p.b, np.zeros_like(p.b), 30)
    assert its30 == 30
    assert np.linalg.norm(x30 - exp) <= 1e-8 * np.linalg.norm(exp)


@pytest.mark.parametrize("name", ["c1", "c2_small", "c3_small", "c4_small", "c5_small"])
def test_dcgs2_iterations_equal_mgs(name):
    """Same Krylov spaces: the iteration counts of the two orthogonalisations
    agree (+-1) at 1e-10 and both meet it on the true residual."""
    p = problem(name)
    h = O.MgHierarchy.from_arrays(p.levels, omega=p.omega)
    _, i1, _, r1 = O.gmres(h, p.b, rtol=1e-10)
    x2, i2, _, r2 = O.gmres_dcgs2(h, p.b, rtol=1e-10)
    assert abs(i1 - i2) <= 1 and r1 <= 1e-10 and r2 <= 1e-10
