"""Pins of the oracle's multigrid/Krylov layer (oracle/mg.py) against textbook
closed forms and brute force:
  * V-cycle == dense error-operator recursion
        E_0 = 0,  E_l = S^nu2 (I - P (I - E_{l-1}) A_{l-1}^{-1} R A_l) S^nu1,
        V_l(x, b) = E_l x + (I - E_l) A_l^{-1} b          (Hackbusch, cited P:23)
  * single level: A_0^{-1} b (Alg. gmg Step 0); linearity in b
  * solves agree with dense LU; GMRES residual monotone
  * h-independent contraction ("varies only slightly"), 5-10 GMRES steps
    on the transport-diffusion operator
  * LFA of the Q1 Laplacian: lambda_max(D^-1 A) -> 3/2 (closed form symbol)
  * O(h^2) L2 convergence with hanging nodes (manufactured solution)."""
import numpy as np
import pytest

import oracle as O
from mgtest_util import problem
from problems import configs as C
from problems import fem as F
from problems import mesh as M


def dense_levels(h):
    out = []
    for l, L in enumerate(h.levels):
        A = O.bsr_to_dense(L.n, L.bs, L.rp, L.col, L.val)
        D = np.zeros_like(A)
        for i in range(L.n):
            s = slice(i * L.bs, (i + 1) * L.bs)
            D[s, s] = np.linalg.inv(A[s, s])
        P = None
        if l > 0:
            rp, col, w = L.P
            nc = h.levels[l - 1].n
            P = np.zeros((L.n * L.bs, nc * L.bs))
            rows = np.repeat(np.arange(L.n), np.diff(rp))
            for t in range(len(col)):
                for c in range(L.bs):
                    P[rows[t] * L.bs + c, col[t] * L.bs + c] = w[t * L.wpe + (c if L.wpe > 1 else 0)]
        out.append((A, D, P))
    return out


def error_operators(h, dl):
    I0 = np.eye(dl[0][0].shape[0])
    E = [np.zeros_like(I0)]
    for l in range(1, len(dl)):
        A, D, P = dl[l]
        Ac = dl[l - 1][0]
        I = np.eye(A.shape[0])
        S = I - h.omega * D @ A
        CGC = I - P @ (np.eye(Ac.shape[0]) - E[l - 1]) @ np.linalg.solve(Ac, P.T @ A)
        E.append(np.linalg.matrix_power(S, h.nu_post) @ CGC @ np.linalg.matrix_power(S, h.nu_pre))
    return E


def tiny(name):
    cfgs = {
        "poisson2d": ((2, 2), (1.0, 1.0), [("uniform",), ("band", [1], 1), ("band", [1], 1)],
                      F.Operator("poisson", 1, True), 0.8),
        "td2d": ((2, 2), (1.0, 1.0), [("uniform",), ("band", [0, 1], 1), ("band", [0, 1], 1)],
                 F.Operator("td", 1, False, C.TD), 0.8),
        "elast3d": ((2, 2, 2), (1.0, 1.0, 1.0), [("band", [0], 1), ("band", [0], 1)],
                    F.Operator("elasticity", 3, True, C.ELAST), 0.5),
    }
    root, box, steps, op, om = cfgs[name]
    return C.make_problem(name, root, box, steps, op, omega=om)


@pytest.mark.parametrize("name", ["poisson2d", "td2d", "elast3d"])
def test_vcycle_equals_dense_recursion(name):
    p = tiny(name)
    h = O.MgHierarchy.from_arrays(p.levels, omega=p.omega)
    dl = dense_levels(h)
    E = error_operators(h, dl)
    rng = np.random.default_rng(1)
    A = dl[-1][0]
    N = A.shape[0]
    x = rng.standard_normal(N)
    b = rng.standard_normal(N)
    got = O.vcycle(h, len(h.levels) - 1, x, b)
    ref = E[-1] @ x + (np.eye(N) - E[-1]) @ np.linalg.solve(A, b)
    assert np.abs(got - ref).max() <= 1e-11 * (np.abs(ref).max() + np.abs(x).max())


def test_vcycle_single_level_linearity_zero():
    p = problem("c1_poisson")
    h = O.MgHierarchy.from_arrays(p.levels[:1], omega=p.omega)
    A = O.bsr_to_dense(p.levels[0].n, 1, p.levels[0].row_ptr, p.levels[0].col, p.levels[0].val)
    b = np.random.default_rng(3).standard_normal(A.shape[0])
    assert np.allclose(O.vcycle(h, 0, np.ones_like(b), b), np.linalg.solve(A, b), rtol=1e-13, atol=1e-14)
    h = O.MgHierarchy.from_arrays(p.levels, omega=p.omega)
    L = len(h.levels) - 1
    rng = np.random.default_rng(4)
    b1, b2 = rng.standard_normal(p.n_dof), rng.standard_normal(p.n_dof)
    z = np.zeros(p.n_dof)
    v = O.vcycle(h, L, z, 2.0 * b1 - 3.0 * b2)
    assert np.allclose(v, 2.0 * O.vcycle(h, L, z, b1) - 3.0 * O.vcycle(h, L, z, b2), rtol=0, atol=1e-12 * np.abs(v).max())
    assert not O.vcycle(h, L, z, z).any()


@pytest.mark.parametrize("name", ["c1", "c1_poisson", "c2_small", "c3_small"])
def test_solves_match_dense_lu(name):
    p = problem(name)
    h = O.MgHierarchy.from_arrays(p.levels, omega=p.omega)
    F_ = p.fine
    A = O.bsr_to_dense(F_.n, F_.bs, F_.row_ptr, F_.col, F_.val)
    xd = np.linalg.solve(A, p.b)
    x, its, hist, rr = O.gmres(h, p.b, rtol=1e-10)
    assert rr <= 1e-10
    kappa = np.linalg.cond(A) if A.shape[0] <= 2000 else 1e6
    assert np.linalg.norm(x - xd) <= 1e-10 * kappa * np.linalg.norm(xd)
    assert all(b <= a * (1 + 1e-12) for a, b in zip(hist, hist[1:]))
    if F_.n * F_.bs <= 2000:
        xr, itr, _ = O.richardson(h, p.b, rtol=1e-10, max_iter=100)
        assert np.linalg.norm(xr - xd) <= 1e-9 * kappa * np.linalg.norm(xd)


def _poisson_uniform(n):
    return C.make_problem("pu", (1, 1), (1.0, 1.0), [("uniform",)] * n, F.Operator("poisson", 1, True))


def test_h_independent_contraction():
    """Richardson-MG V(2,2), omega = 0.8: rho bounded (<= 0.2) on uniform n = 3..6 and its
    growth shrinks (scratch 0.058, 0.066, 0.077, 0.091)."""
    rhos = []
    for n in range(3, 7):
        p = _poisson_uniform(n)
        h = O.MgHierarchy.from_arrays(p.levels, omega=0.8)
        _, its, hist = O.richardson(h, p.b, rtol=1e-14, max_iter=14)
        k = min(len(hist) - 1, 10)
        rhos.append((hist[k] / hist[3]) ** (1.0 / (k - 3)))
    assert max(rhos) <= 0.2
    assert rhos[-1] - rhos[-2] <= 0.05


def test_td_gmres_iterations_5_to_10():
    """with MG preconditioning 'never ... more than 5-10 GMRES steps';
    iteration counts vary only slightly with the level (P:390, S:671 +/-2)."""
    its = []
    for n in (5, 6, 7):
        p = C.make_problem("tdu", (1, 1), (1.0, 1.0), [("uniform",)] * n, F.Operator("td", 1, False, C.TD))
        h = O.MgHierarchy.from_arrays(p.levels, omega=0.8)
        _, it, _, rr = O.gmres(h, p.b, rtol=1e-10)
        assert rr <= 1e-10
        its.append(it)
    assert all(4 <= i <= 10 for i in its), its
    assert max(its) - min(its) <= 2


def test_lfa_lambda_max_q1_laplacian():
    """Q1 Laplacian symbol of D^-1 A: 1 - (c1+c2)/4 - c1 c2/2, max 3/2 at (pi, 0);
    on the Dirichlet 24^2 mesh the largest eigenvalue is just below 1.5."""
    p = C.make_problem("lfa", (24, 24), (1.0, 1.0), [], F.Operator("poisson", 1, True))
    L = p.fine
    A = O.bsr_to_dense(L.n, 1, L.row_ptr, L.col, L.val)
    free = ~L.cmask[:, 0]
    A = A[free][:, free]
    lam = np.linalg.eigvals(A / np.diag(A)[:, None]).real.max()
    assert 1.47 < lam < 1.5
    th = np.linspace(0, np.pi, 201)
    c1, c2 = np.meshgrid(np.cos(th), np.cos(th))
    assert np.isclose((1 - 0.25 * (c1 + c2) - 0.5 * c1 * c2).max(), 1.5)


def test_elasticity_lambda_max_and_omega():
    """Reading Z1: for 3x3 block-Jacobi on M + dt^2 K_e (lambda/mu = 4),
    lambda_max(D^-1 A) grows towards 27/8 > 2/0.8, so omega = 0.8 is unstable and
    omega = 0.5 is used; omega * lambda_max < 2 must hold."""
    lams = []
    for r in (3, 5):
        p = C.make_problem("el", (r, r, r), (1.0, 1.0, 1.0), [], F.Operator("elasticity", 3, True, C.ELAST))
        L = p.fine
        A = O.bsr_to_dense(L.n, 3, L.row_ptr, L.col, L.val)
        free = ~L.cmask.ravel()
        dinv = O.block_diag_inverse(L.n, 3, L.row_ptr, L.col, L.val)
        D = np.zeros_like(A)
        for i in range(L.n):
            D[3 * i:3 * i + 3, 3 * i:3 * i + 3] = dinv[i]
        lams.append(np.linalg.eigvals((D @ A)[free][:, free]).real.max())
    assert lams[0] < lams[1] < 27 / 8 + 1e-9
    assert lams[1] > 2 / 0.8 * 0.95 and 0.5 * lams[1] < 2


def _l2_error(p, x):
    """sqrt(sum_T sum_q w |u_h - u|^2) with the 2-point Gauss rule."""
    L = p.fine
    mesh, nodes = L.mesh, L.nodes
    u = O.mg.apply_H(L.H, x, 1)
    xq, wq = F.gauss2(2)
    phi, _ = F.q1_basis(2, xq)
    h = F.cell_sizes(mesh, p.box)
    x0 = mesh.ijk * h
    vol = np.prod(h, axis=1)
    err = 0.0
    for q in range(len(wq)):
        pts = x0 + xq[q] * h
        uh = sum(phi[q, a] * u[nodes.conn[:, a]] for a in range(4))
        ex = np.sin(np.pi * pts[:, 0]) * np.sin(np.pi * pts[:, 1])
        err += np.sum(wq[q] * vol * (uh - ex) ** 2)
    return np.sqrt(err)


def test_oh2_convergence_with_hanging_nodes():
    """-Lap u = 2 pi^2 sin(pi x) sin(pi y), u = 0 on the boundary, on band-refined meshes
    with hanging nodes refined uniformly u = 0..2 times: L2 error ratio -> 4."""
    f = lambda xy: 2 * np.pi ** 2 * np.sin(np.pi * xy[:, 0]) * np.sin(np.pi * xy[:, 1])  # noqa: E731
    errs = []
    for u in range(3):
        steps = [("uniform",), ("band", [1], 1), ("band", [1], 1)] + [("uniform",)] * u
        p = C.make_problem("mms", (2, 2), (1.0, 1.0), steps, F.Operator("poisson", 1, True), f=f)
        assert p.fine.cmask.any() and M.build_nodes(p.fine.mesh).hanging.any()
        h = O.MgHierarchy.from_arrays(p.levels, omega=0.8)
        x, its, _, rr = O.gmres(h, p.b, rtol=1e-12)
        errs.append(_l2_error(p, x))
    ratios = [errs[i] / errs[i + 1] for i in range(len(errs) - 1)]
    assert all(3.6 < r < 4.4 for r in ratios), ratios


def test_gmres_outer_operator_pin():
    """O.gmres(op=...) (mixed-precision preconditioning): with a
    preconditioner hierarchy built on perturbed (fp32-rounded) operators, GMRES
    must still converge to the solution of the OUTER operator -- pinned by a
    dense LU of that operator -- and must not converge to the perturbed one."""
    from types import SimpleNamespace
    P = C.build("c3_small")
    F = P.fine
    rounded = []
    for L in P.levels:
        R = SimpleNamespace(n=L.n, bs=L.bs, row_ptr=L.row_ptr, col=L.col, P=L.P, wpe=L.wpe,
                            val=L.val.astype(np.float32).astype(np.float64))
        rounded.append(R)
    h32 = O.MgHierarchy.from_arrays(rounded, omega=P.omega)
    op = SimpleNamespace(n=F.n, bs=F.bs, rp=F.row_ptr, col=F.col, val=F.val)
    x, its, hist, rel = O.gmres(h32, P.b, rtol=1e-12, op=op)
    A = O.bsr_to_dense(F.n, F.bs, F.row_ptr, F.col, F.val)
    xe = np.linalg.solve(A, P.b)
    assert np.linalg.norm(x - xe) <= 1e-9 * np.linalg.norm(xe)
    A32 = O.bsr_to_dense(F.n, F.bs, F.row_ptr, F.col, rounded[-1].val)
    x32 = np.linalg.solve(A32, P.b)
    assert np.linalg.norm(x32 - xe) > 1e3 * np.linalg.norm(x - xe)
