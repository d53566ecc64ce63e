"""Mixed-precision mode: the V-cycle's operators A_l are
stored rounded to fp32 (vectors, accumulation, D^-1 of the rounded blocks,
transfers and the coarse inverse stay fp64), the finest level keeps its fp64
operator for GMRES and residuals.

Parity: the oracle runs the same algorithm on the same rounded operators
(rounding is part of the input, done identically on both sides), so per-op
results match at 1e-12 scaled and V-cycles at 1e-10; GMRES with the fp64
outer operator reaches the true fp64 residual 1e-10 with iteration counts
+-1 of the oracle and of the fp64 mode."""
import functools
from types import SimpleNamespace

import numpy as np
import pytest

from gpu_util import TOL_OP, TOL_VCYCLE, absA_x, assert_close_scaled, build_gpu, dev, host
from mgtest_util import problem

import oracle

pytestmark = pytest.mark.gpu

CASES = ["c2_small", "c3_small", "c5_small"]


def rounded(levels):
    out = []
    for L in levels:
        R = SimpleNamespace(**{k: getattr(L, k) for k in ("n", "bs", "row_ptr", "col", "P", "wpe")})
        R.val = L.val.astype(np.float32).astype(np.float64)
        out.append(R)
    return out


@functools.lru_cache(maxsize=None)
def setup(name):
    import paper_2405_05047_b200 as m
    P = problem(name)
    mg = build_gpu(P.levels, P.bs, omega=P.omega, H=P.fine.H, precision=m.MG_PREC_MIXED)
    h32 = oracle.MgHierarchy.from_arrays(rounded(P.levels), omega=P.omega)
    return P, mg, h32


@pytest.mark.parametrize("name", CASES)
def test_mixed_per_op(name):
    import paper_2405_05047_b200 as m
    P, mg, h32 = setup(name)
    bs = P.bs
    Lf = len(P.levels) - 1
    for l, L in enumerate(P.levels):
        g = np.random.default_rng(200 + l)
        x = g.standard_normal(L.n * bs)
        b = g.standard_normal(L.n * bs)
        out = dev(np.zeros(L.n * bs))
        m.mg_sweep(mg.ctx, l, dev(x), dev(b), out)          # V-cycle smoother: rounded A, D^-1 of rounded blocks
        exp = h32.smooth(l, x, b)
        R = h32.levels[l]
        sc = np.abs(x) + P.omega * oracle.spmv(L.n, bs, R.rp, R.col, np.abs(R.val), np.abs(x)) + np.abs(b)
        assert_close_scaled(host(out), exp, sc, tol=10 * TOL_OP, what=f"{name} mixed sweep l={l}")
        m.mg_residual(mg.ctx, l, dev(x), dev(b), out)       # problem operator: fp64 on the finest level
        Lr = L if l == Lf else SimpleNamespace(n=L.n, bs=bs, row_ptr=R.rp, col=R.col, val=R.val)
        exp = oracle.residual(L.n, bs, Lr.row_ptr, Lr.col, Lr.val, x, b)
        assert_close_scaled(host(out), exp, absA_x(Lr, x) + np.abs(b), what=f"{name} mixed residual l={l}")


@pytest.mark.parametrize("name", CASES)
def test_mixed_vcycle(name):
    import paper_2405_05047_b200 as m
    P, mg, h32 = setup(name)
    Lf = len(P.levels) - 1
    z = dev(np.zeros(P.n_dof))
    m.mg_vcycle_zero(mg.ctx, z, dev(P.b))
    exp = oracle.vcycle(h32, Lf, np.zeros(P.n_dof), P.b)
    assert np.linalg.norm(host(z) - exp) <= TOL_VCYCLE * np.linalg.norm(exp)


@pytest.mark.parametrize("name", CASES)
def test_mixed_gmres_reaches_fp64_residual(name):
    import paper_2405_05047_b200 as m
    P, mg, h32 = setup(name)
    F = P.fine
    x = dev(np.zeros(P.n_dof))
    st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(P.b), rtol=1e-10)
    fine64 = SimpleNamespace(n=F.n, bs=F.bs, rp=F.row_ptr, col=F.col, val=F.val)
    xe, ite, _, rele = oracle.gmres(h32, P.b, rtol=1e-10, op=fine64)
    assert conv and abs(its - ite) <= 1, (its, ite)
    # true fp64 residual
    r = oracle.residual(F.n, F.bs, F.row_ptr, F.col, F.val, host(x), P.b)
    assert np.linalg.norm(r) <= 2e-10 * np.linalg.norm(P.b)
    # same iteration count as the all-fp64 solver (+-1)
    h64 = oracle.MgHierarchy.from_arrays(P.levels, omega=P.omega)
    _, it64, _, _ = oracle.gmres(h64, P.b, rtol=1e-10)
    assert abs(its - it64) <= 1


@pytest.mark.parametrize("name", ["c2_small", "c3_small"])
def test_mixed_richardson_defect_correction(name):
    import paper_2405_05047_b200 as m
    P, mg, h32 = setup(name)
    F = P.fine
    x = dev(np.zeros(P.n_dof))
    st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(P.b), method=m.MG_RICHARDSON, rtol=1e-10, max_iter=200)
    assert conv
    r = oracle.residual(F.n, F.bs, F.row_ptr, F.col, F.val, host(x), P.b)
    assert np.linalg.norm(r) <= 2e-10 * np.linalg.norm(P.b)
    # oracle: x += GMG_32(L, 0, b - A_64 x)
    xo = np.zeros(P.n_dof)
    r0 = np.linalg.norm(P.b)
    k = 0
    while k < 200:
        k += 1
        xo = xo + oracle.vcycle(h32, len(P.levels) - 1, np.zeros(P.n_dof),
                                oracle.residual(F.n, F.bs, F.row_ptr, F.col, F.val, xo, P.b))
        if np.linalg.norm(oracle.residual(F.n, F.bs, F.row_ptr, F.col, F.val, xo, P.b)) <= 1e-10 * r0:
            break
    assert abs(its - k) <= 1
