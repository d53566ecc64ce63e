"""GPU parity of the global constraint int p = 0 on every level (SPEC
S:452-474; reading Z25) on the pure-Neumann pressure Poisson of the
projection step (Alg. 2 Step 2): the projection entry points, the
regularised coarse solve, V-cycles, GMRES and MG iteration against the
oracle; the distributed path (LOCAL transport) and value updates."""
import functools
import os
import threading

import numpy as np
import pytest

from gpu_util import TOL_VCYCLE, assert_close_scaled, build_gpu, dev, host
from mgtest_util import problem

import oracle

pytestmark = pytest.mark.gpu

CASES = ["pres_small", "pres_mid"]


def mean_of(P):
    return [(L.mean_w, L.mean_k) for L in P.levels]


@functools.lru_cache(maxsize=None)
def setup(name, precision=0, use_graphs=True):
    P = problem(name)
    mg = build_gpu(P.levels, P.bs, omega=P.omega, H=P.fine.H, precision=precision, use_graphs=use_graphs)
    h = oracle.MgHierarchy.from_arrays(P.levels, omega=P.omega, mean=mean_of(P))
    return P, mg, h


@pytest.mark.parametrize("name", CASES)
def test_projections_every_level(name):
    import paper_2405_05047_b200 as m
    P, mg, h = setup(name)
    for l, L in enumerate(P.levels):
        g = np.random.default_rng(40 + l)
        x = g.standard_normal(L.n) + 3.0
        t = dev(x)
        m.mg_project_zero_mean(mg.ctx, l, t)
        assert_close_scaled(host(t), oracle.project_zero_mean(x, L.mean_w, L.mean_k), np.abs(x),
                            what=f"{name} zero mean l={l}")
        t = dev(x)
        m.mg_make_consistent(mg.ctx, l, t)
        assert_close_scaled(host(t), oracle.consistent(x, L.mean_k), np.abs(x), what=f"{name} consistent l={l}")


@pytest.mark.parametrize("name", CASES)
def test_regularised_coarse_solve(name):
    import paper_2405_05047_b200 as m
    P, mg, h = setup(name)
    L0 = P.levels[0]
    d = oracle.consistent(np.random.default_rng(5).standard_normal(L0.n), L0.mean_k)
    y = dev(np.zeros(L0.n))
    m.mg_coarse_solve(mg.ctx, dev(d), y)
    exp = h.coarse_solve(d)
    assert np.linalg.norm(host(y) - exp) <= TOL_VCYCLE * np.linalg.norm(exp)
    # it solves A_0 y = d on the free DOFs
    r = oracle.residual(L0.n, 1, L0.row_ptr, L0.col, L0.val, host(y), d)
    assert np.linalg.norm(r) <= 1e-10 * np.linalg.norm(d)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("graphs", [True, False])
def test_vcycle_matches_oracle(name, graphs):
    import paper_2405_05047_b200 as m
    P, mg, h = setup(name, use_graphs=graphs)
    F = P.fine
    Lf = len(P.levels) - 1
    b = oracle.consistent(P.b, F.mean_k)
    z = dev(np.zeros(P.n_dof))
    m.mg_vcycle_zero(mg.ctx, z, dev(b))
    exp = oracle.vcycle(h, Lf, np.zeros(P.n_dof), b)
    got = host(z)
    assert np.linalg.norm(got - exp) <= TOL_VCYCLE * np.linalg.norm(exp)
    assert abs(F.mean_w @ got) <= 1e-13 * np.abs(F.mean_w * got).sum()
    x0 = np.random.default_rng(9).standard_normal(P.n_dof)
    x = dev(x0)
    m.mg_vcycle(mg.ctx, x, dev(b))
    exp = oracle.vcycle(h, Lf, x0, b)
    assert np.linalg.norm(host(x) - exp) <= TOL_VCYCLE * np.linalg.norm(exp)


@pytest.mark.parametrize("name", CASES + ["pres"])
def test_gmres_matches_oracle(name):
    import paper_2405_05047_b200 as m
    P, mg, h = setup(name)
    F = P.fine
    b = dev(P.b)                                    # inconsistent: mg_solve projects it (b stays untouched)
    x = dev(np.zeros(P.n_dof))
    st, its, rel, conv = m.mg_solve(mg.ctx, x, b, rtol=1e-10)
    assert np.array_equal(host(b), P.b)
    xe, ite, _, rele = oracle.gmres(h, P.b, rtol=1e-10)
    assert conv and abs(its - ite) <= 1, (its, ite)
    got = host(x)
    assert np.linalg.norm(got - xe) <= 1e-8 * np.linalg.norm(xe)
    assert abs(F.mean_w @ got) <= 1e-13 * np.abs(F.mean_w * got).sum()
    bc = oracle.consistent(P.b, F.mean_k)
    r = oracle.residual(F.n, 1, F.row_ptr, F.col, F.val, got, bc)
    assert np.linalg.norm(r) <= 2e-10 * np.linalg.norm(bc)


@pytest.mark.parametrize("name", CASES)
def test_richardson_matches_oracle(name):
    import paper_2405_05047_b200 as m
    P, mg, h = setup(name)
    x = dev(np.zeros(P.n_dof))
    st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(P.b), method=m.MG_RICHARDSON, rtol=1e-10, max_iter=100)
    xe, ite, hist = oracle.richardson(h, P.b, rtol=1e-10, max_iter=100)
    assert conv and abs(its - ite) <= 1, (its, ite)
    assert np.linalg.norm(host(x) - xe) <= 1e-8 * np.linalg.norm(xe)


@pytest.mark.parametrize("name", CASES)
def test_mixed_precision_reaches_fp64_residual(name):
    import paper_2405_05047_b200 as m
    P, mg, h = setup(name, precision=1)
    F = P.fine
    x = dev(np.zeros(P.n_dof))
    st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(P.b), rtol=1e-10)
    _, ite, _, _ = oracle.gmres(h, P.b, rtol=1e-10)
    assert conv and abs(its - ite) <= 1
    got = host(x)
    bc = oracle.consistent(P.b, F.mean_k)
    r = oracle.residual(F.n, 1, F.row_ptr, F.col, F.val, got, bc)
    assert np.linalg.norm(r) <= 2e-10 * np.linalg.norm(bc)
    assert abs(F.mean_w @ got) <= 1e-13 * np.abs(F.mean_w * got).sum()


def test_update_matrix_rebuilds_regularised_coarse_inverse():
    """mg_update_matrix re-runs the coarse regularisation on the device: the
    updated context equals a fresh build with the new values bit for bit."""
    import copy
    import paper_2405_05047_b200 as m
    P = problem("pres_mid")
    a = build_gpu(P.levels, P.bs, omega=P.omega, H=P.fine.H)
    P2 = copy.deepcopy(P)
    for L in P2.levels:
        L.val = L.val * 3.0
    for l, L in enumerate(P2.levels):
        m.mg_update_matrix(a.ctx, l, np.ascontiguousarray(L.val.reshape(-1)))
    fresh = build_gpu(P2.levels, P2.bs, omega=P2.omega, H=P2.fine.H)
    b = dev(oracle.consistent(P.b, P.fine.mean_k))
    z1, z2 = dev(np.zeros(P.n_dof)), dev(np.zeros(P.n_dof))
    m.mg_vcycle_zero(a.ctx, z1, b)
    m.mg_vcycle_zero(fresh.ctx, z2, b)
    assert np.array_equal(host(z1), host(z2))


def test_constraint_errors_and_removal():
    import paper_2405_05047_b200 as m
    P = problem("pres_small")
    mg = build_gpu(P.levels, P.bs, omega=P.omega)
    F = P.fine
    Lf = len(P.levels) - 1
    m.mg_set_mean_constraint(mg.ctx, Lf, None, None)                    # the levels carried one: remove
    with pytest.raises(m.MgError) as e:
        m.mg_project_zero_mean(mg.ctx, Lf, dev(np.zeros(F.n)))
    assert e.value.status == m.MG_ERR_STATE
    bad = F.mean_w.copy()
    bad[3] = np.nan
    with pytest.raises(m.MgError) as e:
        m.mg_set_mean_constraint(mg.ctx, Lf, bad, F.mean_k)
    assert e.value.status == m.MG_ERR_NONFINITE
    m.mg_set_mean_constraint(mg.ctx, Lf, np.zeros(F.n), F.mean_k)     # w^T k = 0: rejected at setup
    with pytest.raises(m.MgError) as e:
        m.mg_setup(mg.ctx)
    assert e.value.status == m.MG_ERR_INVALID_ARG
    m.mg_set_mean_constraint(mg.ctx, Lf, None, None)                    # removed again
    m.mg_setup(mg.ctx)


def test_distributed_matches_single():
    """Row-partitioned (2 LOCAL ranks): the projections' dots are all-reduced, so
    V-cycles agree to rounding (not bit for bit) and GMRES counts +-1."""
    import paper_2405_05047_b200 as m
    from problems.partition import partition
    P, mg, h = setup("pres_mid")
    parts, extras, ranges = partition(P, 2, min_rows_per_rank=32)
    assert any(not L.replicated for L in parts[0]) and parts[0][-1].mean_w is not None
    key = os.urandom(16)
    Lf = len(P.levels) - 1
    b = oracle.consistent(P.b, P.fine.mean_k)
    out = [None, None]
    errs = []

    def work(r):
        import torch
        torch.cuda.set_device(0)
        try:
            g = build_gpu(parts[r], P.bs, omega=P.omega, H=extras[r][1], comm=(2, r, key, m.MG_TRANSPORT_LOCAL))
            f0, f1 = ranges[-1][r]
            z = dev(np.zeros(f1 - f0))
            m.mg_vcycle_zero(g.ctx, z, dev(b[f0:f1]))
            x = dev(np.zeros(f1 - f0))
            res = m.mg_solve(g.ctx, x, dev(extras[r][0]), rtol=1e-10)
            out[r] = (host(z), host(x), res)
            g.close()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
    th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    if errs:
        raise errs[0]
    z = np.concatenate([o[0] for o in out])
    exp = oracle.vcycle(h, Lf, np.zeros(P.n_dof), b)
    assert np.linalg.norm(z - exp) <= TOL_VCYCLE * np.linalg.norm(exp)
    x = np.concatenate([o[1] for o in out])
    xe, ite, _, _ = oracle.gmres(h, P.b, rtol=1e-10)
    assert out[0][2][3] and abs(out[0][2][1] - ite) <= 1 and out[0][2][1] == out[1][2][1]
    assert np.linalg.norm(x - xe) <= 1e-8 * np.linalg.norm(xe)

