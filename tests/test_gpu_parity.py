"""GPU parity: every step of the hot path through the C
ABI of libmgb200.so against the CPU oracle on the same seeded inputs.

Tolerances (reading Z11): per-op normwise scaled 1e-12
(|A||x| + |b| etc.), whole V-cycle 1e-10 relative in ||.||_2, iteration
counts +-1 at a 1e-10 relative residual.  Integer / layout work is checked
bit-exactly in tests/test_host_logic.py."""
import functools

import numpy as np
import pytest

from gpu_util import (TOL_OP, TOL_VCYCLE, absA_x, assert_close_scaled, build_gpu, build_oracle, dev, host)
from mgtest_util import problem

import oracle

pytestmark = pytest.mark.gpu

FE_CASES = ["c1", "c2_small", "c3_small", "c4_small", "c5_small", "e6_face_l2"]
SYN_CASES = ["syn_bs2", "syn_bs4", "syn_bs3_w1"]


@functools.lru_cache(maxsize=None)
def case(name):
    """(levels, bs, omega, b, H) for an FE config or a synthetic hierarchy."""
    if name.startswith("syn_"):
        from problems.synthetic import random_hierarchy
        if name == "syn_bs2":
            lv, b = random_hierarchy(2, seed_index=11)
        elif name == "syn_bs4":
            lv, b = random_hierarchy(4, seed_index=12)
        else:
            lv, b = random_hierarchy(3, wpe=1, seed_index=13)
        return lv, lv[0].bs, 0.5, b, None
    P = problem(name)
    return P.levels, P.bs, P.omega, P.b, P.fine.H


@functools.lru_cache(maxsize=None)
def gpu_mg(name, coarse_mode=0, use_graphs=True, nu=(2, 2)):
    lv, bs, om, b, H = case(name)
    return build_gpu(lv, bs, omega=om, nu=nu, coarse_mode=coarse_mode, use_graphs=use_graphs, H=H)


@functools.lru_cache(maxsize=None)
def orc_mg(name, coarse="direct", nu=(2, 2)):
    lv, bs, om, b, H = case(name)
    return build_oracle(lv, omega=om, nu=nu, coarse=coarse, H=H)


def rng(seed):
    return np.random.default_rng(1000 + seed)


@pytest.mark.parametrize("name", FE_CASES + SYN_CASES)
def test_residual_and_spmv_every_level(name):
    import paper_2405_05047_b200 as m
    lv, bs, *_ = case(name)
    mg = gpu_mg(name)
    for l, L in enumerate(lv):
        g = rng(l)
        x = g.standard_normal(L.n * bs)
        b = g.standard_normal(L.n * bs)
        y0 = g.standard_normal(L.n * bs)
        r = dev(np.zeros(L.n * bs))
        m.mg_residual(mg.ctx, l, dev(x), dev(b), r)
        exp = oracle.residual(L.n, bs, L.row_ptr, L.col, L.val, x, b)
        assert_close_scaled(host(r), exp, absA_x(L, x) + np.abs(b), what=f"{name} residual l={l}")
        y = dev(y0)
        m.mg_spmv(mg.ctx, l, 1.5, dev(x), -0.5, y)
        exp = oracle.spmv(L.n, bs, L.row_ptr, L.col, L.val, x, 1.5, -0.5, y0)
        assert_close_scaled(host(y), exp, 1.5 * absA_x(L, x) + 0.5 * np.abs(y0), what=f"{name} spmv l={l}")
        y = dev(y0)
        m.mg_spmv(mg.ctx, l, 1.0, dev(x), 0.0, y)       # beta = 0: y not read
        exp = oracle.spmv(L.n, bs, L.row_ptr, L.col, L.val, x)
        assert_close_scaled(host(y), exp, absA_x(L, x), what=f"{name} spmv beta=0 l={l}")


@pytest.mark.parametrize("name", FE_CASES + SYN_CASES)
@pytest.mark.parametrize("sweeps", [1, 2, 3])
def test_smoother_sweeps(name, sweeps):
    import paper_2405_05047_b200 as m
    lv, bs, om, *_ = case(name)
    mg = gpu_mg(name)
    h = orc_mg(name)
    for l, L in enumerate(lv):
        g = rng(10 + l)
        x0 = g.standard_normal(L.n * bs)
        b = g.standard_normal(L.n * bs)
        x = dev(x0)
        m.mg_smooth(mg.ctx, l, x, dev(b), sweeps)
        e = x0
        scale = np.abs(x0)
        for _ in range(sweeps):
            scale = np.abs(e) + om * oracle.spmv(L.n, bs, L.row_ptr, L.col, np.abs(L.val), np.abs(e)) + np.abs(b)
            e = h.smooth(l, e, b)
        assert_close_scaled(host(x), e, scale, tol=TOL_OP * 10 * sweeps, what=f"{name} sweep l={l}")


@pytest.mark.parametrize("name", FE_CASES + SYN_CASES)
def test_restrict_and_prolong(name):
    import paper_2405_05047_b200 as m
    lv, bs, *_ = case(name)
    mg = gpu_mg(name)
    h = orc_mg(name)
    for l in range(1, len(lv)):
        L, C = lv[l], lv[l - 1]
        g = rng(20 + l)
        r = g.standard_normal(L.n * bs)
        d = dev(np.full(C.n * bs, np.nan))               # output fully overwritten
        m.mg_restrict(mg.ctx, l, dev(r), d)
        exp = h.restrict(l, r)
        rrp, rcol, rw = h.levels[l].R
        sc = oracle.transfer(C.n, bs, rrp, rcol, np.abs(rw), L.wpe, np.abs(r))
        assert_close_scaled(host(d), exp, sc, what=f"{name} restrict l={l}")
        y = g.standard_normal(C.n * bs)
        x0 = g.standard_normal(L.n * bs)
        x = dev(x0)
        m.mg_prolong_add(mg.ctx, l, dev(y), x)
        exp = h.prolongate_add(l, x0, y)
        prp, pcol, pw = L.P
        sc = np.abs(x0) + oracle.transfer(L.n, bs, prp, pcol, np.abs(pw), L.wpe, np.abs(y))
        assert_close_scaled(host(x), exp, sc, what=f"{name} prolong l={l}")


@pytest.mark.parametrize("name", FE_CASES + SYN_CASES)
def test_coarse_solve_direct_and_smooth(name):
    import paper_2405_05047_b200 as m
    lv, bs, *_ = case(name)
    L0 = lv[0]
    d = rng(30).standard_normal(L0.n * bs)
    y = dev(np.zeros(L0.n * bs))
    m.mg_coarse_solve(gpu_mg(name).ctx, dev(d), y)
    exp = orc_mg(name).coarse_solve(d)
    # dense inverse vs LU: agree to ~cond(A_0) eps
    A0 = oracle.bsr_to_dense(L0.n, bs, L0.row_ptr, L0.col, L0.val)
    kappa = np.linalg.cond(A0)
    got = host(y)
    assert np.linalg.norm(got - exp) <= 1e-15 * kappa * 50 * np.linalg.norm(exp)
    # paper mode: "several steps of the smoothing iteration"
    y2 = dev(np.zeros(L0.n * bs))
    m.mg_coarse_solve(gpu_mg(name, coarse_mode=1).ctx, dev(d), y2)
    exp2 = orc_mg(name, coarse="smooth").coarse_solve(d)
    assert np.linalg.norm(host(y2) - exp2) <= TOL_VCYCLE * np.linalg.norm(exp2)


@pytest.mark.parametrize("name", FE_CASES + SYN_CASES)
@pytest.mark.parametrize("graphs", [True, False])
def test_vcycle_matches_oracle(name, graphs):
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case(name)
    mg = gpu_mg(name, use_graphs=graphs)
    h = orc_mg(name)
    Lf = len(lv) - 1
    x0 = rng(40).standard_normal(lv[-1].n * bs)
    x = dev(x0)
    bd = dev(b)
    m.mg_vcycle(mg.ctx, x, bd)
    exp = oracle.vcycle(h, Lf, x0.copy(), b)
    assert np.linalg.norm(host(x) - exp) <= TOL_VCYCLE * np.linalg.norm(exp)
    # element-wise as well (every entry, scaled by the largest; the full-size criterion)
    assert np.max(np.abs(host(x) - exp)) <= TOL_VCYCLE * np.max(np.abs(exp))
    # second cycle (graph replay) continues to match
    m.mg_vcycle(mg.ctx, x, bd)
    exp = oracle.vcycle(h, Lf, exp, b)
    assert np.linalg.norm(host(x) - exp) <= TOL_VCYCLE * np.linalg.norm(exp)
    # zero-guess preconditioner form z = GMG(L, 0, v) (A-free first sweep)
    z = dev(np.full(lv[-1].n * bs, np.nan))
    m.mg_vcycle_zero(mg.ctx, z, bd)
    exp = oracle.vcycle(h, Lf, np.zeros_like(b), b)
    assert np.linalg.norm(host(z) - exp) <= TOL_VCYCLE * np.linalg.norm(exp)
    assert np.max(np.abs(host(z) - exp)) <= TOL_VCYCLE * np.max(np.abs(exp))


def test_vcycle_graph_and_eager_bitidentical():
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case("c3_small")
    outs = []
    for graphs in (True, False):
        mg = gpu_mg("c3_small", use_graphs=graphs)
        x = dev(np.zeros(lv[-1].n * bs))
        for _ in range(3):
            m.mg_vcycle(mg.ctx, x, dev(b))
        outs.append(host(x))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("name,nu", [("c2_small", (1, 3)), ("c3_small", (0, 1)), ("c1", (3, 0))])
def test_vcycle_odd_and_zero_sweeps(name, nu):
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case(name)
    mg = gpu_mg(name, nu=nu)
    h = orc_mg(name, nu=nu)
    x0 = rng(41).standard_normal(lv[-1].n * bs)
    x = dev(x0)
    m.mg_vcycle(mg.ctx, x, dev(b))
    exp = oracle.vcycle(h, len(lv) - 1, x0.copy(), b)
    assert np.linalg.norm(host(x) - exp) <= TOL_VCYCLE * np.linalg.norm(exp)
    z = dev(np.zeros(lv[-1].n * bs))
    m.mg_vcycle_zero(mg.ctx, z, dev(b))
    exp = oracle.vcycle(h, len(lv) - 1, np.zeros_like(b), b)
    assert np.linalg.norm(host(z) - exp) <= TOL_VCYCLE * np.linalg.norm(exp)


def test_single_level_hierarchy_is_coarse_solve():
    """n_levels = 1: Alg. gmg Step 0 only."""
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case("c1")
    L0 = lv[0]
    mg = build_gpu([L0], bs, omega=om)
    d = rng(42).standard_normal(L0.n * bs)
    x = dev(np.zeros(L0.n * bs))
    m.mg_vcycle(mg.ctx, x, dev(d))
    A0 = oracle.bsr_to_dense(L0.n, bs, L0.row_ptr, L0.col, L0.val)
    exp = np.linalg.solve(A0, d)
    assert np.linalg.norm(host(x) - exp) <= 1e-12 * np.linalg.cond(A0) * np.linalg.norm(exp)


@pytest.mark.parametrize("name", FE_CASES)
@pytest.mark.parametrize("method", ["gmres", "richardson"])
def test_solve_iteration_counts(name, method):
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case(name)
    mg = gpu_mg(name)
    h = orc_mg(name)
    x = dev(np.zeros(lv[-1].n * bs))
    meth = m.MG_GMRES if method == "gmres" else m.MG_RICHARDSON
    st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(b), method=meth, restart=30, max_iter=200, rtol=1e-10)
    if method == "gmres":
        xe, ite, _, rele = oracle.gmres(h, b, rtol=1e-10, restart=30, max_iter=200)
    else:
        xe, ite, hist = oracle.richardson(h, b, rtol=1e-10, max_iter=200)
        rele = hist[-1] / hist[0]
    assert conv and st == m.MG_OK
    assert abs(its - ite) <= 1, (its, ite)
    assert rel <= 2e-10
    assert np.linalg.norm(host(x) - xe) <= 1e-8 * np.linalg.norm(xe)


def test_gmres_restart_and_maxiter():
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case("c3_small")
    mg = gpu_mg("c3_small")
    h = orc_mg("c3_small")
    x = dev(np.zeros(lv[-1].n * bs))
    st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(b), restart=3, max_iter=200, rtol=1e-10)
    xe, ite, _, _ = oracle.gmres(h, b, rtol=1e-10, restart=3, max_iter=200)
    assert conv and abs(its - ite) <= 1
    x = dev(np.zeros(lv[-1].n * bs))
    st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(b), restart=30, max_iter=2, rtol=1e-14)
    assert st == m.MG_NOT_CONVERGED and its == 2 and not conv and rel < 1.0
    # zero rhs: converged without iterations
    x = dev(np.zeros(lv[-1].n * bs))
    st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(np.zeros_like(b)))
    assert st == m.MG_OK and its == 0 and conv


@pytest.mark.parametrize("restart,max_iter", [(3, 6), (30, 4), (2, 5)])
def test_gmres_truncated_iterate_matches_oracle(restart, max_iter):
    """max_iter truncation and restarts: the GPU iterate after exactly
    max_iter preconditioner applications equals the oracle's, whose GMRES(m) is
    pinned by the minimal-residual property (tests/test_oracle_pins_r2.py)."""
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case("c3_small")
    mg = gpu_mg("c3_small")
    h = orc_mg("c3_small")
    x = dev(np.zeros(lv[-1].n * bs))
    st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(b), restart=restart, max_iter=max_iter, rtol=1e-15)
    xe, ite, _, rele = oracle.gmres(h, b, rtol=1e-15, restart=restart, max_iter=max_iter)
    assert st == m.MG_NOT_CONVERGED and not conv and its == ite == max_iter
    assert np.linalg.norm(host(x) - xe) <= 1e-9 * np.linalg.norm(xe)
    assert abs(rel - rele) <= 1e-6 * rele


def test_gmres_beyond_one_restart_cycle_matches_oracle():
    """A weak preconditioner (V(1,0), coarse problem smoothed twice) so the
    solve needs more than one GMRES(30) cycle; +-1 iterations and x at 1e-8."""
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case("c3_small")
    mg = build_gpu(lv, bs, omega=om, nu=(1, 0), coarse_mode=1, coarse_sweeps=2, H=H)
    h = build_oracle(lv, omega=om, nu=(1, 0), coarse="smooth", coarse_sweeps=2, H=H)
    x = dev(np.zeros(lv[-1].n * bs))
    st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(b), restart=30, max_iter=400, rtol=1e-10)
    xe, ite, _, rele = oracle.gmres(h, b, rtol=1e-10, restart=30, max_iter=400)
    assert ite > 30 and conv and st == m.MG_OK
    assert abs(its - ite) <= 1, (its, ite)
    assert rel <= 1e-10
    assert np.linalg.norm(host(x) - xe) <= 1e-8 * np.linalg.norm(xe)


def test_apply_constraints_and_dot():
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case("c3_small")
    mg = gpu_mg("c3_small")
    x0 = rng(50).standard_normal(lv[-1].n * bs)
    x = dev(x0)
    m.mg_apply_constraints(mg.ctx, x)
    exp = oracle.mg.apply_H(H, x0, bs)
    assert np.array_equal(host(x), exp) or np.max(np.abs(host(x) - exp)) <= TOL_OP * np.max(np.abs(x0))
    a, c = rng(51).standard_normal((2, lv[-1].n * bs))
    d1 = m.mg_dot(mg.ctx, len(lv) - 1, dev(a), dev(c))
    d2 = m.mg_dot(mg.ctx, len(lv) - 1, dev(a), dev(c))
    assert d1 == d2                                                 # deterministic
    assert abs(d1 - oracle.dot(a, c)) <= TOL_OP * np.sum(np.abs(a * c))


def test_error_paths():
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case("c1")
    L = lv[-1]
    ctx = m.mg_create(1, 1)
    try:
        m.mg_create_level(ctx, 0, L.n)
        with pytest.raises(m.MgError) as e:                           # V-cycle before the matrix is set
            m.mg_vcycle(ctx, dev(np.zeros(L.n)), dev(np.zeros(L.n)))
        assert e.value.status == m.MG_ERR_STATE
        bad = L.val.reshape(-1).copy()
        bad[5] = np.nan
        with pytest.raises(m.MgError) as e:
            m.mg_set_matrix(ctx, 0, L.row_ptr, L.col, bad)
        assert e.value.status == m.MG_ERR_NONFINITE
        col = L.col.copy()
        col[[1, 2]] = col[[2, 1]]
        with pytest.raises(m.MgError) as e:
            m.mg_set_matrix(ctx, 0, L.row_ptr, col, L.val.reshape(-1))
        assert e.value.status == m.MG_ERR_STRUCTURE
        m.mg_set_matrix(ctx, 0, L.row_ptr, L.col, L.val.reshape(-1))
        x = dev(np.zeros(L.n))
        with pytest.raises(m.MgError) as e:                           # aliasing
            m.mg_vcycle(ctx, x, x)
        assert e.value.status == m.MG_ERR_INVALID_ARG
        nanb = np.zeros(L.n)
        nanb[3] = np.nan
        with pytest.raises(m.MgError) as e:
            m.mg_solve(ctx, x, dev(nanb))
        assert e.value.status == m.MG_ERR_NONFINITE
        # device-resident inputs are accepted too (mem = DEVICE)
        import torch
        m.mg_set_matrix(ctx, 0, torch.from_numpy(L.row_ptr).cuda(), torch.from_numpy(L.col).cuda(),
                        dev(L.val.reshape(-1)))
        st, its, rel, conv = m.mg_solve(ctx, x, dev(b))
        assert conv and its == 1                                      # exact coarse solve
    finally:
        m.mg_destroy(ctx)
    # singular diagonal block reported when the smoother is built
    val = L.val.copy()
    val[L.row_ptr[4]:L.row_ptr[5]] = 0.0
    ctx = m.mg_create(1, 1, coarse_mode=m.MG_COARSE_SMOOTH)
    try:
        m.mg_create_level(ctx, 0, L.n)
        m.mg_set_matrix(ctx, 0, L.row_ptr, L.col, val.reshape(-1))
        with pytest.raises(m.MgError) as e:
            m.mg_setup(ctx)
        assert e.value.status == m.MG_ERR_SINGULAR
    finally:
        m.mg_destroy(ctx)


def test_user_smoother_override_matches_oracle():
    """mg_set_smoother with explicit D^-1 and per-level omega."""
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case("c2_small")
    mg = gpu_mg("c2_small")
    L = lv[-1]
    Lf = len(lv) - 1
    dinv = oracle.block_diag_inverse(L.n, bs, L.row_ptr, L.col, L.val) * 0.9
    m.mg_set_smoother(mg.ctx, Lf, 0.6, -1, -1, np.ascontiguousarray(dinv.reshape(-1)))
    x0 = rng(60).standard_normal(L.n * bs)
    x = dev(x0)
    m.mg_smooth(mg.ctx, Lf, x, dev(b), 1)
    t = oracle.residual(L.n, bs, L.row_ptr, L.col, L.val, x0, b)
    exp = oracle.jacobi_sweep(L.n, bs, L.row_ptr, L.col, L.val, dinv, 0.6, x0, b)
    sc = np.abs(x0) + 0.6 * np.abs(t)
    assert_close_scaled(host(x), exp, sc + absA_x(L, x0), what="override sweep")
    gpu_mg.cache_clear()


def test_vcycle_profile_split_and_result():
    """mgi_vcycle_profile: per-level split of an eager V-cycle; the result is the
    same V-cycle (bit-identical to the graph-launched one)."""
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case("c3_small")
    mg = gpu_mg("c3_small")
    z1 = dev(np.zeros(lv[-1].n * bs))
    prof = m.vcycle_profile(mg.ctx, z1, dev(b), len(lv))
    z2 = dev(np.zeros(lv[-1].n * bs))
    m.mg_vcycle_zero(mg.ctx, z2, dev(b))
    assert np.array_equal(host(z1), host(z2))
    # levels inside the persistent coarse tail are attributed to the tail's top level
    assert len(prof["level_ms"]) == len(lv) and prof["level_ms"][-1] > 0 and sum(prof["level_ms"]) > 0
    assert all(t == 0 for t in prof["halo_ms"]) and prof["agglomeration_ms"] == 0


@pytest.mark.parametrize("name", ["c2_small", "c3_small", "c4_small"])
def test_condense_rhs_is_HT(name):
    """b_bar = H^T b ("distributing"); hanging entries come out 0."""
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case(name)
    mg = gpu_mg(name)
    F = lv[-1]
    v = rng(70).standard_normal(F.n * bs)
    out = dev(np.full(F.n * bs, np.nan))
    m.mg_condense_rhs(mg.ctx, dev(v), out)
    trp, tcol, tw = oracle.csr_transpose(F.n, F.n, *H)
    exp = oracle.transfer(F.n, bs, trp, tcol, tw, 1, v)
    sc = oracle.transfer(F.n, bs, trp, tcol, np.abs(tw), 1, np.abs(v))
    got = host(out)
    assert_close_scaled(got, exp, sc, what=f"{name} H^T")
    hang = np.diff(H[0]) > 1                       # hanging rows of H hold 2 or 4 master weights
    assert np.all(got.reshape(-1, bs)[hang] == 0.0)  # hanging nodes are never masters: column empty
    # adjoint identity (H^T b, x) = (b, H x) up to rounding
    x0 = rng(71).standard_normal(F.n * bs)
    hx = dev(x0)
    m.mg_apply_constraints(mg.ctx, hx)
    lhs, rhs = float(got @ x0), float(v @ host(hx))
    assert abs(lhs - rhs) <= 1e-12 * (np.abs(got) @ np.abs(x0) + np.abs(v) @ np.abs(host(hx)))


@pytest.mark.parametrize("name", ["c1", "c2_small", "c3_mid", "c5_mid"])
@pytest.mark.parametrize("coarse_mode,precision", [(0, 0), (1, 0), (0, 1)])
def test_coarse_tail_kernel_bitidentical(name, coarse_mode, precision, monkeypatch):
    """The persistent cooperative coarse-tail kernel (levels 0..T in one launch)
    reproduces the standalone kernels bit for bit."""
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case(name)
    outs = []
    for tail in ("1", "c", "0"):                  # grid-barrier tail, cluster tail, standalone kernels
        monkeypatch.setenv("MGB200_TAIL", tail)
        g = build_gpu(lv, bs, omega=om, H=H, coarse_mode=coarse_mode, precision=precision)
        z = dev(np.zeros(lv[-1].n * bs))
        m.mg_vcycle_zero(g.ctx, z, dev(b))
        x = dev(np.zeros(lv[-1].n * bs))
        st, its, rel, conv = m.mg_solve(g.ctx, x, dev(b), rtol=1e-10)
        outs.append((host(z), its, host(x)))
        g.close()
    for o in outs[1:]:
        assert np.array_equal(outs[0][0], o[0])
        assert outs[0][1] == o[1] and np.array_equal(outs[0][2], o[2])


@pytest.mark.parametrize("name", ["c1", "c3_small", "c5_small", "e6_face_l2"])
def test_gmres_device_loop_equals_host_loop(name, monkeypatch):
    """The restart cycle as one conditional graph (while + switch steered by
    k_givens on the device) computes exactly what the per-step host loop
    computes: same iterates bit for bit, same iteration counts."""
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case(name)
    out = []
    for mode in ("host", "device"):
        monkeypatch.setenv("MGB200_GMRES_LOOP", mode)
        mg = build_gpu(lv, bs, omega=om, H=H)
        res = []
        for restart, max_iter, rtol in ((30, 200, 1e-10), (3, 200, 1e-10), (4, 7, 1e-14)):
            x = dev(np.zeros(lv[-1].n * bs))
            st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(b), restart=restart, max_iter=max_iter, rtol=rtol)
            res.append((host(x), its, rel, conv, st))
        out.append(res)
        mg.close()
    for (xh, ih, rh, ch, sh), (xd, idv, rd, cd, sd) in zip(*out):
        assert ih == idv and ch == cd and sh == sd
        assert np.array_equal(xh, xd) and rh == rd


@pytest.mark.parametrize("method", ["mgs", "dcgs2", "richardson"])
def test_solve_from_nonzero_and_zero_guess(method, monkeypatch):
    """A nonzero initial guess takes the full b - A x0 (oracle with the same x0:
    +-1 iterations, x at 1e-8); a zero guess (+0.0 or -0.0) started from r = b
    without the A-pass (MGB200_ZERO_GUESS=1; b - A*0 == b exactly) gives the
    bit-identical iterate of the solve that runs the A-pass (=0)."""
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case("c3_small")
    mg = gpu_mg("c3_small")
    h = orc_mg("c3_small")
    meth = {"mgs": m.MG_GMRES, "dcgs2": m.MG_GMRES_DCGS2, "richardson": m.MG_RICHARDSON}[method]
    x0 = rng(77).standard_normal(lv[-1].n * bs) * 0.3
    x = dev(x0.copy())
    st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(b), method=meth, rtol=1e-10)
    if method == "richardson":
        xe, ite, hist = oracle.richardson(h, b, x0=x0, rtol=1e-10)
    else:
        fn = oracle.gmres if method == "mgs" else oracle.gmres_dcgs2
        xe, ite, _, _ = fn(h, b, x0=x0, rtol=1e-10)
    assert conv and abs(its - ite) <= 1, (its, ite)
    assert np.linalg.norm(host(x) - xe) <= 1e-8 * np.linalg.norm(xe)
    outs = []
    for z, zg in ((0.0, "1"), (-0.0, "1"), (0.0, "0")):
        monkeypatch.setenv("MGB200_ZERO_GUESS", zg)
        x = dev(np.full(lv[-1].n * bs, z))
        st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(b), method=meth, rtol=1e-10)
        outs.append((host(x), its, rel))
    for o in outs[1:]:
        assert np.array_equal(outs[0][0], o[0]) and outs[0][1:] == o[1:]
