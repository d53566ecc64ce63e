"""GPU parity of GMRES with delayed CGS2 reorthogonalisation (MG_GMRES_DCGS2,
reading Z29) against the oracle's `gmres_dcgs2` -- itself pinned by the
minimal-residual property of GMRES (tests/test_oracle_dcgs2.py) -- and against
the paper's MGS GMRES (same Krylov spaces): iteration counts +-1 at 1e-10,
iterates to 1e-8, truncated iterates to 1e-9; the conditional-graph restart
cycle bit-identical to the per-step host loop; the distributed path (LOCAL
ranks) bit-identical to the single-GPU solve."""
import numpy as np
import pytest

from gpu_util import build_gpu, build_oracle, dev, host
from test_gpu_parity import FE_CASES, case, gpu_mg, orc_mg

import oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", FE_CASES)
def test_dcgs2_iterations_and_solution(name):
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case(name)
    mg = gpu_mg(name)
    h = orc_mg(name)
    x = dev(np.zeros(lv[-1].n * bs))
    st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(b), method=m.MG_GMRES_DCGS2, restart=30, max_iter=200,
                                    rtol=1e-10)
    xe, ite, _, _ = oracle.gmres_dcgs2(h, b, rtol=1e-10, restart=30, max_iter=200)
    _, ite_mgs, _, _ = oracle.gmres(h, b, rtol=1e-10, restart=30, max_iter=200)
    assert conv and st == m.MG_OK and rel <= 1e-10
    assert abs(its - ite) <= 1 and abs(its - ite_mgs) <= 1, (its, ite, ite_mgs)
    assert np.linalg.norm(host(x) - xe) <= 1e-8 * np.linalg.norm(xe)


@pytest.mark.parametrize("restart,max_iter", [(3, 6), (30, 4), (2, 5), (30, 7)])
def test_dcgs2_truncated_iterate_matches_oracle(restart, max_iter):
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case("c3_small")
    mg = gpu_mg("c3_small")
    h = orc_mg("c3_small")
    x = dev(np.zeros(lv[-1].n * bs))
    st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(b), method=m.MG_GMRES_DCGS2, restart=restart,
                                    max_iter=max_iter, rtol=1e-15)
    xe, ite, _, rele = oracle.gmres_dcgs2(h, b, rtol=1e-15, restart=restart, max_iter=max_iter)
    assert st == m.MG_NOT_CONVERGED and not conv and its == ite == max_iter
    assert np.linalg.norm(host(x) - xe) <= 1e-9 * np.linalg.norm(xe)
    assert abs(rel - rele) <= 1e-6 * rele


def test_dcgs2_beyond_one_restart_cycle():
    """m = 30 basis vectors (the JB = 32 kernels) and a restart."""
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case("c3_small")
    mg = build_gpu(lv, bs, omega=om, nu=(1, 0), coarse_mode=1, coarse_sweeps=2, H=H)
    h = build_oracle(lv, omega=om, nu=(1, 0), coarse="smooth", coarse_sweeps=2, H=H)
    x = dev(np.zeros(lv[-1].n * bs))
    st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(b), method=m.MG_GMRES_DCGS2, restart=30, max_iter=400,
                                    rtol=1e-10)
    xe, ite, _, _ = oracle.gmres_dcgs2(h, b, rtol=1e-10, restart=30, max_iter=400)
    assert ite > 30 and conv and st == m.MG_OK and rel <= 1e-10
    assert abs(its - ite) <= 1, (its, ite)
    assert np.linalg.norm(host(x) - xe) <= 1e-8 * np.linalg.norm(xe)
    mg.close()


@pytest.mark.parametrize("name", ["c1", "c3_small", "e6_face_l2"])
def test_dcgs2_device_loop_equals_host_loop(name, monkeypatch):
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case(name)
    out = []
    for mode in ("host", "device"):
        monkeypatch.setenv("MGB200_GMRES_LOOP", mode)
        mg = build_gpu(lv, bs, omega=om, H=H)
        res = []
        for restart, max_iter, rtol in ((30, 200, 1e-10), (3, 200, 1e-10), (4, 7, 1e-14)):
            x = dev(np.zeros(lv[-1].n * bs))
            st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(b), method=m.MG_GMRES_DCGS2, restart=restart,
                                            max_iter=max_iter, rtol=rtol)
            res.append((host(x), its, rel, conv, st))
        out.append(res)
        mg.close()
    for (xh, ih, rh, ch, sh), (xd, idv, rd, cd, sd) in zip(*out):
        assert ih == idv and ch == cd and sh == sd
        assert np.array_equal(xh, xd) and rh == rd


def test_dcgs2_zero_rhs_and_graph_keys():
    """zero rhs converges without iterations; MGS and DCGS2 solves alternate on
    one context (separate cycle graphs) and each reproduces itself exactly."""
    import paper_2405_05047_b200 as m
    lv, bs, om, b, H = case("c2_small")
    mg = gpu_mg("c2_small")
    x = dev(np.zeros(lv[-1].n * bs))
    st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(np.zeros_like(b)), method=m.MG_GMRES_DCGS2)
    assert st == m.MG_OK and its == 0 and conv
    res = {}
    for meth in (m.MG_GMRES_DCGS2, m.MG_GMRES, m.MG_GMRES_DCGS2, m.MG_GMRES):
        x = dev(np.zeros(lv[-1].n * bs))
        st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(b), method=meth)
        r = (host(x), its)
        if meth in res:
            assert np.array_equal(res[meth][0], r[0]) and res[meth][1] == r[1]
        res[meth] = r
    assert abs(res[m.MG_GMRES][1] - res[m.MG_GMRES_DCGS2][1]) <= 1


@pytest.mark.parametrize("name,P", [("c3_small", 2), ("c3_mid", 4)])
def test_dcgs2_distributed_matches_single(name, P):
    """Row-partitioned DCGS2 (LOCAL ranks: one multi-dot all-reduce of 2j + 2
    values and one 1-value all-reduce per Arnoldi step): every rank takes the
    same decisions, +-1 iterations and x to 1e-8 against the single-GPU solve."""
    import paper_2405_05047_b200 as m
    from test_gpu_distributed import dist_mg, run_ranks
    Pr, parts, extras, ranges, mgs = dist_mg(name, P)
    bs = Pr.bs
    s = build_gpu(Pr.levels, bs, omega=Pr.omega, H=Pr.fine.H)
    x1 = dev(np.zeros(Pr.n_dof))
    st, its1, rel1, conv1 = m.mg_solve(s.ctx, x1, dev(Pr.b), method=m.MG_GMRES_DCGS2, rtol=1e-10)
    fr = ranges[-1]

    def solve(r):
        f0, f1 = fr[r]
        x = dev(np.zeros((f1 - f0) * bs))
        out = m.mg_solve(mgs[r].ctx, x, dev(extras[r][0]), method=m.MG_GMRES_DCGS2, rtol=1e-10)
        return out, host(x)
    out = run_ranks(P, solve)
    its = {o[0][1] for o in out}
    assert len(its) == 1 and conv1
    assert abs(its.pop() - its1) <= 1 and all(o[0][3] for o in out)
    x = np.concatenate([o[1] for o in out])
    xr = host(x1)
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)


@pytest.mark.parametrize("kernel", ["auto", "reg", "ws", "tma"])
def test_dcgs2_kernel_variants(kernel, monkeypatch):
    """The three implementations of the DCGS2 passes (per-thread accumulators,
    warp-split, bulk-copy ring; MGB200_DCGS_KERNEL) reach the oracle's iterate:
    +-1 iterations and x to 1e-8, a solve beyond j = 8 and a restart."""
    import paper_2405_05047_b200 as m
    if kernel != "auto":
        monkeypatch.setenv("MGB200_DCGS_KERNEL", kernel)
    lv, bs, om, b, H = case("c3_small")
    h = orc_mg("c3_small")
    mg = build_gpu(lv, bs, omega=om, H=H)
    for restart in (30, 11):
        x = dev(np.zeros(lv[-1].n * bs))
        st, its, rel, conv = m.mg_solve(mg.ctx, x, dev(b), method=m.MG_GMRES_DCGS2, restart=restart, rtol=1e-10)
        xe, ite, _, _ = oracle.gmres_dcgs2(h, b, rtol=1e-10, restart=restart)
        assert conv and abs(its - ite) <= 1 and its > 8, (its, ite)
        assert np.linalg.norm(host(x) - xe) <= 1e-8 * np.linalg.norm(xe)
    mg.close()
