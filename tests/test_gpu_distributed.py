"""Multi-GPU path on one B200: the row-partitioned solve with
the LOCAL transport (P virtual ranks = host threads sharing the device; halo
exchange, all-reduced dots and agglomeration go through the same library code
as the NCCL transport, only the copy engine differs).

Each row keeps its CSR summation order after column localisation, R rows are
routed so each lists fine rows ascending, and replicated coarse levels run the
same deterministic kernels -- so the distributed V-cycle must be BIT-IDENTICAL
to the single-GPU V-cycle, and both must match the oracle.  GMRES dots are
all-reduced (sum order differs), so iteration counts are compared +-1."""
import os
import threading

import numpy as np
import pytest

from gpu_util import TOL_OP, TOL_VCYCLE, build_gpu, dev, host
from mgtest_util import problem

import oracle

pytestmark = pytest.mark.gpu


def run_ranks(P, fn):
    res, errs = [None] * P, []

    def work(r):
        import torch
        torch.cuda.set_device(0)
        try:
            res[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            errs.append((r, e))

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if errs:
        raise errs[0][1]
    return res


def dist_mg(name, P, min_rows=32, coarse_mode=0):
    from problems.partition import partition
    import paper_2405_05047_b200 as m
    Pr = problem(name)
    parts, extras, ranges = partition(Pr, P, min_rows_per_rank=min_rows, replicate_level0=(coarse_mode == 0))
    key = os.urandom(16)

    def make(r):
        return build_gpu(parts[r], Pr.bs, omega=Pr.omega, H=extras[r][1], coarse_mode=coarse_mode,
                         comm=(P, r, key, m.MG_TRANSPORT_LOCAL))
    mgs = run_ranks(P, make)
    return Pr, parts, extras, ranges, mgs


def gather(vals, ranges_fine, bs):
    return np.concatenate([v.reshape(-1, bs) for v in vals]).reshape(-1)


CASES = [("c3_small", 2), ("c3_small", 3), ("c2_small", 2), ("c3_mid", 4), ("c4_small", 2), ("c5_mid", 3),
         ("e6_face_l3", 2)]


@pytest.mark.parametrize("name,P", CASES)
def test_partition_has_distributed_and_replicated_levels(name, P):
    from problems.partition import splitters
    Pr = problem(name)
    rg = splitters(Pr, P, min_rows_per_rank=32)
    kinds = ["R" if all(r == (0, Pr.levels[l].n) for r in rg[l]) else "D" for l in range(len(rg))]
    assert kinds[0] == "R" and kinds[-1] == "D"
    for l, k in enumerate(kinds):
        if k == "D":
            b = [r[0] for r in rg[l]] + [rg[l][-1][1]]
            assert b[0] == 0 and b[-1] == Pr.levels[l].n and all(np.diff(b) >= 0)


@pytest.mark.parametrize("name,P", CASES)
def test_distributed_vcycle_bitwise_equals_single_gpu(name, P):
    import paper_2405_05047_b200 as m
    Pr, parts, extras, ranges, mgs = dist_mg(name, P)
    bs = Pr.bs
    x0 = np.random.default_rng(5).standard_normal(Pr.n_dof)
    # single GPU reference
    s = build_gpu(Pr.levels, bs, omega=Pr.omega, H=Pr.fine.H)
    xs = dev(x0)
    m.mg_vcycle(s.ctx, xs, dev(Pr.b))
    zs = dev(np.zeros(Pr.n_dof))
    m.mg_vcycle_zero(s.ctx, zs, dev(Pr.b))
    ref, refz = host(xs), host(zs)
    fr = ranges[-1]

    def cyc(r):
        f0, f1 = fr[r]
        x = dev(x0.reshape(-1, bs)[f0:f1].reshape(-1))
        b = dev(extras[r][0])
        m.mg_vcycle(mgs[r].ctx, x, b)
        z = dev(np.zeros((f1 - f0) * bs))
        m.mg_vcycle_zero(mgs[r].ctx, z, b)
        return host(x), host(z)
    out = run_ranks(P, cyc)
    got = np.concatenate([o[0] for o in out])
    gotz = np.concatenate([o[1] for o in out])
    assert np.array_equal(got, ref), f"max diff {np.max(np.abs(got - ref)):.3e}"
    assert np.array_equal(gotz, refz)
    h = oracle.MgHierarchy.from_arrays(Pr.levels, omega=Pr.omega)
    exp = oracle.vcycle(h, len(Pr.levels) - 1, x0.copy(), Pr.b)
    assert np.linalg.norm(got - exp) <= TOL_VCYCLE * np.linalg.norm(exp)
    for g in mgs:
        g.close()


@pytest.mark.parametrize("name,P", [("c3_small", 2), ("c2_small", 3), ("c4_small", 2)])
def test_distributed_per_op(name, P):
    import paper_2405_05047_b200 as m
    Pr, parts, extras, ranges, mgs = dist_mg(name, P)
    bs = Pr.bs
    Lf = len(Pr.levels) - 1
    g = np.random.default_rng(9)
    xs = [g.standard_normal(L.n * bs) for L in Pr.levels]
    bb = [g.standard_normal(L.n * bs) for L in Pr.levels]

    def sl(v, l, r):
        a, b = ranges[l][r]
        return v.reshape(-1, bs)[a:b].reshape(-1)

    def ops(r):
        res = {}
        for l in range(len(Pr.levels)):
            n = ranges[l][r][1] - ranges[l][r][0]
            x, b = dev(sl(xs[l], l, r)), dev(sl(bb[l], l, r))
            rr = dev(np.zeros(n * bs))
            m.mg_residual(mgs[r].ctx, l, x, b, rr)
            sw = dev(np.zeros(n * bs))
            m.mg_sweep(mgs[r].ctx, l, x, b, sw)
            res[("resid", l)] = host(rr)
            res[("sweep", l)] = host(sw)
            res[("dot", l)] = m.mg_dot(mgs[r].ctx, l, x, b)
            if l > 0:
                nc = ranges[l - 1][r][1] - ranges[l - 1][r][0]
                d = dev(np.zeros(Pr.levels[l - 1].n * bs))       # room for a replicated coarse level
                m.mg_restrict(mgs[r].ctx, l, x, d)
                res[("restrict", l)] = host(d)[:nc * bs] if nc != Pr.levels[l - 1].n else host(d)
                y = dev(sl(xs[l - 1], l - 1, r))
                xp = dev(sl(bb[l], l, r))
                m.mg_prolong_add(mgs[r].ctx, l, y, xp)
                res[("prolong", l)] = host(xp)
        hx = dev(sl(xs[Lf], Lf, r))
        m.mg_apply_constraints(mgs[r].ctx, hx)
        res["H"] = host(hx)
        ht = dev(np.zeros(len(sl(xs[Lf], Lf, r))))
        m.mg_condense_rhs(mgs[r].ctx, dev(sl(bb[Lf], Lf, r)), ht)
        res["HT"] = host(ht)
        return res
    out = run_ranks(P, ops)
    s = build_gpu(Pr.levels, bs, omega=Pr.omega, H=Pr.fine.H)
    for l, L in enumerate(Pr.levels):
        rep = all(rg == (0, L.n) for rg in ranges[l])
        cat = (lambda k: out[0][k]) if rep else (lambda k: np.concatenate([o[k] for o in out]))
        r1 = dev(np.zeros(L.n * bs))
        m.mg_residual(s.ctx, l, dev(xs[l]), dev(bb[l]), r1)
        assert np.array_equal(cat(("resid", l)), host(r1))
        m.mg_sweep(s.ctx, l, dev(xs[l]), dev(bb[l]), r1)
        assert np.array_equal(cat(("sweep", l)), host(r1))
        d1 = m.mg_dot(s.ctx, l, dev(xs[l]), dev(bb[l]))
        for o in out:
            assert abs(o[("dot", l)] - d1) <= TOL_OP * np.sum(np.abs(xs[l] * bb[l]))
        if l > 0:
            C = Pr.levels[l - 1]
            d = dev(np.zeros(C.n * bs))
            m.mg_restrict(s.ctx, l, dev(xs[l]), d)
            crep = all(rg == (0, C.n) for rg in ranges[l - 1])
            got = out[0][("restrict", l)] if crep else np.concatenate([o[("restrict", l)] for o in out])
            assert np.array_equal(got, host(d))
            xp = dev(bb[l])
            m.mg_prolong_add(s.ctx, l, dev(xs[l - 1]), xp)
            assert np.array_equal(cat(("prolong", l)), host(xp))
    hx = dev(xs[Lf])
    m.mg_apply_constraints(s.ctx, hx)
    assert np.array_equal(np.concatenate([o["H"] for o in out]), host(hx))
    ht = dev(np.zeros(Pr.n_dof))
    m.mg_condense_rhs(s.ctx, dev(bb[Lf]), ht)
    assert np.array_equal(np.concatenate([o["HT"] for o in out]), host(ht))


@pytest.mark.parametrize("name,P", [("c3_small", 2), ("c3_mid", 4), ("c2_small", 3), ("c5_mid", 2)])
def test_distributed_gmres_matches(name, P):
    import paper_2405_05047_b200 as m
    Pr, parts, extras, ranges, mgs = dist_mg(name, P)
    bs = Pr.bs
    s = build_gpu(Pr.levels, bs, omega=Pr.omega, H=Pr.fine.H)
    x1 = dev(np.zeros(Pr.n_dof))
    st, its1, rel1, conv1 = m.mg_solve(s.ctx, x1, dev(Pr.b), rtol=1e-10)
    fr = ranges[-1]

    def solve(r):
        f0, f1 = fr[r]
        x = dev(np.zeros((f1 - f0) * bs))
        out = m.mg_solve(mgs[r].ctx, x, dev(extras[r][0]), rtol=1e-10)
        m.mg_apply_constraints(mgs[r].ctx, x)
        return out, host(x)
    out = run_ranks(P, solve)
    its = {o[0][1] for o in out}
    assert len(its) == 1                                   # all ranks take identical decisions
    it = its.pop()
    assert abs(it - its1) <= 1 and all(o[0][3] for o in out)
    x = np.concatenate([o[1] for o in out])
    m.mg_apply_constraints(s.ctx, x1)
    xr = host(x1)
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)


def test_distributed_coarse_smoothing_mode():
    """coarse_mode = smooth: level 0 may stay distributed (sweeps with halos)."""
    import paper_2405_05047_b200 as m
    Pr, parts, extras, ranges, mgs = dist_mg("c3_mid", 2, min_rows=8, coarse_mode=1)
    assert not all(rg == (0, Pr.levels[0].n) for rg in ranges[0])
    s = build_gpu(Pr.levels, Pr.bs, omega=Pr.omega, H=Pr.fine.H, coarse_mode=1)
    z1 = dev(np.zeros(Pr.n_dof))
    m.mg_vcycle_zero(s.ctx, z1, dev(Pr.b))
    fr = ranges[-1]

    def cyc(r):
        f0, f1 = fr[r]
        z = dev(np.zeros((f1 - f0) * Pr.bs))
        m.mg_vcycle_zero(mgs[r].ctx, z, dev(extras[r][0]))
        return host(z)
    got = np.concatenate(run_ranks(2, cyc))
    assert np.array_equal(got, host(z1))


@pytest.mark.parametrize("overlap", ["1", "0"])
def test_distributed_mixed_precision_and_overlap(overlap, monkeypatch):
    """Row-partitioned mixed-precision V-cycle and GMRES, with and without the
    halo / interior overlap (interior and boundary parts): bit-identical V-cycle
    to the single-GPU mixed solver."""
    import paper_2405_05047_b200 as m
    from problems.partition import partition
    monkeypatch.setenv("MGB200_OVERLAP", overlap)
    Pr = problem("c3_mid")
    parts, extras, ranges = partition(Pr, 3, min_rows_per_rank=32)
    key = os.urandom(16)
    mgs = run_ranks(3, lambda r: build_gpu(parts[r], Pr.bs, omega=Pr.omega, H=extras[r][1],
                                           precision=m.MG_PREC_MIXED, comm=(3, r, key, m.MG_TRANSPORT_LOCAL)))
    s = build_gpu(Pr.levels, Pr.bs, omega=Pr.omega, H=Pr.fine.H, precision=m.MG_PREC_MIXED)
    z = dev(np.zeros(Pr.n_dof))
    m.mg_vcycle_zero(s.ctx, z, dev(Pr.b))
    x1 = dev(np.zeros(Pr.n_dof))
    _, its1, _, _ = m.mg_solve(s.ctx, x1, dev(Pr.b), rtol=1e-10)
    fr = ranges[-1]

    def work(r):
        f0, f1 = fr[r]
        zz = dev(np.zeros((f1 - f0) * Pr.bs))
        m.mg_vcycle_zero(mgs[r].ctx, zz, dev(extras[r][0]))
        xx = dev(np.zeros((f1 - f0) * Pr.bs))
        out = m.mg_solve(mgs[r].ctx, xx, dev(extras[r][0]), rtol=1e-10)
        return host(zz), out
    out = run_ranks(3, work)
    assert np.array_equal(np.concatenate([o[0] for o in out]), host(z))
    assert all(o[1][3] for o in out) and abs(out[0][1][1] - its1) <= 1
    for g in mgs:
        g.close()


def test_distributed_rank_without_rows():
    """Edge case: rank 1 owns no rows of a distributed level (NULL vectors from
    empty tensors); the V-cycle stays bit-identical and GMRES matches."""
    import paper_2405_05047_b200 as m
    from problems.partition import partition
    Pr = problem("c3_small")                        # levels [125, 455, 2925]
    n0, n1, n2 = (L.n for L in Pr.levels)
    ranges = [[(0, n0), (0, n0)], [(0, n1), (n1, n1)], [(0, 1400), (1400, n2)]]
    parts, extras, _ = partition(Pr, 2, ranges=ranges)
    key = os.urandom(16)
    mgs = run_ranks(2, lambda r: build_gpu(parts[r], Pr.bs, omega=Pr.omega, H=extras[r][1],
                                           comm=(2, r, key, m.MG_TRANSPORT_LOCAL)))
    s = build_gpu(Pr.levels, Pr.bs, omega=Pr.omega, H=Pr.fine.H)
    z = dev(np.zeros(Pr.n_dof))
    m.mg_vcycle_zero(s.ctx, z, dev(Pr.b))
    _, its1, _, _ = m.mg_solve(s.ctx, dev(np.zeros(Pr.n_dof)), dev(Pr.b), rtol=1e-10)

    def work(r):
        f0, f1 = ranges[-1][r]
        zz = dev(np.zeros((f1 - f0) * Pr.bs))
        m.mg_vcycle_zero(mgs[r].ctx, zz, dev(extras[r][0]))
        # per-op calls on the level this rank owns no rows of: empty (NULL) vectors
        e = dev(np.zeros((ranges[1][r][1] - ranges[1][r][0]) * Pr.bs))
        e2 = dev(np.zeros_like(host(e)))
        m.mg_residual(mgs[r].ctx, 1, e, e2, dev(np.zeros_like(host(e))))
        out = m.mg_solve(mgs[r].ctx, dev(np.zeros((f1 - f0) * Pr.bs)), dev(extras[r][0]), rtol=1e-10)
        return host(zz), out
    out = run_ranks(2, work)
    assert np.array_equal(np.concatenate([o[0] for o in out]), host(z))
    assert all(o[1][3] for o in out) and abs(out[0][1][1] - its1) <= 1


@pytest.mark.parametrize("name,P", [("c3_small", 2), ("c2_small", 3)])
def test_distributed_zero_guess_shortcut(name, P, monkeypatch):
    """The zero-guess test is all-reduced across ranks: with it forced on
    (MGB200_ZERO_GUESS=1) every rank starts from r = b and the solve is bit-identical
    to the one that runs the distributed A-pass (=0)."""
    import paper_2405_05047_b200 as m
    Pr, parts, extras, ranges, mgs = dist_mg(name, P)
    fr = ranges[-1]
    res = []
    for zg in ("1", "0"):
        monkeypatch.setenv("MGB200_ZERO_GUESS", zg)

        def solve(r):
            f0, f1 = fr[r]
            x = dev(np.zeros((f1 - f0) * Pr.bs))
            out = m.mg_solve(mgs[r].ctx, x, dev(extras[r][0]), rtol=1e-10)
            return out, host(x)
        res.append(run_ranks(P, solve))
    for (o1, x1), (o0, x0) in zip(*res):
        assert o1 == o0 and np.array_equal(x1, x0)
