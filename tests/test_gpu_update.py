"""mg_update_matrix: value-only re-upload (the Newton / time-step re-upload of
P:821).  After updating every level to the operator of a different
time step on the same mesh, V-cycles and GMRES must be BIT-IDENTICAL to a
context built from scratch with the new values (the device scatter, the device
D^-1 and the device coarse Gauss-Jordan are the setup path's own kernels), in
fp64 and mixed precision, single GPU and row-partitioned."""
import copy
import os

import numpy as np
import pytest

from gpu_util import build_gpu, dev, host

from problems import configs

pytestmark = pytest.mark.gpu


def retimed(name, factor):
    """Same mesh/hierarchy, operator of a different time step (new values)."""
    root, box, steps, op, omega, si = configs.CONFIGS[name]
    op2 = copy.deepcopy(op)
    op2.params["dt"] = op.params["dt"] * factor
    kw = {"g_fun": configs.lid(len(root), op.bs)} if op.name == "stokes" else {}
    return configs.make_problem(name, root, box, steps, op2, seed_index=si, omega=omega, **kw)


@pytest.mark.parametrize("name", ["c2_small", "c3_small", "c4_small", "c5_small"])
@pytest.mark.parametrize("precision", [0, 1])
def test_update_matches_fresh_build(name, precision):
    import paper_2405_05047_b200 as m
    P0 = configs.build(name)
    P1 = retimed(name, 1.7)
    for l in range(len(P0.levels)):
        assert np.array_equal(P0.levels[l].row_ptr, P1.levels[l].row_ptr)
        assert np.array_equal(P0.levels[l].col, P1.levels[l].col)
        assert not np.array_equal(P0.levels[l].val, P1.levels[l].val)
    a = build_gpu(P0.levels, P0.bs, omega=P0.omega, H=P0.fine.H, precision=precision)
    b = dev(P1.b)
    z = dev(np.zeros(P0.n_dof))
    m.mg_vcycle_zero(a.ctx, z, b)                       # capture graphs with the old values
    for l, L in enumerate(P1.levels):
        vals = L.val.reshape(-1)
        m.mg_update_matrix(a.ctx, l, dev(vals) if l % 2 else np.ascontiguousarray(vals))   # device and host inputs
    fresh = build_gpu(P1.levels, P1.bs, omega=P1.omega, H=P1.fine.H, precision=precision)
    z1, z2 = dev(np.zeros(P0.n_dof)), dev(np.zeros(P0.n_dof))
    m.mg_vcycle_zero(a.ctx, z1, b)                      # replayed graph, new values
    m.mg_vcycle_zero(fresh.ctx, z2, b)
    assert np.array_equal(host(z1), host(z2))
    x1, x2 = dev(np.zeros(P0.n_dof)), dev(np.zeros(P0.n_dof))
    r1 = m.mg_solve(a.ctx, x1, b, rtol=1e-10)
    r2 = m.mg_solve(fresh.ctx, x2, b, rtol=1e-10)
    assert r1[1] == r2[1] and np.array_equal(host(x1), host(x2))
    # the context really changed operator: old and new solutions differ
    a0 = build_gpu(P0.levels, P0.bs, omega=P0.omega, H=P0.fine.H, precision=precision)
    x0 = dev(np.zeros(P0.n_dof))
    m.mg_solve(a0.ctx, x0, b, rtol=1e-10)
    assert not np.allclose(host(x0), host(x1))


def test_update_errors():
    import paper_2405_05047_b200 as m
    P = configs.build("c3_small")
    a = build_gpu(P.levels, P.bs, omega=P.omega, H=P.fine.H)
    bad = P.fine.val.reshape(-1).copy()
    bad[7] = np.inf
    with pytest.raises(m.MgError) as e:
        m.mg_update_matrix(a.ctx, len(P.levels) - 1, bad)
    assert e.value.status == m.MG_ERR_NONFINITE
    sing = P.levels[0].val.copy()
    rp = P.levels[0].row_ptr
    for k in range(rp[3], rp[4]):
        if P.levels[0].col[k] == 3:
            sing[k] = 0.0
    with pytest.raises(m.MgError) as e:
        m.mg_update_matrix(a.ctx, 0, sing.reshape(-1))
    assert e.value.status == m.MG_ERR_SINGULAR
    ctx = m.mg_create(1, P.bs)
    m.mg_create_level(ctx, 0, P.levels[0].n)
    with pytest.raises(m.MgError) as e:
        m.mg_update_matrix(ctx, 0, P.levels[0].val.reshape(-1))
    assert e.value.status == m.MG_ERR_STATE
    m.mg_destroy(ctx)


def test_update_distributed_matches_single():
    import threading
    import paper_2405_05047_b200 as m
    from problems.partition import partition
    P0 = configs.build("c3_mid")
    P1 = retimed("c3_mid", 0.6)
    parts0, extras0, ranges = partition(P0, 2, min_rows_per_rank=32)
    parts1, extras1, _ = partition(P1, 2, min_rows_per_rank=32)
    key = os.urandom(16)
    out = [None, None]

    def work(r):
        import torch
        torch.cuda.set_device(0)
        g = build_gpu(parts0[r], P0.bs, omega=P0.omega, H=extras0[r][1], comm=(2, r, key, m.MG_TRANSPORT_LOCAL))
        for l, L in enumerate(parts1[r]):
            m.mg_update_matrix(g.ctx, l, np.ascontiguousarray(L.val.reshape(-1)))
        z = dev(np.zeros(len(extras1[r][0])))
        m.mg_vcycle_zero(g.ctx, z, dev(extras1[r][0]))
        out[r] = host(z)
        g.close()
    th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    fresh = build_gpu(P1.levels, P1.bs, omega=P1.omega, H=P1.fine.H)
    z = dev(np.zeros(P1.n_dof))
    m.mg_vcycle_zero(fresh.ctx, z, dev(P1.b))
    assert np.array_equal(np.concatenate(out), host(z))
