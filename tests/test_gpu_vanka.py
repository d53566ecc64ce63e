"""GPU parity of the Vanka-type patch smoother (mg_set_vanka)
against the oracle's vanka_sweep on the same generated systems, patches = the
cells of each level's mesh (m = 2^d * bs unknowns: 4 .. 32).

Tolerance: the device inverts each A_pp by Gauss-Jordan with partial pivoting,
the oracle by LAPACK, so a sweep agrees to ~kappa(A_pp) * eps times the
magnitude of the computation (reading Z11 extended):
  |x_gpu - x_orc| <= 64 eps max_p kappa(A_pp) * max(|x| + omega W |A_pp^-1| (|b| + |A||x|)).
Whole V-cycles 1e-9 relative, GMRES iteration counts +-1; mg_update_matrix
rebuilds the patch inverses bit-identically to a fresh context."""
import functools

import numpy as np
import pytest

from gpu_util import absA_x, dev, host

import oracle
from oracle.mg import vanka_setup, vanka_sweep
from problems import channel as CH
from problems import configs

pytestmark = pytest.mark.gpu

EPS = np.finfo(np.float64).eps


@functools.lru_cache(maxsize=None)
def cfg(name):
    return configs.build(name)


@functools.lru_cache(maxsize=None)
def channel(name):
    P = CH.build(name)
    u = CH.initial_state(P)
    rng = np.random.default_rng(11)
    w = CH.full_field(P, u + 0.2 * rng.standard_normal(u.shape) * (~P.fine.cmask))
    return P, CH.with_values(P, CH.jacobians(P, w, u)), -CH.residual(P, w, u)


def case(name):
    if name.startswith("c4ns"):
        P, levels, b = channel(name)
        return levels, 3, P.omega, b
    P = cfg(name)
    return P.levels, P.bs, P.omega, P.b


def gpu(levels, bs, omega, **kw):
    from paper_2405_05047_b200 import Multigrid
    return Multigrid(levels, bs, omega=omega, vanka=True, **kw)


@pytest.mark.parametrize("name", ["c2_small", "c3_small", "c5_small", "c4ns_small", "c4ns_mid"])
def test_vanka_sweep_matches_oracle(name):
    import paper_2405_05047_b200 as m
    levels, bs, omega, _ = case(name)
    g = gpu(levels, bs, omega)
    rng = np.random.default_rng(5)
    for l in (len(levels) - 1, 1):
        L = levels[l]
        lv = oracle.mg.MgLevel(L.n, bs, L.row_ptr, L.col, np.asarray(L.val, np.float64))
        vk = vanka_setup(lv, L.patches)
        N = L.n * bs
        x, b = rng.standard_normal(N), rng.standard_normal(N)
        out = dev(np.zeros(N))
        m.mg_sweep(g.ctx, l, dev(x), dev(b), out)
        got = host(out)
        exp = vanka_sweep(lv, vk, omega, x, b)
        patches, inv, w = vk
        ra = (np.abs(b) + absA_x(L, x)).reshape(-1, bs)[patches].reshape(len(patches), -1)
        acc = np.zeros((L.n, bs))
        np.add.at(acc, patches.ravel(), np.einsum("pij,pj->pi", np.abs(inv), ra).reshape(-1, bs))
        scale = np.abs(x) + omega * (w[:, None] * acc).reshape(-1)
        kappa = max(np.linalg.cond(inv[q]) for q in range(0, len(inv), max(1, len(inv) // 200)))
        err = np.abs(got - exp).max()
        assert err <= 64 * EPS * kappa * scale.max(), (name, l, err, kappa, scale.max())
    g.close()


@pytest.mark.parametrize("name", ["c3_small", "c4ns_mid", "c5_small"])
def test_vanka_vcycle_and_gmres_match_oracle(name):
    levels, bs, omega, b = case(name)
    g = gpu(levels, bs, omega)
    h = oracle.MgHierarchy.from_arrays(levels, omega=omega, vanka=True)
    rng = np.random.default_rng(7)
    x0 = rng.standard_normal(len(b))
    x = dev(x0)
    g.vcycle(x, dev(b))
    exp = oracle.vcycle(h, len(levels) - 1, x0, b)
    assert np.linalg.norm(host(x) - exp) <= 1e-9 * np.linalg.norm(exp)
    x = dev(np.zeros(len(b)))
    st, its, rel, conv = g.solve(x, dev(b), rtol=1e-10)
    _, its_o, _, rel_o = oracle.gmres(h, b, rtol=1e-10)
    assert conv and abs(its - its_o) <= 1, (its, its_o)
    g.close()


def test_vanka_update_matrix_rebuilds_inverses():
    import paper_2405_05047_b200 as m
    P, levels, b = channel("c4ns_mid")
    u = CH.initial_state(P)
    vals2 = CH.jacobians(P, CH.full_field(P, u + 0.5 * (~P.fine.cmask)), u)
    levels2 = CH.with_values(P, vals2)
    a = gpu(levels, 3, P.omega)
    for l, v in enumerate(vals2):
        m.mg_update_matrix(a.ctx, l, np.ascontiguousarray(v.reshape(-1)))
    f = gpu(levels2, 3, P.omega)
    bd = dev(b)
    xa, xf = dev(np.zeros(len(b))), dev(np.zeros(len(b)))
    a.vcycle(xa, bd)
    f.vcycle(xf, bd)
    assert np.array_equal(host(xa), host(xf))
    a.close()
    f.close()


def test_vanka_errors_and_switch_back():
    import paper_2405_05047_b200 as m
    levels, bs, omega, b = case("c4ns_small")
    g = gpu(levels, bs, omega)
    L = len(levels) - 1
    with pytest.raises(m.MgError):
        m.mg_set_vanka(g.ctx, L, np.array([[0, 0, 1, 2]]))          # repeated node
    with pytest.raises(m.MgError):
        m.mg_set_vanka(g.ctx, L, np.array([[0, 1, 2, 3]]))          # rows not covered
    with pytest.raises(m.MgError):
        m.mg_set_vanka(g.ctx, L, np.arange(22).reshape(2, 11))      # 11 * 3 > 32 unknowns
    m.mg_set_vanka(g.ctx, L, None)                                  # back to block-Jacobi on the finest level
    h = oracle.MgHierarchy.from_arrays(levels, omega=omega, vanka=True)
    h.levels[-1].vanka = None
    x = dev(np.zeros(len(b)))
    g.vcycle(x, dev(b))
    exp = oracle.vcycle(h, L, np.zeros(len(b)), b)
    assert np.linalg.norm(host(x) - exp) <= 1e-9 * np.linalg.norm(exp)
    g.close()
