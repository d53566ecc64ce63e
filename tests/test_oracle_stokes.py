"""Pins of the C4/C5 NS-shaped operator (reading Z23): equal-order Q1
generalised Stokes with PSPG stabilisation and eps*M_p regularisation, unknowns
(p, u_1..u_d) node-major, velocity-only Dirichlet.  The paper prints no
values for this reading ("parity unpinned vs the paper"); these
tests pin it to closed forms and invariants:

* the constant pressure is annihilated by every unconstrained velocity row
  (int div v = 0 for v vanishing on the boundary) and by the PSPG term, so
  A (p=1, u=0) = eps * (int phi_i) on pressure rows (the Q1 mass row sum);
* the velocity-pressure coupling is exactly skew (B / -B^T) before
  condensation, the velocity-velocity and pressure-pressure blocks symmetric;
* MG-preconditioned GMRES converges with h-independent iteration counts.
"""
import numpy as np
import pytest

from problems import configs
from problems import fem as F
from problems import mesh as M

import oracle


def _assembled(name):
    root, box, steps, op, omega, si = configs.CONFIGS[name]
    m = configs.build_mesh(root, steps)
    nodes = M.build_nodes(m, m.max_level)
    H = F.hanging_matrix(nodes)
    rp, col, val = F.assemble(m, nodes, op, box, H)
    return m, nodes, op, box, rp, col, val


@pytest.mark.parametrize("name", ["c4_small", "c5_small"])
def test_constant_pressure_mode(name):
    P = configs.build(name)
    L = P.fine
    bs = P.bs
    x = np.zeros((L.n, bs))
    x[:, 0] = 1.0
    x[L.cmask[:, 0], 0] = 0.0                      # hanging pressure DOFs are constrained
    y = oracle.spmv(L.n, bs, L.row_ptr, L.col, L.val, x.reshape(-1)).reshape(L.n, bs)
    free_u = ~L.cmask[:, 1:]
    # interior (unconstrained) velocity rows: int p div v = 0 for p = 1
    # (exact up to summation of O(h^{d-1}) terms)
    scale = np.max(np.abs(L.val))
    assert np.max(np.abs(y[:, 1:][free_u])) <= 1e-12 * scale
    # pressure rows: eps * int phi_i (lumped mass of the condensed space), positive
    eps = configs.CONFIGS[name][3].params["eps"]
    pr = y[~L.cmask[:, 0], 0]
    assert np.all(pr > 0)
    box = configs.CONFIGS[name][1]
    assert abs(pr.sum() - eps * np.prod(box)) <= 1e-9 * eps * np.prod(box)


@pytest.mark.parametrize("name", ["c4_small", "c5_small"])
def test_block_structure_skew_coupling(name):
    m, nodes, op, box, rp, col, val = _assembled(name)
    n, bs = len(nodes.keys), op.bs
    A = oracle.bsr_to_dense(n, bs, rp, col, val).reshape(n, bs, n, bs)
    vv = A[:, 1:, :, 1:].reshape(n * (bs - 1), -1)
    pp = A[:, 0, :, 0]
    up = A[:, 1:, :, 0]                             # velocity rows, pressure cols
    pu = A[:, 0, :, 1:]                             # pressure rows, velocity cols
    sc = np.max(np.abs(A))
    assert np.max(np.abs(vv - vv.T)) <= 1e-13 * sc
    assert np.max(np.abs(pp - pp.T)) <= 1e-13 * sc
    assert np.max(np.abs(up + np.transpose(pu, (1, 2, 0)))) <= 1e-13 * sc
    # symmetric part positive definite (velocity mass + PSPG + eps M_p) on the
    # regular DOFs (condensed hanging rows/columns are zero): Cholesky succeeds
    reg = np.repeat(~nodes.hanging, bs)
    Ad = A.reshape(n * bs, n * bs)[np.ix_(reg, reg)]
    np.linalg.cholesky(0.5 * (Ad + Ad.T))


def test_stokes_transfers_per_component():
    P = configs.build("c4_small")
    for l in range(1, len(P.levels)):
        L, C = P.levels[l], P.levels[l - 1]
        assert L.wpe == P.bs
        rp, col, w = L.P
        w = w.reshape(-1, P.bs)
        rows = F.row_of(rp)
        # weights vanish exactly on constrained (row or column) components
        assert np.all(w[L.cmask[rows]] == 0.0)
        assert np.all(w[C.cmask[col]] == 0.0)
        # pressure (never Dirichlet) keeps interpolation rows summing to 1 at regular fine nodes
        reg = ~L.cmask[:, 0]
        s = np.zeros(L.n)
        np.add.at(s, rows, w[:, 0])
        assert np.allclose(s[reg], 1.0, atol=0, rtol=0) or np.max(np.abs(s[reg] - 1.0)) <= 1e-15


def test_stokes_gmres_h_independent_3d():
    its = []
    for k in (2, 3):
        P = configs.make_problem("t", (2, 2, 4), (1.0, 1.0, 2.0), [("uniform",)] * k,
                                 F.Operator("stokes", 4, False, configs.STOKES3), seed_index=4,
                                 omega=0.6, g_fun=configs.lid(3, 4))
        h = oracle.MgHierarchy.from_arrays(P.levels, omega=0.6)
        x, it, hist, rel = oracle.gmres(h, P.b, rtol=1e-10, max_iter=120)
        assert rel <= 1e-10 * 1.5
        its.append(it)
    assert its[1] - its[0] <= 3 and max(its) <= 35


def test_stokes_gmres_2d_c4_small():
    P = configs.build("c4_small")
    h = oracle.MgHierarchy.from_arrays(P.levels, omega=P.omega)
    x, it, hist, rel = oracle.gmres(h, P.b, rtol=1e-10)
    assert it <= 20 and rel <= 1.5e-10
