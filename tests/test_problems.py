"""Pins of the seeded input generator (problems/) against the paper's printed
values, closed forms and invariants."""
import itertools

import numpy as np
import pytest

from problems import configs as C
from problems import fem as F
from problems import mesh as M
from mgtest_util import problem


def _pattern_meshes(axes, L):
    m = M.uniform((8, 8, 8))
    out = [m]
    for _ in range(L - 1):
        m = M.refine(m, M.band_mark(m, axes, 1))
        out.append(m)
    return out


@pytest.mark.parametrize("pattern,axes", [("face", [0]), ("edge", [0, 1]), ("vertex", [0, 1, 2])])
def test_table_ndofs_exact(G, pattern, axes):
    """P:457-477 Table `ndofs`: all node counts exactly; edge-midpoint hanging
    fraction to the printed precision (reading Z15; face L4 typo 6.33 vs 6.38)."""
    ref = G["table_ndofs"][pattern]
    for L, m in enumerate(_pattern_meshes(axes, 6 if pattern != "face" else 5), start=1):
        ns = M.build_nodes(m)
        assert len(ns.keys) == ref["nodes"][L - 1]
        pct = 100.0 * np.mean(ns.h_kind == 2)
        digits = 2 if ref["pct"][L - 1] < 10 else 1
        if pattern == "face" and L == 4:
            assert round(pct, 2) == 6.38  # paper prints 6.33 (presumed typo, Z15)
        else:
            assert round(pct, digits) == pytest.approx(ref["pct"][L - 1], abs=1e-9)


def test_table_ndofs_face_L6_and_dofs(G):
    m = _pattern_meshes([0], 6)[-1]
    assert len(M.build_nodes(m).keys) == G["table_ndofs"]["face"]["nodes"][5]
    for pat in ("face", "edge", "vertex"):
        rows = G["elasticity_dofs"][pat]
        ref = G["table_ndofs"][pat]["nodes"]
        for L, dofs in rows:
            assert dofs == 6 * ref[L - 1]       # P:445 "six times this number of mesh nodes"


def test_edge_L6_hanging_dofs():
    """'about 25 600' of the 209,910 DOFs at edge L6 are hanging."""
    m = _pattern_meshes([0, 1], 6)[-1]
    ns = M.build_nodes(m)
    assert abs(6 * int(np.sum(ns.h_kind == 2)) - 25600) < 200


def test_uniform_counts(G):
    """(2^n+1)^2 nodes for uniform refinement (Table td)."""
    for n, dofs in zip(G["td_dofs"]["n"][:2], G["td_dofs"]["dofs"][:2]):
        m = C.build_mesh((1, 1), [("uniform",)] * n)
        assert len(M.build_nodes(m).keys) == dofs
    for n, dofs in zip(G["td_dofs"]["n"], G["td_dofs"]["dofs"]):
        assert (2 ** n + 1) ** 2 == dofs


def test_refine_spec_examples():
    """1 element -> 4, 9 nodes, 0 hanging; 2x2 mark one -> 7 elements,
    2 hanging nodes; marking a corner twice triggers the closure."""
    m = M.refine(M.uniform((1, 1)), np.ones(1, bool))
    ns = M.build_nodes(m)
    assert m.n_cells == 4 and len(ns.keys) == 9 and not ns.hanging.any()
    m = M.uniform((2, 2))
    mark = np.zeros(4, bool)
    mark[0] = True
    m = M.refine(m, mark)
    ns = M.build_nodes(m)
    assert m.n_cells == 7 and int(ns.hanging.sum()) == 2
    assert np.all(ns.h_weights[ns.hanging][:, :2] == 0.5)
    # refine the corner child again: closure must refine the neighbours of the new level
    sel = (m.lev == 1) & (m.ijk[:, 0] == 1) & (m.ijk[:, 1] == 1)
    m2 = M.refine(m, sel)
    assert not M.balance_violations(m2).any()
    assert m2.n_cells > 7 + 3


def _exhaustive_balance_ok(m: M.Mesh) -> bool:
    """Brute force 2:1 check over every pair of leaves sharing a face or edge."""
    R = m.max_level
    lo = m.ijk << (R - m.lev)[:, None]
    hi = (m.ijk + 1) << (R - m.lev)[:, None]
    for i in range(m.n_cells):
        ov_lo = np.maximum(lo[i], lo)
        ov_hi = np.minimum(hi[i], hi)
        touch = np.all(ov_lo <= ov_hi, axis=1)
        dimsh = np.sum(ov_hi > ov_lo, axis=1)      # dimension of the shared set
        share = touch & (dimsh >= max(m.dim - 2, 1)) & (np.arange(m.n_cells) != i)
        if m.dim == 2:
            share = touch & (dimsh >= 1) & (np.arange(m.n_cells) != i)
        if np.any(np.abs(m.lev[share] - m.lev[i]) > 1):
            return False
    return True


def test_balance_exhaustive_and_hierarchy_invariants():
    """S:227 exhaustive 2:1 scan; S:229 nesting of hierarchy levels; P:490 the
    number of MG levels grows by one per refinement step; root never merged."""
    m = C.build_mesh((4, 4), [("band", [1], 1)] * 3)
    assert _exhaustive_balance_ok(m)
    H = M.hierarchy(m)
    assert len(H) == m.max_level + 1
    for c, f in zip(H[:-1], H[1:]):
        assert _exhaustive_balance_ok(c)
        ck = set(zip(c.lev.tolist(), M.cell_key_any(c.root, c.lev, c.ijk).tolist()))
        for lv, key, ijk in zip(f.lev, M.cell_key_any(f.root, f.lev, f.ijk), f.ijk):
            par = M.cell_key(f.root, int(lv) - 1, (ijk >> 1)[None])[0] if lv > 0 else None
            assert (int(lv), int(key)) in ck or (int(lv) - 1, int(par)) in ck
    assert H[0].max_level == 0 and H[0].n_cells == 16


def test_hierarchy_regression_values():
    """Global-coarsening hierarchies cross-checked by two independent scratch
    methods: face L4 (8^3) and the C2/C3 configs."""
    m = _pattern_meshes([0], 4)[-1]
    assert [len(M.build_nodes(x, m.max_level).keys) for x in M.hierarchy(m)] == [729, 1434, 6509, 43861]
    m = C.build_mesh((32, 32), [("band", [1], 20)] * 7)
    assert [len(M.build_nodes(x, m.max_level).keys) for x in M.hierarchy(m)] == \
        [1089, 1315, 2055, 4688, 16009, 61701, 244489, 973329]


@pytest.mark.slow
def test_c3_hierarchy_sizes():
    m = C.build_mesh((9, 9, 9), [("band", [0], 1)] * 6)
    assert [len(M.build_nodes(x, m.max_level).keys) for x in M.hierarchy(m)] == \
        [1000, 1883, 5268, 18517, 70934, 474473, 3443281]


def test_uniform_roundtrip():
    """refine then coarsen a uniform mesh returns the original count."""
    m0 = M.uniform((3, 2, 2))
    m1 = M.refine(m0, np.ones(m0.n_cells, bool))
    assert M.coarsen_step(m1).n_cells == m0.n_cells


def test_element_matrices_closed_forms(G):
    """Q1 unit-square M and K entries; K.1 = 0; bit symmetry."""
    Mref, Gt, _ = F.reference_tensors(2)
    K = Gt[0, 0] + Gt[1, 1]
    gm = G["q1_element"][0]
    gk = G["q1_element"][1]
    # corner 0 = (0,0); 1 = (1,0) edge neighbour; 3 = (1,1) opposite
    assert Mref[0, 0] == pytest.approx(gm["diag"], abs=1e-15)
    assert Mref[0, 1] == pytest.approx(gm["edge"], abs=1e-15)
    assert Mref[0, 3] == pytest.approx(gm["opposite"], abs=1e-15)
    assert K[0, 0] == pytest.approx(gk["diag"], abs=1e-15)
    assert K[0, 1] == pytest.approx(gk["edge"], abs=1e-15)
    assert K[0, 3] == pytest.approx(gk["opposite"], abs=1e-15)
    assert np.abs(K @ np.ones(4)).max() < 1e-15
    assert np.array_equal(K, K.T) and np.array_equal(Mref, Mref.T)
    assert Mref.sum() == pytest.approx(1.0, abs=1e-15)
    # 3d Laplacian stencil of a unit cube: centre 8h/3, face 0, edge -h/6, corner -h/12
    _, G3, _ = F.reference_tensors(3)
    K3 = G3[0, 0] + G3[1, 1] + G3[2, 2]
    assert K3[0, 0] == pytest.approx(1 / 3, abs=1e-15)
    assert K3[0, 7] == pytest.approx(-1 / 12, abs=1e-15)


def test_elasticity_rigid_modes():
    """translations and linearised rotations lie in ker K_e."""
    op = F.Operator("elasticity", 3, True, dict(lam=8e4, mu=2e4, dt=1.0))
    T, S = F.element_terms(op, 3, np.array([[0.5, 0.5, 0.5]]))
    Ke = sum(S[0, t] * T[t] for t in range(1, T.shape[0]))   # drop the mass term
    assert np.array_equal(Ke, Ke.T)
    xyz = F.M._corner_offsets(3) * 0.5
    modes = []
    for c in range(3):
        u = np.zeros((8, 3)); u[:, c] = 1.0; modes.append(u)
    for (a, b) in ((0, 1), (0, 2), (1, 2)):
        u = np.zeros((8, 3)); u[:, a] = -xyz[:, b]; u[:, b] = xyz[:, a]; modes.append(u)
    for u in modes:
        assert np.abs(Ke @ u.ravel()).max() < 1e-12 * np.abs(Ke).max()


def test_constrain_and_dirichlet_spec_examples(G):
    """S:352 (H^T A H with identity hanging row) and S:361 (symmetric elimination)."""
    ex = G["constrain_system"][0]
    A = np.array(ex["A"], float)
    Hm = np.array(ex["H"], float)
    Abar = Hm.T @ A @ Hm
    Abar[2, :] = 0; Abar[:, 2] = 0; Abar[2, 2] = 1
    assert np.allclose(Abar, ex["Abar"], atol=0)
    # same via the generator's C assembler: one 'element' with 3 local nodes is
    # not a Q1 cell, so exercise apply_constraints for the Dirichlet example
    ex = G["dirichlet"][0]
    rp = np.array([0, 2, 4]); col = np.array([0, 1, 0, 1]); val = np.array(ex["A"], float).reshape(4, 1, 1)
    cm = np.array([[False], [True]]); g = np.array([[0.0], [ex["fix"][1]]]); b = np.array(ex["b"], float)[:, None]
    F.apply_constraints(rp, col, val, cm, g, b)
    assert np.array_equal(val.reshape(2, 2), np.array(ex["Aout"], float))
    assert np.array_equal(b.ravel(), np.array(ex["bout"], float))


def _dense(l):
    from oracle import bsr_to_dense
    return bsr_to_dense(l.n, l.bs, l.row_ptr, l.col, l.val)


@pytest.mark.parametrize("name", ["c1_poisson", "c3_small", "face_poisson"])
def test_condensed_symmetry_and_identity_rows(name):
    """S:377 symmetry preserved bit-exactly; constrained rows are identity."""
    p = problem(name)
    for l in p.levels:
        if l.n * l.bs > 4000:
            continue
        A = _dense(l)
        assert np.array_equal(A, A.T)
        cm = l.cmask.ravel()
        assert np.array_equal(A[cm][:, cm], np.eye(cm.sum()))
        assert not A[cm][:, ~cm].any()


def test_H_invariants():
    """H^2 = H, H 1 = 1, weights in {1/2, 1/4}, rows sum to 1."""
    p = problem("face_poisson")
    for l in p.levels:
        rp, col, w = l.H
        Hd = np.zeros((l.n, l.n))
        for i in range(l.n):
            Hd[i, col[rp[i]:rp[i + 1]]] = w[rp[i]:rp[i + 1]]
        assert np.array_equal(Hd @ Hd, Hd)
        assert np.array_equal(Hd @ np.ones(l.n), np.ones(l.n))
        assert set(np.unique(w)).issubset({0.25, 0.5, 1.0})


@pytest.mark.parametrize("name", ["c1_poisson", "c2_small", "c3_small", "face_poisson"])
def test_P_invariants(name):
    """P:331 reference chi_ij weights (dyadic), P.1 = 1 on unconstrained fine rows
    away from the boundary, empty rows at constrained fine DOFs (reading G6)."""
    p = problem(name)
    for lc, lf in zip(p.levels[:-1], p.levels[1:]):
        rp, col, w = lf.P
        assert np.all(np.diff(rp) >= 0) and rp[-1] == len(col)
        for i in range(lf.n):
            assert np.all(np.diff(col[rp[i]:rp[i + 1]]) > 0)
        assert set(np.round(w * 64).astype(int) / 64) == set(w)      # dyadic
        cm = lf.cmask[:, 0]
        assert np.all(np.diff(rp)[cm] == 0)
        assert not lc.cmask[col, 0].any()
        # interpolation of the constant: fine rows whose every coarse neighbour is free sum to 1
        Pd = np.zeros((lf.n, lc.n))
        rows = np.repeat(np.arange(lf.n), np.diff(rp))
        Pd[rows, col] = w
        # E H 1 = 1: rebuild P without the Pi masks and check the row sums
    # unmasked composition: E H_c Pi_c with Pi dropped reproduces constants exactly
    lc, lf = p.levels[-2], p.levels[-1]
    rp, col, w = F.prolongation(lc.mesh, lc.nodes, lc.H, np.ones(lc.n, bool), lf.mesh, lf.nodes, np.ones(lf.n, bool))
    sums = np.add.reduceat(w, rp[:-1]) if len(w) else np.zeros(0)
    assert np.array_equal(sums, np.ones(lf.n))


def test_theta_ex(G):
    ex = G["theta_ex"]
    assert C.theta_ex(ex["t"], ex["x"], ex["y"]) == ex["value"]


def test_seeded_rhs_deterministic():
    a = C.build("c1").b
    b = C.build("c1").b
    assert np.array_equal(a, b)
