"""N4: the paper's own 6-component elasticity system (u, v) (P:441-445,
backward Euler) on the Table `ndofs` face meshes.  Pins: DOF counts equal the
paper's elasticity table (DOFs = 6 x nodes), the backward-Euler
block structure reduces exactly to C3's eliminated operator M + dt^2 K_e
(reading Z14) by a Schur complement, and MG-preconditioned GMRES converges
with h-independent iteration counts."""
import numpy as np
import pytest

from problems import configs
from problems import fem as F
from problems import mesh as M

import oracle


@pytest.mark.parametrize("name,dofs", [("e6_face_l2", 17550), ("e6_face_l3", 67686), ("e6_edge_l6", 209910),
                                       ("e6_vertex_l6", 22494)])
def test_dof_counts_match_paper_table(name, dofs):
    P = configs.build(name)
    assert P.n_dof == dofs and P.bs == 6


def test_face_l5_dof_count_matches_paper():
    root, box, steps, op, omega, si = configs.CONFIGS["e6_face_l5"]
    m = configs.build_mesh(root, steps)
    assert 6 * len(M.build_nodes(m, m.max_level).keys) == 1035030


def test_schur_complement_is_eliminated_operator():
    """[[M, -dt M], [dt K, M]] (u, v) with v eliminated: M + dt^2 K (Z14) on the
    unconstrained system, checked densely on a small mesh."""
    p = configs.ELAST
    m = configs.build_mesh((2, 2, 2), [])
    nodes = M.build_nodes(m, m.max_level)
    H = F.hanging_matrix(nodes)
    n = len(nodes.keys)
    rp6, c6, v6 = F.assemble(m, nodes, F.Operator("elasticity6", 6, False, p), (1.0, 1.0, 1.0), H)
    rp3, c3, v3 = F.assemble(m, nodes, F.Operator("elasticity", 3, True, p), (1.0, 1.0, 1.0), H)
    A6 = oracle.bsr_to_dense(n, 6, rp6, c6, v6).reshape(n, 6, n, 6)
    A3 = oracle.bsr_to_dense(n, 3, rp3, c3, v3)
    Muu = A6[:, :3, :, :3].reshape(3 * n, 3 * n)
    Muv = A6[:, :3, :, 3:].reshape(3 * n, 3 * n)
    Kvu = A6[:, 3:, :, :3].reshape(3 * n, 3 * n)
    Mvv = A6[:, 3:, :, 3:].reshape(3 * n, 3 * n)
    dt = p["dt"]
    assert np.allclose(Muv, -dt * Muu, rtol=0, atol=1e-15) and np.allclose(Mvv, Muu, rtol=0, atol=1e-15)
    # v = (M u - rhs)/(dt M) -> Schur: M + dt K M^-1 dt M = M + dt^2 K  (times M^-1 M)
    S = Muu - Muv @ np.linalg.solve(Mvv, Kvu)
    assert np.allclose(S, A3, rtol=1e-11, atol=1e-11 * np.abs(A3).max())


def test_gmres_iterations_h_independent():
    its = []
    for name in ("e6_face_l2", "e6_face_l3"):
        P = configs.build(name)
        h = oracle.MgHierarchy.from_arrays(P.levels, omega=P.omega)
        x, it, hist, rel = oracle.gmres(h, P.b, rtol=1e-10, max_iter=100)
        assert rel <= 1.5e-10
        its.append(it)
    assert abs(its[1] - its[0]) <= 3 and max(its) <= 30
