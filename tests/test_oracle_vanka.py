"""Pins of the oracle's Vanka-type patch smoother:
x <- x + omega sum_p R_p^T W A_pp^{-1} R_p (b - A x), W = 1/multiplicity.

  * one patch holding every node and omega = 1: one sweep is the exact solve
    (A_pp = A) from any x;
  * one-node patches: the sweep IS the block-Jacobi sweep (pinned elsewhere
    against dense algebra);
  * listing every patch twice changes nothing (the multiplicity weights);
  * the V-cycle with Vanka smoothing equals the dense error-operator
    recursion with S = I - omega M A, M = sum_p R_p^T W A_pp^{-1} R_p
    (textbook two-grid / multigrid recursion);
  * on the C4 channel Jacobians (reading Z28) GMRES + V(2,2)-Vanka needs no
    more iterations than block-Jacobi and converges for omega in [0.6, 1]."""
import numpy as np
import pytest

import oracle as O
from oracle.mg import vanka_setup, vanka_sweep
from problems import channel as CH
from problems import synthetic as SY
from test_oracle_mg import dense_levels, tiny


def syn_level(n=8, bs=3, seed=0):
    rng = np.random.default_rng(seed)
    rp, col, val = SY.random_bsr(n, bs, rng, avg_nnz=3, band=4)
    return O.mg.MgLevel(n, bs, rp, col, val)


def test_single_patch_is_exact_solve():
    L = syn_level()
    A = O.bsr_to_dense(L.n, L.bs, L.rp, L.col, L.val)
    vk = vanka_setup(L, np.arange(L.n)[None, :])
    rng = np.random.default_rng(1)
    x, b = rng.standard_normal(L.n * L.bs), rng.standard_normal(L.n * L.bs)
    got = vanka_sweep(L, vk, 1.0, x, b)
    exp = np.linalg.solve(A, b)
    assert np.abs(got - exp).max() <= 1e-12 * np.abs(exp).max()


def test_one_node_patches_are_block_jacobi():
    L = syn_level(n=30, seed=2)
    vk = vanka_setup(L, np.arange(L.n)[:, None])
    dinv = O.block_diag_inverse(L.n, L.bs, L.rp, L.col, L.val)
    rng = np.random.default_rng(3)
    x, b = rng.standard_normal(L.n * L.bs), rng.standard_normal(L.n * L.bs)
    got = vanka_sweep(L, vk, 0.7, x, b)
    exp = O.jacobi_sweep(L.n, L.bs, L.rp, L.col, L.val, dinv, 0.7, x, b)
    assert np.abs(got - exp).max() <= 1e-13 * np.abs(exp).max()


def test_duplicate_patches_change_nothing():
    L = syn_level(n=30, seed=4)
    rng = np.random.default_rng(5)
    patches = np.stack([np.arange(L.n), (np.arange(L.n) + 1) % L.n, (np.arange(L.n) + 7) % L.n], axis=1)
    x, b = rng.standard_normal(L.n * L.bs), rng.standard_normal(L.n * L.bs)
    a = vanka_sweep(L, vanka_setup(L, patches), 0.8, x, b)
    c = vanka_sweep(L, vanka_setup(L, np.concatenate([patches, patches])), 0.8, x, b)
    assert np.abs(a - c).max() <= 1e-14 * np.abs(a).max()


@pytest.mark.parametrize("name", ["poisson2d", "elast3d"])
def test_vcycle_with_vanka_equals_dense_recursion(name):
    p = tiny(name)
    h = O.MgHierarchy.from_arrays(p.levels, omega=p.omega, vanka=True)
    dl = dense_levels(h)
    Ms = []
    for L in h.levels:
        patches, inv, w = L.vanka
        M = np.zeros((L.n * L.bs,) * 2)
        for q, nodes in enumerate(patches):
            idx = (nodes[:, None] * L.bs + np.arange(L.bs)).ravel()
            M[np.ix_(idx, idx)] += np.repeat(w[nodes], L.bs)[:, None] * inv[q]
        Ms.append(M)
    I0 = np.eye(dl[0][0].shape[0])
    E = [np.zeros_like(I0)]
    for l in range(1, len(dl)):
        A, _, P = dl[l]
        Ac = dl[l - 1][0]
        I = np.eye(A.shape[0])
        S = I - h.omega * Ms[l] @ A
        CGC = I - P @ (np.eye(Ac.shape[0]) - E[l - 1]) @ np.linalg.solve(Ac, P.T @ A)
        E.append(np.linalg.matrix_power(S, h.nu_post) @ CGC @ np.linalg.matrix_power(S, h.nu_pre))
    rng = np.random.default_rng(6)
    A = dl[-1][0]
    N = A.shape[0]
    x, b = rng.standard_normal(N), rng.standard_normal(N)
    got = O.vcycle(h, len(h.levels) - 1, x, b)
    ref = E[-1] @ x + (np.eye(N) - E[-1]) @ np.linalg.solve(A, b)
    assert np.abs(got - ref).max() <= 1e-11 * (np.abs(ref).max() + np.abs(x).max())


def test_vanka_on_channel_jacobians():
    P = CH.build("c4ns_mid")
    u = CH.initial_state(P)
    F = CH.residual(P, u, u)
    levels = CH.with_values(P, CH.jacobians(P, u, u))
    _, its_j, _, _ = O.gmres(O.MgHierarchy.from_arrays(levels, omega=P.omega), -F, rtol=1e-10)
    for om in (0.6, 0.8, 1.0):
        _, its_v, _, rel = O.gmres(O.MgHierarchy.from_arrays(levels, omega=om, vanka=True), -F, rtol=1e-10)
        assert rel <= 1e-10 and its_v <= its_j and its_v <= 15, (om, its_v, its_j)
