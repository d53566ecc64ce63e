"""Pins of the oracle's per-op definitions (oracle/csrc/oracle.c) against the
SPEC worked examples (tests/golden/) and brute force with numpy/scipy dense
linear algebra on random block-CSR matrices (ragged rows, empty rows, every
block size of the configs)."""
import math

import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O


def dense_to_csr(A):
    A = np.asarray(A, float)
    S = sp.csr_matrix(A)
    S.sort_indices()
    return (S.indptr.astype(np.int64), S.indices.astype(np.int64), S.data.copy())


def random_bsr(n, bs, density, rng, empty_rows=True, with_diag=True):
    rows = []
    for i in range(n):
        cols = np.nonzero(rng.random(n) < density)[0]
        if with_diag:
            cols = np.union1d(cols, [i])
        if empty_rows and i % 7 == 3 and not with_diag:
            cols = np.zeros(0, int)
        rows.append(np.sort(cols))
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(c) for c in rows])
    col = np.concatenate(rows).astype(np.int64) if rp[-1] else np.zeros(0, np.int64)
    val = rng.standard_normal((rp[-1], bs, bs))
    if with_diag:
        for i in range(n):
            k = rp[i] + np.searchsorted(col[rp[i]:rp[i + 1]], i)
            val[k] += 4 * bs * np.eye(bs)
    return rp, col, val


# ------------------------------------------------------------------ SPEC examples


def test_spec_spmv(G):
    for ex in G["spmv"]:
        rp, col, w = dense_to_csr(ex["A"])
        y = O.spmv(len(rp) - 1, 1, rp, col, w.reshape(-1, 1, 1), np.array(ex["x"], float),
                   ex["alpha"], ex["beta"], np.array(ex["y0"], float))
        assert np.array_equal(y, np.array(ex["y"], float)), ex["cite"]


def test_spec_spmv_transpose(G):
    for ex in G["spmv_transpose"]:
        A = np.array(ex["A"], float)
        rp, col, w = dense_to_csr(A)
        trp, tcol, tw = O.csr_transpose(A.shape[0], A.shape[1], rp, col, w)
        y = O.transfer(A.shape[1], 1, trp, tcol, tw, 1, np.array(ex["x"], float))
        assert np.array_equal(y, np.array(ex["y"], float)), ex["cite"]


def test_spec_blas1_diag_transpose(G):
    d, n2 = G["blas1"]
    assert O.dot(np.array(d["a"], float), np.array(d["b"], float)) == d["out"]
    assert O.nrm2(np.array(n2["a"], float)) == n2["out"]
    ex = G["diag_apply"][0]
    D = np.diag(np.array(ex["D"], float))
    rp, col, w = dense_to_csr(D)
    dinv = O.block_diag_inverse(2, 1, rp, col, w.reshape(-1, 1, 1))
    assert np.array_equal(dinv.ravel() * np.array(ex["x"]), np.array(ex["out"], float))
    ex = G["csr_transpose"][0]
    r, c, v = ex["entries"][0]
    rp = np.array([0, 1, 1]); col = np.array([c]); w = np.array([float(v)])
    trp, tcol, tw = O.csr_transpose(ex["rows"], ex["cols"], rp, col, w)
    assert list(trp) == [0, 0, 0, 1] and list(tcol) == [0] and list(tw) == [5.0]


def test_spec_lu_and_jacobi(G):
    for ex in G["dense_lu_solve"]:
        lu, piv = O.lu_factor(np.array(ex["A"], float))
        assert np.array_equal(O.lu_solve(lu, piv, np.array(ex["b"], float)), np.array(ex["x"], float))
    for ex in G["jacobi"]:
        A = np.array(ex["A"], float)
        rp, col, w = dense_to_csr(A)
        val = w.reshape(-1, 1, 1)
        dinv = O.block_diag_inverse(2, 1, rp, col, val)
        x = O.jacobi_sweep(2, 1, rp, col, val, dinv, ex["omega"], np.zeros(2), np.array(ex["b"], float))
        assert np.array_equal(x, np.array(ex["x"], float)), ex["cite"]


def test_spec_gmres(G):
    """S:449-450 with precond = I."""
    class L:
        pass
    for ex in G["gmres"]:
        A = np.array(ex["A"], float)
        rp, col, w = dense_to_csr(A)
        lv = L(); lv.n, lv.bs, lv.row_ptr, lv.col, lv.val, lv.P = 2, 1, rp, col, w.reshape(-1, 1, 1), None
        h = O.MgHierarchy.from_arrays([lv])
        x, its, hist, rr = O.gmres(h, np.array(ex["b"], float), rtol=1e-12, precondition=False)
        assert its <= ex["max_iters"]
        assert np.allclose(x, ex["x"], rtol=0, atol=1e-14)
        assert rr <= 1e-12


# ------------------------------------------------------------------ brute force


@pytest.mark.parametrize("bs", [1, 2, 3, 4])
def test_spmv_residual_vs_dense(bs):
    rng = np.random.default_rng(100 + bs)
    for n, dens, ed in ((1, 1.0, False), (37, 0.15, True), (64, 0.3, True)):
        rp, col, val = random_bsr(n, bs, dens, rng, empty_rows=ed, with_diag=False)
        A = O.bsr_to_dense(n, bs, rp, col, val)
        Sd = sp.bsr_matrix((val, col, rp), shape=(n * bs, n * bs)).toarray()
        assert np.array_equal(A, Sd)                         # expansion agrees with scipy
        x = rng.standard_normal(n * bs)
        y0 = rng.standard_normal(n * bs)
        b = rng.standard_normal(n * bs)
        y = O.spmv(n, bs, rp, col, val, x, 1.5, -0.5, y0)
        ref = 1.5 * (Sd @ x) - 0.5 * y0
        scale = 1.5 * (np.abs(Sd) @ np.abs(x)) + 0.5 * np.abs(y0)
        assert np.all(np.abs(y - ref) <= 1e-14 * scale + 1e-300)
        r = O.residual(n, bs, rp, col, val, x, b)
        assert np.all(np.abs(r - (b - Sd @ x)) <= 1e-14 * (np.abs(b) + np.abs(Sd) @ np.abs(x)))


@pytest.mark.parametrize("bs", [1, 2, 3, 4])
def test_block_inverse_and_sweep_vs_dense(bs):
    rng = np.random.default_rng(200 + bs)
    n = 41
    rp, col, val = random_bsr(n, bs, 0.2, rng)
    dinv = O.block_diag_inverse(n, bs, rp, col, val)
    A = O.bsr_to_dense(n, bs, rp, col, val)
    for i in range(n):
        blk = A[i * bs:(i + 1) * bs, i * bs:(i + 1) * bs]
        assert np.allclose(dinv[i], np.linalg.inv(blk), rtol=1e-13, atol=1e-15)
    x, b = rng.standard_normal(n * bs), rng.standard_normal(n * bs)
    D = np.zeros_like(A)
    for i in range(n):
        D[i * bs:(i + 1) * bs, i * bs:(i + 1) * bs] = np.linalg.inv(A[i * bs:(i + 1) * bs, i * bs:(i + 1) * bs])
    ref = x + 0.7 * D @ (b - A @ x)
    out = O.jacobi_sweep(n, bs, rp, col, val, dinv, 0.7, x, b)
    assert np.allclose(out, ref, rtol=1e-12, atol=1e-12)


def test_block_inverse_errors():
    rp = np.array([0, 1, 2]); col = np.array([0, 1])
    val = np.zeros((2, 2, 2)); val[0] = np.eye(2)
    with pytest.raises(ValueError):
        O.block_diag_inverse(2, 2, rp, col, val)              # singular block
    rp = np.array([0, 1, 1]); col = np.array([0]); val = np.ones((1, 1, 1))
    with pytest.raises(ValueError):
        O.block_diag_inverse(2, 1, rp, col, val)              # missing diagonal


@pytest.mark.parametrize("bs,wpe", [(1, 1), (3, 1), (4, 1), (4, 4), (2, 2)])
def test_transfer_and_transpose_vs_dense(bs, wpe):
    rng = np.random.default_rng(300 + bs + wpe)
    nf, nc = 53, 17
    dens = rng.random((nf, nc)) < 0.12
    rp = np.zeros(nf + 1, np.int64); rp[1:] = np.cumsum(dens.sum(1))
    col = np.nonzero(dens)[1].astype(np.int64)
    w = rng.integers(1, 8, size=len(col) * wpe) / 8.0
    P = np.zeros((nf * bs, nc * bs))
    rows = np.repeat(np.arange(nf), np.diff(rp))
    for t in range(len(col)):
        for c in range(bs):
            P[rows[t] * bs + c, col[t] * bs + c] = w[t * wpe + (c if wpe > 1 else 0)]
    y = rng.standard_normal(nc * bs); x0 = rng.standard_normal(nf * bs)
    assert np.allclose(O.transfer(nf, bs, rp, col, w, wpe, y, x0), x0 + P @ y, rtol=1e-14, atol=1e-14)
    trp, tcol, tw = O.csr_transpose(nf, nc, rp, col, w, wpe)
    S = sp.csr_matrix((np.arange(1, len(col) + 1, dtype=float), col, rp), shape=(nf, nc)).T.tocsr()
    S.sort_indices()
    assert np.array_equal(trp, S.indptr) and np.array_equal(tcol, S.indices)
    r = rng.standard_normal(nf * bs)
    assert np.allclose(O.transfer(nc, bs, trp, tcol, tw, wpe, r), P.T @ r, rtol=1e-14, atol=1e-14)
    rrp, rcol, rw = O.csr_transpose(nc, nf, trp, tcol, tw, wpe)
    assert np.array_equal(rrp, rp) and np.array_equal(rcol, col) and np.array_equal(rw, w)  # involution S:117


def test_lu_vs_numpy_and_dot():
    rng = np.random.default_rng(7)
    A = rng.standard_normal((60, 60)) + 8 * np.eye(60)
    b = rng.standard_normal(60)
    lu, piv = O.lu_factor(A)
    x = O.lu_solve(lu, piv, b)
    assert np.allclose(x, np.linalg.solve(A, b), rtol=1e-12, atol=1e-13)
    with pytest.raises(ValueError):
        O.lu_factor(np.zeros((3, 3)))
    a, c = rng.standard_normal(10001), rng.standard_normal(10001)
    exact = math.fsum(a * c)
    assert abs(O.dot(a, c) - exact) <= 1e-13 * np.sum(np.abs(a * c))
