"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 reference for the hot path of arXiv
2405.05047: the geometric-multigrid V-cycle (Alg. `gmg`) on
assembled block systems, with the block-Jacobi smoother, transfer
matrices P and R = P^T, the coarse solve (P:127 / P:341), GMRES
with modified Gram-Schmidt and Givens rotations and hanging-node
interpolation x <- H x; the global constraint int p = 0 on every
level; the explicit pressure-correction Navier-Stokes step of Alg. 2
 in oracle/ns.py.

Who may use it: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` leg.  The product (paper_2405_05047_b200)
never imports it; the two share no code.  Per-op kernels are plain C
(oracle/csrc/oracle.c, -ffp-contract=off, rows summed sequentially); the
recursion and Krylov logic are written out in Python in the paper's order
(oracle/mg.py).

Pins (tests/test_oracle_*.py): SPEC worked examples (tests/golden/), dense
numpy/scipy brute force on random BSR matrices, dense two-grid / multi-level
error-operator recursion, dense LU on small systems, O(h^2) manufactured
convergence, LFA lambda_max(D^-1 A) -> 1.5, h-independent contraction.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "csrc", "oracle.c")
LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC",
                               "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        P, I64, D, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        L.or_bsr_spmv.argtypes = [I64, I, P, P, P, D, P, D, P]
        L.or_bsr_spmv.restype = None
        L.or_bsr_residual.argtypes = [I64, I, P, P, P, P, P, P]
        L.or_bsr_residual.restype = None
        L.or_block_diag_inverse.argtypes = [I64, I, P, P, P, P]
        L.or_block_diag_inverse.restype = I
        L.or_jacobi_sweep.argtypes = [I64, I, P, P, P, P, D, P, P, P]
        L.or_jacobi_sweep.restype = None
        L.or_transfer.argtypes = [I64, I, P, P, P, I, P, P, I]
        L.or_transfer.restype = None
        L.or_csr_transpose.argtypes = [I64, I64, P, P, P, I, P, P, P]
        L.or_csr_transpose.restype = None
        L.or_lu_factor.argtypes = [I64, P, P]
        L.or_lu_factor.restype = I
        L.or_lu_solve.argtypes = [I64, P, P, P, P]
        L.or_lu_solve.restype = None
        L.or_dot.argtypes = [I64, P, P]
        L.or_dot.restype = D
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def set_threads(n: int) -> None:
    """OpenMP thread count for the row-parallel kernels (results do not depend on it)."""
    os.environ["OMP_NUM_THREADS"] = str(n)
    try:
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(n))
    except OSError:
        pass


# ----------------------------------------------------------------------------
# per-op definitions
# ----------------------------------------------------------------------------


def spmv(n, bs, rp, col, val, x, alpha=1.0, beta=0.0, y=None):
    """y = alpha A x + beta y."""
    rp, col, val, x = _c(rp, np.int64), _c(col, np.int64), _c(val, np.float64), _c(x, np.float64)
    y = np.zeros(n * bs) if y is None else _c(y, np.float64).copy()
    lib().or_bsr_spmv(n, bs, _p(rp), _p(col), _p(val), alpha, _p(x), beta, _p(y))
    return y


def residual(n, bs, rp, col, val, x, b):
    """r = b - A x  (Alg. gmg Step 2)."""
    rp, col, val, x, b = (_c(rp, np.int64), _c(col, np.int64), _c(val, np.float64),
                          _c(x, np.float64), _c(b, np.float64))
    r = np.empty(n * bs)
    lib().or_bsr_residual(n, bs, _p(rp), _p(col), _p(val), _p(x), _p(b), _p(r))
    return r


def block_diag_inverse(n, bs, rp, col, val):
    """D^{-1} = inverse diagonal blocks (block-Jacobi S)."""
    rp, col, val = _c(rp, np.int64), _c(col, np.int64), _c(val, np.float64)
    d = np.empty((n, bs, bs))
    st = lib().or_block_diag_inverse(n, bs, _p(rp), _p(col), _p(val), _p(d))
    if st != 0:
        raise ValueError(f"block_diag_inverse failed with status {st}")
    return d


def jacobi_sweep(n, bs, rp, col, val, dinv, omega, x, b):
    """x + omega D^{-1}(b - A x)."""
    rp, col, val, dinv, x, b = (_c(rp, np.int64), _c(col, np.int64), _c(val, np.float64),
                                _c(dinv, np.float64), _c(x, np.float64), _c(b, np.float64))
    out = np.empty(n * bs)
    lib().or_jacobi_sweep(n, bs, _p(rp), _p(col), _p(val), _p(dinv), omega, _p(x), _p(b), _p(out))
    return out


def transfer(n_rows, bs, rp, col, w, wpe, x, y=None):
    """P x (y is None) or y + P x  (P:333 prolongation; R = P^T for restriction)."""
    rp, col, w, x = _c(rp, np.int64), _c(col, np.int64), _c(w, np.float64), _c(x, np.float64)
    acc = y is not None
    out = _c(y, np.float64).copy() if acc else np.empty(n_rows * bs)
    lib().or_transfer(n_rows, bs, _p(rp), _p(col), _p(w), wpe, _p(x), _p(out), int(acc))
    return out


def csr_transpose(n_rows, n_cols, rp, col, w, wpe=1):
    """Stable transpose (R = P^T)."""
    rp, col, w = _c(rp, np.int64), _c(col, np.int64), _c(w, np.float64)
    nnz = int(rp[-1])
    orp = np.empty(n_cols + 1, np.int64)
    ocol = np.empty(nnz, np.int64)
    ow = np.empty(nnz * wpe)
    lib().or_csr_transpose(n_rows, n_cols, _p(rp), _p(col), _p(w), wpe, _p(orp), _p(ocol), _p(ow))
    return orp, ocol, ow


def lu_factor(A):
    a = _c(A, np.float64).copy()
    n = a.shape[0]
    piv = np.empty(n, np.int64)
    st = lib().or_lu_factor(n, _p(a), _p(piv))
    if st != 0:
        raise ValueError("singular matrix in lu_factor")
    return a, piv


def lu_solve(lu, piv, b):
    b = _c(b, np.float64)
    x = np.empty_like(b)
    lib().or_lu_solve(lu.shape[0], _p(lu), _p(piv), _p(b), _p(x))
    return x


def dot(a, b) -> float:
    a, b = _c(a, np.float64), _c(b, np.float64)
    return float(lib().or_dot(a.shape[0], _p(a), _p(b)))


def nrm2(a) -> float:
    return float(np.sqrt(dot(a, a)))


def bsr_to_dense(n, bs, rp, col, val):
    """Dense expansion of a BSR matrix (oracle-side helper for small cases)."""
    A = np.zeros((n * bs, n * bs))
    for i in range(n):
        for k in range(rp[i], rp[i + 1]):
            A[i * bs:(i + 1) * bs, col[k] * bs:(col[k] + 1) * bs] += val[k]
    return A


from .mg import (MgHierarchy, MgLevel, consistent, gmres, gmres_dcgs2, project_zero_mean, richardson,  # noqa: E402,F401
                 vcycle)
