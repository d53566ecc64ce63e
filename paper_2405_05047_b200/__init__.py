"""paper_2405_05047_b200 -- B200-native fp64 geometric multigrid (arXiv 2405.05047).

Thin ctypes binding over libmgb200.so (include/mg.h): the same names as the C
ABI, argument marshalling only.  Every step of the solve runs in the CUDA
library; there is no CPU fallback -- importing this package fails loudly if
the extension has not been built (``python paper_2405_05047_b200/build.py`` or
``python __graft_entry__.py``).

Vectors and arrays may be torch tensors (CUDA -> device pointer, CPU -> host
pointer) or numpy arrays (host pointer).  Compute calls take CUDA tensors.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MGB200_LIB: an alternative build of the same library (same-box A/B of compile-time
# kernel variants, scripts/); the default is the in-tree build
LIB_PATH = os.environ.get("MGB200_LIB") or os.path.join(_HERE, "libmgb200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2405_05047_b200/build.py` "
                      "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

MG_OK, MG_NOT_CONVERGED = 0, 1
MG_ERR_INVALID_ARG, MG_ERR_DIMENSION, MG_ERR_STRUCTURE, MG_ERR_NONFINITE = -1, -2, -3, -4
MG_ERR_SINGULAR, MG_ERR_STATE, MG_ERR_CUDA, MG_ERR_NCCL, MG_ERR_OOM = -5, -6, -7, -8, -9
MG_MEM_HOST, MG_MEM_DEVICE = 0, 1
MG_COARSE_DIRECT, MG_COARSE_SMOOTH = 0, 1
MG_GMRES, MG_RICHARDSON, MG_GMRES_DCGS2 = 0, 1, 2
MG_TRANSPORT_NCCL, MG_TRANSPORT_LOCAL, MG_TRANSPORT_IPC = 0, 1, 2
MG_PREC_FP64, MG_PREC_MIXED = 0, 1

STATUS_NAMES = {0: "MG_OK", 1: "MG_NOT_CONVERGED", -1: "MG_ERR_INVALID_ARG", -2: "MG_ERR_DIMENSION",
                -3: "MG_ERR_STRUCTURE", -4: "MG_ERR_NONFINITE", -5: "MG_ERR_SINGULAR", -6: "MG_ERR_STATE",
                -7: "MG_ERR_CUDA", -8: "MG_ERR_NCCL", -9: "MG_ERR_OOM"}


class mg_config(ctypes.Structure):
    _fields_ = [("n_levels", ctypes.c_int), ("block_size", ctypes.c_int), ("nu_pre", ctypes.c_int),
                ("nu_post", ctypes.c_int), ("omega", ctypes.c_double), ("coarse_mode", ctypes.c_int),
                ("coarse_sweeps", ctypes.c_int), ("use_graphs", ctypes.c_int), ("precision", ctypes.c_int)]


class mg_comm(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int), ("rank", ctypes.c_int), ("transport", ctypes.c_int),
                ("nccl_id", ctypes.c_ubyte * 128)]


class mg_solve_opts(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int), ("restart", ctypes.c_int), ("max_iter", ctypes.c_int),
                ("rtol", ctypes.c_double)]


class mg_solve_info(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("rel_residual", ctypes.c_double), ("converged", ctypes.c_int)]


class MgError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.mg_last_error().decode()
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}: {msg}")


_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_D = ctypes.c_double

_SIGS = {
    "mg_get_unique_id": [_P],
    "mg_create": [ctypes.POINTER(_P), ctypes.POINTER(mg_config), _I, _P, ctypes.POINTER(mg_comm)],
    "mg_create_level": [_P, _I, _I64, _I64, _I64],
    "mg_set_matrix": [_P, _I, _P, _P, _P, _I64, _I],
    "mg_update_matrix": [_P, _I, _P, _I],
    "mg_set_transfer": [_P, _I, _P, _P, _P, _I64, _I, _I],
    "mg_set_smoother": [_P, _I, _D, _I, _I, _P, _I],
    "mg_set_vanka": [_P, _I, _I64, _I, _P, _I],
    "mg_set_constraints": [_P, _P, _P, _P, _I64, _I],
    "mg_set_mean_constraint": [_P, _I, _P, _P, _I],
    "mg_project_zero_mean": [_P, _I, _P],
    "mg_make_consistent": [_P, _I, _P],
    "mg_setup": [_P],
    "mg_destroy": [_P],
    "mg_vcycle": [_P, _P, _P],
    "mg_vcycle_zero": [_P, _P, _P],
    "mg_solve": [_P, _P, _P, ctypes.POINTER(mg_solve_opts), ctypes.POINTER(mg_solve_info)],
    "mg_spmv": [_P, _I, _D, _P, _D, _P],
    "mg_sweep": [_P, _I, _P, _P, _P],
    "mg_residual": [_P, _I, _P, _P, _P],
    "mg_smooth": [_P, _I, _P, _P, _I],
    "mg_restrict": [_P, _I, _P, _P],
    "mg_prolong_add": [_P, _I, _P, _P],
    "mg_coarse_solve": [_P, _P, _P],
    "mg_apply_constraints": [_P, _P],
    "mg_condense_rhs": [_P, _P, _P],
    "mg_dot": [_P, _I, _P, _P, ctypes.POINTER(_D)],
    "mg_axpy": [_P, _I, _D, _P, _P],
}
for _name, _args in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = ctypes.c_int
_lib.mg_last_error.restype = ctypes.c_char_p
_lib.mg_last_error.argtypes = []
_lib.mg_version.restype = ctypes.c_char_p
_lib.mg_version.argtypes = []
_lib.mgi_launch_count.restype = ctypes.c_int64
_lib.mgi_launch_count.argtypes = [_P]
_lib.mgi_vcycle_profile.restype = ctypes.c_int
_lib.mgi_vcycle_profile.argtypes = [_P, _P, _P, _I, _P, _I]
_lib.mgi_level_info.restype = ctypes.c_int
_lib.mgi_level_info.argtypes = [_P, _I] + [ctypes.POINTER(ctypes.c_int64)] * 6

# --- Navier-Stokes step (include/ns.h) ---
class ns_step_info(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("rel_residual", ctypes.c_double), ("converged", ctypes.c_int),
                ("ms", ctypes.c_double * 4)]


_NS_SIGS = {
    "ns_create": [ctypes.POINTER(_P), _P, _I64, _I64],
    "ns_destroy": [_P],
    "ns_set_momentum": [_P, _P, _P, _P, _I64, _I],
    "ns_set_coupling": [_P, _P, _P, _P, _I64, _P, _P, _P, _I64, _I],
    "ns_set_mass": [_P, _P, _P, _I],
    "ns_set_dirichlet": [_P, _P, _P, _I64, _I],
    "ns_set_force": [_P, _P, _I],
    "ns_set_params": [_P, _D, _D, _D, _I, _I, _I],
    "ns_set_state": [_P, _P, _P, _P, _I],
    "ns_get_state": [_P, _P, _P, _P, _I],
    "ns_step": [_P, ctypes.POINTER(ns_step_info)],
    "ns_momentum": [_P, _P, _I],
    "ns_get_divergence": [_P, _P, _I],
}
for _name, _args in _NS_SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
_lib.ns_launch_count.restype = ctypes.c_int64
_lib.ns_launch_count.argtypes = [_P]

# --- Newton's method (include/newton.h) ---
MG_NEWTON_MAX_HIST = 32


class mg_newton_opts(ctypes.Structure):
    _fields_ = [("max_newton", ctypes.c_int), ("ntol", ctypes.c_double), ("atol", ctypes.c_double),
                ("reuse_rate", ctypes.c_double), ("lin", mg_solve_opts)]


class mg_newton_info(ctypes.Structure):
    _fields_ = [("newton_its", ctypes.c_int), ("gmres_its", ctypes.c_int), ("jacobians", ctypes.c_int),
                ("converged", ctypes.c_int),
                ("lin_its", ctypes.c_int * MG_NEWTON_MAX_HIST), ("res_norm", ctypes.c_double * (MG_NEWTON_MAX_HIST + 1)),
                ("ms_assemble", ctypes.c_double), ("ms_upload", ctypes.c_double), ("ms_solve", ctypes.c_double)]


MG_NEWTON_ASSEMBLE_FN = ctypes.CFUNCTYPE(ctypes.c_int, _P, ctypes.POINTER(_D), ctypes.POINTER(_D),
                                         ctypes.POINTER(ctypes.POINTER(_D)))
_lib.mg_newton.restype = ctypes.c_int
_lib.mg_newton.argtypes = [_P, _P, MG_NEWTON_ASSEMBLE_FN, _P, ctypes.POINTER(mg_newton_opts),
                           ctypes.POINTER(mg_newton_info)]

EXPORTED = sorted(list(_SIGS) + list(_NS_SIGS) + ["mg_last_error", "mg_version", "ns_launch_count", "mg_newton"])


def lib():
    return _lib


def _check(st: int, where: str, ok=(MG_OK,)) -> int:
    if st not in ok:
        raise MgError(st, where)
    return st


def _ptr(a, dtype=None):
    """(pointer, mem) of a torch tensor or numpy array (contiguity and dtype checked)."""
    if a is None:
        return None, MG_MEM_HOST
    if isinstance(a, np.ndarray):
        if dtype is not None and a.dtype != dtype:
            raise TypeError(f"expected {dtype}, got {a.dtype}")
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data, MG_MEM_HOST
    # torch tensor
    if not a.is_contiguous():
        raise ValueError("tensor must be contiguous")
    if dtype is not None and str(a.dtype).replace("torch.", "") != np.dtype(dtype).name:
        raise TypeError(f"expected {dtype}, got {a.dtype}")
    return a.data_ptr(), (MG_MEM_DEVICE if a.is_cuda else MG_MEM_HOST)


def _dptr(a) -> int:
    """device pointer of a CUDA fp64 tensor (compute calls)."""
    if not getattr(a, "is_cuda", False):
        raise TypeError("compute calls take CUDA tensors")
    p, _ = _ptr(a, np.float64)
    return p


def _same_mem(*arrs):
    mems = {_ptr(a)[1] for a in arrs if a is not None}
    if len(mems) > 1:
        raise ValueError("all arrays of one call must live in the same memory (host or device)")
    return mems.pop() if mems else MG_MEM_HOST


# Per-context facts the binding needs to check buffer sizes and devices before
# handing raw pointers to the C side (which trusts them): device, block size,
# number of levels; level row counts are queried (mgi_level_info) and cached.
_CTX: dict = {}
_NS: dict = {}


def _numel(a) -> int:
    return int(a.size) if isinstance(a, np.ndarray) else int(a.numel())


def _need(a, count: int, what: str, device=None):
    """Raise ValueError unless `a` holds at least `count` elements (and, for a
    CUDA tensor, lives on `device`)."""
    if a is None:
        return
    if _numel(a) < count:
        raise ValueError(f"{what}: {_numel(a)} elements, the call reads/writes {count}")
    if device is not None and getattr(a, "is_cuda", False) and a.device.index != device:
        raise ValueError(f"{what}: tensor on cuda:{a.device.index}, context on cuda:{device}")


def _rows(ctx, level) -> int:
    info = _CTX.get(ctx)
    if info is None:
        return -1
    n = info["rows"].get(level)
    if n is None:
        n = level_info(ctx, level)["n"] if 0 <= level < info["n_levels"] else -1
        if n > 0:
            info["rows"][level] = n
    return n


def _vec(ctx, level, a, what):
    """Device pointer of a level vector [n_rows(level) * bs] (size and device checked)."""
    p = _dptr(a)
    info = _CTX.get(ctx)
    if info is not None:
        n = _rows(ctx, level)
        _need(a, max(n, 0) * info["bs"], what, info["device"])
    return p


def _fine(ctx) -> int:
    info = _CTX.get(ctx)
    return info["n_levels"] - 1 if info is not None else 0


# ----------------------------------------------------------------------------
# the C ABI, same names
# ----------------------------------------------------------------------------

def mg_version() -> str:
    return _lib.mg_version().decode()


def mg_last_error() -> str:
    return _lib.mg_last_error().decode()


def mg_get_unique_id() -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    _check(_lib.mg_get_unique_id(buf), "mg_get_unique_id")
    return bytes(buf)


def mg_create(n_levels, block_size, *, nu_pre=2, nu_post=2, omega=0.8, coarse_mode=MG_COARSE_DIRECT,
              coarse_sweeps=20, use_graphs=True, device=0, stream=None, comm=None, precision=MG_PREC_FP64):
    """Returns an opaque context handle (int).  stream: a torch.cuda.Stream, a
    raw cudaStream_t int, or None (internal blocking stream).  comm: None
    (single GPU) or (nranks, rank, id_bytes[, transport])."""
    cfg = mg_config(n_levels, block_size, nu_pre, nu_post, omega, coarse_mode, coarse_sweeps, int(bool(use_graphs)),
                    precision)
    h = _P()
    s = getattr(stream, "cuda_stream", stream)
    cm = None
    if comm is not None:
        nranks, rank, uid = comm[:3]
        transport = comm[3] if len(comm) > 3 else MG_TRANSPORT_NCCL
        uid = bytes(uid).ljust(128, b"\0")[:128]
        cm = mg_comm(nranks, rank, transport, (ctypes.c_ubyte * 128)(*uid))
    _check(_lib.mg_create(ctypes.byref(h), ctypes.byref(cfg), device, s, ctypes.byref(cm) if cm else None),
           "mg_create")
    _CTX[h.value] = {"device": int(device), "bs": int(block_size), "n_levels": int(n_levels), "rows": {}}
    return h.value


def mg_create_level(ctx, level, n_rows_global, row_begin=0, row_end=None):
    _check(_lib.mg_create_level(ctx, level, n_rows_global, row_begin,
                                n_rows_global if row_end is None else row_end), "mg_create_level")


def mg_set_matrix(ctx, level, row_ptr, col, vals):
    mem = _same_mem(row_ptr, col, vals)
    nnzb = int(col.shape[0])
    _check(_lib.mg_set_matrix(ctx, level, _ptr(row_ptr, np.int64)[0], _ptr(col, np.int64)[0],
                              _ptr(vals, np.float64)[0], nnzb, mem), "mg_set_matrix")


def mg_update_matrix(ctx, level, vals):
    info = _CTX.get(ctx)
    if info is not None and 0 <= level < info["n_levels"]:
        _need(vals, level_info(ctx, level)["nnzb"] * info["bs"] ** 2, "mg_update_matrix vals", info["device"])
    p, mem = _ptr(vals, np.float64)
    _check(_lib.mg_update_matrix(ctx, level, p, mem), "mg_update_matrix")


def mg_set_transfer(ctx, fine_level, row_ptr, col, w, weights_per_entry=1):
    mem = _same_mem(row_ptr, col, w)
    _check(_lib.mg_set_transfer(ctx, fine_level, _ptr(row_ptr, np.int64)[0], _ptr(col, np.int64)[0],
                                _ptr(w, np.float64)[0], int(col.shape[0]), weights_per_entry, mem),
           "mg_set_transfer")


def mg_set_smoother(ctx, level, omega=0.0, nu_pre=-1, nu_post=-1, dinv=None):
    info = _CTX.get(ctx)
    if info is not None and dinv is not None:
        _need(dinv, max(_rows(ctx, level), 0) * info["bs"] ** 2, "mg_set_smoother dinv", info["device"])
    p, mem = _ptr(dinv, np.float64)
    _check(_lib.mg_set_smoother(ctx, level, omega, nu_pre, nu_post, p, mem), "mg_set_smoother")


def mg_set_vanka(ctx, level, patch_nodes):
    """patch_nodes: (n_patches, nloc) int64 rows of the level (None / empty: block-Jacobi)."""
    if patch_nodes is None or len(patch_nodes) == 0:
        _check(_lib.mg_set_vanka(ctx, level, 0, 1, None, MG_MEM_HOST), "mg_set_vanka")
        return
    pn = np.ascontiguousarray(patch_nodes, dtype=np.int64)
    _check(_lib.mg_set_vanka(ctx, level, pn.shape[0], pn.shape[1], pn.ctypes.data, MG_MEM_HOST), "mg_set_vanka")


def mg_set_constraints(ctx, row_ptr, col, w):
    mem = _same_mem(row_ptr, col, w)
    _check(_lib.mg_set_constraints(ctx, _ptr(row_ptr, np.int64)[0], _ptr(col, np.int64)[0],
                                   _ptr(w, np.float64)[0], int(col.shape[0]), mem), "mg_set_constraints")


def mg_set_mean_constraint(ctx, level, w, k):
    """Global constraint w^T x = 0 of a singular level operator with kernel
    span{k} (int p = 0 on every level); w=None removes it."""
    if w is None:
        _check(_lib.mg_set_mean_constraint(ctx, level, None, None, MG_MEM_HOST), "mg_set_mean_constraint")
        return
    mem = _same_mem(w, k)
    info = _CTX.get(ctx)
    if info is not None:
        n = max(_rows(ctx, level), 0) * info["bs"]
        _need(w, n, "mg_set_mean_constraint w", info["device"])
        _need(k, n, "mg_set_mean_constraint k", info["device"])
    _check(_lib.mg_set_mean_constraint(ctx, level, _ptr(w, np.float64)[0], _ptr(k, np.float64)[0], mem),
           "mg_set_mean_constraint")


def mg_project_zero_mean(ctx, level, x):
    _check(_lib.mg_project_zero_mean(ctx, level, _vec(ctx, level, x, "x")), "mg_project_zero_mean")


def mg_make_consistent(ctx, level, b):
    _check(_lib.mg_make_consistent(ctx, level, _vec(ctx, level, b, "b")), "mg_make_consistent")


def mg_setup(ctx):
    _check(_lib.mg_setup(ctx), "mg_setup")


def mg_destroy(ctx):
    _check(_lib.mg_destroy(ctx), "mg_destroy")
    _CTX.pop(ctx, None)


def mg_vcycle(ctx, x, b):
    f = _fine(ctx)
    _check(_lib.mg_vcycle(ctx, _vec(ctx, f, x, "x"), _vec(ctx, f, b, "b")), "mg_vcycle")


def mg_vcycle_zero(ctx, z, v):
    f = _fine(ctx)
    _check(_lib.mg_vcycle_zero(ctx, _vec(ctx, f, z, "z"), _vec(ctx, f, v, "v")), "mg_vcycle_zero")


def mg_solve(ctx, x, b, method=MG_GMRES, restart=30, max_iter=200, rtol=1e-10, raise_on_nonconv=False):
    """Returns (status, iterations, rel_residual, converged)."""
    o = mg_solve_opts(method, restart, max_iter, rtol)
    info = mg_solve_info()
    f = _fine(ctx)
    st = _lib.mg_solve(ctx, _vec(ctx, f, x, "x"), _vec(ctx, f, b, "b"), ctypes.byref(o), ctypes.byref(info))
    _check(st, "mg_solve", ok=(MG_OK,) if raise_on_nonconv else (MG_OK, MG_NOT_CONVERGED))
    return st, info.iterations, info.rel_residual, bool(info.converged)


def mg_spmv(ctx, level, alpha, x, beta, y):
    _check(_lib.mg_spmv(ctx, level, alpha, _vec(ctx, level, x, "x"), beta, _vec(ctx, level, y, "y")), "mg_spmv")


def mg_sweep(ctx, level, x, b, x_out):
    _check(_lib.mg_sweep(ctx, level, _vec(ctx, level, x, "x"), _vec(ctx, level, b, "b"),
                         _vec(ctx, level, x_out, "x_out")), "mg_sweep")


def mg_residual(ctx, level, x, b, r):
    _check(_lib.mg_residual(ctx, level, _vec(ctx, level, x, "x"), _vec(ctx, level, b, "b"),
                            _vec(ctx, level, r, "r")), "mg_residual")


def mg_smooth(ctx, level, x, b, sweeps=1):
    _check(_lib.mg_smooth(ctx, level, _vec(ctx, level, x, "x"), _vec(ctx, level, b, "b"), sweeps), "mg_smooth")


def mg_restrict(ctx, fine_level, r_fine, d_coarse):
    _check(_lib.mg_restrict(ctx, fine_level, _vec(ctx, fine_level, r_fine, "r_fine"),
                            _vec(ctx, fine_level - 1, d_coarse, "d_coarse")), "mg_restrict")


def mg_prolong_add(ctx, fine_level, y_coarse, x_fine):
    _check(_lib.mg_prolong_add(ctx, fine_level, _vec(ctx, fine_level - 1, y_coarse, "y_coarse"),
                               _vec(ctx, fine_level, x_fine, "x_fine")), "mg_prolong_add")


def mg_coarse_solve(ctx, d, y):
    _check(_lib.mg_coarse_solve(ctx, _vec(ctx, 0, d, "d"), _vec(ctx, 0, y, "y")), "mg_coarse_solve")


def mg_apply_constraints(ctx, x):
    f = _fine(ctx)
    _check(_lib.mg_apply_constraints(ctx, _vec(ctx, f, x, "x")), "mg_apply_constraints")


def mg_condense_rhs(ctx, b, b_bar):
    f = _fine(ctx)
    _check(_lib.mg_condense_rhs(ctx, _vec(ctx, f, b, "b"), _vec(ctx, f, b_bar, "b_bar")), "mg_condense_rhs")


def mg_dot(ctx, level, a, b) -> float:
    out = _D()
    _check(_lib.mg_dot(ctx, level, _vec(ctx, level, a, "a"), _vec(ctx, level, b, "b"), ctypes.byref(out)), "mg_dot")
    return out.value


def mg_axpy(ctx, level, alpha, x, y):
    _check(_lib.mg_axpy(ctx, level, alpha, _vec(ctx, level, x, "x"), _vec(ctx, level, y, "y")), "mg_axpy")


def mg_newton(ctx, x, assemble, n_fine_dof, level_sizes, *, max_newton=3, ntol=1e-8, atol=0.0, reuse_rate=0.0,
              method=MG_GMRES, restart=30, max_iter=200, rtol=1e-10):
    """Newton's method on the device (include/newton.h).  assemble(w, F, vals)
    is the caller's CPU assembly: w (n_fine_dof,) read-only view of the current
    iterate; F (n_fine_dof,) to fill with F(w), or None; vals a list of
    per-level views (level_sizes[l],) to fill with the Jacobian values, or
    None.  level_sizes: nnzb_l*bs*bs per level.  Returns (status, info dict)."""
    err = []

    def cb(_user, w_p, F_p, vals_p):
        try:
            w = np.ctypeslib.as_array(w_p, shape=(n_fine_dof,))
            F = np.ctypeslib.as_array(F_p, shape=(n_fine_dof,)) if bool(F_p) else None
            vals = None
            if bool(vals_p):
                vals = [np.ctypeslib.as_array(vals_p[l], shape=(int(sz),)) for l, sz in enumerate(level_sizes)]
            assemble(w, F, vals)
            return MG_OK
        except Exception as e:  # reported after the call returns
            err.append(e)
            return MG_ERR_INVALID_ARG

    fn = MG_NEWTON_ASSEMBLE_FN(cb)
    o = mg_newton_opts(max_newton, ntol, atol, reuse_rate, mg_solve_opts(method, restart, max_iter, rtol))
    info = mg_newton_info()
    st = _lib.mg_newton(ctx, _vec(ctx, _fine(ctx), x, "x"), fn, None, ctypes.byref(o), ctypes.byref(info))
    if err:
        raise err[0]
    _check(st, "mg_newton", ok=(MG_OK, MG_NOT_CONVERGED))
    k = info.newton_its
    return st, {"newton_its": k, "gmres_its": info.gmres_its, "jacobians": info.jacobians,
                "converged": bool(info.converged), "lin_its": list(info.lin_its[:k]),
                "res_norm": list(info.res_norm[:k + 1]), "ms_assemble": info.ms_assemble,
                "ms_upload": info.ms_upload, "ms_solve": info.ms_solve}


def launch_count(ctx) -> int:
    """Kernels launched by the context so far (eager + CUDA-graph kernel nodes)."""
    return int(_lib.mgi_launch_count(ctx))


def vcycle_profile(ctx, x, b, n_levels, zero=True) -> dict:
    """Per-level time split of one eager V-cycle (mgi_vcycle_profile), ms."""
    out = (ctypes.c_double * (2 * n_levels + 1))()
    _check(_lib.mgi_vcycle_profile(ctx, _dptr(x), _dptr(b), int(zero), out, 2 * n_levels + 1), "mgi_vcycle_profile")
    v = list(out)
    return {"level_ms": v[:n_levels], "halo_ms": v[n_levels:2 * n_levels], "agglomeration_ms": v[2 * n_levels]}


def level_info(ctx, level) -> dict:
    v = [ctypes.c_int64() for _ in range(6)]
    _check(_lib.mgi_level_info(ctx, level, *[ctypes.byref(x) for x in v]), "mgi_level_info")
    keys = ("n", "nnzb", "sell_entries", "nnz_p", "sell_entries_p", "sell_entries_r")
    return {k: x.value for k, x in zip(keys, v)}


from .solver import Multigrid  # noqa: E402,F401


# ----------------------------------------------------------------------------
# Navier-Stokes step (include/ns.h): same names, argument marshalling only
# ----------------------------------------------------------------------------

def ns_create(pressure_ctx, n_u, n_p):
    h = _P()
    _check(_lib.ns_create(ctypes.byref(h), pressure_ctx, int(n_u), int(n_p)), "ns_create")
    _NS[h.value] = {"n_u": int(n_u), "n_p": int(n_p)}
    return h


def ns_destroy(ctx):
    _check(_lib.ns_destroy(ctx), "ns_destroy")
    _NS.pop(getattr(ctx, "value", ctx), None)


def ns_set_momentum(ctx, row_ptr, col, vals):
    mem = _same_mem(row_ptr, col, vals)
    _check(_lib.ns_set_momentum(ctx, _ptr(row_ptr, np.int64)[0], _ptr(col, np.int64)[0], _ptr(vals, np.float64)[0],
                                int(col.shape[0]), mem), "ns_set_momentum")


def ns_set_coupling(ctx, pi, g):
    prp, pcol, pw = pi
    grp, gcol, gv = g
    mem = _same_mem(prp, pcol, pw, grp, gcol, gv)
    _check(_lib.ns_set_coupling(ctx, _ptr(prp, np.int64)[0], _ptr(pcol, np.int64)[0], _ptr(pw, np.float64)[0],
                                int(pcol.shape[0]), _ptr(grp, np.int64)[0], _ptr(gcol, np.int64)[0],
                                _ptr(gv, np.float64)[0], int(gcol.shape[0]), mem), "ns_set_coupling")


def ns_set_mass(ctx, m_u, m_p):
    sz = _ns_sizes(ctx)
    if sz is not None:
        _need(m_u, sz["n_u"], "ns_set_mass m_u")
        _need(m_p, sz["n_p"], "ns_set_mass m_p")
    mem = _same_mem(m_u, m_p)
    _check(_lib.ns_set_mass(ctx, _ptr(m_u, np.float64)[0], _ptr(m_p, np.float64)[0], mem), "ns_set_mass")


def ns_set_dirichlet(ctx, rows, vals):
    mem = _same_mem(rows, vals)
    _check(_lib.ns_set_dirichlet(ctx, _ptr(rows, np.int64)[0], _ptr(vals, np.float64)[0], int(rows.shape[0]), mem),
           "ns_set_dirichlet")


def _ns_sizes(ctx):
    return _NS.get(getattr(ctx, "value", ctx))


def ns_set_force(ctx, F):
    sz = _ns_sizes(ctx)
    if sz is not None and F is not None:
        _need(F, 3 * sz["n_u"], "ns_set_force F")
    p, mem = _ptr(F, np.float64)
    _check(_lib.ns_set_force(ctx, p, mem), "ns_set_force")


def ns_set_params(ctx, nu, dt, rtol=1e-6, restart=30, max_iter=200, timing=False):
    _check(_lib.ns_set_params(ctx, float(nu), float(dt), float(rtol), int(restart), int(max_iter), int(bool(timing))),
           "ns_set_params")


def _ns_state_sizes(ctx, u, p, q):
    sz = _ns_sizes(ctx)
    if sz is not None:
        _need(u, 3 * sz["n_u"], "u")
        _need(p, sz["n_p"], "p")
        _need(q, sz["n_p"], "q")


def ns_set_state(ctx, u, p, q):
    _ns_state_sizes(ctx, u, p, q)
    mem = _same_mem(u, p, q)
    _check(_lib.ns_set_state(ctx, _ptr(u, np.float64)[0], _ptr(p, np.float64)[0], _ptr(q, np.float64)[0], mem),
           "ns_set_state")


def ns_get_state(ctx, u, p, q):
    """Fill u [n_u*3], p, q [n_p] (numpy arrays or CUDA tensors, same memory)."""
    _ns_state_sizes(ctx, u, p, q)
    mem = _same_mem(u, p, q)
    _check(_lib.ns_get_state(ctx, _ptr(u, np.float64)[0], _ptr(p, np.float64)[0], _ptr(q, np.float64)[0], mem),
           "ns_get_state")


def ns_step(ctx):
    """One time step; returns (status, iterations, rel_residual, converged, ms[4])."""
    info = ns_step_info()
    st = _lib.ns_step(ctx, ctypes.byref(info))
    _check(st, "ns_step", ok=(MG_OK, MG_NOT_CONVERGED))
    return st, info.iterations, info.rel_residual, bool(info.converged), list(info.ms)


def ns_momentum(ctx, u_new):
    sz = _ns_sizes(ctx)
    if sz is not None:
        _need(u_new, 3 * sz["n_u"], "u_new")
    p, mem = _ptr(u_new, np.float64)
    _check(_lib.ns_momentum(ctx, p, mem), "ns_momentum")


def ns_get_divergence(ctx, d):
    sz = _ns_sizes(ctx)
    if sz is not None:
        _need(d, sz["n_p"], "d")
    p, mem = _ptr(d, np.float64)
    _check(_lib.ns_get_divergence(ctx, p, mem), "ns_get_divergence")


def ns_launch_count(ctx) -> int:
    return int(_lib.ns_launch_count(ctx))
from .navier_stokes import NavierStokes  # noqa: E402,F401
