"""Helpers for the -m gpu parity tests: device tensors, building the CUDA
multigrid and the oracle hierarchy from the same generated inputs, and the
scaled tolerances of reading Z11."""
import numpy as np

import oracle

TOL_OP = 1e-12      # per-op, normwise scaled (BASELINE north_star "1e-12 relative", reading Z11)
TOL_VCYCLE = 1e-10  # whole V-cycle, ||.||_2 relative (reading Z11)


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def host(t):
    import torch
    torch.cuda.synchronize()
    return t.double().cpu().numpy()


def build_gpu(levels, bs, *, omega=0.8, nu=(2, 2), coarse_mode=0, coarse_sweeps=20, use_graphs=True, H=None,
              omegas=None, **kw):
    from paper_2405_05047_b200 import Multigrid
    return Multigrid(levels, bs, omega=omega, nu_pre=nu[0], nu_post=nu[1], coarse_mode=coarse_mode,
                     coarse_sweeps=coarse_sweeps, use_graphs=use_graphs, H=H, omegas=omegas, **kw)


def build_oracle(levels, *, omega=0.8, nu=(2, 2), coarse="direct", coarse_sweeps=20, H=None):
    return oracle.MgHierarchy.from_arrays(levels, omega=omega, nu_pre=nu[0], nu_post=nu[1], coarse=coarse,
                                          coarse_sweeps=coarse_sweeps, H=H)


def absA_x(lv, x):
    """|A||x| by the oracle's spmv on absolute values (scale of Z11)."""
    return oracle.spmv(lv.n, lv.bs, lv.row_ptr, lv.col, np.abs(lv.val), np.abs(x))


def assert_close_scaled(got, exp, scale, tol=TOL_OP, what=""):
    err = np.max(np.abs(got - exp)) if got.size else 0.0
    sc = np.max(np.abs(scale)) if scale.size else 0.0
    assert err <= tol * max(sc, 1e-300), f"{what}: max err {err:.3e} > {tol:g} * scale {sc:.3e}"
