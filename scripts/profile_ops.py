"""Profiling driver for ncu (run under `ncu --profile-from-start off`).

mode step:    one bench step (GMRES+MG solve from 0 + x <- Hx) inside the
              profiler range -> the launch list of a step.
mode kernels: the fine-level kernels once each (fused sweep, residual, SpMV,
              restriction, prolongation, A-free first sweep via a V-cycle
              from zero) -> `--set full` captures.
"""
import argparse
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2405_05047_b200 as m  # noqa: E402
from problems import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("mode", choices=["step", "kernels", "vcycle"])
ap.add_argument("--config", default="c3")
ap.add_argument("--mixed", action="store_true")
ap.add_argument("--orth", choices=["mgs", "dcgs2"], default="mgs", help="GMRES orthogonalisation (step mode)")
ap.add_argument("--level", type=int, default=-1, help="kernels mode: level to profile (default finest)")
a = ap.parse_args()

t = time.time()
P = configs.build(a.config, keep_geometry=False)
print(f"gen {a.config} {P.n_dof} DOFs {time.time() - t:.1f}s", file=sys.stderr, flush=True)
S = m.Multigrid(P.levels, P.bs, omega=P.omega, H=P.fine.H, precision=m.MG_PREC_MIXED if a.mixed else 0)
ctx = S.ctx
Lf = len(P.levels) - 1
b = torch.from_numpy(P.b).cuda()
x = torch.zeros_like(b)
meth = m.MG_GMRES_DCGS2 if a.orth == "dcgs2" else m.MG_GMRES
for _ in range(3):
    x.zero_()
    S.solve(x, b, method=meth)
torch.cuda.synchronize()
if a.mode == "step":
    torch.cuda.profiler.start()
    x.zero_()
    st, its, rel, conv = S.solve(x, b, method=meth)
    S.apply_constraints(x)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"step: {its} iterations, rel {rel:.2e}", file=sys.stderr)
elif a.mode == "vcycle":
    z = torch.zeros_like(b)
    for _ in range(3):
        S.precondition(z, b)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    S.precondition(z, b)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
else:
    if a.level >= 0:
        Lf = a.level
        nl = P.levels[Lf].n * P.bs
        b = torch.randn(nl, dtype=torch.float64, device="cuda")
    xin = torch.randn_like(b)
    out = torch.empty_like(b)
    nc = P.levels[Lf - 1].n * P.bs
    d = torch.empty(nc, dtype=torch.float64, device="cuda")
    m.mg_sweep(ctx, Lf, xin, b, out)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    m.mg_sweep(ctx, Lf, xin, b, out)            # k_sell_apply<3,2,1>
    m.mg_residual(ctx, Lf, xin, b, out)         # k_sell_apply<3,1,1>
    m.mg_spmv(ctx, Lf, 1.0, xin, 0.0, out)      # k_sell_apply<3,0,1>
    m.mg_restrict(ctx, Lf, out, d)              # k_transfer<3,1,0,1>
    m.mg_prolong_add(ctx, Lf, d, out)           # k_transfer<3,1,1,1>
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
