"""Profiling driver for ncu (run under `ncu --profile-from-start off`).

mode ns_step:    one step of the paper's NS cavity (Alg. 2; 545,025 velocity /
                 70,785 pressure nodes) inside the profiler range -> launch list.
mode c4ns_sweep: on the C4 channel's finest Newton Jacobian (1,045,686 DOFs):
                 one block-Jacobi sweep (k_sell_apply<3,SWEEP>) and one Vanka
                 sweep (residual + k_vanka_patch + k_vanka_update).
"""
import argparse
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2405_05047_b200 as m  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("mode", choices=["ns_step", "c4ns_sweep"])
a = ap.parse_args()

if a.mode == "ns_step":
    from problems import ns as NSP
    P = NSP.build_ns("ns")
    g = m.NavierStokes(P, rtol=1e-6)
    g.set_state(*NSP.initial_state(P))
    for _ in range(3):
        g.step()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    st = g.step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"ns step: {st[1]} pressure iterations", file=sys.stderr)
    g.close()
else:
    from problems import channel as C
    t = time.time()
    P = C.build("c4ns")
    u = C.initial_state(P)
    levels = C.with_values(P, C.jacobians(P, u, u))
    print(f"gen c4ns {time.time() - t:.1f}s", file=sys.stderr, flush=True)
    J = m.Multigrid(levels, 3, omega=P.omega)
    V = m.Multigrid(levels, 3, omega=1.0, vanka=True)
    L = len(levels) - 1
    N = P.n_dof
    xin = torch.randn(N, dtype=torch.float64, device="cuda")
    b = torch.randn(N, dtype=torch.float64, device="cuda")
    out = torch.empty_like(xin)
    for S in (J, V):
        m.mg_sweep(S.ctx, L, xin, b, out)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    m.mg_sweep(J.ctx, L, xin, b, out)
    m.mg_sweep(V.ctx, L, xin, b, out)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    J.close()
    V.close()
