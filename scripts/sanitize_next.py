"""compute-sanitizer driver for the NEXT-row entry points: the NS step
(include/ns.h), Newton (include/newton.h), the Vanka smoother (mg_set_vanka,
incl. mg_update_matrix rebuilds) and the single-CTA mean projection."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2405_05047_b200 as m  # noqa: E402
from problems import channel as C  # noqa: E402
from problems import configs  # noqa: E402
from problems import ns as NSP  # noqa: E402

torch.cuda.set_device(0)

# NS step, Jacobi and Vanka pressure smoother
P = NSP.build_ns("ns_small")
for vk in (False, True):
    g = m.NavierStokes(P, rtol=1e-6, vanka=vk, omega=0.8 if vk else None, timing=True)
    g.set_state(*NSP.random_state(P, scale=0.3))
    g.momentum()
    g.step()
    g.step()
    g.divergence()
    g.get_state()
    g.close()
print("ns ok", flush=True)

# Newton on the channel (Jacobian reuse on), Vanka on every level
Pc = C.build("c4ns_small")
u = C.initial_state(Pc)
for vk in (False, True):
    S = m.Multigrid(C.with_values(Pc, C.jacobians(Pc, u, u)), 3, omega=Pc.omega, H=Pc.fine.H, vanka=vk)
    x = torch.from_numpy(u.reshape(-1).copy()).cuda()
    S.newton(x, C.assemble_callback(Pc, u), max_newton=4, ntol=1e-8, reuse_rate=0.3 if vk else 0.0)
    L = len(Pc.levels) - 1
    xin = torch.randn_like(x)
    out = torch.empty_like(x)
    m.mg_sweep(S.ctx, L, xin, x, out)
    m.mg_axpy(S.ctx, L, 0.5, xin, out)
    S.close()
print("newton ok", flush=True)

# Vanka on 3D bs 4 (m = 32) and bs 1, mixed precision
for name in ("c5_small", "c2_small"):
    Pp = configs.build(name)
    for prec in (0, 1):
        S = m.Multigrid(Pp.levels, Pp.bs, omega=Pp.omega, H=Pp.fine.H, vanka=True, precision=prec)
        b = torch.from_numpy(Pp.b).cuda()
        z = torch.zeros_like(b)
        S.solve(z, b, rtol=1e-8)
        S.close()
print("vanka ok", flush=True)
