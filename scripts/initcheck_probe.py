"""initcheck probe: the NS pressure solve and a channel solve with CUDA graphs
off, so a flagged memcpy shows its call site."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2405_05047_b200 as m  # noqa: E402
from problems import channel as C  # noqa: E402
from problems import ns as NSP  # noqa: E402

torch.cuda.set_device(0)
mode = sys.argv[1]
graphs = len(sys.argv) > 2 and sys.argv[2] == "graphs"
if mode == "ns":
    P = NSP.build_ns("ns_small")
    g = m.NavierStokes(P, rtol=1e-6, use_graphs=graphs)
    g.set_state(*NSP.random_state(P, scale=0.3))
    g.step()
    g.step()
    g.close()
else:
    Pc = C.build("c4ns_small")
    u = C.initial_state(Pc)
    S = m.Multigrid(C.with_values(Pc, C.jacobians(Pc, u, u)), 3, omega=Pc.omega, H=Pc.fine.H, use_graphs=graphs)
    b = torch.from_numpy(-C.residual(Pc, u, u)).cuda()
    x = torch.zeros_like(b)
    S.solve(x, b, rtol=1e-8)
    x.zero_()
    S.solve(x, b, rtol=1e-8)
    S.close()
print("done", flush=True)
