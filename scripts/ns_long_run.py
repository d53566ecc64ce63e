"""The paper's whole NS experiment on the device: the 3D cavity of P:706 (Re 1000,
dt 1e-4), Alg. 2 from rest for `--steps` time steps (the paper: "8/dt = 40 000",
reading Z19), timing the run and sampling the kinetic energy 1/2 sum m_u |u|^2
and the discrete divergence |G^T u| of the projected velocity."""
import argparse
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2405_05047_b200 as m  # noqa: E402
from problems import ns as NSP  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=40000)
ap.add_argument("--sample", type=int, default=5000)
ap.add_argument("--vanka", action="store_true")
a = ap.parse_args()

P = NSP.build_ns("ns")
g = m.NavierStokes(P, rtol=1e-6, vanka=a.vanka, omega=0.8 if a.vanka else None)
g.set_state(*NSP.initial_state(P))
stream = torch.cuda.current_stream()
samples = []
its_total = 0
t0 = time.perf_counter()
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record(stream)
dev_ms = 0.0
for k in range(1, a.steps + 1):
    st, its, rel, conv, ms = g.step()
    its_total += its
    if not conv:
        raise RuntimeError(f"pressure solve did not converge at step {k}: {its} its, rel {rel}")
    if k % a.sample == 0 or k == a.steps:
        e1.record(stream)
        torch.cuda.synchronize()
        dev_ms += e0.elapsed_time(e1)
        u, p, q = g.get_state()
        d = g.divergence()
        samples.append({"step": k, "t": k * P.dt, "kinetic_energy": 0.5 * float(P.m_u @ (u * u).sum(1)),
                         "max_abs_u": float(np.abs(u).max()), "divergence_l2": float(np.linalg.norm(d)),
                         "pressure_its": its})
        print(json.dumps(samples[-1]), flush=True)
        e0.record(stream)
wall = time.perf_counter() - t0
print(json.dumps({"steps": a.steps, "smoother": "vanka" if a.vanka else "jacobi", "wall_s": wall,
                  "device_s": dev_ms / 1e3, "ms_per_step": dev_ms / a.steps,
                  "pressure_its_per_step": its_total / a.steps,
                  "paper_gpu_s_h100": 1660.0, "paper_cpu_s_8threads": 26754.2}), flush=True)
g.close()
