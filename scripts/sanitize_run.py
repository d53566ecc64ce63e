"""Exercise every library entry point on small configs (single GPU and LOCAL
distributed) for compute-sanitizer runs (memcheck / racecheck / initcheck /
synccheck)."""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2405_05047_b200 as m  # noqa: E402
from problems import configs  # noqa: E402
from problems.partition import partition  # noqa: E402

torch.cuda.set_device(0)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


for name in sys.argv[1:] or ["c1", "c3_small", "c5_small"]:
    P = configs.build(name)
    bs = P.bs
    for coarse_mode in (0, 1):
        S = m.Multigrid(P.levels, bs, omega=P.omega, H=P.fine.H, coarse_mode=coarse_mode)
        ctx = S.ctx
        for l, L in enumerate(P.levels):
            x = torch.randn(L.n * bs, dtype=torch.float64, device="cuda")
            b = torch.randn_like(x)
            r = torch.empty_like(x)
            m.mg_residual(ctx, l, x, b, r)
            m.mg_sweep(ctx, l, x, b, r)
            m.mg_spmv(ctx, l, 2.0, x, 0.5, r)
            m.mg_smooth(ctx, l, x, b, 3)
            m.mg_dot(ctx, l, x, b)
            if l > 0:
                d = torch.empty(P.levels[l - 1].n * bs, dtype=torch.float64, device="cuda")
                m.mg_restrict(ctx, l, r, d)
                m.mg_prolong_add(ctx, l, d, x)
        b = dev(P.b)
        z = torch.zeros_like(b)
        S.precondition(z, b)
        S.vcycle(z, b)
        z.zero_()
        S.solve(z, b, rtol=1e-8)
        z.zero_()
        S.solve(z, b, method=m.MG_RICHARDSON, rtol=1e-6, max_iter=20)
        S.apply_constraints(z)
        torch.cuda.synchronize()
        S.close()
    # distributed (LOCAL transport, 2 virtual ranks)
    parts, extras, ranges = partition(P, 2, min_rows_per_rank=16)
    key = os.urandom(16)
    out = [None, None]

    def work(r):
        torch.cuda.set_device(0)
        D = m.Multigrid(parts[r], bs, omega=P.omega, H=extras[r][1], comm=(2, r, key, m.MG_TRANSPORT_LOCAL))
        bb = dev(extras[r][0])
        zz = torch.zeros_like(bb)
        D.vcycle(zz, bb)
        zz.zero_()
        out[r] = D.solve(zz, bb, rtol=1e-8)
        D.apply_constraints(zz)
        torch.cuda.synchronize()
        D.close()
    th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join() for t in th]
    print(name, "ok", out, flush=True)
