"""Time the SELL-C transfer kernels (k_tsell) on every level of a config for
each (ks, nsl) variant (MGB200_TSELL_R / MGB200_TSELL_P, read at launch).
CUDA events around 20 launches each, median; alg. bytes per SURVEY §8(d)."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_05047_b200 as m  # noqa: E402
from problems import configs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
P = configs.build(cfg, keep_geometry=False)
S = m.Multigrid(P.levels, P.bs, omega=P.omega, H=P.fine.H)
os.environ["MGB200_TSELL"] = "0"             # read at setup: the fp64 SELL-32 transfer kernels
S_old = m.Multigrid(P.levels, P.bs, omega=P.omega, H=P.fine.H)
del os.environ["MGB200_TSELL"]
bs = P.bs
L = len(P.levels) - 1
peak = 6456.8
st = torch.cuda.current_stream()


def timeit(fn, reps=20):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


variants = ["1,1", "2,1", "4,1"]
for l in (L, L - 1):
    nf, nc = P.levels[l].n, P.levels[l - 1].n
    zp = m.level_info(S.ctx, l)["nnz_p"]
    r = torch.randn(nf * bs, dtype=torch.float64, device="cuda")
    d = torch.empty(nc * bs, dtype=torch.float64, device="cuda")
    x = torch.randn(nf * bs, dtype=torch.float64, device="cuda")
    rb = 12 * zp + 8 * (nc + 1) + 8 * bs * (nf + nc)
    pb = 12 * zp + 8 * (nf + 1) + 8 * bs * (nc + 2 * nf)
    tr = timeit(lambda: m.mg_restrict(S_old.ctx, l, r, d))
    tp = timeit(lambda: m.mg_prolong_add(S_old.ctx, l, d, x))
    print(f"{cfg} level {l} SELL-32 fp64 (round 1): restrict {tr:7.1f} us ({rb / tr / 1e3 / peak:.3f} of peak)  "
          f"prolong {tp:7.1f} us ({pb / tp / 1e3 / peak:.3f})", flush=True)
    for v in variants:
        os.environ["MGB200_TSELL_R"] = v
        os.environ["MGB200_TSELL_P"] = v
        tr = timeit(lambda: m.mg_restrict(S.ctx, l, r, d))
        tp = timeit(lambda: m.mg_prolong_add(S.ctx, l, d, x))
        print(f"{cfg} level {l} ks,nsl={v}: restrict {tr:7.1f} us ({rb / tr / 1e3 / peak:.3f} of peak)  "
              f"prolong {tp:7.1f} us ({pb / tp / 1e3 / peak:.3f})", flush=True)
