"""One rank of a multi-PROCESS distributed solve with the IPC transport
(include/mg.h MG_TRANSPORT_IPC), launched by tests/test_gpu_ipc.py.

usage: python ipc_worker.py <case> <P> <rank> <key-hex> <out.npz> [min_rows] [coarse_mode]
Builds the case, keeps its own rank's rows of the row partition,
and records: one V-cycle from a seeded x, one zero-guess V-cycle, one
GMRES+MG solve to 1e-10 (iterations, rel. residual), per-op results and the
per-level time split of one eager V-cycle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def main():
    name, P, rank, key, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), bytes.fromhex(sys.argv[4]), sys.argv[5]
    min_rows = int(sys.argv[6]) if len(sys.argv) > 6 else 32
    coarse_mode = int(sys.argv[7]) if len(sys.argv) > 7 else 0
    import torch
    torch.cuda.set_device(0)
    import paper_2405_05047_b200 as m
    from gpu_util import build_gpu, dev, host
    from mgtest_util import problem
    from problems.partition import partition
    if name.startswith("c5w"):
        # per-rank generated structured C5 (problems/structured.py): no global build at all
        from problems import structured as S
        levels, b_np, ranges = S.build_rank(P, rank, root=(2, 2, 4), R=int(name[3:]), min_rows_per_rank=min_rows)
        bs, n_dof = 4, levels[-1].n_global * 4
        mg = build_gpu(levels, bs, omega=S.OMEGA, H=None, coarse_mode=coarse_mode,
                       comm=(P, rank, key, m.MG_TRANSPORT_IPC))
        f0, f1 = levels[-1].row_begin, levels[-1].row_end
        b = dev(b_np)
    else:
        Pr = problem(name)
        bs, n_dof = Pr.bs, Pr.n_dof
        parts, extras, ranges = partition(Pr, P, min_rows_per_rank=min_rows, replicate_level0=(coarse_mode == 0),
                                          only_rank=rank)
        mg = build_gpu(parts[rank], bs, omega=Pr.omega, H=extras[rank][1], coarse_mode=coarse_mode,
                       comm=(P, rank, key, m.MG_TRANSPORT_IPC))
        f0, f1 = ranges[-1][rank]
        b = dev(extras[rank][0])
    x0 = np.random.default_rng(5).standard_normal(n_dof).reshape(-1, bs)[f0:f1].reshape(-1)
    x = dev(x0)
    m.mg_vcycle(mg.ctx, x, b)
    z = dev(np.zeros((f1 - f0) * bs))
    m.mg_vcycle_zero(mg.ctx, z, b)
    Lf = len(mg.n) - 1
    r = dev(np.zeros((f1 - f0) * bs))
    m.mg_residual(mg.ctx, Lf, x, b, r)
    dot = m.mg_dot(mg.ctx, Lf, r, r)
    xs = dev(np.zeros((f1 - f0) * bs))
    st, its, rel, conv = m.mg_solve(mg.ctx, xs, b, rtol=1e-10)
    if not name.startswith("c5w"):
        m.mg_apply_constraints(mg.ctx, xs)
    prof = m.vcycle_profile(mg.ctx, z, b, len(mg.n))
    np.savez(out, x=host(x), z=host(z), r=host(r), dot=dot, xs=host(xs), its=its, rel=rel, conv=conv,
             level_ms=np.array(prof["level_ms"]), halo_ms=np.array(prof["halo_ms"]),
             agg_ms=prof["agglomeration_ms"], f0=f0, f1=f1)
    mg.close()


if __name__ == "__main__":
    main()
