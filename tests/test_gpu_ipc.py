"""Multi-PROCESS row-partitioned solve on one B200 (VERDICT r1
"next" 3): P separate processes, one rank each, all on cuda:0, talking through
the IPC transport (CUDA IPC mailboxes + inter-process events + a shared-memory
host barrier; NCCL refuses several ranks on one GPU).  This is a real process
boundary, unlike the in-process LOCAL transport of test_gpu_distributed.py.

Same expectations as the LOCAL tests: the distributed V-cycle is BIT-IDENTICAL
to the single-GPU V-cycle (row sums keep CSR order after localisation, routed R
rows keep fine order, replicated coarse levels run the same kernels, the
all-reduce sums ranks in a fixed order), and GMRES+MG matches +-1 iteration."""
import os
import subprocess
import sys

import numpy as np
import pytest

from gpu_util import TOL_VCYCLE, build_gpu, dev, host
from mgtest_util import problem

import oracle

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def run_procs(name, P, tmp_path, min_rows=32, coarse_mode=0):
    key = os.urandom(16).hex()
    outs = [str(tmp_path / f"rank{r}.npz") for r in range(P)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "ipc_worker.py"), name, str(P), str(r), key,
                               outs[r], str(min_rows), str(coarse_mode)], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(P)]
    logs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(out)
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"rank {r} failed:\n{logs[r][-3000:]}"
    return [dict(np.load(o)) for o in outs]


@pytest.mark.parametrize("name,P", [("c3_small", 2), ("c2_small", 3), ("c4_small", 2), ("c3_mid", 4)])
def test_ipc_processes_vcycle_bitwise_and_gmres(name, P, tmp_path):
    import paper_2405_05047_b200 as m
    res = run_procs(name, P, tmp_path)
    Pr = problem(name)
    bs = Pr.bs
    x0 = np.random.default_rng(5).standard_normal(Pr.n_dof)
    s = build_gpu(Pr.levels, bs, omega=Pr.omega, H=Pr.fine.H)
    xs = dev(x0)
    m.mg_vcycle(s.ctx, xs, dev(Pr.b))
    zs = dev(np.zeros(Pr.n_dof))
    m.mg_vcycle_zero(s.ctx, zs, dev(Pr.b))
    got = np.concatenate([r["x"] for r in res])
    gotz = np.concatenate([r["z"] for r in res])
    assert np.array_equal(got, host(xs)), f"max diff {np.max(np.abs(got - host(xs))):.3e}"
    assert np.array_equal(gotz, host(zs))
    h = oracle.MgHierarchy.from_arrays(Pr.levels, omega=Pr.omega)
    exp = oracle.vcycle(h, len(Pr.levels) - 1, x0.copy(), Pr.b)
    assert np.linalg.norm(got - exp) <= TOL_VCYCLE * np.linalg.norm(exp)
    # all ranks agree on the all-reduced dot and on the GMRES decisions
    dots = [float(r["dot"]) for r in res]
    assert all(d == dots[0] for d in dots)
    rr = np.concatenate([r["r"] for r in res])
    assert abs(dots[0] - np.dot(rr, rr)) <= 1e-12 * dots[0]
    its = {int(r["its"]) for r in res}
    assert len(its) == 1 and all(bool(r["conv"]) for r in res)
    xsol = np.concatenate([r["xs"] for r in res])
    xe, ite, _, _ = oracle.gmres(h, Pr.b, rtol=1e-10)
    from oracle.mg import apply_H
    xe = apply_H(Pr.fine.H, xe, bs)
    assert abs(its.pop() - ite) <= 1
    assert np.linalg.norm(xsol - xe) <= 1e-8 * np.linalg.norm(xe)
    # the per-level split reports halo time on the distributed levels
    assert all(len(r["level_ms"]) == len(Pr.levels) for r in res)
    s.close()


def test_ipc_smoothing_coarse_mode(tmp_path):
    """Distributed level 0 (coarse problem smoothed): no agglomeration."""
    import paper_2405_05047_b200 as m
    name, P = "c3_small", 2
    res = run_procs(name, P, tmp_path, coarse_mode=1)
    Pr = problem(name)
    x0 = np.random.default_rng(5).standard_normal(Pr.n_dof)
    s = build_gpu(Pr.levels, Pr.bs, omega=Pr.omega, H=Pr.fine.H, coarse_mode=1)
    xs = dev(x0)
    m.mg_vcycle(s.ctx, xs, dev(Pr.b))
    got = np.concatenate([r["x"] for r in res])
    assert np.array_equal(got, host(xs))
    s.close()


@pytest.mark.parametrize("P", [1, 2, 3])
def test_ipc_structured_c5_per_rank_generation(P, tmp_path):
    """C5 weak-scaling path: each process generates only its own rows
    (problems/structured.py) -- the distributed V-cycle equals the single-GPU
    V-cycle of the globally generated system bit for bit, both match the
    oracle, and GMRES+MG agrees +-1 iteration with the oracle."""
    import paper_2405_05047_b200 as m
    from problems import structured as S
    R = 3
    res = run_procs(f"c5w{R}", P, tmp_path, min_rows=8) if P > 1 else None
    glob, b, _ = S.build_rank(1, 0, root=(2, 2, 4), R=R)
    n_dof = glob[-1].n * 4
    x0 = np.random.default_rng(5).standard_normal(n_dof)
    s = build_gpu(glob, 4, omega=S.OMEGA, H=None)
    xs = dev(x0)
    m.mg_vcycle(s.ctx, xs, dev(b))
    h = oracle.MgHierarchy.from_arrays(glob, omega=S.OMEGA)
    exp = oracle.vcycle(h, R, x0.copy(), b)
    assert np.linalg.norm(host(xs) - exp) <= TOL_VCYCLE * np.linalg.norm(exp)
    xe, ite, _, _ = oracle.gmres(h, b, rtol=1e-10)
    if res is None:
        x = dev(np.zeros(n_dof))
        st, its, rel, conv = m.mg_solve(s.ctx, x, dev(b), rtol=1e-10)
        assert conv and abs(its - ite) <= 1 and np.linalg.norm(host(x) - xe) <= 1e-8 * np.linalg.norm(xe)
    else:
        got = np.concatenate([r["x"] for r in res])
        assert np.array_equal(got, host(xs))
        its = {int(r["its"]) for r in res}
        assert len(its) == 1 and abs(its.pop() - ite) <= 1
        xsol = np.concatenate([r["xs"] for r in res])
        assert np.linalg.norm(xsol - xe) <= 1e-8 * np.linalg.norm(xe)
    s.close()
