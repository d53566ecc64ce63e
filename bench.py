#!/usr/bin/env python
"""bench.py -- throughput of the fp64 GMG hot path of arXiv 2405.05047 on B200.

A step = one pass of the whole hot path over the
synthetic workload: GMRES(30) preconditioned by one V(2,2)-cycle per
iteration (Alg. gmg; GMRES P:343-347), from x0 = 0 to a 1e-10
relative residual, followed by the hanging-node interpolation x <- H x
(P:144).  Metric (BASELINE.json): V-cycles/s (= preconditioner applications
per second inside the solve), with DOF-cycles/s and the fine-level fused
smoother's HBM roofline fraction alongside.

Default workload: C3 -- 3D Q1 linear elasticity, 3x3 blocks,
face-refined octree with hanging nodes, 10,329,843 DOFs, 7 levels: the
north-star ">=10M-DOF adaptive 3D mesh" configuration.  Inputs (7 GB of
operators) are far larger than L2 (126 MB), so no explicit flush is needed.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]
        N > 1: torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "c3": "C3: 3D Q1 elasticity (M + dt^2 K_e), 3x3 blocks, face-refined octree (9^3 root, 6 band steps), "
          "hanging nodes, 7 levels, GMRES(30)+V(2,2) block-Jacobi omega=0.5, direct coarse solve",
    "c2": "C2: 2D transport-diffusion Q1, quadtree band-refined toward y=0 (32^2 root, 7 steps), 8 levels, "
          "GMRES(30)+V(2,2) Jacobi omega=0.8, direct coarse solve",
    "c1": "C1: 2D transport-diffusion Q1, uniform 32x32 (1089 DOFs), 4 levels",
    "c4": "C4: 2D NS-shaped generalised Stokes (PSPG, eps M_p), Q1 3x3 blocks (p,u,v), lid cavity band-refined "
          "toward the lid (32^2 root, 6 steps), 7 levels, per-component transfers, GMRES(30)+V(2,2) omega=0.8",
    "e6": "N4: the paper's 6-component elasticity system (u, v), backward Euler (P:441-445), 6x6 blocks, "
          "Table ndofs face mesh L5 (8^3 root, K=1 band toward x=0): 1,035,030 DOFs as in P:537, "
          "GMRES(30)+V(2,2) block-Jacobi omega=0.5, direct coarse solve",
    "c4ns": "C4 (SURVEY §8(d)): 2D instationary Navier-Stokes flow around a cylinder (DFG 2D-2 channel, "
            "Re 100, disk as Dirichlet obstacle), equal-order Q1 (PSPG + streamline diffusion), 3x3 blocks, "
            "quadtree band-refined toward the cylinder (44x8 root, 2 uniform + 6 band steps), 9 levels, backward "
            "Euler dt=0.01, Newton (CPU-assembled Jacobians re-uploaded every step) + GMRES(30)/V(2,2) omega=0.6",
    "ns": "N2: the paper's explicit pressure-correction Navier-Stokes step (Alg. 2) on its 3D driven cavity "
          "(0,1)^2x(0,2), graded 32x32x64 pressure mesh (Q1, 70,785 nodes) and Q1-iso-Q2 velocity (545,025 "
          "nodes), Re 1000, dt 1e-4, pressure Poisson GMRES+MG with int p = 0 to rtol 1e-6",
    "e6_edge": "N4: the paper's 6-component elasticity (u, v) on Table ndofs edge mesh L6 (8^3 root, K=1 band toward "
               "x=y=0): 209,910 DOFs as in P:554, GMRES(30)+V(2,2) block-Jacobi omega=0.5",
    "e6_vertex": "N4: the paper's 6-component elasticity (u, v) on Table ndofs vertex mesh L6 (band toward the vertex "
                 "0): 22,494 DOFs as in P:571, GMRES(30)+V(2,2) block-Jacobi omega=0.5",
    "td_l10": "the paper's transport-diffusion case L10 (P:402-405): uniform 1024x1024 Q1 mesh of the unit square, "
              "1,050,625 DOFs, M^l/dt + lambda K + B (lambda 0.01, b = (0,-1), dt 0.02), 9 levels, GMRES(30)+V(2,2) "
              "Jacobi omega 0.8, direct coarse solve",
    "c5": "C5 weak scaling: 3D NS-shaped generalised Stokes (PSPG, eps M_p), Q1 4x4 blocks (p,u,v,w), "
          "(0,1)^2x(0,2) lid cavity of equal cubic cells, root*2^R per GPU count (P=1 128^2x256 = 17.1M DOFs, "
          "P=2 160^2x320, P=4 192^2x384, P=8 256^2x512 = 135.5M DOFs), lexicographic numbering, each rank "
          "generates its own z-slab of every level, per-component transfers, GMRES(30)+V(2,2) omega=0.6",
    "pres": "N2: pure-Neumann pressure Poisson of the projection step (Alg. 2 Step 2, P:618-636) on the NS cavity "
            "(0,1)^2x(0,2), Q1, 128x128x256 cells (4,293,249 DOFs), 6 levels, int p = 0 imposed on every level "
            "(P:158), GMRES(30)+V(2,2) Jacobi omega=0.8, regularised direct coarse solve",
}


WEAK_CONFIGS = {"c5"}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# the paper's own numbers for the same workload (other hardware and code: context)
PAPER_CONTEXT = {
    "td_l10": {"gpu_ms_per_solve_h100": 90.0, "cpu_ms_per_solve_8threads": 3047.5,
               "source": "P:405: 9.0 s (GPU) / 304.75 s (CPU) per 100 time steps = 100 linear solves"},
    "e6_edge": {"gpu_ms_per_solve_h100": 147.0, "cpu_ms_per_solve_8threads": 3055.8,
                "source": "P:554: 14.7 s (GPU) / 305.58 s (CPU) per 100 time steps"},
    "e6_vertex": {"gpu_ms_per_solve_h100": 79.0, "cpu_ms_per_solve_8threads": 282.1,
                  "source": "P:571: 7.9 s (GPU) / 28.21 s (CPU) per 100 time steps"},
    "e6": {"gpu_ms_per_solve_h100": 1225.7, "cpu_ms_per_solve_8threads": 44319.4,
           "source": "P:537: 122.57 s (GPU) / 4431.94 s (CPU) per 100 time steps"},
}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def level_bytes(info, bs, zero, vb=8):
    """Algorithmic bytes of one V(2,2) on one level; info from mgi_level_info.
    vb: bytes per stored matrix value (8 fp64, 4 in the mixed-precision V-cycle)."""
    n, z = info["n"], info["nnzb"]
    a_stream = z * (vb * bs * bs + 4) + 8 * (n + 1)
    sweep = a_stream + 8 * bs * n * 3 + 8 * bs * bs * n
    sweep0 = 16 * bs * n + 8 * bs * bs * n
    resid = a_stream + 24 * bs * n
    return sweep, sweep0, resid


def vcycle_bytes(infos, bs, nu=(2, 2), zero=True, coarse_direct=True, vb=8):
    """Algorithmic bytes of one V-cycle (fine level from zero guess if zero)."""
    total = 0
    L = len(infos) - 1
    for l in range(L, 0, -1):
        sweep, sweep0, resid = level_bytes(infos[l], bs, zero, vb)
        first_zero = zero or l < L
        total += (sweep0 + (nu[0] - 1) * sweep) if first_zero else nu[0] * sweep
        total += resid + nu[1] * sweep
        nf, nc = infos[l]["n"], infos[l - 1]["n"]
        zp = infos[l]["nnz_p"]
        total += 12 * zp + 8 * (nc + 1) + 8 * bs * (nf + nc)         # restrict
        total += 12 * zp + 8 * (nf + 1) + 8 * bs * (nc + 2 * nf)     # prolong-add
    n0 = infos[0]["n"] * bs
    total += 8 * n0 * n0 if coarse_direct else 0
    return total


def build_problem(name):
    from problems import configs
    t = time.time()
    P = configs.build({"e6": "e6_face_l5", "e6_edge": "e6_edge_l6", "e6_vertex": "e6_vertex_l6",
                       "pres": "pres_l5"}.get(name, name), keep_geometry=False)
    log(f"[bench] generated {name}: {P.n_dof} DOFs, levels {[l.n for l in P.levels]} in {time.time() - t:.1f}s")
    return P


class StructuredProblem:
    """This rank's part of the per-rank generated C5 workload, with the fields
    of problems.configs.Problem that bench.py uses."""

    def __init__(self, levels, b, ranges, ws, n_dof):
        from problems import structured as S
        self.levels, self.b, self.ranges = levels, b, ranges
        self.bs, self.omega, self.nu_pre, self.nu_post = 4, S.OMEGA, 2, 2
        self.n_dof = n_dof
        self.level_kinds = (["single"] * len(levels) if ws == 1 else
                            ["replicated" if all(r == (0, L.n_global) for r in ranges[l]) else "distributed"
                             for l, L in enumerate(levels)])

    @property
    def fine(self):
        class _F:
            H = None
            mean_w = None
        return _F()


def build_structured(args, ws, rank):
    from problems import structured as S
    if ws not in S.C5_WEAK:
        raise SystemExit(f"c5 weak scaling is defined for 1/2/4/8 ranks (SURVEY §8(d)), not {ws}")
    t = time.time()
    levels, b, ranges = S.build_rank(ws, rank, min_rows_per_rank=args.min_rows_per_rank)
    P = StructuredProblem(levels, b, ranges, ws, S.n_dof(ws))
    log(f"[bench] rank {rank}: generated its C5 rows ({levels[-1].n * 4} of {P.n_dof} DOFs, levels "
        f"{[L.n for L in levels]}) in {time.time() - t:.1f}s")
    return P


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


_ORACLE_H = {}


def oracle_vcycle_rate(P, n_cycles=1, warmup=0, threads=None):
    """The oracle (as it stands) timed on the host cores: V-cycles/s of
    GMG(L, 0, b) -- the preconditioner application of one GMRES step."""
    import oracle
    cores = threads or cpu_cores()
    oracle.set_threads(cores)
    if id(P) in _ORACLE_H:
        h = _ORACLE_H[id(P)]
        L = len(P.levels) - 1
        times = []
        for _ in range(n_cycles):
            t = time.perf_counter()
            oracle.vcycle(h, L, np.zeros_like(P.b), P.b)
            times.append(time.perf_counter() - t)
        return times, cores
    t = time.time()
    mean = [(L.mean_w, L.mean_k) for L in P.levels] if P.fine.mean_w is not None else None
    h = oracle.MgHierarchy.from_arrays(P.levels, omega=P.omega, nu_pre=P.nu_pre, nu_post=P.nu_post, mean=mean)
    _ORACLE_H[id(P)] = h
    log(f"[bench] oracle setup {time.time() - t:.1f}s on {cores} cores")
    L = len(P.levels) - 1
    for _ in range(warmup):
        oracle.vcycle(h, L, np.zeros_like(P.b), P.b)
    times = []
    for _ in range(n_cycles):
        t = time.perf_counter()
        oracle.vcycle(h, L, np.zeros_like(P.b), P.b)
        times.append(time.perf_counter() - t)
    return times, cores


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    P = build_structured(args, 1, 0) if args.config in WEAK_CONFIGS else build_problem(args.config)
    times, cores = oracle_vcycle_rate(P, n_cycles=args.steps, warmup=args.warmup)
    tot = sum(times)
    val = args.steps / tot
    line = {
        "impl": "reference", "metric": "V-cycles/s", "value": val, "unit": "V-cycles/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
        "scaling": "weak" if args.config in WEAK_CONFIGS else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "n_dof": P.n_dof, "levels": len(P.levels)},
        "cpu_baseline": {"value": val, "unit": "V-cycles/s", "cores": cores, "kind": "oracle",
                         "sample": f"each step = one oracle V(2,2) GMG(L,0,b) on the full {args.config} "
                                   f"({P.n_dof} DOFs): one preconditioner application of the GMRES step"},
        "e2e": {"value": val, "unit": "V-cycles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "dof_cycles_per_s": val * P.n_dof,
    }
    print(json.dumps(line), flush=True)


def init_dist(ws, local):
    """One process per rank.  One GPU per rank: torch.distributed over NCCL for
    the plumbing and the library's NCCL transport.  Fewer GPUs than ranks
    (e.g. the one-GPU build box; NCCL refuses two ranks on one device): gloo
    for the plumbing and the library's IPC transport (CUDA IPC mailboxes,
    inter-process events, shared-memory barrier).  MGB200_TRANSPORT=ipc forces
    the IPC transport.  Returns (device, transport, reduction device)."""
    import torch
    import torch.distributed as dist
    import paper_2405_05047_b200 as mg
    ngpu = torch.cuda.device_count()
    ipc = ngpu < ws or os.environ.get("MGB200_TRANSPORT", "").lower() == "ipc"
    dev = local % max(ngpu, 1)
    torch.cuda.set_device(dev)
    if ipc:
        dist.init_process_group("gloo")
        return dev, mg.MG_TRANSPORT_IPC, "cpu"
    dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    return dev, mg.MG_TRANSPORT_NCCL, "cuda"


def group_key(transport):
    """128-byte group key from rank 0: an NCCL unique id, or random bytes naming
    the IPC transport's shared-memory segment."""
    import torch
    import paper_2405_05047_b200 as mg
    rank = torch.distributed.get_rank()
    box = [None]
    if rank == 0:
        box[0] = mg.mg_get_unique_id() if transport == mg.MG_TRANSPORT_NCCL else os.urandom(128)
    torch.distributed.broadcast_object_list(box, src=0)
    return box[0]


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    dev, transport, red = local, None, "cuda"
    if ws > 1:
        dev, transport, red = init_dist(ws, local)
        # host threads per rank for the generator's OpenMP helper
        os.environ["OMP_NUM_THREADS"] = str(max(1, cpu_cores() // ws))
    torch.cuda.set_device(dev)
    import paper_2405_05047_b200 as mg

    cleanup = None
    if args.config in WEAK_CONFIGS:
        # C5 weak scaling: every rank generates its own rows of every level
        # (problems/structured.py), ~17M DOFs per rank, no data-path broadcast
        P = build_structured(args, ws, rank)
    elif ws > 1:
        # one generation on rank 0, arrays shared through memory-mapped .npy files
        from problems.share import shared_build

        def bcast(tok):
            box = [tok]
            torch.distributed.broadcast_object_list(box, src=0)
            return box[0]
        P, cleanup = shared_build(lambda: build_problem(args.config), args.config, rank,
                                  torch.distributed.barrier, bcast)
    else:
        P = build_problem(args.config)
    bs = P.bs
    prec = mg.MG_PREC_MIXED if args.precision == "mixed" else mg.MG_PREC_FP64
    vb = 4 if args.precision == "mixed" else 8
    stream = torch.cuda.current_stream()
    t = time.time()
    if args.config in WEAK_CONFIGS:
        H = None
        b_np = P.b
        n_global = P.n_dof
        comm = (ws, rank, group_key(transport), transport) if ws > 1 else None
        solver = mg.Multigrid(P.levels, bs, omega=P.omega, nu_pre=P.nu_pre, nu_post=P.nu_post, H=None,
                              device=dev, stream=stream, use_graphs=not args.no_graphs, precision=prec, comm=comm)
        level_kinds = P.level_kinds
    elif ws > 1:
        # row partition: nnz-balanced Morton splitters on every
        # level; levels with < 16k rows per rank are replicated (agglomerated)
        from problems.partition import partition
        parts, extras, ranges = partition(P, ws, min_rows_per_rank=args.min_rows_per_rank, only_rank=rank)
        uid = group_key(transport)
        levels, (b_np, H) = parts[rank], extras[rank]
        del parts, extras
        cleanup()
        solver = mg.Multigrid(levels, bs, omega=P.omega, nu_pre=P.nu_pre, nu_post=P.nu_post, H=H, device=dev,
                              stream=stream, use_graphs=not args.no_graphs, precision=prec,
                              comm=(ws, rank, uid, transport))
        n_global = P.n_dof
        level_kinds = ["replicated" if all(r == (0, P.levels[l].n) for r in ranges[l]) else "distributed"
                       for l in range(len(P.levels))]
    else:
        H = P.fine.H
        solver = mg.Multigrid(P.levels, bs, omega=P.omega, nu_pre=P.nu_pre, nu_post=P.nu_post, H=H,
                              device=dev, stream=stream, use_graphs=not args.no_graphs, precision=prec)
        b_np = P.b
        n_global = P.n_dof
        level_kinds = ["single"] * len(P.levels)
    torch.cuda.synchronize()
    log(f"[bench] rank {rank}: library setup {time.time() - t:.1f}s")
    ctx = solver.ctx
    L = len(P.levels) - 1
    infos = [mg.level_info(ctx, l) for l in range(L + 1)]
    N = infos[L]["n"] * bs                      # this rank's fine DOFs
    b_host = torch.from_numpy(np.ascontiguousarray(b_np)).pin_memory()
    b = b_host.cuda()
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    orth_method = {"mgs": mg.MG_GMRES, "dcgs2": mg.MG_GMRES_DCGS2}
    opts = dict(restart=30, max_iter=200, rtol=args.rtol, method=orth_method[args.orth])

    def step(xv, bv):
        xv.zero_()
        st, its, rel, conv = solver.solve(xv, bv, **opts)
        if not conv:
            raise RuntimeError(f"solve did not converge: {its} its, rel {rel:.3e}")
        if H is not None:
            solver.apply_constraints(xv)
        return its, rel

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        its0, rel0 = step(x, b)
    # ---------------- timed region (device events, max over ranks) ------------
    sampler = ClockSampler(dev)
    sampler.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    l0 = mg.launch_count(ctx)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    ncu_range = os.environ.get("MGB200_PROFILE_TIMED") == "1"   # ncu --profile-from-start off: timed steps only
    if ncu_range:
        torch.cuda.profiler.start()
    e0.record(stream)
    total_its = 0
    for _ in range(args.steps):
        its, rel = step(x, b)
        total_its += its
    e1.record(stream)
    torch.cuda.synchronize()
    if ncu_range:
        torch.cuda.profiler.stop()
    barrier()
    t_ms = e0.elapsed_time(e1)
    launches = mg.launch_count(ctx) - l0
    clocks = sampler.stop()
    if ws > 1:
        tt = torch.tensor([t_ms, float(launches)], dtype=torch.float64, device=red)
        tmax = tt[:1].clone()
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(tt[1:], op=torch.distributed.ReduceOp.SUM)
        t_ms, launches = float(tmax[0]), int(tt[1])
    # every rank takes part in the same global V-cycles (strong scaling):
    # units = global V-cycles of the whole job
    value = total_its / (t_ms / 1e3)
    # a fixed global problem (C2/C3/...) is strong scaling at every N; C5's
    # per-rank generated rows are weak scaling
    scaling = "weak" if args.config in WEAK_CONFIGS else "strong"

    # ---------------- e2e: host buffers through the public API -----------------
    # Every step copies its rhs host -> device and its solution device -> host
    # (pinned buffers).  Double-buffered: step k+1's upload and step k's download
    # run on a copy stream while step k / k+1 solve.
    xs = [x, torch.zeros_like(x)]
    bd = [b, torch.empty_like(b)]
    x_hosts = [torch.empty(N, dtype=torch.float64).pin_memory() for _ in range(2)]
    cs = torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    bd[1].copy_(b)
    step(xs[1], bd[1])        # warm the second buffer pair (its CUDA graphs are captured here)
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    e2e_its = 0
    with torch.cuda.stream(cs):
        bd[0].copy_(b_host, non_blocking=True)
        ev_in[0].record(cs)
    for k in range(args.steps):
        cur, nxt = k % 2, (k + 1) % 2
        if k + 1 < args.steps:
            with torch.cuda.stream(cs):
                bd[nxt].copy_(b_host, non_blocking=True)   # step k-1 (its user) has finished
                ev_in[nxt].record(cs)
        stream.wait_event(ev_in[cur])
        if k >= 2:
            stream.wait_event(ev_out[cur])                  # x_hosts[cur]'s download of step k-2 done
        its, _ = step(xs[cur], bd[cur])
        ev_out[cur].record(stream)
        with torch.cuda.stream(cs):
            cs.wait_event(ev_out[cur])
            x_hosts[cur].copy_(xs[cur], non_blocking=True)
            ev_out[cur].record(cs)
        e2e_its += its
    stream.wait_stream(cs)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    if ws > 1:
        tt = torch.tensor([e2e_ms], dtype=torch.float64, device=red)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(tt[0])
    e2e_val = e2e_its / (e2e_ms / 1e3)

    # ---------------- pure V-cycle rate (graph replay of mg_vcycle_zero) -------
    # SURVEY §8(d) protocol: 5 warm-up cycles, then 5 batches of 50 graph-launched
    # mg_vcycle_zero calls timed with CUDA events; the median batch is reported
    z = torch.zeros_like(x)
    for _ in range(5):
        solver.precondition(z, b)
    nv, batches = 50, []
    for _ in range(5):
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(nv):
            solver.precondition(z, b)
        e1.record(stream)
        torch.cuda.synchronize()
        batches.append(e0.elapsed_time(e1) / nv)
    vc_ms = statistics.median(batches)
    vc_bytes = vcycle_bytes(infos, bs, (P.nu_pre, P.nu_post), zero=True, vb=vb)

    # ---------------- value-only re-upload of every level (Newton / time step) --
    upd = None
    if ws == 1:
        dvals = [torch.from_numpy(np.ascontiguousarray(Lv.val.reshape(-1))).cuda() for Lv in P.levels]
        for l in range(L + 1):
            mg.mg_update_matrix(ctx, l, dvals[l])          # warm
        torch.cuda.synchronize()
        t = time.perf_counter()
        for l in range(L + 1):
            mg.mg_update_matrix(ctx, l, dvals[l])
        torch.cuda.synchronize()
        upd_ms = 1e3 * (time.perf_counter() - t)
        hv = np.ascontiguousarray(P.levels[L].val.reshape(-1))
        hp = torch.from_numpy(hv).pin_memory()

        def _host_upd(src):  # best of 3 (the first call also sizes the staging buffers)
            best = float("inf")
            for _ in range(3):
                torch.cuda.synchronize()
                t = time.perf_counter()
                mg.mg_update_matrix(ctx, L, src)
                torch.cuda.synchronize()
                best = min(best, 1e3 * (time.perf_counter() - t))
            return best
        fin_pageable, fin_pinned = _host_upd(hv), _host_upd(hp)
        gb = hv.nbytes / 1e9
        upd = {"all_levels_device_ms": upd_ms, "finest_from_host_ms": fin_pageable,
               "finest_from_pinned_host_ms": fin_pinned, "finest_gb": gb,
               "finest_from_host_gbs": gb / (fin_pageable / 1e3),
               "finest_from_pinned_host_gbs": gb / (fin_pinned / 1e3),
               "note": "mg_update_matrix of the finest level from host memory (pageable numpy / pinned torch), "
                       "wall time of the whole call incl. device scatter through the entry map, device D^-1 "
                       "and the host sync, best of 3; all_levels_device_ms = every level from device memory; "
                       "graphs stay valid"}
        del hp
        del dvals

    # ---------------- per-level split of one (eager) V-cycle --------------------
    prof = mg.vcycle_profile(ctx, z, b, L + 1)

    # ---------------- dominant kernel: fine-level fused block-Jacobi sweep -----
    peak, peak_src = measured_peaks()
    xin = torch.randn(N, dtype=torch.float64, device="cuda")
    xout = torch.empty_like(xin)
    for _ in range(3):
        mg.mg_sweep(ctx, L, xin, b, xout)
    ns = 20
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ns)]
    torch.cuda.synchronize()
    for a, c in evs:
        a.record(stream)
        mg.mg_sweep(ctx, L, xin, b, xout)
        c.record(stream)
    torch.cuda.synchronize()
    sw_ms = sum(a.elapsed_time(c) for a, c in evs) / ns
    sweep_b, _, _ = level_bytes(infos[L], bs, False, vb)
    achieved = sweep_b / (sw_ms / 1e3) / 1e9
    # plain SpMV y = A x of the finest level (the GMRES operator; BASELINE metric
    # "SpMV HBM GB/s as % of peak"): z (8 bs^2 + 4) + 8 (n + 1) + 16 bs n bytes
    for _ in range(3):
        mg.mg_spmv(ctx, L, 1.0, xin, 0.0, xout)
    torch.cuda.synchronize()
    for a, c_ in evs:
        a.record(stream)
        mg.mg_spmv(ctx, L, 1.0, xin, 0.0, xout)
        c_.record(stream)
    torch.cuda.synchronize()
    spmv_ms = sum(a.elapsed_time(c_) for a, c_ in evs) / ns
    nL, zL = infos[L]["n"], infos[L]["nnzb"]
    spmv_b = zL * (8 * bs * bs + 4) + 8 * (nL + 1) + 16 * bs * nL
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(args.config, {}).get("sweep_fine_dram_bytes")

    # ---------------- the other GMRES orthogonalisation on the same workload ----
    # MGS (the paper's) vs delayed CGS2 (reading Z29): same solver, same
    # graphs for the V-cycles, only the Arnoldi orthogonalisation differs
    orth_side = None
    if not args.no_orth_side:
        other = "dcgs2" if args.orth == "mgs" else "mgs"
        o_opts = dict(opts, method=orth_method[other])

        def ostep(xv, bv):
            xv.zero_()
            st, its, rel, conv = solver.solve(xv, bv, **o_opts)
            if not conv:
                raise RuntimeError(f"{other} solve did not converge: {its} its, rel {rel:.3e}")
            if H is not None:
                solver.apply_constraints(xv)
            return its, rel
        for _ in range(args.warmup):
            ostep(x, b)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        o_its = 0
        for _ in range(args.steps):
            its, rel = ostep(x, b)
            o_its += its
        e1.record(stream)
        torch.cuda.synchronize()
        o_ms = e0.elapsed_time(e1)
        if ws > 1:
            tt = torch.tensor([o_ms], dtype=torch.float64, device=red)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            o_ms = float(tt[0])
        orth_side = {"orth": other, "value": o_its / (o_ms / 1e3), "unit": "V-cycles/s",
                     "solve_ms": o_ms / args.steps, "iterations_per_solve": o_its / args.steps,
                     "true_rel_residual": rel,
                     "allreduces_per_arnoldi_step": "2" if other == "dcgs2" else "j + 2 (step j)",
                     "vector_passes_per_arnoldi_step": "2j + 6" if other == "dcgs2" else "4j + 7",
                     "note": "same solve with the other Arnoldi orthogonalisation: mgs = the paper's modified "
                             "Gram-Schmidt (P:346), dcgs2 = classical Gram-Schmidt with one delayed "
                             "reorthogonalisation (DESIGN.md Z29)"}

    # ---------------- mixed precision on the same workload ---------
    mixed = None
    if ws == 1 and args.precision == "fp64" and not args.no_mixed:
        solver.close()
        t = time.time()
        solver = mg.Multigrid(P.levels, bs, omega=P.omega, nu_pre=P.nu_pre, nu_post=P.nu_post, H=P.fine.H,
                              device=dev, stream=stream, use_graphs=not args.no_graphs, precision=mg.MG_PREC_MIXED)
        log(f"[bench] mixed-precision setup {time.time() - t:.1f}s")
        for _ in range(args.warmup):
            step(x, b)
        torch.cuda.synchronize()
        e0.record(stream)
        m_its = 0
        for _ in range(args.steps):
            its, rel = step(x, b)
            m_its += its
        e1.record(stream)
        torch.cuda.synchronize()
        m_ms = e0.elapsed_time(e1)
        mixed = {"value": m_its / (m_ms / 1e3), "unit": "V-cycles/s", "solve_ms": m_ms / args.steps,
                 "iterations_per_solve": m_its // args.steps, "true_rel_residual": rel,
                 "note": "V-cycle operators A_l stored fp32 (fp64 vectors, accumulation, D^-1, transfers, "
                         "coarse inverse), fp64 GMRES operator; converges to the fp64 1e-10 residual"}

    # ---------------- CPU baseline: the oracle on the host cores ----------------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        times, cores = oracle_vcycle_rate(P, n_cycles=1)
        cpu = {"value": 1.0 / times[0], "unit": "V-cycles/s", "cores": cores, "kind": "oracle",
               "sample": f"one oracle V(2,2) GMG(L,0,b) on the full {args.config} ({N} DOFs), "
                         f"{times[0]:.2f} s, OpenMP over rows"}
        # thread scan (1 thread, the paper's 8 threads, all cores); results are
        # bit-identical across thread counts
        scan = {}
        for th in sorted({1, min(8, cores), cores}):
            if th == cores:
                scan[str(th)] = cpu["value"]
                continue
            tt, _ = oracle_vcycle_rate(P, n_cycles=1, threads=th)
            scan[str(th)] = 1.0 / tt[0]
        cpu["threads_scan_vcycles_per_s"] = scan
        import oracle
        oracle.set_threads(cores)
        # time-to-1e-10 of the oracle's GMRES(30) + V(2,2) on the same system
        if not args.no_cpu_solve:
            h = _ORACLE_H[id(P)]
            t = time.perf_counter()
            _, o_its, _, o_rel = oracle.gmres(h, P.b, rtol=args.rtol)
            cpu["solve"] = {"seconds": time.perf_counter() - t, "iterations": o_its, "rel_residual": o_rel,
                            "dofs_per_s": P.n_dof / (time.perf_counter() - t)}

    if rank == 0:
        line = {
            "metric": "V-cycles/s", "value": value, "unit": "V-cycles/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            # config = the workload only, identical in the reference arm's line; run details below
            "config": {"workload": WORKLOADS[args.config], "n_dof": n_global, "levels": len(P.levels)},
            "run": {"n_dof_per_gpu": N, "level_rows_rank0": [i["n"] for i in infos],
                       "level_kinds": level_kinds,
                       "nnzb_fine_rank0": infos[L]["nnzb"],
                       "parallelism": (f"row-partition x{ws} ({'NCCL' if transport == mg.MG_TRANSPORT_NCCL else 'IPC'}"
                                       f" transport: halos, allreduce dots, agglomeration"
                                       + (f"; {ws} ranks share {torch.cuda.device_count()} GPU(s)"
                                          if torch.cuda.device_count() < ws else "") + ")")
                       if ws > 1 else "single GPU",
                       "solver": "GMRES(30) + V(2,2) block-Jacobi, rtol 1e-10, x0 = 0, then x <- Hx",
                       "precision": ("fp64" if vb == 8 else
                                     "mixed: V-cycle A_l stored fp32 (fp64 vectors/accumulation/D^-1/transfers), "
                                     "fp64 GMRES operator; true fp64 residual 1e-10"),
                       "l2": (f"finest operator {infos[L]['nnzb'] * (8 * bs * bs + 4) / 1e9:.2f} GB vs L2 126 MB: "
                              + ("no flush needed" if infos[L]["nnzb"] * (8 * bs * bs + 4) > 1e9
                                 else "partly L2-resident (small config)")),
                       "iterations_per_solve": total_its // args.steps},
            "dof_cycles_per_s": value * n_global,
            "solve_ms": t_ms / args.steps,
            "solve_dofs_per_s": n_global / (t_ms / args.steps / 1e3),
            "vcycle_levels": {"rows_rank0": [i["n"] for i in infos], "ms": prof["level_ms"],
                              "eager_total_ms": sum(prof["level_ms"]) + sum(prof["halo_ms"])
                              + prof["agglomeration_ms"],
                              "halo_ms": prof["halo_ms"], "agglomeration_ms": prof["agglomeration_ms"],
                              "note": "one eager V(2,2) from zero, CUDA events between phases"},
            "paper_context": PAPER_CONTEXT.get(args.config),
            "orth": args.orth,
            "orth_other": orth_side,
            "mixed_precision": mixed,
            "update_matrix": upd,
            "vcycle_only": {"ms": vc_ms, "per_s": 1e3 / vc_ms, "batch_ms": batches,
                            "protocol": "5 warm-up, 5 batches x 50 graph-launched V(2,2) from zero, median",
                            "alg_bytes": vc_bytes,
                            "alg_gbs": vc_bytes / (vc_ms / 1e3) / 1e9,
                            "frac": vc_bytes / (vc_ms / 1e3) / 1e9 / peak},
            "roofline": {"bound": "hbm", "kernel": f"k_sell_apply<{bs},SWEEP> (fused block-Jacobi sweep), finest level",
                         "achieved": achieved,
                         "peak": peak, "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "alg_bytes_per_launch": sweep_b, "avg_launch_ms": sw_ms},
            "spmv_hbm": {"kernel": f"k_sell_apply<{bs},SPMV> finest level (fp64)", "avg_launch_ms": spmv_ms,
                         "alg_bytes_per_launch": spmv_b, "gbs": spmv_b / (spmv_ms / 1e3) / 1e9,
                         "frac": spmv_b / (spmv_ms / 1e3) / 1e9 / peak},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "V-cycles/s", "h2d_bytes_per_step": 8 * n_global,
                    "d2h_bytes_per_step": 8 * n_global},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    solver.close()
    if ws > 1:
        torch.distributed.destroy_process_group()


def run_newton(args):
    """C4 as SURVEY §8(d) states it (BASELINE config 4): flow around a cylinder,
    backward Euler, Newton + GMRES(30)/V(2,2) per time step with every level's
    Jacobian assembled on the CPU and re-uploaded value-only.  Step =
    one time step through mg_newton (the public API): `value` = V-cycles/s of
    the GPU linear solves (device time: CUDA events inside mg_newton), `e2e` =
    the same V-cycles over the whole time step's wall time including the CPU
    assembly and the host<->device copies."""
    import torch
    ws, rank, local = dist_env()
    if ws > 1 and rank != 0:
        return          # single-GPU workload: replicas only
    torch.cuda.set_device(local)
    import paper_2405_05047_b200 as mg
    from problems import channel as C
    t = time.time()
    P = C.build("c4ns")
    log(f"[bench] generated c4ns: {P.n_dof} DOFs, levels {[L.data.n for L in P.levels]} in {time.time() - t:.1f}s")
    stream = torch.cuda.current_stream()
    u = C.initial_state(P)
    omega = args.omega if args.omega else (1.0 if args.vanka else P.omega)
    solver = mg.Multigrid(C.with_values(P, C.jacobians(P, u, u)), 3, omega=omega, H=P.fine.H, device=local,
                          stream=stream, vanka=args.vanka)
    ctx = solver.ctx
    L = len(P.levels) - 1
    infos = [mg.level_info(ctx, l) for l in range(L + 1)]
    x = torch.from_numpy(u.reshape(-1).copy()).cuda()

    def time_step():
        u_old = x.cpu().numpy().reshape(-1, 3)
        t0 = time.perf_counter()
        st, info = solver.newton(x, C.assemble_callback(P, u_old), max_newton=4, ntol=1e-8)
        if not info["converged"]:
            raise RuntimeError(f"Newton did not converge: {info}")
        return time.perf_counter() - t0, info

    for _ in range(args.warmup):
        time_step()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    l0 = mg.launch_count(ctx)
    wall, its, newton, upl, sol, asm, lin = 0.0, 0, 0, 0.0, 0.0, 0.0, []
    for _ in range(args.steps):
        w_s, info = time_step()
        wall += w_s
        its += info["gmres_its"]
        newton += info["newton_its"]
        upl += info["ms_upload"]
        sol += info["ms_solve"]
        asm += info["ms_assemble"]
        lin.append(info["lin_its"])
    launches = mg.launch_count(ctx) - l0
    clocks = sampler.stop()
    value = its / (sol / 1e3)
    # dominant kernel: fine-level fused sweep of the current Jacobian
    peak, peak_src = measured_peaks()
    N = P.n_dof
    xin = torch.randn(N, dtype=torch.float64, device="cuda")
    bb = torch.randn(N, dtype=torch.float64, device="cuda")
    xout = torch.empty_like(xin)
    for _ in range(3):
        mg.mg_sweep(ctx, L, xin, bb, xout)
    ns = 20
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ns)]
    torch.cuda.synchronize()
    for a, c_ in evs:
        a.record(stream)
        mg.mg_sweep(ctx, L, xin, bb, xout)
        c_.record(stream)
    torch.cuda.synchronize()
    sw_ms = sum(a.elapsed_time(c_) for a, c_ in evs) / ns
    sweep_b, _, _ = level_bytes(infos[L], 3, False)
    cpu = None
    if not args.no_cpu_baseline:
        import oracle
        cores = cpu_cores()
        oracle.set_threads(cores)
        h = oracle.MgHierarchy.from_arrays(C.with_values(P, C.jacobians(P, u, u)), omega=P.omega)
        bh = np.random.default_rng(0).standard_normal(N)
        t = time.perf_counter()
        oracle.vcycle(h, L, np.zeros(N), bh)
        dt_o = time.perf_counter() - t
        cpu = {"value": 1.0 / dt_o, "unit": "V-cycles/s", "cores": cores, "kind": "oracle",
               "sample": f"one oracle V(2,2) GMG(L,0,b) on the c4ns Jacobian hierarchy ({N} DOFs), {dt_o:.2f} s"}
    line = {
        "metric": "V-cycles/s", "value": value, "unit": "V-cycles/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS["c4ns"], "n_dof": N, "levels": L + 1,
                   "level_rows": [i["n"] for i in infos], "nnzb_fine": infos[L]["nnzb"],
                   "parallelism": "single GPU", "l2": "finest Jacobian 0.29 GB > L2 126 MB",
                   "smoother": ("Vanka (cell patches, mg_set_vanka)" if args.vanka else "block-Jacobi")
                   + f", omega {omega}",
                   "newton_per_step": newton / args.steps, "gmres_per_step": its / args.steps,
                   "lin_its": lin},
        "dof_cycles_per_s": value * N,
        "time_step": {"wall_ms": 1e3 * wall / args.steps, "cpu_assembly_ms": asm / args.steps,
                      "upload_device_ms": upl / args.steps, "solve_device_ms": sol / args.steps,
                      "note": "CPU assembly of F and of 9 levels' Jacobians (numpy + C helper, the paper's CPU side)"},
        "roofline": {"bound": "hbm", "kernel": "k_sell_apply<3,SWEEP> (fused block-Jacobi sweep), finest level",
                     "achieved": sweep_b / (sw_ms / 1e3) / 1e9, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": sweep_b / (sw_ms / 1e3) / 1e9 / peak, "traffic": None, "alg_bytes_per_launch": sweep_b,
                     "avg_launch_ms": sw_ms},
        "cpu_baseline": cpu,
        "e2e": {"value": its / wall, "unit": "V-cycles/s",
                "h2d_bytes_per_step": int(newton / args.steps * (8 * N + sum(8 * 9 * i["nnzb"] for i in infos))),
                "d2h_bytes_per_step": int((newton / args.steps + 1) * 8 * N)},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    solver.close()


def run_ns(args):
    """The paper's explicit pressure-correction NS step (Alg. 2; SURVEY
    N2) on its 3D cavity (32x32x64 graded pressure mesh = 70,785 nodes,
    velocity on the midpoint refinement = 545,025 nodes), from rest.  Step = one
    ns_step (momentum kernel, divergence, pressure GMRES+MG with int q = 0,
    pressure update).  value = time steps/s; the line carries the Table `ns`
    split per step for context (the paper: H100 PCIe, its GPU column
    sums to 1660 s over "40 000" steps = 41.5 ms per step; reading Z19)."""
    import torch
    ws, rank, local = dist_env()
    if ws > 1 and rank != 0:
        return
    torch.cuda.set_device(local)
    import paper_2405_05047_b200 as mg
    from problems import ns as NSP
    t = time.time()
    P = NSP.build_ns("ns")
    log(f"[bench] generated ns: n_u {P.n_u}, n_p {P.n_p}, pressure levels {[L.n for L in P.pres_levels]} "
        f"in {time.time() - t:.1f}s")
    g = mg.NavierStokes(P, rtol=1e-6, timing=True, vanka=args.vanka, omega=args.omega or None)
    u, p, q = NSP.initial_state(P)
    g.set_state(u, p, q)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        g.step()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    l0 = mg.ns_launch_count(g.ctx)   # includes the pressure solve (thread-local tally)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    comp = np.zeros(4)
    its = 0
    for _ in range(args.steps):
        st, it, rel, conv, ms = g.step()
        comp += np.array(ms)
        its += it
    e1.record(stream)
    torch.cuda.synchronize()
    t_ms = e0.elapsed_time(e1)
    launches = mg.ns_launch_count(g.ctx) - l0
    clocks = sampler.stop()
    # e2e: the state from/to pinned host buffers around every step
    uh, ph, qh = (np.ascontiguousarray(a) for a in g.get_state())
    t0 = time.perf_counter()
    for _ in range(args.steps):
        g.set_state(uh, ph, qh)
        g.step()
        uh, ph, qh = (np.ascontiguousarray(a) for a in g.get_state())
    e2e_s = time.perf_counter() - t0
    value = args.steps / (t_ms / 1e3)
    # the same steps with the Vanka-type cell-patch smoother in the pressure MG
    vk = None
    if not args.vanka:
        gv = mg.NavierStokes(P, rtol=1e-6, timing=True, vanka=True, omega=0.8)
        gv.set_state(u, p, q)
        for _ in range(args.warmup):
            gv.step()
        torch.cuda.synchronize()
        e0.record(stream)
        vcomp, vits = np.zeros(4), 0
        for _ in range(args.steps):
            st, it, rel, conv, ms = gv.step()
            vcomp += np.array(ms)
            vits += it
        e1.record(stream)
        torch.cuda.synchronize()
        v_ms = e0.elapsed_time(e1)
        vk = {"value": args.steps / (v_ms / 1e3), "unit": "time steps/s", "ms_per_step": v_ms / args.steps,
              "pressure_gmres_per_step": vits / args.steps,
              "split_ms_per_step": dict(zip(("momentum", "pres-rhs", "pres-solve", "pres-up"),
                                            (vcomp / args.steps).tolist())),
              "note": "pressure MG smoothed by mg_set_vanka on the mesh cells, omega 0.8 (point Jacobi needs "
                      "omega 0.4 on the graded mesh, reading Z27)"}
        gv.close()
    cpu = None
    if not args.no_cpu_baseline:
        import oracle
        from oracle import ns as ons
        cores = cpu_cores()
        oracle.set_threads(cores)
        ops = ons.NsOperators.from_arrays(P.n_u, P.n_p, P.mom_rp, P.mom_col, P.mom_val, P.G, P.m_u, P.m_p,
                                          P.dir_rows, P.dir_vals, P.nu, P.dt)
        h = oracle.MgHierarchy.from_arrays(P.pres_levels, omega=P.omega,
                                           mean=[(L.mean_w, L.mean_k) for L in P.pres_levels])
        t = time.perf_counter()
        ons.step(ops, h, uh, ph, qh, rtol=1e-6)
        dt_o = time.perf_counter() - t
        cpu = {"value": 1.0 / dt_o, "unit": "time steps/s", "cores": cores, "kind": "oracle",
               "sample": f"one oracle Alg. 2 step on the paper's cavity, {dt_o:.2f} s"}
    n = args.steps
    line = {
        "metric": "NS time steps/s", "value": value, "unit": "time steps/s", "n_gpus": 1, "steps": n,
        "warmup": args.warmup, "ms_per_step": t_ms / n, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS["ns"], "n_u": P.n_u, "n_p": P.n_p,
                   "pressure_levels": [L.n for L in P.pres_levels], "pressure_gmres_per_step": its / n,
                   "pressure_rtol": 1e-6, "parallelism": "single GPU",
                   "pressure_smoother": ("Vanka (cell patches)" if args.vanka else "point Jacobi")
                   + f", omega {args.omega or P.omega}",
                   "l2": "per-step operators ~0.6 GB > L2 126 MB"},
        "table_ns_split_ms_per_step": {"momentum": comp[0] / n, "pres-rhs": comp[1] / n, "pres-solve": comp[2] / n,
                                       "pres-up": comp[3] / n},
        "vanka_pressure": vk,
        "paper_context": {"gpu_ms_per_step_h100": 41.5, "split_ms_per_step_h100": {
            "momentum": 5.78, "pres-rhs": 1.33, "pres-solve": 32.6, "pres-up": 1.81},
            "note": "Table ns GPU column / 40 000 steps (P:757-790); other hardware and code: context only"},
        "cpu_baseline": cpu,
        "e2e": {"value": n / e2e_s, "unit": "time steps/s", "h2d_bytes_per_step": 8 * (3 * P.n_u + 2 * P.n_p),
                "d2h_bytes_per_step": 8 * (3 * P.n_u + 2 * P.n_p)},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    g.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(WORKLOADS), default="c3")
    ap.add_argument("--rtol", type=float, default=1e-10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu-solve", action="store_true", help="skip the oracle's full GMRES solve in cpu_baseline")
    ap.add_argument("--no-graphs", action="store_true")
    ap.add_argument("--no-mixed", action="store_true", help="skip the mixed-precision side measurement")
    ap.add_argument("--orth", choices=["mgs", "dcgs2"], default="mgs",
                    help="GMRES orthogonalisation of the timed solve: mgs (the paper's, P:346) or dcgs2 (Z29)")
    ap.add_argument("--no-orth-side", action="store_true", help="skip timing the other orthogonalisation")
    ap.add_argument("--precision", choices=["fp64", "mixed"], default="fp64",
                    help="mixed: fp32-stored V-cycle operators inside fp64 GMRES (SURVEY N1)")
    ap.add_argument("--vanka", action="store_true", help="c4ns / ns: Vanka-type cell-patch smoother (P:822)")
    ap.add_argument("--omega", type=float, default=0.0, help="c4ns / ns: smoother damping (0: config default)")
    ap.add_argument("--min-rows-per-rank", type=int, default=16384,
                    help="multi-GPU: levels with fewer rows per rank are replicated (agglomerated)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("[bench] warmup raised to 3 (timing rules)")
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "c4ns":
        run_newton(args)
    elif args.config == "ns":
        run_ns(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
