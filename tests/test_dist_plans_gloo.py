"""World-size-2 CPU test (torch.distributed, gloo) of the multi-GPU host logic
(SURVEY §8(e)): each rank takes its rows from problems.partition, builds its
ghost list with the library's mgi_localize_columns / mgi_owner, exchanges halo
requests and P entries over gloo exactly as the library's transports do, and
assembles its restriction rows with mgi_assemble_routed_rows.  Checked:
send/recv lists are mutually consistent, a distributed SpMV (oracle per rank
on ghost-extended x) equals the global oracle SpMV bit-for-bit, and the routed
R rows equal the rows of the global stable transpose."""
import ctypes
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import paper_2405_05047_b200 as m
        from problems import configs
        from problems.partition import partition
        L = m.lib()
        L.mgi_localize_columns.argtypes = [ctypes.c_int64] * 3 + [ctypes.c_void_p] * 5
        L.mgi_owner.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int]
        L.mgi_assemble_routed_rows.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_int64,
                                                                                           ctypes.c_int64] + \
            [ctypes.c_void_p] * 3
        Pr = configs.build("c3_small")
        parts, extras, ranges = partition(Pr, world, min_rows_per_rank=32)
        bs = Pr.bs
        Lf = len(Pr.levels) - 1
        me = parts[rank][Lf]
        F = Pr.levels[Lf]
        bounds = np.array([r[0] for r in ranges[Lf]] + [F.n], np.int64)
        # ---- ghosts of A's columns and their owners (library routines) ----
        nnz = len(me.col)
        loc = np.zeros(nnz, np.int64)
        gh = np.zeros(nnz, np.int64)
        ng = ctypes.c_int64()
        assert L.mgi_localize_columns(me.n, me.row_begin, me.row_end, _p(me.row_ptr), _p(me.col), _p(loc), _p(gh),
                                      ctypes.byref(ng)) == 0
        ghosts = gh[:ng.value].copy()
        owners = np.array([L.mgi_owner(int(g), _p(bounds), world) for g in ghosts])
        assert np.all((owners >= 0) & (owners < world) & (owners != rank))
        req = [ghosts[owners == r].tolist() for r in range(world)]
        got = [None] * world
        dist.all_gather_object(got, req)
        send = {r: got[r][rank] for r in range(world) if r != rank}   # rows others need from me
        for r, rows in send.items():
            assert all(me.row_begin <= g < me.row_end for g in rows)
        # ---- distributed SpMV: oracle on [own | ghosts] vs global oracle ----
        x = np.random.default_rng(3).standard_normal(F.n * bs)        # same global x on every rank
        xown = x.reshape(-1, bs)[me.row_begin:me.row_end]
        # ghost values travel over gloo (each rank only sends its own rows)
        vals = [None] * world
        dist.all_gather_object(vals, {r: xown[np.array(rows, np.int64) - me.row_begin] for r, rows in send.items()
                                      if len(rows)})
        gvals = np.zeros((len(ghosts), bs))
        for r in range(world):
            if r != rank and rank in vals[r]:
                gvals[owners == r] = vals[r][rank]
        xext = np.concatenate([xown, gvals]).reshape(-1)
        y_loc = oracle.spmv(me.n, bs, me.row_ptr, loc, me.val, xext)
        y_glob = oracle.spmv(F.n, bs, F.row_ptr, F.col, F.val, x).reshape(-1, bs)[me.row_begin:me.row_end]
        assert np.array_equal(y_loc.reshape(-1, bs), y_glob)
        # ---- restriction rows routed to the coarse owners ----
        C = Pr.levels[Lf - 1]
        cb = np.array([r[0] for r in ranges[Lf - 1]] + [C.n], np.int64)
        prp, pcol, pw = me.P
        rows = np.repeat(np.arange(me.n), np.diff(prp)) + me.row_begin
        dest = np.array([L.mgi_owner(int(j), _p(cb), world) for j in pcol])
        out = [(pcol[dest == r], rows[dest == r], pw[dest == r]) for r in range(world)]
        allout = [None] * world
        dist.all_gather_object(allout, out)
        J = np.concatenate([allout[r][rank][0] for r in range(world)]).astype(np.int64)
        I = np.concatenate([allout[r][rank][1] for r in range(world)]).astype(np.int64)
        W = np.concatenate([allout[r][rank][2] for r in range(world)]).astype(np.float64)
        r0, nr = int(cb[rank]), int(cb[rank + 1] - cb[rank])
        orp = np.zeros(nr + 1, np.int64)
        ocol = np.zeros(max(1, len(J)), np.int64)
        ow = np.zeros(max(1, len(J)))
        assert L.mgi_assemble_routed_rows(len(J), _p(J), _p(I), _p(W), 1, r0, nr, _p(orp), _p(ocol), _p(ow)) == 0
        grp, gcol, gw = oracle.csr_transpose(F.n, C.n, *F.P)
        a, b = grp[r0], grp[r0 + nr]
        assert np.array_equal(orp, grp[r0:r0 + nr + 1] - a)
        assert np.array_equal(ocol[:len(J)], gcol[a:b]) and np.array_equal(ow[:len(J)], gw[a:b])
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except BaseException as e:  # noqa: BLE001
        import traceback
        q.put((rank, f"{type(e).__name__}: {e}\n{traceback.format_exc()}"))


def test_multirank_plans_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000)
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
