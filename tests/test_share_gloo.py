"""problems/share.py: rank 0 generates, the other ranks load the arrays
memory-mapped (world size 2, gloo, CPU) -- the partition each rank builds
from the shared problem is identical to one built from its own generation."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from problems import configs
        from problems.partition import partition
        from problems.share import shared_build

        def bcast(tok):
            box = [tok]
            dist.broadcast_object_list(box, src=0)
            return box[0]
        P, cleanup = shared_build(lambda: configs.build("c3_small", keep_geometry=False), "t", rank, dist.barrier,
                                  bcast)
        parts, extras, ranges = partition(P, ws, min_rows_per_rank=16, only_rank=rank)
        cleanup()
        ref = configs.build("c3_small", keep_geometry=False)
        rparts, rextras, rranges = partition(ref, ws, min_rows_per_rank=16, only_rank=rank)
        ok = ranges == rranges and np.array_equal(extras[rank][0], rextras[rank][0])
        for a, b in zip(parts[rank], rparts[rank]):
            ok &= a.n == b.n and np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col, b.col)
            ok &= np.array_equal(a.val, b.val) and (a.P is None or all(np.array_equal(x, y) for x, y in zip(a.P, b.P)))
        out[rank] = bool(ok)
    finally:
        dist.destroy_process_group()


def test_shared_problem_two_ranks():
    ws = 2
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_worker, args=(ws, _port(), out), nprocs=ws, join=True)
        assert out.get(0) and out.get(1), dict(out)


def test_shared_build_roundtrip_and_fallback(tmp_path, monkeypatch):
    """Single process: dump/load round trip of a problem (arrays memory-mapped,
    identical), and the no-room fallback (every rank builds its own copy)."""
    from problems import configs
    from problems import share
    P = configs.build("c2_small", keep_geometry=False)
    share.dump(P, str(tmp_path / "p"))
    Q = share.load(str(tmp_path / "p"))
    assert Q.n_dof == P.n_dof and Q.omega == P.omega and np.array_equal(Q.b, P.b)
    for a, b in zip(P.levels, Q.levels):
        assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.val, b.val)
        assert isinstance(b.val, np.memmap)
    built = []
    monkeypatch.setattr(share.shutil, "disk_usage", lambda p: type("U", (), {"free": 0})())
    P2, cleanup = share.shared_build(lambda: built.append(1) or P, "t", 0, lambda: None, lambda tok: tok)
    cleanup()
    assert P2 is P and built == [1]
    P3, cleanup = share.shared_build(lambda: built.append(2) or P, "t", 1, lambda: None, lambda tok: None)
    cleanup()
    assert P3 is P and built == [1, 2]        # rank 1 saw no directory: built its own
