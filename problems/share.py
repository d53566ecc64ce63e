"""Share one generated problem between the ranks of a job on one node
(SEEDED INPUT PREPARATION; no solve arithmetic).

Generating a 10M-DOF hierarchy takes ~30 s and ~10 GB of host memory; with N
ranks each generating it the scaling run would cost N times both.  Rank 0
generates once and writes every numpy array of the problem as its own .npy
file (the object skeleton is pickled with the arrays replaced by file ids);
the other ranks load the arrays memory-mapped, so each rank pages in only the
rows its partition touches and the page cache is shared.
"""
from __future__ import annotations

import os
import pickle
import shutil

import numpy as np

_MARK = "__mgb200_npy__"


def _strip(obj, out, memo):
    if isinstance(obj, np.ndarray):
        key = id(obj)
        if key not in memo:
            memo[key] = len(out)
            out.append(obj)
        return (_MARK, memo[key])
    if isinstance(obj, tuple):
        return tuple(_strip(v, out, memo) for v in obj)
    if isinstance(obj, list):
        return [_strip(v, out, memo) for v in obj]
    if isinstance(obj, dict):
        return {k: _strip(v, out, memo) for k, v in obj.items()}
    if hasattr(obj, "__dict__") and not isinstance(obj, type):
        clone = object.__new__(type(obj))
        clone.__dict__.update({k: _strip(v, out, memo) for k, v in obj.__dict__.items()})
        return clone
    return obj


def _fill(obj, arrays):
    if isinstance(obj, tuple) and len(obj) == 2 and obj[0] == _MARK:
        return arrays[obj[1]]
    if isinstance(obj, tuple):
        return tuple(_fill(v, arrays) for v in obj)
    if isinstance(obj, list):
        return [_fill(v, arrays) for v in obj]
    if isinstance(obj, dict):
        return {k: _fill(v, arrays) for k, v in obj.items()}
    if hasattr(obj, "__dict__") and not isinstance(obj, type):
        obj.__dict__.update({k: _fill(v, arrays) for k, v in obj.__dict__.items()})
        return obj
    return obj


def dump(problem, directory: str) -> None:
    os.makedirs(directory, exist_ok=True)
    arrays: list = []
    skel = _strip(problem, arrays, {})
    for i, a in enumerate(arrays):
        np.save(os.path.join(directory, f"{i}.npy"), np.ascontiguousarray(a), allow_pickle=False)
    with open(os.path.join(directory, "skeleton.pkl.tmp"), "wb") as f:
        pickle.dump((len(arrays), skel), f)
    os.replace(os.path.join(directory, "skeleton.pkl.tmp"), os.path.join(directory, "skeleton.pkl"))


def load(directory: str, mmap: bool = True):
    with open(os.path.join(directory, "skeleton.pkl"), "rb") as f:
        n, skel = pickle.load(f)
    arrays = [np.load(os.path.join(directory, f"{i}.npy"), mmap_mode="r" if mmap else None) for i in range(n)]
    return _fill(skel, arrays)


def remove(directory: str) -> None:
    shutil.rmtree(directory, ignore_errors=True)


def _nbytes(obj) -> int:
    arrays: list = []
    _strip(obj, arrays, {})
    return sum(a.nbytes for a in arrays)


def shared_build(build, tag: str, rank: int, barrier, broadcast_token, base: str | None = None):
    """build(): the generator call (rank 0 only).  barrier(): a collective barrier;
    broadcast_token(tok or None) -> tok: a collective broadcast of a small string
    from rank 0.  Rank 0 writes to the first of (base, /dev/shm, the temp dir) with
    room for the arrays; if none has room every rank builds its own copy.
    Returns (problem, cleanup) -- call cleanup() collectively once every rank has
    taken what it needs."""
    import tempfile
    directory = None
    if rank == 0:
        P = build()
        need = _nbytes(P) + (64 << 20)
        for cand in (base, "/dev/shm", tempfile.gettempdir()):
            if not cand or not os.path.isdir(cand) or not os.access(cand, os.W_OK):
                continue
            if shutil.disk_usage(cand).free < need:
                continue
            directory = os.path.join(cand, f"mgb200_{tag}_{os.getpid()}_{os.urandom(4).hex()}")
            try:
                dump(P, directory)
                break
            except OSError:
                remove(directory)
                directory = None
    directory = broadcast_token(directory if rank == 0 else None)
    if rank != 0:
        P = load(directory) if directory else build()

    def cleanup():
        barrier()
        if rank == 0 and directory:
            remove(directory)
    return P, cleanup
