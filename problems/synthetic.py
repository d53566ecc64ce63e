"""Seeded random block-sparse hierarchies (SEEDED INPUT GENERATOR; no solve
arithmetic).  Used to cover block sizes and transfer weight layouts the FE
configs do not exercise (bs = 2, 4; weights_per_entry = bs) in per-op and
V-cycle parity tests.  Matrices are block diagonally dominant (so D^-1 exists
and smoothing is stable); transfers have 0-4 entries per row with ragged and
empty rows."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEED_BASE = 240505047


@dataclass
class SynLevel:
    n: int
    bs: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    P: tuple | None = None
    wpe: int = 1

    @property
    def nnzb(self) -> int:
        return int(self.row_ptr[-1])


def random_bsr(n, bs, rng, avg_nnz=7, band=40):
    rows, cols = [], []
    for i in range(n):
        k = int(rng.integers(0, 2 * avg_nnz))
        nb = rng.integers(max(0, i - band), min(n, i + band + 1), size=k)
        c = np.unique(np.concatenate([[i], nb]))
        rows.append(np.full(len(c), i))
        cols.append(c)
    r = np.concatenate(rows)
    c = np.concatenate(cols).astype(np.int64)
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    rp = np.cumsum(rp)
    val = rng.standard_normal((len(c), bs, bs))
    absrow = np.zeros(n)
    np.add.at(absrow, r, np.abs(val).sum(axis=(1, 2)))
    diag = np.nonzero(r == c)[0]
    val[diag] += (absrow[r[diag]] + 1.0)[:, None, None] * np.eye(bs)[None]
    return rp, c, val


def random_transfer(nf, nc, wpe, rng):
    rows, cols = [], []
    for i in range(nf):
        k = int(rng.integers(0, 5))                     # 0..4 entries, empty rows included
        c = np.unique(rng.integers(0, nc, size=k))
        rows.append(np.full(len(c), i))
        cols.append(c)
    r = np.concatenate(rows)
    c = np.concatenate(cols).astype(np.int64)
    rp = np.zeros(nf + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    rp = np.cumsum(rp)
    w = rng.uniform(0.0, 0.5, size=len(c) * wpe)
    return rp, c, w


def random_hierarchy(bs, sizes=(21, 77, 301), wpe=None, seed_index=10):
    rng = np.random.Generator(np.random.PCG64(SEED_BASE + seed_index))
    wpe = bs if wpe is None else wpe
    levels = []
    for l, n in enumerate(sizes):
        rp, c, v = random_bsr(n, bs, rng)
        lv = SynLevel(n, bs, rp, c, v)
        if l > 0:
            lv.P = random_transfer(n, sizes[l - 1], wpe, rng)
            lv.wpe = wpe
        levels.append(lv)
    b = rng.standard_normal(sizes[-1] * bs)
    return levels, b
