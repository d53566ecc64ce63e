"""Row partition of a generated hierarchy over ranks (SEEDED INPUT PREPARATION;
no solve arithmetic) -- SURVEY §8(e):

* the finest level is cut into contiguous ranges of its Morton order,
  balanced on block nonzeros (adaptive meshes have non-uniform rows);
* the SAME splitters apply on every level: a node belongs to the rank whose
  Morton-key range contains it (keys are lattice coordinates at the finest
  level, so a coarse node goes with the coincident fine node);
* levels with fewer than `min_rows_per_rank` rows per rank (and level 0 when
  the coarse solve is direct) are REPLICATED: every rank holds all rows and the
  library agglomerates the restricted residual onto them.

Each rank gets its owned rows of A_l (global columns), of P_{l-1} (fine rows
of level l, global coarse columns), of H and of b.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class RankLevel:
    n: int                # owned rows
    n_global: int
    row_begin: int
    row_end: int
    bs: int
    row_ptr: np.ndarray
    col: np.ndarray       # global block columns
    val: np.ndarray
    P: tuple | None = None
    wpe: int = 1
    mean_w: np.ndarray | None = None   # owned rows of the level's constraint weights (pure Neumann)
    mean_k: np.ndarray | None = None

    @property
    def replicated(self) -> bool:
        return self.row_begin == 0 and self.row_end == self.n_global


def _rows(rp, col, val, r0, r1, vpe_shape):
    a, b = int(rp[r0]), int(rp[r1])
    return (np.ascontiguousarray(rp[r0:r1 + 1] - rp[r0]), np.ascontiguousarray(col[a:b]),
            np.ascontiguousarray(val[a:b]) if val is not None else None)


def splitters(problem, nranks, min_rows_per_rank=64, replicate_level0=True):
    """Per level: list of (row_begin, row_end) per rank."""
    levels = problem.levels
    fine = levels[-1]
    rp = fine.row_ptr
    target = rp[-1] * np.arange(1, nranks) / nranks
    cut = np.searchsorted(rp, target)                  # nnzb-balanced row cuts of the finest level
    kcut = fine.keys[np.minimum(cut, fine.n - 1)]
    out = []
    replicate = False
    for l in range(len(levels) - 1, -1, -1):
        L = levels[l]
        if L.n < min_rows_per_rank * nranks or (l == 0 and replicate_level0):
            replicate = True
        if replicate:
            out.append([(0, L.n)] * nranks)
            continue
        b = np.concatenate([[0], np.searchsorted(L.keys, kcut), [L.n]]).astype(np.int64)
        b = np.maximum.accumulate(b)
        out.append([(int(b[r]), int(b[r + 1])) for r in range(nranks)])
    return out[::-1]


def partition(problem, nranks, min_rows_per_rank=64, replicate_level0=True, only_rank=None, ranges=None):
    """Returns (per-rank list of RankLevel lists, per-rank (b_local, H_local), ranges).
    only_rank: build the data of that rank only (the other entries are None).
    ranges: explicit per-level row ranges (overrides the splitters; edge-case tests)."""
    if ranges is None:
        ranges = splitters(problem, nranks, min_rows_per_rank, replicate_level0)
    bs = problem.bs
    ranks = []
    extras = []
    for r in range(nranks):
        if only_rank is not None and r != only_rank:
            ranks.append(None)
            extras.append(None)
            continue
        lv = []
        for l, L in enumerate(problem.levels):
            r0, r1 = ranges[l][r]
            rp, col, val = _rows(L.row_ptr, L.col, L.val, r0, r1, None)
            RL = RankLevel(r1 - r0, L.n, r0, r1, bs, rp, col, val)
            if l > 0:
                prp, pcol, pw = L.P
                wpe = getattr(L, "wpe", 1)
                a, b = int(prp[r0]), int(prp[r1])
                RL.P = (np.ascontiguousarray(prp[r0:r1 + 1] - prp[r0]), np.ascontiguousarray(pcol[a:b]),
                        np.ascontiguousarray(pw[a * wpe:b * wpe]))
                RL.wpe = wpe
            if getattr(L, "mean_w", None) is not None:
                RL.mean_w = np.ascontiguousarray(L.mean_w.reshape(-1, bs)[r0:r1].reshape(-1))
                RL.mean_k = np.ascontiguousarray(L.mean_k.reshape(-1, bs)[r0:r1].reshape(-1))
            lv.append(RL)
        f0, f1 = ranges[-1][r]
        b_loc = np.ascontiguousarray(problem.b.reshape(-1, bs)[f0:f1].reshape(-1))
        H = problem.fine.H
        hrp, hcol, hw = _rows(H[0], H[1], H[2], f0, f1, None)
        ranks.append(lv)
        extras.append((b_loc, (hrp, hcol, hw)))
    return ranks, extras, ranges
