"""The per-rank C5 generator (problems/structured.py) against the generic
octree generator (problems/configs.py) and against itself across partitions.

* Same system: on c5_small (root (2,2,4), two uniform steps) every level's
  matrix, every prolongation and the constrained right-hand side equal the
  generic generator's after renumbering Morton -> lexicographic (values to
  rounding of the summation order, structure and transfer weights exactly).
* Partition independence: the rows that ranks 0..P-1 generate for P = 2, 3
  are, concatenated, BIT-IDENTICAL to the single-rank rows (matrices,
  transfers, right-hand side), and every coarse node of a distributed level is
  owned by the owner of its coincident fine node."""
import numpy as np
import pytest

from problems import configs as C
from problems import structured as S


def _perm(level_nodes, g, R, l):
    """generic node index -> lexicographic id on level l."""
    c = level_nodes.coords >> (R - l)
    return c[:, 0] + (g[0] + 1) * (c[:, 1] + (g[1] + 1) * c[:, 2])


def _dense_blocks(rp, col, val, perm=None):
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    if perm is not None:
        rows, col = perm[rows], perm[col]
    return {(int(r), int(c)): v for r, c, v in zip(rows, col, val)}


def test_structured_equals_generic_c5_small():
    gen = C.build("c5_small")
    root, R = (2, 2, 4), 2
    bs = 4
    # raw rhs of the generic generator (same seed and draw order), renumbered
    rng = np.random.Generator(np.random.PCG64(C.SEED_BASE + S.SEED_INDEX))
    fine = gen.levels[-1]
    raw = rng.standard_normal((fine.n, bs))
    gF = S.grid(root, R)
    pf = _perm(fine.nodes, gF, R, R)
    raw_s = np.empty_like(raw)
    raw_s[pf] = raw
    levels, b, ranges = S.build_rank(1, 0, root=root, R=R, raw_b=raw_s)
    assert [L.n for L in levels] == [L.n for L in gen.levels]
    for l, (Ls, Lg) in enumerate(zip(levels, gen.levels)):
        g = S.grid(root, l)
        pm = _perm(Lg.nodes, g, R, l)
        assert np.array_equal(np.sort(pm), np.arange(Lg.n))
        A_g = _dense_blocks(Lg.row_ptr, Lg.col, Lg.val, pm)
        A_s = _dense_blocks(Ls.row_ptr, Ls.col, Ls.val)
        assert A_g.keys() == A_s.keys()
        scale = max(np.max(np.abs(Lg.val)), 1.0)
        err = max(np.max(np.abs(A_g[k] - A_s[k])) for k in A_g)
        assert err <= 1e-14 * scale, (l, err)
        # columns ascending in every row (library requirement)
        for i in range(0, Ls.n, 97):
            c = Ls.col[Ls.row_ptr[i]:Ls.row_ptr[i + 1]]
            assert np.all(np.diff(c) > 0)
        if l > 0:
            pc = _perm(gen.levels[l - 1].nodes, S.grid(root, l - 1), R, l - 1)
            rp, col, w = Lg.P
            Pg = _dense_blocks(rp, col, w.reshape(-1, bs), None)
            Pg = {(int(pm[r]), int(pc[c])): v for (r, c), v in Pg.items()}
            rp, col, w = Ls.P
            Ps = _dense_blocks(rp, col, w.reshape(-1, bs))
            assert Pg.keys() == Ps.keys() and Ls.wpe == Lg.wpe == bs
            assert all(np.array_equal(Pg[k], Ps[k]) for k in Pg)      # exact dyadics
    bg = np.empty_like(gen.b.reshape(-1, bs))
    bg[pf] = gen.b.reshape(-1, bs)
    assert np.max(np.abs(bg - b.reshape(-1, bs))) <= 1e-13 * np.max(np.abs(bg))


@pytest.mark.parametrize("P", [2, 3])
def test_rank_rows_equal_global_rows_bitwise(P):
    root, R = (2, 2, 4), 3
    glob, bg, _ = S.build_rank(1, 0, root=root, R=R)
    parts = [S.build_rank(P, r, root=root, R=R, min_rows_per_rank=8) for r in range(P)]
    ranges = parts[0][2]
    kinds = ["R" if all(rg == (0, S.n_nodes(S.grid(root, l))) for rg in ranges[l]) else "D"
             for l in range(R + 1)]
    assert kinds[0] == "R" and kinds[-1] == "D"
    for l in range(R + 1):
        G = glob[l]
        lv = [p[0][l] for p in parts]
        for r in range(P):
            assert (lv[r].row_begin, lv[r].row_end) == ranges[l][r] and lv[r].n_global == G.n
        if kinds[l] == "R":
            for L in lv:
                assert np.array_equal(L.row_ptr, G.row_ptr) and np.array_equal(L.col, G.col)
                assert np.array_equal(L.val, G.val)
            continue
        assert [L.row_begin for L in lv] == sorted(L.row_begin for L in lv) and lv[-1].row_end == G.n
        rp = np.concatenate([[0]] + [L.row_ptr[1:] + sum(x.nnzb for x in lv[:i]) for i, L in enumerate(lv)])
        assert np.array_equal(rp, G.row_ptr)
        assert np.array_equal(np.concatenate([L.col for L in lv]), G.col)
        assert np.array_equal(np.concatenate([L.val for L in lv]), G.val)
        if l > 0:
            assert np.array_equal(np.concatenate([L.P[1] for L in lv]), G.P[1])
            assert np.array_equal(np.concatenate([L.P[2] for L in lv]), G.P[2])
    assert np.array_equal(np.concatenate([p[1] for p in parts]), bg)
    # coarse node (i,j,k) of a distributed level lives with fine node (2i,2j,2k)
    for l in range(1, R):
        if kinds[l] != "D":
            continue
        g, gf = S.grid(root, l), S.grid(root, R)
        s = 1 << (R - l)
        for r in range(P):
            c0, c1 = ranges[l][r]
            for cid in (c0, c1 - 1):
                if c1 <= c0:
                    continue
                pl = (g[0] + 1) * (g[1] + 1)
                k, rest = divmod(cid, pl)
                j, i = divmod(rest, g[0] + 1)
                fid = i * s + (gf[0] + 1) * (j * s + (gf[1] + 1) * k * s)
                f0, f1 = ranges[R][r]
                assert f0 <= fid < f1


def test_weak_scaling_sizes():
    """17.1M / 33.3M / 57.4M / 135.5M DOFs at P = 1/2/4/8."""
    sizes = {P: S.n_dof(P) for P in (1, 2, 4, 8)}
    assert sizes[1] == 17_106_948 and sizes[8] == 135_532_548
    per_gpu = [sizes[P] / P / 1e6 for P in (1, 2, 4, 8)]
    assert all(14.0 < v < 17.2 for v in per_gpu)
