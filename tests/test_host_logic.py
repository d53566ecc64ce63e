"""CPU tests of libmgb200.so without a GPU: the library loads, exports every
symbol declared in include/*.h, and its host-side setup logic (validation,
SELL-32-sigma layout, R = P^T, inverse blocks, dense inverse, column
localisation) agrees with the oracle / brute force.  Integer results are
compared bit-exactly."""
import ctypes
import os
import re

import numpy as np
import pytest

from mgtest_util import ROOT, problem

import oracle

HDRS = [os.path.join(ROOT, "include", h) for h in ("mg.h", "mg_internal.h", "ns.h", "newton.h")]


def _lib():
    import paper_2405_05047_b200 as m
    return m.lib()


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def declared_symbols():
    names = set()
    for h in HDRS:
        txt = open(h).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        txt = re.sub(r"typedef[^;]*;", "", txt)            # function-pointer types are not symbols
        for m in re.finditer(r"\b((?:mgi?|ns)_[a-z0-9_]+)\s*\(", txt):
            names.add(m.group(1))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    import paper_2405_05047_b200 as m
    names = declared_symbols()
    assert "mg_vcycle" in names and "mg_solve" in names and "mgi_sell_fill" in names and "ns_step" in names
    L = m.lib()
    for n in names:
        assert hasattr(L, n), f"{n} declared in include/ but not exported"
    # the python binding exposes the same names as the C ABI
    for n in [x for x in names if x.startswith(("mg_", "ns_"))]:
        assert hasattr(m, n), f"binding lacks {n}"
    assert m.mg_version().startswith("mgb200")


def _sell(rp, col, val, vpe, sigma=4096):
    L = _lib()
    n = len(rp) - 1
    ns, ne = ctypes.c_int64(), ctypes.c_int64()
    L.mgi_sell_size.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    assert L.mgi_sell_size(n, _p(rp), sigma, ctypes.byref(ns), ctypes.byref(ne)) == 0
    sp = np.zeros(ns.value + 1, np.int64)
    perm = np.zeros(ns.value * 32, np.int32)
    c = np.zeros(ne.value, np.int32)
    v = np.zeros(ne.value * vpe)
    L.mgi_sell_fill.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    assert L.mgi_sell_fill(n, _p(rp), _p(col), _p(val), vpe, sigma, _p(sp), _p(perm), _p(c), _p(v)) == 0
    return sp, perm, c, v


def _unsell(sp, perm, c, v, vpe, n):
    """Reconstruct CSR rows from the documented layout (mg_internal.h)."""
    rows = {}
    for s in range(len(sp) - 1):
        ln = (sp[s + 1] - sp[s]) // 32
        for lane in range(32):
            r = perm[s * 32 + lane]
            ents = []
            for k in range(ln):
                e = sp[s] + 32 * k + lane
                base = (e - lane) * vpe
                vals = []
                for j in range(vpe // 2):
                    vals += [v[base + 64 * j + 2 * lane], v[base + 64 * j + 2 * lane + 1]]
                if vpe & 1:
                    vals.append(v[base + 64 * (vpe // 2) + lane])
                ents.append((int(c[e]), vals))
            if r >= 0:
                rows[int(r)] = ents
            else:
                assert all(all(x == 0.0 for x in vals) for _, vals in ents)
    assert sorted(rows) == list(range(n))
    return rows


@pytest.mark.parametrize("name,sigma", [("c2_small", 32), ("c2_small", 4096), ("c3_small", 64)])
def test_sell_layout_roundtrip_bitexact(name, sigma):
    P = problem(name)
    lv = P.levels[-1]
    bs = lv.bs
    val = np.ascontiguousarray(lv.val.reshape(-1))
    sp, perm, c, v = _sell(lv.row_ptr, lv.col, val, bs * bs, sigma)
    rows = _unsell(sp, perm, c, v, bs * bs, lv.n)
    for i in range(lv.n):
        a, b = lv.row_ptr[i], lv.row_ptr[i + 1]
        got = rows[i]
        # true entries in CSR order, then zero padding
        for k in range(b - a):
            assert got[k][0] == lv.col[a + k]
            assert np.array_equal(np.array(got[k][1]), lv.val[a + k].reshape(-1))
        for k in range(b - a, len(got)):
            assert all(x == 0.0 for x in got[k][1])
            assert got[k][0] == (lv.col[b - 1] if b > a else 0)   # padding column stays in range
    # entry count = sum over windows of (sorted) slice maxima, brute force
    ln = np.diff(lv.row_ptr)
    expect = 0
    for w0 in range(0, lv.n, sigma):
        srt = np.sort(ln[w0:w0 + sigma])[::-1]
        expect += 32 * int(sum(srt[k] for k in range(0, len(srt), 32)))
    assert len(c) == expect
    if sigma >= 4096:
        assert len(c) <= 1.05 * lv.nnzb + 32 * 64


def test_sell_transfer_layout_wpe():
    P = problem("c3_small")
    lv = P.levels[-1]
    rp, col, w = lv.P
    w3 = np.ascontiguousarray(np.repeat(w, 3) * np.tile([1.0, 2.0, 3.0], len(w)))
    sp, perm, c, v = _sell(rp, col, w3, 3, 128)
    rows = _unsell(sp, perm, c, v, 3, lv.n)
    for i in range(0, lv.n, 7):
        for k in range(rp[i], rp[i + 1]):
            cc, vals = rows[i][k - rp[i]]
            assert cc == col[k] and vals == [w[k], 2 * w[k], 3 * w[k]]
    nc = P.levels[-2].n
    assert c.min() >= 0 and c.max() < nc          # rectangular: every stored column < n_coarse


def _tsell(rp, col, w, wpe, C, sigma):
    L = _lib()
    n = len(rp) - 1
    ns, ne = ctypes.c_int64(), ctypes.c_int64()
    assert L.mgi_tsell_size(ctypes.c_int64(n), _p(rp), C, sigma, ctypes.byref(ns), ctypes.byref(ne)) == 0
    sp = np.zeros(ns.value + 1, np.int64)
    perm = np.zeros(ns.value * C, np.int32)
    c = np.zeros(ne.value, np.int32)
    wf = np.zeros(ne.value * wpe, np.float32)
    st = L.mgi_tsell_fill(ctypes.c_int64(n), _p(rp), _p(col), _p(w), wpe, C, sigma, _p(sp), _p(perm), _p(c), _p(wf))
    return st, sp, perm, c, wf


@pytest.mark.parametrize("name,C,sigma", [("c3_small", 10, 40), ("c3_small", 10, 4100), ("c5_small", 8, 64),
                                           ("c2_small", 32, 4096)])
def test_transfer_sellc_layout_bitexact(name, C, sigma):
    """SELL-C transfer layout (mgi_tsell_fill, include/mg_internal.h): every
    P and R = P^T row reappears entry by entry in CSR order at
    slice_ptr[s] + k*C + r, weights bit-exact in fp32 (dyadic, G6), padding
    with weight 0 at an in-range column; rows are a permutation within the
    sigma windows."""
    P = problem(name)
    L = _lib()
    lv = P.levels[-1]
    nc = P.levels[-2].n
    rp, col, w = lv.P
    wpe = lv.wpe
    rrp = np.zeros(nc + 1, np.int64)
    rcol = np.zeros(len(col), np.int64)
    rw = np.zeros(len(w))
    assert L.mgi_csr_transpose(ctypes.c_int64(lv.n), ctypes.c_int64(nc), _p(rp), _p(col), _p(w), wpe,
                               _p(rrp), _p(rcol), _p(rw)) == 0
    for (trp, tcol, tw, n, ncols) in ((rp, col, w, lv.n, nc), (rrp, rcol, rw, nc, lv.n)):
        st, sp, perm, c, wf = _tsell(trp, tcol, np.ascontiguousarray(tw), wpe, C, sigma)
        assert st == 0
        seen = np.zeros(n, bool)
        for s in range(len(sp) - 1):
            ln = (sp[s + 1] - sp[s]) // C
            assert (sp[s + 1] - sp[s]) % C == 0
            for r in range(C):
                i = perm[s * C + r]
                if i < 0:
                    continue
                assert s * C // sigma == i // sigma          # permutation inside the window
                seen[i] = True
                a, b = trp[i], trp[i + 1]
                assert b - a <= ln
                for k in range(ln):
                    e = sp[s] + k * C + r
                    if k < b - a:
                        assert c[e] == tcol[a + k]
                        assert np.array_equal(wf[e * wpe:(e + 1) * wpe].astype(np.float64),
                                              tw[(a + k) * wpe:(a + k + 1) * wpe])
                    else:
                        assert np.all(wf[e * wpe:(e + 1) * wpe] == 0.0) and 0 <= c[e] < ncols
        assert seen.all()
    # a weight that is not exact in fp32 keeps the fp64 layout (status 2)
    w2 = np.ascontiguousarray(w.copy())
    w2[0] = 0.1
    assert _tsell(rp, col, w2, wpe, C, sigma)[0] == 2


@pytest.mark.parametrize("name", ["c2_small", "c3_small"])
def test_transpose_bitexact_vs_oracle(name):
    L = _lib()
    P = problem(name)
    for l in range(1, len(P.levels)):
        lv = P.levels[l]
        rp, col, w = lv.P
        nc = P.levels[l - 1].n
        orp = np.zeros(nc + 1, np.int64)
        ocol = np.zeros(len(col), np.int64)
        ow = np.zeros(len(w))
        L.mgi_csr_transpose.argtypes = [ctypes.c_int64, ctypes.c_int64] + [ctypes.c_void_p] * 3 + [ctypes.c_int] + \
            [ctypes.c_void_p] * 3
        assert L.mgi_csr_transpose(lv.n, nc, _p(rp), _p(col), _p(w), 1, _p(orp), _p(ocol), _p(ow)) == 0
        erp, ecol, ew = oracle.csr_transpose(lv.n, nc, rp, col, w)
        assert np.array_equal(orp, erp) and np.array_equal(ocol, ecol) and np.array_equal(ow, ew)


@pytest.mark.parametrize("name", ["c1", "c3_small"])
def test_block_inverse_vs_oracle(name):
    L = _lib()
    P = problem(name)
    lv = P.levels[-1]
    bs = lv.bs
    val = np.ascontiguousarray(lv.val.reshape(-1))
    d = np.zeros(lv.n * bs * bs)
    L.mgi_block_diag_inverse.argtypes = [ctypes.c_int64, ctypes.c_int] + [ctypes.c_void_p] * 4
    assert L.mgi_block_diag_inverse(lv.n, bs, _p(lv.row_ptr), _p(lv.col), _p(val), _p(d)) == 0
    e = oracle.block_diag_inverse(lv.n, bs, lv.row_ptr, lv.col, lv.val).reshape(-1)
    assert np.max(np.abs(d - e)) <= 1e-12 * np.max(np.abs(e))


def test_block_inverse_singular_and_missing_diag():
    L = _lib()
    rp = np.array([0, 1, 2], np.int64)
    col = np.array([0, 1], np.int64)
    val = np.array([1.0, 2.0, 2.0, 4.0, 1.0, 0.0, 0.0, 1.0])   # first block singular
    d = np.zeros(8)
    L.mgi_block_diag_inverse.argtypes = [ctypes.c_int64, ctypes.c_int] + [ctypes.c_void_p] * 4
    assert L.mgi_block_diag_inverse(2, 2, _p(rp), _p(col), _p(val), _p(d)) == -5
    col2 = np.array([1, 1], np.int64)
    assert L.mgi_block_diag_inverse(2, 2, _p(rp), _p(col2), _p(val), _p(d)) == -3


def test_dense_inverse_vs_numpy():
    L = _lib()
    rng = np.random.default_rng(5)
    for N in (1, 7, 64):
        A = rng.standard_normal((N, N)) + N * np.eye(N)
        a = A.copy()
        inv = np.zeros((N, N))
        L.mgi_dense_inverse.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        assert L.mgi_dense_inverse(N, _p(a), _p(inv)) == 0
        assert np.allclose(inv @ A, np.eye(N), atol=1e-12 * N)
    S = np.ones((3, 3))
    inv = np.zeros((3, 3))
    assert L.mgi_dense_inverse(3, _p(S), _p(inv)) == -5


def test_validate_csr_errors():
    L = _lib()
    L.mgi_validate_csr.argtypes = [ctypes.c_int64, ctypes.c_int64] + [ctypes.c_void_p] * 3 + [
        ctypes.c_int64, ctypes.c_int, ctypes.c_int64]
    rp = np.array([0, 2, 3], np.int64)
    col = np.array([0, 1, 1], np.int64)
    val = np.ones(3)
    assert L.mgi_validate_csr(2, 2, _p(rp), _p(col), _p(val), 1, 1, 0) == 0
    bad = np.array([1, 0, 1], np.int64)                       # unsorted
    assert L.mgi_validate_csr(2, 2, _p(rp), _p(bad), _p(val), 1, 0, 0) == -3
    oob = np.array([0, 2, 1], np.int64)                       # out of range
    assert L.mgi_validate_csr(2, 2, _p(rp), _p(oob), _p(val), 1, 0, 0) == -3
    nod = np.array([0, 1, 0], np.int64)                       # row 1 lacks its diagonal
    assert L.mgi_validate_csr(2, 2, _p(rp), _p(nod), _p(val), 1, 1, 0) == -3
    rpb = np.array([0, 3, 2], np.int64)                       # decreasing row_ptr
    assert L.mgi_validate_csr(2, 2, _p(rpb), _p(col), _p(val), 1, 0, 0) == -3
    nan = np.array([1.0, np.nan, 1.0])
    assert L.mgi_validate_csr(2, 2, _p(rp), _p(col), _p(nan), 1, 1, 0) == -4


def test_localize_columns_bruteforce():
    L = _lib()
    P = problem("c2_small")
    lv = P.levels[-1]
    n = lv.n
    L.mgi_localize_columns.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64] + [ctypes.c_void_p] * 5
    for r0, r1 in [(0, n // 3), (n // 3, 2 * n // 3), (2 * n // 3, n)]:
        rp = lv.row_ptr[r0:r1 + 1] - lv.row_ptr[r0]
        col = np.ascontiguousarray(lv.col[lv.row_ptr[r0]:lv.row_ptr[r1]])
        loc = np.zeros(len(col), np.int64)
        gh = np.zeros(len(col), np.int64)
        ng = ctypes.c_int64()
        assert L.mgi_localize_columns(r1 - r0, r0, r1, _p(np.ascontiguousarray(rp)), _p(col), _p(loc), _p(gh),
                                      ctypes.byref(ng)) == 0
        ghosts = sorted({int(c) for c in col if c < r0 or c >= r1})
        assert list(gh[:ng.value]) == ghosts
        back = np.where(loc < r1 - r0, loc + r0, np.array(ghosts + [0])[np.maximum(loc - (r1 - r0), 0)])
        assert np.array_equal(back, col)


def test_nccl_transport_loads_and_makes_unique_id():
    """The NCCL transport is dlopen'd: the library loads without it, and
    mg_get_unique_id (rank 0's bootstrap id) works without a GPU."""
    import paper_2405_05047_b200 as m
    uid = m.mg_get_unique_id()
    assert len(uid) == 128 and any(uid)
    assert uid != m.mg_get_unique_id()


def test_bench_byte_model_matches_survey():
    """bench.py's algorithmic-byte model on a hand-checkable level."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    info = {"n": 10, "nnzb": 27, "nnz_p": 5}
    sweep, sweep0, resid = bench.level_bytes(info, 3, False)
    a_stream = 27 * (8 * 9 + 4) + 8 * 11
    assert sweep == a_stream + 8 * 3 * 10 * 3 + 8 * 9 * 10
    assert sweep0 == 16 * 3 * 10 + 8 * 9 * 10
    assert resid == a_stream + 24 * 3 * 10
    sweep32, _, _ = bench.level_bytes(info, 3, False, vb=4)
    assert sweep - sweep32 == 27 * 4 * 9


def test_sell_entry_map_places_values_like_fill():
    """mgi_sell_entry_map (mg_update_matrix): scattering original entries through
    the map reproduces the layout mgi_sell_fill builds, bit for bit."""
    L = _lib()
    P = problem("c3_small")
    lv = P.levels[-1]
    V = lv.bs * lv.bs
    val = np.ascontiguousarray(lv.val.reshape(-1))
    sp, perm, c, v = _sell(lv.row_ptr, lv.col, val, V, 4096)
    m = np.zeros(lv.nnzb, np.int64)
    pos = np.zeros(lv.n, np.int32)
    L.mgi_sell_entry_map.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 5
    assert L.mgi_sell_entry_map(lv.n, _p(lv.row_ptr), _p(sp), _p(perm), _p(m), _p(pos)) == 0
    out = np.zeros_like(v)
    for k in range(lv.nnzb):
        e = m[k]
        lane = e % 32
        base = (e - lane) * V
        for j in range(V // 2):
            out[base + 64 * j + 2 * lane] = val[k * V + 2 * j]
            out[base + 64 * j + 2 * lane + 1] = val[k * V + 2 * j + 1]
        if V & 1:
            out[base + 64 * (V // 2) + lane] = val[k * V + V - 1]
        assert c[e] == lv.col[k]
    assert np.array_equal(out, v)
    assert np.array_equal(perm[pos], np.arange(lv.n))
