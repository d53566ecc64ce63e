"""Q1 finite elements on box cells: element matrices, condensed assembly,
hanging-node matrix H, Dirichlet elimination and grid transfers P.

SEEDED INPUT GENERATOR (test/bench infrastructure) -- produces the matrices the
hot path consumes; holds none of the solve arithmetic (see problems/mesh.py).

Paper passages (P:n = PAPER.md line n; S:n = SPEC.md line n):
  * P:93-108   Q^r elements, r = 1 only (A11); equal-order systems with n_c
               components stored node-major, matrix entries are n_c x n_c blocks.
  * P:143-144  hanging-node matrix H (identity rows for regular nodes, master
               weights in hanging rows); H^T in assembly.
  * P:327-337  prolongation u^{l+1} = P_l u^l with the reference coefficients
               chi_ij "the same for each mesh element"; R_l = P_l^T.
  * P:375-392  transport-diffusion: lambda = 0.01, b = (0,-1), BE dt = 0.02,
               exact solution theta_ex; lumped mass (Z13).
  * P:431-444, P:480  elasticity: lambda = 8e4, mu = 2e4, f = (0,-1,0),
               homogeneous Dirichlet, BE dt = 0.025 (reading Z14: 3x3 blocks of
               M + dt^2 K_e).
Readings G4-G6 / Z7-Z9: 2-point Gauss per direction, condensed
A_bar = H^T A H with identity hanging rows, symmetric Dirichlet elimination,
P = Pi_f E H_c Pi_c.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

from . import mesh as M
from ._native import lib, ptr

# --------------------------------------------------------------------------
# Reference Q1 element on [0,1]^d, 2-point Gauss rule
# --------------------------------------------------------------------------


def gauss2(dim: int):
    g = np.array([0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0)])
    pts = np.array(list(itertools.product(g, repeat=dim)))[:, ::-1]  # axis 0 fastest
    w = np.full(len(pts), 0.5 ** dim)
    return pts, w


def q1_basis(dim: int, xi: np.ndarray):
    """phi (nq, 2^d) and grad (nq, 2^d, d) of the Q1 basis; corner c has bit a
    of c = offset along axis a (matches mesh._corner_offsets)."""
    xi = np.atleast_2d(xi)
    nq = xi.shape[0]
    nloc = 1 << dim
    phi = np.ones((nq, nloc))
    grad = np.ones((nq, nloc, dim))
    for c in range(nloc):
        for a in range(dim):
            bit = (c >> a) & 1
            f = xi[:, a] if bit else 1.0 - xi[:, a]
            df = 1.0 if bit else -1.0
            phi[:, c] *= f
            for b in range(dim):
                grad[:, c, b] *= (df if b == a else f)
    return phi, grad


def _sym(A):
    """Mirror the upper triangle: bit-exact symmetry for symmetric integrands."""
    U = np.triu(A)
    return U + np.triu(A, 1).T


def reference_tensors(dim: int):
    """Unit-cube integrals by quadrature: M[i,j] = ∫φ_iφ_j,
    G[a][b][i,j] = ∫∂_aφ_i ∂_bφ_j, C[a][i,j] = ∫φ_i ∂_aφ_j."""
    xq, wq = gauss2(dim)
    phi, grad = q1_basis(dim, xq)
    Mref = _sym(np.einsum("q,qi,qj->ij", wq, phi, phi))
    G = np.einsum("q,qia,qjb->abij", wq, grad, grad)
    for a in range(dim):
        G[a, a] = _sym(G[a, a])
    C = np.einsum("q,qi,qja->aij", wq, phi, grad)
    return Mref, G, C


# --------------------------------------------------------------------------
# Operators: element matrix = sum_t S[e,t] T_t, T_t of shape (nloc*bs)^2
# --------------------------------------------------------------------------


@dataclass
class Operator:
    name: str
    bs: int
    symmetric: bool
    params: dict = field(default_factory=dict)


def element_terms(op: Operator, dim: int, h: np.ndarray):
    """Reference tensors T (n_terms, nl, nl) and per-element scales S (n_e, n_terms)
    for box cells of size h (n_e, d).  Physical integrals on a box:
    ∫φφ = vol M, ∫∂_aφ∂_bφ = vol/(h_a h_b) G_ab, ∫φ∂_aφ = vol/h_a C_a."""
    Mref, G, C = reference_tensors(dim)
    nloc = 1 << dim
    vol = np.prod(h, axis=1)
    T, S = [], []
    p = op.params
    if op.name == "poisson":
        for a in range(dim):
            T.append(G[a, a])
            S.append(vol / h[:, a] ** 2)
    elif op.name == "td":
        # M^l/dt + lambda K + B  (reading Z13: lumped mass)
        Ml = np.diag(Mref.sum(axis=1))
        T.append(Ml)
        S.append(vol / p["dt"])
        for a in range(dim):
            T.append(G[a, a])
            S.append(p["lam"] * vol / h[:, a] ** 2)
        for a in range(dim):
            if p["b"][a] != 0.0:
                T.append(C[a])
                S.append(p["b"][a] * vol / h[:, a])
    elif op.name == "elasticity":
        # M + dt^2 K_e, K_e[(i,c),(j,d)] = lam ∫∂_cφ_i∂_dφ_j
        #                 + mu (δ_cd ∇φ_i·∇φ_j + ∫∂_dφ_i∂_cφ_j)   (reading Z14)
        bs = dim
        lam, mu, dt = p["lam"], p["mu"], p["dt"]
        E = np.eye(bs)
        T.append(np.kron(Mref, E))  # node-major (i,c),(j,d)
        S.append(vol)
        for a in range(dim):
            for b in range(dim):
                Tab = np.zeros((nloc, bs, nloc, bs))
                # lam term: c=a, d=b  -> ∂_aφ_i ∂_bφ_j
                Tab[:, a, :, b] += lam * G[a, b]
                # mu ∫∂_dφ_i ∂_cφ_j with d=a, c=b
                Tab[:, b, :, a] += mu * G[a, b]
                if a == b:
                    for c in range(bs):
                        Tab[:, c, :, c] += mu * G[a, a]
                T.append(Tab.reshape(nloc * bs, nloc * bs))
                S.append(dt * dt * vol / (h[:, a] * h[:, b]))
        # make the sum of the (a,b) and (b,a) terms bit-symmetric: merge pairs
        T2, S2 = [T[0]], [S[0]]
        for a in range(dim):
            for b in range(a, dim):
                ia, ib = 1 + a * dim + b, 1 + b * dim + a
                if a == b:
                    T2.append(_sym(T[ia]))
                else:
                    T2.append(_sym(T[ia] + T[ib]))
                S2.append(S[ia])
        T, S = T2, S2
    elif op.name == "elasticity6":
        # The paper's first-order system for (u, v), backward Euler,
        # unknowns (u_1..u_d, v_1..v_d) node-major (reading N4):
        #   (u^m - u^{m-1})/dt - v^m = 0        ->  M u - dt M v        = M u^{m-1}
        #   (v^m - v^{m-1})/dt - div s(u^m) = f  ->  dt K_e u + M v      = M v^{m-1} + dt M f
        bs = 2 * dim
        lam, mu, dt = p["lam"], p["mu"], p["dt"]
        E = np.eye(dim)

        def place(Auu=None, Auv=None, Avu=None, Avv=None):
            Tb = np.zeros((nloc, bs, nloc, bs))
            for (blk, r0, c0) in ((Auu, 0, 0), (Auv, 0, dim), (Avu, dim, 0), (Avv, dim, dim)):
                if blk is not None:
                    Tb[:, r0:r0 + dim, :, c0:c0 + dim] = blk
            return Tb.reshape(nloc * bs, nloc * bs)

        Mb = np.einsum("ij,cd->icjd", Mref, E)
        T.append(place(Auu=Mb, Avv=Mb))
        S.append(vol)
        T.append(place(Auv=-Mb))
        S.append(dt * vol)
        for a in range(dim):
            for b in range(dim):
                Kab = np.zeros((nloc, dim, nloc, dim))
                Kab[:, a, :, b] += lam * G[a, b]
                Kab[:, b, :, a] += mu * G[a, b]
                if a == b:
                    for c in range(dim):
                        Kab[:, c, :, c] += mu * G[a, a]
                T.append(place(Avu=Kab))
                S.append(dt * vol / (h[:, a] * h[:, b]))
    elif op.name == "stokes":
        # Generalised Stokes, equal-order Q1, unknowns (p, u_1..u_d) node-major
        # (P:108), PSPG stabilisation + pressure-mass regularisation (reading Z23):
        #   (u/dt, v) + nu (grad u, grad v) - (p, div v) + (div u, q)
        #   + sum_T delta_T (grad p, grad q)_T + eps (p, q),
        #   delta_T = alpha (1/dt + nu/h_T^2)^-1.
        bs = dim + 1
        nu, dt = p["nu"], p["dt"]
        eps, alpha = p.get("eps", 1e-2), p.get("alpha", 1.0)
        hT = h.max(axis=1)
        delta = alpha / (1.0 / dt + nu / hT ** 2)

        def blk(A, r, c):
            Tb = np.zeros((nloc, bs, nloc, bs))
            Tb[:, r, :, c] = A
            return Tb.reshape(nloc * bs, nloc * bs)

        T.append(sum(blk(Mref, c, c) for c in range(1, bs)))
        S.append(vol / dt)
        for a in range(dim):
            T.append(sum(blk(G[a, a], c, c) for c in range(1, bs)))
            S.append(nu * vol / h[:, a] ** 2)
            T.append(blk(G[a, a], 0, 0))
            S.append(delta * vol / h[:, a] ** 2)
        T.append(blk(Mref, 0, 0))
        S.append(eps * vol)
        for a in range(dim):
            # velocity row (i, 1+a), pressure col j: -int phi_j d_a phi_i ;
            # pressure row i, velocity col (j, 1+a): +int phi_i d_a phi_j
            T.append(blk(-C[a].T, 1 + a, 0) + blk(C[a], 0, 1 + a))
            S.append(vol / h[:, a])
    else:
        raise ValueError(op.name)
    return np.ascontiguousarray(np.stack(T)), np.ascontiguousarray(np.stack(S, axis=1))


# --------------------------------------------------------------------------
# Hanging-node matrix H and expansion
# --------------------------------------------------------------------------


def hanging_matrix(nodes: M.NodeSet):
    """H as CSR (row_ptr, col, w): identity rows for regular nodes, master
    weights in hanging rows.  Chains (a master that is itself hanging)
    are resolved by substitution so that masters are always regular."""
    N = len(nodes.keys)
    kind = nodes.h_kind
    cnt = np.where(kind > 0, kind, 1)
    rp = np.zeros(N + 1, np.int64)
    rp[1:] = np.cumsum(cnt)
    col = np.empty(rp[-1], np.int64)
    w = np.empty(rp[-1])
    reg = kind == 0
    col[rp[:-1][reg]] = np.nonzero(reg)[0]
    w[rp[:-1][reg]] = 1.0
    for k in (2, 4):
        m = kind == k
        if m.any():
            base = rp[:-1][m]
            for t in range(k):
                col[base + t] = nodes.h_masters[m, t]
                w[base + t] = nodes.h_weights[m, t]
    if np.any(kind[col] > 0):
        rp, col, w = _resolve_chains(rp, col, w, kind > 0)
    # CSR invariant: strictly increasing columns within a row
    rows = np.repeat(np.arange(N, dtype=np.int64), np.diff(rp))
    order = np.lexsort((col, rows))
    return rp, col[order], w[order]


def _resolve_chains(rp, col, w, hang):
    N = len(rp) - 1
    for _ in range(8):
        if not np.any(hang[col]):
            return rp, col, w
        rows = []
        for i in range(N):
            acc = {}
            for t in range(rp[i], rp[i + 1]):
                c = col[t]
                if hang[c] and c != i:
                    for u in range(rp[c], rp[c + 1]):
                        acc[col[u]] = acc.get(col[u], 0.0) + w[t] * w[u]
                else:
                    acc[c] = acc.get(c, 0.0) + w[t]
            rows.append(sorted(acc.items()))
        rp = np.zeros(N + 1, np.int64)
        rp[1:] = np.cumsum([len(r) for r in rows])
        col = np.array([c for r in rows for c, _ in r], np.int64)
        w = np.array([v for r in rows for _, v in r])
    raise RuntimeError("hanging-node chains did not resolve")


# --------------------------------------------------------------------------
# Assembly
# --------------------------------------------------------------------------


def cell_sizes(mesh: M.Mesh, box) -> np.ndarray:
    h0 = np.array([box[a] / mesh.root[a] for a in range(mesh.dim)])
    return h0[None, :] / (2.0 ** mesh.lev)[:, None]


def assemble(mesh: M.Mesh, nodes: M.NodeSet, op: Operator, box, H):
    """Condensed BSR  A_bar = H^T A H  (before Dirichlet / hanging identity rows).
    Returns row_ptr (n+1) int64, col (nnzb) int64, val (nnzb, bs, bs)."""
    T, S = element_terms(op, mesh.dim, cell_sizes(mesh, box))
    return assemble_terms(mesh, nodes, T, S, op.bs, op.symmetric, H)


def assemble_terms(mesh: M.Mesh, nodes: M.NodeSet, T: np.ndarray, S: np.ndarray, bs: int, symmetric: bool, H,
                   row_ptr=None):
    """Condensed BSR of the element matrices A_e = sum_t S[e, t] T_t (T (n_terms,
    nloc*bs, nloc*bs), S (n_e, n_terms)); the sparsity pattern depends on the
    mesh connectivity only, never on the values (row_ptr: a known pattern's row
    pointer skips the counting pass)."""
    N = len(nodes.keys)
    nloc = 1 << mesh.dim
    T = np.ascontiguousarray(T, np.float64)
    S = np.ascontiguousarray(S, np.float64)
    conn = np.ascontiguousarray(nodes.conn, np.int64)
    rp_h, col_h, w_h = (np.ascontiguousarray(a) for a in H)
    L = lib()
    if row_ptr is None:
        row_ptr = np.zeros(N + 1, np.int64)
        rc = L.asm_condensed(N, bs, nloc, mesh.n_cells, ptr(conn), ptr(rp_h), ptr(col_h), ptr(w_h),
                             T.shape[0], ptr(T), ptr(S), 0, 0, ptr(row_ptr), None, None)
        if rc != 0:
            raise RuntimeError("assembly pass 0 failed")
    else:
        row_ptr = np.array(row_ptr, np.int64)
    nnzb = int(row_ptr[-1])
    col = np.empty(nnzb, np.int64)
    val = np.empty((nnzb, bs, bs))
    rc = L.asm_condensed(N, bs, nloc, mesh.n_cells, ptr(conn), ptr(rp_h), ptr(col_h), ptr(w_h),
                         T.shape[0], ptr(T), ptr(S), 1, int(symmetric), ptr(row_ptr), ptr(col), ptr(val))
    if rc != 0:
        raise RuntimeError("assembly pass 1 failed")
    return row_ptr, col, val


def row_of(row_ptr: np.ndarray) -> np.ndarray:
    return np.repeat(np.arange(len(row_ptr) - 1, dtype=np.int64), np.diff(row_ptr))


def apply_constraints(row_ptr, col, val, cmask: np.ndarray, g: np.ndarray, b: np.ndarray | None):
    """Identity rows at constrained DOFs (hanging and Dirichlet) and symmetric
    elimination of their columns (readings Z7, Z9).
    cmask (n, bs) bool; g (n, bs) values at constrained DOFs (0 at hanging);
    b (n, bs) rhs updated in place: b_i -= A_ik g_k, b_k = g_k."""
    n, bs = cmask.shape
    rows = row_of(row_ptr)
    touch = cmask[rows].any(axis=1) | cmask[col].any(axis=1)
    k = np.nonzero(touch)[0]
    vk = val[k]
    if b is not None:
        gc = np.where(cmask, g, 0.0)
        corr = np.einsum("kij,kj->ki", vk, gc[col[k]])
        np.add.at(b, rows[k], -corr)
    rmask = ~cmask[rows[k]]            # (m, bs)
    cm = ~cmask[col[k]]
    vk = vk * rmask[:, :, None] * cm[:, None, :]
    diag = rows[k] == col[k]
    idx = np.nonzero(diag)[0]
    for c in range(bs):
        sel = idx[cmask[rows[k][idx], c]]
        vk[sel, c, c] = 1.0
    val[k] = vk
    if b is not None:
        b[cmask] = g[cmask]


def constraint_plan(row_ptr, col, cmask: np.ndarray):
    """The value-only part of apply_constraints (homogeneous g, no rhs) as a
    reusable plan for repeated assemblies on one pattern (Newton Jacobians):
    (entries touched, 0/1 keep mask per block entry, identity positions)."""
    n, bs = cmask.shape
    rows = row_of(row_ptr)
    touch = cmask[rows].any(axis=1) | cmask[col].any(axis=1)
    k = np.nonzero(touch)[0]
    keep = (~cmask[rows[k]])[:, :, None] & (~cmask[col[k]])[:, None, :]
    diag = np.nonzero(rows[k] == col[k])[0]
    ident = [(k[diag[cmask[rows[k][diag], c]]], c) for c in range(bs)]
    return k, keep.astype(np.float64), ident


def apply_constraint_plan(val, plan):
    """Same values as apply_constraints(..., g = 0, b = None)."""
    k, keep, ident = plan
    val[k] *= keep
    for idx, c in ident:
        val[idx, c, c] = 1.0


# --------------------------------------------------------------------------
# Transfers  P = Pi_f E H_c Pi_c   (reading G6 / Z8)
# --------------------------------------------------------------------------


def prolongation(coarse: M.Mesh, cnodes: M.NodeSet, Hc, c_free: np.ndarray,
                 fine: M.Mesh, fnodes: M.NodeSet, f_free: np.ndarray):
    """Scalar-weight P (n_f x n_c) CSR.  E[i,j] = phi_j^coarse(x_i^fine) from the
    finest coarse leaf containing fine node i (the reference chi_ij of Eq.
    `prolongation`; set, not summed), composed with the coarse
    hanging matrix H_c; rows of constrained fine nodes and columns of
    constrained coarse nodes are dropped (Pi_f, Pi_c).  c_free / f_free: (n,)
    bool "node is unconstrained" (all components share the mask here)."""
    dim = fine.dim
    nloc = 1 << dim
    offs = M._corner_offsets(dim)
    R = fnodes.R
    # coarse leaf lookup: for each fine leaf, its coarse leaf is itself or its parent
    ckeys = M.cell_key_any(coarse.root, coarse.lev, coarse.ijk)
    cid_sorted = np.lexsort((ckeys, coarse.lev))
    ck_lev = coarse.lev[cid_sorted]
    ck_key = ckeys[cid_sorted]
    comb = ck_lev * (np.int64(1) << 50) + ck_key
    fself = fine.lev * (np.int64(1) << 50) + M.cell_key_any(fine.root, fine.lev, fine.ijk)
    found_self, pos_self = M.lookup(comb, fself)
    plev = np.maximum(fine.lev - 1, 0)
    fpar = plev * (np.int64(1) << 50) + M.cell_key_any(fine.root, plev, fine.ijk >> 1)
    found_par, pos_par = M.lookup(comb, fpar)
    if not np.all(found_self | found_par):
        raise RuntimeError("fine leaf without coarse leaf: hierarchy not nested")
    cidx = np.where(found_self, cid_sorted[pos_self], cid_sorted[pos_par])
    clev = coarse.lev[cidx]
    # position of fine corners in the coarse cell's reference coords, in units of 1/2
    sub = np.where(found_self[:, None], 0, fine.ijk & 1)           # child offset in parent
    # xi2 (n_f, nloc, d) in {0,1,2}
    xi2 = np.where(found_self[:, None, None], 2 * offs[None], sub[:, None, :] + offs[None])
    # weights of coarse corner cc at xi2/2: prod_a (xi/2 if bit else 1 - xi/2)
    cbits = offs  # (nloc_c, d)
    x = xi2[:, :, None, :] / 2.0                                     # (n_f, nloc_f, 1, d)
    wts = np.prod(np.where(cbits[None, None, :, :] == 1, x, 1.0 - x), axis=3)  # (n_f, nloc_f, nloc_c)
    fnode = fnodes.conn                                              # (n_f, nloc)
    cnode = cnodes.conn[cidx]                                        # (n_f, nloc)
    # choose for each fine node the entry from the finest coarse leaf
    fn = fnode.ravel()
    lv = np.repeat(clev, nloc)
    order = np.lexsort((-lv, fn))
    fn_s = fn[order]
    first = np.ones(len(fn_s), bool)
    first[1:] = fn_s[1:] != fn_s[:-1]
    pick = order[first]                                              # one (leaf, corner) per fine node
    e_of = pick // nloc
    a_of = pick % nloc
    nf = len(fnodes.keys)
    assert len(pick) == nf
    W = wts[e_of, a_of]                                              # (nf, nloc_c)
    C = cnode[e_of]                                                  # (nf, nloc_c)
    # compose with coarse H: expand each coarse corner by its H row
    hrp, hcol, hw = Hc
    rows_i, cols_j, vals = [], [], []
    for cc in range(nloc):
        wcc = W[:, cc]
        nz = wcc != 0.0
        j = C[nz, cc]
        i = np.nonzero(nz)[0]
        cnt = hrp[j + 1] - hrp[j]
        rr = np.repeat(i, cnt)
        base = np.repeat(hrp[j], cnt)
        off = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        t = base + off
        rows_i.append(rr)
        cols_j.append(hcol[t])
        vals.append(np.repeat(wcc[nz], cnt) * hw[t])
    r = np.concatenate(rows_i)
    c = np.concatenate(cols_j)
    v = np.concatenate(vals)
    keep = f_free[r] & c_free[c]
    r, c, v = r[keep], c[keep], v[keep]
    # combine duplicates (sums of dyadics: exact)
    key = r * len(cnodes.keys) + c
    uk, inv = np.unique(key, return_inverse=True)
    vv = np.zeros(len(uk))
    np.add.at(vv, inv, v)
    rr = uk // len(cnodes.keys)
    cc_ = uk % len(cnodes.keys)
    nz = vv != 0.0
    rr, cc_, vv = rr[nz], cc_[nz], vv[nz]
    rp = np.zeros(nf + 1, np.int64)
    np.add.at(rp, rr + 1, 1)
    rp = np.cumsum(rp)
    return rp, cc_.astype(np.int64), vv
