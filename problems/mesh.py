"""Hierarchical quadtree/octree meshes with hanging nodes and global coarsening.

SEEDED INPUT GENERATOR (test/bench infrastructure). This module produces the
*inputs* of the hot path (meshes -> assembled systems -> transfer matrices).
It holds none of the multigrid solve arithmetic: the V-cycle, smoother,
transfers and Krylov ops live in the CUDA library (product) and, independently,
in `oracle/` (test reference). Both consume what this module generates.

Paper passages followed (PAPER.md line numbers, "P:n"):
  * P:106, P:143  local refinement 1 -> 4 (2d) / 1 -> 8 (3d) children, level
                  jump <= 1 between neighbours, "at most 1 hanging node per face".
  * P:143-144     hanging nodes are replaced by interpolation of their direct
                  neighbours (edge midpoint: 2 masters x 1/2, face centre:
                  4 masters x 1/4).
  * P:156-158     global coarsening: "an element is coarsened, if it belongs to a
                  group of four (in 3d eight) elements on the same mesh level that
                  all arise from splitting the same common father element"; "as
                  many refinements as possible are taken back" per step; every
                  level spans the whole domain.
  * P:445, Table `ndofs`  refinement towards a face / edge / vertex;
                  reading Z16: the 4h band rule reproduces all 18
                  node counts of Table `ndofs` exactly (pinned in tests).

Representation: a mesh is a set of leaf cells (level, integer cell coords at
that level) over a root box of `root` cells.  Nodes live on an integer lattice
at a reference level R (>= every leaf level of the hierarchy); node keys are
Morton codes of lattice coordinates, so sorting by key gives the Morton node
numbering used on every level (reading G2 in DESIGN.md).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

# --------------------------------------------------------------------------
# Morton codes (bit interleaving), int64
# --------------------------------------------------------------------------


def _spread2(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64) & np.uint64(0xFFFFFFFF)
    v = (v | (v << np.uint64(16))) & np.uint64(0x0000FFFF0000FFFF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF00FF00FF)
    v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F0F0F0F0F)
    v = (v | (v << np.uint64(2))) & np.uint64(0x3333333333333333)
    v = (v | (v << np.uint64(1))) & np.uint64(0x5555555555555555)
    return v


def _spread3(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64) & np.uint64(0x1FFFFF)
    v = (v | (v << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
    v = (v | (v << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
    v = (v | (v << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
    v = (v | (v << np.uint64(2))) & np.uint64(0x1249249249249249)
    return v


def morton(coords: np.ndarray) -> np.ndarray:
    """Morton key of integer lattice coordinates `coords` (n, d); axis 0 is the
    least significant bit of each interleaved group."""
    coords = np.asarray(coords)
    d = coords.shape[1]
    if d == 2:
        k = _spread2(coords[:, 0]) | (_spread2(coords[:, 1]) << np.uint64(1))
    elif d == 3:
        k = (_spread3(coords[:, 0]) | (_spread3(coords[:, 1]) << np.uint64(1))
             | (_spread3(coords[:, 2]) << np.uint64(2)))
    else:
        raise ValueError("dim must be 2 or 3")
    return k.astype(np.int64)


def lookup(sorted_keys: np.ndarray, q: np.ndarray):
    """(found mask, index) of keys `q` in the sorted unique array `sorted_keys`."""
    idx = np.searchsorted(sorted_keys, q)
    idx_c = np.minimum(idx, max(len(sorted_keys) - 1, 0))
    found = (idx < len(sorted_keys)) & (sorted_keys[idx_c] == q) if len(sorted_keys) else np.zeros(len(q), bool)
    return found, idx_c


# --------------------------------------------------------------------------
# Mesh
# --------------------------------------------------------------------------


@dataclass
class Mesh:
    dim: int
    root: tuple          # number of root cells per axis
    lev: np.ndarray      # (n,) int64 leaf level (0 = root cell)
    ijk: np.ndarray      # (n, dim) int64 cell coords at the leaf's own level

    @property
    def n_cells(self) -> int:
        return int(self.lev.shape[0])

    @property
    def max_level(self) -> int:
        return int(self.lev.max()) if self.n_cells else 0

    def cell_keys(self, level: int, ijk: np.ndarray) -> np.ndarray:
        return cell_key(self.root, level, ijk)

    def sorted(self) -> "Mesh":
        """Canonical leaf order: by (level, key) -- makes meshes comparable."""
        order = np.lexsort((cell_key_any(self.root, self.lev, self.ijk), self.lev))
        return Mesh(self.dim, self.root, self.lev[order], self.ijk[order])


def cell_key(root, level: int, ijk: np.ndarray) -> np.ndarray:
    """Linear key of cells `ijk` (n, d) at one level (row-major, axis 0 fastest)."""
    ijk = np.asarray(ijk, np.int64)
    n = [int(r) << level for r in root]
    key = ijk[:, -1].copy()
    for a in range(len(root) - 2, -1, -1):
        key = key * n[a] + ijk[:, a]
    return key


def cell_key_any(root, lev: np.ndarray, ijk: np.ndarray) -> np.ndarray:
    out = np.empty(lev.shape[0], np.int64)
    for q in np.unique(lev):
        m = lev == q
        out[m] = cell_key(root, int(q), ijk[m])
    return out


def uniform(root, dim: int | None = None) -> Mesh:
    root = tuple(int(r) for r in root)
    dim = len(root) if dim is None else dim
    grids = np.meshgrid(*[np.arange(r) for r in root], indexing="ij")
    ijk = np.stack([g.ravel(order="F") for g in grids], axis=1).astype(np.int64)
    return Mesh(dim, root, np.zeros(ijk.shape[0], np.int64), ijk)


def _corner_offsets(dim: int) -> np.ndarray:
    """Corner c of a cell: bit a of c is the offset along axis a."""
    return np.array([[(c >> a) & 1 for a in range(dim)] for c in range(1 << dim)], np.int64)


def _ring_offsets(dim: int) -> np.ndarray:
    """Offsets o (relative to 2*ijk) of the level-(l+1) cells that share a face
    (or, in 3d, an edge) with a level-l cell.  Vertex-only neighbours are
    excluded: the 2:1 rule constrains faces and edges only."""
    out = []
    for o in itertools.product((-1, 0, 1, 2), repeat=dim):
        outside = sum(1 for v in o if v in (-1, 2))
        if 1 <= outside <= dim - 1:
            out.append(o)
    return np.array(out, np.int64)


def _children(lev, ijk, dim):
    offs = _corner_offsets(dim)
    cl = np.repeat(lev + 1, len(offs))
    cijk = (2 * ijk[:, None, :] + offs[None, :, :]).reshape(-1, dim)
    return cl, cijk


def internal_sets(mesh: Mesh) -> dict:
    """Sorted keys of refined (internal) cells per level: all strict ancestors
    of leaves."""
    L = mesh.max_level
    out = {}
    prev = np.zeros((0, mesh.dim), np.int64)
    for q in range(L - 1, -1, -1):
        fine = np.concatenate([mesh.ijk[mesh.lev == q + 1], prev], axis=0)
        par = fine >> 1
        keys = cell_key(mesh.root, q, par)
        keys, first = np.unique(keys, return_index=True)
        out[q] = keys
        prev = par[first]
    return out


def _in_domain(root, level, ijk):
    ok = np.ones(ijk.shape[0], bool)
    for a, r in enumerate(root):
        ok &= (ijk[:, a] >= 0) & (ijk[:, a] < (int(r) << level))
    return ok


def _touches_refined(mesh: Mesh, lev_q: int, ijk: np.ndarray, internal_next: np.ndarray) -> np.ndarray:
    """For cells at level q: does any face/edge-adjacent level-(q+1) cell have
    children, i.e. is there a leaf of level >= q+2 across a face or edge?"""
    ring = _ring_offsets(mesh.dim)
    bad = np.zeros(ijk.shape[0], bool)
    if len(internal_next) == 0 or ijk.shape[0] == 0:
        return bad
    for o in ring:
        nb = 2 * ijk + o[None, :]
        ok = _in_domain(mesh.root, lev_q + 1, nb)
        keys = cell_key(mesh.root, lev_q + 1, np.where(ok[:, None], nb, 0))
        found, _ = lookup(internal_next, keys)
        bad |= found & ok
    return bad


def refine(mesh: Mesh, mask: np.ndarray) -> Mesh:
    """Replace marked leaves by their 2^d children, then close to 2:1 face (and,
    in 3d, edge) balance by refining transitively ("the actual refinement
    can therefore extend further into the domain")."""
    mask = np.asarray(mask, bool)
    while True:
        keep_l, keep_ijk = mesh.lev[~mask], mesh.ijk[~mask]
        cl, cijk = _children(mesh.lev[mask], mesh.ijk[mask], mesh.dim)
        mesh = Mesh(mesh.dim, mesh.root, np.concatenate([keep_l, cl]),
                    np.concatenate([keep_ijk, cijk], axis=0))
        mask = balance_violations(mesh)
        if not mask.any():
            return mesh


def balance_violations(mesh: Mesh) -> np.ndarray:
    """Leaves that have a face/edge neighbour two or more levels finer."""
    internal = internal_sets(mesh)
    bad = np.zeros(mesh.n_cells, bool)
    for q in range(mesh.max_level - 1):
        m = mesh.lev == q
        if m.any() and (q + 1) in internal:
            bad[m] = _touches_refined(mesh, q, mesh.ijk[m], internal[q + 1])
    return bad


def band_mark(mesh: Mesh, axes, K: int = 1) -> np.ndarray:
    """Band rule (reading Z16/G1): mark every leaf of the current finest level
    whose infinity-distance from the target entity {x_a = 0 : a in axes} is
    < 4*K*h, h the finest cell size.  In lattice units of the finest level that
    is max_a ijk_a < 4K (exact integer test)."""
    L = mesh.max_level
    m = mesh.lev == L
    d = np.max(mesh.ijk[:, list(axes)], axis=1)
    return m & (d < 4 * K)


def coarsen_step(mesh: Mesh) -> Mesh:
    """One global-coarsening step (reading G3 in DESIGN.md).

    Candidates: parents whose 2^d children are all leaves of the input mesh
    (each element merges at most once per step).  Processed deepest level
    first; a merge of parent Q (level q) is rejected if, after the deeper merges
    of this step, a cell of level q+1 sharing a face/edge with Q is still
    refined (that would leave a level-(q+2) leaf next to the new level-q leaf,
    breaking 2:1).  Same-level merges never affect each other's legality, so
    the result is independent of the order inside a level."""
    dim, root = mesh.dim, mesh.root
    nch = 1 << dim
    has_parent = mesh.lev > 0
    plev = mesh.lev - 1
    pijk = mesh.ijk >> 1
    pkey = np.where(has_parent, cell_key_any(root, np.maximum(plev, 0), pijk), -1)
    # group leaves by (plev, pkey)
    gid = np.where(has_parent, plev * (np.int64(1) << 50) + pkey, -1)
    ug, inv, cnt = np.unique(gid, return_inverse=True, return_counts=True)
    cand_group = (cnt == nch) & (ug >= 0)
    internal = internal_sets(mesh)
    merged_keys = {}
    L = mesh.max_level
    for q in range(L - 1, -1, -1):
        sel = cand_group & ((ug >> 50) == q)
        if not sel.any():
            continue
        # representative parent coords: first child of each group
        leaf_mask = cand_group[inv] & (plev == q)
        lidx = np.nonzero(leaf_mask)[0]
        g_of_leaf = inv[lidx]
        _, first = np.unique(g_of_leaf, return_index=True)
        qijk = pijk[lidx[first]]
        inext = internal.get(q + 1, np.zeros(0, np.int64))
        if (q + 1) in merged_keys and len(merged_keys[q + 1]):
            inext = np.setdiff1d(inext, merged_keys[q + 1], assume_unique=True)
        bad = _touches_refined(mesh, q, qijk, inext)
        merged_keys[q] = np.sort(cell_key(root, q, qijk[~bad]))
    # build new leaf set
    keep = np.ones(mesh.n_cells, bool)
    new_l, new_ijk = [], []
    for q, keys in merged_keys.items():
        if len(keys) == 0:
            continue
        m = (plev == q) & has_parent
        found, _ = lookup(keys, np.where(m, pkey, -1))
        kill = m & found
        keep &= ~kill
        # one parent per merged key
        ijk_q = np.stack(np.unravel_index(keys, [int(r) << q for r in root][::-1]), axis=1)[:, ::-1]
        new_l.append(np.full(len(keys), q, np.int64))
        new_ijk.append(ijk_q.astype(np.int64))
    lev = np.concatenate([mesh.lev[keep]] + new_l)
    ijk = np.concatenate([mesh.ijk[keep]] + new_ijk, axis=0)
    return Mesh(dim, root, lev, ijk)


def hierarchy(fine: Mesh, max_levels: int = 64) -> list:
    """Ω_0 ⪯ ... ⪯ Ω_L by repeated global coarsening until the root mesh
    (root cells are never merged: Ω_0 is "the coarse starting mesh").
    Returned coarse -> fine."""
    levels = [fine]
    while levels[-1].max_level > 0 and len(levels) < max_levels:
        c = coarsen_step(levels[-1])
        if c.n_cells == levels[-1].n_cells:
            raise RuntimeError("global coarsening stalled before reaching the root mesh")
        levels.append(c)
    return levels[::-1]


# --------------------------------------------------------------------------
# Nodes, connectivity, hanging nodes
# --------------------------------------------------------------------------


@dataclass
class NodeSet:
    R: int                  # lattice reference level
    keys: np.ndarray        # (N,) sorted Morton keys
    coords: np.ndarray      # (N, d) lattice coords at level R
    conn: np.ndarray        # (n_cells, 2^d) node index per cell corner
    hanging: np.ndarray     # (N,) bool
    h_kind: np.ndarray      # (N,) 0 regular, 2 edge-midpoint, 4 face-centre
    h_masters: np.ndarray   # (N, 4) master node ids (-1 padded)
    h_weights: np.ndarray   # (N, 4) master weights


def build_nodes(mesh: Mesh, R: int | None = None) -> NodeSet:
    dim = mesh.dim
    R = mesh.max_level if R is None else R
    offs = _corner_offsets(dim)
    sh = (R - mesh.lev)[:, None, None]
    corners = (mesh.ijk[:, None, :] + offs[None, :, :]) << sh
    ck = morton(corners.reshape(-1, dim))
    keys, inv = np.unique(ck, return_inverse=True)
    conn = inv.reshape(mesh.n_cells, 1 << dim).astype(np.int64)
    coords = np.empty((len(keys), dim), np.int64)
    coords[inv] = corners.reshape(-1, dim)
    N = len(keys)
    kind = np.zeros(N, np.int64)
    masters = -np.ones((N, 4), np.int64)
    weights = np.zeros((N, 4))
    # candidate hanging points: edge midpoints and (3d) face centres of leaves
    m = mesh.lev < R
    base = mesh.ijk[m] << (R - mesh.lev[m])[:, None]
    s = (np.int64(1) << (R - mesh.lev[m] - 1))[:, None]
    # edges: direction a, the other coordinates at {0, 2s}
    for a in range(dim):
        others = [b for b in range(dim) if b != a]
        for sel in itertools.product((0, 2), repeat=dim - 1):
            e = np.zeros(dim, np.int64)
            for b, v in zip(others, sel):
                e[b] = v
            mid = base + s * e[None, :]
            mid[:, a] += s[:, 0]
            found, idx = lookup(keys, morton(mid))
            if not found.any():
                continue
            p0 = mid[found].copy(); p0[:, a] -= s[found, 0]
            p1 = mid[found].copy(); p1[:, a] += s[found, 0]
            _, i0 = lookup(keys, morton(p0))
            _, i1 = lookup(keys, morton(p1))
            hid = idx[found]
            kind[hid] = 2
            masters[hid, 0] = i0
            masters[hid, 1] = i1
            weights[hid, :2] = 0.5
    if dim == 3:
        for a in range(3):
            b, c = [x for x in range(3) if x != a]
            for side in (0, 2):
                e = np.zeros(3, np.int64)
                e[a] = side
                e[b] = 1
                e[c] = 1
                ctr = base + s * e[None, :]
                found, idx = lookup(keys, morton(ctr))
                if not found.any():
                    continue
                hid = idx[found]
                cf = ctr[found]
                sf = s[found, 0]
                ms = []
                for db, dc in ((-1, -1), (1, -1), (-1, 1), (1, 1)):
                    p = cf.copy()
                    p[:, b] += db * sf
                    p[:, c] += dc * sf
                    ms.append(lookup(keys, morton(p))[1])
                kind[hid] = 4
                masters[hid] = np.stack(ms, axis=1)
                weights[hid] = 0.25
    return NodeSet(R, keys, coords, conn, kind > 0, kind, masters, weights)


def boundary_nodes(mesh: Mesh, nodes: NodeSet) -> np.ndarray:
    """Nodes on ∂Ω of the root box (lattice coordinate 0 or max on any axis)."""
    mx = np.array([int(r) << nodes.R for r in mesh.root], np.int64)
    c = nodes.coords
    return np.any((c == 0) | (c == mx[None, :]), axis=1)
