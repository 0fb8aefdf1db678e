"""ORACLE (test infrastructure only) — mesh preparation on the host.

Implements the canonical flat-array contract of SURVEY.md §8(b) C1-C10 with
plain numpy.  The paper's mesh handling is libMesh; it
allows "level-one mesh incompatibility" only, which we
read as 2:1 balance across edges (2D) / faces and edges (3D) (C10).
Hanging nodes are interpolated linearly from the unconstrained DOFs
(Eq. 6): weight 1/2 at mid-edge nodes and 1/4 at 3D
face centres.
"""
from __future__ import annotations

from dataclasses import dataclass
import itertools

import numpy as np

from inputs import Problem, density_at


def morton(coords: np.ndarray) -> np.ndarray:
    """Morton key: bit b of axis c goes to bit d*b + c (x least significant), C2."""
    coords = np.asarray(coords, dtype=np.int64)
    d = coords.shape[1]
    key = np.zeros(coords.shape[0], dtype=np.int64)
    top = int(coords.max()) if coords.size else 0
    assert coords.size == 0 or (int(coords.min()) >= 0 and top < (1 << 21))
    for b in range(max(1, top.bit_length())):          # higher bits are all zero
        for c in range(d):
            key |= ((coords[:, c] >> b) & 1) << (d * b + c)
    return key


def _dirs(dim: int):
    """Neighbour directions for the balance rule: edges in 2D; faces+edges in 3D (C10)."""
    out = []
    for v in itertools.product((-1, 0, 1), repeat=dim):
        nz = sum(1 for t in v if t != 0)
        if dim == 2 and nz == 1:
            out.append(v)
        if dim == 3 and nz in (1, 2):
            out.append(v)
    return np.array(out, dtype=np.int64)


def balance(prob: Problem, level: np.ndarray, anchor: np.ndarray, max_rounds: int = 64):
    """2:1 balance (C10): refine the coarser leaf until no face/edge neighbour
    differs by more than one level.  Point location by Morton search in the
    sorted linear tree."""
    dim, L = prob.dim, prob.L
    ext = np.array(prob.lattice_extent, dtype=np.int64)
    lev = level.astype(np.int64).copy()
    anc = anchor.astype(np.int64).copy()
    dirs = _dirs(dim)
    for _ in range(max_rounds):
        keys = morton(anc)
        order = np.argsort(keys, kind="stable")
        lev, anc, keys = lev[order], anc[order], keys[order]
        s = (1 << (L - lev))
        mark = np.zeros(lev.shape[0], dtype=bool)
        for dvec in dirs:
            q = anc + dvec[None, :] * s[:, None]
            inside = np.all((q >= 0) & (q < ext[None, :]), axis=1)
            ii = np.nonzero(inside)[0]
            if ii.size == 0:
                continue
            j = np.searchsorted(keys, morton(q[ii]), side="right") - 1
            bad = lev[j] < lev[ii] - 1
            mark[j[bad]] = True
        if not mark.any():
            return lev.astype(np.int8), anc.astype(np.int32)
        ref = np.nonzero(mark)[0]
        keep = ~mark
        half = (s[ref] // 2)
        kids = []
        for corner in range(1 << dim):
            off = np.array([(corner >> c) & 1 for c in range(dim)], dtype=np.int64)
            kids.append(anc[ref] + off[None, :] * half[:, None])
        anc = np.concatenate([anc[keep]] + kids)
        lev = np.concatenate([lev[keep]] + [lev[ref] + 1] * (1 << dim))
    raise RuntimeError("balance did not converge")


@dataclass
class OracleMesh:
    dim: int
    L: int
    hL: float
    elem_level: np.ndarray    # int8 [n_el]          C2 order
    elem_anchor: np.ndarray   # int32 [n_el, dim]
    elem_node: np.ndarray     # int32 [n_el, 2^dim]  C4 corner order
    node_coord: np.ndarray    # int64 [n_node, dim]  lattice coordinates, C3 order
    hang_node: np.ndarray     # int32 [n_hang]       ascending
    hang_ptr: np.ndarray      # int32 [n_hang+1]
    hang_parent: np.ndarray   # int32 [nnz]          ascending within a row
    hang_weight: np.ndarray   # float64 [nnz]
    fixed_dof: np.ndarray     # int64 [n_fixed]      ascending, no hanging DOFs
    load: np.ndarray          # float64 [dim*n_node] consistent nodal loads (before projection)
    filt_ptr: np.ndarray      # int64 [n_el+1]
    filt_idx: np.ndarray      # int32 [nnz]
    density: np.ndarray       # float64 [n_el]  input density (raw, before any presmoothing)

    @property
    def n_el(self):
        return self.elem_level.shape[0]

    @property
    def n_node(self):
        return self.node_coord.shape[0]

    @property
    def n_dof(self):
        return self.dim * self.n_node

    def size(self):
        return (1 << (self.L - self.elem_level.astype(np.int64)))

    def centers(self):
        """C1: (a + s/2) h_L."""
        return (self.elem_anchor.astype(np.float64) + 0.5 * self.size()[:, None]) * self.hL

    def volumes(self):
        """C1: V_e = (s h_L)^d."""
        return (self.size().astype(np.float64) * self.hL) ** self.dim

    def h(self):
        return self.size().astype(np.float64) * self.hL


def corner_offsets(dim):
    """Local corner c = cx + 2 cy + 4 cz (C4)."""
    return np.array([[(c >> k) & 1 for k in range(dim)] for c in range(1 << dim)], dtype=np.int64)


def _node_lookup(keys_sorted, coords):
    k = morton(coords)
    idx = np.searchsorted(keys_sorted, k)
    idx_c = np.minimum(idx, keys_sorted.shape[0] - 1)
    found = keys_sorted[idx_c] == k
    return np.where(found, idx_c, -1)


def hanging_constraints(dim, elem_anchor, size, node_keys):
    """C6: a node is hanging iff it lies in the relative interior of an edge
    (or, in 3D, a face) of some leaf; with 2:1 balance it is then that edge's
    midpoint (parents: 2 endpoints, w = 1/2) or that face's centre (parents: 4
    corners, w = 1/4).  Returns dict node -> tuple(sorted parents)."""
    offs = corner_offsets(dim)
    hang = {}
    coarse = size >= 2
    A = elem_anchor[coarse].astype(np.int64)
    S = size[coarse].astype(np.int64)
    # edges: pairs of corners differing in exactly one axis
    edges = [(a, b) for a in range(1 << dim) for b in range(a + 1, 1 << dim)
             if bin(a ^ b).count("1") == 1]
    faces = []
    if dim == 3:
        for axis in range(3):
            for side in (0, 1):
                faces.append([c for c in range(8) if ((c >> axis) & 1) == side])
    for group, w in [(e, 0.5) for e in edges] + [(f, 0.25) for f in faces]:
        pts = [A + offs[c][None, :] * S[:, None] for c in group]
        mid = sum(pts) // len(group)
        nid = _node_lookup(node_keys, mid)
        has = np.nonzero(nid >= 0)[0]
        if has.size == 0:
            continue
        par = np.stack([_node_lookup(node_keys, p[has]) for p in pts], axis=1)
        assert np.all(par >= 0)
        par.sort(axis=1)
        for n, prow in zip(nid[has].tolist(), par.tolist()):
            t = tuple(prow)
            if n in hang:
                assert hang[n] == t, "inconsistent hanging classification"
            else:
                hang[n] = t
    return hang


def build_mesh(prob: Problem, with_filter: bool = True, density: bool = True) -> OracleMesh:
    dim, L = prob.dim, prob.L
    lev, anc = balance(prob, prob.leaf_level, prob.leaf_anchor)
    keys = morton(anc)
    order = np.argsort(keys, kind="stable")
    lev, anc = lev[order], anc[order].astype(np.int64)
    size = (1 << (L - lev.astype(np.int64)))
    offs = corner_offsets(dim)
    corners = anc[:, None, :] + offs[None, :, :] * size[:, None, None]       # [n_el, 2^d, d]
    flat = corners.reshape(-1, dim)
    ck = morton(flat)
    uk, first = np.unique(ck, return_index=True)
    node_coord = flat[first]
    node_keys = uk
    elem_node = np.searchsorted(node_keys, ck).reshape(-1, 1 << dim).astype(np.int32)
    n_node = node_coord.shape[0]

    hang = hanging_constraints(dim, anc, size, node_keys)
    hn = np.array(sorted(hang), dtype=np.int32)
    hptr = np.zeros(hn.shape[0] + 1, dtype=np.int32)
    hpar, hw = [], []
    for i, n in enumerate(hn.tolist()):
        ps = hang[n]
        hptr[i + 1] = hptr[i] + len(ps)
        hpar.extend(ps)
        hw.extend([1.0 / len(ps)] * len(ps))
    hpar = np.array(hpar, dtype=np.int32)
    hw = np.array(hw, dtype=np.float64)
    is_hang = np.zeros(n_node, dtype=bool)
    is_hang[hn] = True

    # C7: fixed DOFs by geometric predicate, excluding hanging nodes
    fixed = []
    for lo, hi, mask in prob.fixed:
        lo = np.array(lo, dtype=np.int64)
        hi = np.array(hi, dtype=np.int64)
        sel = np.all((node_coord >= lo) & (node_coord <= hi), axis=1) & ~is_hang
        for c in range(dim):
            if (mask >> c) & 1:
                fixed.append(np.nonzero(sel)[0] * dim + c)
    fixed_dof = np.unique(np.concatenate(fixed)) if fixed else np.zeros(0, dtype=np.int64)

    # C8: consistent nodal loads
    load = np.zeros(dim * n_node, dtype=np.float64)
    hL = prob.hL
    for kind, lo, hi, vec in prob.loads:
        lo = np.array(lo, dtype=np.int64)
        hi = np.array(hi, dtype=np.int64)
        vec = np.array(vec, dtype=np.float64)
        if kind == "point":
            nid = _node_lookup(node_keys, lo[None, :])[0]
            assert nid >= 0, "point load not on a node"
            load[dim * nid:dim * nid + dim] += vec
            continue
        span = [c for c in range(dim) if hi[c] != lo[c]]
        fixed_axes = [c for c in range(dim) if hi[c] == lo[c]]
        if kind == "line":
            assert len(span) == 1
        elif kind == "face":
            assert len(span) == 2 and dim == 3
        # leaves having a (d-1 or 1)-dimensional boundary piece inside the region
        sel = np.ones(anc.shape[0], dtype=bool)
        for c in fixed_axes:
            sel &= (anc[:, c] == lo[c]) | (anc[:, c] + size == lo[c])
        for c in span:
            sel &= (anc[:, c] >= lo[c]) & (anc[:, c] + size <= hi[c])
        # each boundary piece spreads vec * measure equally over its 2^len(span) corners
        es = np.nonzero(sel)[0]
        s = size[es].astype(np.int64)
        measure = (s.astype(np.float64) * hL) ** len(span)
        npts = 1 << len(span)
        for m in range(npts):
            p = np.empty((es.shape[0], dim), dtype=np.int64)
            for c in fixed_axes:
                p[:, c] = lo[c]
            for t, c in enumerate(span):
                p[:, c] = anc[es, c] + ((m >> t) & 1) * s
            nid = _node_lookup(node_keys, p)
            assert np.all(nid >= 0)
            for c in range(dim):
                np.add.at(load, dim * nid.astype(np.int64) + c, vec[c] * (measure / npts))

    mesh = OracleMesh(dim=dim, L=L, hL=hL, elem_level=lev.astype(np.int8),
                      elem_anchor=anc.astype(np.int32), elem_node=elem_node,
                      node_coord=node_coord, hang_node=hn, hang_ptr=hptr, hang_parent=hpar,
                      hang_weight=hw, fixed_dof=fixed_dof.astype(np.int64), load=load,
                      filt_ptr=np.zeros(1, dtype=np.int64), filt_idx=np.zeros(0, dtype=np.int32),
                      density=np.zeros(0))
    if density:
        mesh.density = density_at(prob, mesh.elem_level, mesh.elem_anchor)
    if with_filter:
        mesh.filt_ptr, mesh.filt_idx = filter_neighbours(mesh, prob.rmin)
    return mesh


def filter_neighbours(mesh: OracleMesh, rmin: float):
    """C9: for each element (C2 order) every d with |c_d - c_e|^2 < rmin^2,
    ascending, self included (Eq. 4: H_de > 0)."""
    from scipy.spatial import cKDTree
    c = mesh.centers()
    n = c.shape[0]
    tree = cKDTree(c)
    lists = tree.query_ball_point(c, r=rmin, p=2.0, eps=0.0)
    ptr = np.zeros(n + 1, dtype=np.int64)
    idx = []
    r2 = rmin * rmin
    for e in range(n):
        cand = np.array(sorted(lists[e]), dtype=np.int64)
        if cand.size:
            d2 = ((c[cand] - c[e][None, :]) ** 2).sum(axis=1)
            cand = cand[d2 < r2]
        idx.append(cand)
        ptr[e + 1] = ptr[e] + cand.size
    idx = np.concatenate(idx).astype(np.int32) if idx else np.zeros(0, dtype=np.int32)
    return ptr, idx


def filter_neighbours_bruteforce(mesh: OracleMesh, rmin: float):
    """O(n^2) twin of C9 for tiny meshes."""
    c = mesh.centers()
    n = c.shape[0]
    ptr = [0]
    idx = []
    for e in range(n):
        for d in range(n):
            if ((c[d] - c[e]) ** 2).sum() < rmin * rmin:
                idx.append(d)
        ptr.append(len(idx))
    return np.array(ptr, dtype=np.int64), np.array(idx, dtype=np.int32)
