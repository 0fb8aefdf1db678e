"""Morton-range partition of the general (AMR) path over ranks (SURVEY §8(e):
"contiguous C2 (Morton) element ranges ... each node is owned by ... ;
hanging-node parents on another rank join the halo"), host side.

The device decomposition of the general path is already "owner computes"
over contiguous ranges of the canonical (Morton, C3) node order
(kernels_genfused.cuh).  The multi-GPU partition is the same cut one level
up: rank r owns the nodes [n_r, n_{r+1}) (a union of whole blocks' worth of
nodes, balanced by incidence count).  Its local mesh holds

* every element that contributes to an owned node -- directly, or through a
  hanging corner whose Eq. 6 parent is owned;
* the local nodes: owned nodes first (in canonical order), then the ghosts
  (every other non-hanging corner of a local element and every parent of a
  local hanging corner: "hanging-node parents on another rank join the
  halo"), then the hanging corner nodes that are not owned;
* the hanging constraints of its hanging nodes (parents remapped, all local),
  the fixed DOFs and loads of its nodes (a hanging node's load reaches its
  owned parents through C^T, so b = Pi_F C^T f is exact on owned DOFs).

Per PCG iteration a rank needs, for its ghosts, the previous iterate's r, q
and p from their owners (send/recv lists below), the same data the
structured z-slab path pushes into its ghost planes; the dots are all-reduced
exactly as there.  Everything here is index bookkeeping (no method
arithmetic); tests/test_amr_shard_host.py checks that the owned part of the
operator computed from a rank's local mesh alone equals the global operator.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .api import HostMesh, Mesh, ipc_close, ipc_open


def node_incidence(host: HostMesh):
    """Node -> contributing elements (direct corner, or hanging corner whose
    parent is the node), as CSR (ptr, elems), elements ascending per node."""
    d = host.dim
    nc = 1 << d
    en = host.elem_node.reshape(-1, nc).astype(np.int64)
    hang_row = np.full(host.n_node, -1, dtype=np.int64)
    hang_row[host.hang_node] = np.arange(host.hang_node.shape[0])
    rows, cols = [], []
    h = hang_row[en]                                          # [n_el, nc]
    direct = h < 0
    rows.append(en[direct])
    cols.append(np.nonzero(direct)[0])
    e_h, c_h = np.nonzero(~direct)
    for e, row in zip(e_h, h[e_h, c_h]):
        ps = host.hang_parent[host.hang_ptr[row]:host.hang_ptr[row + 1]].astype(np.int64)
        rows.append(ps)
        cols.append(np.full(ps.shape[0], e, dtype=np.int64))
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    o = np.lexsort((cols, rows))
    rows, cols = rows[o], cols[o]
    keep = np.ones(rows.shape[0], dtype=bool)
    keep[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
    rows, cols = rows[keep], cols[keep]
    ptr = np.searchsorted(rows, np.arange(host.n_node + 1))
    return ptr, cols


def partition(host: HostMesh, nranks: int, ptr=None):
    """Contiguous node ranges [(n_r, n_{r+1})] of about equal incidence count
    (the per-node work of the owner-computes operator)."""
    if nranks < 1 or nranks > host.n_node:
        raise ValueError("bad rank count")
    if ptr is None:
        ptr, _ = node_incidence(host)
    cost = np.diff(ptr).astype(np.float64) + 1.0
    cum = np.concatenate([[0.0], np.cumsum(cost)])
    cuts = [0]
    for r in range(1, nranks):
        c = int(np.searchsorted(cum, cum[-1] * r / nranks))
        cuts.append(max(cuts[-1] + 1, min(c, host.n_node - (nranks - r))))
    cuts.append(host.n_node)
    return list(zip(cuts[:-1], cuts[1:]))


@dataclass
class AmrSlab:
    rank: int
    n0: int                          # owned global nodes [n0, n1)
    n1: int
    host: HostMesh                   # local mesh: owned nodes are local [0, n_own)
    n_own: int
    n_ghost: int                     # ghosts: local [n_own, n_own + n_ghost)
    node_global: np.ndarray          # local node -> global node
    elem_global: np.ndarray          # local element -> global element
    ghost_owner: np.ndarray          # [n_ghost] owning rank of each ghost
    recv: dict = field(default_factory=dict)   # rank s -> local ghost indices whose values come from s
    send: dict = field(default_factory=dict)   # rank s -> local owned indices that s needs


def slice_host(host: HostMesh, nranks: int, rank: int, ranges=None, inc=None) -> AmrSlab:
    """Rank `rank`'s local mesh and exchange lists (module docstring)."""
    d = host.dim
    nc = 1 << d
    if inc is None:
        inc = node_incidence(host)
    ptr, els_of = inc
    if ranges is None:
        ranges = partition(host, nranks, ptr)
    n0, n1 = ranges[rank]
    elems = np.unique(els_of[ptr[n0]:ptr[n1]])
    en = host.elem_node.reshape(-1, nc)[elems].astype(np.int64)
    is_hang = np.zeros(host.n_node, dtype=bool)
    is_hang[host.hang_node] = True
    hang_row = np.full(host.n_node, -1, dtype=np.int64)
    hang_row[host.hang_node] = np.arange(host.hang_node.shape[0])
    corners = np.unique(en)
    hang_c = corners[is_hang[corners]]
    parents = [host.hang_parent[host.hang_ptr[hang_row[g]]:host.hang_ptr[hang_row[g] + 1]] for g in hang_c]
    parents = np.unique(np.concatenate(parents).astype(np.int64)) if parents else np.zeros(0, np.int64)
    nonhang = np.union1d(corners[~is_hang[corners]], parents)
    owned = np.arange(n0, n1, dtype=np.int64)
    ghosts = np.setdiff1d(nonhang, owned)
    extra_hang = np.setdiff1d(hang_c, owned)                  # hanging corners outside the owned range
    node_global = np.concatenate([owned, ghosts, extra_hang])
    loc = np.full(host.n_node, -1, dtype=np.int64)
    loc[node_global] = np.arange(node_global.shape[0])
    # hanging constraints of the local hanging nodes (owned ones included), parents remapped
    lh = node_global[is_hang[node_global]]
    lh_local = loc[lh]
    order = np.argsort(lh_local, kind="stable")
    hptr, hpar, hw = [0], [], []
    for g in lh[order]:
        row = hang_row[g]
        ps = host.hang_parent[host.hang_ptr[row]:host.hang_ptr[row + 1]]
        ws = host.hang_weight[host.hang_ptr[row]:host.hang_ptr[row + 1]]
        lp = loc[ps]
        if np.any(lp < 0):
            raise AssertionError("a parent of a local hanging node is not local")
        o = np.argsort(lp)
        hpar.extend(lp[o].tolist())
        hw.extend(ws[o].tolist())
        hptr.append(len(hpar))
    fixed_g = host.fixed_dof
    fnode = fixed_g // d
    lf = loc[fnode]
    sel = lf >= 0
    fixed = np.sort(lf[sel] * d + fixed_g[sel] % d).astype(np.int64)
    load = host.load.reshape(-1, d)[node_global].reshape(-1).copy()
    local = HostMesh(
        dim=d, L=host.L, h0=host.h0,
        elem_node=loc[en].astype(np.int32), elem_anchor=host.elem_anchor[elems].copy(),
        elem_level=host.elem_level[elems].copy(), node_coord=host.node_coord[node_global].copy(),
        hang_node=np.sort(lh_local).astype(np.int32), hang_ptr=np.array(hptr, dtype=np.int32),
        hang_parent=np.array(hpar, dtype=np.int32), hang_weight=np.array(hw, dtype=np.float64),
        fixed_dof=fixed, load=load, filt_ptr=None, filt_idx=None, rmin=0.0)
    starts = np.array([a for a, _ in ranges])
    ghost_owner = np.searchsorted(starts, ghosts, side="right") - 1
    slab = AmrSlab(rank=rank, n0=n0, n1=n1, host=local, n_own=int(n1 - n0), n_ghost=int(ghosts.shape[0]),
                   node_global=node_global, elem_global=elems, ghost_owner=ghost_owner)
    for s in np.unique(ghost_owner).tolist():
        slab.recv[int(s)] = (n1 - n0) + np.nonzero(ghost_owner == s)[0]
    return slab


def exchange_lists(slabs):
    """send[s] of every slab from the recv lists of the others (the global
    node ids a rank receives are the ones its owner sends, same order)."""
    for sl in slabs:
        sl.send = {}
    for sl in slabs:
        for s, idx in sl.recv.items():
            g = sl.node_global[idx]
            owner = slabs[s]
            owner.send[sl.rank] = g - owner.n0
    return slabs


def send_entries_from(recvs, rank, n0):
    """Rank `rank`'s ghost-store list for to_gshard_attach from every rank's
    receive lists: recvs[r] = {source rank: (r's local ghost nodes, their
    global node ids)}; n0 = this rank's first owned global node.  Returns
    (destination rank, local owned node, the destination's local ghost node)
    per entry, destinations in rank order."""
    dst, loc, rem = [], [], []
    for r, rv in enumerate(recvs):
        if r == rank or rank not in rv:
            continue
        idx, g = rv[rank]                                       # r's ghost slots fed by this rank
        idx = np.asarray(idx)
        dst.append(np.full(idx.shape[0], r, dtype=np.int32))
        loc.append((np.asarray(g) - n0).astype(np.int32))
        rem.append(idx.astype(np.int32))
    if not dst:
        return np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.int32)
    return np.concatenate(dst), np.concatenate(loc), np.concatenate(rem)


def recv_lists(slab):
    """What a rank publishes to its peers: per source rank, its local ghost
    nodes and their global ids (the owner turns them into its send list)."""
    return {s: (idx, slab.node_global[idx]) for s, idx in slab.recv.items()}


def send_entries(slabs, rank):
    """send_entries_from for a group whose slabs all live in this process."""
    return send_entries_from([recv_lists(sl) for sl in slabs], rank, slabs[rank].n0)


def element_owner(host: HostMesh, ranges):
    """The rank that reports each element's sensitivity when results are
    gathered: the owner of its corner 0 (of corner 0's first Eq. 6 parent when
    that corner is hanging).  Every local element's dc is exact on every rank
    holding it; this only avoids double counting."""
    d = host.dim
    nc = 1 << d
    c0 = host.elem_node.reshape(-1, nc)[:, 0].astype(np.int64)
    hang_row = np.full(host.n_node, -1, dtype=np.int64)
    hang_row[host.hang_node] = np.arange(host.hang_node.shape[0])
    h = hang_row[c0]
    node = c0.copy()
    sel = h >= 0
    node[sel] = host.hang_parent[host.hang_ptr[h[sel]]]
    starts = np.array([a for a, _ in ranges])
    return np.searchsorted(starts, node, side="right") - 1


class AmrShardGroup:
    """Every rank of a general-path shard group in one process, on one device
    (tosolve_cg_group drives them in lockstep; the ghost stores are
    device-to-device, the all-reduce the slot / flag protocol)."""

    def __init__(self, host: HostMesh, nranks: int, E0=1.0, Emin=1e-9, nu=0.3, device=0):
        self.host = host
        inc = node_incidence(host)
        self.ranges = partition(host, nranks, inc[0])
        self.slabs = exchange_lists([slice_host(host, nranks, r, self.ranges, inc) for r in range(nranks)])
        self.meshes = [Mesh(sl.host, E0=E0, Emin=Emin, nu=nu, rmin=0.0, device=device, n_owned=sl.n_own)
                       for sl in self.slabs]
        bufs = [m.shard_buffers() for m in self.meshes]
        for r, m in enumerate(self.meshes):
            m.gshard_attach(r, nranks, bufs, *send_entries(self.slabs, r))
        owner = element_owner(host, self.ranges)
        self.elem_owned = [owner[sl.elem_global] == sl.rank for sl in self.slabs]

    def scatter_elems(self, x_global):
        import torch
        return [x_global.index_select(0, torch.as_tensor(sl.elem_global, device=x_global.device))
                for sl in self.slabs]

    def solve(self, penal, xs, us, rtol=1e-10, max_iter=20000, flags=0):
        from . import _lib as L
        from .api import tosolve_cg_group
        return tosolve_cg_group(self.meshes, penal, xs, us, rtol, max_iter, flags | L.TO_NO_TRUE_RES)

    def gather_nodes(self, us):
        d = self.host.dim
        out = np.zeros(self.host.n_dof)
        for sl, u in zip(self.slabs, us):
            un = u.detach().cpu().numpy().reshape(-1, d)
            out.reshape(-1, d)[sl.node_global[:sl.n_own]] = un[:sl.n_own]
        return out

    def gather_elems(self, vs):
        out = np.zeros(self.host.n_el)
        for sl, v, own in zip(self.slabs, vs, self.elem_owned):
            out[sl.elem_global[own]] = v.detach().cpu().numpy()[own]
        return out


class AmrShardRank:
    """One Morton node range per process and GPU (torchrun), the general-path
    counterpart of shard.ShardRank: every rank cuts its own local mesh from
    the global host mesh (the partition is a deterministic function of it),
    the receive lists and the CUDA IPC handles of the CG vectors, Dinv, x and
    the all-reduce slots / flags travel through ``dist.all_gather_object``
    (plumbing), every peer's buffers are mapped (one mapping per IPC handle),
    and tosolve_cg_group drives this rank's handle alone: the exchanges and
    the all-reduce are the device-side peer stores and flags."""

    FIELDS = [("rb", 0), ("rb", 1), ("pb", 0), ("pb", 1), ("qb", 0), ("qb", 1), ("x", None), ("slots", None),
              ("flags", None), ("dinv", None)]

    def __init__(self, host: HostMesh, E0=1.0, Emin=1e-9, nu=0.3, device=0, group=None):
        import torch.distributed as dist
        from . import _lib as L
        single = not (dist.is_available() and dist.is_initialized())
        rank, nranks = (0, 1) if single else (dist.get_rank(group), dist.get_world_size(group))
        inc = node_incidence(host)
        self.ranges = partition(host, nranks, inc[0])
        self.slab = slice_host(host, nranks, rank, self.ranges, inc)
        self.device = device
        self.mesh = Mesh(self.slab.host, E0=E0, Emin=Emin, nu=nu, rmin=0.0, device=device, n_owned=self.slab.n_own)
        mine = self.mesh.shard_buffers()

        def ptr(b, f, i):
            v = getattr(b, f)
            return v[i] if i is not None else v

        exported = {"recv": recv_lists(self.slab),
                    "ipc": [self.mesh.ipc_export(ptr(mine, f, i)) for f, i in self.FIELDS]}
        allx = [None] * nranks
        if single:
            allx[0] = exported
        else:
            dist.all_gather_object(allx, exported, group=group)
        self._opened = []
        opened = {}   # one mapping per IPC handle (small buffers may share an allocation block)

        def open_ptr(h, off):
            if h not in opened:
                opened[h] = ipc_open(device, h, 0)
                self._opened.append(opened[h])
            return opened[h] + off

        peers = []
        for r, ex in enumerate(allx):
            if r == rank:
                peers.append(mine)
                continue
            b = L.ToShardBufs()
            for (f, i), (h, off) in zip(self.FIELDS, ex["ipc"]):
                p = open_ptr(h, off)
                if i is not None:
                    getattr(b, f)[i] = p
                else:
                    setattr(b, f, p)
            peers.append(b)
        self.mesh.gshard_attach(rank, nranks, peers,
                                *send_entries_from([ex["recv"] for ex in allx], rank, self.slab.n0))
        self.elem_owned = element_owner(host, self.ranges)[self.slab.elem_global] == rank
        if not single:
            dist.barrier(group=group)

    def solve(self, penal, x, u, rtol=1e-10, max_iter=20000, flags=0, stream=None):
        from . import _lib as L
        from .api import tosolve_cg_group
        return tosolve_cg_group([self.mesh], penal, [x], [u], rtol, max_iter, flags | L.TO_NO_TRUE_RES,
                                None if stream is None else [stream])[0]

    def close(self):
        for p in self._opened:
            try:
                ipc_close(self.device, p)
            except Exception:
                pass
        self._opened = []
        self.mesh.close()
