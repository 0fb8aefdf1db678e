"""z-slab sharding of the structured path.

The path "shards naturally, with one exchange step per matvec plus scalar
reductions".  Host side, this module:

* ``slab_plan`` cuts the node planes of a uniform H8 box along z into
  contiguous owned ranges [a_r, b_r) (sizes within one plane of each other,
  at least two planes per rank);
* ``slice_host`` builds rank r's local mesh: the element layers
  [a_r - 2, b_r + 1) and node planes [a_r - 2, b_r + 2) clipped to the box,
  with the loads and Dirichlet DOFs sliced from the GLOBAL host mesh (so a
  slab cut never becomes a boundary), plus the index maps local -> global;
* ``ShardGroup`` uploads every slab of one process (all on one device) and
  attaches them to each other (to_shard_attach);
* ``ShardRank`` is the one-process-per-GPU form: each rank uploads its own
  slab and the exchange buffers are shared with CUDA IPC handles exchanged
  through torch.distributed (gloo or nccl; plumbing only).

Everything the solve computes runs in libtomesh (tosolve_cg_group; the
exchange is fused into the iteration kernel, the scalar reductions are
device-side).  This module only partitions index arrays and marshals
pointers.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .api import HostMesh, Mesh, ipc_close, ipc_open, tosolve_cg_group

GHOST = 2   # ghost node planes (and element layers) per interior side


def slab_plan(nz_nodes: int, nranks: int):
    """Owned node-plane ranges [(a, b)], contiguous, covering [0, nz_nodes)."""
    if nranks < 1 or nranks > L.TO_SHARD_MAX:
        raise ValueError(f"nranks must be in [1, {L.TO_SHARD_MAX}]")
    if nz_nodes < 2 * nranks:
        raise ValueError(f"{nz_nodes} node planes cannot give {nranks} ranks two planes each")
    base, extra = divmod(nz_nodes, nranks)
    out, a = [], 0
    for r in range(nranks):
        b = a + base + (1 if r < extra else 0)
        out.append((a, b))
        a = b
    return out


def _box(host: HostMesh):
    if host.dim != 3 or host.hang_node.shape[0] != 0:
        raise ValueError("sharding needs a uniform 3D (H8) box")
    lev = host.elem_level
    if lev.min() != lev.max():
        raise ValueError("sharding needs every element at one level")
    s = 1 << (host.L - int(lev[0]))
    ext = host.elem_anchor.max(axis=0) // s + 1
    if int(np.prod(ext)) != host.n_el:
        raise ValueError("the elements do not tile a box")
    return s, [int(e) for e in ext]


@dataclass
class Slab:
    rank: int
    a: int                      # owned global node planes [a, b)
    b: int
    gz_lo: int                  # global node plane of local plane 0
    own_lo: int                 # owned local planes [own_lo, own_hi)
    own_hi: int
    host: HostMesh              # the local mesh (upload it with Mesh)
    elem_global: np.ndarray     # local element -> global element id
    node_global: np.ndarray     # local node -> global node id
    elem_owned: np.ndarray      # bool per local element: its layer is owned
    node_owned: np.ndarray      # bool per local node: its plane is owned


def slice_host(host: HostMesh, nranks: int, rank: int) -> Slab:
    s, ext = _box(host)
    nz = ext[2] + 1
    a, b = slab_plan(nz, nranks)[rank]
    gz_lo, gz_hi = max(a - GHOST, 0), min(b + GHOST, nz)          # local node planes
    layer = host.elem_anchor[:, 2] // s
    els = np.nonzero((layer >= gz_lo) & (layer < gz_hi - 1))[0]
    en = host.elem_node[els]
    nodes = np.unique(en)
    anchor = host.elem_anchor[els].copy()
    anchor[:, 2] -= gz_lo * s
    coord = host.node_coord[nodes].copy()
    coord[:, 2] -= gz_lo * s
    fx = host.fixed_dof
    fn = fx // 3
    pos = np.searchsorted(nodes, fn)
    keep = (pos < nodes.shape[0]) & (nodes[np.minimum(pos, nodes.shape[0] - 1)] == fn)
    fixed = (pos[keep] * 3 + fx[keep] % 3).astype(np.int64)
    load = host.load.reshape(-1, 3)[nodes].reshape(-1).copy()
    ne = els.shape[0]
    local = HostMesh(
        dim=3, L=host.L, h0=host.h0,
        elem_node=np.searchsorted(nodes, en).astype(np.int32),
        elem_anchor=anchor.astype(np.int32), elem_level=host.elem_level[els].copy(),
        node_coord=coord.astype(np.int32),
        hang_node=np.zeros(0, np.int32), hang_ptr=np.zeros(1, np.int32), hang_parent=np.zeros(0, np.int32),
        hang_weight=np.zeros(0, np.float64), fixed_dof=fixed, load=load,
        # the structured path filters with its lattice stencil: no neighbour lists
        filt_ptr=np.zeros(ne + 1, np.int64) if host.rmin > 0 else None,
        filt_idx=np.zeros(0, np.int32) if host.rmin > 0 else None,
        rmin=host.rmin)
    el_layer = layer[els]
    return Slab(rank=rank, a=a, b=b, gz_lo=gz_lo, own_lo=a - gz_lo, own_hi=b - gz_lo, host=local,
                elem_global=els.astype(np.int64), node_global=nodes.astype(np.int64),
                elem_owned=(el_layer >= a) & (el_layer < min(b, ext[2])),
                node_owned=(host.node_coord[nodes, 2] // s >= a) & (host.node_coord[nodes, 2] // s < b))


def check_filter_reach(host: HostMesh):
    """The ghost layers cover filter neighbourhoods of one element layer."""
    s, _ = _box(host)
    h = host.h0 / (1 << host.L) * s
    if host.rmin > 2.0 * h + 1e-12:
        raise ValueError("sharded filter supports rmin <= 2 element edges (one ghost layer of reach)")


class ShardGroup:
    """All slabs of a box in one process, on one device (tosolve_cg_group
    drives them in lockstep; the ghost exchange is a device-to-device store,
    the all-reduce the same slot/flag protocol as across GPUs)."""

    def __init__(self, host: HostMesh, nranks: int, E0=1.0, Emin=1e-9, nu=0.3, rmin=None, device=0):
        check_filter_reach(host)
        self.host = host
        self.slabs = [slice_host(host, nranks, r) for r in range(nranks)]
        self.meshes = [Mesh(sl.host, E0=E0, Emin=Emin, nu=nu, rmin=rmin, device=device) for sl in self.slabs]
        for m in self.meshes:
            if not m.info()["structured"]:
                raise ValueError("a slab did not take the structured path")
        bufs = [m.shard_buffers() for m in self.meshes]
        gz = [sl.gz_lo for sl in self.slabs]
        for sl, m in zip(self.slabs, self.meshes):
            m.shard_attach(sl.rank, nranks, gz, sl.own_lo, sl.own_hi, bufs)

    def scatter_elems(self, x_global):
        """Per-slab copies of a global element array (input marshalling)."""
        import torch
        return [x_global.index_select(0, torch.as_tensor(sl.elem_global, device=x_global.device))
                for sl in self.slabs]

    def solve(self, penal, xs, us, rtol=1e-10, max_iter=20000, flags=0):
        return tosolve_cg_group(self.meshes, penal, xs, us, rtol, max_iter, flags | L.TO_NO_TRUE_RES)

    def gather_nodes(self, us):
        """Global canonical DOF vector from the owned nodes of every slab (host)."""
        out = np.zeros(self.host.n_dof)
        for sl, u in zip(self.slabs, us):
            un = u.detach().cpu().numpy().reshape(-1, 3)
            out.reshape(-1, 3)[sl.node_global[sl.node_owned]] = un[sl.node_owned]
        return out

    def gather_elems(self, vs):
        out = np.zeros(self.host.n_el)
        for sl, v in zip(self.slabs, vs):
            out[sl.elem_global[sl.elem_owned]] = v.detach().cpu().numpy()[sl.elem_owned]
        return out


class ShardRank:
    """One slab per process and GPU (torchrun): the exchange buffers of the
    neighbours and every rank's all-reduce slots are mapped with CUDA IPC;
    the handles travel through ``dist.all_gather_object`` (plumbing)."""

    def __init__(self, host: HostMesh = None, E0=1.0, Emin=1e-9, nu=0.3, rmin=None, device=0, group=None,
                 slab: Slab = None):
        """host: the global mesh (this rank's slab is sliced from it), or
        slab: this rank's slab built by the caller (e.g. a weak-scaling box
        whose global mesh is never formed)."""
        import torch.distributed as dist
        single = not (dist.is_available() and dist.is_initialized())
        rank, nranks = (0, 1) if single else (dist.get_rank(group), dist.get_world_size(group))
        if slab is None:
            check_filter_reach(host)
            slab = slice_host(host, nranks, rank)
        else:
            check_filter_reach(slab.host)
            if slab.rank != rank:
                raise ValueError(f"slab of rank {slab.rank} given to rank {rank}")
        self.slab = slab
        self.mesh = Mesh(self.slab.host, E0=E0, Emin=Emin, nu=nu, rmin=rmin, device=device)
        self.device = device
        mine = self.mesh.shard_buffers()
        fields = [("rb", 0), ("rb", 1), ("pb", 0), ("pb", 1), ("qb", 0), ("qb", 1), ("x", None), ("slots", None),
                  ("flags", None)]

        def ptr(b, f, i):
            v = getattr(b, f)
            return v[i] if i is not None else v

        exported = {"gz_lo": self.slab.gz_lo, "nx": mine.nx, "ny": mine.ny, "nz": mine.nz,
                    "plane": mine.plane_doubles,
                    "ipc": [self.mesh.ipc_export(ptr(mine, f, i)) for f, i in fields]}
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
            b = L.ToShardBufs()
            b.nx, b.ny, b.nz, b.plane_doubles = ex["nx"], ex["ny"], ex["nz"], ex["plane"]
            if r == rank:
                peers.append(mine)
                continue
            need = range(len(fields)) if abs(r - rank) == 1 else (7, 8)   # neighbours: vectors; all: slots
            vals = {}
            for k in need:
                h, off = ex["ipc"][k]
                vals[k] = open_ptr(h, off)
            for k, (f, i) in enumerate(fields):
                p = vals.get(k, 0)
                if f in ("rb", "pb", "qb"):
                    getattr(b, f)[i] = p
                else:
                    setattr(b, f, p if p else None)
            peers.append(b)
        gz = [ex["gz_lo"] for ex in allx]
        self.mesh.shard_attach(rank, nranks, gz, self.slab.own_lo, self.slab.own_hi, peers)
        if not single:
            dist.barrier(group=group)

    def solve(self, penal, x, u, rtol=1e-10, max_iter=20000, flags=0, stream=None):
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
