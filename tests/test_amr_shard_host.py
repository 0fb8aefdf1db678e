"""Morton-range partition of the general (AMR) path (paper_1009_4975_b200/
amr_shard.py): host slicing on CPU, and a gloo world-2 run of
the per-rank slicing and exchange lists.

The decisive check: the owned part of the operator A v = Pi_F C^T K C Pi_F v
(Eq. 8) evaluated from a rank's LOCAL mesh alone (its
elements, ghosts and hanging constraints; a plain numpy element loop in this
test) equals the oracle's global operator (oracle/sample.py apply_full) on the
owned DOFs -- so no contributing element, ghost or hanging parent is missing.
"""
import os
import socket
import sys

import numpy as np
import pytest

import paper_1009_4975_b200 as pb
from paper_1009_4975_b200 import amr_shard
from inputs import config, density_at
from oracle import fe, mesh as omesh, sample
from tests.helpers import cantilever2d, cantilever3d, hanging_load3d, refine_some

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = {
    "amr2d": lambda: cantilever2d((5, 3), L=3, leaves=refine_some(2, (5, 3), 3, [(1, 1), (3, 0)]), rmin=0.3),
    "amr3d": lambda: cantilever3d((3, 2, 2), L=2, leaves=refine_some(3, (3, 2, 2), 2, [(1, 1, 0)]), rmin=0.4),
    "c4s": lambda: config("c4", base=(6, 3, 3), L=2, n_gauss=30),
    "hload3d": hanging_load3d,
}


def local_owned_apply(sl, x_loc, v_glob, penal, E0, Emin, nu):
    """A v on the owned DOFs from the rank's local mesh only (element loop)."""
    h = sl.host
    d, nc = h.dim, 1 << h.dim
    n = h.n_dof
    free = np.ones(n, dtype=bool)
    free[h.fixed_dof] = False
    for c in range(d):
        free[h.hang_node.astype(np.int64) * d + c] = False
    v_raw = v_glob.reshape(-1, d)[sl.node_global].reshape(-1)
    v = v_raw * free
    u = v.copy()
    rows = {int(g): (h.hang_ptr[i], h.hang_ptr[i + 1]) for i, g in enumerate(h.hang_node)}
    for g, (a, b) in rows.items():                           # u = C v (Eq. 6)
        for c in range(d):
            u[d * g + c] = sum(h.hang_weight[k] * v[d * h.hang_parent[k] + c] for k in range(a, b))
    q = np.zeros(n)
    en = h.elem_node.reshape(-1, nc)
    hs = (1 << (h.L - h.elem_level.astype(np.int64))) * h.hL
    E = fe.simp(x_loc, penal, E0, Emin)
    K0s = {}
    for e in range(h.n_el):
        hv = float(hs[e])
        if hv not in K0s:
            K0s[hv] = fe.element_stiffness(d, 1.0, nu, hv)
        dofs = (en[e][:, None] * d + np.arange(d)[None, :]).reshape(-1)
        y = E[e] * (K0s[hv] @ u[dofs])
        for c in range(nc):
            g = int(en[e][c])
            if g in rows:                                        # C^T: to the parents
                a, b = rows[g]
                for k in range(a, b):
                    p = int(h.hang_parent[k])
                    q[d * p:d * p + d] += h.hang_weight[k] * y[d * c:d * c + d]
            else:
                q[d * g:d * g + d] += y[d * c:d * c + d]
    own = sl.n_own * d
    return np.where(free[:own], q[:own], v_raw[:own])     # unit rows on hanging and fixed DOFs


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("nranks", [2, 3])
def test_slices_reproduce_the_global_operator(name, nranks):
    prob = CASES[name]()
    hm = pb.prepare(prob)
    om = omesh.build_mesh(prob, with_filter=False)
    x = density_at(prob, hm.elem_level, hm.elem_anchor)
    v = np.random.default_rng(3).standard_normal(hm.n_dof)
    ref = sample.apply_full(om, x, v, prob.penal, prob.E0, prob.Emin, prob.nu)
    inc = amr_shard.node_incidence(hm)
    ranges = amr_shard.partition(hm, nranks, inc[0])
    assert ranges[0][0] == 0 and ranges[-1][1] == hm.n_node
    assert all(ranges[r][1] == ranges[r + 1][0] for r in range(nranks - 1))
    slabs = amr_shard.exchange_lists([amr_shard.slice_host(hm, nranks, r, ranges, inc) for r in range(nranks)])
    d = hm.dim
    for sl in slabs:
        # local mesh arrays are consistent and every constraint parent is local
        assert sl.host.elem_node.max() < sl.host.n_node and sl.host.hang_parent.max(initial=-1) < sl.host.n_node
        assert np.array_equal(sl.node_global[:sl.n_own], np.arange(sl.n0, sl.n1))
        q = local_owned_apply(sl, x[sl.elem_global], v, prob.penal, prob.E0, prob.Emin, prob.nu)
        np.testing.assert_allclose(q, ref[sl.n0 * d:sl.n1 * d], rtol=1e-12, atol=1e-12 * np.abs(ref).max())
        # the exchange lists pair up: what s receives from r is what r sends to s
        for s, idx in sl.recv.items():
            assert s != sl.rank
            got = sl.node_global[idx]
            assert np.array_equal(got, slabs[s].n0 + slabs[s].send[sl.rank])
            assert np.all((got >= slabs[s].n0) & (got < slabs[s].n1))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import paper_1009_4975_b200 as pb_
    from paper_1009_4975_b200 import amr_shard as ash
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        prob = CASES["c4s"]()
        hm = pb_.prepare(prob)
        sl = ash.slice_host(hm, ws, rank)                     # each rank slices its own part only
        recv = {s: sl.node_global[idx].tolist() for s, idx in sl.recv.items()}
        allr = [None] * ws
        dist.all_gather_object(allr, {"rank": rank, "n0": sl.n0, "n1": sl.n1, "recv": recv})
        # what every other rank receives from me lies in my owned range
        ok = all(all(sl.n0 <= g < sl.n1 for g in a["recv"].get(rank, [])) for a in allr if a["rank"] != rank)
        cover = sorted((a["n0"], a["n1"]) for a in allr)
        ok &= cover[0][0] == 0 and cover[-1][1] == hm.n_node and all(cover[i][1] == cover[i + 1][0]
                                                                      for i in range(ws - 1))
        out.put((rank, bool(ok), sl.n_ghost))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_amr_partition_gloo_world2():
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    res = [q.get(timeout=10) for _ in range(2)]
    assert all(ok for _, ok, _ in res) and all(ng > 0 for _, _, ng in res)


def _rank_worker(rank, ws, port, out):
    """AmrShardRank's host plumbing with the device calls replaced by fakes:
    the receive lists and IPC handles through all_gather_object, every peer
    buffer mapped once per handle at the right offset, and the send entries it
    hands to to_gshard_attach equal to the ones the in-process group builds."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import paper_1009_4975_b200 as pb_
    from paper_1009_4975_b200 import _lib as L
    from paper_1009_4975_b200 import amr_shard as ash
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        base = 1 << 40 | rank << 32            # fake device addresses of this rank
        opened, seen = [], {}
        offs = {("rb", 0): 0x100, ("rb", 1): 0x200, ("pb", 0): 0x300, ("pb", 1): 0x400, ("qb", 0): 0x500,
                ("qb", 1): 0x600, ("x", None): 0x700, ("dinv", None): 0x800, ("slots", None): 0x10000,
                ("flags", None): 0x10100}       # slots + flags share one allocation block

        class FakeMesh:
            def __init__(self, host, **kw):
                self.host, self.kw = host, kw

            def shard_buffers(self):
                b = L.ToShardBufs()
                for (f, i), o in offs.items():
                    if i is None:
                        setattr(b, f, base + o)
                    else:
                        getattr(b, f)[i] = base + o
                return b

            def ipc_export(self, ptr):
                blk = ptr & ~0xFFFF
                return (f"r{rank}-{blk:x}".encode().ljust(64, b"\0"), ptr - blk)

            def gshard_attach(self, r, n, peers, dst, loc, rem):
                seen.update(rank=r, n=n, send=(dst.tolist(), loc.tolist(), rem.tolist()),
                            peers=[{(f, i): ((getattr(p, f)[i] if i is not None else getattr(p, f)) or 0)
                                    for f, i in offs} for p in peers])

            def close(self):
                pass

        def fake_open(device, h, off):
            opened.append(h)
            owner = int(h.split(b"-")[0][1:])
            blk = int(h.rstrip(b"\0").split(b"-")[1], 16)
            assert blk >> 32 == (1 << 8 | owner) and off == 0
            return blk

        ash.Mesh, ash.ipc_open, ash.ipc_close = FakeMesh, fake_open, lambda d, p: None
        hm = pb_.prepare(CASES["c4s"]())
        sr = ash.AmrShardRank(hm)
        ok = seen["rank"] == rank and seen["n"] == ws and sr.mesh.kw["n_owned"] == sr.slab.n_own
        ok &= len(set(opened)) == len(opened) == 2 * (ws - 1)   # one mapping per handle: vectors block, slots block
        for r, p in enumerate(seen["peers"]):
            ok &= all(p[k] == (1 << 40 | r << 32) + o for k, o in offs.items())
        # the same entries as the in-process group's (which slices every rank here)
        slabs = ash.exchange_lists([ash.slice_host(hm, ws, r) for r in range(ws)])
        dst, loc, rem = ash.send_entries(slabs, rank)
        ok &= seen["send"] == (dst.tolist(), loc.tolist(), rem.tolist()) and len(seen["send"][0]) > 0
        ok &= all(0 <= l < sr.slab.n_own for l in seen["send"][1])
        # every element is reported by exactly one rank
        allown = [None] * ws
        dist.all_gather_object(allown, sr.slab.elem_global[sr.elem_owned].tolist())
        flat = sorted(e for a in allown for e in a)
        ok &= flat == list(range(hm.n_el))
        out.put((rank, bool(ok)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_amr_shard_rank_plumbing_gloo_world3():
    pytest.importorskip("torch")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in range(3))
    assert res == {0: True, 1: True, 2: True}
