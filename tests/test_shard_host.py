"""Host logic of the z-slab sharding (paper_1009_4975_b200/shard.py; SURVEY
§8(e)), on CPU: the slab plan, the local meshes sliced from the global host
mesh, the per-rank slicing under torch.distributed (gloo, world size 2), and
the one-process-per-GPU plumbing of ShardRank (IPC handle exchange, which peer
buffers are mapped, the attach arguments) with fake device calls (gloo, world
size 3).  The device side (the fused exchange and the all-reduce) is covered
by tests/test_gpu_shard.py."""
import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import paper_1009_4975_b200 as pb  # noqa: E402
from paper_1009_4975_b200 import shard  # noqa: E402
from inputs import config  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_slab_plan():
    for nz in (4, 11, 14, 129):
        for R in range(1, min(16, nz // 2) + 1):
            plan = shard.slab_plan(nz, R)
            assert plan[0][0] == 0 and plan[-1][1] == nz
            assert all(b0 == a1 for (_, b0), (a1, _) in zip(plan, plan[1:]))
            sizes = [b - a for a, b in plan]
            assert min(sizes) >= 2 and max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.slab_plan(5, 3)
    with pytest.raises(ValueError):
        shard.slab_plan(100, 17)


@pytest.mark.parametrize("name,kw,R", [("c5", dict(nx=20, ny=10, nz=10), 3), ("c3", dict(nx=37, ny=9, nz=13), 4),
                                       ("c5", dict(nx=6, ny=4, nz=7), 4)])
def test_slices_partition_and_match_global(name, kw, R):
    hm = pb.prepare(config(name, **kw))
    s = 1
    slabs = [shard.slice_host(hm, R, r) for r in range(R)]
    own_n = np.concatenate([sl.node_global[sl.node_owned] for sl in slabs])
    own_e = np.concatenate([sl.elem_global[sl.elem_owned] for sl in slabs])
    assert np.array_equal(np.sort(own_n), np.arange(hm.n_node))            # every node owned exactly once
    assert np.array_equal(np.sort(own_e), np.arange(hm.n_el))              # every element owned exactly once
    gfixed = set(hm.fixed_dof.tolist())
    for sl in slabs:
        h = sl.host
        # local box: anchors from 0, element corners at anchor + offsets (C4 corner order)
        assert h.elem_anchor.min(axis=0).tolist() == [0, 0, 0]
        off = np.array([[c & 1, (c >> 1) & 1, c >> 2] for c in range(8)]) * s
        assert np.array_equal(h.node_coord[h.elem_node], h.elem_anchor[:, None, :] + off[None])
        # loads and Dirichlet DOFs are the global ones at the local nodes (a cut is no boundary)
        assert np.array_equal(h.load.reshape(-1, 3), hm.load.reshape(-1, 3)[sl.node_global])
        want = sorted(3 * i + c for i, n in enumerate(sl.node_global) for c in range(3) if 3 * n + c in gfixed)
        assert h.fixed_dof.tolist() == want
        # two ghost planes (and element layers) per interior side, planes relative to gz_lo
        zc = hm.node_coord[sl.node_global, 2]
        assert zc.min() == sl.gz_lo and sl.own_lo == sl.a - sl.gz_lo and sl.own_hi == sl.b - sl.gz_lo
        assert sl.own_lo == (0 if sl.rank == 0 else 2)
        top = hm.node_coord[:, 2].max()
        assert zc.max() == min(sl.b + 1, top)
        # owned elements: layers [a, b) (the last rank up to the top layer)
        ez = hm.elem_anchor[sl.elem_global, 2]
        assert np.array_equal(sl.elem_owned, (ez >= sl.a) & (ez < min(sl.b, top)))


def test_reach_and_box_checks():
    hm = pb.prepare(config("c5", nx=8, ny=4, nz=6))
    hm.rmin = 2.5
    with pytest.raises(ValueError):
        shard.check_filter_reach(hm)
    amr = pb.prepare(config("c4", base=(6, 3, 3), L=1, n_gauss=20))
    if amr.hang_node.shape[0] or amr.elem_level.min() != amr.elem_level.max():
        with pytest.raises(ValueError):
            shard.slice_host(amr, 2, 0)


def _free_port():
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    p = so.getsockname()[1]
    so.close()
    return p


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    sys.path.insert(0, ROOT)
    import paper_1009_4975_b200 as pb_
    from paper_1009_4975_b200 import shard as sh
    from inputs import config as cfg
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        hm = pb_.prepare(cfg("c5", nx=12, ny=6, nz=9))
        sl = sh.slice_host(hm, dist.get_world_size(), dist.get_rank())
        mine = {"nodes": sl.node_global[sl.node_owned].tolist(), "elems": sl.elem_global[sl.elem_owned].tolist(),
                "gz_lo": sl.gz_lo, "own": (sl.own_lo, sl.own_hi), "nz": int(sl.host.node_coord[:, 2].max()) + 1,
                "load": float(sl.host.load.reshape(-1, 3)[sl.node_owned].sum())}
        allx = [None] * ws
        dist.all_gather_object(allx, mine)
        if rank == 0:
            nodes = sorted(n for a in allx for n in a["nodes"])
            elems = sorted(e for a in allx for e in a["elems"])
            ok = nodes == list(range(hm.n_node)) and elems == list(range(hm.n_el))
            ok &= abs(sum(a["load"] for a in allx) - hm.load.sum()) < 1e-12
            # the lower rank's box holds the upper rank's first two owned planes (its ghost planes b, b+1)
            lo, hi = allx
            ok &= lo["gz_lo"] + lo["nz"] >= hi["gz_lo"] + hi["own"][0] + 2
            out.put(bool(ok))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_slices_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


def _rank_worker(rank, ws, port, out):
    """ShardRank's host plumbing with the device calls replaced by fakes: the
    IPC exchange through all_gather_object, which peer buffers each rank maps
    (neighbours' vectors, everyone's slots and flags), one mapping per handle,
    and the arguments it hands to to_shard_attach."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    sys.path.insert(0, ROOT)
    import paper_1009_4975_b200 as pb_
    from paper_1009_4975_b200 import _lib as L
    from paper_1009_4975_b200 import shard as sh
    from inputs import config as cfg
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        base = 1 << 40 | rank << 32            # fake device addresses of this rank
        opened = []
        seen = {}

        class FakeMesh:
            def __init__(self, host, **kw):
                self.host = host

            def shard_buffers(self):
                b = L.ToShardBufs()
                for i in range(2):
                    b.rb[i], b.pb[i], b.qb[i] = base + 0x100 * (1 + i), base + 0x100 * (3 + i), base + 0x100 * (5 + i)
                b.x, b.slots, b.flags = base + 0x700, base + 0x10000, base + 0x10100   # slots+flags: one block
                b.nx, b.ny, b.nz, b.plane_doubles = 13, 7, int(self.host.node_coord[:, 2].max()) + 1, 3 * 14 * 7
                return b

            def ipc_export(self, ptr):
                blk = ptr & ~0xFFFF
                return (f"r{rank}-{blk:x}".encode().ljust(64, b"\0"), ptr - blk)

            def shard_attach(self, r, n, gz, lo, hi, peers):
                seen.update(rank=r, n=n, gz=list(gz), own=(lo, hi),
                            peers=[(p.x or 0, p.rb[0] or 0, p.slots or 0, p.flags or 0) for p in peers])

            def close(self):
                pass

        def fake_open(device, h, off):
            opened.append(h)
            owner = int(h.split(b"-")[0][1:])
            blk = int(h.rstrip(b"\0").split(b"-")[1], 16)
            assert blk >> 32 == (1 << 8 | owner)
            return blk + off

        sh.Mesh, sh.ipc_open, sh.ipc_close = FakeMesh, fake_open, lambda d, p: None
        hm = pb_.prepare(cfg("c5", nx=12, ny=6, nz=11))
        sr = sh.ShardRank(hm)
        ok = seen["rank"] == rank and seen["n"] == ws and seen["own"] == (sr.slab.own_lo, sr.slab.own_hi)
        ok &= len(set(opened)) == len(opened)                   # one mapping per handle
        for r, (x, rb0, slots, flags) in enumerate(seen["peers"]):
            owner = (1 << 40 | r << 32)
            ok &= slots == owner + 0x10000 and flags == owner + 0x10100
            if abs(r - rank) <= 1:
                ok &= x == owner + 0x700 and rb0 == owner + 0x100
            else:
                ok &= x == 0 and rb0 == 0                        # non-neighbours' vectors are never mapped
        allseen = [None] * ws
        dist.all_gather_object(allseen, seen["gz"])
        ok &= all(g == allseen[0] for g in allseen)
        out.put((rank, bool(ok)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_shard_rank_plumbing_gloo_world3():
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


@pytest.mark.parametrize("nranks", [1, 2, 3])
def test_weak_slab_matches_slice_of_global_mesh(nranks):
    """bench.py's weak-scaling slabs, built without the global mesh, equal the
    slabs shard.slice_host cuts from the global c5-recipe box: loads and
    Dirichlet DOFs bit-exact by global node, element and node ownership, and
    densities from the one global lexicographic field."""
    import bench
    from inputs import config
    from paper_1009_4975_b200 import shard
    nx, ny, nz = 8, 4, 4
    glob = pb.prepare(config("c5", nx=nx, ny=ny, nz=nz * nranks))
    gc = glob.node_coord.astype(np.int64)
    gid = gc[:, 0] + (nx + 1) * (gc[:, 1] + (ny + 1) * gc[:, 2])
    gload = dict(zip(gid.tolist(), map(tuple, glob.load.reshape(-1, 3).tolist())))
    gfix = {(int(gid[f // 3]), int(f % 3)) for f in glob.fixed_dof}
    field = np.random.default_rng(5).uniform(0.001, 1.0, nx * ny * nz * nranks)
    for r in range(nranks):
        sl, x, _ = bench.weak_slab(nranks, r, nx=nx, ny=ny, nz=nz)
        ref = shard.slice_host(glob, nranks, r)
        assert (sl.a, sl.b, sl.gz_lo, sl.own_lo, sl.own_hi) == (ref.a, ref.b, ref.gz_lo, ref.own_lo, ref.own_hi)
        assert sl.host.n_el == ref.host.n_el and sl.host.n_node == ref.host.n_node
        loads = sl.host.load.reshape(-1, 3)
        assert all(tuple(loads[i]) == gload[int(g)] for i, g in enumerate(sl.node_global))
        fix = {(int(sl.node_global[f // 3]), int(f % 3)) for f in sl.host.fixed_dof}
        assert fix == {fg for fg in gfix if fg[0] in set(sl.node_global.tolist())}
        assert sl.elem_owned.sum() == ref.elem_owned.sum() and sl.node_owned.sum() == ref.node_owned.sum()
        assert np.array_equal(x, field[sl.elem_global])
