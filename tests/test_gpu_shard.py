"""GPU parity of the z-slab sharded structured path (include/tomesh.h
to_shard_* / tosolve_cg_group) against the oracle.

All slabs of a group live on the one GPU of the test box and are driven in
lockstep by tosolve_cg_group (every kernel runs to completion before the
next one starts on the stream, so no rank ever waits on a kernel that is not
running); the ghost exchange and the all-reduce go through exactly the
device code a multi-GPU group uses (peer-pointer stores, slot pushes, flags).

Tolerances as tests/test_gpu_parity.py (north_star): converged u, the
compliance, dc and the filtered dc at 1e-8 relative L2; every rank of a group
reports the same iteration count and residual (identical scalars by
construction).  The summation order of the dots differs from the unsharded
solve, so iterates are compared at convergence only."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1009_4975_b200 as pb
from paper_1009_4975_b200 import shard
from inputs import config
from oracle import mesh as omesh, pipeline
from tests.gpu_helpers import cuda, host, rel

pytestmark = pytest.mark.gpu

CASES = {
    "c5s": lambda: config("c5", nx=20, ny=10, nz=10),
    "c3s": lambda: config("c3", nx=16, ny=8, nz=8),
    "c3s_ragged": lambda: config("c3", nx=37, ny=9, nz=13),
}
_cache = {}


def _ref(name):
    if name not in _cache:
        prob = CASES[name]()
        om = omesh.build_mesh(prob)
        x = pipeline.input_density(prob, om)
        ref = pipeline.run(prob, rtol=1e-10, m=om, x=x)
        _cache[name] = (prob, om, x, ref, pb.prepare(prob))
    return _cache[name]


@pytest.mark.parametrize("name,nranks", [("c5s", 1), ("c5s", 2), ("c5s", 3), ("c5s", 5), ("c3s", 2),
                                         ("c3s_ragged", 4)])
def test_sharded_solve_matches_oracle(name, nranks):
    prob, om, x, ref, hm = _ref(name)
    g = shard.ShardGroup(hm, nranks, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
    xs = g.scatter_elems(cuda(x))
    us = [torch.zeros(m.n_dof, dtype=torch.float64, device="cuda") for m in g.meshes]
    sts = g.solve(prob.penal, xs, us, rtol=1e-10, max_iter=50000)
    assert len({(s.iters, s.relres) for s in sts}) == 1          # one decision on every rank
    assert sts[0].status == 0 and sts[0].relres <= 1e-10
    assert abs(sts[0].iters - ref.cg.iters) <= max(5, 0.05 * ref.cg.iters)
    assert abs(sts[0].bnorm - np.linalg.norm(ref.b)) <= 1e-12 * np.linalg.norm(ref.b)
    u = g.gather_nodes(us)
    assert rel(u, ref.u) <= 1e-8
    # the ghost planes the sensitivities and filter of the owned elements need
    # (global planes a-1, b, b+1) hold the neighbours' values
    for sl, ul in zip(g.slabs, us):
        z = hm.node_coord[sl.node_global, 2]
        need = (z >= sl.a - 1) & (z <= sl.b + 1)
        assert rel(host(ul).reshape(-1, 3)[need], ref.u.reshape(-1, 3)[sl.node_global[need]]) <= 1e-8
    dcs, dfs, c = [], [], 0.0
    for m, xl, ul in zip(g.meshes, xs, us):
        dc = torch.empty(m.n_el, dtype=torch.float64, device="cuda")
        c += m.to_sensitivity(prob.penal, xl, ul, dc, compliance=True)
        out = torch.empty_like(dc)
        m.to_filter(pb.TO_FILTER_SENS, xl, dc, out)
        dcs.append(dc)
        dfs.append(out)
    assert abs(c - ref.compliance) <= 1e-8 * abs(ref.compliance)
    assert rel(g.gather_elems(dcs), ref.dc) <= 1e-8
    assert rel(g.gather_elems(dfs), ref.dc_filtered) <= 1e-8


def test_sharded_fixed_iterations_and_repeat():
    """TO_FIXED_ITERS: exactly N iterations on every rank; a second solve on
    the same group (sequence numbers continue) reproduces the first bit for
    bit (deterministic reductions); the iterate is close to the unsharded
    one after the same N iterations."""
    prob, om, x, ref, hm = _ref("c5s")
    g = shard.ShardGroup(hm, 3, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
    xs = g.scatter_elems(cuda(x))
    runs = []
    for _ in range(2):
        us = [torch.zeros(m.n_dof, dtype=torch.float64, device="cuda") for m in g.meshes]
        sts = g.solve(prob.penal, xs, us, max_iter=40, flags=pb.TO_FIXED_ITERS)
        assert all(s.iters == 40 and s.status == 0 for s in sts)
        runs.append(g.gather_nodes(us))
    assert np.array_equal(runs[0], runs[1])
    # re-attaching the whole group restarts the sequence numbers (flags cleared)
    bufs = [m.shard_buffers() for m in g.meshes]
    for sl, m in zip(g.slabs, g.meshes):
        m.shard_attach(sl.rank, 3, [t.gz_lo for t in g.slabs], sl.own_lo, sl.own_hi, bufs)
    us = [torch.zeros(m.n_dof, dtype=torch.float64, device="cuda") for m in g.meshes]
    g.solve(prob.penal, xs, us, max_iter=40, flags=pb.TO_FIXED_ITERS)
    assert np.array_equal(g.gather_nodes(us), runs[0])
    m1 = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
    u1 = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
    m1.tosolve_cg(prob.penal, cuda(x), u1, max_iter=40, flags=pb.TO_FIXED_ITERS)
    assert rel(runs[0], host(u1)) <= 1e-6
    # zero iterations: u = 0
    us = [torch.ones(m.n_dof, dtype=torch.float64, device="cuda") for m in g.meshes]
    sts = g.solve(prob.penal, xs, us, max_iter=0, flags=pb.TO_FIXED_ITERS)
    assert all(s.iters == 0 for s in sts) and all(float(u.abs().max()) == 0.0 for u in us)


def test_sharded_errors():
    prob, om, x, ref, hm = _ref("c5s")
    g = shard.ShardGroup(hm, 2, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
    xs = g.scatter_elems(cuda(x))
    us = [torch.zeros(m.n_dof, dtype=torch.float64, device="cuda") for m in g.meshes]
    with pytest.raises(pb.TomeshError):                                  # warm start unsupported
        g.solve(prob.penal, xs, us, flags=pb.TO_WARM)
    bufs = [m.shard_buffers() for m in g.meshes]
    sl = g.slabs[1]
    with pytest.raises(pb.TomeshError):                                  # one owned plane
        g.meshes[1].shard_attach(1, 2, [s.gz_lo for s in g.slabs], sl.own_lo, sl.own_lo + 1, bufs)
    with pytest.raises(pb.TomeshError):                                  # no ghost planes below
        g.meshes[1].shard_attach(1, 2, [s.gz_lo for s in g.slabs], 0, sl.own_hi, bufs)
    with pytest.raises(pb.TomeshError):                                  # peers[rank] is another handle
        g.meshes[1].shard_attach(1, 2, [s.gz_lo for s in g.slabs], sl.own_lo, sl.own_hi, bufs[::-1])
    lone = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
    with pytest.raises(pb.TomeshError):                                  # not attached
        pb.api.tosolve_cg_group([lone], prob.penal, [cuda(x)], [torch.zeros(hm.n_dof, dtype=torch.float64,
                                                                              device="cuda")])
    amr = pb.prepare(config("c4", base=(12, 6, 6), L=2, n_gauss=60))
    with pytest.raises(ValueError):                                      # not a uniform box
        shard.ShardGroup(amr, 2)
    # an invalid density on one rank stops every rank with TO_EINVAL
    xs_bad = [t.clone() for t in xs]
    xs_bad[1][3] = 0.0
    with pytest.raises(pb.TomeshError):
        g.solve(prob.penal, xs_bad, us)
    # the group recovers: a valid solve right after
    sts = g.solve(prob.penal, xs, us, rtol=1e-10, max_iter=50000)
    assert sts[0].status == 0 and rel(g.gather_nodes(us), ref.u) <= 1e-8


def test_ipc_export_open_in_another_process():
    """CUDA IPC of the exchange buffers (the one-process-per-GPU form): the
    handle + offset of two addresses inside one buffer reopen in another
    process at the same distance (no kernel runs; nobody waits)."""
    import subprocess
    import sys
    prob, om, x, ref, hm = _ref("c5s")
    m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
    b = m.shard_buffers()
    h1, o1 = m.ipc_export(b.x)
    h2, o2 = m.ipc_export(b.x + 64)
    assert o2 - o1 == 64
    hs, os_ = m.ipc_export(b.slots)
    assert h1 == h2                                                       # one allocation, one handle
    code = ("import sys; import paper_1009_4975_b200 as pb; import torch; torch.cuda.init();"
            "a = pb.api.ipc_open(0, bytes.fromhex(sys.argv[1]), int(sys.argv[2]));"
            "pb.api.ipc_close(0, a - int(sys.argv[2])); print(a % 8)")
    r = subprocess.run([sys.executable, "-c", code, h1.hex(), str(o1)], capture_output=True,
                       text=True, timeout=300, cwd=__import__("os").path.dirname(__import__("os").path.dirname(
                           __import__("os").path.abspath(__file__))))
    assert r.returncode == 0, r.stderr[-2000:]
    assert int(r.stdout.strip().splitlines()[-1]) == 0                     # an aligned double address
    with pytest.raises(pb.TomeshError):                                   # not a buffer of this handle
        m.ipc_export(xs_ptr := torch.zeros(8, dtype=torch.float64, device="cuda").data_ptr())
    assert hs and os_ >= 0 and xs_ptr


def test_sharded_full_size_c5_matches_unsharded():
    """BASELINE.json's full c5 (4.19M elements) as 2 z-slabs against the
    unsharded handle, same 30 fixed PCG iterations, then sensitivities and the
    SENS filter: only the summation order of the dots differs, so u, dc and
    the filtered dc agree to 1e-8 relative (the unsharded c5 path itself is
    checked against the oracle in tests/test_gpu_fullsize.py)."""
    from inputs import density_at
    prob = config("c5")
    hm = pb.prepare(prob)
    x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda")
    m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
    u1 = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
    st1 = m.tosolve_cg(prob.penal, x, u1, max_iter=30, flags=pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES)
    dc1 = torch.empty(hm.n_el, dtype=torch.float64, device="cuda")
    m.to_sensitivity(prob.penal, x, u1, dc1)
    df1 = torch.empty_like(dc1)
    m.to_filter(pb.TO_FILTER_SENS, x, dc1, df1)
    u1h, df1h = host(u1), host(df1)
    m.close()
    del u1, dc1, df1
    torch.cuda.empty_cache()
    g = shard.ShardGroup(hm, 2, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
    xs = g.scatter_elems(x)
    us = [torch.zeros(mm.n_dof, dtype=torch.float64, device="cuda") for mm in g.meshes]
    sts = g.solve(prob.penal, xs, us, max_iter=30, flags=pb.TO_FIXED_ITERS)
    assert all(s.iters == 30 for s in sts) and abs(sts[0].relres - st1.relres) <= 1e-8 * st1.relres
    assert rel(g.gather_nodes(us), u1h) <= 1e-8
    dfs = []
    for mm, xl, ul in zip(g.meshes, xs, us):
        dc = torch.empty(mm.n_el, dtype=torch.float64, device="cuda")
        mm.to_sensitivity(prob.penal, xl, ul, dc)
        out = torch.empty_like(dc)
        mm.to_filter(pb.TO_FILTER_SENS, xl, dc, out)
        dfs.append(out)
    assert rel(g.gather_elems(dfs), df1h) <= 1e-8
