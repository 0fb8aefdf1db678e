"""GPU parity of the sharded general (AMR) path (paper_1009_4975_b200/
amr_shard.py, include/tomesh.h to_gshard_attach / tosolve_cg_group).

All ranks of a group live on the one GPU of the test box and are driven in
lockstep by tosolve_cg_group, with the same ghost stores, slot pushes and
flags a multi-GPU group uses.  Each group solve is compared with the oracle
(SURVEY §8(c) L2): u gathered from the owned nodes, c = the sum of the ranks'
f.u partials, dc gathered from the elements each rank reports, at 1e-8
relative; every rank takes the same iteration count, and a repeat solve is
bit-identical."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1009_4975_b200 as pb  # noqa: E402
from paper_1009_4975_b200 import amr_shard  # noqa: E402
from inputs import config, density_at  # noqa: E402
from oracle import mesh as omesh, pipeline  # noqa: E402
from tests.gpu_helpers import cuda, host, rel  # noqa: E402
from tests.helpers import cantilever2d, cantilever3d, hanging_load3d, refine_some  # noqa: E402

pytestmark = pytest.mark.gpu

CASES = {
    "amr2d": lambda: cantilever2d((5, 3), L=3, leaves=refine_some(2, (5, 3), 3, [(1, 1), (3, 0)]), rmin=0.3),
    "amr3d": lambda: cantilever3d((3, 2, 2), L=2, leaves=refine_some(3, (3, 2, 2), 2, [(1, 1, 0)]), rmin=0.4),
    "c4s": lambda: config("c4", base=(12, 6, 6), L=2, n_gauss=60),
    "hload3d": hanging_load3d,
}


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("nranks", [1, 2, 3])
def test_amr_sharded_solve_matches_oracle(name, nranks):
    prob = CASES[name]()
    hm = pb.prepare(prob)
    om = omesh.build_mesh(prob)
    x = density_at(prob, hm.elem_level, hm.elem_anchor)
    ref = pipeline.run(prob, rtol=1e-10, m=om, x=x)
    g = amr_shard.AmrShardGroup(hm, nranks, E0=prob.E0, Emin=prob.Emin, nu=prob.nu)
    xs = g.scatter_elems(cuda(x))
    us = [torch.zeros(m.n_dof, dtype=torch.float64, device="cuda") for m in g.meshes]
    st = g.solve(prob.penal, xs, us, rtol=1e-10, max_iter=50000)
    assert len({s.iters for s in st}) == 1 and all(s.status == 0 for s in st)
    assert abs(st[0].iters - ref.cg.iters) <= max(5, 0.05 * ref.cg.iters)
    u = g.gather_nodes(us)
    assert rel(u, ref.u) <= 1e-8
    c = 0.0
    dcs = []
    for m, xi, ui in zip(g.meshes, xs, us):
        dc = torch.empty(m.n_el, dtype=torch.float64, device="cuda")
        c += m.to_sensitivity(prob.penal, xi, ui, dc, compliance=True)
        dcs.append(dc)
    assert abs(c - ref.compliance) <= 1e-8 * abs(ref.compliance)
    assert rel(g.gather_elems(dcs), ref.dc) <= 1e-8
    # a repeat solve: bit-identical (fixed summation orders, rank-order all-reduce)
    us2 = [torch.zeros_like(v) for v in us]
    st2 = g.solve(prob.penal, xs, us2, rtol=1e-10, max_iter=50000)
    assert st2[0].iters == st[0].iters and all(torch.equal(a, b) for a, b in zip(us, us2))


def test_amr_sharded_fixed_iterations_and_errors():
    prob = CASES["c4s"]()
    hm = pb.prepare(prob)
    g = amr_shard.AmrShardGroup(hm, 2, E0=prob.E0, Emin=prob.Emin, nu=prob.nu)
    x = density_at(prob, hm.elem_level, hm.elem_anchor)
    xs = g.scatter_elems(cuda(x))
    us = [torch.zeros(m.n_dof, dtype=torch.float64, device="cuda") for m in g.meshes]
    st = g.solve(prob.penal, xs, us, rtol=0.0, max_iter=25, flags=pb.TO_FIXED_ITERS)
    assert all(s.iters == 25 for s in st)
    # the 25-iteration iterate equals the unsharded general path's to rounding
    m1 = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=0.0)
    u1 = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
    m1.tosolve_cg(prob.penal, cuda(x), u1, rtol=0.0, max_iter=25, flags=pb.TO_FIXED_ITERS)
    assert rel(g.gather_nodes(us), host(u1)) <= 1e-10
    # a density outside (0, 1] on one rank stops every rank with TO_EINVAL
    xb = [v.clone() for v in xs]
    xb[1][0] = 0.0
    with pytest.raises(pb.TomeshError) as ei:
        g.solve(prob.penal, xb, us, rtol=1e-8, max_iter=100)
    assert ei.value.code == pb.TO_EINVAL


def test_amr_shard_rank_single_process_form():
    """AmrShardRank (one Morton range per process; here world size 1, no
    process group): the real IPC export of its buffers, the attach with an
    empty send list and the group solve of its one handle equal the oracle."""
    prob = CASES["hload3d"]()
    hm = pb.prepare(prob)
    om = omesh.build_mesh(prob)
    x = density_at(prob, hm.elem_level, hm.elem_anchor)
    ref = pipeline.run(prob, rtol=1e-10, m=om, x=x)
    sr = amr_shard.AmrShardRank(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu)
    try:
        assert sr.slab.n_own == hm.n_node and sr.elem_owned.all()
        xd = cuda(x)[torch.as_tensor(sr.slab.elem_global, device="cuda")]
        u = torch.zeros(sr.mesh.n_dof, dtype=torch.float64, device="cuda")
        st = sr.solve(prob.penal, xd, u, rtol=1e-10, max_iter=50000)
        assert st.status == 0 and abs(st.iters - ref.cg.iters) <= max(5, 0.05 * ref.cg.iters)
        un = np.zeros(hm.n_dof)
        d = hm.dim
        un.reshape(-1, d)[sr.slab.node_global[:sr.slab.n_own]] = host(u).reshape(-1, d)[:sr.slab.n_own]
        assert rel(un, ref.u) <= 1e-8
    finally:
        sr.close()
