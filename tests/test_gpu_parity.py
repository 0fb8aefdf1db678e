"""GPU parity: the CUDA path (through the C ABI) vs the oracle on the same
seeded inputs.  Tolerances: L1 operator outputs 1e-12
relative L2 (fp64 rounding of a few hundred terms), converged u, compliance,
dc and filtered dc 1e-8 relative L2 (north_star), certificate <= 10 rtol."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from inputs import config
from oracle import fe, mesh as omesh, pipeline, topopt
from tests.gpu_helpers import cuda, host, product_input_density, product_mesh, rel
from tests.helpers import cantilever2d, cantilever3d, hanging_load2d, hanging_load3d, refine_some

pytestmark = pytest.mark.gpu

CASES = {
    "c1": lambda: config("c1"),
    "c2": lambda: config("c2"),
    "c3s": lambda: config("c3", nx=16, ny=8, nz=8),
    "c4s": lambda: config("c4", base=(12, 6, 6), L=2, n_gauss=60),
    "c5s": lambda: config("c5", nx=20, ny=10, nz=10),
    "c5s_general": lambda: config("c5", nx=20, ny=10, nz=10),     # uniform H8 forced onto the general path
    "c3s_ragged": lambda: config("c3", nx=37, ny=9, nz=13),       # several CTA tiles + ragged tails in x, y, z
    "c1_launched": lambda: config("c1"),     # one launch per iteration (default for c1: the cluster solver)
    "c1_coop": lambda: config("c1"),         # the whole loop in one cooperative kernel (k_gen_persist)
    "c2_launched": lambda: config("c2"),
    "amr2d": lambda: cantilever2d((5, 3), L=3, leaves=refine_some(2, (5, 3), 3, [(1, 1), (3, 0)]), rmin=0.3),
    "amr3d": lambda: cantilever3d((3, 2, 2), L=2, leaves=refine_some(3, (3, 2, 2), 2, [(1, 1, 0)]), rmin=0.4),
    "hload2d": hanging_load2d,       # loads on hanging nodes (C8): b = Pi_F C^T f, c = f^T u with them
    "hload3d": hanging_load3d,
    # the element-partitioned iteration (TO_UPLOAD_EP, kernels_genep.cuh: each element once,
    # partial sums in per-block slots, Chronopoulos-Gear form of the same PCG)
    "c2_ep": lambda: config("c2"),
    "c4s_ep": lambda: config("c4", base=(12, 6, 6), L=2, n_gauss=60),
    "amr3d_ep": lambda: cantilever3d((3, 2, 2), L=2, leaves=refine_some(3, (3, 2, 2), 2, [(1, 1, 0)]), rmin=0.4),
    "hload3d_ep": hanging_load3d,
}

_cache = {}


def _setup(name):
    if name not in _cache:
        prob = CASES[name]()
        om = omesh.build_mesh(prob)
        import paper_1009_4975_b200 as pb
        opts = (pb.TO_UPLOAD_GENERAL if name.endswith("_general") else 0) | \
               (pb.TO_UPLOAD_LAUNCHED if name.endswith("_launched") else 0) | \
               (pb.TO_UPLOAD_NO_CLUSTER if name.endswith("_coop") else 0) | \
               (pb.TO_UPLOAD_EP if name.endswith("_ep") else 0)
        hm, m = product_mesh(prob, options=opts)
        if name.startswith(("c3s", "c5s")):
            assert m.info()["structured"] == (0 if name.endswith("_general") else 1)
        # which device path runs the loop (include/tomesh.h matvec_variant)
        want = {"c1": 5, "c2": 4, "c1_launched": 4, "c2_launched": 4, "c1_coop": 3, "amr2d": 5, "hload2d": 5,
                "c2_ep": 6, "c4s_ep": 6, "amr3d_ep": 6, "hload3d_ep": 6}
        if name in want:
            assert m.info()["matvec_variant"] == want[name], (name, m.info())
        x_dev = product_input_density(prob, hm, m)
        _cache[name] = (prob, om, hm, m, x_dev)
    return _cache[name]


@pytest.mark.parametrize("name", list(CASES))
def test_L1_operators(name):
    prob, om, hm, m, x_dev = _setup(name)
    x = pipeline.input_density(prob, om)
    assert rel(host(x_dev), x) <= 1e-12                       # includes the c3 DENS pass
    xd = cuda(x)
    K = fe.assemble_K(om, x, prob.penal, prob.E0, prob.Emin, prob.nu)
    A, b, C = fe.projected_system(om, K)
    rng = np.random.default_rng(7)
    v = rng.standard_normal(om.n_dof)
    q = torch.empty(om.n_dof, dtype=torch.float64, device="cuda")
    m.to_apply_A(prob.penal, xd, cuda(v), q)
    assert rel(host(q), A @ v) <= 1e-12
    d = torch.empty_like(q)
    m.to_jacobi_diag(prob.penal, xd, d)
    assert rel(host(d), A.diagonal()) <= 1e-12
    bd = torch.empty_like(q)
    m.to_project_rhs(bd)
    assert rel(host(bd), b) <= 1e-14
    u = torch.empty_like(q)
    m.to_recover(cuda(v), u)
    assert rel(host(u), C @ v) <= 1e-14
    # sensitivities and compliance from an identical u
    uu = C @ v
    dc = torch.empty(om.n_el, dtype=torch.float64, device="cuda")
    c = m.to_sensitivity(prob.penal, xd, cuda(uu), dc, compliance=True)
    dco = topopt.sensitivities(om, x, uu, prob.penal, prob.E0, prob.Emin, prob.nu)
    assert rel(host(dc), dco) <= 1e-12
    assert abs(c - fe.compliance(om.load, uu)) <= 1e-12 * max(1.0, abs(c))
    # filter from identical (x, dc)
    out = torch.empty_like(dc)
    m.to_filter(0, xd, cuda(dco), out)
    assert rel(host(out), topopt.filter_sens(om, prob.rmin, x, dco)) <= 1e-12
    m.to_filter(1, xd, cuda(dco), out)
    assert rel(host(out), topopt.filter_dens(om, prob.rmin, dco)) <= 1e-12


@pytest.mark.parametrize("name", list(CASES))
def test_L2_converged_solve(name):
    prob, om, hm, m, x_dev = _setup(name)
    x = pipeline.input_density(prob, om)
    ref = pipeline.run(prob, rtol=1e-10, m=om, x=x)
    xd = cuda(x)
    u = torch.zeros(om.n_dof, dtype=torch.float64, device="cuda")
    st = m.tosolve_cg(prob.penal, xd, u, rtol=1e-10, max_iter=50000)
    assert st.status == 0 and st.relres <= 1e-10
    ud = host(u)
    assert rel(ud, ref.u) <= 1e-8
    dc = torch.empty(om.n_el, dtype=torch.float64, device="cuda")
    c = m.to_sensitivity(prob.penal, xd, u, dc, compliance=True)
    assert abs(c - ref.compliance) <= 1e-8 * abs(ref.compliance)
    assert rel(host(dc), ref.dc) <= 1e-8
    out = torch.empty_like(dc)
    m.to_filter(0, xd, dc, out)
    assert rel(host(out), ref.dc_filtered) <= 1e-8
    # L3 certificate: the oracle's own A, b judge the device solution
    uhat = ud.copy()
    for k, hn in enumerate(om.hang_node):
        uhat[om.dim * hn:om.dim * hn + om.dim] = 0.0
    cert = np.linalg.norm(ref.b - ref.A @ uhat) / np.linalg.norm(ref.b)
    assert cert <= 10 * 1e-10
    assert abs(st.relres_true - cert) <= 1e-11
    # iteration counts of two correct fp64 PCGs differ by rounding only
    assert abs(st.iters - ref.cg.iters) <= max(5, 0.05 * ref.cg.iters)


@pytest.mark.parametrize("name", ["c1", "c2", "c1_launched", "c1_coop", "c5s", "c4s_ep", "c2_ep"])
def test_warm_start_and_fixed_iterations(name):
    prob, om, hm, m, x_dev = _setup(name)
    u = torch.zeros(om.n_dof, dtype=torch.float64, device="cuda")
    st = m.tosolve_cg(prob.penal, x_dev, u, rtol=1e-10, max_iter=50000)
    st2 = m.tosolve_cg(prob.penal, x_dev, u, rtol=1e-8, max_iter=50000, flags=1)   # TO_WARM
    assert st2.iters <= 1
    u2 = torch.zeros_like(u)
    st3 = m.tosolve_cg(prob.penal, x_dev, u2, rtol=1e-30, max_iter=37, flags=2 | 4)  # FIXED | HISTORY
    assert st3.iters == 37 and st3.status == 0
    h = m.history(100)
    assert h.shape[0] == 37 and np.all(np.isfinite(h))
    # same 37 iterations again: bit-identical (atomic-free operator, reductions in fixed order)
    u3 = torch.zeros_like(u)
    m.tosolve_cg(prob.penal, x_dev, u3, rtol=1e-30, max_iter=37, flags=2)
    assert torch.equal(u2, u3)


def test_zero_load_gives_zero_solution():
    prob = cantilever2d((4, 2))
    prob.loads = []
    hm, m = product_mesh(prob)
    x = cuda(np.full(hm.n_el, 0.5))
    u = torch.full((hm.n_dof,), 3.0, dtype=torch.float64, device="cuda")
    st = m.tosolve_cg(3.0, x, u, rtol=1e-10, max_iter=100)
    assert st.iters == 0 and torch.count_nonzero(u) == 0


@pytest.mark.parametrize("name", ["c2", "c5s", "c4s_ep"])
def test_solver_edge_cases(name):
    """Status codes of include/tomesh.h on both paths: densities outside (0, 1]
    (incl. NaN) -> TO_EINVAL; max_iter = 0 -> no iteration, TO_NOT_CONVERGED, u
    = 0; a too small iteration cap -> TO_NOT_CONVERGED with a usable iterate
    whose recurrence residual matches the true one."""
    import paper_1009_4975_b200 as pb
    from paper_1009_4975_b200._lib import TomeshError
    prob, om, hm, m, x_dev = _setup(name)
    u = torch.zeros(om.n_dof, dtype=torch.float64, device="cuda")
    for bad in (0.0, -0.5, 1.5, float("nan")):
        xb = x_dev.clone()
        xb[om.n_el // 2] = bad
        with pytest.raises(TomeshError) as ei:
            m.tosolve_cg(prob.penal, xb, u, rtol=1e-8, max_iter=100)
        assert ei.value.code == pb.TO_EINVAL
    st = m.tosolve_cg(prob.penal, x_dev, u, rtol=1e-10, max_iter=0)
    assert st.iters == 0 and st.status == pb.TO_NOT_CONVERGED and torch.count_nonzero(u) == 0
    assert abs(st.relres - 1.0) < 1e-12                 # r0 = b
    st = m.tosolve_cg(prob.penal, x_dev, u, rtol=1e-12, max_iter=7)
    assert st.iters == 7 and st.status == pb.TO_NOT_CONVERGED
    assert np.isfinite(host(u)).all()
    assert abs(st.relres_true - st.relres) <= 1e-6 * st.relres


@pytest.mark.parametrize("name", ["c4s", "amr3d", "c1_launched", "c1", "c2"])
def test_upload_is_deterministic(name):
    """Two uploads of the same mesh solve to bit-identical u: nothing at upload
    depends on timing (no timing-based kernel or grid choice), and every
    reduction sums in a fixed order."""
    prob, om, hm, m, x_dev = _setup(name)
    import paper_1009_4975_b200 as pb
    opts = pb.TO_UPLOAD_LAUNCHED if name.endswith("_launched") else 0
    us = []
    for _ in range(2):
        _, m2 = product_mesh(prob, options=opts)
        u = torch.zeros(om.n_dof, dtype=torch.float64, device="cuda")
        m2.tosolve_cg(prob.penal, x_dev, u, rtol=1e-10, max_iter=50000)
        us.append(u)
        m2.close()
    assert torch.equal(us[0], us[1])


def _stop_targets(h, lo=8):
    """An odd and an even iteration k >= lo at which a solve with rtol just
    above h[k-1] stops (every earlier residual, and ||r_0|| = ||b||, clearly
    above it)."""
    out = {}
    for k in range(lo, len(h) + 1):
        if h[k - 1] < 0.99 * min(h[:k - 1].min(), 1.0) and (k & 1) not in out:
            out[k & 1] = k
    assert set(out) == {0, 1}, h
    return [out[1], out[0]]


def test_structured_deferred_x_update():
    """The structured kernel defers x (kernels_cg.cuh cg_x_coef): an odd kernel
    k leaves x alone and kernel k+1 adds alpha_{k-1} p_{k-1} = (alpha_{k-1} /
    beta_{k-1}) (p_k - z_k) to its own term; k_final_s3 adds what is pending
    after N iterations or at a stop.  Against the general path's textbook
    update (x += alpha p in every iteration) on the same mesh: u after every
    fixed count N = 0..12 (both parities) to rounding (1e-11; two fp64 CG runs
    in different summation orders drift apart exponentially on this problem,
    ~1e-13 at 40 iterations and ~1e-4 at 97, whatever the parity).  Solves that
    stop at an odd and at an even iteration k, unsharded and as a 2-slab
    group: ||b - A u|| / ||b|| of the returned u (the operator applied by the
    library to u) equals the recurrence residual the solve reports (a missing
    alpha p term changes it at O(1e-1))."""
    import paper_1009_4975_b200 as pb
    from paper_1009_4975_b200 import shard
    prob, om, hm, m, x_dev = _setup("c5s")
    _, _, _, mg, _ = _setup("c5s_general")
    n = om.n_dof
    fixed = pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES
    for N in range(13):
        us = torch.zeros(n, dtype=torch.float64, device="cuda")
        ug = torch.zeros_like(us)
        m.tosolve_cg(prob.penal, x_dev, us, rtol=0.0, max_iter=N, flags=fixed)
        mg.tosolve_cg(prob.penal, x_dev, ug, rtol=0.0, max_iter=N, flags=fixed)
        if N == 0:
            assert torch.count_nonzero(us) == 0 and torch.count_nonzero(ug) == 0
        else:
            assert rel(host(us), host(ug)) <= 1e-11, N
    b = torch.empty(n, dtype=torch.float64, device="cuda")
    m.to_project_rhs(b)
    q = torch.empty_like(b)

    def true_res(u):
        m.to_apply_A(prob.penal, x_dev, u, q)
        return float(torch.linalg.norm(b - q) / torch.linalg.norm(b))

    u = torch.zeros(n, dtype=torch.float64, device="cuda")
    m.tosolve_cg(prob.penal, x_dev, u, rtol=0.0, max_iter=400, flags=pb.TO_FIXED_ITERS | pb.TO_HISTORY)
    h = m.history(400)     # ||r_k|| / ||b|| is not monotone: the first new minima below 1 come late
    ks = _stop_targets(h)
    g = shard.ShardGroup(hm, 2, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
    xs = g.scatter_elems(x_dev)
    for k in ks:
        rtol = float(h[k - 1]) * (1 + 1e-6)   # stops at k: h[j-1] > rtol for every j < k
        us = torch.zeros(n, dtype=torch.float64, device="cuda")
        st = m.tosolve_cg(prob.penal, x_dev, us, rtol=rtol, max_iter=1000)
        assert st.iters == k and st.status == 0
        assert abs(st.relres_true - st.relres) <= 1e-8 * st.relres
        assert abs(true_res(us) - st.relres) <= 1e-8 * st.relres
        uss = [torch.zeros(mm.n_dof, dtype=torch.float64, device="cuda") for mm in g.meshes]
        sts = g.solve(prob.penal, xs, uss, rtol=rtol, max_iter=1000)
        assert all(s.iters == k and s.status == 0 for s in sts), (k, [s.iters for s in sts])
        ug = cuda(g.gather_nodes(uss))
        assert abs(true_res(ug) - sts[0].relres) <= 1e-8 * sts[0].relres, k


@pytest.mark.parametrize("name", ["c4s", "amr3d", "c2_launched", "c5s_general", "c4s_ep"])
def test_general_block_decomposition(name):
    """The owner-computes decomposition the general kernel runs on
    (to_mesh_info.gen_*): every element is staged by at least one block and
    every unconstrained node is owned by exactly one (local slots >= nodes),
    and the kernel's shared memory fits two CTAs per SM (the block builder
    splits blocks until it does)."""
    prob, om, hm, m, x_dev = _setup(name)
    info = m.info()
    assert info["structured"] == 0
    assert info["gen_blocks"] >= 1
    assert info["gen_local_el"] >= info["n_elem"]
    assert info["gen_local_nodes"] >= info["n_node"] - info["n_hang"]
    assert 0 < info["gen_smem_bytes"] <= 113664
    assert info["gen_max_el"] <= 2047 and info["gen_max_loc"] <= 1536


@pytest.mark.parametrize("name", ["c4s_ep", "amr3d_ep", "c2_ep"])
def test_element_partitioned_matches_default_path(name):
    """The element-partitioned iteration equals the default general path
    iterate by iterate up to rounding (Chronopoulos-Gear and Hestenes-Stiefel
    PCG coincide in exact arithmetic): u after 25 fixed iterations at 1e-9,
    the converged u at 1e-9 with iteration counts within 2."""
    import paper_1009_4975_b200 as pb
    prob, om, hm, m, x_dev = _setup(name)
    _, m0 = product_mesh(prob, options=pb.TO_UPLOAD_LAUNCHED | pb.TO_UPLOAD_NO_EP)
    assert m0.info()["matvec_variant"] == 4
    for rtol, n, flags in ((0.0, 25, pb.TO_FIXED_ITERS), (1e-10, 50000, 0)):
        ua = torch.zeros(om.n_dof, dtype=torch.float64, device="cuda")
        ub = torch.zeros_like(ua)
        sa = m.tosolve_cg(prob.penal, x_dev, ua, rtol=rtol, max_iter=n, flags=flags)
        sb = m0.tosolve_cg(prob.penal, x_dev, ub, rtol=rtol, max_iter=n, flags=flags)
        assert rel(host(ua), host(ub)) <= 1e-9
        assert abs(sa.iters - sb.iters) <= 2
    m0.close()
