"""GPU parity of the paper's solver (tosolve_minres) against
oracle/minres.py on the same seeded problems.

Tolerances: converged solutions (rtol 1e-12 on |eta|) against the oracle's
direct solve 1e-8 relative (north_star's u tolerance); iteration counts of two
correct fp64 MINRES runs differ by rounding only (within 5%); |eta| is the
M^-1-norm of the residual, so the reported eta_rel bounds the true residual
through the condition of the rescaled system."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

torch = pytest.importorskip("torch")

import paper_1009_4975_b200 as pb
from inputs import config
from oracle import fe, mesh as omesh, minres as om, pipeline
from tests.gpu_helpers import cuda, host, product_mesh, rel
from tests.helpers import cantilever2d, cantilever3d, refine_some

pytestmark = pytest.mark.gpu

CASES = {
    "c1": lambda: config("c1"),
    "c2": lambda: config("c2"),
    "c3s": lambda: config("c3", nx=16, ny=8, nz=8),
    "amr2d": lambda: cantilever2d((5, 3), L=3, leaves=refine_some(2, (5, 3), 3, [(1, 1), (3, 0)]), rmin=0.3),
    "amr3d": lambda: cantilever3d((3, 2, 2), L=2, leaves=refine_some(3, (3, 2, 2), 2, [(1, 1, 0)]), rmin=0.4),
}
_cache = {}


def _setup(name):
    if name not in _cache:
        prob = CASES[name]()
        om_ = omesh.build_mesh(prob)
        hm, m = product_mesh(prob)
        x = pipeline.input_density(prob, om_)
        K = fe.assemble_K(om_, x, prob.penal, prob.E0, prob.Emin, prob.nu)
        A, b, C = fe.projected_system(om_, K)
        _cache[name] = (prob, om_, hm, m, x, A, b, C)
    return _cache[name]


@pytest.mark.parametrize("name", list(CASES))
def test_minres_jacobi_parity(name):
    prob, om_, hm, m, x, A, b, C = _setup(name)
    u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
    st = m.tosolve_minres(prob.penal, cuda(x), u, rtol=1e-12, max_iter=50000, precond=pb.TO_PC_JACOBI)
    assert st["status"] == 0 and st["eta_rel"] <= 1e-12
    ud = fe.recover(C, spla.spsolve(A.tocsc(), b))
    assert rel(host(u), ud) <= 1e-8
    _, r = om.solve_paper(A, b, rtol=1e-12, precond="none")
    assert abs(st["iters"] - r.iters) <= max(3, 0.05 * r.iters)
    assert st["relres_true"] <= 1e-8


def test_minres_edge_cases():
    prob, om_, hm, m, x, A, b, C = _setup("c1")
    u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
    st = m.tosolve_minres(prob.penal, cuda(x), u, rtol=1e-12, max_iter=5)
    assert st["status"] == pb.TO_NOT_CONVERGED and st["iters"] == 5
    _, r = om.solve_paper(A, b, rtol=0.0, max_iter=5, precond="none")
    assert abs(st["eta_rel"] - r.eta[-1] / r.eta[0]) <= 1e-9
    st = m.tosolve_minres(prob.penal, cuda(x), u, rtol=1e-12, max_iter=0)
    assert st["iters"] == 0 and np.all(host(u) == 0)
    for bad in ({"precond": 7}, {"flags": pb.TO_WARM}, {"rtol": -1.0}):
        with pytest.raises(pb.TomeshError):
            m.tosolve_minres(prob.penal, cuda(x), u, **bad)
    xb = x.copy()
    xb[3] = 0.0
    with pytest.raises(pb.TomeshError):
        m.tosolve_minres(prob.penal, cuda(xb), u)


@pytest.mark.parametrize("name", ["c1", "c2", "amr2d", "amr3d"])
def test_minres_ic0_parity(name):
    """MINRES + IC(0) of the rescaled matrix: the same shift as the oracle's,
    iteration counts within rounding, solution at the direct solve's."""
    prob, om_, hm, m, x, A, b, C = _setup(name)
    u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
    st = m.tosolve_minres(prob.penal, cuda(x), u, rtol=1e-12, max_iter=20000, precond=pb.TO_PC_IC0)
    _, r = om.solve_paper(A, b, rtol=1e-12, precond="ic0")
    assert st["status"] == 0 and st["ic0_shift"] == r.shift
    assert min(st["ic0_levels"]) >= 1
    assert abs(st["iters"] - r.iters) <= max(3, 0.05 * r.iters)
    ud = fe.recover(C, spla.spsolve(A.tocsc(), b))
    assert rel(host(u), ud) <= 1e-8
    # fewer iterations than the rescaling alone (the point of the preconditioner)
    st_j = m.tosolve_minres(prob.penal, cuda(x), u, rtol=1e-12, max_iter=50000, precond=pb.TO_PC_JACOBI)
    assert st["iters"] < st_j["iters"]


def test_minres_ic0_structured_rejected():
    prob, om_, hm, m, x, A, b, C = _setup("c3s")
    u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
    with pytest.raises(pb.TomeshError) as e:
        m.tosolve_minres(prob.penal, cuda(x), u, precond=pb.TO_PC_IC0)
    assert e.value.code == pb.TO_EINVAL
