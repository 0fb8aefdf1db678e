"""GPU parity of the dynamic AMR strategy (§4 :360-492): the device
marking (to_amr_mark) against oracle/amr.py bit-exactly, and the whole Fig. 1
loop with adaptation (paper_1009_4975_b200.amr.optimize_amr: device steps,
device marks, C++ mesh update) against oracle.amr.optimize_amr.

Tolerances: marks are integers (bit-exact).  The loop compares meshes
exactly (element counts, adaptation steps, final leaf set) and floating-point
trajectories at 1e-8 relative (converged PCG to 1e-12 vs the oracle's direct
solve, compounded over the steps, as in test_gpu_oc.py)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1009_4975_b200 as pb
from inputs import config, uniform_leaves
from oracle import amr, mesh as omesh
from tests.gpu_helpers import cuda, host, product_mesh
from tests.helpers import cantilever2d, cantilever3d, refine_some

pytestmark = pytest.mark.gpu

CASES = {
    "amr2d": lambda: cantilever2d((6, 3), L=3, leaves=refine_some(2, (6, 3), 3, [(1, 1), (4, 0)]), rmin=0.9),
    "amr3d": lambda: cantilever3d((3, 2, 2), L=2, leaves=refine_some(3, (3, 2, 2), 2, [(1, 1, 0)]), rmin=0.7),
    "c2": lambda: config("c2"),
    "uniform3d_s": lambda: cantilever3d((6, 4, 4), L=2, leaves=uniform_leaves(3, (6, 4, 4), 2, 1), rmin=0.8),
    "no_filter": lambda: cantilever2d((6, 3), L=2, leaves=refine_some(2, (6, 3), 2, [(2, 1)]), rmin=0.0),
}


@pytest.mark.parametrize("name", list(CASES))
def test_amr_mark_parity(name):
    prob = CASES[name]()
    om = omesh.build_mesh(prob, density=False)
    hm, m = product_mesh(prob)
    if name == "uniform3d_s":
        assert m.info()["structured"] == 1
    rng = np.random.default_rng(3)
    marks = torch.empty(om.n_el, dtype=torch.int8, device="cuda")
    for trial in range(3):
        x = rng.uniform(1e-3, 1.0, om.n_el) ** (1 + trial)
        for rho_s in (0.5, 0.3):
            m.to_amr_mark(cuda(x), marks, rho_s)
            want = amr.mark(om, x, rho_s, prob.rmin)
            assert np.array_equal(marks.cpu().numpy(), want)
    with pytest.raises(pb.TomeshError):
        m.to_amr_mark(cuda(x), marks, 0.0)


@pytest.mark.parametrize("dim", [2, 3])
def test_dynamic_amr_loop_parity(dim):
    if dim == 2:
        prob = cantilever2d((8, 4), L=2, leaves=uniform_leaves(2, (8, 4), 2, 0), rmin=0.8)
        steps = 24
    else:
        prob = cantilever3d((4, 2, 2), L=1, leaves=uniform_leaves(3, (4, 2, 2), 1, 0), rmin=0.8)
        steps = 14
    om, xo, H = amr.optimize_amr(prob, 0.5, steps, stage_steps=8)
    run = pb.amr.optimize_amr(prob, 0.5, steps, stage_steps=8, rtol=1e-12)
    assert len(run.steps) == steps
    assert [s["n_elem"] for s in run.steps] == H.n_elem
    assert [s["adapted"] for s in run.steps] == H.adapted
    assert any(H.adapted)
    assert [s["penal"] for s in run.steps] == H.penal
    np.testing.assert_allclose([s["compliance"] for s in run.steps], H.compliance, rtol=1e-8)
    np.testing.assert_allclose([s["volume"] for s in run.steps], H.volume, rtol=0, atol=1e-11)
    assert np.array_equal(run.host.elem_level, om.elem_level) and np.array_equal(run.host.elem_anchor,
                                                                                  om.elem_anchor)
    np.testing.assert_allclose(host(run.x), xo, rtol=1e-8, atol=1e-12)


def test_static_refine_only_and_stop_on_converge():
    """The refine-only baseline never derefines and only adds levels; with
    stop_on_converge the dynamic run ends converged at p_max (or at the cap)."""
    prob = cantilever2d((8, 4), L=2, leaves=uniform_leaves(2, (8, 4), 2, 0), rmin=1.2)
    run = pb.amr.optimize_amr(prob, 0.5, 120, mode="static", level_steps=30, rtol=1e-10)
    assert run.adaptations and all(a["n_groups"] == 0 for a in run.adaptations)
    counts = [a["n_elem_after"] for a in run.adaptations]
    assert all(b >= a for a, b in zip(counts, counts[1:]))
    assert all(abs(s["volume"] - 0.5) <= 1e-10 for s in run.steps)
    run = pb.amr.optimize_amr(prob, 0.5, 300, stop_on_converge=True, change_tol=0.02, rtol=1e-10)
    last = run.steps[-1]
    assert len(run.steps) == 300 or (last["penal"] == 3.0 and last["change"] < 0.02)
    with pytest.raises(ValueError):
        pb.amr.optimize_amr(prob, 0.5, 5, mode="bogus")
    with pytest.raises(ValueError):
        pb.amr.optimize_amr(prob, 0.5, 5, stop_rule="bogus")
    # reading R25: stop once the design re-converges within min_steps of a
    # converged adaptation (never later than the mesh rule on the same run)
    run2 = pb.amr.optimize_amr(prob, 0.5, 300, stop_on_converge=True, change_tol=0.02, rtol=1e-10,
                               stop_rule="design")
    last = run2.steps[-1]
    assert len(run2.steps) == 300 or (last["penal"] == 3.0 and last["change"] < 0.02)
    assert len(run2.steps) <= len(run.steps)
    # the two rules see the same (deterministic) trajectory until the design rule stops
    assert [t["compliance"] for t in run2.steps] == [t["compliance"] for t in run.steps[:len(run2.steps)]]
