"""GPU parity of the OC design update (to_oc_update, reading R18) and of the
Fig. 1 loop (to_optimize, reading R19) against oracle/oc.py.

Tolerances.  The device evaluates x_e (g_e/lam)^eta as a_e lam^-eta and sums
the volumes in another order, so vol(lam) agrees to a few ulp; the bisection
then takes the oracle's decisions (a flip needs vol(lam) within rounding of
the target, and moves lam by at most the 1e-12 bracket tolerance), so lam and
x_new agree to ~1e-12 relative.  The loop compounds a converged PCG solve
(rtol 1e-12 vs the oracle's direct solve) with that update for a dozen
steps: 1e-8 relative on compliance and x."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1009_4975_b200 as pb
from inputs import config
from oracle import mesh as omesh, oc
from tests.gpu_helpers import cuda, host, product_mesh
from tests.helpers import cantilever2d, cantilever3d, refine_some

pytestmark = pytest.mark.gpu

CASES = {
    "c1": lambda: config("c1"),
    "c3s": lambda: config("c3", nx=16, ny=8, nz=8),               # structured handle (uniform V)
    "amr2d": lambda: cantilever2d((5, 3), L=3, leaves=refine_some(2, (5, 3), 3, [(1, 1), (3, 0)]), rmin=0.3),
    "amr3d": lambda: cantilever3d((3, 2, 2), L=2, leaves=refine_some(3, (3, 2, 2), 2, [(1, 1, 0)]), rmin=0.4),
}
_cache = {}


def _setup(name):
    if name not in _cache:
        prob = CASES[name]()
        om = omesh.build_mesh(prob)
        hm, m = product_mesh(prob)
        _cache[name] = (prob, om, hm, m)
    return _cache[name]


def _instance(rng, V, kind="generic"):
    n = V.shape[0]
    x = rng.uniform(1e-3, 1.0, n)
    dc = -np.exp(rng.uniform(-6, 2, n)) * V
    if kind == "generic":
        dc[rng.random(n) < 0.05] = 0.0
    return x, dc


def _check(om_V, x, dc, volfrac, m, **kw):
    r = oc.oc_update(x, dc, om_V, volfrac, **kw)
    xd, dcd = cuda(x), cuda(dc)
    xn = torch.empty_like(xd)
    st = m.to_oc_update(xd, dcd, volfrac, xn, **kw)
    state = {"active": 0, "inactive": 1, "infeasible": 2}[r.status]
    assert st.state == state
    assert abs(st.lam - r.lam) <= 1e-10 * max(r.lam, 1e-300)
    assert abs(st.steps - r.steps) <= 2
    np.testing.assert_allclose(host(xn), r.x, rtol=1e-11, atol=1e-15)
    assert abs(st.volume - r.volume) <= 1e-12
    assert abs(st.change - r.change) <= 1e-11
    assert np.all(host(xd) == x)                     # inputs untouched
    return st, r, xn


@pytest.mark.parametrize("name", list(CASES))
def test_oc_update_parity(name):
    prob, om, hm, m = _setup(name)
    rng = np.random.default_rng(7)
    V = om.volumes()
    for volfrac in (0.5, 0.3, 0.12):
        x, dc = _instance(rng, V)
        st, r, _ = _check(V, x, dc, volfrac, m)
        if r.status == "active":
            assert abs(st.volume - volfrac) <= 1e-10


@pytest.mark.parametrize("name", ["c1", "amr2d"])
def test_oc_update_variants(name):
    """eta != 1/2 (pow path), another move limit and lower bound, in-place update."""
    prob, om, hm, m = _setup(name)
    rng = np.random.default_rng(11)
    V = om.volumes()
    x, dc = _instance(rng, V)
    _check(V, x, dc, 0.4, m, eta=0.3, move=0.1, rho_o=1e-2)
    _check(V, x, dc, 0.4, m, eta=1.0)
    r = oc.oc_update(x, dc, V, 0.4)
    xd = cuda(x)
    m.to_oc_update(xd, cuda(dc), 0.4, xd)             # x_new aliases x
    np.testing.assert_allclose(host(xd), r.x, rtol=1e-11, atol=1e-15)


@pytest.mark.parametrize("name", ["c1", "c3s", "amr3d"])
def test_oc_update_edge_cases(name):
    prob, om, hm, m = _setup(name)
    rng = np.random.default_rng(5)
    V = om.volumes()
    n = V.shape[0]
    x, dc = _instance(rng, V)
    st, r, _ = _check(V, x, dc, 1.0, m)                          # budget above what the move limit allows
    assert st.state == 1 and st.lam == 0.0
    st, r, xn = _check(V, x, np.zeros(n), 0.5, m)                # dc = 0: all to max(rho_o, x - move)
    np.testing.assert_array_equal(host(xn), np.maximum(1e-3, x - 0.2))
    # move = 0: unchanged (budget a hair above the current volume so that the
    # inactive-limit test vol_0 <= target is not a rounding tie)
    st, r, xn = _check(V, x, dc, float(np.sum(V * x) / V.sum()) + 1e-9, m, move=0.0)
    np.testing.assert_array_equal(host(xn), x)
    st, r, _ = _check(V, np.ones(n), dc, 0.05, m)                # x = 1, lo = 0.8 > budget: infeasible
    assert st.state == 2
    xu = np.full(n, 0.5)                                          # symmetric instance -> uniform volfrac
    st, r, xn = _check(V, xu, -1.3 * V, 0.45, m)
    np.testing.assert_allclose(host(xn), 0.45, rtol=1e-12)
    # errors
    xd, dcd = cuda(x), cuda(dc)
    out = torch.empty_like(xd)
    bad = dc.copy()
    bad[n // 2] = np.nan
    with pytest.raises(pb.TomeshError) as e:
        m.to_oc_update(xd, cuda(bad), 0.5, out)
    assert e.value.code == pb.TO_ENAN
    for kw in ({"volfrac": 0.0}, {"volfrac": 1.5}, {"volfrac": 0.5, "move": -0.1}, {"volfrac": 0.5, "eta": 0.0},
               {"volfrac": 0.5, "rho_o": 0.0}):
        with pytest.raises(pb.TomeshError) as e:
            m.to_oc_update(xd, dcd, x_new=out, **kw)
        assert e.value.code == pb.TO_EINVAL
    with pytest.raises(pb.TomeshError):
        m.to_oc_update(xd, dcd, 0.5, dcd)                          # x_new aliases dc


@pytest.mark.parametrize("name,steps,stage", [("c1", 12, 4), ("amr2d", 10, 3), ("c3s", 8, 3), ("amr3d", 8, 3)])
def test_optimize_loop_parity(name, steps, stage):
    """to_optimize vs oracle.optimize: solve (warm-started PCG to 1e-12 vs direct)
    -> sensitivities -> Eq. 5 filter -> OC, with p-continuation."""
    prob, om, hm, m = _setup(name)
    volfrac = 0.4
    x0 = np.full(om.n_el, volfrac)
    xo, H = oc.optimize(om, x0, volfrac, steps, prob.rmin, stage_steps=stage, E0=prob.E0, Emin=prob.Emin,
                        nu=prob.nu)
    xd = cuda(x0)
    u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
    launches0 = m.info()["launches_total"]
    rc, hist = m.to_optimize(xd, u, steps, volfrac, stage_steps=stage, rtol=1e-12)
    assert rc == pb.TO_OK and len(hist) == steps
    assert m.info()["launches_total"] > launches0 + 4 * steps
    np.testing.assert_allclose([h["compliance"] for h in hist], H.compliance, rtol=1e-8)
    assert [h["penal"] for h in hist] == H.penal
    np.testing.assert_allclose([h["volume"] for h in hist], H.volume, rtol=0, atol=1e-11)
    np.testing.assert_allclose([h["change"] for h in hist], H.change, rtol=1e-7, atol=1e-12)
    np.testing.assert_allclose(host(xd), xo, rtol=1e-8, atol=1e-12)
    assert all(h["cg_iters"] > 0 for h in hist)


def test_optimize_stop_on_converge():
    prob, om, hm, m = _setup("c1")
    x0 = np.full(om.n_el, 0.5)
    xo, H = oc.optimize(om, x0, 0.5, 40, prob.rmin, penal0=1.0, penal_max=1.0, stop_on_converge=True,
                        change_tol=0.05, E0=prob.E0, Emin=prob.Emin, nu=prob.nu)
    xd = cuda(x0)
    u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
    rc, hist = m.to_optimize(xd, u, 40, 0.5, penal0=1.0, penal_max=1.0, stop_on_converge=True, change_tol=0.05,
                             rtol=1e-12)
    assert len(hist) == len(H.compliance) < 40
    assert hist[-1]["change"] < 0.05
    np.testing.assert_allclose(host(xd), xo, rtol=1e-8, atol=1e-12)
