"""Pins for oracle/oc.py (OC update, reading R18; Fig. 1 loop).

Each pin checks the oracle against something other than its own formula:
the closed-form multiplier when no bound is active, symmetry, the move = 0
and dc = 0 special cases, a brute-force lambda grid, and the KKT conditions
of the convex p = 1 problem reached by the loop.
"""
import numpy as np
import pytest

from oracle import fe, mesh as omesh, oc, topopt
from tests.helpers import cantilever2d, refine_some


def _rand_instance(rng, n, spread=0.1):
    x = rng.uniform(0.3, 0.6, n)
    V = rng.choice([1.0, 0.25, 0.0625], n)
    lam0 = 2.5
    dc = -lam0 * V * (1.0 + rng.uniform(-spread, spread, n))
    return x, dc, V, lam0


def test_closed_form_multiplier(rng):
    """No bound active: x_new = x (-dc/(lam V))^eta, so sum V x_new = target
    gives lam = (sum V x (-dc/V)^eta / target)^(1/eta) in closed form."""
    x, dc, V, _ = _rand_instance(rng, 50)
    for eta in (0.5, 0.3, 1.0):
        lam_true = 2.8
        xn_true = x * (-dc / (lam_true * V)) ** eta
        assert np.all(np.abs(xn_true - x) < oc.MOVE) and np.all(xn_true < 1.0)
        volfrac = np.sum(V * xn_true) / V.sum()
        r = oc.oc_update(x, dc, V, volfrac, eta=eta)
        lam_cf = (np.sum(V * x * (-dc / V) ** eta) / (volfrac * V.sum())) ** (1.0 / eta)
        assert r.status == "active"
        assert abs(lam_cf - lam_true) <= 1e-13 * lam_true
        assert abs(r.lam - lam_cf) <= 1e-11 * lam_cf
        np.testing.assert_allclose(r.x, xn_true, rtol=1e-11, atol=0)
        assert abs(r.volume - volfrac) <= 1e-11


def test_uniform_symmetry():
    """Identical sensitivities and volumes, uniform start -> uniform x = V0."""
    n = 40
    for x0 in (0.5, 0.35, 0.6):
        r = oc.oc_update(np.full(n, x0), np.full(n, -1.7), np.ones(n), 0.5)
        np.testing.assert_allclose(r.x, 0.5, rtol=1e-11)
        assert r.change == pytest.approx(abs(0.5 - x0), abs=1e-11)


def test_move_zero_keeps_x(rng):
    x, dc, V, _ = _rand_instance(rng, 30, spread=0.8)
    volfrac = np.sum(V * x) / V.sum()
    r = oc.oc_update(x, dc, V, volfrac, move=0.0)
    np.testing.assert_array_equal(r.x, x)
    assert r.change == 0.0


def test_zero_sensitivity_goes_to_lower_bound(rng):
    """dc = 0: B = 0, every element goes to max(rho_o, x - move); volume falls, constraint inactive."""
    x = rng.uniform(0.0011, 1.0, 25)
    r = oc.oc_update(x, np.zeros_like(x), np.ones_like(x), 0.5)
    assert r.status == "inactive" and r.lam == 0.0
    np.testing.assert_array_equal(r.x, np.maximum(1e-3, x - 0.2))


def test_inactive_constraint_moves_up(rng):
    """A volume budget above what the move limit allows: every loaded element takes hi."""
    x = rng.uniform(0.1, 0.3, 25)
    r = oc.oc_update(x, -rng.uniform(0.1, 1.0, 25), np.ones(25), 0.9)
    assert r.status == "inactive"
    np.testing.assert_allclose(r.x, np.minimum(1.0, x + 0.2), rtol=0, atol=0)


def test_lambda_grid_bruteforce(rng):
    """Random 4x2-sized instances with bounds active: vol(lam) evaluated on a fine
    log grid straight from the definition brackets the oracle's lam."""
    for trial in range(5):
        n = 8
        x = rng.uniform(0.001, 1.0, n)
        V = rng.choice([1.0, 0.25], n)
        dc = -np.exp(rng.uniform(-4, 2, n)) * V
        volfrac = 0.4
        r = oc.oc_update(x, dc, V, volfrac)
        if r.status != "active":
            continue
        grid = np.exp(np.linspace(np.log(1e-8), np.log(1e8), 200001))
        vols = []
        for lam in grid[::1]:
            B = -dc / (lam * V)
            xc = np.clip(x * np.sqrt(B), np.maximum(1e-3, x - 0.2), np.minimum(1.0, x + 0.2))
            vols.append(np.sum(V * xc))
        vols = np.array(vols)
        assert np.all(np.diff(vols) <= 1e-12)            # vol non-increasing in lam
        tgt = volfrac * V.sum()
        k = np.nonzero(vols <= tgt)[0][0]                 # first grid lam with vol <= target
        assert grid[k - 1] * (1 - 1e-9) <= r.lam <= grid[k] * (1 + 1e-9)
        assert abs(np.sum(V * r.x) - tgt) <= 1e-9 * tgt


def test_invariants_random(rng):
    """Bounds, move limit, and volume equality when active."""
    for _ in range(20):
        n = int(rng.integers(5, 200))
        x = rng.uniform(0.001, 1.0, n)
        V = rng.choice([1.0, 0.5, 0.125], n)
        dc = -np.abs(rng.standard_normal(n)) * 10 ** rng.uniform(-3, 3)
        dc[rng.random(n) < 0.1] = 0.0
        volfrac = rng.uniform(0.1, 0.9)
        r = oc.oc_update(x, dc, V, volfrac)
        assert np.all(r.x >= 1e-3) and np.all(r.x <= 1.0)
        assert np.all(np.abs(r.x - x) <= 0.2 + 1e-15)
        if r.status == "active":
            assert abs(r.volume - volfrac) <= 1e-10
        else:
            assert r.volume <= volfrac + 1e-12 or r.status == "infeasible"


def test_convergence_condition():
    assert oc.converged(0.0099) and not oc.converged(0.01) and not oc.converged(0.02)


def _kkt_check(m, x, penal, lam_tol):
    V = m.volumes()
    u = oc.solve_u(m, x, penal)
    dc = topopt.sensitivities(m, x, u, penal)
    r = oc.oc_update(x, dc, V, 0.5)
    ratio = -dc / (r.lam * V)
    inner = (x > 0.02) & (x < 0.999)
    assert inner.sum() > 3
    np.testing.assert_allclose(ratio[inner], 1.0, atol=lam_tol)
    assert np.all(ratio[x <= 0.02] <= 1.0 + lam_tol)   # at (or decaying to) the lower bound: <= lam
    assert np.all(ratio[x >= 0.999] >= 1.0 - lam_tol)  # at upper bound: marginal value >= lam


@pytest.mark.parametrize("amr", [False, True])
def test_loop_reaches_kkt_point_p1(amr):
    """p = 1 without filter is the convex variable-thickness-sheet problem; the
    loop's fixed point must satisfy its KKT conditions: -dc_e / V_e = lam on
    elements strictly inside the bounds (the OC criterion, Bendsoe's book)."""
    if amr:
        prob = cantilever2d((6, 3), L=1, leaves=refine_some(2, (6, 3), 1, [(5, 0), (4, 1)]))
    else:
        prob = cantilever2d((8, 4))
    m = omesh.build_mesh(prob)
    V = m.volumes()
    x0 = np.full(m.n_el, 0.5)
    x, H = oc.optimize(m, x0, 0.5, 300, rmin=0.0, penal0=1.0, penal_max=1.0)
    for v in H.volume:
        assert abs(v - 0.5) <= 1e-10
    assert H.change[-1] < 1e-3   # OC creeps towards the bounds: linear but slow
    # the p = 1 compliance decreases monotonically along the loop
    assert all(b <= a * (1 + 1e-12) for a, b in zip(H.compliance[5:], H.compliance[6:]))
    assert abs(np.sum(V * x) / V.sum() - 0.5) <= 1e-10
    _kkt_check(m, x, 1.0, 5e-3)


def test_loop_continuation_schedule():
    """p-continuation (reading R19): starts at 1, steps by 0.5, capped."""
    m = omesh.build_mesh(cantilever2d((6, 3)))
    _, H = oc.optimize(m, np.full(m.n_el, 0.5), 0.5, 14, rmin=1.5, stage_steps=3)
    assert H.penal[0] == 1.0 and max(H.penal) == 3.0
    assert all(b - a in (0.0, 0.5) for a, b in zip(H.penal, H.penal[1:]))
    assert all(abs(v - 0.5) <= 1e-10 for v in H.volume)
