"""Pins for oracle/topopt.py."""
import numpy as np
import pytest

from inputs import DensitySpec
from oracle import fe, mesh as omesh, solve, topopt
from tests.helpers import cantilever2d, cantilever3d, refine_some


def _solve(m, x, penal, Emin=1e-9):
    K = fe.assemble_K(m, x, penal, 1.0, Emin)
    A, b, C = fe.projected_system(m, K)
    return fe.recover(C, solve.dense_solve(A, b))


def test_sensitivity_finite_differences(rng):
    """central differences with exact solves agree to 1e-4 on a 4x2 mesh."""
    m = omesh.build_mesh(cantilever2d((4, 2)))
    x = rng.uniform(0.3, 0.9, m.n_el)
    u = _solve(m, x, 3.0)
    dc = topopt.sensitivities(m, x, u, 3.0)
    delta = 1e-6
    for e in range(m.n_el):
        xp, xm = x.copy(), x.copy()
        xp[e] += delta
        xm[e] -= delta
        cp = fe.compliance(m.load, _solve(m, xp, 3.0))
        cm = fe.compliance(m.load, _solve(m, xm, 3.0))
        fd = (cp - cm) / (2 * delta)
        assert abs(fd - dc[e]) <= 1e-4 * abs(dc[e])
    assert np.all(dc <= 0)


def test_sensitivity_fd_with_hanging_nodes(rng):
    prob = cantilever2d((3, 2), L=1, leaves=refine_some(2, (3, 2), 1, [(1, 0)]))
    m = omesh.build_mesh(prob)
    assert m.hang_node.size > 0
    x = rng.uniform(0.3, 0.9, m.n_el)
    u = _solve(m, x, 3.0)
    dc = topopt.sensitivities(m, x, u, 3.0)
    delta = 1e-6
    for e in rng.choice(m.n_el, 6, replace=False):
        xp, xm = x.copy(), x.copy()
        xp[e] += delta
        xm[e] -= delta
        fd = (fe.compliance(m.load, _solve(m, xp, 3.0)) - fe.compliance(m.load, _solve(m, xm, 3.0))) / (2 * delta)
        assert abs(fd - dc[e]) <= 1e-4 * abs(dc[e])


@pytest.mark.parametrize("dim", [2, 3])
def test_sensitivity_homogeneity_identity(dim, rng):
    """sum_e x_e dc_e = -p (c - E_min sum_e u_e^T K0 u_e) (degree -p homogeneity)."""
    if dim == 2:
        m = omesh.build_mesh(cantilever2d((5, 3), L=1, leaves=refine_some(2, (5, 3), 1, [(2, 1)])))
    else:
        m = omesh.build_mesh(cantilever3d((3, 2, 2), L=1, leaves=refine_some(3, (3, 2, 2), 1, [(1, 0, 0)])))
    x = rng.uniform(0.05, 1, m.n_el)
    Emin = 1e-3
    u = _solve(m, x, 3.0, Emin)
    c = fe.compliance(m.load, u)
    dc = topopt.sensitivities(m, x, u, 3.0, 1.0, Emin)
    en = topopt.element_energy(m, u)
    lhs = (x * dc).sum()
    rhs = -3.0 * (c - Emin * en.sum())
    assert abs(lhs - rhs) <= 1e-10 * abs(rhs)


def test_sensitivity_special_cases(rng):
    m = omesh.build_mesh(cantilever2d((4, 2)))
    x = rng.uniform(0.3, 0.9, m.n_el)
    u = _solve(m, x, 1.0)
    dc = topopt.sensitivities(m, x, u, 1.0, 1.0, 1e-9)
    assert np.allclose(dc, -(1 - 1e-9) * topopt.element_energy(m, u), rtol=1e-15, atol=0)
    # element with all corners at zero displacement -> 0
    uz = u.copy()
    uz[fe.element_dofs(m)[0]] = 0.0
    assert topopt.sensitivities(m, x, uz, 3.0)[0] == 0.0


def _amr_mesh(rmin):
    prob = cantilever2d((4, 2), L=2, leaves=refine_some(2, (4, 2), 2, [(1, 0), (2, 1)]), rmin=rmin)
    return omesh.build_mesh(prob), prob


def test_filter_bruteforce_and_invariants(rng):
    m, prob = _amr_mesh(0.9)
    x = rng.uniform(0.05, 1, m.n_el)
    dc = -rng.uniform(0.1, 2, m.n_el)
    out = topopt.filter_sens(m, prob.rmin, x, dc)
    bf = topopt.filter_bruteforce(m, prob.rmin, x, dc, "sens")
    assert np.max(np.abs(out - bf)) <= 1e-12 * np.max(np.abs(bf))
    outd = topopt.filter_dens(m, prob.rmin, dc)
    bfd = topopt.filter_bruteforce(m, prob.rmin, x, dc, "dens")
    assert np.max(np.abs(outd - bfd)) <= 1e-12 * np.max(np.abs(bfd))
    # linear in dc
    out2 = topopt.filter_sens(m, prob.rmin, x, 3.0 * dc)
    assert np.max(np.abs(out2 - 3.0 * out)) <= 1e-13 * np.max(np.abs(out))
    # convex combination of x_d dc_d / x_e
    for e in range(m.n_el):
        nb = m.filt_idx[m.filt_ptr[e]:m.filt_ptr[e + 1]]
        vals = x[nb] * dc[nb] / x[e]
        assert vals.min() - 1e-12 <= out[e] <= vals.max() + 1e-12
    # DENS preserves a constant field; SENS of uniform x, dc is unchanged
    assert np.allclose(topopt.filter_dens(m, prob.rmin, np.full(m.n_el, 0.7)), 0.7, rtol=1e-15)
    assert np.allclose(topopt.filter_sens(m, prob.rmin, np.full(m.n_el, 0.4),
                                          np.full(m.n_el, -2.0)), -2.0, rtol=1e-15)


def test_filter_small_radius_is_identity(rng):
    """the filter is deactivated below the smallest element size."""
    m, prob = _amr_mesh(0.2)        # finest centre distance is 0.25
    x = rng.uniform(0.05, 1, m.n_el)
    dc = -rng.uniform(0.1, 2, m.n_el)
    assert np.all(np.diff(m.filt_ptr) == 1)
    assert np.allclose(topopt.filter_sens(m, prob.rmin, x, dc), dc, rtol=1e-15, atol=0)


def test_filter_stencil_counts_uniform():
    """rmin = 1.5: 9 neighbours in 2D interior (|d|^2 in {0,1,2}); 3D: 19 with rmin 1.5,
    27 with rmin 2.0 (the config-3 and config-5 stencils)."""
    from inputs import make_problem
    m2 = omesh.build_mesh(make_problem("u2", 2, (5, 5), rmin=1.5))
    assert np.diff(m2.filt_ptr).max() == 9
    m3 = omesh.build_mesh(make_problem("u3", 3, (5, 5, 5), rmin=1.5))
    assert np.diff(m3.filt_ptr).max() == 19
    m3b = omesh.build_mesh(make_problem("u3b", 3, (5, 5, 5), rmin=2.0))
    assert np.diff(m3b.filt_ptr).max() == 27
