"""Pins for oracle/sample.py: the element-by-element / output-by-output
evaluation used at full configuration sizes must reproduce the assembled
oracle (fe.py, itself pinned by closed forms and brute force) and the O(n^2)
brute-force filter twin on meshes where both run."""
import numpy as np
import pytest

from inputs import config
from oracle import fe, mesh as omesh, sample, topopt
from tests.helpers import cantilever2d, cantilever3d, refine_some

CASES = {
    "c1": lambda: config("c1"),
    "amr2d": lambda: cantilever2d((5, 3), L=3, leaves=refine_some(2, (5, 3), 3, [(1, 1), (3, 0)]), rmin=0.3),
    "amr3d": lambda: cantilever3d((3, 2, 2), L=2, leaves=refine_some(3, (3, 2, 2), 2, [(1, 1, 0)]), rmin=0.4),
    "c5s": lambda: config("c5", nx=6, ny=3, nz=3),
}


@pytest.mark.parametrize("name", list(CASES))
def test_apply_full_equals_assembled_projected_operator(name, rng):
    prob = CASES[name]()
    m = omesh.build_mesh(prob)
    x = rng.uniform(0.01, 1.0, m.n_el)
    K = fe.assemble_K(m, x, 3.0, 1.0, 1e-9, 0.3)
    A, b, C = fe.projected_system(m, K)
    v = rng.standard_normal(m.n_dof)
    q = sample.apply_full(m, x, v, 3.0)
    assert np.linalg.norm(q - A @ v) <= 1e-13 * np.linalg.norm(A @ v)
    assert np.array_equal(sample.rhs(m), b)
    u = C @ rng.standard_normal(m.n_dof)
    uhat = u.copy()
    for c in range(m.dim):
        uhat[m.hang_node.astype(np.int64) * m.dim + c] = 0.0
    ref = np.linalg.norm(b - A @ uhat) / np.linalg.norm(b)
    assert abs(sample.residual_norm(m, x, u, 3.0) - ref) <= 1e-12 * ref


@pytest.mark.parametrize("name", ["c1", "amr2d", "amr3d"])
def test_filter_rows_equals_bruteforce(name, rng):
    prob = CASES[name]()
    m = omesh.build_mesh(prob)
    x = rng.uniform(0.01, 1.0, m.n_el)
    dc = -rng.uniform(0.0, 1.0, m.n_el)
    elems = rng.choice(m.n_el, size=min(25, m.n_el), replace=False)
    for mode in ("sens", "dens"):
        full = topopt.filter_bruteforce(m, prob.rmin, x, dc, mode=mode)
        got = sample.filter_rows(m, prob.rmin, x, dc, elems, mode=mode)
        assert np.allclose(got, full[elems], rtol=1e-13, atol=0)
