"""Pins for oracle/minres.py (the paper's solver).

MINRES: iterates against scipy.sparse.linalg.minres (a library routine, the
same method), |eta_j| equal to the true M^-1-norm of the residual, monotone,
and the textbook special cases.  IC(0): equal to the exact Cholesky factor
when the pattern has no fill (tridiagonal), sqrt of a diagonal, and the
defining property (L L^T)_ij = A_ij on the pattern of tril(A)."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import fe, mesh as omesh, minres as om
from tests.helpers import cantilever2d, refine_some


def _spd(rng, n, density=0.15):
    R = sp.random(n, n, density=density, random_state=np.random.RandomState(int(rng.integers(1 << 30))))
    A = (R @ R.T + sp.eye(n) * n * 0.05).tocsr()
    return A


def _laplace2d(m):
    T = sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(m, m))
    return (sp.kron(sp.eye(m), T) + sp.kron(T, sp.eye(m))).tocsr()


def test_minres_matches_scipy_iterates(rng):
    A = _spd(rng, 60)
    b = rng.standard_normal(60)
    xs = []
    spla.minres(A, b, rtol=1e-14, maxiter=12, callback=lambda xk: xs.append(xk.copy()))
    for k in range(1, 9):
        r = om.minres(A, b, rtol=0.0, max_iter=k)
        np.testing.assert_allclose(r.x, xs[k - 1], rtol=1e-9, atol=1e-12)


def test_preconditioned_minres_matches_scipy(rng):
    A = _spd(rng, 50)
    b = rng.standard_normal(50)
    d = A.diagonal()
    Minv = spla.LinearOperator(A.shape, matvec=lambda v: v / d)
    xs = []
    spla.minres(A, b, M=Minv, rtol=1e-14, maxiter=10, callback=lambda xk: xs.append(xk.copy()))
    for k in range(1, 8):
        r = om.minres(A, b, msolve=lambda v: v / d, rtol=0.0, max_iter=k)
        np.testing.assert_allclose(r.x, xs[k - 1], rtol=1e-9, atol=1e-12)


def test_eta_is_preconditioned_residual_norm_and_monotone(rng):
    A = _spd(rng, 40)
    b = rng.standard_normal(40)
    d = A.diagonal()
    for k in range(1, 25, 3):
        r = om.minres(A, b, msolve=lambda v: v / d, rtol=0.0, max_iter=k)
        res = b - A @ r.x
        true = np.sqrt(res @ (res / d))
        assert abs(r.eta[-1] - true) <= 1e-9 * r.eta[0]
    r = om.minres(A, b, msolve=lambda v: v / d, rtol=1e-12, max_iter=200)
    assert all(b2 <= a2 * (1 + 1e-12) for a2, b2 in zip(r.eta, r.eta[1:]))
    np.testing.assert_allclose(r.x, spla.spsolve(A.tocsc(), b), rtol=1e-9)


def test_minres_special_cases():
    b = np.array([1.0, 2.0, 3.0])
    r = om.minres(sp.eye(3).tocsr(), b, rtol=1e-14)
    assert r.iters == 1 and np.allclose(r.x, b)
    r = om.minres(sp.diags([1.0, 2.0, 3.0]).tocsr(), b, rtol=1e-14)
    assert r.iters == 3 and np.allclose(r.x, 1.0, rtol=1e-13)


def test_ic0_tridiagonal_is_cholesky(rng):
    n = 30
    main = 2.0 + rng.uniform(0, 1, n)
    off = -rng.uniform(0.1, 0.9, n - 1)
    A = sp.diags([off, main, off], [-1, 0, 1]).tocsr()
    L = om.ic0(A).toarray()
    np.testing.assert_allclose(L, np.linalg.cholesky(A.toarray()), rtol=1e-13, atol=1e-15)
    Ld = om.ic0(sp.diags(main).tocsr()).toarray()
    np.testing.assert_allclose(Ld, np.diag(np.sqrt(main)), rtol=1e-15)


def test_ic0_defining_property():
    A = _laplace2d(7)
    L = om.ic0(A)
    P = (L @ L.T).toarray()
    T = sp.tril(A).tocoo()
    for i, j, v in zip(T.row, T.col, T.data):
        assert abs(P[i, j] - v) <= 1e-13
    pat = set(zip(T.row.tolist(), T.col.tolist()))
    Lc = L.tocoo()
    assert set(zip(Lc.row.tolist(), Lc.col.tolist())) <= pat
    # fill positions differ from A (this pattern has fill), so IC(0) != Cholesky here
    assert np.max(np.abs(P - A.toarray())) > 1e-3


def test_ic0_preconditioning_reduces_iterations():
    """4x4 Laplacian, preconditioned MINRES strictly fewer iterations."""
    A = _laplace2d(4)
    b = np.ones(16)
    plain = om.minres(A, b, rtol=1e-10)
    L = om.ic0(A)
    pre = om.minres(A, b, msolve=lambda v: om.ic0_solve(L, v), rtol=1e-10)
    assert pre.iters < plain.iters
    np.testing.assert_allclose(pre.x, spla.spsolve(A.tocsc(), b), rtol=1e-8)


@pytest.mark.parametrize("amr", [False, True])
def test_paper_solver_on_fe_system(amr):
    """MINRES + IC(0) on the rescaled projected system reaches the direct solution,
    in fewer iterations than without the preconditioner."""
    if amr:
        prob = cantilever2d((8, 4), L=2, leaves=refine_some(2, (8, 4), 2, [(3, 1), (6, 2)]))
    else:
        prob = cantilever2d((16, 8))
    m = omesh.build_mesh(prob)
    x = np.random.default_rng(2).uniform(0.05, 1.0, m.n_el)
    K = fe.assemble_K(m, x, 3.0)
    A, b, C = fe.projected_system(m, K)
    u_ic, r_ic = om.solve_paper(A, b, rtol=1e-12, precond="ic0")
    u_j, r_j = om.solve_paper(A, b, rtol=1e-12, precond="none")
    ud = spla.spsolve(A.tocsc(), b)
    np.testing.assert_allclose(u_ic, ud, rtol=1e-7, atol=1e-9 * np.abs(ud).max())
    np.testing.assert_allclose(u_j, ud, rtol=1e-7, atol=1e-9 * np.abs(ud).max())
    assert r_ic.iters < r_j.iters / 2
    assert r_ic.shift is not None


def test_shifted_ic0_picks_smallest_working_shift():
    """Laplacian (an M-matrix): no shift; a matrix with a negative pivot under
    IC(0): the returned shift works and half of it does not."""
    L, a = om.ic0_shifted(_laplace2d(5))
    assert a == 0.0
    prob = cantilever2d((16, 8))
    m = omesh.build_mesh(prob)
    x = np.random.default_rng(2).uniform(0.05, 1.0, m.n_el)
    A, b, C = fe.projected_system(m, fe.assemble_K(m, x, 3.0))
    Kt, bt, s = om.rescale(A, b)
    L, a = om.ic0_shifted(Kt)
    if a > 0:
        n = Kt.shape[0]
        if a > 1e-3:
            with pytest.raises(ArithmeticError):
                om.ic0(Kt + (a / 2) * sp.eye(n, format="csr"))
        with pytest.raises(ArithmeticError):
            om.ic0(Kt)
