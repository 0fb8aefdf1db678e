"""Pins for oracle/solve.py."""
import numpy as np
import pytest
import scipy.sparse as sp

from inputs import config, DensitySpec, make_problem, uniform_leaves
from oracle import fe, mesh as omesh, solve, pipeline
from tests.helpers import cantilever2d, cantilever3d, refine_some


def test_toys():
    I = sp.identity(5, format="csr")
    b = np.arange(1.0, 6.0)
    r = solve.pcg_jacobi(I, b, rtol=1e-14)
    assert r.iters == 1 and np.array_equal(r.x, b)
    D = sp.diags([1.0, 2.0, 3.0]).tocsr()
    r = solve.pcg_jacobi(D, np.array([1.0, 2.0, 3.0]), rtol=1e-14)
    assert np.allclose(r.x, 1.0, atol=1e-15, rtol=0) and r.iters == 1


def test_random_spd_vs_dense(rng):
    M = rng.standard_normal((50, 50))
    A = sp.csr_matrix(M @ M.T + 50 * np.eye(50))
    b = rng.standard_normal(50)
    r = solve.pcg_jacobi(A, b, rtol=1e-13)
    xd = np.linalg.solve(A.toarray(), b)
    assert np.linalg.norm(r.x - xd) <= 1e-11 * np.linalg.norm(xd)
    assert r.relres_true <= 10 * 1e-13


def test_warm_start_from_exact_takes_no_iterations(rng):
    m = omesh.build_mesh(cantilever2d((4, 2)))
    K = fe.assemble_K(m, rng.uniform(0.2, 1, m.n_el), 3.0)
    A, b, C = fe.projected_system(m, K)
    x = solve.dense_solve(A, b)
    r = solve.pcg_jacobi(A, b, rtol=1e-8, x0=x)
    assert r.iters <= 1


def test_c1_pcg_vs_dense_direct():
    """P9 on config 1 (2562 DOFs)."""
    prob = config("c1")
    res = pipeline.run(prob)
    xd = solve.dense_solve(res.A, res.b)
    assert np.linalg.norm(res.cg.x - xd) <= 1e-10 * np.linalg.norm(xd)
    assert res.cg.relres <= 1e-10
    assert res.cg.relres_true <= 1e-9


def test_jacobi_pcg_equals_rescaled_cg(rng):
    """P10: CG on D^-1/2 A D^-1/2 produces the Jacobi-PCG iterates."""
    m = omesh.build_mesh(cantilever2d((6, 3)))
    K = fe.assemble_K(m, rng.uniform(0.01, 1, m.n_el), 3.0)
    A, b, C = fe.projected_system(m, K)
    xs = solve.cg_rescaled(A, b, 8)
    for k in range(1, 9):
        r = solve.pcg_jacobi(A, b, fixed_iters=k)
        assert np.linalg.norm(r.x - xs[k - 1]) <= 1e-11 * np.linalg.norm(xs[k - 1])


@pytest.mark.parametrize("dim", [2, 3])
def test_patch_test_with_hanging_nodes(dim, rng):
    """P5: a linear displacement field is reproduced exactly (interior + hanging)."""
    if dim == 2:
        prob = cantilever2d((4, 4), L=2, leaves=refine_some(2, (4, 4), 2, [(1, 1), (2, 2)]))
    else:
        prob = cantilever3d((3, 3, 3), L=1, leaves=refine_some(3, (3, 3, 3), 1, [(1, 1, 1)]))
    m = omesh.build_mesh(prob)
    assert m.hang_node.size > 0
    x = np.full(m.n_el, 0.6)          # patch test: homogeneous material
    K = fe.assemble_K(m, x, 3.0)
    C = fe.constraint_matrix(m)
    KC = (C.T @ K @ C).toarray()
    a0 = rng.standard_normal(dim)
    B = rng.standard_normal((dim, dim))
    X = m.node_coord.astype(float) * m.hL
    ulin = (a0[None, :] + X @ B.T).ravel()
    ext = np.array(prob.lattice_extent)
    onb = np.any((m.node_coord == 0) | (m.node_coord == ext[None, :]), axis=1)
    is_h = np.zeros(m.n_node, dtype=bool)
    is_h[m.hang_node] = True
    interior = np.repeat(~onb & ~is_h, dim)
    bound = np.repeat(onb & ~is_h, dim)
    uhat = np.where(is_h.repeat(dim), 0.0, ulin)
    # residual of C^T K C at interior free DOFs vanishes for a linear field
    res = KC @ uhat
    assert np.max(np.abs(res[interior])) < 1e-11 * np.max(np.abs(KC))
    # solve with the linear field prescribed on the boundary
    I = np.nonzero(interior)[0]
    Bd = np.nonzero(bound)[0]
    uI = np.linalg.solve(KC[np.ix_(I, I)], -KC[np.ix_(I, Bd)] @ ulin[Bd])
    uh = np.zeros(m.n_dof)
    uh[I] = uI
    uh[Bd] = ulin[Bd]
    u = C @ uh
    assert np.max(np.abs(u - ulin)) < 1e-12 * np.max(np.abs(ulin))


def test_galerkin_nesting_amr_stiffer_than_fine(rng):
    """P8: with densities replicated onto the level-L grid, c_AMR <= c_fine; equal when
    the AMR mesh is fully refined."""
    L = 2
    base = (4, 2)
    prob = cantilever2d(base, L=L, leaves=refine_some(2, base, L, [(2, 0), (3, 1)]))
    ma = omesh.build_mesh(prob)
    xa = rng.uniform(0.05, 1, ma.n_el)
    fine = cantilever2d(base, L=L, leaves=uniform_leaves(2, base, L, L))
    mf = omesh.build_mesh(fine)
    # replicate: fine cell -> containing AMR leaf
    xf = np.empty(mf.n_el)
    for e in range(mf.n_el):
        p = mf.elem_anchor[e]
        hit = np.nonzero(np.all((ma.elem_anchor <= p) & (p < ma.elem_anchor + ma.size()[:, None]), axis=1))[0]
        xf[e] = xa[hit[0]]
    cs = []
    for m, x in ((ma, xa), (mf, xf)):
        K = fe.assemble_K(m, x, 3.0)
        A, b, C = fe.projected_system(m, K)
        u = fe.recover(C, solve.dense_solve(A, b))
        cs.append(fe.compliance(m.load, u))
    assert cs[0] < cs[1]
