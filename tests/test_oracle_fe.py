"""Pins for oracle/fe.py."""
import os

import numpy as np
import pytest
import scipy.sparse as sp

from inputs import DensitySpec, make_problem, uniform_leaves
from oracle import fe, mesh as omesh, solve
from tests.helpers import cantilever2d, cantilever3d, refine_some

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rigid_modes(dim, h=1.0):
    nc = 1 << dim
    X = np.array([[((c >> k) & 1) * h for k in range(dim)] for c in range(nc)], dtype=float)
    modes = []
    for k in range(dim):
        v = np.zeros((nc, dim))
        v[:, k] = 1.0
        modes.append(v.ravel())
    rots = [(0, 1)] if dim == 2 else [(0, 1), (1, 2), (0, 2)]
    for a, b in rots:
        v = np.zeros((nc, dim))
        v[:, a] = -X[:, b]
        v[:, b] = X[:, a]
        modes.append(v.ravel())
    return np.array(modes).T


def _load_q4_closed_form(nu):
    lines = [l.strip() for l in open(os.path.join(GOLD, "q4_ke_closed_form.txt"))
             if l.strip() and not l.startswith("#")]
    k = []
    for l in lines[:8]:
        expr = l.split("=", 1)[1]
        k.append(eval(expr, {"nu": nu}))
    pat = np.array([[int(t) for t in l.split()] for l in lines[8:16]])
    return np.array(k)[pat - 1] / (1 - nu * nu)


# P1 -------------------------------------------------------------------------
def test_q4_K00_closed_form():
    K = fe.element_stiffness(2, 1.0, 0.3, 1.0)
    assert abs(K[0, 0] - (0.5 - 0.3 / 6) / (1 - 0.09)) < 1e-15


@pytest.mark.parametrize("nu", [0.0, 0.3, 0.45])
def test_q4_matches_published_element_matrix(nu):
    KE = _load_q4_closed_form(nu)          # CCW node order (0,0),(1,0),(1,1),(0,1)
    perm_nodes = [0, 1, 3, 2]               # C4 corners in that order
    perm = np.array([[2 * n, 2 * n + 1] for n in perm_nodes]).ravel()
    K = fe.element_stiffness(2, 1.0, nu, 1.0)
    assert np.max(np.abs(K[np.ix_(perm, perm)] - KE)) < 1e-14


@pytest.mark.parametrize("dim", [2, 3])
def test_K0_symmetry_rank_rigid_modes(dim):
    K = fe.element_stiffness(dim, 1.0, 0.3, 1.0)
    assert np.max(np.abs(K - K.T)) < 1e-15
    R = _rigid_modes(dim)
    assert np.max(np.abs(K @ R)) < 1e-14
    assert np.linalg.matrix_rank(K, tol=1e-10) == (5 if dim == 2 else 18)
    ev = np.linalg.eigvalsh(K)
    assert ev.min() > -1e-14


@pytest.mark.parametrize("dim", [2, 3])
def test_K0_gauss_exactness_and_h_scaling(dim):
    K2 = fe.element_stiffness(dim, 1.0, 0.3, 1.0, ngauss=2)
    K3 = fe.element_stiffness(dim, 1.0, 0.3, 1.0, ngauss=3)
    assert np.max(np.abs(K2 - K3)) < 1e-14
    Kh = fe.element_stiffness(dim, 1.0, 0.3, 0.5)
    if dim == 2:
        assert np.max(np.abs(Kh - K2)) < 1e-14          # 2D: independent of h
    else:
        assert np.max(np.abs(Kh - 0.5 * K2)) < 1e-14    # 3D: linear in h (Q14)


# P2 -------------------------------------------------------------------------
def test_h8_K00_closed_form_and_dense():
    nu = 0.3
    K = fe.element_stiffness(3, 1.0, nu, 1.0)
    assert abs(K[0, 0] - (2 - 3 * nu) / (9 * (1 + nu) * (1 - 2 * nu))) < 1e-15
    assert np.count_nonzero(np.abs(K) > 1e-14) == 576


@pytest.mark.parametrize("dim", [2, 3])
def test_K0_constant_strain_energy(dim, rng):
    """Patch identity: for u = eps x (constant strain), u^T K0 u = V eps^T D eps."""
    h = 0.75
    K = fe.element_stiffness(dim, 2.5, 0.3, h)
    D = fe.constitutive(2.5, 0.3, dim)
    nc = 1 << dim
    X = np.array([[((c >> k) & 1) * h for k in range(dim)] for c in range(nc)], dtype=float)
    for _ in range(5):
        G = rng.standard_normal((dim, dim))
        u = (X @ G.T).ravel()                        # u_i = G_ij x_j
        E = 0.5 * (G + G.T)
        if dim == 2:
            ev = np.array([E[0, 0], E[1, 1], 2 * E[0, 1]])
        else:
            ev = np.array([E[0, 0], E[1, 1], E[2, 2], 2 * E[0, 1], 2 * E[1, 2], 2 * E[0, 2]])
        assert abs(u @ K @ u - h ** dim * ev @ D @ ev) < 1e-12 * abs(h ** dim * ev @ D @ ev)


# P3 -------------------------------------------------------------------------
def test_simp_values():
    assert fe.simp(1.0, 3, 1.0, 1e-9) == 1.0
    assert abs(fe.simp(0.5, 3, 1.0, 1e-9) - (1e-9 + 0.125 * (1 - 1e-9))) < 1e-17
    assert abs((1e-3) ** 3 - 1e-9) < 1e-24
    assert abs(fe.simp(0.0, 3, 1.0, 1e-9) - 1e-9) < 1e-24


# P4 -------------------------------------------------------------------------
def _dense_assembly(m, x, penal, nu=0.3):
    n = m.n_dof
    K = np.zeros((n, n))
    for e in range(m.n_el):
        K0 = fe.element_stiffness(m.dim, 1.0, nu, float(m.h()[e]))
        dofs = [m.dim * int(m.elem_node[e, c]) + k for c in range(1 << m.dim) for k in range(m.dim)]
        for a in range(len(dofs)):
            for b in range(len(dofs)):
                K[dofs[a], dofs[b]] += fe.simp(x[e], penal) * K0[a, b]
    return K


@pytest.mark.parametrize("dim", [2, 3])
def test_assembly_vs_dense_loop(dim, rng):
    prob = cantilever2d((2, 2)) if dim == 2 else cantilever3d((2, 2, 1))
    m = omesh.build_mesh(prob)
    x = rng.uniform(0.1, 1.0, m.n_el)
    K = fe.assemble_K(m, x, 3.0).toarray()
    Kd = _dense_assembly(m, x, 3.0)
    assert np.max(np.abs(K - Kd)) < 1e-14
    assert np.max(np.abs(K - K.T)) < 1e-15 * np.max(np.abs(K))
    # rigid modes annihilated before BCs
    X = m.node_coord.astype(float) * m.hL
    R = np.zeros((m.n_dof, dim))
    for k in range(dim):
        R[k::dim, k] = 1.0
    rot = np.zeros(m.n_dof)
    rot[0::dim] = -X[:, 1]
    rot[1::dim] = X[:, 0]
    R = np.column_stack([R, rot])
    assert np.max(np.abs(K @ R)) < 1e-12 * np.max(np.abs(K))


def test_single_fully_fixed_element_zero_compliance():
    prob = make_problem("one", 2, (1, 1), fixed=[((0, 0), (1, 1), 0b11)],
                        loads=[("point", (1, 1), (1, 1), (0.0, -1.0))])
    m = omesh.build_mesh(prob)
    K = fe.assemble_K(m, np.ones(1), 3.0)
    A, b, C = fe.projected_system(m, K)
    assert np.all(b == 0.0)
    u = fe.recover(C, solve.dense_solve(A, b))
    assert fe.compliance(m.load, u) == 0.0


def test_p1_linearity_doubling_density_halves_u():
    prob = cantilever2d((4, 2), Emin=0.0)
    m = omesh.build_mesh(prob)
    def solve_u(x):
        K = fe.assemble_K(m, x, 1.0, 1.0, 0.0)
        A, b, C = fe.projected_system(m, K)
        return fe.recover(C, solve.dense_solve(A, b))
    x = np.linspace(0.2, 0.5, m.n_el)
    u1, u2 = solve_u(x), solve_u(2 * x)
    assert np.max(np.abs(u1 - 2 * u2)) < 1e-12 * np.max(np.abs(u1))


# P6 -------------------------------------------------------------------------
def test_projection_without_hanging_is_dirichlet_reduced_K(rng):
    m = omesh.build_mesh(cantilever2d((3, 2)))
    x = rng.uniform(0.1, 1, m.n_el)
    K = fe.assemble_K(m, x, 3.0).toarray()
    A, b, C = fe.projected_system(m, sp.csr_matrix(K))
    Kr = K.copy()
    Kr[m.fixed_dof, :] = 0
    Kr[:, m.fixed_dof] = 0
    Kr[m.fixed_dof, m.fixed_dof] = 1.0
    assert np.max(np.abs(A.toarray() - Kr)) == 0.0


@pytest.mark.parametrize("dim", [2, 3])
def test_projected_system_vs_dense_elimination(dim, rng):
    """Eqs. 6-9 vs eliminating u_c = P u_f directly with a transformation T."""
    if dim == 2:
        prob = cantilever2d((3, 3), L=1, leaves=refine_some(2, (3, 3), 1, [(1, 1)]))
    else:
        prob = cantilever3d((3, 2, 2), L=1, leaves=refine_some(3, (3, 2, 2), 1, [(1, 0, 0)]))
    m = omesh.build_mesh(prob)
    assert m.hang_node.size > 0
    x = rng.uniform(0.1, 1, m.n_el)
    K = fe.assemble_K(m, x, 3.0)
    A, b, C = fe.projected_system(m, K)
    Ad = A.toarray()
    # unit rows on hanging DOFs
    for hn in m.hang_node:
        for c in range(dim):
            i = dim * hn + c
            row = Ad[i].copy()
            assert row[i] == 1.0
            row[i] = 0.0
            assert np.all(row == 0.0)
    u_proj = fe.recover(C, solve.dense_solve(A, b))
    # independent elimination: T maps independent DOFs (free, non-hanging) to all DOFs
    fm = fe.free_mask(m)
    indep = np.nonzero(fm)[0]
    col = {int(i): k for k, i in enumerate(indep)}
    T = np.zeros((m.n_dof, indep.size))
    for i in indep:
        T[i, col[int(i)]] = 1.0
    for k, hn in enumerate(m.hang_node):
        for j in range(m.hang_ptr[k], m.hang_ptr[k + 1]):
            for c in range(dim):
                pd = dim * int(m.hang_parent[j]) + c
                if pd in col:
                    T[dim * hn + c, col[pd]] += m.hang_weight[j]
    Kd = K.toarray()
    y = np.linalg.solve(T.T @ Kd @ T, T.T @ m.load)
    u_elim = T @ y
    assert np.linalg.norm(u_proj - u_elim) < 1e-10 * np.linalg.norm(u_elim)


# P13 ------------------------------------------------------------------------
def test_compliance_identities(rng):
    prob = cantilever2d((6, 3), L=1, leaves=refine_some(2, (6, 3), 1, [(2, 1), (3, 1)]))
    m = omesh.build_mesh(prob)
    x = rng.uniform(0.05, 1, m.n_el)
    K = fe.assemble_K(m, x, 3.0)
    A, b, C = fe.projected_system(m, K)
    u = fe.recover(C, solve.dense_solve(A, b))
    c = fe.compliance(m.load, u)
    assert abs(c - u @ (K @ u)) < 1e-10 * abs(c)
    # element-wise energy sum
    en = 0.0
    for e in range(m.n_el):
        K0 = fe.element_stiffness(2, 1.0, 0.3, float(m.h()[e]))
        dofs = [2 * int(m.elem_node[e, k]) + j for k in range(4) for j in range(2)]
        en += fe.simp(x[e], 3.0) * u[dofs] @ K0 @ u[dofs]
    assert abs(c - en) < 1e-10 * abs(c)
    assert c > 0
    # f = 0 -> 0
    assert fe.compliance(np.zeros(m.n_dof), u) == 0.0
    # monotone: stiffening one element lowers compliance
    x2 = x.copy()
    x2[5] = min(1.0, x2[5] + 0.3)
    K2 = fe.assemble_K(m, x2, 3.0)
    A2, b2, C2 = fe.projected_system(m, K2)
    u2 = fe.recover(C2, solve.dense_solve(A2, b2))
    assert fe.compliance(m.load, u2) < c


# P12 ------------------------------------------------------------------------
def _tip_deflection(nely):
    Lb, H = 10.0, 1.0
    h = H / nely
    nelx = int(Lb / h)
    prob = make_problem("beam", 2, (nelx, nely), h0=h,
                        fixed=[((0, 0), (0, nely), 0b11)],
                        loads=[("line", (nelx, 0), (nelx, nely), (0.0, -1.0))],
                        Emin=0.0)
    m = omesh.build_mesh(prob, with_filter=False)
    K = fe.assemble_K(m, np.ones(m.n_el), 1.0, 1.0, 0.0)
    A, b, C = fe.projected_system(m, K)
    u = fe.recover(C, solve.pcg_jacobi(A, b, rtol=1e-12).x)
    tip = np.nonzero(m.node_coord[:, 0] == nelx)[0]
    return -u[2 * tip + 1].mean()


def test_beam_theory_tip_deflection():
    """Slender cantilever (L/H = 10): Timoshenko PL^3/(3EI) + PL/(kGA)."""
    E, nu, P, Lb, H = 1.0, 0.3, 1.0, 10.0, 1.0   # line load of intensity 1 over H -> P = 1
    I = H ** 3 / 12
    G = E / (2 * (1 + nu))
    # plane stress beam: E; unit thickness
    ref = P * Lb ** 3 / (3 * E * I) + P * Lb / (5.0 / 6.0 * G * H)
    d4, d8 = _tip_deflection(4), _tip_deflection(8)
    err4, err8 = abs(d4 - ref) / ref, abs(d8 - ref) / ref
    assert err8 < 0.03
    assert err8 < err4
