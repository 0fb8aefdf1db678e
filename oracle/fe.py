"""ORACLE (test infrastructure only) — finite-element operators.

* Element stiffness by Gauss quadrature (bi/tri-linear displacement,
  PAPER.md:288-293; plane stress, unit thickness in 2D).
* SIMP, Eq. 2 in the modified form of north_star /
  SURVEY Q1:  E_e = E_min + x_e^p (E0 - E_min).
* Assembled K(x), the interpolation C = [I 0; P 0]
  (Eq. 6), the projected operator with unit diagonal on the
  constrained DOFs (Eq. 8) extended to Dirichlet DOFs by
  symmetric elimination, its rhs (Eq. 7), recovery (Eq. 9,
  PAPER.md:684-686) and compliance f^T u (Eq. 1).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .mesh import OracleMesh


def lame(E: float, nu: float, dim: int):
    mu = E / (2.0 * (1.0 + nu))
    if dim == 2:   # plane stress
        lam = E * nu / (1.0 - nu * nu)
    else:
        lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    return lam, mu


def constitutive(E: float, nu: float, dim: int) -> np.ndarray:
    """Voigt D: 2D (xx, yy, xy); 3D (xx, yy, zz, xy, yz, zx), engineering shear."""
    if dim == 2:
        return E / (1.0 - nu * nu) * np.array([[1.0, nu, 0.0], [nu, 1.0, 0.0],
                                               [0.0, 0.0, 0.5 * (1.0 - nu)]])
    lam, mu = lame(E, nu, 3)
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[0, 0] = D[1, 1] = D[2, 2] = lam + 2 * mu
    D[3, 3] = D[4, 4] = D[5, 5] = mu
    return D


def element_stiffness(dim: int, E: float, nu: float, h: float, ngauss: int = 2) -> np.ndarray:
    """K0 = sum_gp B^T D B |J| w on the cube [0,h]^d, corner c = cx+2cy+4cz,
    local DOF = d*c + component (C4)."""
    xg, wg = np.polynomial.legendre.leggauss(ngauss)
    nc = 1 << dim
    sgn = np.array([[2 * ((c >> k) & 1) - 1 for k in range(dim)] for c in range(nc)], dtype=float)
    D = constitutive(E, nu, dim)
    nstr = 3 if dim == 2 else 6
    K = np.zeros((dim * nc, dim * nc))
    J = h / 2.0
    for idx in np.ndindex(*([ngauss] * dim)):
        xi = np.array([xg[i] for i in idx])
        w = np.prod([wg[i] for i in idx])
        dN = np.zeros((nc, dim))     # d N_c / d x_k
        for c in range(nc):
            f = 1.0 + sgn[c] * xi     # (1 + s_k xi_k)
            for k in range(dim):
                prod = sgn[c, k]
                for m in range(dim):
                    if m != k:
                        prod *= f[m]
                dN[c, k] = prod / (2.0 ** dim) / J
        B = np.zeros((nstr, dim * nc))
        for c in range(nc):
            if dim == 2:
                B[0, 2 * c] = dN[c, 0]
                B[1, 2 * c + 1] = dN[c, 1]
                B[2, 2 * c] = dN[c, 1]
                B[2, 2 * c + 1] = dN[c, 0]
            else:
                B[0, 3 * c] = dN[c, 0]
                B[1, 3 * c + 1] = dN[c, 1]
                B[2, 3 * c + 2] = dN[c, 2]
                B[3, 3 * c] = dN[c, 1]
                B[3, 3 * c + 1] = dN[c, 0]
                B[4, 3 * c + 1] = dN[c, 2]
                B[4, 3 * c + 2] = dN[c, 1]
                B[5, 3 * c] = dN[c, 2]
                B[5, 3 * c + 2] = dN[c, 0]
        K += B.T @ D @ B * (w * J ** dim)
    return K


def simp(x, penal, E0=1.0, Emin=1e-9):
    """Modified SIMP (Eq. 2 with the void floor)."""
    return Emin + np.asarray(x, dtype=np.float64) ** penal * (E0 - Emin)


def element_dofs(mesh: OracleMesh) -> np.ndarray:
    d = mesh.dim
    en = mesh.elem_node.astype(np.int64)
    return (en[:, :, None] * d + np.arange(d)[None, None, :]).reshape(en.shape[0], -1)


def assemble_K(mesh: OracleMesh, x, penal, E0=1.0, Emin=1e-9, nu=0.3, elems=None) -> sp.csr_matrix:
    """K = sum_e E_e P_e^T K0(h_e) P_e (optionally over a subset of elements)."""
    n = mesh.n_dof
    dofs = element_dofs(mesh)
    E = simp(x, penal, E0, Emin)
    hs = mesh.h()
    if elems is None:
        elems = np.arange(mesh.n_el)
    elems = np.asarray(elems, dtype=np.int64)
    ne = dofs.shape[1]
    K = sp.csr_matrix((n, n))
    chunk = max(1, (1 << 22) // (ne * ne))
    parts = []
    for hval in np.unique(hs[elems]):
        K0 = element_stiffness(mesh.dim, 1.0, nu, float(hval))
        sel = elems[hs[elems] == hval]
        for i0 in range(0, sel.shape[0], chunk):
            es = sel[i0:i0 + chunk]
            dd = dofs[es]
            rows = np.repeat(dd, ne, axis=1).ravel()
            cols = np.tile(dd, (1, ne)).ravel()
            vals = (E[es][:, None, None] * K0[None, :, :]).ravel()
            parts.append(sp.csr_matrix((vals, (rows, cols)), shape=(n, n)))
            if len(parts) >= 16:
                K = K + sum(parts[1:], parts[0])
                parts = []
    if parts:
        K = K + sum(parts[1:], parts[0])
    return K.tocsr()


def constraint_matrix(mesh: OracleMesh) -> sp.csr_matrix:
    """C: identity on unconstrained DOFs, rows of P on hanging DOFs (Eq. 6)."""
    d = mesh.dim
    n = mesh.n_dof
    is_h = np.zeros(mesh.n_node, dtype=bool)
    is_h[mesh.hang_node] = True
    rows, cols, vals = [], [], []
    free_nodes = np.nonzero(~is_h)[0]
    for c in range(d):
        rows.append(free_nodes * d + c)
        cols.append(free_nodes * d + c)
        vals.append(np.ones(free_nodes.shape[0]))
    for i, hnode in enumerate(mesh.hang_node.tolist()):
        for k in range(mesh.hang_ptr[i], mesh.hang_ptr[i + 1]):
            par = int(mesh.hang_parent[k])
            for c in range(d):
                rows.append(np.array([hnode * d + c]))
                cols.append(np.array([par * d + c]))
                vals.append(np.array([mesh.hang_weight[k]]))
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(n, n))


def free_mask(mesh: OracleMesh) -> np.ndarray:
    """Pi_F: DOFs that are neither hanging nor fixed."""
    m = np.ones(mesh.n_dof, dtype=bool)
    for c in range(mesh.dim):
        m[mesh.hang_node.astype(np.int64) * mesh.dim + c] = False
    m[mesh.fixed_dof] = False
    return m


def projected_system(mesh: OracleMesh, K: sp.csr_matrix, f=None):
    """A = Pi_F C^T K C Pi_F + (I - Pi_F),  b = Pi_F C^T f  (Eqs. 7-8 + Dirichlet rows)."""
    C = constraint_matrix(mesh)
    F = sp.diags(free_mask(mesh).astype(np.float64))
    I = sp.identity(mesh.n_dof, format="csr")
    A = (F @ (C.T @ K @ C) @ F + (I - F)).tocsr()
    if f is None:
        f = mesh.load
    b = F @ (C.T @ f)
    return A, np.asarray(b).ravel(), C


def recover(C: sp.csr_matrix, uhat: np.ndarray) -> np.ndarray:
    """Eq. 9: u = C u_hat."""
    return C @ uhat


def compliance(f: np.ndarray, u: np.ndarray) -> float:
    """Eq. 1 objective f^T u."""
    return float(np.dot(f, u))
