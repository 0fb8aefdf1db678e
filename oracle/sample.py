"""ORACLE (test infrastructure only) — the hot path's outputs at full
configuration sizes, where the assembled system of `fe.py` would not fit
(config 5: 1.03e9 nonzeros).  Same definitions, evaluated element by element
or output by output; nothing here is blocked, fused or reordered beyond
splitting a sum over elements into chunks.

apply_full    A v = Pi_F C^T K C Pi_F v + (I - Pi_F) v  (Eq. 8, PAPER.md:678-682,
              with Dirichlet rows), K v = sum_e P_e^T (E_e K0(h_e)) P_e v, the
              definition of the assembled stiffness, and
              C the hanging-node interpolation of Eq. 6 (:653-663).
filter_rows   Eq. 5 or the DENS variant for selected
              elements, by brute force over all elements (Eq. 4 weights,
              strict dist < rmin tested on exact squared distances, C9).
residual_norm ||b - A u_hat|| / ||b|| with b = Pi_F C^T f (Eq. 7).
"""
from __future__ import annotations

import numpy as np

from .fe import constraint_matrix, element_dofs, element_stiffness, free_mask, simp
from .mesh import OracleMesh


def stiffness_apply(mesh: OracleMesh, x, w, penal, E0=1.0, Emin=1e-9, nu=0.3, chunk=1 << 18) -> np.ndarray:
    """K w = sum_e P_e^T E_e K0(h_e) P_e w, element by element (chunks of elements)."""
    dofs = element_dofs(mesh)
    E = simp(x, penal, E0, Emin)
    hs = mesh.h()
    out = np.zeros(mesh.n_dof)
    for hval in np.unique(hs):
        K0 = element_stiffness(mesh.dim, 1.0, nu, float(hval))
        sel = np.nonzero(hs == hval)[0]
        for i0 in range(0, sel.shape[0], chunk):
            es = sel[i0:i0 + chunk]
            dd = dofs[es]
            ye = E[es][:, None] * (w[dd] @ K0.T)
            out += np.bincount(dd.ravel(), weights=ye.ravel(), minlength=mesh.n_dof)
    return out


def apply_full(mesh: OracleMesh, x, v, penal, E0=1.0, Emin=1e-9, nu=0.3) -> np.ndarray:
    """A v for the projected operator (Eq. 8 + Dirichlet rows)."""
    F = free_mask(mesh)
    C = constraint_matrix(mesh)
    vF = np.where(F, v, 0.0)
    Kw = stiffness_apply(mesh, x, C @ vF, penal, E0, Emin, nu)
    return np.where(F, C.T @ Kw, v)


def rhs(mesh: OracleMesh) -> np.ndarray:
    """b = Pi_F C^T f (Eq. 7)."""
    F = free_mask(mesh)
    C = constraint_matrix(mesh)
    return np.where(F, C.T @ mesh.load, 0.0)


def residual_norm(mesh: OracleMesh, x, u, penal, E0=1.0, Emin=1e-9, nu=0.3) -> float:
    """||b - A u_hat|| / ||b||, u_hat = u with the hanging DOFs zeroed (they are
    the unit rows of A, whose rhs is 0)."""
    uhat = np.array(u, dtype=np.float64, copy=True)
    for c in range(mesh.dim):
        uhat[mesh.hang_node.astype(np.int64) * mesh.dim + c] = 0.0
    b = rhs(mesh)
    r = b - apply_full(mesh, x, uhat, penal, E0, Emin, nu)
    return float(np.linalg.norm(r) / np.linalg.norm(b))


def filter_rows(mesh: OracleMesh, rmin, x, val, elems, mode="sens") -> np.ndarray:
    """Eq. 5 ('sens') or the DENS average for the given elements, brute force."""
    c = mesh.centers()
    V = mesh.volumes()
    x = np.asarray(x, dtype=np.float64)
    val = np.asarray(val, dtype=np.float64)
    out = np.empty(len(elems))
    for k, e in enumerate(np.asarray(elems).tolist()):
        d2 = ((c - c[e]) ** 2).sum(axis=1)
        nb = np.nonzero(d2 < rmin * rmin)[0]
        H = rmin - np.sqrt(d2[nb])
        w = H * V[nb]
        if mode == "sens":
            out[k] = np.sum(w * x[nb] * val[nb]) / (x[e] * np.sum(w))
        else:
            out[k] = np.sum(w * val[nb]) / np.sum(w)
    return out
