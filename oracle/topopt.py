"""ORACLE (test infrastructure only) — sensitivities and filters.

Sensitivity (the formula is not printed, SURVEY Q2 /
SPEC.md:332): dc_e = -p x_e^(p-1) (E0 - E_min) u_e^T K0(h_e) u_e, where
u_e is the element gather of the recovered u = C u_hat (so hanging corners
carry their interpolated values).

Filter:
  Eq. 4  H_de = max(rmin - dist(d, e), 0), dist between element centres;
  Eq. 5  out_e = sum_d x_d H_de V_d dc_d / (x_e sum_d H_de V_d)  ('sens');
  'dens': out_e = sum_d H_de V_d in_d / sum_d H_de V_d.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .fe import element_stiffness, element_dofs
from .mesh import OracleMesh


def element_energy(mesh: OracleMesh, u: np.ndarray, nu=0.3, elems=None) -> np.ndarray:
    """u_e^T K0(h_e) u_e with unit modulus."""
    dofs = element_dofs(mesh)
    hs = mesh.h()
    if elems is None:
        elems = np.arange(mesh.n_el)
    elems = np.asarray(elems, dtype=np.int64)
    out = np.zeros(elems.shape[0])
    for hval in np.unique(hs[elems]):
        K0 = element_stiffness(mesh.dim, 1.0, nu, float(hval))
        m = hs[elems] == hval
        ue = u[dofs[elems[m]]]
        out[m] = np.einsum("ea,ab,eb->e", ue, K0, ue)
    return out


def sensitivities(mesh: OracleMesh, x, u, penal, E0=1.0, Emin=1e-9, nu=0.3, elems=None):
    x = np.asarray(x, dtype=np.float64)
    if elems is None:
        xe = x
    else:
        xe = x[np.asarray(elems)]
    return -penal * xe ** (penal - 1.0) * (E0 - Emin) * element_energy(mesh, u, nu, elems)


def filter_weights(mesh: OracleMesh, rmin: float) -> sp.csr_matrix:
    """W[e, d] = H_de V_d over the neighbour lists (C9)."""
    c = mesh.centers()
    V = mesh.volumes()
    ptr, idx = mesh.filt_ptr, mesh.filt_idx.astype(np.int64)
    rows = np.repeat(np.arange(mesh.n_el), np.diff(ptr))
    dist = np.sqrt(((c[idx] - c[rows]) ** 2).sum(axis=1))
    H = np.maximum(rmin - dist, 0.0)
    return sp.csr_matrix((H * V[idx], (rows, idx)), shape=(mesh.n_el, mesh.n_el))


def filter_sens(mesh: OracleMesh, rmin, x, dc):
    W = filter_weights(mesh, rmin)
    x = np.asarray(x, dtype=np.float64)
    return (W @ (x * dc)) / (x * np.asarray(W.sum(axis=1)).ravel())


def filter_dens(mesh: OracleMesh, rmin, v):
    W = filter_weights(mesh, rmin)
    return (W @ v) / np.asarray(W.sum(axis=1)).ravel()


def filter_bruteforce(mesh: OracleMesh, rmin, x, val, mode="sens"):
    """Direct double loop over all pairs (tiny meshes)."""
    c = mesh.centers()
    V = mesh.volumes()
    n = mesh.n_el
    out = np.zeros(n)
    for e in range(n):
        num = 0.0
        den = 0.0
        for d in range(n):
            H = max(rmin - np.sqrt(((c[d] - c[e]) ** 2).sum()), 0.0)
            if mode == "sens":
                num += x[d] * H * V[d] * val[d]
            else:
                num += H * V[d] * val[d]
            den += H * V[d]
        out[e] = num / (x[e] * den) if mode == "sens" else num / den
    return out
