"""ORACLE (test infrastructure only) — linear solvers.

The paper rescales K symmetrically so that its diagonal is 1
(K~ = D^-1/2 K D^-1/2) and runs (R)MINRES with IC(0).
This build's hot path runs CG on that rescaled system without IC(0)
(SURVEY Q3), which in exact arithmetic is Jacobi-preconditioned CG on A.
`pcg_jacobi` is the textbook Hestenes-Stiefel recurrence;
`cg_rescaled` runs plain CG on the explicitly rescaled matrix (pin P10).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp


@dataclass
class CGResult:
    x: np.ndarray
    iters: int
    relres: float              # recurrence residual ||r_k|| / ||b||
    relres_true: float         # ||b - A x|| / ||b||
    converged: bool
    alphas: list = field(default_factory=list)
    betas: list = field(default_factory=list)
    history: list = field(default_factory=list)


def pcg_jacobi(A, b, rtol=1e-10, max_iter=100000, x0=None, fixed_iters=None, record=False):
    """Jacobi-PCG on A x = b, stopping when ||r_k||_2 / ||b||_2 <= rtol
    (SURVEY Q9), or after exactly `fixed_iters` iterations."""
    n = b.shape[0]
    dinv = 1.0 / A.diagonal()
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    r = b - A @ x if x0 is not None else b.copy()
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return CGResult(np.zeros(n), 0, 0.0, 0.0, True)
    z = dinv * r
    p = z.copy()
    rho = float(r @ z)
    res = CGResult(x, 0, np.linalg.norm(r) / bnorm, 0.0, False)
    k = 0
    limit = fixed_iters if fixed_iters is not None else max_iter
    while k < limit:
        if fixed_iters is None and np.linalg.norm(r) / bnorm <= rtol:
            break
        q = A @ p
        pq = float(p @ q)
        if not pq > 0.0:
            raise FloatingPointError("CG breakdown: p^T A p <= 0")
        alpha = rho / pq
        x += alpha * p
        r -= alpha * q
        z = dinv * r
        rho_new = float(r @ z)
        beta = rho_new / rho
        p = z + beta * p
        rho = rho_new
        k += 1
        if record:
            res.alphas.append(alpha)
            res.betas.append(beta)
            res.history.append(np.linalg.norm(r) / bnorm)
    res.x = x
    res.iters = k
    res.relres = float(np.linalg.norm(r) / bnorm)
    res.relres_true = float(np.linalg.norm(b - A @ x) / bnorm)
    res.converged = res.relres <= rtol
    return res


def cg_rescaled(A, b, iters):
    """Plain CG on K~ = D^-1/2 A D^-1/2, x = D^-1/2 x~."""
    d = A.diagonal()
    s = 1.0 / np.sqrt(d)
    S = sp.diags(s)
    At = (S @ A @ S).tocsr()
    bt = s * b
    x = np.zeros_like(b)
    r = bt.copy()
    p = r.copy()
    rr = float(r @ r)
    xs = []
    for _ in range(iters):
        q = At @ p
        alpha = rr / float(p @ q)
        x += alpha * p
        r -= alpha * q
        rr_new = float(r @ r)
        p = r + (rr_new / rr) * p
        rr = rr_new
        xs.append(s * x)
    return xs


def dense_solve(A, b):
    Ad = A.toarray() if sp.issparse(A) else np.asarray(A)
    return np.linalg.solve(Ad, b)
