"""ORACLE (test infrastructure only) — the paper's own solver (§5).

The systems are solved on the explicitly rescaled matrix
  K~ = D^-1/2 K D^-1/2,  D = diag(K)              (:511-523)
with an incomplete Cholesky factor of zero fill-in,
  K~ ~ L~ L~^T                                    (:524-530),
by (preconditioned) MINRES (:541-551; recycling, RMINRES, is out of scope:
its algorithm lives in another paper).  Here K is the projected operator A
of Eq. 8 with Dirichlet rows (reading R5), so D = diag(A) (reading R4).

ic0(A)        IC(0) of a sparse SPD matrix, row by row in the textbook
              order: for row i and each k < i in the pattern of row i,
                L_ik = (A_ik - sum_{j<k} L_ij L_kj) / L_kk,
                L_ii = sqrt(A_ii - sum_{k<i} L_ik^2),
              with every product that would land outside the pattern of
              tril(A) dropped (zero fill-in).  A non-positive pivot raises.
ic0_shifted   elasticity matrices are not M-matrices and IC(0) of K~ can
              break down; reading R24: Manteuffel's shifted IC(0), the factor
              of K~ + a I (K~ has a unit diagonal) with a = 0, then
              1e-3 * 2^t, t = 0, 1, ... until every pivot is positive.
minres(...)   preconditioned MINRES in the Lanczos / Givens form of Paige and
              Saunders (as laid out in Elman, Silvester & Wathen, Alg. 2.4):
              z_j = M^-1 v_j normalised by gamma_j = sqrt(<z_j, v_j>); the QR
              factorisation of the tridiagonal Lanczos matrix by Givens
              rotations gives the update directions w_j and |eta|, the
              M^-1-norm of the residual, which is non-increasing.
              Stops when |eta| <= rtol |eta_0|.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp


def ic0(A) -> sp.csr_matrix:
    """Lower-triangular IC(0) factor (CSR, diagonal last in every row)."""
    T = sp.tril(sp.csr_matrix(A), format="csr")
    T.sort_indices()
    n = T.shape[0]
    ptr, idx, val = T.indptr, T.indices, T.data.astype(np.float64)
    L = val.copy()
    rows = [dict() for _ in range(n)]          # row i: column -> position, for the pattern test
    for i in range(n):
        for t in range(ptr[i], ptr[i + 1]):
            rows[i][idx[t]] = t
    for i in range(n):
        a, b = ptr[i], ptr[i + 1]
        if b == a or idx[b - 1] != i:
            raise ValueError(f"row {i}: structurally zero diagonal")
        for t in range(a, b - 1):               # off-diagonal k = idx[t] < i, ascending
            k = idx[t]
            acc = L[t]
            for u in range(a, t):               # j < k in row i, and (k, j) in the pattern
                j = idx[u]
                pk = rows[k].get(j)
                if pk is not None:
                    acc -= L[u] * L[pk]
            L[t] = acc / L[ptr[k + 1] - 1]
        d = L[b - 1]
        for u in range(a, b - 1):
            d -= L[u] * L[u]
        if not (d > 0.0):
            raise ArithmeticError(f"IC(0): non-positive pivot {d} in row {i}")
        L[b - 1] = np.sqrt(d)
    return sp.csr_matrix((L, idx.copy(), ptr.copy()), shape=(n, n))


def ic0_shifted(A, max_tries=30):
    """IC(0) of A + a I with the smallest a in {0, 1e-3 2^t} that succeeds; returns (L, a)."""
    A = sp.csr_matrix(A)
    n = A.shape[0]
    for t in range(-1, max_tries):
        a = 0.0 if t < 0 else 1e-3 * 2.0 ** t
        try:
            return ic0(A + a * sp.eye(n, format="csr") if a > 0 else A), a
        except ArithmeticError:
            continue
    raise ArithmeticError("IC(0) breaks down for every shift tried")


def ic0_solve(L: sp.csr_matrix, r: np.ndarray) -> np.ndarray:
    """(L L^T)^-1 r by a forward and a backward substitution."""
    from scipy.sparse.linalg import spsolve_triangular
    y = spsolve_triangular(L, r, lower=True)
    return spsolve_triangular(sp.csr_matrix(L.T), y, lower=False)


@dataclass
class MinresResult:
    x: np.ndarray
    iters: int
    eta: list = field(default_factory=list)      # |eta_j|, the M^-1-norm of the residual, j = 0..iters
    converged: bool = False


def minres(A, b, msolve=None, x0=None, rtol=1e-10, max_iter=10000) -> MinresResult:
    """Preconditioned MINRES (ESW Alg. 2.4).  msolve(v) = M^-1 v (identity if None)."""
    n = b.shape[0]
    ms = (lambda v: v.copy()) if msolve is None else msolve
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    v_old = np.zeros(n)
    v = b - A @ x
    z = ms(v)
    gamma = np.sqrt(float(z @ v))
    res = MinresResult(x, 0, [gamma])
    if gamma == 0.0:
        res.converged = True
        return res
    eta = gamma
    s_old = s = 0.0
    c_old = c = 1.0
    gamma_old = 1.0
    w_old = np.zeros(n)
    w = np.zeros(n)
    for j in range(1, max_iter + 1):
        z = z / gamma
        Az = A @ z
        delta = float(Az @ z)
        v_new = Az - (delta / gamma) * v - (gamma / gamma_old) * v_old
        z_new = ms(v_new)
        gamma_new = np.sqrt(max(float(z_new @ v_new), 0.0))
        a0 = c * delta - c_old * s * gamma
        a1 = np.sqrt(a0 * a0 + gamma_new * gamma_new)
        a2 = s * delta + c_old * c * gamma
        a3 = s_old * gamma
        c_new, s_new = a0 / a1, gamma_new / a1
        w_new = (z - a3 * w_old - a2 * w) / a1
        x = x + c_new * eta * w_new
        eta = -s_new * eta
        res.eta.append(abs(eta))
        res.iters = j
        v_old, v = v, v_new
        z = z_new
        gamma_old, gamma = gamma, gamma_new
        w_old, w = w, w_new
        c_old, c = c, c_new
        s_old, s = s, s_new
        if abs(eta) <= rtol * res.eta[0] or gamma == 0.0:
            res.converged = True
            break
    res.x = x
    return res


def rescale(A, b):
    """K~ = D^-1/2 A D^-1/2, b~ = D^-1/2 b (:511-523); returns (K~, b~, d^-1/2)."""
    d = np.asarray(sp.csr_matrix(A).diagonal(), dtype=np.float64)
    if np.any(d <= 0):
        raise ArithmeticError("non-positive diagonal")
    s = 1.0 / np.sqrt(d)
    S = sp.diags(s)
    Kt = sp.csr_matrix(S @ A @ S)
    Kt.eliminate_zeros()      # the IC(0) pattern is the nonzero structure (explicit zeros of the projection dropped)
    return Kt, s * b, s


def solve_paper(A, b, rtol=1e-10, max_iter=10000, precond="ic0"):
    """MINRES on the rescaled system, preconditioned by IC(0) of K~ ('ic0') or
    not at all ('none', i.e. Jacobi on A).  Returns (u, MinresResult)."""
    Kt, bt, s = rescale(A, b)
    ms = None
    shift = None
    if precond == "ic0":
        L, shift = ic0_shifted(Kt)
        ms = lambda v: ic0_solve(L, v)   # noqa: E731
    r = minres(Kt, bt, ms, rtol=rtol, max_iter=max_iter)
    r.shift = shift
    return s * r.x, r
