"""ORACLE (test infrastructure only) — the whole hot path on one problem.

Plain definition: u* = C A^-1 b, c = f^T u*,
dc = sensitivities(u*), dc~ = Eq. 5 filter(x, dc).  Computed here with the
assembled matrices and the textbook Jacobi-PCG.
"""
from __future__ import annotations

from dataclasses import dataclass
import time

import numpy as np

from inputs import Problem
from . import fe, mesh as omesh, solve, topopt


@dataclass
class OracleResult:
    mesh: omesh.OracleMesh
    x: np.ndarray
    u: np.ndarray
    uhat: np.ndarray
    compliance: float
    dc: np.ndarray
    dc_filtered: np.ndarray
    cg: solve.CGResult
    A: object
    b: np.ndarray
    timings: dict


def input_density(prob: Problem, m: omesh.OracleMesh) -> np.ndarray:
    """Input x: the raw field, plus one DENS pass when the config asks for it (c3)."""
    x = m.density.copy()
    if prob.presmooth_rmin is not None:
        if prob.presmooth_rmin != prob.rmin:
            raise NotImplementedError
        x = topopt.filter_dens(m, prob.presmooth_rmin, x)
    return x


def run(prob: Problem, rtol=None, fixed_iters=None, m=None, x=None, record=False) -> OracleResult:
    t = {}
    t0 = time.perf_counter()
    if m is None:
        m = omesh.build_mesh(prob)
    t["mesh"] = time.perf_counter() - t0
    if x is None:
        x = input_density(prob, m)
    t0 = time.perf_counter()
    K = fe.assemble_K(m, x, prob.penal, prob.E0, prob.Emin, prob.nu)
    A, b, C = fe.projected_system(m, K)
    t["assembly"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    cg = solve.pcg_jacobi(A, b, rtol=prob.rtol if rtol is None else rtol,
                          max_iter=prob.max_iter, fixed_iters=fixed_iters, record=record)
    t["cg"] = time.perf_counter() - t0
    u = fe.recover(C, cg.x)
    c = fe.compliance(m.load, u)
    t0 = time.perf_counter()
    dc = topopt.sensitivities(m, x, u, prob.penal, prob.E0, prob.Emin, prob.nu)
    t["sens"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    dcf = topopt.filter_sens(m, prob.rmin, x, dc)
    t["filter"] = time.perf_counter() - t0
    return OracleResult(m, x, u, cg.x, c, dc, dcf, cg, A, b, t)
