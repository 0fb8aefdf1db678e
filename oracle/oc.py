"""ORACLE (test infrastructure only) — the design update and the Fig. 1 loop.

OC update.  PAPER.md:350-354 (§3): "In the next step, we compute an update of
the design variables ... we use Optimality Criteria (OC), a simple approach
based on a set of intuitive criteria [BendsoeBk2003, Bendsoe1988]"; also
:586-587 (§6).  The formula itself is not printed.  Reading R18 (
the standard heuristic form SPEC.md:349-357, constants SPEC.md:376):

  B_e(lam) = max(-dc_e, 0) / (lam V_e)        (d vol / d x_e = V_e, Eq. 1)
  x_e(lam) = min(hi_e, max(lo_e, x_e B_e(lam)^eta))
  lo_e     = max(rho_o, x_e - move),  hi_e = min(1, x_e + move)

with rho_o the density lower bound ("typically 10^-3"),
move = 0.2 and eta = 1/2, and the volume multiplier lam chosen so that
vol(lam) = sum_e V_e x_e(lam) equals the target V0 sum_e V_e (the volume
constraint of Eq. 1, with V0 a fraction, :309).
vol(lam) is non-increasing in lam; lam is found by bisection (reading R18):

  vol_0 = lim_{lam->0+} vol(lam) = sum_e V_e (dc_e < 0 ? hi_e : lo_e)
  if vol_0 <= target: the constraint is inactive, lam = 0, x_new = that limit
  l1 = 0, l2 = lam_hi;  while vol(l2) > target and l2 < 1e300: l2 *= 1e3
  repeat  lm = (l1 + l2) / 2;  vol(lm) > target ? l1 = lm : l2 = lm
  until   l2 - l1 <= tol (l1 + l2)  or  max_steps bisections
  lam = (l1 + l2) / 2,  x_new = x(lam)

Design change (Condition 1): max_e |x_new_e - x_e|,
converged when < 0.01 (strict).

Fig. 1 loop: solve K(x)u = f -> sensitivities -> filter
(Eq. 5) -> OC update -> convergence check, with p-continuation (PAPER.md:
331-333: "start with p = 1 and slowly increase p as the design converges";
schedule reading R19: p += 0.5 up to p_max when the change is < 0.01 or
after `stage_steps` steps at the current p).  The solve here is
the direct sparse solve of the projected system (the plain definition
u* = C A^-1 b); mesh adaptation is out of scope.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse.linalg as spla

from . import fe, topopt
from .mesh import OracleMesh

RHO_O = 1e-3
MOVE = 0.2        # SPEC.md:376 (reading R18)
ETA = 0.5         # SPEC.md:376 (reading R18)
LAM_HI = 1e9      # initial upper bracket (SPEC.md:322 lambda_bracket)
TOL = 1e-12       # relative bisection tolerance on lam (reading R18)
MAX_STEPS = 200


@dataclass
class OCResult:
    x: np.ndarray
    lam: float
    steps: int          # bisections + bracket widenings
    volume: float       # sum V x_new / sum V
    change: float       # max |x_new - x|
    status: str         # 'active' | 'inactive' | 'infeasible'


def oc_candidate(x, dc, V, lam, move=MOVE, eta=ETA, rho_o=RHO_O):
    """x_e(lam) of reading R18, elementwise, as written above."""
    lo = np.maximum(rho_o, x - move)
    hi = np.minimum(1.0, x + move)
    B = np.maximum(-dc, 0.0) / (lam * V)
    return np.minimum(hi, np.maximum(lo, x * B ** eta))


def oc_update(x, dc, V, volfrac, move=MOVE, eta=ETA, rho_o=RHO_O, lam_hi=LAM_HI, tol=TOL,
              max_steps=MAX_STEPS) -> OCResult:
    x = np.asarray(x, dtype=np.float64)
    dc = np.asarray(dc, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    Vtot = V.sum()
    target = volfrac * Vtot
    lo = np.maximum(rho_o, x - move)
    hi = np.minimum(1.0, x + move)
    x0 = np.where(dc < 0.0, hi, lo)
    if np.sum(V * x0) <= target:
        return OCResult(x0, 0.0, 0, float(np.sum(V * x0) / Vtot), float(np.max(np.abs(x0 - x))), "inactive")

    def vol(lam):
        return np.sum(V * oc_candidate(x, dc, V, lam, move, eta, rho_o))

    steps = 0
    l1, l2 = 0.0, lam_hi
    while vol(l2) > target and l2 < 1e300:
        l2 *= 1e3
        steps += 1
    status = "active" if vol(l2) <= target else "infeasible"
    nb = 0
    while status == "active" and nb < max_steps and not (l2 - l1 <= tol * (l1 + l2)):
        lm = 0.5 * (l1 + l2)
        if vol(lm) > target:
            l1 = lm
        else:
            l2 = lm
        nb += 1
    lam = 0.5 * (l1 + l2) if status == "active" else l2
    xn = oc_candidate(x, dc, V, lam, move, eta, rho_o)
    return OCResult(xn, float(lam), steps + nb, float(np.sum(V * xn) / Vtot), float(np.max(np.abs(xn - x))), status)


def converged(change, tol=0.01) -> bool:
    """Condition 1, strict."""
    return change < tol


@dataclass
class LoopHistory:
    compliance: list = field(default_factory=list)
    penal: list = field(default_factory=list)
    volume: list = field(default_factory=list)
    change: list = field(default_factory=list)
    lam: list = field(default_factory=list)


def solve_u(mesh: OracleMesh, x, penal, E0=1.0, Emin=1e-9, nu=0.3):
    """u* = C A^-1 b (Eqs. 7-9), direct sparse solve."""
    K = fe.assemble_K(mesh, x, penal, E0, Emin, nu)
    A, b, C = fe.projected_system(mesh, K)
    uhat = spla.spsolve(A.tocsc(), b)
    return fe.recover(C, uhat)


def optimize(mesh: OracleMesh, x0, volfrac, n_steps, rmin, penal0=1.0, penal_max=3.0, penal_step=0.5,
             stage_steps=30, E0=1.0, Emin=1e-9, nu=0.3, move=MOVE, eta=ETA, rho_o=RHO_O,
             stop_on_converge=False, change_tol=0.01):
    """The Fig. 1 loop on a fixed mesh for n_steps design updates (or until
    converged at penal_max when stop_on_converge)."""
    x = np.asarray(x0, dtype=np.float64).copy()
    V = mesh.volumes()
    H = LoopHistory()
    penal, at_stage = penal0, 0
    for _ in range(n_steps):
        u = solve_u(mesh, x, penal, E0, Emin, nu)
        c = fe.compliance(mesh.load, u)
        dc = topopt.sensitivities(mesh, x, u, penal, E0, Emin, nu)
        if rmin > 0:
            dc = topopt.filter_sens(mesh, rmin, x, dc)
        r = oc_update(x, dc, V, volfrac, move, eta, rho_o)
        H.compliance.append(c)
        H.penal.append(penal)
        H.volume.append(r.volume)
        H.change.append(r.change)
        H.lam.append(r.lam)
        x = r.x
        at_stage += 1
        if stop_on_converge and penal >= penal_max and converged(r.change, change_tol):
            break
        if penal < penal_max and (converged(r.change, change_tol) or at_stage >= stage_steps):
            penal, at_stage = min(penal_max, penal + penal_step), 0
    return x, H
