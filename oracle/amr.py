"""ORACLE (test infrastructure only) — the dynamic AMR strategy of §4
 around the Fig. 1 loop.

Trigger (reading R23): adapt after a design step when
  CASE (i)  the design change max|dx| < change_tol (0.01, "Condition 1 ...
            the maximum change in the design variables is smaller than a
            certain tolerance (which we usually set to 0.01)") and at least
            min_steps (5) steps were taken since the last adaptation, or
  CASE (ii) max_steps (10) steps were taken since the last adaptation.

Marking (reading R21): element e is solid when x_e >= rho_s
(rho_s = 0.5).  e is marked for refinement when a solid element d lies
within r_amr of it, dist(c_d, c_e) < r_amr between element centres (the
filter's neighbourhood, r_amr = rmin as in PAPER.md:606-607; strict, as C9),
d = e included; otherwise (void with no solid element within r_amr) for
derefinement.  Refinement stops at the finest lattice level L, derefinement
at level 0.

Compatibility sweeps (reading R22):
  sweep 1  a derefinement mark survives only if every sibling (the 2^d
           children of the parent) is a leaf marked for derefinement;
  sweep 2  a sibling group survives only if no leaf of level >= l + 1 (l the
           siblings' level) touches the parent across a face or an edge in 3D,
           an edge in 2D (the C10 adjacency) — "level two or higher edge
           incompatibility" — in the mesh after this pass's refinements and
           their 2:1 closure (so the final balance never has to re-refine a
           derefined parent).

Mesh update: refined leaves are replaced by their 2^d children, which inherit
the density; derefined groups by the parent, whose density is the mean of the
children's (equal volumes: the volume-weighted mean), summed in corner order
c = cx + 2cy + 4cz.  The new pre-balance leaf set then goes through the same
2:1 balance and numbering as any mesh (mesh.build_mesh); a leaf split by the
balance inherits the density of the pre-balance leaf containing it.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from inputs import Problem
from . import fe, mesh as omesh, oc, topopt
from .mesh import OracleMesh, _dirs, morton

RHO_S = 0.5      # reading R21 (the Costa-Alves "density 0.5 or larger")
MIN_STEPS = 5
MAX_STEPS = 10


def should_adapt(change, since, change_tol=0.01, min_steps=MIN_STEPS, max_steps=MAX_STEPS) -> bool:
    return (change < change_tol and since >= min_steps) or since >= max_steps


def mark(mesh: OracleMesh, x, rho_s=RHO_S, r_amr=None) -> np.ndarray:
    """+1 refine, -1 derefine, 0 neither (capped at levels L and 0), int8 per element."""
    x = np.asarray(x, dtype=np.float64)
    solid = x >= rho_s
    if r_amr is None or r_amr <= 0:
        near = solid.copy()
    else:
        ptr, idx = omesh.filter_neighbours(mesh, r_amr)
        near = np.array([bool(solid[idx[ptr[e]:ptr[e + 1]]].any()) for e in range(mesh.n_el)])
    m = np.where(near, 1, -1).astype(np.int8)
    m[(m == 1) & (mesh.elem_level.astype(np.int64) >= mesh.L)] = 0
    m[(m == -1) & (mesh.elem_level.astype(np.int64) == 0)] = 0
    return m


def _corner_offsets(dim):
    return [np.array([(c >> k) & 1 for k in range(dim)], dtype=np.int64) for c in range(1 << dim)]


@dataclass
class AdaptResult:
    leaf_level: np.ndarray      # int8 [n]  pre-balance leaves (refined / derefined / kept), sorted by Morton key
    leaf_anchor: np.ndarray     # int32 [n, dim]
    leaf_x: np.ndarray          # float64 [n]
    marks: np.ndarray           # int8 per old element after the sweeps
    n_refined: int = 0
    n_groups: int = 0
    n_unmarked_sibling: int = 0
    n_unmarked_incompat: int = 0


def sweeps(mesh: OracleMesh, marks) -> tuple:
    """Sweeps 1 and 2 on the marks; returns (marks, n_unmarked_sibling, n_unmarked_incompat)."""
    dim, L = mesh.dim, mesh.L
    lev = mesh.elem_level.astype(np.int64)
    anc = mesh.elem_anchor.astype(np.int64)
    m = np.asarray(marks, dtype=np.int8).copy()
    where = {(int(lev[e]), tuple(int(v) for v in anc[e])): e for e in range(mesh.n_el)}
    offs = _corner_offsets(dim)

    def group(e):
        s = 1 << (L - lev[e])
        pa = (anc[e] // (2 * s)) * (2 * s)
        return pa, [where.get((int(lev[e]), tuple(int(v) for v in pa + o * s))) for o in offs]

    # sweep 1: siblings
    n1 = 0
    m1 = m.copy()
    for e in np.nonzero(m == -1)[0]:
        _, sib = group(e)
        if any(d is None or m[d] != -1 for d in sib):
            m1[e] = 0
            n1 += 1
    m = m1
    # sweep 2: level-two incompatibility around the would-be parent, judged on
    # the mesh after this pass's refinements and their 2:1 closure (C10)
    ext = np.array(_extent(mesh), dtype=np.int64)
    rl, ra = [], []
    for e in range(mesh.n_el):
        if m[e] == 1:
            s = 1 << (L - lev[e])
            for o in offs:
                rl.append(lev[e] + 1)
                ra.append(anc[e] + o * (s // 2))
        else:
            rl.append(lev[e])
            ra.append(anc[e])
    box = _Box(dim, L, tuple(int(v) for v in ext))
    cl, ca = omesh.balance(box, np.array(rl, dtype=np.int64), np.array(ra, dtype=np.int64).reshape(-1, dim))
    cl = cl.astype(np.int64)
    ca = ca.astype(np.int64)
    order = np.argsort(morton(ca), kind="stable")
    cl, ca = cl[order], ca[order]
    keys = morton(ca)
    n2 = 0
    done = set()
    for e in np.nonzero(m == -1)[0]:
        pa, sib = group(e)
        gk = (int(lev[e]), tuple(int(v) for v in pa))
        if gk in done:
            continue
        done.add(gk)
        l = int(lev[e])
        bad = False
        if l < L:
            S = 2 * (1 << (L - l))         # parent edge in lattice units
            t = (1 << (L - l)) // 2        # edge of a level-(l+1) cell
            for dv in _dirs(dim):
                rng = []
                for c in range(dim):
                    if dv[c] < 0:
                        rng.append([pa[c] - t])
                    elif dv[c] > 0:
                        rng.append([pa[c] + S])
                    else:
                        rng.append(list(range(int(pa[c]), int(pa[c] + S), t)))
                for q in _product(rng):
                    q = np.array(q, dtype=np.int64)
                    if np.any(q < 0) or np.any(q >= ext):
                        continue
                    j = int(np.searchsorted(keys, morton(q[None, :]), side="right")[0]) - 1
                    if cl[j] >= l + 1:
                        bad = True
                        break
                if bad:
                    break
        if bad:
            for d in sib:
                if m[d] == -1:
                    m[d] = 0
                    n2 += 1
    return m, n1, n2


@dataclass
class _Box:
    """What mesh.balance needs to know about the domain."""
    dim: int
    L: int
    lattice_extent: tuple


def _product(lists):
    out = [[]]
    for lst in lists:
        out = [p + [v] for p in out for v in lst]
    return out


def _extent(mesh: OracleMesh):
    """Lattice extent of the box (max over leaves of anchor + size)."""
    s = 1 << (mesh.L - mesh.elem_level.astype(np.int64))
    return tuple(int(v) for v in (mesh.elem_anchor.astype(np.int64) + s[:, None]).max(axis=0))


def adapt(mesh: OracleMesh, x, marks) -> AdaptResult:
    """Sweeps, then the new pre-balance leaf set with transferred densities."""
    dim, L = mesh.dim, mesh.L
    x = np.asarray(x, dtype=np.float64)
    m, n1, n2 = sweeps(mesh, marks)
    lev = mesh.elem_level.astype(np.int64)
    anc = mesh.elem_anchor.astype(np.int64)
    offs = _corner_offsets(dim)
    where = {(int(lev[e]), tuple(int(v) for v in anc[e])): e for e in range(mesh.n_el)}
    out_l, out_a, out_x = [], [], []
    nref = ngrp = 0
    for e in range(mesh.n_el):
        s = 1 << (L - lev[e])
        if m[e] == 1:
            nref += 1
            for o in offs:
                out_l.append(lev[e] + 1)
                out_a.append(anc[e] + o * (s // 2))
                out_x.append(x[e])
        elif m[e] == -1:
            pa = (anc[e] // (2 * s)) * (2 * s)
            if np.array_equal(pa, anc[e]):              # emit the parent once, from corner 0
                sib = [where[(int(lev[e]), tuple(int(v) for v in pa + o * s))] for o in offs]
                acc = 0.0
                for d in sib:                            # corner order
                    acc += x[d]
                ngrp += 1
                out_l.append(lev[e] - 1)
                out_a.append(pa)
                out_x.append(acc / len(sib))
        else:
            out_l.append(lev[e])
            out_a.append(anc[e])
            out_x.append(x[e])
    nl = np.array(out_l, dtype=np.int64)
    na = np.array(out_a, dtype=np.int64).reshape(-1, dim)
    nx = np.array(out_x, dtype=np.float64)
    order = np.argsort(morton(na), kind="stable")
    return AdaptResult(nl[order].astype(np.int8), na[order].astype(np.int32), nx[order], m,
                       nref, ngrp, n1, n2)


def transfer(new_mesh: OracleMesh, res: AdaptResult) -> np.ndarray:
    """Density of each (balanced) new leaf = that of the pre-balance leaf containing it."""
    keys = morton(res.leaf_anchor.astype(np.int64))
    j = np.searchsorted(keys, morton(new_mesh.elem_anchor.astype(np.int64)), side="right") - 1
    return res.leaf_x[j].copy()


def rebuild(prob: Problem, res: AdaptResult, with_filter=True) -> OracleMesh:
    p2 = replace(prob, leaf_level=res.leaf_level, leaf_anchor=res.leaf_anchor)
    return omesh.build_mesh(p2, with_filter=with_filter, density=False)


@dataclass
class AmrHistory:
    compliance: list = field(default_factory=list)
    penal: list = field(default_factory=list)
    volume: list = field(default_factory=list)
    change: list = field(default_factory=list)
    n_elem: list = field(default_factory=list)
    adapted: list = field(default_factory=list)


def optimize_amr(prob: Problem, volfrac, n_steps, penal0=1.0, penal_max=3.0, penal_step=0.5, stage_steps=30,
                 rho_s=RHO_S, min_steps=MIN_STEPS, max_steps=MAX_STEPS, change_tol=0.01, x0=None):
    """Fig. 1 with dynamic AMR: per step solve -> sensitivities -> Eq. 5 filter
    -> OC (oc.py) -> continuation; then the adaptation trigger, marking (r_amr =
    rmin), sweeps, mesh update and density transfer.  Returns the final mesh,
    x and the history."""
    mesh = omesh.build_mesh(prob, density=False)
    x = np.full(mesh.n_el, volfrac) if x0 is None else np.asarray(x0, dtype=np.float64).copy()
    H = AmrHistory()
    penal, at_stage, since = penal0, 0, 0
    for _ in range(n_steps):
        V = mesh.volumes()
        u = oc.solve_u(mesh, x, penal, prob.E0, prob.Emin, prob.nu)
        c = fe.compliance(mesh.load, u)
        dc = topopt.sensitivities(mesh, x, u, penal, prob.E0, prob.Emin, prob.nu)
        if prob.rmin > 0:
            dc = topopt.filter_sens(mesh, prob.rmin, x, dc)
        r = oc.oc_update(x, dc, V, volfrac)
        H.compliance.append(c)
        H.penal.append(penal)
        H.volume.append(r.volume)
        H.change.append(r.change)
        H.n_elem.append(mesh.n_el)
        x = r.x
        at_stage += 1
        since += 1
        if penal < penal_max and (oc.converged(r.change, change_tol) or at_stage >= stage_steps):
            penal, at_stage = min(penal_max, penal + penal_step), 0
        adapted = False
        if should_adapt(r.change, since, change_tol, min_steps, max_steps):
            res = adapt(mesh, x, mark(mesh, x, rho_s, prob.rmin))
            mesh = rebuild(prob, res)
            x = transfer(mesh, res)
            since, adapted = 0, True
        H.adapted.append(adapted)
    return mesh, x, H
