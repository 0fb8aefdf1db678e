"""Problem definitions and seeded generators (shared input, no method arithmetic).

Conventions:

* The domain is a box of ``base`` level-0 cells of edge ``h0``.  The finest
  lattice is level ``L``: lattice unit ``h_L = h0 / 2**L``.  A leaf has a
  level ``l`` and an integer anchor ``a`` (its minimum corner on the finest
  lattice, a multiple of ``2**(L-l)``); its size is ``s = 2**(L-l)`` lattice
  units.
* Boundary conditions are geometric predicates on lattice coordinates
  (inclusive boxes); loads are point loads, line loads (intensity per unit
  length along a domain-boundary segment) or face tractions (per unit area
  on a domain-boundary rectangle).  Turning them into nodal values is the
  consumer's job (C7, C8).
* Random draws use ``numpy.random.default_rng(seed)`` in the order stated in
  SURVEY.md §8(d); per-element i.i.d. draws are made in lexicographic
  element order (x fastest) on the uniform grid.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np


@dataclass
class DensitySpec:
    kind: str                       # 'const' | 'iid' | 'gauss'
    value: float = 0.5              # const
    lo: float = 0.0                 # iid: U(lo, hi)
    hi: float = 1.0
    seed: int = 0
    n_gauss: int = 0                # gauss: sum of n isotropic Gaussians
    width_lo: float = 0.02          # widths U(width_lo, width_hi) * extent[0]
    width_hi: float = 0.1
    thr: float = 0.5                # rho = clip(sigmoid(k (g - thr)), clip_lo, 1)
    k: float = 20.0
    clip_lo: float = 1e-3


@dataclass
class Problem:
    name: str
    dim: int
    L: int
    base: tuple
    h0: float
    leaf_level: np.ndarray          # int8 [n]   pre-balance leaf set (C11)
    leaf_anchor: np.ndarray         # int32 [n, dim]
    density: DensitySpec
    fixed: list                     # [(lo, hi, mask)] lattice boxes, mask bit c = component c
    loads: list                     # [(kind, lo, hi, vec)] kind in point|line|face
    E0: float = 1.0
    Emin: float = 1e-9
    nu: float = 0.3
    penal: float = 3.0
    rmin: float = 1.5               # physical filter radius
    rtol: float = 1e-10
    max_iter: int = 20000
    fixed_iters: Optional[int] = None
    presmooth_rmin: Optional[float] = None   # c3: one DENS filter pass of the raw field
    notes: str = ""

    @property
    def hL(self) -> float:
        return self.h0 / (1 << self.L)

    @property
    def lattice_extent(self) -> tuple:
        return tuple(int(b) << self.L for b in self.base)


# ---------------------------------------------------------------------------
# leaf sets
# ---------------------------------------------------------------------------

def uniform_leaves(dim: int, base, L: int, level: int = 0):
    """All level-``level`` cells of the box (lexicographic order, x fastest)."""
    base = tuple(int(b) for b in base)
    n = [b << level for b in base]
    s = 1 << (L - level)
    grids = np.meshgrid(*[np.arange(k, dtype=np.int64) for k in n], indexing="ij")
    # lexicographic x fastest: flatten with axis 0 fastest -> use Fortran order
    coords = np.stack([g.ravel(order="F") for g in grids], axis=1) * s
    lev = np.full(coords.shape[0], level, dtype=np.int8)
    return lev, coords.astype(np.int32)


def leaf_centers(prob: Problem, level: np.ndarray, anchor: np.ndarray) -> np.ndarray:
    """Physical centers (a + s/2) h_L.  Pure geometry of the input."""
    s = (1 << (prob.L - level.astype(np.int64)))[:, None]
    return (anchor.astype(np.float64) + 0.5 * s) * prob.hL


def _gauss_params(spec: DensitySpec, dim: int, extent_phys):
    rng = np.random.default_rng(spec.seed)
    centers = rng.random((spec.n_gauss, dim)) * np.asarray(extent_phys, dtype=np.float64)
    widths = rng.uniform(spec.width_lo, spec.width_hi, spec.n_gauss) * float(extent_phys[0])
    return centers, widths


def _gauss_density(spec: DensitySpec, dim: int, extent_phys, pts: np.ndarray) -> np.ndarray:
    centers, widths = _gauss_params(spec, dim, extent_phys)
    out = np.empty(pts.shape[0], dtype=np.float64)
    chunk = 1 << 16
    inv2w2 = 1.0 / (2.0 * widths * widths)
    for i0 in range(0, pts.shape[0], chunk):
        p = pts[i0:i0 + chunk]
        d2 = np.zeros((p.shape[0], spec.n_gauss))
        for c in range(dim):
            d2 += (p[:, c:c + 1] - centers[None, :, c]) ** 2
        g = np.exp(-d2 * inv2w2[None, :]).sum(axis=1)
        rho = 1.0 / (1.0 + np.exp(-spec.k * (g - spec.thr)))
        out[i0:i0 + chunk] = np.clip(rho, spec.clip_lo, 1.0)
    return out


def raw_iid_field(prob: Problem) -> np.ndarray:
    """i.i.d. U(lo, hi) per finest-grid element, lexicographic order (x fastest)."""
    spec = prob.density
    n = int(np.prod(prob.lattice_extent))
    rng = np.random.default_rng(spec.seed)
    return rng.uniform(spec.lo, spec.hi, n)


def density_at(prob: Problem, level: np.ndarray, anchor: np.ndarray) -> np.ndarray:
    """Input density of each given leaf (evaluated by the caller on its own leaf set).

    For 'iid' the mesh must be uniform at the finest level; the raw field is
    looked up by lexicographic element index.  For c3 the raw field is the
    input *before* the one DENS smoothing pass; the pass
    itself is method arithmetic and is done by each side.
    """
    spec = prob.density
    n = level.shape[0]
    if spec.kind == "const":
        return np.full(n, spec.value, dtype=np.float64)
    if spec.kind == "iid":
        if np.any(level != prob.L):
            raise ValueError("iid density requires a uniform finest-level mesh")
        ext = prob.lattice_extent
        a = anchor.astype(np.int64)
        lex = a[:, 0].copy()
        stride = 1
        for c in range(1, prob.dim):
            stride *= ext[c - 1]
            lex += a[:, c] * stride
        return raw_iid_field(prob)[lex]
    if spec.kind == "gauss":
        extent_phys = [b * prob.h0 for b in prob.base]
        return _gauss_density(spec, prob.dim, extent_phys, leaf_centers(prob, level, anchor))
    raise ValueError(spec.kind)


# ---------------------------------------------------------------------------
# synthetic refinement rule R (input generation)
# ---------------------------------------------------------------------------

def refine_rule_R(prob_like: Problem, lo: float = 0.05, hi: float = 0.95):
    """Pre-balance leaf set: for k = 0..L-1 refine the level-k leaves whose
    density lies in (lo, hi) plus every level-k leaf whose closed box touches
    one of them.  Returns (level int8, anchor int32)."""
    dim, L = prob_like.dim, prob_like.L
    lev, anc = uniform_leaves(dim, prob_like.base, L, 0)
    for k in range(L):
        at_k = lev == k
        idx = np.nonzero(at_k)[0]
        if idx.size == 0:
            break
        rho = density_at(prob_like, lev[idx], anc[idx])
        S = (rho > lo) & (rho < hi)
        s = 1 << (L - k)
        g = anc[idx].astype(np.int64) // s                      # level-k grid coords
        shape = [b << k for b in prob_like.base]
        present = np.zeros(shape, dtype=bool)
        inS = np.zeros(shape, dtype=bool)
        present[tuple(g.T)] = True
        inS[tuple(g[S].T)] = True
        dil = inS.copy()
        # Chebyshev-1 dilation (closed boxes of same-size cells touch)
        for axis in range(dim):
            tmp = dil.copy()
            sl_a = [slice(None)] * dim
            sl_b = [slice(None)] * dim
            sl_a[axis] = slice(1, None)
            sl_b[axis] = slice(None, -1)
            tmp[tuple(sl_a)] |= dil[tuple(sl_b)]
            tmp[tuple(sl_b)] |= dil[tuple(sl_a)]
            dil = tmp
        T = dil[tuple(g.T)] & present[tuple(g.T)]
        ref = idx[T]
        if ref.size == 0:
            continue
        keep = np.ones(lev.shape[0], dtype=bool)
        keep[ref] = False
        half = s // 2
        kids_a = []
        for corner in range(1 << dim):
            off = np.array([((corner >> c) & 1) * half for c in range(dim)], dtype=np.int64)
            kids_a.append(anc[ref].astype(np.int64) + off[None, :])
        kids_a = np.concatenate(kids_a, axis=0)
        kids_l = np.full(kids_a.shape[0], k + 1, dtype=np.int8)
        lev = np.concatenate([lev[keep], kids_l])
        anc = np.concatenate([anc[keep].astype(np.int64), kids_a]).astype(np.int32)
    return lev, anc


# ---------------------------------------------------------------------------
# problems
# ---------------------------------------------------------------------------

def make_problem(name, dim, base, L=0, h0=1.0, leaves=None, density=None, fixed=(),
                 loads=(), **kw) -> Problem:
    if leaves is None:
        leaves = uniform_leaves(dim, base, L, L)
    lev, anc = leaves
    return Problem(name=name, dim=dim, L=L, base=tuple(int(b) for b in base), h0=float(h0),
                   leaf_level=np.asarray(lev, dtype=np.int8),
                   leaf_anchor=np.asarray(anc, dtype=np.int32).reshape(-1, dim),
                   density=density or DensitySpec("const", value=1.0),
                   fixed=list(fixed), loads=list(loads), **kw)


def _c1(scale=1):
    nx, ny = 60 * scale, 20 * scale
    return make_problem(
        "c1_mbb_60x20" if scale == 1 else f"c1_mbb_{nx}x{ny}", 2, (nx, ny), L=0,
        density=DensitySpec("const", value=0.5),
        fixed=[((0, 0), (0, ny), 0b01), ((nx, 0), (nx, 0), 0b10)],
        loads=[("point", (0, ny), (0, ny), (0.0, -1.0))],
        rmin=1.5, rtol=1e-10,
        notes="MBB half-beam: x-symmetry on x=0, y-support at (nx,0), unit load at (0,ny)")


def _c2(L=4, base=(32, 16), seed=2):
    tmp = make_problem("tmp", 2, base, L=L, leaves=(np.zeros(0), np.zeros((0, 2))),
                       density=DensitySpec("gauss", seed=seed, n_gauss=40, thr=0.5))
    leaves = refine_rule_R(tmp)
    ext = [b << L for b in base]
    return make_problem(
        f"c2_cantilever2d_amr_{base[0]}x{base[1]}_L{L}", 2, base, L=L, leaves=leaves,
        density=tmp.density,
        fixed=[((0, 0), (0, ext[1]), 0b11)],
        loads=[("point", (ext[0], ext[1] // 2), (ext[0], ext[1] // 2), (0.0, -1.0))],
        rmin=1.5 / (1 << L), rtol=1e-10)


def _c3(nx=96, ny=48, nz=48, seed=3):
    return make_problem(
        f"c3_cantilever3d_{nx}x{ny}x{nz}", 3, (nx, ny, nz), L=0,
        density=DensitySpec("iid", lo=0.01, hi=1.0, seed=seed),
        fixed=[((0, 0, 0), (0, ny, nz), 0b111)],
        loads=[("line", (nx, 0, 0), (nx, 0, nz), (0.0, -1.0, 0.0))],
        rmin=1.5, rtol=1e-8, presmooth_rmin=1.5)


def _c4(L=4, base=(24, 12, 12), seed=4, n_gauss=200):
    tmp = make_problem("tmp", 3, base, L=L, leaves=(np.zeros(0), np.zeros((0, 3))),
                       density=DensitySpec("gauss", seed=seed, n_gauss=n_gauss, thr=0.3))
    leaves = refine_rule_R(tmp)
    ext = [b << L for b in base]
    return make_problem(
        f"c4_bridge3d_amr_{base[0]}x{base[1]}x{base[2]}_L{L}", 3, base, L=L, leaves=leaves,
        density=tmp.density,
        fixed=[((0, 0, 0), (0, ext[1], ext[2]), 0b111)],
        loads=[("line", (ext[0], 0, 0), (ext[0], 0, ext[2]), (0.0, -1.0, 0.0))],
        rmin=1.5 / (1 << L), rtol=1e-8)


def _c5(nx=256, ny=128, nz=128, seed=5):
    return make_problem(
        f"c5_uniform3d_{nx}x{ny}x{nz}", 3, (nx, ny, nz), L=0,
        density=DensitySpec("iid", lo=0.001, hi=1.0, seed=seed),
        fixed=[((0, 0, 0), (0, ny, nz), 0b111)],
        loads=[("face", (nx, 0, 0), (nx, ny, nz), (0.0, -1.0, 0.0))],
        rmin=2.0, rtol=1e-8, fixed_iters=500)


def config_c4L():
    """c4 recipe with one more refinement level (L = 5, finest-equivalent
    768x384x384): 1,486,742 active elements, the "~1-2M active elements" that
    BASELINE.json's config 4 names (the L = 4 recipe gives 225,090;
    DESIGN.md §3, reading R26)."""
    return _c4(L=5)


_CONFIGS = {
    "c1": _c1, "c2": _c2, "c3": _c3, "c4": _c4, "c5": _c5,
}


def config_names():
    return list(_CONFIGS)


def config(name: str, **kw) -> Problem:
    """BASELINE.json configs c1..c5; keyword overrides give
    scaled-down variants with the same recipe (e.g. ``config('c5', nx=16, ny=8, nz=8)``)."""
    return _CONFIGS[name](**kw)
