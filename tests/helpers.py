"""Small problem builders used by several tests (no method arithmetic)."""
import numpy as np

from inputs import DensitySpec, make_problem, uniform_leaves


def refine_some(dim, base, L, cells):
    """Uniform level-0 mesh with the given level-0 cells (grid coords) refined
    down to level L along their first child (pre-balance leaf set)."""
    lev, anc = uniform_leaves(dim, base, L, 0)
    leaves = {(int(l), tuple(int(v) for v in a)) for l, a in zip(lev, anc)}
    for cell in cells:
        s = 1 << L
        a = tuple(int(c) * s for c in cell)
        cur = (0, a)
        for lvl in range(L):
            leaves.discard(cur)
            size = 1 << (L - cur[0])
            half = size // 2
            kids = []
            for corner in range(1 << dim):
                off = tuple(((corner >> k) & 1) * half for k in range(dim))
                kids.append((cur[0] + 1, tuple(cur[1][k] + off[k] for k in range(dim))))
            leaves.update(kids)
            cur = kids[0]
    lv = np.array([l for l, _ in sorted(leaves)], dtype=np.int8)
    an = np.array([a for _, a in sorted(leaves)], dtype=np.int32).reshape(-1, dim)
    return lv, an


def cantilever2d(base=(4, 2), L=0, leaves=None, density=None, h0=1.0, **kw):
    ext = [b << L for b in base]
    return make_problem("cant2d", 2, base, L=L, h0=h0, leaves=leaves,
                        density=density or DensitySpec("const", value=1.0),
                        fixed=[((0, 0), (0, ext[1]), 0b11)],
                        loads=[("point", (ext[0], 0), (ext[0], 0), (0.0, -1.0))], **kw)


def cantilever3d(base=(4, 2, 2), L=0, leaves=None, density=None, h0=1.0, **kw):
    ext = [b << L for b in base]
    return make_problem("cant3d", 3, base, L=L, h0=h0, leaves=leaves,
                        density=density or DensitySpec("const", value=1.0),
                        fixed=[((0, 0, 0), (0, ext[1], ext[2]), 0b111)],
                        loads=[("line", (ext[0], 0, 0), (ext[0], 0, ext[2]), (0.0, -1.0, 0.0))],
                        **kw)


def hanging_load2d():
    """Loads on hanging nodes: base 4x2, L = 1, level-0 cell (2, 0)
    refined once.  Lattice node (5, 2) is the midpoint of the bottom edge of
    the coarse cell (2, 1) and (6, 1) of the left edge of (3, 0): both are
    hanging (parents at half weight) and both carry a point load besides the
    tip load."""
    base, L = (4, 2), 1
    prob = cantilever2d(base, L=L, leaves=refine_some(2, base, L, [(2, 0)]), rmin=0.8,
                        density=DensitySpec("gauss", seed=21, n_gauss=6, thr=0.0, k=3.0))
    prob.loads = prob.loads + [("point", (5, 2), (5, 2), (0.25, -1.0)), ("point", (6, 1), (6, 1), (-0.5, 0.75))]
    prob.name = "hload2d"
    return prob


def hanging_load3d():
    """3D loads on hanging nodes: base 3x2x2, L = 1, level-0 cell
    (2, 0, 0) refined once.  Lattice node (6, 2, 1) is the midpoint of an edge
    of the coarse cell (2, 1, 0) on the loaded face x = 6 (two parents, 1/2
    each) and (5, 2, 1) the centre of its face y = 2 (four parents, 1/4
    each); both carry point loads besides the line load on the tip edge."""
    base, L = (3, 2, 2), 1
    prob = cantilever3d(base, L=L, leaves=refine_some(3, base, L, [(2, 0, 0)]), rmin=0.8,
                        density=DensitySpec("gauss", seed=22, n_gauss=8, thr=0.0, k=3.0))
    prob.loads = prob.loads + [("point", (6, 2, 1), (6, 2, 1), (0.0, -1.0, 0.5)),
                               ("point", (5, 2, 1), (5, 2, 1), (0.3, -1.0, 0.0))]
    prob.name = "hload3d"
    return prob
