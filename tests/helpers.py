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
