"""Pins for oracle/amr.py (§4 :360-492; readings R21-R23).

Independent checks: the trigger examples of PAPER.md:421-455, marking against
an all-pairs distance scan, the sibling rule on hand-built meshes, sweep 2
against brute force (a derefinement it keeps never gets re-refined by the 2:1
balance; one it drops would leave a two-level jump), transfer conservation and
the refine/derefine inverse pair."""
import itertools

import numpy as np
import pytest

from inputs import make_problem, uniform_leaves, DensitySpec
from oracle import amr, mesh as omesh
from tests.helpers import cantilever2d, cantilever3d, refine_some
from tests.test_oracle_mesh import _check_tiling_and_balance, _shared_measure


def _mesh(prob):
    return omesh.build_mesh(prob, density=False)


def test_should_adapt_cases():
    """CASE (i): change < 0.01 and >= 5 steps; CASE (ii): >= 10 steps."""
    assert amr.should_adapt(0.005, 6)
    assert amr.should_adapt(0.5, 10)
    assert not amr.should_adapt(0.5, 3)
    assert not amr.should_adapt(0.005, 4)
    assert amr.should_adapt(0.0099, 5) and not amr.should_adapt(0.01, 5)


def _pairs_within(mesh, r):
    c = mesh.centers()
    n = mesh.n_el
    out = []
    for e in range(n):
        out.append([d for d in range(n) if np.sum((c[d] - c[e]) ** 2) < r * r])
    return out


@pytest.mark.parametrize("dim", [2, 3])
def test_mark_vs_all_pairs(dim, rng):
    if dim == 2:
        prob = cantilever2d((6, 3), L=2, leaves=refine_some(2, (6, 3), 2, [(1, 1), (4, 0)]), rmin=1.3)
    else:
        prob = cantilever3d((3, 2, 2), L=2, leaves=refine_some(3, (3, 2, 2), 2, [(1, 1, 0)]), rmin=0.8)
    m = _mesh(prob)
    for trial in range(4):
        x = rng.uniform(0.0, 1.0, m.n_el) ** 3
        for r_amr in (prob.rmin, 0.3, 2.5):
            got = amr.mark(m, x, 0.5, r_amr)
            near = _pairs_within(m, r_amr)
            for e in range(m.n_el):
                want = 1 if any(x[d] >= 0.5 for d in near[e]) else -1
                if want == 1 and m.elem_level[e] == m.L:
                    want = 0
                if want == -1 and m.elem_level[e] == 0:
                    want = 0
                assert got[e] == want
    # r_amr <= 0: only the solid elements themselves
    got = amr.mark(m, x, 0.5, 0.0)
    assert np.all((got == 1) == ((x >= 0.5) & (m.elem_level < m.L)))


def test_single_solid_element_fig2():
    """Fig. 2: a void element with a solid one within r_amr is refined (a),
    a void element with none is derefined (b)."""
    prob = cantilever2d((4, 2), L=1, leaves=uniform_leaves(2, (4, 2), 1, 1), rmin=1.2)
    m = _mesh(prob)
    x = np.full(m.n_el, 1e-3)
    c = m.centers()
    e0 = int(np.argmin(np.sum((c - np.array([2.25, 0.75])) ** 2, axis=1)))
    x[e0] = 1.0
    mk = amr.mark(m, x, 0.5, 1.2)
    d = np.sqrt(np.sum((c - c[e0]) ** 2, axis=1))
    # at the finest level refinement is capped: solid and near elements get 0, far ones -1
    assert np.all(mk[d < 1.2] == 0) and np.all(mk[d >= 1.2] == -1)


def _group_mesh():
    # 4x2 base, L = 2: cell (1,0) refined to level 1; cell (2,0) refined to level 1
    # and its child at the shared edge refined to level 2
    lev, anc = uniform_leaves(2, (4, 2), 2, 0)
    leaves = {(int(l), tuple(int(v) for v in a)) for l, a in zip(lev, anc)}
    for cell in [(4, 0), (8, 0)]:
        leaves.discard((0, cell))
        for o in itertools.product((0, 2), repeat=2):
            leaves.add((1, (cell[0] + o[0], cell[1] + o[1])))
    leaves.discard((1, (8, 0)))
    for o in itertools.product((0, 1), repeat=2):
        leaves.add((2, (8 + o[0], 0 + o[1])))
    ls = sorted(leaves)
    return cantilever2d((4, 2), L=2, leaves=(np.array([l for l, _ in ls], dtype=np.int8),
                                            np.array([a for _, a in ls], dtype=np.int32)))


def _idx(m, level, anchor):
    for e in range(m.n_el):
        if m.elem_level[e] == level and tuple(m.elem_anchor[e]) == tuple(anchor):
            return e
    raise KeyError


def test_sweep1_siblings():
    """3 of 4 siblings marked -> all 4 unmarked."""
    m = _mesh(_group_mesh())
    kids = [_idx(m, 1, (4 + a, b)) for a, b in itertools.product((0, 2), repeat=2)]
    mk = np.zeros(m.n_el, dtype=np.int8)
    mk[kids[:3]] = -1
    out, n1, n2 = amr.sweeps(m, mk)
    assert np.all(out == 0) and n1 == 3 and n2 == 0


def test_sweep2_level_two_incompatibility():
    """Derefining (1,0)'s children would put a level-0 parent next to the
    level-2 leaves of (2,0): unmarked; derefinements whose
    parent touches only leaves at most one level finer are kept."""
    m = _mesh(_group_mesh())
    kids_a = [_idx(m, 1, (4 + a, b)) for a, b in itertools.product((0, 2), repeat=2)]
    mk = np.zeros(m.n_el, dtype=np.int8)
    mk[kids_a] = -1
    out, n1, n2 = amr.sweeps(m, mk)
    assert np.all(out[kids_a] == 0) and n2 == 4
    # the level-2 leaves of (2,0) derefine to level 1: the parent (8,0) touches only
    # level <= 1 leaves -> kept
    kids_b = [_idx(m, 2, (8 + a, b)) for a, b in itertools.product((0, 1), repeat=2)]
    mk = np.zeros(m.n_el, dtype=np.int8)
    mk[kids_b] = -1
    out, _, n2 = amr.sweeps(m, mk)
    assert np.all(out[kids_b] == -1) and n2 == 0
    # refinement in the same pass counts: cells (1,0), (2,0) at level 1; derefining
    # (1,0)'s children is fine unless (2,0)'s child at the shared edge is refined
    lev, anc = uniform_leaves(2, (4, 2), 2, 0)
    leaves = {(int(l), tuple(int(v) for v in a)) for l, a in zip(lev, anc)}
    for cell in [(4, 0), (8, 0)]:
        leaves.discard((0, cell))
        for o in itertools.product((0, 2), repeat=2):
            leaves.add((1, (cell[0] + o[0], cell[1] + o[1])))
    ls = sorted(leaves)
    m = _mesh(cantilever2d((4, 2), L=2, leaves=(np.array([l for l, _ in ls], dtype=np.int8),
                                                np.array([a for _, a in ls], dtype=np.int32))))
    kids_a = [_idx(m, 1, (4 + a, b)) for a, b in itertools.product((0, 2), repeat=2)]
    mk = np.zeros(m.n_el, dtype=np.int8)
    mk[kids_a] = -1
    out, _, n2 = amr.sweeps(m, mk)
    assert np.all(out[kids_a] == -1) and n2 == 0
    mk[_idx(m, 1, (8, 0))] = 1
    out, _, n2 = amr.sweeps(m, mk)
    assert np.all(out[kids_a] == 0) and n2 == 4
    mk[_idx(m, 1, (8, 0))] = 0
    mk[_idx(m, 1, (10, 0))] = 1          # not touching (1,0): its closure refines (8,0)? no: kept
    out, _, n2 = amr.sweeps(m, mk)
    assert np.all(out[kids_a] == -1) and n2 == 0


@pytest.mark.parametrize("dim", [2, 3])
def test_sweep2_vs_bruteforce(dim, rng):
    """Random marks: every derefinement sweep 2 keeps stays a leaf through the
    2:1 balance of the new leaf set, and every group it drops would have been
    re-refined by that balance (brute force with mesh.balance)."""
    if dim == 2:
        prob = cantilever2d((4, 3), L=3, leaves=refine_some(2, (4, 3), 3, [(1, 1), (2, 1), (3, 2)]))
    else:
        prob = cantilever3d((2, 2, 2), L=3, leaves=refine_some(3, (2, 2, 2), 3, [(0, 0, 0), (1, 1, 0)]))
    m = _mesh(prob)
    n_dropped = n_kept = 0
    for trial in range(12):
        mk = rng.choice(np.array([-1, 0, 1], dtype=np.int8), m.n_el, p=[0.7, 0.2, 0.1])
        mk[(mk == 1) & (m.elem_level == m.L)] = 0
        mk[(mk == -1) & (m.elem_level == 0)] = 0
        s, n1, n2 = amr.sweeps(m, mk)
        res = amr.adapt(m, np.full(m.n_el, 0.5), mk)
        new = amr.rebuild(prob, res, with_filter=False)
        newset = {(int(l), tuple(int(v) for v in a)) for l, a in zip(new.elem_level, new.elem_anchor)}
        for e in np.nonzero(s == -1)[0]:
            assert _parent(m, e) in newset, "a derefined parent was re-refined by the balance"
            n_kept += 1
        after1 = _sweep1_only(m, mk)
        for e in np.nonzero((after1 == -1) & (s == 0))[0]:
            forced = np.where(s == 1, 1, 0).astype(np.int8)
            forced[_siblings(m, e)] = -1
            lv, an = _apply_marks(m, forced)
            bl, ba = omesh.balance(prob, lv.astype(np.int8), an.astype(np.int32))
            bset = {(int(l), tuple(int(v) for v in a)) for l, a in zip(bl, ba)}
            assert _parent(m, e) not in bset, "sweep 2 dropped a compatible derefinement"
            n_dropped += 1
    assert n_kept > 0 and n_dropped > 0


def _parent(m, e):
    s = 1 << (m.L - int(m.elem_level[e]))
    pa = (m.elem_anchor[e].astype(np.int64) // (2 * s)) * (2 * s)
    return (int(m.elem_level[e]) - 1, tuple(int(v) for v in pa))


def _siblings(m, e):
    s = 1 << (m.L - int(m.elem_level[e]))
    pa = (m.elem_anchor[e].astype(np.int64) // (2 * s)) * (2 * s)
    out = []
    for o in itertools.product((0, 1), repeat=m.dim):
        out.append(_idx(m, int(m.elem_level[e]), tuple(pa + np.array(o) * s)))
    return out


def _sweep1_only(m, mk):
    out = mk.copy()
    for e in np.nonzero(mk == -1)[0]:
        try:
            sib = _siblings(m, e)
        except KeyError:
            out[e] = 0
            continue
        if any(mk[d] != -1 for d in sib):
            out[e] = 0
    return out


def _apply_marks(m, mk):
    """Pre-balance leaf set for marks that already satisfy sweep 1 (no sweep 2)."""
    lv, an = [], []
    done = set()
    for e in range(m.n_el):
        l, a = int(m.elem_level[e]), m.elem_anchor[e].astype(np.int64)
        s = 1 << (m.L - l)
        if mk[e] == 1:
            for o in itertools.product((0, 1), repeat=m.dim):
                lv.append(l + 1)
                an.append(a + np.array(o) * (s // 2))
        elif mk[e] == -1:
            pa = tuple((a // (2 * s)) * (2 * s))
            if pa not in done:
                done.add(pa)
                lv.append(l - 1)
                an.append(np.array(pa))
        else:
            lv.append(l)
            an.append(a)
    return np.array(lv), np.array(an)


@pytest.mark.parametrize("dim", [2, 3])
def test_transfer_conserves_material(dim, rng):
    """sum x V before = after (refinement: exact; derefinement: the mean, to rounding),
    and the result tiles the box with 2:1 balance."""
    if dim == 2:
        prob = cantilever2d((4, 3), L=3, leaves=refine_some(2, (4, 3), 3, [(1, 1), (2, 1)]), rmin=0.7)
    else:
        prob = cantilever3d((2, 2, 2), L=2, leaves=refine_some(3, (2, 2, 2), 2, [(0, 0, 0)]), rmin=0.6)
    m = _mesh(prob)
    x = rng.uniform(1e-3, 1.0, m.n_el)
    for trial in range(5):
        mk = amr.mark(m, x, 0.5, prob.rmin)
        res = amr.adapt(m, x, mk)
        new = amr.rebuild(prob, res)
        xn = amr.transfer(new, res)
        before = np.sum(x * m.volumes())
        after = np.sum(xn * new.volumes())
        assert abs(after - before) <= 1e-12 * before
        ext = [b << prob.L for b in prob.base]
        _check_tiling_and_balance(new, ext)
        m, x = new, np.clip(xn + rng.normal(0, 0.2, new.n_el), 1e-3, 1.0)


def test_refine_then_derefine_is_identity(rng):
    """Refine everything once, then derefine every new group: the leaf set
    returns and the densities to rounding of the mean."""
    prob = cantilever2d((4, 2), L=1, leaves=uniform_leaves(2, (4, 2), 1, 0))
    m = _mesh(prob)
    x = rng.uniform(1e-3, 1.0, m.n_el)
    res = amr.adapt(m, x, np.ones(m.n_el, dtype=np.int8))
    m2 = amr.rebuild(prob, res)
    x2 = amr.transfer(m2, res)
    assert m2.n_el == 4 * m.n_el and np.all(m2.elem_level == 1)
    res2 = amr.adapt(m2, x2, -np.ones(m2.n_el, dtype=np.int8))
    m3 = amr.rebuild(prob, res2)
    x3 = amr.transfer(m3, res2)
    assert np.array_equal(m3.elem_level, m.elem_level) and np.array_equal(m3.elem_anchor, m.elem_anchor)
    np.testing.assert_allclose(x3, x, rtol=1e-15, atol=0)


def test_mean_of_children():
    """Children (0.1, 0.1, 0.3, 0.5) -> parent 0.25."""
    prob = cantilever2d((1, 1), L=1, leaves=uniform_leaves(2, (1, 1), 1, 1))
    m = _mesh(prob)
    x = np.array([0.1, 0.1, 0.3, 0.5])
    res = amr.adapt(m, x, -np.ones(4, dtype=np.int8))
    assert res.leaf_level.tolist() == [0] and res.leaf_x[0] == pytest.approx(0.25, abs=1e-16)


def test_dynamic_loop_small():
    """Fig. 1 with AMR on a small 2D cantilever: volume kept at every step, the
    mesh adapts on the CASE (i)/(ii) schedule, and after every adaptation the
    solid elements (x >= rho_s) below L were refined."""
    prob = cantilever2d((8, 4), L=2, leaves=uniform_leaves(2, (8, 4), 2, 0), rmin=0.8)
    mesh, x, H = amr.optimize_amr(prob, 0.5, 24, stage_steps=8)
    assert all(abs(v - 0.5) <= 1e-10 for v in H.volume)
    ad = [i for i, a in enumerate(H.adapted) if a]
    assert ad and ad[0] <= 9
    assert all(b - a <= 10 for a, b in zip([-1] + ad, ad))
    assert max(H.n_elem) > H.n_elem[0]
    # material conservation across adaptations: the volume after OC is V0 and the transfer keeps it
    assert abs(np.sum(x * mesh.volumes()) / mesh.volumes().sum() - 0.5) <= 1e-10
