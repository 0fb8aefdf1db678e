"""Pins for oracle/mesh.py (Table 1)."""
import os
import itertools

import numpy as np
import pytest

from inputs import config, make_problem, uniform_leaves, DensitySpec
from oracle import mesh as omesh, fe, solve
from tests.helpers import cantilever2d, cantilever3d, refine_some

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _boxes(m):
    s = m.size()
    return m.elem_anchor.astype(np.int64), s


def _shared_measure(a1, s1, a2, s2):
    """Dimension of the intersection of two closed boxes (-1 if empty)."""
    dims = 0
    for c in range(a1.shape[0]):
        lo = max(a1[c], a2[c])
        hi = min(a1[c] + s1, a2[c] + s2)
        if lo > hi:
            return -1
        if hi > lo:
            dims += 1
    return dims


def _check_tiling_and_balance(m, ext):
    a, s = _boxes(m)
    dim = m.dim
    vol = (s.astype(np.int64) ** dim).sum()
    assert vol == int(np.prod(ext))
    n = a.shape[0]
    # exhaustive pairwise: balance across (d-1)-faces, and edges in 3D (C10)
    need = {2: (1,), 3: (1, 2)}[dim]
    for i in range(n):
        for j in range(i + 1, n):
            k = _shared_measure(a[i], s[i], a[j], s[j])
            assert k < dim, "overlap"
            if k in need:
                assert abs(int(m.elem_level[i]) - int(m.elem_level[j])) <= 1


def test_table1_unknown_convention():
    rows = [l.split() for l in open(os.path.join(GOLD, "paper_table1_unknowns.txt"))
            if l.strip() and not l.startswith("#")]
    for nx, ny, ne, nu in rows:
        prob = make_problem("t1", 2, (int(nx), int(ny)))
        m = omesh.build_mesh(prob, with_filter=False, density=False)
        assert m.n_el == int(ne)
        assert m.n_dof == int(nu)


def test_2x1_mesh_six_nodes():
    m = omesh.build_mesh(make_problem("2x1", 2, (2, 1)), with_filter=False)
    assert m.n_node == 6 and m.hang_node.size == 0


def test_one_refined_element_four_hanging_2d():
    prob = cantilever2d((3, 3), L=1, leaves=refine_some(2, (3, 3), 1, [(1, 1)]))
    m = omesh.build_mesh(prob)
    assert m.hang_node.size == 4
    assert np.all(m.hang_weight == 0.5)


def test_one_refined_element_eighteen_hanging_3d():
    prob = cantilever3d((3, 3, 3), L=1, leaves=refine_some(3, (3, 3, 3), 1, [(1, 1, 1)]))
    m = omesh.build_mesh(prob)
    assert m.hang_node.size == 18
    nper = np.diff(m.hang_ptr)
    assert (nper == 2).sum() == 12 and (nper == 4).sum() == 6


@pytest.mark.parametrize("case", ["2d", "3d"])
def test_mesh_invariants(case):
    if case == "2d":
        prob = cantilever2d((4, 2), L=3, leaves=refine_some(2, (4, 2), 3, [(1, 0), (2, 1)]))
    else:
        prob = cantilever3d((3, 2, 2), L=2, leaves=refine_some(3, (3, 2, 2), 2, [(1, 0, 1)]))
    m = omesh.build_mesh(prob)
    ext = prob.lattice_extent
    _check_tiling_and_balance(m, ext)
    # C2: Morton order of anchors; C3: Morton order of nodes
    assert np.all(np.diff(omesh.morton(m.elem_anchor)) > 0)
    assert np.all(np.diff(omesh.morton(m.node_coord)) > 0)
    # C4 corner geometry
    offs = omesh.corner_offsets(m.dim)
    s = m.size()
    for c in range(1 << m.dim):
        assert np.all(m.node_coord[m.elem_node[:, c]] == m.elem_anchor + offs[c] * s[:, None])
    # C6: hanging node = mean of parents exactly; parents are not hanging
    hang = set(m.hang_node.tolist())
    for i, hn in enumerate(m.hang_node):
        ps = m.hang_parent[m.hang_ptr[i]:m.hang_ptr[i + 1]]
        assert np.all(np.diff(ps) > 0)
        assert np.all(m.node_coord[ps].sum(axis=0) == len(ps) * m.node_coord[hn])
        assert not (set(ps.tolist()) & hang)
        assert abs(m.hang_weight[m.hang_ptr[i]:m.hang_ptr[i + 1]].sum() - 1.0) == 0.0
    # brute-force twin of C6: node in the relative interior of a leaf edge/face
    a, sz = _boxes(m)
    brute = set()
    for n in range(m.n_node):
        p = m.node_coord[n]
        for e in range(m.n_el):
            inside = (p >= a[e]) & (p <= a[e] + sz[e])
            if not inside.all():
                continue
            on_bound = (p == a[e]) | (p == a[e] + sz[e])
            free_axes = int((~on_bound).sum())
            # relative interior of an edge: dim-1 axes on the boundary, 1 interior;
            # of a face (3D): 1 axis on the boundary, 2 interior
            if free_axes in ((1,) if m.dim == 2 else (1, 2)):
                brute.add(n)
    assert brute == hang
    # C7: fixed DOFs exclude hanging nodes and are sorted
    assert np.all(np.diff(m.fixed_dof) > 0)
    assert not (set((m.fixed_dof // m.dim).tolist()) & hang)


def test_filter_csr_vs_bruteforce():
    prob = cantilever2d((4, 2), L=2, leaves=refine_some(2, (4, 2), 2, [(1, 0)]), rmin=0.6)
    m = omesh.build_mesh(prob)
    p, i = omesh.filter_neighbours_bruteforce(m, prob.rmin)
    assert np.array_equal(p, m.filt_ptr) and np.array_equal(i, m.filt_idx)


def test_fully_refined_amr_equals_uniform():
    """P7: an AMR tree refined everywhere to L gives bit-identical arrays to the
    uniform mesh of the same geometry, and identical u."""
    L = 2
    base = (3, 2)
    leaves = uniform_leaves(2, base, L, L)
    amr = cantilever2d(base, L=L, leaves=leaves)
    uni = cantilever2d((base[0] << L, base[1] << L), L=0, h0=1.0 / (1 << L))
    ma = omesh.build_mesh(amr)
    mu = omesh.build_mesh(uni)
    for f in ["elem_anchor", "elem_node", "node_coord", "fixed_dof", "load", "hang_node",
              "filt_ptr", "filt_idx"]:
        assert np.array_equal(getattr(ma, f), getattr(mu, f)), f
    assert np.array_equal(ma.centers(), mu.centers())
    x = np.linspace(0.1, 1.0, ma.n_el)
    us = []
    for m in (ma, mu):
        K = fe.assemble_K(m, x, 3.0)
        A, b, C = fe.projected_system(m, K)
        us.append(fe.recover(C, solve.dense_solve(A, b)))
    assert np.array_equal(us[0], us[1])


def test_balance_resolves_level_jumps():
    # deep refinement in one corner cell forces ripple refinement of its neighbours
    prob = cantilever2d((4, 4), L=4, leaves=refine_some(2, (4, 4), 4, [(1, 1)]))
    m = omesh.build_mesh(prob)
    _check_tiling_and_balance(m, prob.lattice_extent)
    assert m.n_el > prob.leaf_level.shape[0]


def test_loads_consistent_totals():
    p3 = config("c3", nx=6, ny=3, nz=3)
    m = omesh.build_mesh(p3)
    assert abs(m.load.sum() - (-3.0)) < 1e-15           # line of length nz=3, intensity 1
    p5 = config("c5", nx=4, ny=2, nz=3)
    m = omesh.build_mesh(p5)
    assert abs(m.load.sum() - (-6.0)) < 1e-15           # face 2 x 3, traction 1
    fy = m.load[1::3]
    face = m.node_coord[:, 0] == 4
    vals = sorted(set(fy[face].tolist()))
    assert vals == [-1.0, -0.5, -0.25]
    p1 = config("c1")
    m = omesh.build_mesh(p1)
    assert m.fixed_dof.size == 22 and m.n_dof == 2562
