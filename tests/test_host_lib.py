"""CPU tests of the product's host side: the library loads and exports every
symbol of include/*.h, and the C++ host builder reproduces the oracle's
canonical arrays bit-exactly."""
import ctypes
import os
import re

import numpy as np
import pytest

from inputs import config
from oracle import mesh as omesh, fe
import paper_1009_4975_b200 as pb
from paper_1009_4975_b200 import _lib
from tests.helpers import cantilever2d, cantilever3d, refine_some, hanging_load2d, hanging_load3d

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    names = set()
    for h in ("tomesh.h", "tomesh_host.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?(?:int|void|char)\s*\*?\s*(\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    declared = _declared_symbols()
    assert {"tomesh_upload", "tosolve_cg", "to_sensitivity", "to_filter", "tomesh_free",
            "to_last_error", "tomesh_host_build"} <= declared
    for name in declared:
        assert hasattr(lib, name), name
    assert declared <= set(_lib.EXPORTS)


def test_struct_layouts_match_header(tmp_path):
    """offsetof/sizeof of every ABI struct, from the C headers via g++, match ctypes."""
    import shutil
    import subprocess
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("no g++")
    structs = {"to_mesh_desc": _lib.ToMeshDesc, "to_cg_stats": _lib.ToCgStats,
               "to_mesh_info": _lib.ToMeshInfo, "tomesh_host_spec": _lib.HostSpec,
               "tomesh_host_arrays": _lib.HostArrays, "to_oc_stats": _lib.ToOcStats,
               "to_opt_params": _lib.ToOptParams, "to_opt_step": _lib.ToOptStep,
               "to_opt_state": _lib.ToOptState, "tomesh_adapt_result": _lib.AdaptResult,
               "to_minres_stats": _lib.ToMinresStats, "to_shard_bufs": _lib.ToShardBufs}
    lines = ['#include <cstdio>', '#include <cstddef>', '#include "tomesh.h"', '#include "tomesh_host.h"',
             "int main(){"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f.rstrip("_")}));')
    lines.append("return 0;}")
    src = tmp_path / "abi.cpp"
    src.write_text("\n".join(lines))
    exe = tmp_path / "abi"
    subprocess.run([gxx, "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {}
    for line in out:
        if line.strip():
            a, b, c = line.split()
            got[(a, b)] = int(c)
    for cname, cls in structs.items():
        assert got[(cname, "sizeof")] == ctypes.sizeof(cls), cname
        for f, _ in cls._fields_:
            assert got[(cname, f)] == getattr(cls, f).offset, (cname, f)


def _compare(prob):
    hm = pb.prepare(prob)
    om = omesh.build_mesh(prob)
    assert np.array_equal(hm.elem_level, om.elem_level)
    assert np.array_equal(hm.elem_anchor, om.elem_anchor)
    assert np.array_equal(hm.elem_node, om.elem_node)
    assert np.array_equal(hm.node_coord.astype(np.int64), om.node_coord)
    assert np.array_equal(hm.hang_node, om.hang_node)
    assert np.array_equal(hm.hang_ptr, om.hang_ptr)
    assert np.array_equal(hm.hang_parent, om.hang_parent)
    assert np.array_equal(hm.hang_weight, om.hang_weight)
    assert np.array_equal(hm.fixed_dof, om.fixed_dof)
    assert np.array_equal(hm.load, om.load)
    assert np.array_equal(hm.filt_ptr, om.filt_ptr)
    assert np.array_equal(hm.filt_idx, om.filt_idx)
    return hm, om


@pytest.mark.parametrize("case", [
    "c1", "c2", "c3", "c4", "c3s", "c5s", "c4s",
    "amr2d", "amr3d", "ripple2d", "hload2d", "hload3d"])
def test_host_builder_bit_exact_vs_oracle(case):
    if case == "c1":
        prob = config("c1")
    elif case == "c2":
        prob = config("c2")
    elif case in ("c3", "c4"):
        prob = config(case)                            # full BASELINE.json sizes
    elif case == "c3s":
        prob = config("c3", nx=12, ny=6, nz=6)
    elif case == "c5s":
        prob = config("c5", nx=16, ny=8, nz=8)
    elif case == "c4s":
        prob = config("c4", base=(12, 6, 6), L=2, n_gauss=60)
    elif case == "amr2d":
        prob = cantilever2d((5, 3), L=3, leaves=refine_some(2, (5, 3), 3, [(1, 1), (3, 0)]), rmin=0.3)
    elif case == "amr3d":
        prob = cantilever3d((3, 2, 2), L=2, leaves=refine_some(3, (3, 2, 2), 2, [(1, 1, 0)]), rmin=0.4)
    elif case == "hload2d":
        prob = hanging_load2d()
    elif case == "hload3d":
        prob = hanging_load3d()
    else:
        prob = cantilever2d((4, 4), L=4, leaves=refine_some(2, (4, 4), 4, [(1, 1)]), rmin=0.2)
    hm, om = _compare(prob)
    if case.startswith("hload"):
        # C8: loads on hanging nodes stay in f (both sides); two loaded nodes are hanging
        d = om.dim
        loaded = {n for n in range(om.n_node) if np.any(om.load[d * n:d * n + d] != 0.0)}
        assert len(loaded & set(om.hang_node.tolist())) == 2
    if case in ("c2", "c4", "c4s", "amr2d", "amr3d", "ripple2d"):
        assert hm.hang_node.size > 0


def test_host_builder_rejects_bad_leaves():
    prob = cantilever2d((2, 2))
    with pytest.raises(pb.TomeshError):
        pb.tomesh_host_build(2, 0, (2, 2), 1.0, prob.leaf_level[:-1], prob.leaf_anchor[:-1],
                             prob.fixed, prob.loads, 1.5)
    with pytest.raises(pb.TomeshError):
        pb.tomesh_host_build(2, 0, (2, 2), 1.0, prob.leaf_level, prob.leaf_anchor, prob.fixed,
                             [("point", (1, 5), (1, 5), (0.0, 1.0))], 1.5)


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("nu", [0.0, 0.3, 0.45])
def test_product_K0_closed_form_vs_oracle_quadrature(dim, nu):
    """L1: the kernels' K0 (Kronecker closed form) vs the oracle's Gauss quadrature."""
    n = dim << dim
    K = np.zeros((n, n))
    assert _lib.lib().to_element_matrix(dim, nu, K.ctypes.data) == 0
    Ko = fe.element_stiffness(dim, 1.0, nu, 1.0)
    assert np.max(np.abs(K - Ko)) <= 1e-15 * np.max(np.abs(Ko)) * 4


@pytest.mark.parametrize("nu", [0.0, 0.3, 0.45])
def test_product_hadamard_factorisation(nu, rng):
    """y = K0 x via the Hadamard form equals the oracle's dense product."""
    diag = np.zeros((3, 8))
    off = np.zeros((3, 3, 8))
    assert _lib.lib().to_element_hadamard(nu, diag.ctypes.data, off.ctypes.data) == 0
    Ko = fe.element_stiffness(3, 1.0, nu, 1.0)
    H1 = np.array([[1, 1], [1, -1]])
    H3 = np.kron(np.kron(H1, H1), H1)          # index m = m_z m_y m_x (x least significant)
    for _ in range(5):
        x = rng.standard_normal(24)
        X = x.reshape(8, 3)                   # [corner][component]
        Xh = H3 @ X
        Yh = np.zeros_like(Xh)
        for m in range(8):
            for i in range(3):
                acc = diag[i, m] * Xh[m, i]
                for j in range(3):
                    if j != i and ((m >> i) & 1) != ((m >> j) & 1):
                        acc += off[i, j, m] * Xh[m ^ ((1 << i) | (1 << j)), j]
                Yh[m, i] = acc
        y = (H3 @ Yh).reshape(-1)
        assert np.max(np.abs(y - Ko @ x)) <= 1e-14 * np.max(np.abs(Ko @ x)) * 10


# ---- dynamic AMR mesh update: C++ host code vs oracle/amr.py (bit-exact) ----------------

def _amr_cases():
    from tests.helpers import cantilever2d, cantilever3d, refine_some, hanging_load2d, hanging_load3d
    return [
        cantilever2d((6, 3), L=3, leaves=refine_some(2, (6, 3), 3, [(1, 1), (4, 0), (2, 2)]), rmin=0.9),
        cantilever3d((3, 2, 2), L=2, leaves=refine_some(3, (3, 2, 2), 2, [(1, 1, 0), (0, 0, 1)]), rmin=0.7),
    ]


@pytest.mark.parametrize("case", [0, 1])
def test_host_adapt_matches_oracle(case):
    """tomesh_host_adapt + tomesh_host_build + tomesh_host_transfer reproduce the
    oracle's sweeps, leaf set, densities and balanced mesh exactly, over a
    sequence of adaptations driven by random density fields (oracle marks)."""
    from oracle import amr
    prob = _amr_cases()[case]
    rng = np.random.default_rng(21 + case)
    om = omesh.build_mesh(prob, density=False)
    hm = pb.prepare(prob, keep_handle=True)
    x = rng.uniform(1e-3, 1.0, om.n_el) ** 2
    for it in range(4):
        assert np.array_equal(hm.elem_level, om.elem_level) and np.array_equal(hm.elem_anchor, om.elem_anchor)
        mk = amr.mark(om, x, 0.5, prob.rmin)
        if it == 3:   # random marks exercise both sweeps harder
            mk = rng.choice(np.array([-1, 0, 1], dtype=np.int8), om.n_el, p=[0.6, 0.3, 0.1])
            mk[(mk == 1) & (om.elem_level == om.L)] = 0
            mk[(mk == -1) & (om.elem_level == 0)] = 0
        ro = amr.adapt(om, x, mk)
        rh = pb.api.tomesh_host_adapt(hm, mk, x)
        assert np.array_equal(rh.marks, ro.marks)
        assert (rh.n_refined, rh.n_groups, rh.n_unmarked_sibling, rh.n_unmarked_incompat) == \
            (ro.n_refined, ro.n_groups, ro.n_unmarked_sibling, ro.n_unmarked_incompat)
        assert np.array_equal(rh.leaf_level, ro.leaf_level) and np.array_equal(rh.leaf_anchor, ro.leaf_anchor)
        assert np.array_equal(rh.leaf_x, ro.leaf_x)                       # bit-exact means
        om = amr.rebuild(prob, ro)
        hm = pb.api.rebuild(prob, rh)
        xo = amr.transfer(om, ro)
        xh = pb.api.tomesh_host_transfer(hm, rh)
        assert np.array_equal(xh, xo)
        for f in ("elem_node", "hang_node", "hang_parent", "fixed_dof", "load", "filt_ptr", "filt_idx"):
            assert np.array_equal(getattr(hm, f), getattr(om, f)), f
        x = np.clip(xo + rng.normal(0, 0.25, om.n_el), 1e-3, 1.0)


def test_host_adapt_rejects_bad_marks():
    prob = _amr_cases()[0]
    hm = pb.prepare(prob, keep_handle=True)
    x = np.full(hm.n_el, 0.5)
    bad = np.zeros(hm.n_el, dtype=np.int8)
    bad[int(np.nonzero(hm.elem_level == 0)[0][0])] = -1            # derefine at level 0
    with pytest.raises(pb.TomeshError):
        pb.api.tomesh_host_adapt(hm, bad, x)
    bad[:] = 0
    bad[0] = 3
    with pytest.raises(pb.TomeshError):
        pb.api.tomesh_host_adapt(hm, bad, x)
    with pytest.raises(ValueError):
        pb.api.tomesh_host_adapt(pb.prepare(prob), np.zeros(hm.n_el, dtype=np.int8), x)   # no handle kept
