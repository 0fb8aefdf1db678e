"""tomesh_upload rejects inconsistent meshes before touching the GPU (runs on
CPU): include/tomesh.h promises TO_EMESH for out-of-range indices, a
constraint parent that is itself hanging, a hanging DOF listed as fixed,
weights not summing to 1 and unsorted lists, and TO_EINVAL for
bad scalars / empty meshes."""
import copy
import ctypes as C

import numpy as np
import pytest

import paper_1009_4975_b200 as pb
from paper_1009_4975_b200 import _lib as L
from paper_1009_4975_b200.api import make_desc
from tests.helpers import cantilever2d, refine_some


@pytest.fixture(scope="module")
def hanging_mesh():
    prob = cantilever2d((5, 3), L=3, leaves=refine_some(2, (5, 3), 3, [(1, 1), (3, 0)]), rmin=0.3)
    hm = pb.prepare(prob)
    assert hm.hang_node.size > 0
    return hm


def _upload(hm, E0=1.0, Emin=1e-9, nu=0.3, rmin=None):
    d, keep = make_desc(hm, E0, Emin, nu, hm.rmin if rmin is None else rmin)
    h = C.c_void_p()
    rc = L.lib().tomesh_upload(C.byref(d), 0, None, C.byref(h))
    msg = L.lib().to_last_error().decode()
    return rc, msg


def _mutated(hm, **arrays):
    m = copy.deepcopy(hm)
    for k, v in arrays.items():
        setattr(m, k, v)
    return m


def test_out_of_range_node_index(hanging_mesh):
    en = hanging_mesh.elem_node.copy()
    en[3, 2] = hanging_mesh.n_node
    rc, msg = _upload(_mutated(hanging_mesh, elem_node=en))
    assert rc == L.TO_EMESH and "elem_node" in msg


def test_chained_constraint_rejected(hanging_mesh):
    # make the first hanging node's first parent another hanging node
    hp = hanging_mesh.hang_parent.copy()
    other = int(hanging_mesh.hang_node[1])
    k0, k1 = hanging_mesh.hang_ptr[0], hanging_mesh.hang_ptr[1]
    row = sorted(set(hp[k0:k1].tolist()[1:] + [other]))
    if len(row) != k1 - k0:
        pytest.skip("degenerate parent row")
    hp[k0:k1] = row
    rc, msg = _upload(_mutated(hanging_mesh, hang_parent=hp))
    assert rc == L.TO_EMESH and "hanging" in msg


def test_hanging_dof_fixed_rejected(hanging_mesh):
    fd = np.unique(np.concatenate([hanging_mesh.fixed_dof, [2 * int(hanging_mesh.hang_node[0])]])).astype(np.int64)
    rc, msg = _upload(_mutated(hanging_mesh, fixed_dof=fd))
    assert rc == L.TO_EMESH and "hanging" in msg


def test_weights_must_sum_to_one(hanging_mesh):
    hw = hanging_mesh.hang_weight.copy()
    hw[0] *= 1.5
    rc, msg = _upload(_mutated(hanging_mesh, hang_weight=hw))
    assert rc == L.TO_EMESH and "sum" in msg


def test_unsorted_fixed_list_rejected(hanging_mesh):
    fd = hanging_mesh.fixed_dof[::-1].copy()
    rc, msg = _upload(_mutated(hanging_mesh, fixed_dof=fd))
    assert rc == L.TO_EMESH


def test_bad_scalars_rejected(hanging_mesh):
    assert _upload(hanging_mesh, nu=0.5)[0] == L.TO_EINVAL
    assert _upload(hanging_mesh, E0=0.0)[0] == L.TO_EINVAL
    assert _upload(hanging_mesh, Emin=-1.0)[0] == L.TO_EINVAL


def test_empty_mesh_rejected(hanging_mesh):
    m = _mutated(hanging_mesh, elem_node=np.zeros((0, 4), np.int32), elem_anchor=np.zeros((0, 2), np.int32),
                 elem_level=np.zeros(0, np.int8))
    rc, _ = _upload(m)
    assert rc == L.TO_EINVAL


def test_null_arguments():
    h = C.c_void_p()
    assert L.lib().tomesh_upload(None, 0, None, C.byref(h)) == L.TO_EINVAL
    assert L.lib().tosolve_cg(None, C.c_double(3.0), None, None, C.c_double(1e-8), 10, 0, None, None) == L.TO_EINVAL
