"""ctypes declarations of libtomesh.so (include/tomesh.h, include/tomesh_host.h).

Loading fails loudly: there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libtomesh.so")

TO_OK, TO_NOT_CONVERGED = 0, 1
TO_EINVAL, TO_ECUDA, TO_ENOMEM, TO_EMESH, TO_ENAN, TO_EBREAKDOWN, TO_ENONPOS_DIAG = -1, -2, -3, -4, -5, -6, -7
TO_WARM, TO_FIXED_ITERS, TO_HISTORY, TO_NO_TRUE_RES, TO_PROFILE, TO_PROFILE_LOOP = 1, 2, 4, 8, 16, 32
TO_FILTER_SENS, TO_FILTER_DENS = 0, 1
TO_UPLOAD_GENERAL, TO_UPLOAD_LAUNCHED, TO_UPLOAD_NO_CLUSTER, TO_UPLOAD_EP, TO_UPLOAD_NO_EP = 1, 2, 4, 8, 16
TO_PC_JACOBI, TO_PC_IC0 = 0, 1
TOH_LOAD_POINT, TOH_LOAD_LINE, TOH_LOAD_FACE = 0, 1, 2

STATUS_NAMES = {0: "TO_OK", 1: "TO_NOT_CONVERGED", -1: "TO_EINVAL", -2: "TO_ECUDA", -3: "TO_ENOMEM",
                -4: "TO_EMESH", -5: "TO_ENAN", -6: "TO_EBREAKDOWN", -7: "TO_ENONPOS_DIAG"}

P = C.c_void_p


class ToMeshDesc(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("max_level", C.c_int32), ("h0", C.c_double),
        ("n_elem", C.c_int64), ("n_node", C.c_int64),
        ("elem_node", P), ("elem_anchor", P), ("elem_level", P),
        ("n_hang", C.c_int64), ("hang_node", P), ("hang_ptr", P), ("hang_parent", P), ("hang_weight", P),
        ("n_fixed", C.c_int64), ("fixed_dof", P),
        ("load", P),
        ("E0", C.c_double), ("Emin", C.c_double), ("nu", C.c_double),
        ("rmin", C.c_double), ("filt_nnz", C.c_int64), ("filt_ptr", P), ("filt_idx", P),
        ("options", C.c_uint32), ("n_owned", C.c_int32),
    ]


class ToCgStats(C.Structure):
    _fields_ = [("iters", C.c_int32), ("status", C.c_int32), ("relres", C.c_double),
                ("relres_true", C.c_double), ("ms", C.c_double), ("bnorm", C.c_double)]


class ToMeshInfo(C.Structure):
    _fields_ = [("dim", C.c_int32), ("structured", C.c_int32),
                ("n_elem", C.c_int64), ("n_node", C.c_int64), ("n_dof", C.c_int64), ("n_hang", C.c_int64),
                ("n_fixed", C.c_int64), ("filt_nnz", C.c_int64), ("grid", C.c_int64 * 3),
                ("device_bytes", C.c_int64), ("kernel_launches", C.c_int32), ("matvec_variant", C.c_int32),
                ("launches_total", C.c_int64), ("gen_blocks", C.c_int32), ("gen_smem_bytes", C.c_int32),
                ("gen_max_loc", C.c_int32), ("gen_max_el", C.c_int32), ("gen_local_el", C.c_int64),
                ("gen_local_nodes", C.c_int64)]


class ToMinresStats(C.Structure):
    _fields_ = [("iters", C.c_int32), ("status", C.c_int32), ("eta_rel", C.c_double), ("relres_true", C.c_double),
                ("ms", C.c_double), ("ic0_shift", C.c_double), ("ic0_levels", C.c_int32 * 2)]


class ToOcStats(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("volume", C.c_double), ("change", C.c_double), ("ms", C.c_double),
                ("steps", C.c_int32), ("state", C.c_int32), ("passes", C.c_int32)]


class ToOptParams(C.Structure):
    _fields_ = [("volfrac", C.c_double), ("move", C.c_double), ("eta", C.c_double), ("rho_o", C.c_double),
                ("penal0", C.c_double), ("penal_max", C.c_double), ("penal_step", C.c_double),
                ("stage_steps", C.c_int32), ("stop_on_converge", C.c_int32), ("change_tol", C.c_double),
                ("rtol", C.c_double), ("max_iter", C.c_int32), ("filter", C.c_int32),
                ("adapt_min_steps", C.c_int32), ("adapt_max_steps", C.c_int32)]


class ToOptState(C.Structure):
    _fields_ = [("penal", C.c_double), ("at_stage", C.c_int32), ("since_adapt", C.c_int32),
                ("adapt_due", C.c_int32), ("converged", C.c_int32)]


class AdaptResult(C.Structure):
    _fields_ = [("n_leaf", C.c_int64), ("leaf_level", P), ("leaf_anchor", P), ("leaf_x", P), ("marks", P),
                ("n_refined", C.c_int64), ("n_groups", C.c_int64), ("n_unmarked_sibling", C.c_int64),
                ("n_unmarked_incompat", C.c_int64)]


class ToOptStep(C.Structure):
    _fields_ = [("compliance", C.c_double), ("penal", C.c_double), ("volume", C.c_double),
                ("change", C.c_double), ("lambda_", C.c_double), ("solve_ms", C.c_double), ("oc_ms", C.c_double),
                ("cg_iters", C.c_int32), ("status", C.c_int32)]


class HostSpec(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("max_level", C.c_int32), ("base", C.c_int32 * 3), ("h0", C.c_double),
        ("n_leaf", C.c_int64), ("leaf_level", P), ("leaf_anchor", P),
        ("n_fixed_box", C.c_int32), ("fixed_box", P), ("fixed_mask", P),
        ("n_load", C.c_int32), ("load_kind", P), ("load_box", P), ("load_vec", P),
        ("rmin", C.c_double),
    ]


class HostArrays(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("max_level", C.c_int32), ("h0", C.c_double),
        ("n_elem", C.c_int64), ("n_node", C.c_int64), ("n_hang", C.c_int64), ("n_hang_nnz", C.c_int64),
        ("n_fixed", C.c_int64), ("filt_nnz", C.c_int64),
        ("elem_node", P), ("elem_anchor", P), ("elem_level", P), ("node_coord", P),
        ("hang_node", P), ("hang_ptr", P), ("hang_parent", P), ("hang_weight", P),
        ("fixed_dof", P), ("load", P), ("filt_ptr", P), ("filt_idx", P),
    ]


TO_SHARD_MAX = 16


class ToShardBufs(C.Structure):
    _fields_ = [("rb", P * 2), ("pb", P * 2), ("qb", P * 2), ("x", P), ("slots", P), ("flags", P),
                ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("pad", C.c_int32),
                ("plane_doubles", C.c_int64), ("dinv", P)]


EXPORTS = {
    # name: (restype, argtypes)
    "tomesh_upload": (C.c_int, [C.POINTER(ToMeshDesc), C.c_int, P, C.POINTER(P)]),
    "tomesh_free": (None, [P]),
    "tomesh_get_info": (C.c_int, [P, C.POINTER(ToMeshInfo)]),
    "tosolve_cg": (C.c_int, [P, C.c_double, P, P, C.c_double, C.c_int32, C.c_uint32, C.POINTER(ToCgStats), P]),
    "tosolve_minres": (C.c_int, [P, C.c_double, P, P, C.c_double, C.c_int32, C.c_int32, C.c_uint32,
                                 C.POINTER(ToMinresStats), P]),
    "tosolve_history": (C.c_int, [P, P, C.c_int32]),
    "tosolve_profile": (C.c_int, [P, P, C.c_int32]),
    "to_sensitivity": (C.c_int, [P, C.c_double, P, P, P, C.POINTER(C.c_double), P]),
    "to_filter": (C.c_int, [P, C.c_int32, P, P, P, P]),
    "to_oc_update": (C.c_int, [P, P, P, C.c_double, C.c_double, C.c_double, C.c_double, P,
                               C.POINTER(ToOcStats), P]),
    "to_optimize": (C.c_int, [P, C.POINTER(ToOptParams), C.c_int32, P, P, C.POINTER(ToOptStep),
                              C.POINTER(C.c_int32), C.POINTER(ToOptState), P]),
    "to_amr_mark": (C.c_int, [P, P, C.c_double, P, P]),
    "tomesh_host_adapt": (C.c_int, [P, P, P, C.POINTER(P)]),
    "tomesh_adapt_get": (C.c_int, [P, C.POINTER(AdaptResult)]),
    "tomesh_host_transfer": (C.c_int, [P, P, P]),
    "tomesh_adapt_free": (None, [P]),
    "to_apply_A": (C.c_int, [P, C.c_double, P, P, P, P]),
    "to_jacobi_diag": (C.c_int, [P, C.c_double, P, P, P]),
    "to_project_rhs": (C.c_int, [P, P, P]),
    "to_recover": (C.c_int, [P, P, P, P]),
    "to_element_matrix": (C.c_int, [C.c_int32, C.c_double, P]),
    "to_element_hadamard": (C.c_int, [C.c_double, P, P]),
    "to_last_error": (C.c_char_p, []),
    "to_shard_buffers": (C.c_int, [P, C.POINTER(ToShardBufs), P]),
    "to_shard_attach": (C.c_int, [P, C.c_int32, C.c_int32, P, C.c_int32, C.c_int32, C.POINTER(ToShardBufs), P]),
    "to_gshard_attach": (C.c_int, [P, C.c_int32, C.c_int32, C.POINTER(ToShardBufs), C.c_int64, P, P, P, P]),
    "tosolve_cg_group": (C.c_int, [P, C.c_int32, C.c_double, P, P, C.c_double, C.c_int32, C.c_uint32,
                                   C.POINTER(ToCgStats), P]),
    "to_ipc_export": (C.c_int, [P, P, P, C.POINTER(C.c_uint64)]),
    "to_ipc_open": (C.c_int, [C.c_int, P, C.c_uint64, C.POINTER(P)]),
    "to_ipc_close": (C.c_int, [C.c_int, P]),
    "tomesh_host_build": (C.c_int, [C.POINTER(HostSpec), C.POINTER(P)]),
    "tomesh_host_get": (C.c_int, [P, C.POINTER(HostArrays)]),
    "tomesh_host_filter": (C.c_int, [P, C.c_double]),
    "tomesh_host_free": (None, [P]),
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libtomesh.so not built ({LIB_PATH}); run __graft_entry__.build() "
                              "or python -m paper_1009_4975_b200.build — there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class TomeshError(RuntimeError):
    def __init__(self, code: int, where: str):
        msg = lib().to_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS_NAMES.get(code, code)} ({code}): {msg}")
        self.code = code


def check(code: int, where: str, ok_positive: bool = True) -> int:
    if code < 0 or (code > 0 and not ok_positive):
        raise TomeshError(code, where)
    return code
