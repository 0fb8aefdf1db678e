"""Thin Python binding of libtomesh (argument marshalling only).

Every step of the hot path runs in the library's CUDA kernels (device
calls) or its C++ host builder (mesh preparation).  torch is used for device
memory and streams only.  Names follow include/tomesh.h.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib as L


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _copy(ptr, dtype, count, shape=None):
    if count == 0 or not ptr:
        out = np.zeros(0 if shape is None else (0,) + tuple(shape[1:]), dtype=dtype)
        return out
    buf = (C.c_byte * (count * np.dtype(dtype).itemsize)).from_address(ptr)
    out = np.frombuffer(buf, dtype=dtype, count=count).copy()
    return out.reshape(shape) if shape is not None else out


# ---------------------------------------------------------------------------
# host mesh preparation (C++ host builder, include/tomesh_host.h)
# ---------------------------------------------------------------------------

@dataclass
class HostMesh:
    dim: int
    L: int
    h0: float
    elem_node: np.ndarray
    elem_anchor: np.ndarray
    elem_level: np.ndarray
    node_coord: np.ndarray
    hang_node: np.ndarray
    hang_ptr: np.ndarray
    hang_parent: np.ndarray
    hang_weight: np.ndarray
    fixed_dof: np.ndarray
    load: np.ndarray
    filt_ptr: Optional[np.ndarray]
    filt_idx: Optional[np.ndarray]
    rmin: float
    handle: Optional["_HostHandle"] = None   # the tomesh_host* (kept for tomesh_host_adapt)

    @property
    def n_el(self):
        return int(self.elem_level.shape[0])

    @property
    def n_node(self):
        return int(self.node_coord.shape[0])

    @property
    def n_dof(self):
        return self.dim * self.n_node

    @property
    def hL(self):
        return self.h0 / (1 << self.L)


class _HostHandle:
    """Owns a tomesh_host* (freed with the object)."""

    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            if self.h and self.h.value:
                L.lib().tomesh_host_free(self.h)
        except Exception:
            pass


_KIND = {"point": L.TOH_LOAD_POINT, "line": L.TOH_LOAD_LINE, "face": L.TOH_LOAD_FACE}


def tomesh_host_build(dim, max_level, base, h0, leaf_level, leaf_anchor, fixed, loads, rmin,
                      keep_handle=False) -> HostMesh:
    """fixed: [(lo, hi, mask)], loads: [(kind, lo, hi, vec)] (lattice boxes, inclusive).
    keep_handle: keep the C mesh alive (needed by tomesh_host_adapt / _transfer)."""
    lib = L.lib()
    leaf_level = np.ascontiguousarray(leaf_level, dtype=np.int8)
    leaf_anchor = np.ascontiguousarray(leaf_anchor, dtype=np.int32).reshape(-1, dim)
    fb = np.ascontiguousarray([list(lo) + list(hi) for lo, hi, _ in fixed] or [[0] * 2 * dim], dtype=np.int32)
    fm = np.ascontiguousarray([m for _, _, m in fixed] or [0], dtype=np.int32)
    lk = np.ascontiguousarray([_KIND[k] for k, _, _, _ in loads] or [0], dtype=np.int32)
    lb = np.ascontiguousarray([list(lo) + list(hi) for _, lo, hi, _ in loads] or [[0] * 2 * dim], dtype=np.int32)
    lv = np.ascontiguousarray([list(v) for _, _, _, v in loads] or [[0.0] * dim], dtype=np.float64)
    spec = L.HostSpec()
    spec.dim = dim
    spec.max_level = max_level
    for c in range(3):
        spec.base[c] = int(base[c]) if c < dim else 1
    spec.h0 = h0
    spec.n_leaf = leaf_level.shape[0]
    spec.leaf_level = _ptr(leaf_level)
    spec.leaf_anchor = _ptr(leaf_anchor)
    spec.n_fixed_box = len(fixed)
    spec.fixed_box = _ptr(fb)
    spec.fixed_mask = _ptr(fm)
    spec.n_load = len(loads)
    spec.load_kind = _ptr(lk)
    spec.load_box = _ptr(lb)
    spec.load_vec = _ptr(lv)
    spec.rmin = float(rmin)
    h = C.c_void_p()
    L.check(lib.tomesh_host_build(C.byref(spec), C.byref(h)), "tomesh_host_build")
    handle = _HostHandle(h)
    a = L.HostArrays()
    L.check(lib.tomesh_host_get(h, C.byref(a)), "tomesh_host_get")
    nc = 1 << dim
    ne, nn = a.n_elem, a.n_node
    return HostMesh(
        dim=dim, L=max_level, h0=h0,
        elem_node=_copy(a.elem_node, np.int32, ne * nc, (ne, nc)),
        elem_anchor=_copy(a.elem_anchor, np.int32, ne * dim, (ne, dim)),
        elem_level=_copy(a.elem_level, np.int8, ne),
        node_coord=_copy(a.node_coord, np.int32, nn * dim, (nn, dim)),
        hang_node=_copy(a.hang_node, np.int32, a.n_hang),
        hang_ptr=_copy(a.hang_ptr, np.int32, a.n_hang + 1),
        hang_parent=_copy(a.hang_parent, np.int32, a.n_hang_nnz),
        hang_weight=_copy(a.hang_weight, np.float64, a.n_hang_nnz),
        fixed_dof=_copy(a.fixed_dof, np.int64, a.n_fixed),
        load=_copy(a.load, np.float64, nn * dim),
        filt_ptr=_copy(a.filt_ptr, np.int64, ne + 1) if a.filt_ptr else None,
        filt_idx=_copy(a.filt_idx, np.int32, a.filt_nnz) if a.filt_ptr else None,
        rmin=float(rmin),
        handle=handle if keep_handle else None,
    )


def prepare(problem, keep_handle=False) -> HostMesh:
    """Host mesh for an ``inputs.Problem`` (its pre-balance leaves and predicates)."""
    p = problem
    return tomesh_host_build(p.dim, p.L, p.base, p.h0, p.leaf_level, p.leaf_anchor, p.fixed, p.loads, p.rmin,
                             keep_handle)


@dataclass
class Adaptation:
    """Result of tomesh_host_adapt: the new pre-balance leaves (ascending Morton
    order) with transferred densities, the marks after the two sweeps, counts."""
    leaf_level: np.ndarray
    leaf_anchor: np.ndarray
    leaf_x: np.ndarray
    marks: np.ndarray
    n_refined: int
    n_groups: int
    n_unmarked_sibling: int
    n_unmarked_incompat: int
    handle: object = None


class _AdaptHandle:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            if self.h and self.h.value:
                L.lib().tomesh_adapt_free(self.h)
        except Exception:
            pass


def tomesh_host_adapt(host: HostMesh, marks, x) -> Adaptation:
    """Sweeps + refine/derefine on the host (include/tomesh_host.h)."""
    if host.handle is None:
        raise ValueError("host mesh built without keep_handle=True")
    marks = np.ascontiguousarray(marks, dtype=np.int8)
    x = np.ascontiguousarray(x, dtype=np.float64)
    if marks.shape[0] != host.n_el or x.shape[0] != host.n_el:
        raise ValueError("marks and x need one value per element")
    h = C.c_void_p()
    L.check(L.lib().tomesh_host_adapt(host.handle.h, _ptr(marks), _ptr(x), C.byref(h)), "tomesh_host_adapt")
    ah = _AdaptHandle(h)
    r = L.AdaptResult()
    L.check(L.lib().tomesh_adapt_get(h, C.byref(r)), "tomesh_adapt_get")
    n, dim = r.n_leaf, host.dim
    return Adaptation(_copy(r.leaf_level, np.int8, n), _copy(r.leaf_anchor, np.int32, n * dim, (n, dim)),
                      _copy(r.leaf_x, np.float64, n), _copy(r.marks, np.int8, host.n_el),
                      r.n_refined, r.n_groups, r.n_unmarked_sibling, r.n_unmarked_incompat, ah)


def tomesh_host_transfer(host_new: HostMesh, ad: Adaptation) -> np.ndarray:
    out = np.empty(host_new.n_el, dtype=np.float64)
    L.check(L.lib().tomesh_host_transfer(host_new.handle.h, ad.handle.h, _ptr(out)), "tomesh_host_transfer")
    return out


def rebuild(problem, ad: Adaptation) -> HostMesh:
    """Host mesh of the adapted leaf set with the problem's boundary boxes and loads."""
    p = problem
    return tomesh_host_build(p.dim, p.L, p.base, p.h0, ad.leaf_level, ad.leaf_anchor, p.fixed, p.loads, p.rmin,
                             keep_handle=True)


# ---------------------------------------------------------------------------
# device handle (include/tomesh.h)
# ---------------------------------------------------------------------------

@dataclass
class CgStats:
    iters: int
    status: int
    relres: float
    relres_true: float
    ms: float
    bnorm: float


@dataclass
class OcStats:
    lam: float
    volume: float
    change: float
    ms: float
    steps: int
    state: int          # 0 active, 1 inactive, 2 infeasible
    passes: int         # passes over the elements


def _dptr(t):
    import torch
    if t is None:
        return None
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError("expected a contiguous float64 CUDA tensor")
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def make_desc(host: HostMesh, E0, Emin, nu, rmin, options=0, n_owned=0):
    """to_mesh_desc of a host mesh (argument marshalling only); returns the
    struct and the numpy arrays it points into (keep them alive)."""
    keep = []

    def arr(a, dt):
        a = np.ascontiguousarray(a, dtype=dt)
        keep.append(a)
        return _ptr(a)

    d = L.ToMeshDesc()
    d.dim = host.dim
    d.max_level = host.L
    d.h0 = host.h0
    d.n_elem = host.n_el
    d.n_node = host.n_node
    d.elem_node = arr(host.elem_node, np.int32)
    d.elem_anchor = arr(host.elem_anchor, np.int32)
    d.elem_level = arr(host.elem_level, np.int8)
    d.n_hang = host.hang_node.shape[0]
    d.hang_node = arr(host.hang_node, np.int32)
    d.hang_ptr = arr(host.hang_ptr, np.int32)
    d.hang_parent = arr(host.hang_parent, np.int32)
    d.hang_weight = arr(host.hang_weight, np.float64)
    d.n_fixed = host.fixed_dof.shape[0]
    d.fixed_dof = arr(host.fixed_dof, np.int64)
    d.load = arr(host.load, np.float64)
    d.E0, d.Emin, d.nu = E0, Emin, nu
    d.rmin = rmin if host.filt_ptr is not None else 0.0
    if host.filt_ptr is not None and rmin > 0:
        d.filt_nnz = host.filt_idx.shape[0]
        d.filt_ptr = arr(host.filt_ptr, np.int64)
        d.filt_idx = arr(host.filt_idx, np.int32)
    d.options = int(options)
    d.n_owned = int(n_owned)
    return d, keep


class Mesh:
    """Device copy of a mesh + CG workspace (tomesh_upload / tomesh_free)."""

    def __init__(self, host: HostMesh, E0=1.0, Emin=1e-9, nu=0.3, rmin=None, device=0, stream=None, options=0,
                 n_owned=0):
        """options: TO_UPLOAD_* bits of include/tomesh.h (which device code
        applies the operator; the operator itself does not change).  n_owned
        > 0: a rank's local mesh of a general-path shard group (nodes
        [0, n_owned) owned; paper_1009_4975_b200.amr_shard)."""
        import torch
        self.host = host
        self.device = torch.device("cuda", device)
        self.dim = host.dim
        self.n_el, self.n_node, self.n_dof = host.n_el, host.n_node, host.n_dof
        self.E0, self.Emin, self.nu = E0, Emin, nu
        rmin = host.rmin if rmin is None else rmin
        d, self._keep = make_desc(host, E0, Emin, nu, rmin, options, n_owned)
        self._h = C.c_void_p()
        with torch.cuda.device(self.device):
            L.check(L.lib().tomesh_upload(C.byref(d), device, _stream(stream), C.byref(self._h)), "tomesh_upload")

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            L.lib().tomesh_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        i = L.ToMeshInfo()
        L.check(L.lib().tomesh_get_info(self._h, C.byref(i)), "tomesh_get_info")
        return {f: (list(getattr(i, f)) if f == "grid" else getattr(i, f)) for f, _ in L.ToMeshInfo._fields_}

    # -- the four calls of the boundary --------------------------------------------------
    def tosolve_cg(self, penal, x, u, rtol=1e-10, max_iter=20000, flags=0, stream=None) -> CgStats:
        st = L.ToCgStats()
        rc = L.lib().tosolve_cg(self._h, float(penal), _dptr(x), _dptr(u), float(rtol), int(max_iter),
                                int(flags), C.byref(st), _stream(stream))
        L.check(rc, "tosolve_cg")
        return CgStats(st.iters, st.status, st.relres, st.relres_true, st.ms, st.bnorm)

    # -- z-slab sharding (include/tomesh.h to_shard_*; paper_1009_4975_b200.shard) -------
    def shard_buffers(self, stream=None) -> "L.ToShardBufs":
        b = L.ToShardBufs()
        L.check(L.lib().to_shard_buffers(self._h, C.byref(b), _stream(stream)), "to_shard_buffers")
        return b

    def shard_attach(self, rank, nranks, gz_lo, own_lo, own_hi, peers, stream=None):
        gz = np.ascontiguousarray(gz_lo, dtype=np.int32)
        arr = (L.ToShardBufs * nranks)(*peers)
        L.check(L.lib().to_shard_attach(self._h, int(rank), int(nranks), _ptr(gz), int(own_lo), int(own_hi), arr,
                                        _stream(stream)), "to_shard_attach")

    def gshard_attach(self, rank, nranks, peers, send_rank, send_local, send_remote, stream=None):
        """to_gshard_attach: send entry i stores owned local node send_local[i]
        into ghost node send_remote[i] of rank send_rank[i]."""
        arr = (L.ToShardBufs * nranks)(*peers)
        sr = np.ascontiguousarray(send_rank, dtype=np.int32)
        sl = np.ascontiguousarray(send_local, dtype=np.int32)
        sm = np.ascontiguousarray(send_remote, dtype=np.int32)
        L.check(L.lib().to_gshard_attach(self._h, int(rank), int(nranks), arr, int(sr.shape[0]), _ptr(sr), _ptr(sl),
                                         _ptr(sm), _stream(stream)), "to_gshard_attach")

    def ipc_export(self, dev_ptr):
        h = (C.c_byte * 64)()
        off = C.c_uint64()
        L.check(L.lib().to_ipc_export(self._h, C.c_void_p(dev_ptr), h, C.byref(off)), "to_ipc_export")
        return bytes(h), int(off.value)

    def tosolve_minres(self, penal, x, u, rtol=1e-10, max_iter=20000, precond=0, flags=0, stream=None) -> dict:
        """The paper's solver: MINRES on the rescaled system, precond 0 = rescaling
        only (TO_PC_JACOBI), 1 = IC(0) of the rescaled matrix (TO_PC_IC0)."""
        st = L.ToMinresStats()
        rc = L.lib().tosolve_minres(self._h, float(penal), _dptr(x), _dptr(u), float(rtol), int(max_iter),
                                    int(precond), int(flags), C.byref(st), _stream(stream))
        L.check(rc, "tosolve_minres")
        out = {f: getattr(st, f) for f, _ in L.ToMinresStats._fields_}
        out["ic0_levels"] = list(out["ic0_levels"])
        return out

    def history(self, n):
        out = np.zeros(max(1, n))
        k = L.lib().tosolve_history(self._h, _ptr(out), int(n))
        L.check(k, "tosolve_history")
        return out[:k]

    def profile(self):
        out = np.zeros(6)
        L.check(L.lib().tosolve_profile(self._h, _ptr(out), 6), "tosolve_profile")
        return {"apply_ms": out[0], "alpha_ms": out[1], "u1_ms": out[2], "u2_ms": out[3], "iters": int(out[4]),
                "loop_ms": out[5]}

    def to_sensitivity(self, penal, x, u, dc, compliance=False, stream=None):
        c = C.c_double(0.0)
        L.check(L.lib().to_sensitivity(self._h, float(penal), _dptr(x), _dptr(u), _dptr(dc),
                                       C.byref(c) if compliance else None, _stream(stream)), "to_sensitivity")
        return c.value if compliance else None

    def to_filter(self, mode, x, inp, out, stream=None):
        L.check(L.lib().to_filter(self._h, int(mode), _dptr(x), _dptr(inp), _dptr(out), _stream(stream)),
                "to_filter")
        return out

    # -- the design update and the Fig. 1 loop ----------------------------------------------
    def to_oc_update(self, x, dc, volfrac, x_new, move=0.2, eta=0.5, rho_o=1e-3, stream=None) -> OcStats:
        st = L.ToOcStats()
        L.check(L.lib().to_oc_update(self._h, _dptr(x), _dptr(dc), float(volfrac), float(move), float(eta),
                                     float(rho_o), _dptr(x_new), C.byref(st), _stream(stream)), "to_oc_update")
        return OcStats(st.lambda_, st.volume, st.change, st.ms, st.steps, st.state, st.passes)

    def to_optimize(self, x, u, n_steps, volfrac, penal0=1.0, penal_max=3.0, penal_step=0.5, stage_steps=30,
                    stop_on_converge=False, change_tol=0.01, move=0.2, eta=0.5, rho_o=1e-3, rtol=1e-10,
                    max_iter=20000, filter=True, adapt_min_steps=0, adapt_max_steps=0, state=None, stream=None):
        """Runs the Fig. 1 loop in the library; x is updated in place.  `state`
        (an _lib.ToOptState) carries continuation/adaptation counters across
        calls.  Returns (status, list of per-step dicts)."""
        P = L.ToOptParams(volfrac=volfrac, move=move, eta=eta, rho_o=rho_o, penal0=penal0, penal_max=penal_max,
                          penal_step=penal_step, stage_steps=stage_steps, stop_on_converge=int(stop_on_converge),
                          change_tol=change_tol, rtol=rtol, max_iter=max_iter, filter=int(filter),
                          adapt_min_steps=adapt_min_steps, adapt_max_steps=adapt_max_steps)
        hist = (L.ToOptStep * max(1, n_steps))()
        done = C.c_int32(0)
        rc = L.lib().to_optimize(self._h, C.byref(P), int(n_steps), _dptr(x), _dptr(u), hist, C.byref(done),
                                 C.byref(state) if state is not None else None, _stream(stream))
        L.check(rc, "to_optimize")
        out = [{f: getattr(hist[k], f) for f, _ in L.ToOptStep._fields_} for k in range(done.value)]
        for h in out:
            h["lam"] = h.pop("lambda_")
        return rc, out

    def to_amr_mark(self, x, marks, rho_s=0.5, stream=None):
        """marks: int8 CUDA tensor [n_el] (+1 refine, -1 derefine, 0 keep)."""
        import torch
        if not (marks.is_cuda and marks.dtype == torch.int8 and marks.is_contiguous()):
            raise ValueError("marks must be a contiguous int8 CUDA tensor")
        L.check(L.lib().to_amr_mark(self._h, _dptr(x), float(rho_s), C.c_void_p(marks.data_ptr()),
                                    _stream(stream)), "to_amr_mark")
        return marks

    # -- operator-level calls -------------------------------------------------------------
    def to_apply_A(self, penal, x, v, q, stream=None):
        L.check(L.lib().to_apply_A(self._h, float(penal), _dptr(x), _dptr(v), _dptr(q), _stream(stream)), "to_apply_A")
        return q

    def to_jacobi_diag(self, penal, x, d, stream=None):
        L.check(L.lib().to_jacobi_diag(self._h, float(penal), _dptr(x), _dptr(d), _stream(stream)), "to_jacobi_diag")
        return d

    def to_project_rhs(self, b, stream=None):
        L.check(L.lib().to_project_rhs(self._h, _dptr(b), _stream(stream)), "to_project_rhs")
        return b

    def to_recover(self, v, u, stream=None):
        L.check(L.lib().to_recover(self._h, _dptr(v), _dptr(u), _stream(stream)), "to_recover")
        return u


def tosolve_cg_group(meshes, penal, xs, us, rtol=1e-10, max_iter=20000, flags=0, streams=None):
    """tosolve_cg on attached shard handles in lockstep (include/tomesh.h)."""
    n = len(meshes)
    hs = (C.c_void_p * n)(*[m._h for m in meshes])
    xp = (C.c_void_p * n)(*[_dptr(x) for x in xs])
    up = (C.c_void_p * n)(*[_dptr(u) for u in us])
    sp = (C.c_void_p * n)(*[_stream(None if streams is None else streams[i]) for i in range(n)])
    st = (L.ToCgStats * n)()
    rc = L.lib().tosolve_cg_group(hs, n, float(penal), xp, up, float(rtol), int(max_iter), int(flags), st, sp)
    L.check(rc, "tosolve_cg_group")
    return [CgStats(s.iters, s.status, s.relres, s.relres_true, s.ms, s.bnorm) for s in st]


def ipc_open(device, handle: bytes, offset: int) -> int:
    h = (C.c_byte * 64).from_buffer_copy(handle)
    p = C.c_void_p()
    L.check(L.lib().to_ipc_open(int(device), h, C.c_uint64(offset), C.byref(p)), "to_ipc_open")
    return int(p.value)


def ipc_close(device, base_ptr: int):
    L.check(L.lib().to_ipc_close(int(device), C.c_void_p(base_ptr)), "to_ipc_close")
