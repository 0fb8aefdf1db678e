"""Keys and paths of the cached converged oracle references (test
infrastructure; written by tools/oracle_reference.py, which calls only
`oracle/`).  The key hashes the oracle's own input arrays and the solve
tolerance, so a changed recipe or oracle mesh never matches a stale file."""
from __future__ import annotations

import hashlib
import os

import numpy as np

from inputs import config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CACHE_DIR = os.path.join(ROOT, "cache", "oracle_ref")


def variant(name: str):
    """BASELINE configs by name; 'c4L' is the documented large c4 recipe
    variant."""
    if name == "c4L":
        from inputs.problems import config_c4L
        return config_c4L()
    return config(name)


def input_key(prob, om, x, rtol) -> str:
    h = hashlib.sha256()
    h.update(repr((prob.name, prob.dim, prob.L, prob.base, prob.E0, prob.Emin, prob.nu,
                   prob.penal, prob.rmin, float(rtol))).encode())
    for a in (om.elem_node, om.hang_node, om.hang_ptr, om.hang_parent, om.hang_weight,
              om.fixed_dof, om.load, np.asarray(x, dtype=np.float64)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def cache_path(name: str, key: str) -> str:
    return os.path.join(CACHE_DIR, f"{name}_{key}.npz")
