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


# A committed digest of each cached reference (tests/golden/, ~1 MB per
# config): u at 65,536 sampled DOFs, dc and the filtered dc at 32,768 sampled
# elements, the compliance and the iteration count, written by
# tools/oracle_reference.py from the oracle's own solution.  The full-size L2
# test falls back to it when cache/oracle_ref/ (git-ignored, 100+ MB for c5)
# is not there, so the converged 1e-8 comparison never depends on a directory
# that a re-created container loses.
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")
N_SAMPLE_DOF, N_SAMPLE_EL = 65536, 32768


def digest_path(name: str, key: str) -> str:
    return os.path.join(GOLDEN_DIR, f"oracle_ref_digest_{name}_{key}.npz")


def sample_indices(key: str, n: int, k: int, salt: int) -> np.ndarray:
    """k distinct indices of range(n), a function of the input key alone."""
    rng = np.random.default_rng([int(key, 16), salt])
    return np.sort(rng.choice(n, size=min(k, n), replace=False)).astype(np.int64)
