"""The committed digests of the cached oracle references (tests/golden/
oracle_ref_digest_*.npz, written by tools/oracle_reference.py from the
oracle's own converged solutions): each one is self-consistent, i.e. its sample
indices are reproduced from its key, its sizes match the config it names, and
the oracle solve it was cut from had converged to the stated tolerance."""
import glob
import json
import os

import numpy as np
import pytest

from tests.oracle_cache import GOLDEN_DIR, N_SAMPLE_DOF, N_SAMPLE_EL, sample_indices

FILES = sorted(glob.glob(os.path.join(GOLDEN_DIR, "oracle_ref_digest_*.npz")))


def test_digests_present():
    assert {os.path.basename(f).split("_")[3] for f in FILES} >= {"c3", "c4", "c4L"}


@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(f) for f in FILES])
def test_digest_self_consistent(path):
    name, key = os.path.basename(path)[:-4].split("_")[3:5]
    d = np.load(path)
    meta = json.loads(str(d["meta"]))
    assert meta["config"] == name and meta["key"] == key and meta["converged"] and meta["relres"] <= 1e-10
    n_dof, n_el = int(d["n_dof"]), int(d["n_el"])
    assert (n_dof, n_el) == (meta["n_dof"], meta["n_el"])
    sd = sample_indices(key, n_dof, N_SAMPLE_DOF, 1)
    se = sample_indices(key, n_el, N_SAMPLE_EL, 2)
    assert int(d["idx_sum"]) == int(sd.sum() + se.sum())
    assert d["u"].shape == sd.shape and d["dc"].shape == se.shape == d["dcf"].shape
    assert np.all(np.diff(sd) > 0) and np.all(np.diff(se) > 0)
    assert np.all(np.isfinite(d["u"])) and np.all(d["dc"] <= 0.0) and float(d["compliance"]) > 0.0
