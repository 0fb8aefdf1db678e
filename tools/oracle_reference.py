"""Converged oracle references for the full-size L2 parity tests (SURVEY §8(c)
"Configs 4-5 compare against a cached oracle reference").

Calls only `oracle/` (pipeline.run: assembled A, textbook Jacobi-PCG to
rel-residual `rtol`, recovery Eq. 9, compliance, sensitivities, Eq. 5 filter)
and writes u, c, dc and the filtered dc to
`cache/oracle_ref/<config>_<key>.npz`, where <key> hashes the oracle's own
input arrays (tests/oracle_cache.py recomputes it).  The directory is
git-ignored (c5's u alone is 103 MB) but travels to the GPU box with the
gpurun snapshot.  Nothing here ever reads a device output.

    python tools/oracle_reference.py c3 c4 [--rtol 1e-10]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from inputs import config  # noqa: E402
from oracle import mesh as omesh, pipeline  # noqa: E402
from tests.oracle_cache import (N_SAMPLE_DOF, N_SAMPLE_EL, cache_path, digest_path, input_key,  # noqa: E402
                                sample_indices, variant)


def write_digest(name, key, path):
    """tests/golden/oracle_ref_digest_<name>_<key>.npz from the cached oracle
    solution at `path`: sampled entries of u, dc and the filtered dc (indices a
    function of the key), the compliance and the solve's meta."""
    ref = np.load(path)
    u, dc, dcf = ref["u"], ref["dc"], ref["dcf"]
    sd = sample_indices(key, u.shape[0], N_SAMPLE_DOF, 1)
    se = sample_indices(key, dc.shape[0], N_SAMPLE_EL, 2)
    out = digest_path(name, key)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    np.savez_compressed(out, u=u[sd], dc=dc[se], dcf=dcf[se], compliance=ref["compliance"], meta=ref["meta"],
                        n_dof=np.int64(u.shape[0]), n_el=np.int64(dc.shape[0]),
                        idx_sum=np.int64(sd.sum() + se.sum()))
    print(f"{name}: digest {os.path.relpath(out, ROOT)} ({os.path.getsize(out) / 1e6:.2f} MB)", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+")
    ap.add_argument("--rtol", type=float, default=1e-10)
    args = ap.parse_args()
    for name in args.names:
        t0 = time.perf_counter()
        prob = variant(name)
        om = omesh.build_mesh(prob)
        x = pipeline.input_density(prob, om)
        key = input_key(prob, om, x, args.rtol)
        path = cache_path(name, key)
        if os.path.exists(path):
            print(f"{name}: {path} exists", flush=True)
            if not os.path.exists(digest_path(name, key)):
                write_digest(name, key, path)
            continue
        t_mesh = time.perf_counter() - t0
        print(f"{name}: n_el={om.n_el} n_dof={om.n_dof} n_hang={om.hang_node.shape[0]} "
              f"mesh {t_mesh:.1f}s key {key}", flush=True)
        r = pipeline.run(prob, rtol=args.rtol, m=om, x=x)
        meta = dict(config=name, key=key, rtol=args.rtol, iters=r.cg.iters, relres=r.cg.relres,
                    relres_true=r.cg.relres_true, converged=bool(r.cg.converged),
                    n_el=int(om.n_el), n_dof=int(om.n_dof), timings=r.timings, t_mesh=t_mesh,
                    threads=1, wall_s=time.perf_counter() - t0)
        os.makedirs(os.path.dirname(path), exist_ok=True)
        tmp = path + ".tmp.npz"
        np.savez(tmp, u=r.u, dc=r.dc, dcf=r.dc_filtered, compliance=np.float64(r.compliance),
                 meta=json.dumps(meta))
        os.replace(tmp, path)
        write_digest(name, key, path)
        print(json.dumps(meta), flush=True)


if __name__ == "__main__":
    main()
