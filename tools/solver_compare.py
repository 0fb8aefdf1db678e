"""The paper's solver against the B200 path's, per config:
Jacobi-PCG (tosolve_cg), MINRES on the rescaled system (tosolve_minres,
TO_PC_JACOBI) and MINRES + IC(0) (TO_PC_IC0), to the config's tolerance on
the config's input density.  One JSON line per config and solver.

    python tools/solver_compare.py [c1 c2 c4]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1009_4975_b200 as pb
from inputs import config, density_at


def main(names):
    for name in names:
        prob = config(name)
        hm = pb.prepare(prob)
        m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
        x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda")
        u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
        rtol = prob.rtol
        m.tosolve_cg(prob.penal, x, u, rtol=rtol, max_iter=100000)          # warm-up
        st = m.tosolve_cg(prob.penal, x, u, rtol=rtol, max_iter=100000)
        rows = [{"solver": "jacobi_pcg", "iters": st.iters, "ms": st.ms, "relres_true": st.relres_true}]
        for pc, label in ((pb.TO_PC_JACOBI, "minres_rescaled"), (pb.TO_PC_IC0, "minres_ic0")):
            if pc == pb.TO_PC_IC0 and hm.n_dof > 60000:
                # natural-order IC(0) solves are dependency chains: ~n levels, tens of ms per
                # iteration at c2 size already (measured); skipped above that size
                rows.append({"solver": label, "skipped": "natural-order triangular solves too deep", "iters": 0,
                             "ms": 0.0})
                continue
            t0 = time.perf_counter()
            s1 = m.tosolve_minres(prob.penal, x, u, rtol=rtol, max_iter=100000, precond=pc)   # includes IC(0) setup once
            first_s = time.perf_counter() - t0
            s2 = m.tosolve_minres(prob.penal, x, u, rtol=rtol, max_iter=100000, precond=pc)
            rows.append({"solver": label, "iters": s2["iters"], "ms": s2["ms"], "relres_true": s2["relres_true"],
                         "ic0_shift": s2["ic0_shift"], "ic0_levels": s2["ic0_levels"], "first_call_s": first_s})
        for r in rows:
            r.update({"config": name, "n_dof": hm.n_dof, "rtol": rtol,
                      "us_per_iter": 1000.0 * r["ms"] / max(1, r["iters"])})
            print(json.dumps(r), flush=True)
        m.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c4"])
