"""The paper's Test 2 comparison (Fig. 7-8), synthetic stand-in:
a 3D 2:1:1 cantilever optimised on a fixed uniform 128x32x32 H8 mesh and with
the dynamic AMR strategy started from 64x16x16 (one refinement level, so the
finest local resolution equals the uniform mesh), V0 = 25%, filter radius =
r_amr = 1.5 fine elements, p-continuation.  The paper's load case is only in a
figure; here the x = 0 face is clamped and a unit line load acts in -y along
the edge {x = 128, y = 0} (the c3 load case).  Everything runs through the
library (to_optimize on the uniform mesh; paper_1009_4975_b200.amr for AMR).

Prints one JSON line: total device-side wall time, CG iterations, element /
DOF counts of both runs, the compliance of each, and the design difference D
of Eq. 10 between the final designs on the fine lattice.

    python tools/amr_test2.py [steps] [rmin] [change_tol] [stop_rule]
    (change_tol > 0: run to convergence at p = 3; stop_rule "mesh" (default) or "design")
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1009_4975_b200 as pb
from inputs import DensitySpec, make_problem, uniform_leaves

NX, NY, NZ = 128, 32, 32


def problem(amr, rmin=1.5):
    base = (NX // 2, NY // 2, NZ // 2) if amr else (NX, NY, NZ)
    L = 1 if amr else 0
    return make_problem("test2_cantilever3d_" + ("amr" if amr else "uniform"), 3, base, L=L,
                        h0=2.0 if amr else 1.0, leaves=uniform_leaves(3, base, L, 0),
                        density=DensitySpec("const", value=0.25),
                        fixed=[((0, 0, 0), (0, NY, NZ), 0b111)],
                        loads=[("line", (NX, 0, 0), (NX, 0, NZ), (0.0, -1.0, 0.0))], rmin=rmin, rtol=1e-8)


def raster(host, x):
    """Densities on the fine lattice (lexicographic NX x NY x NZ)."""
    out = np.zeros((NZ, NY, NX))
    s = 1 << (host.L - host.elem_level.astype(np.int64))
    for e in range(host.n_el):
        a = host.elem_anchor[e]
        out[a[2]:a[2] + s[e], a[1]:a[1] + s[e], a[0]:a[0] + s[e]] = x[e]
    return out


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    rmin = float(sys.argv[2]) if len(sys.argv) > 2 else 1.5
    tol = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
    stop_rule = sys.argv[4] if len(sys.argv) > 4 else "mesh"
    conv = tol > 0
    volfrac, stage = 0.25, 12
    # uniform fine mesh
    pu = problem(False, rmin)
    hu = pb.prepare(pu)
    mu = pb.Mesh(hu, E0=pu.E0, Emin=pu.Emin, nu=pu.nu, rmin=pu.rmin)
    xu = torch.full((hu.n_el,), volfrac, dtype=torch.float64, device="cuda")
    uu = torch.zeros(hu.n_dof, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, hist_u = mu.to_optimize(xu, uu, steps, volfrac, stage_steps=stage, rtol=1e-8, stop_on_converge=conv,
                               change_tol=tol if conv else 0.01)
    torch.cuda.synchronize()
    wall_u = time.perf_counter() - t0
    # dynamic AMR
    pa = problem(True, rmin)
    t0 = time.perf_counter()
    run = pb.amr.optimize_amr(pa, volfrac, steps, stage_steps=stage, rtol=1e-8, stop_on_converge=conv,
                              change_tol=tol if conv else 0.01, stop_rule=stop_rule)
    torch.cuda.synchronize()
    wall_a = time.perf_counter() - t0
    ru = raster(hu, xu.cpu().numpy())
    ra = raster(run.host, run.x.cpu().numpy())
    D = float(np.abs(ru - ra).sum() / ru.sum())
    line = {
        "workload": "test2_cantilever3d_128x32x32", "step_cap": steps, "rmin": rmin, "change_tol": tol,
        "stop_rule": stop_rule,
        "volfrac": volfrac,
        "uniform": {"steps": len(hist_u), "n_elem": hu.n_el, "n_dof": hu.n_dof, "wall_s": wall_u,
                    "solve_ms": float(sum(h["solve_ms"] for h in hist_u)),
                    "cg_iters": int(sum(h["cg_iters"] for h in hist_u)),
                    "compliance_last": hist_u[-1]["compliance"], "structured": mu.info()["structured"]},
        "amr": {"steps": len(run.steps), "n_elem_first_last": [run.steps[0]["n_elem"], run.host.n_el],
                "n_dof_last": run.host.n_dof,
                "wall_s": wall_a, "solve_ms": float(sum(h["solve_ms"] for h in run.steps)),
                "cg_iters": int(sum(h["cg_iters"] for h in run.steps)),
                "compliance_last": run.steps[-1]["compliance"], "adaptations": len(run.adaptations),
                "mean_n_elem": float(np.mean([h["n_elem"] for h in run.steps]))},
        "design_difference_D": D,
        "time_ratio_uniform_over_amr": wall_u / wall_a,
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
