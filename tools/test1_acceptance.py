"""The paper's Test 1 claim at desk scale (SPEC.md:541-543 A1-A3),
entirely on the device path:

  uniform  the 2:1 cantilever on a uniform 128x64 Q4 mesh
  dynamic  the dynamic AMR strategy from 32x16 with two refinement levels
           (finest resolution = the uniform mesh)
  static   the refine-only scheme of Costa / Stainko that the paper argues
           against: converge, refine the marked elements, repeat

Left edge clamped, unit point load at the middle of the right edge, V0 = 50%,
filter radius = r_amr = 1.5 fine elements, p-continuation 1 -> 3; every run
stops when the design change is < 0.01 at p = 3 (and, for the adaptive runs,
the mesh would not change) or after `steps` design steps.

  A1  D(uniform, dynamic) < 0.02              (paper: 0.168% at full scale)
  A2  D(uniform, static) > 0.05 and > 3 A1    (paper: 19.6%)
  A3  the dynamic run ends with fewer elements and accumulates fewer CG
      iterations and unknowns than the uniform run

D is Eq. 10 on the fine lattice.  Prints one JSON line.

    python tools/test1_acceptance.py [steps] [rmin] [change_tol] [stop_rule]
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

NX, NY = 128, 64


def problem(adaptive, rmin=1.5):
    L = 2 if adaptive else 0
    base = (NX >> L, NY >> L)
    return make_problem("test1_cantilever2d_" + ("amr" if adaptive else "uniform"), 2, base, L=L,
                        h0=float(1 << L), leaves=uniform_leaves(2, base, L, 0),
                        density=DensitySpec("const", value=0.5),
                        fixed=[((0, 0), (0, NY), 0b11)],
                        loads=[("point", (NX, NY // 2), (NX, NY // 2), (0.0, -1.0))], rmin=rmin, rtol=1e-8)


def raster(host, x):
    out = np.zeros((NY, NX))
    s = 1 << (host.L - host.elem_level.astype(np.int64))
    for e in range(host.n_el):
        a = host.elem_anchor[e]
        out[a[1]:a[1] + s[e], a[0]:a[0] + s[e]] = x[e]
    return out


def summary(steps, host, wall):
    return {"steps": len(steps), "wall_s": wall, "n_elem_last": host.n_el,
            "cg_iters_total": int(sum(h["cg_iters"] for h in steps)),
            "unknowns_total": int(sum(h.get("n_dof", host.n_dof) for h in steps)),
            "compliance_last": steps[-1]["compliance"], "penal_last": steps[-1]["penal"],
            "change_last": steps[-1]["change"]}


def main():
    cap = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    rmin = float(sys.argv[2]) if len(sys.argv) > 2 else 1.5
    tol = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
    stop_rule = sys.argv[4] if len(sys.argv) > 4 else "mesh"
    volfrac = 0.5
    pu = problem(False, rmin)
    hu = pb.prepare(pu)
    mu = pb.Mesh(hu, E0=pu.E0, Emin=pu.Emin, nu=pu.nu, rmin=pu.rmin)
    xu = torch.full((hu.n_el,), volfrac, dtype=torch.float64, device="cuda")
    uu = torch.zeros(hu.n_dof, dtype=torch.float64, device="cuda")
    t0 = time.perf_counter()
    _, hist_u = mu.to_optimize(xu, uu, cap, volfrac, stop_on_converge=True, change_tol=tol, rtol=1e-8)
    wall_u = time.perf_counter() - t0
    for h in hist_u:
        h["n_dof"] = hu.n_dof
    ru = raster(hu, xu.cpu().numpy())
    out = {"workload": "test1_cantilever2d_128x64", "step_cap": cap, "rmin": rmin, "change_tol": tol,
           "stop_rule": stop_rule,
           "uniform": summary(hist_u, hu, wall_u)}
    pa = problem(True, rmin)
    for mode in ("dynamic", "static"):
        t0 = time.perf_counter()
        run = pb.amr.optimize_amr(pa, volfrac, cap, mode=mode, stop_on_converge=True, change_tol=tol, rtol=1e-8,
                                  stop_rule=stop_rule)
        wall = time.perf_counter() - t0
        ra = raster(run.host, run.x.cpu().numpy())
        out[mode] = summary(run.steps, run.host, wall)
        out[mode]["adaptations"] = len(run.adaptations)
        out[mode]["levels_last"] = int(run.host.elem_level.max())
        out[mode]["D_vs_uniform"] = float(np.abs(ru - ra).sum() / ru.sum())
    d1, d2 = out["dynamic"]["D_vs_uniform"], out["static"]["D_vs_uniform"]
    out["A1_dynamic_close"] = d1 < 0.02
    out["A2_static_far"] = d2 > 0.05 and d2 > 3 * d1
    out["A3_dynamic_cheaper"] = (out["dynamic"]["n_elem_last"] < hu.n_el
                                 and out["dynamic"]["cg_iters_total"] < out["uniform"]["cg_iters_total"]
                                 and out["dynamic"]["unknowns_total"] < out["uniform"]["unknowns_total"])
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
