"""Dynamic-AMR topology optimization run (Fig. 1 + §4) on the device path, on
the paper's Test 1 geometry (2D 2:1 cantilever): a 64x32
start refined up to the 256x128 resolution of the uniform reference (L = 2),
V0 = 50%, filter radius = r_amr = 1.5 finest elements.  Prints one JSON line:
per-step device times, adaptations (element counts, host times) and the final
element count against the uniform fine mesh.

    python tools/amr_bench.py [steps] [--oracle]   (--oracle: also time the CPU oracle loop)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1009_4975_b200 as pb
from inputs import make_problem, uniform_leaves, DensitySpec


def test1_problem(L=2, base=(64, 32)):
    ext = [b << L for b in base]
    return make_problem("test1_cantilever2d_amr", 2, base, L=L, leaves=uniform_leaves(2, base, L, 0),
                        density=DensitySpec("const", value=0.5),
                        fixed=[((0, 0), (0, ext[1]), 0b11)],
                        loads=[("point", (ext[0], ext[1] // 2), (ext[0], ext[1] // 2), (0.0, -1.0))],
                        rmin=1.5 / (1 << L))


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else 40
    prob = test1_problem()
    t0 = time.perf_counter()
    run = pb.amr.optimize_amr(prob, 0.5, steps, stage_steps=10, rtol=1e-8)
    wall = time.perf_counter() - t0
    st = run.steps
    fine = (prob.base[0] << prob.L) * (prob.base[1] << prob.L)
    line = {
        "workload": prob.name, "steps": len(st), "wall_s": wall,
        "solve_ms_per_step": float(np.mean([s["solve_ms"] for s in st])),
        "oc_ms_per_step": float(np.mean([s["oc_ms"] for s in st])),
        "cg_iters_per_step": float(np.mean([s["cg_iters"] for s in st])),
        "compliance_first_last": [st[0]["compliance"], st[-1]["compliance"]],
        "n_elem_first_last": [st[0]["n_elem"], run.host.n_el], "uniform_fine_elems": fine,
        "final_fraction_of_fine": run.host.n_el / fine,
        "adaptations": run.adaptations,
    }
    if "--oracle" in sys.argv:
        from oracle import amr
        t0 = time.perf_counter()
        n_or = min(steps, 12)
        amr.optimize_amr(prob, 0.5, n_or, stage_steps=10)
        line["oracle_s_per_step"] = (time.perf_counter() - t0) / n_or
        line["oracle_steps_timed"] = n_or
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
