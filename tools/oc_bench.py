"""Device time of to_oc_update (one cooperative kernel) on seeded inputs at
config sizes; prints one JSON line per config.  usage: python tools/oc_bench.py [c5 c4 ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1009_4975_b200 as pb
from inputs import config


def main(names):
    for name in names:
        prob = config(name)
        hm = pb.prepare(prob)
        m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=0.0)
        rng = np.random.default_rng(3)
        V = (2.0 ** (hm.L - hm.elem_level.astype(np.float64)) * hm.hL) ** hm.dim
        x = torch.as_tensor(rng.uniform(1e-3, 1.0, hm.n_el), device="cuda")
        dc = torch.as_tensor(-np.exp(rng.uniform(-6, 2, hm.n_el)) * V, device="cuda")
        vf = float(np.sum(V * x.cpu().numpy()) / V.sum()) - 0.05
        xn = torch.empty_like(x)
        runs = [m.to_oc_update(x, dc, vf, xn) for _ in range(5)]
        best = min(runs, key=lambda r: r.ms)
        passes = best.passes
        lvl = 0 if m.info()["structured"] else 1
        byts = hm.n_el * (24 + 16 * (passes - 2) + 24 + lvl * passes)
        print(json.dumps({"config": name, "n_elem": hm.n_el, "ms": best.ms, "steps": best.steps, "passes": passes, "state": best.state,
                          "us_per_pass": 1000 * best.ms / passes, "gbs": byts / (best.ms / 1e3) / 1e9,
                          "all_ms": [r.ms for r in runs]}), flush=True)
        m.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["c5", "c4", "c3"])
