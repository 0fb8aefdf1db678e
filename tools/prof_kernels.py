"""Per-kernel device time per PCG iteration (TO_PROFILE), in microseconds.

    python tools/prof_kernels.py [config]
"""
import sys, json
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1009_4975_b200 as pb
from inputs import config, density_at
prob = config(sys.argv[1] if len(sys.argv) > 1 else "c4")
hm = pb.prepare(prob)
m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda")
u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
for _ in range(2):
    st = m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=200, flags=pb.TO_FIXED_ITERS | pb.TO_PROFILE | pb.TO_NO_TRUE_RES)
p = m.profile()
print(json.dumps({k: (v / p["iters"] * 1000 if k.endswith("_ms") else v) for k, v in p.items()}), m.info()["matvec_variant"])
