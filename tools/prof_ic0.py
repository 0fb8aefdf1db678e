"""A few MINRES + IC(0) iterations on one config, for ncu captures of k_ic0_tri.
    python tools/prof_ic0.py c2 [max_iter]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1009_4975_b200 as pb
from inputs import config, density_at

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
mi = int(sys.argv[2]) if len(sys.argv) > 2 else 6
prob = config(name)
hm = pb.prepare(prob)
m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda")
u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
st = m.tosolve_minres(prob.penal, x, u, rtol=prob.rtol, max_iter=mi, precond=1)
torch.cuda.synchronize()
print(st)
