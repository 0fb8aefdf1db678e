"""A mid-size 3D AMR mesh (c4 recipe, base 12x6x6, L = 3: 66,519 elements by
default) for general-path latency measurements: 200 fixed PCG iterations,
per-iteration time.

    python tools/prof_c4mid.py [bx by bz L n_gauss]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1009_4975_b200 as pb
from inputs import config, density_at

a = [int(v) for v in sys.argv[1:]] or [12, 6, 6, 3, 60]
prob = config("c4", base=tuple(a[:3]), L=a[3], n_gauss=a[4])
hm = pb.prepare(prob)
m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda")
u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
for _ in range(2):
    st = m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=200, flags=pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES)
print("n_el", hm.n_el, "n_dof", hm.n_dof, "variant", m.info()["matvec_variant"], "us/iter", 1000 * st.ms / st.iters)
