"""Fixed-iteration general-path solve of a config for ncu captures.

    python tools/prof_gen.py c4 [iters]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1009_4975_b200 as pb  # noqa: E402
from inputs import config, density_at  # noqa: E402
from tests.oracle_cache import variant  # noqa: E402

name = sys.argv[1]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
prob = variant(name)
hm = pb.prepare(prob)
m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin, device=0)
x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda:0")
u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda:0")
st = m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=iters, flags=pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES)
print(name, hm.n_el, hm.n_dof, st.iters, round(st.ms * 1e3 / iters, 2), "us/it", m.info())
