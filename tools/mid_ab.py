"""us per iteration on mid-size general-path meshes (A/B of block sizing).

    python tools/mid_ab.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1009_4975_b200 as pb  # noqa: E402
from inputs import config, density_at  # noqa: E402

cases = {"c2": lambda: config("c2"), "c4_b12L3": lambda: config("c4", base=(12, 6, 6), L=3),
         "c4_b12L2": lambda: config("c4", base=(12, 6, 6), L=2, n_gauss=60), "c4": lambda: config("c4")}
out = {}
for name, mk in cases.items():
    prob = mk()
    hm = pb.prepare(prob)
    m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin, options=pb.TO_UPLOAD_LAUNCHED)
    x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda")
    u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
    m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=100, flags=pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES)
    st = m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=500, flags=pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES)
    out[name] = (hm.n_el, round(st.ms * 1e3 / 500, 2))
    m.close()
print(json.dumps(out))
