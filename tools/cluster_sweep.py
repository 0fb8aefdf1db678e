"""us per PCG iteration of the general-path loop variants on small 2D/3D
meshes of growing size: the cluster-resident solver (variant 5), the
cooperative kernel (3) and one kernel per iteration (4).  Fixed iterations.

    python tools/cluster_sweep.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1009_4975_b200 as pb  # noqa: E402
from inputs import config, density_at  # noqa: E402

CASES = [("c1", {}), ("c1", {"scale": 2}), ("c2", {"L": 2}), ("c2", {"L": 3}), ("c2", {"base": (16, 8)}),
         ("c2", {}), ("c4", {"base": (6, 3, 3), "L": 2, "n_gauss": 30}), ("c4", {"base": (12, 6, 6), "L": 2, "n_gauss": 60})]
for name, kw in CASES:
    prob = config(name, **kw)
    hm = pb.prepare(prob)
    out = {"config": name, "kw": {k: list(v) if isinstance(v, tuple) else v for k, v in kw.items()},
           "n_el": hm.n_el, "n_node": hm.n_node}
    for opts in (0, pb.TO_UPLOAD_NO_CLUSTER, pb.TO_UPLOAD_LAUNCHED):
        m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin, options=opts)
        x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda")
        u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
        m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=300, flags=pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES)
        st = m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=2000, flags=pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES)
        out[f"v{m.info()['matvec_variant']}_us"] = round(st.ms * 1e3 / 2000, 2)
        m.close()
    print(json.dumps(out), flush=True)
