"""us per PCG iteration of the small configs on the general-path variants
(the cluster-resident solver, the persistent cooperative kernel and one
kernel per iteration), fixed iterations.

    python tools/small_cfg.py [c1 c2]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1009_4975_b200 as pb  # noqa: E402
from inputs import config, density_at  # noqa: E402

for name in sys.argv[1:] or ["c1", "c2"]:
    prob = config(name)
    hm = pb.prepare(prob)
    for opts in (0, pb.TO_UPLOAD_NO_CLUSTER, pb.TO_UPLOAD_LAUNCHED):
        m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin, options=opts)
        x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda")
        u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
        m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=500, flags=pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES)
        st = m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=2000, flags=pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES)
        u.zero_()
        st2 = m.tosolve_cg(prob.penal, x, u, rtol=prob.rtol, max_iter=100000)
        print(json.dumps({"config": name, "variant": m.info()["matvec_variant"],
                          "us_per_iter": round(st.ms * 1e3 / 2000, 2), "to_rtol_iters": st2.iters,
                          "to_rtol_ms": round(st2.ms, 3)}), flush=True)
        m.close()
