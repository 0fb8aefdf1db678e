"""Element-partitioned general path (TO_UPLOAD_EP) against the default
general path on the same mesh: u after a solve to 1e-10, after 25 fixed
iterations, iteration counts, and us per iteration.

    python tools/ep_check.py [names...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1009_4975_b200 as pb  # noqa: E402
from inputs import config, density_at  # noqa: E402
from tests.helpers import cantilever3d, hanging_load3d, refine_some  # noqa: E402
from tests.oracle_cache import variant  # noqa: E402

CASES = {
    "amr3d": lambda: cantilever3d((3, 2, 2), L=2, leaves=refine_some(3, (3, 2, 2), 2, [(1, 1, 0)]), rmin=0.4),
    "hload3d": hanging_load3d,
    "c4s": lambda: config("c4", base=(12, 6, 6), L=2, n_gauss=60),
    "c5s": lambda: config("c5", nx=20, ny=10, nz=10),
    "c2": lambda: config("c2"),
    "c4": lambda: variant("c4"),
    "c4L": lambda: variant("c4L"),
}


def rel(a, b):
    return float(torch.linalg.norm(a - b) / max(float(torch.linalg.norm(b)), 1e-300))


def run(name):
    prob = CASES[name]()
    hm = pb.prepare(prob)
    out = {"case": name, "n_el": hm.n_el}
    res = {}
    for tag, opt in (("ref", pb.TO_UPLOAD_LAUNCHED | pb.TO_UPLOAD_GENERAL | pb.TO_UPLOAD_NO_EP),
                     ("ep", pb.TO_UPLOAD_EP | pb.TO_UPLOAD_GENERAL)):
        m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin, options=opt)
        x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda")
        u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
        st = m.tosolve_cg(prob.penal, x, u, rtol=1e-10, max_iter=100000)
        u25 = torch.zeros_like(u)
        m.tosolve_cg(prob.penal, x, u25, rtol=0.0, max_iter=25, flags=pb.TO_FIXED_ITERS)
        u200 = torch.zeros_like(u)
        fx = m.tosolve_cg(prob.penal, x, u200, rtol=0.0, max_iter=200, flags=pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES)
        u2 = torch.zeros_like(u)
        m.tosolve_cg(prob.penal, x, u2, rtol=1e-10, max_iter=100000)
        info = m.info()
        res[tag] = (u, u25, u2)
        out[tag] = {"iters": st.iters, "status": st.status, "relres_true": st.relres_true,
                    "us_per_iter": round(fx.ms * 1e3 / 200, 2), "variant": info["matvec_variant"],
                    "blocks": info["gen_blocks"], "smem": info["gen_smem_bytes"],
                    "el_per_node": round(info["gen_local_el"] / max(1, hm.n_el), 3)}
        m.close()
    out["u_rel"] = rel(res["ep"][0], res["ref"][0])
    out["u25_rel"] = rel(res["ep"][1], res["ref"][1])
    out["ep_repeat_identical"] = bool(torch.equal(res["ep"][0], res["ep"][2]))
    return out


if __name__ == "__main__":
    for n in sys.argv[1:] or list(CASES):
        print(json.dumps(run(n)), flush=True)
