"""Short workload for ncu captures: one solve of `iters` fixed PCG iterations on
a config, then sensitivities and the SENS filter (the bench step, shortened).

    python tools/prof_run.py [config] [iters]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1009_4975_b200 as pb  # noqa: E402
from inputs import config, density_at  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    prob = config(name)
    hm = pb.prepare(prob)
    m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin, device=0)
    x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda:0")
    if prob.presmooth_rmin is not None:
        xs = torch.empty_like(x)
        m.to_filter(pb.TO_FILTER_DENS, x, x, xs)
        x = xs
    u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda:0")
    dc = torch.empty(hm.n_el, dtype=torch.float64, device="cuda:0")
    dcf = torch.empty_like(dc)
    st = m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=iters, flags=pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES)
    m.to_sensitivity(prob.penal, x, u, dc)
    m.to_filter(pb.TO_FILTER_SENS, x, dc, dcf)
    torch.cuda.synchronize()
    print(name, "iters", st.iters, "n_dof", hm.n_dof, "n_el", hm.n_el)


if __name__ == "__main__":
    main()
