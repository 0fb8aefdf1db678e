"""Small runs of every device code path, for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck).  Each case uploads a small mesh and runs a
few iterations of its path plus the calls around it.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1009_4975_b200 as pb  # noqa: E402
from inputs import config, density_at  # noqa: E402

CASES = {
    "c1": (lambda: config("c1"), 0),                                   # 2D cluster-resident solver
    "c1_coop": (lambda: config("c1"), pb.TO_UPLOAD_NO_CLUSTER),        # 2D cooperative general kernel
    "c1_launched": (lambda: config("c1"), pb.TO_UPLOAD_LAUNCHED),      # 2D kernel per iteration, step inside
    "c2L2": (lambda: config("c2", L=2), 0),                            # 2D cluster solver with hanging nodes
    "c2": (lambda: config("c2"), 0),                                   # 2D general kernel per iteration, step inside
    "c4s": (lambda: config("c4", base=(6, 3, 3), L=2, n_gauss=30), 0),  # 3D cluster solver (hanging nodes)
    "c4s_launched": (lambda: config("c4", base=(6, 3, 3), L=2, n_gauss=30), pb.TO_UPLOAD_LAUNCHED),
    "c3s": (lambda: config("c3", nx=37, ny=9, nz=13), 0),              # structured K1 (TMA, ragged tiles)
    "c5s": (lambda: config("c5", nx=20, ny=10, nz=10), 0),
}


def run_case(name, iters=6):
    mk, opts = CASES[name]
    prob = mk()
    hm = pb.prepare(prob)
    m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin, options=opts)
    x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda")
    if prob.presmooth_rmin is not None:
        xs = torch.empty_like(x)
        m.to_filter(pb.TO_FILTER_DENS, x, x, xs)
        x = xs
    u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
    st = m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=iters, flags=pb.TO_FIXED_ITERS)
    st2 = m.tosolve_cg(prob.penal, x, u, rtol=1e-3, max_iter=200, flags=pb.TO_WARM)   # warm start + rtol stop
    dc = torch.empty(hm.n_el, dtype=torch.float64, device="cuda")
    c = m.to_sensitivity(prob.penal, x, u, dc, compliance=True)
    out = torch.empty_like(dc)
    m.to_filter(pb.TO_FILTER_SENS, x, dc, out)
    q = torch.empty_like(u)
    m.to_apply_A(prob.penal, x, u, q)
    xn = torch.empty_like(x)
    oc = m.to_oc_update(x, out, float(x.mean()) - 0.05, xn)
    marks = torch.empty(hm.n_el, dtype=torch.int8, device="cuda")
    m.to_amr_mark(x, marks, 0.5)
    torch.cuda.synchronize()
    print(f"{name}: iters {st.iters} warm {st2.iters} c {c:.6g} oc state {oc.state}", flush=True)
    m.close()


def run_shard(nranks=2, iters=6):
    from paper_1009_4975_b200 import shard
    prob = config("c5", nx=12, ny=6, nz=10)
    hm = pb.prepare(prob)
    g = shard.ShardGroup(hm, nranks, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
    xg = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda")
    xs = g.scatter_elems(xg)
    us = [torch.zeros(m.n_dof, dtype=torch.float64, device="cuda") for m in g.meshes]
    st = g.solve(prob.penal, xs, us, rtol=0.0, max_iter=iters, flags=pb.TO_FIXED_ITERS)
    st2 = g.solve(prob.penal, xs, us, rtol=1e-6, max_iter=2000)
    torch.cuda.synchronize()
    print(f"shard{nranks}: iters {st[0].iters} / {st2[0].iters}", flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES) + ["shard2"]
    for n in names:
        if n.startswith("shard"):
            run_shard(int(n[5:]))
        else:
            run_case(n)
    print("SANITIZE_CASES_OK")
