"""Short workload for ncu: c5, 6 fixed PCG iterations unsharded, then the same
as a 1-slab and a 2-slab group (tosolve_cg_group) on one GPU.

    python tools/shard_prof.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1009_4975_b200 as pb  # noqa: E402
from paper_1009_4975_b200 import shard  # noqa: E402
from inputs import config, density_at  # noqa: E402

prob = config("c5")
hm = pb.prepare(prob)
x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda")
m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
m.tosolve_cg(prob.penal, x, u, max_iter=6, flags=pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES)
del m, u
for R in (1, 2):
    g = shard.ShardGroup(hm, R, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
    xs = g.scatter_elems(x)
    us = [torch.zeros(mm.n_dof, dtype=torch.float64, device="cuda") for mm in g.meshes]
    g.solve(prob.penal, xs, us, max_iter=6, flags=pb.TO_FIXED_ITERS)
    del g, xs, us
torch.cuda.synchronize()
print("ok")
