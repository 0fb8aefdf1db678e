"""The z-slab sharded solve of c5 on ONE GPU (all slabs in one process,
tosolve_cg_group): the cost of the shard machinery (ghost-plane stores in K1,
one step kernel per iteration) and the per-slab iteration time that a
multi-GPU run would overlap.  Fixed 200 PCG iterations per solve, the
iteration loop timed with one event pair (TO_PROFILE_LOOP).  Slabs run one
after another here, so loop_ms / R is the average slab iteration: an
estimate of the per-GPU iteration time at R GPUs (NVLink latency not
included), labeled as such.

    python tools/shard_bench.py [R ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1009_4975_b200 as pb  # noqa: E402
from paper_1009_4975_b200 import shard  # noqa: E402
from inputs import config, density_at  # noqa: E402


def main():
    Rs = [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]
    prob = config("c5")
    hm = pb.prepare(prob)
    x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda")
    it = 200
    m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
    u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
    loops = []
    for _ in range(3):
        m.tosolve_cg(prob.penal, x, u, max_iter=it, flags=pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES | pb.TO_PROFILE_LOOP)
        loops.append(m.profile()["loop_ms"] / it)
    base = sorted(loops)[1]
    print(json.dumps({"workload": "c5", "mode": "unsharded", "iter_ms": base}), flush=True)
    del m, u
    torch.cuda.empty_cache()
    for R in Rs:
        g = shard.ShardGroup(hm, R, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin)
        xs = g.scatter_elems(x)
        us = [torch.zeros(mm.n_dof, dtype=torch.float64, device="cuda") for mm in g.meshes]
        loops = []
        for _ in range(3):
            g.solve(prob.penal, xs, us, max_iter=it, flags=pb.TO_FIXED_ITERS | pb.TO_PROFILE_LOOP)
            loops.append(g.meshes[0].profile()["loop_ms"] / it)
        grp = sorted(loops)[1]
        print(json.dumps({"workload": "c5", "mode": f"zslab{R} on one GPU", "group_iter_ms": grp,
                          "overhead_vs_unsharded": grp / base - 1.0,
                          "est_per_gpu_iter_ms_at_R_gpus": grp / R,
                          "est_strong_speedup": base / (grp / R),
                          "slab_planes": [[s.a, s.b] for s in g.slabs]}), flush=True)
        del g, xs, us
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
