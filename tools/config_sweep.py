"""Per-config solve timings on one GPU (CUDA events inside tosolve_cg).

    python tools/config_sweep.py [c1 c2 ...]

For each config: host prepare + upload time, one warm-up solve, then a
solve to the config's tolerance (iterations, ms, it/s, true residual) and a
fixed 200-iteration solve (it/s), plus sensitivities + filter time.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1009_4975_b200 as pb  # noqa: E402
from inputs import density_at  # noqa: E402
from tests.oracle_cache import variant  # noqa: E402


def run(name):
    prob = variant(name)
    t0 = time.perf_counter()
    hm = pb.prepare(prob)
    t1 = time.perf_counter()
    m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin, device=0)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda:0")
    if prob.presmooth_rmin is not None:
        xs = torch.empty_like(x)
        m.to_filter(pb.TO_FILTER_DENS, x, x, xs)
        x = xs
    u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda:0")
    rtol = prob.rtol
    m.tosolve_cg(prob.penal, x, u, rtol=rtol, max_iter=100000)
    u.zero_()
    st = m.tosolve_cg(prob.penal, x, u, rtol=rtol, max_iter=100000)
    u.zero_()
    fx = m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=200, flags=pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES)
    dc = torch.empty(hm.n_el, dtype=torch.float64, device="cuda:0")
    dcf = torch.empty_like(dc)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        m.to_sensitivity(prob.penal, x, u, dc)
        m.to_filter(pb.TO_FILTER_SENS, x, dc, dcf)
    e1.record()
    torch.cuda.synchronize()
    info = m.info()
    return {"config": name, "n_el": hm.n_el, "n_dof": hm.n_dof, "structured": info["structured"],
            "prepare_s": round(t1 - t0, 3), "upload_s": round(t2 - t1, 3),
            "rtol": rtol, "iters": st.iters, "solve_ms": round(st.ms, 3), "relres_true": st.relres_true,
            "it_per_s_to_tol": round(st.iters / (st.ms / 1e3), 1) if st.ms else None,
            "it_per_s_fixed200": round(200 / (fx.ms / 1e3), 1),
            "us_per_iter_fixed200": round(fx.ms * 1e3 / 200, 2),
            "sens_plus_filter_ms": round(e0.elapsed_time(e1) / 5, 3), "variant": info["matvec_variant"],
            **{k: info[k] for k in ("gen_blocks", "gen_smem_bytes", "gen_max_loc", "gen_max_el", "gen_local_el",
                                    "gen_local_nodes")}}


if __name__ == "__main__":
    names = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c4L", "c5"]
    for n in names:
        print(json.dumps(run(n)), flush=True)
