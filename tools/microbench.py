"""Micro-timings on c5 (CUDA events): plain operator apply (k_apply_s3<PLAIN>),
one PCG iteration (k_apply_s3<CG>), and a torch copy of the same vector size.

    python tools/microbench.py [config]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1009_4975_b200 as pb  # noqa: E402
from inputs import config, density_at  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    prob = config(name)
    hm = pb.prepare(prob)
    m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin, device=0)
    x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda:0")
    v = torch.randn(hm.n_dof, dtype=torch.float64, device="cuda:0")
    q = torch.empty_like(v)
    t_apply = timed(lambda: m.to_apply_A(prob.penal, x, v, q))      # includes mask/permute passes
    u = torch.zeros_like(v)
    st = m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=200, flags=pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES
                      | pb.TO_PROFILE)
    prof = m.profile()
    big = torch.empty(hm.n_dof * 4, dtype=torch.float64, device="cuda:0")
    big2 = torch.empty_like(big)
    t_copy = timed(lambda: big2.copy_(big))
    print(f"{name}: to_apply_A (with boundary permutes) {t_apply * 1e3:.1f} us; "
          f"CG iteration kernel {prof['apply_ms'] / prof['iters'] * 1e3:.1f} us; "
          f"copy of 4 vectors ({8 * 8 * hm.n_dof / 1e6:.0f} MB moved) {t_copy * 1e3:.1f} us "
          f"= {8 * 8 * hm.n_dof / t_copy / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
