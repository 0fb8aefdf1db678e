"""Run-to-run determinism of every solver path (a race in the hand-rolled
synchronisation -- mbarrier rings, last-block-done reductions, PDL chains,
shard flags -- would show up as differing bits): 10 fixed-iteration solves
per path, all bit-identical to the first.

    python tools/repeat_check.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1009_4975_b200 as pb  # noqa: E402
from inputs import config, density_at  # noqa: E402
from tools.sanitize_cases import CASES  # noqa: E402

ok = True
for name, (mk, opts) in list(CASES.items()) + [("c4", (lambda: config("c4"), 0))]:
    prob = mk()
    hm = pb.prepare(prob)
    m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin, options=opts)
    x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda")
    ref = None
    for rep in range(10):
        u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda")
        m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=60, flags=pb.TO_FIXED_ITERS)
        if ref is None:
            ref = u.clone()
        elif not torch.equal(u, ref):
            ok = False
            print(f"{name}: repetition {rep} differs (max |du| {float((u - ref).abs().max()):.3e})")
    print(f"{name}: 10 solves of 60 iterations, bit-identical: {torch.equal(u, ref)}", flush=True)
    m.close()
print("REPEAT_OK" if ok else "REPEAT_FAILED")
sys.exit(0 if ok else 1)
