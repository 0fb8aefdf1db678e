"""Phase timing of the general-path kernel (A/B build with -DTOMESH_GF_TRACE):
per-block durations of its phases in the last iteration of a fixed solve.

    python tools/gf_trace.py c4 [iters]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1009_4975_b200 as pb  # noqa: E402
from paper_1009_4975_b200 import _lib as L  # noqa: E402
from inputs import density_at  # noqa: E402
from tests.oracle_cache import variant  # noqa: E402

name = sys.argv[1]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
prob = variant(name)
hm = pb.prepare(prob)
m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin, device=0)
x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device="cuda:0")
u = torch.zeros(hm.n_dof, dtype=torch.float64, device="cuda:0")
st = m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=iters, flags=pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES)
buf = np.zeros((16384, 8), dtype=np.uint64)
L.lib().to_debug_gf_trace(buf.ctypes.data_as(C.c_void_p))
t = buf[np.any(buf[:, :7] != 0, axis=1)].astype(np.int64)
nb = t.shape[0]
t0 = t[:, 0].min()
names = ["meta+issue+pdl", "S+owned", "mbar+halo", "virt+elem+acc", "q+dots", "grid_sum"]
print(name, "blocks", nb, "us/it", round(st.ms * 1e3 / iters, 2), "kernel span us", round((t[:, 6].max() - t0) / 1e3, 2))
for k in range(6):
    d = (t[:, k + 1] - t[:, k]) / 1e3
    print(f"  {names[k]:16s} mean {d.mean():7.2f} us  p50 {np.median(d):7.2f}  p90 {np.percentile(d, 90):7.2f}")
el = t[:, 7] / 1e3
print(f"  (elements+barrier mean {el.mean():7.2f} us  p50 {np.median(el):7.2f})")
life = (t[:, 6] - t[:, 0]) / 1e3
print(f"  block lifetime   mean {life.mean():7.2f} us  p50 {np.median(life):7.2f}  max {life.max():7.2f}")
start = (t[:, 0] - t0) / 1e3
print("  start times (us) percentiles 0/25/50/75/100:", np.percentile(start, [0, 25, 50, 75, 100]).round(2))
