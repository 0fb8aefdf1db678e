"""Helpers for the -m gpu parity tests: build the product handle and the
oracle for the same seeded problem (no method arithmetic here)."""
import numpy as np

from inputs import density_at


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def product_mesh(prob, options=0):
    import paper_1009_4975_b200 as pb
    hm = pb.prepare(prob)
    m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin, options=options)
    return hm, m


def cuda(a):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


def host(t):
    return t.detach().cpu().numpy()


def product_input_density(prob, hm, m):
    """The product's own input x: raw field at its leaves (+ its DENS pass for c3)."""
    import torch
    import paper_1009_4975_b200 as pb
    x = cuda(density_at(prob, hm.elem_level, hm.elem_anchor))
    if prob.presmooth_rmin is not None:
        out = torch.empty_like(x)
        m.to_filter(pb.TO_FILTER_DENS, x, x, out)
        x = out
    return x
