"""Fig. 1 with dynamic AMR (PAPER.md:336-358 and §4 :360-492) on top of the
C ABI: the design steps run in the library (`to_optimize`, every step a
device solve, sensitivity, filter and OC update) until the adaptation
trigger fires; then the marks are computed on the device (`to_amr_mark`),
the mesh is updated by the C++ host code (`tomesh_host_adapt`, the
compatibility sweeps and refine/derefine with density transfer), rebuilt
(`tomesh_host_build`), the densities moved onto it (`tomesh_host_transfer`)
and the new mesh uploaded.  This module only sequences those calls.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .api import Mesh, prepare, rebuild, tomesh_host_adapt, tomesh_host_transfer


@dataclass
class AmrRun:
    host: object                       # final HostMesh
    x: object                          # final densities (CUDA tensor, final mesh order)
    steps: list = field(default_factory=list)         # per-step dicts (+ "n_elem", "adapted")
    adaptations: list = field(default_factory=list)   # per adaptation: counts


def optimize_amr(problem, volfrac, n_steps, penal0=1.0, penal_max=3.0, penal_step=0.5, stage_steps=30,
                 rho_s=0.5, min_steps=5, max_steps=10, change_tol=0.01, rtol=1e-10, max_iter=20000,
                 device=0, x0=None, mode="dynamic", stop_on_converge=False, level_steps=150,
                 stop_rule="mesh") -> AmrRun:
    """mode "dynamic": the paper's strategy (§4).  mode "static": the
    refine-only baseline the paper argues against (Costa/Stainko, PAPER.md:
    754-790): optimise to convergence at p_max, refine the marked elements
    (no derefinement; after at most level_steps steps on a level if it does not
    converge), repeat until nothing is refined.  stop_on_converge:
    end when the design change is < change_tol at p_max and the adaptation
    that follows would not change the mesh (stop_rule "mesh"),
    or (stop_rule "design", reading R25) when the design converges
    again within min_steps steps of an adaptation that was itself made at a
    converged design: "if the local minimum is not an artifact of the mesh,
    the design will remain the same after mesh adaptation"."""
    static = mode == "static"
    if mode not in ("dynamic", "static"):
        raise ValueError("mode must be 'dynamic' or 'static'")
    if stop_rule not in ("mesh", "design"):
        raise ValueError("stop_rule must be 'mesh' or 'design'")
    last_adapt_at_conv = False
    import torch
    dev = torch.device("cuda", device)
    host = prepare(problem, keep_handle=True)
    mesh = Mesh(host, E0=problem.E0, Emin=problem.Emin, nu=problem.nu, rmin=problem.rmin, device=device)
    x = torch.full((host.n_el,), float(volfrac), dtype=torch.float64, device=dev) if x0 is None else x0
    state = L.ToOptState(penal=penal0, at_stage=0, since_adapt=0)
    run = AmrRun(host, x)
    done = 0
    while done < n_steps:
        u = torch.zeros(host.n_dof, dtype=torch.float64, device=dev)
        n_call = min(n_steps - done, level_steps) if static else n_steps - done
        _, hist = mesh.to_optimize(x, u, n_call, volfrac, penal0=penal0, penal_max=penal_max,
                                   penal_step=penal_step, stage_steps=stage_steps, change_tol=change_tol,
                                   rtol=rtol, max_iter=max_iter, adapt_min_steps=0 if static else min_steps,
                                   adapt_max_steps=0 if static else max_steps,
                                   stop_on_converge=stop_on_converge or static, state=state)
        for h in hist:
            h["n_elem"] = host.n_el
            h["n_dof"] = host.n_dof
            h["adapted"] = False
        run.steps.extend(hist)
        done += len(hist)
        converged = bool(state.converged)
        if done >= n_steps or (not static and not state.adapt_due and not converged):
            break                                        # step budget used up
        if (converged and not static and stop_rule == "design" and last_adapt_at_conv
                and state.since_adapt <= min_steps):
            break                                        # re-converged right after a converged adaptation
        t0 = time.perf_counter()
        marks = torch.empty(host.n_el, dtype=torch.int8, device=dev)
        mesh.to_amr_mark(x, marks, rho_s)
        mk, xh = marks.cpu().numpy(), x.cpu().numpy()
        if static:
            mk[mk < 0] = 0                               # refinement only
        t1 = time.perf_counter()
        ad = tomesh_host_adapt(host, mk, xh)
        if ad.n_refined == 0 and ad.n_groups == 0:
            if converged:
                break                                    # converged on a mesh the strategy keeps
            if static:
                continue                                 # finest level reached: keep optimising
        new_host = rebuild(problem, ad)
        xn = tomesh_host_transfer(new_host, ad)
        t2 = time.perf_counter()
        mesh.close()
        host = new_host
        mesh = Mesh(host, E0=problem.E0, Emin=problem.Emin, nu=problem.nu, rmin=problem.rmin, device=device)
        x = torch.as_tensor(xn, device=dev)
        torch.cuda.synchronize(dev)
        t3 = time.perf_counter()
        run.adaptations.append({"step": done, "n_elem_before": len(mk), "n_elem_after": host.n_el,
                                "n_refined": ad.n_refined, "n_groups": ad.n_groups,
                                "n_unmarked_sibling": ad.n_unmarked_sibling,
                                "n_unmarked_incompat": ad.n_unmarked_incompat,
                                "mark_s": t1 - t0, "host_adapt_rebuild_s": t2 - t1, "upload_s": t3 - t2})
        run.steps[-1]["adapted"] = True
        last_adapt_at_conv = converged
        state.since_adapt = 0
        state.adapt_due = 0
    mesh.close()
    run.host, run.x = host, x
    return run
