"""bench.py — PCG iterations/s of the B200 hot path on BASELINE.json's config 5.

One step = the whole hot path on the c5 workload
(uniform 256x128x128 H8, 4.19M elements, 12.83M DOFs, x ~ U(0.001, 1)):
SIMP scale, Jacobi diagonal, projected rhs, exactly 500 PCG iterations,
recovery, sensitivities + compliance, Eq. 5 filter (rmin = 2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun): weak scaling of ONE sharded solve: the c5
box stacked N times along z (256 x 128 x 128N elements), rank r owning one
c5-sized z-slab; every PCG iteration is one kernel per rank with the ghost
planes stored into the neighbours' buffers (NVLink peer stores, CUDA IPC) and
the dots all-reduced on the device ("scaling": "weak", "comm":
"device_peer_stores").  value = c5-box iterations/s (N boxes per global
iteration).  --replicas: N independent c5 solves instead (no data-path
collective).  --shard: ONE c5 solve split into z-slabs over the N ranks
("scaling": "strong"; paper_1009_4975_b200/shard.py).
--impl reference times the oracle (plain numpy/scipy CPU program) on a
bounded sample of the same workload, rank 0 only.
"""
from __future__ import annotations

import os as _os

# the oracle legs (cpu_baseline, --impl reference) run on ONE host thread:
# pinned before numpy / scipy load their BLAS
for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    _os.environ.setdefault(_v, "1")

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(mx)) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def x_touch_fraction(iters):
    """Share of the structured kernel's launches that read and write x: with
    the deferred x update (kernels_cg.cuh cg_x_coef) kernel 0 and every odd
    kernel leave x alone and the even kernels k >= 2 apply two steps' terms,
    so floor((iters - 1) / 2) of `iters` launches touch x."""
    if not iters:
        return 1.0
    return max(0, (iters - 1) // 2) / iters


def kernel_bytes(dim, n_el, n_node, n_dof, structured, iters=None):
    """Algorithmic bytes per launch of the PCG kernels.

    Structured path, one kernel per iteration (k1): s (8/elem) + Dinv
    (8/node) + read r_{k-1}, q_{k-1}, p_{k-1} and write r_k, p_k, q_k (6 x
    8/DOF) + read and write x (2 x 8/DOF) in the launches that touch x
    (x_touch_fraction of `iters` launches; all of them when iters is None),
    averaged per launch; k2 = 0.
    General path (k_gen_fused, one kernel per iteration + a one-CTA step):
    read r, q, p, Dinv, x and write r, p, q, x (9 x 8/DOF) + s and
    connectivity per element (8 + 4 * 2^dim); k2 = 0."""
    nc = 1 << dim
    if structured:
        return {"k1": 8 * n_el + 8 * n_node + 48 * n_dof + round(16 * n_dof * x_touch_fraction(iters)), "k2": 0}
    return {"k1": 72 * n_dof + n_el * (8 + 4 * nc), "k2": 0}


def general_bytes(hm):
    """SURVEY §8(d) algorithmic bytes of one general-path PCG iteration with
    the minimal V = 7 vector passes: 8 n_dof V + n_el (8 + 4 * 2^d) + the fixed
    bitmask n_dof / 8 + n_hang * 4 + (hanging parent entries) * 12."""
    nc = 1 << hm.dim
    return (8 * hm.n_dof * 7 + hm.n_el * (8 + 4 * nc) + hm.n_dof // 8 + 4 * hm.hang_node.shape[0]
            + 12 * hm.hang_parent.shape[0])


def general_path_record(dev, hbm, peak_kind, its=200):
    """The general (AMR) path on c4L, BASELINE.json's config 4 at its "~1-2M
    active elements" (the c4 recipe at L = 5, reading R26), measured
    in the same run: iteration time (the block kernel k_gen_fused + the step
    kernel, launched back to back, one event pair around 200 iterations,
    median of three), the block kernel alone (events around every launch),
    §8(d) bytes and roofline fraction, and the solve to the config's rtol."""
    import torch
    import paper_1009_4975_b200 as pb
    from inputs import density_at
    from inputs.problems import config_c4L
    prob = config_c4L()
    t0 = time.perf_counter()
    hm = pb.prepare(prob)
    t_prep = time.perf_counter() - t0
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin, device=dev.index, stream=stream)
        x = torch.as_tensor(density_at(prob, hm.elem_level, hm.elem_anchor), device=dev)
        u = torch.zeros(hm.n_dof, dtype=torch.float64, device=dev)
    flags = pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES
    m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=its, flags=flags, stream=stream)
    loops = []
    for _ in range(3):
        m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=its, flags=flags | pb.TO_PROFILE_LOOP, stream=stream)
        loops.append(m.profile())
    loop = sorted(loops, key=lambda p: p["loop_ms"])[1]
    it_ms = loop["loop_ms"] / max(1, loop["iters"])
    m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=its, flags=flags | pb.TO_PROFILE, stream=stream)
    pr = m.profile()
    k_ms = pr["apply_ms"] / max(1, pr["iters"])
    step_ms = pr["u1_ms"] / max(1, pr["iters"])
    u.zero_()
    st = m.tosolve_cg(prob.penal, x, u, rtol=prob.rtol, max_iter=200000, stream=stream)
    B = general_bytes(hm)
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(prob.name, {}).get("k1_dram_bytes")
        except Exception:
            traffic = None
    info = m.info()
    m.close()
    # BASELINE.json's config 4 as written (L = 4, 225k elements: L2-resident, latency-bound): iteration time only
    from inputs import config
    p4 = config("c4")
    h4 = pb.prepare(p4)
    with torch.cuda.stream(stream):
        m4 = pb.Mesh(h4, E0=p4.E0, Emin=p4.Emin, nu=p4.nu, rmin=p4.rmin, device=dev.index, stream=stream)
        x4 = torch.as_tensor(density_at(p4, h4.elem_level, h4.elem_anchor), device=dev)
        u4 = torch.zeros(h4.n_dof, dtype=torch.float64, device=dev)
    m4.tosolve_cg(p4.penal, x4, u4, rtol=0.0, max_iter=its, flags=flags, stream=stream)
    l4 = []
    for _ in range(3):
        m4.tosolve_cg(p4.penal, x4, u4, rtol=0.0, max_iter=its, flags=flags | pb.TO_PROFILE_LOOP, stream=stream)
        l4.append(m4.profile())
    l4 = sorted(l4, key=lambda q: q["loop_ms"])[1]
    it4 = l4["loop_ms"] / max(1, l4["iters"])
    B4 = general_bytes(h4)
    c4_line = {"workload": p4.name, "n_elem": h4.n_el, "n_dof": h4.n_dof, "n_hang": int(h4.hang_node.shape[0]),
               "us_per_iter": 1000.0 * it4, "iters_per_sec": 1000.0 / it4, "algorithmic_bytes_per_iter": B4,
               "iteration_frac": B4 / (it4 / 1000.0) / 1e9 / hbm,
               "note": "working set below the 126 MB L2: latency-bound, the HBM fraction is context only"}
    m4.close()
    return {
        "c4": c4_line,
        "workload": prob.name, "n_elem": hm.n_el, "n_dof": hm.n_dof, "n_hang": int(hm.hang_node.shape[0]),
        "matvec_variant": info["matvec_variant"], "iters_per_sec": 1000.0 / it_ms, "us_per_iter": 1000.0 * it_ms,
        "roofline": {"bound": "hbm", "achieved": B / (k_ms / 1000.0) / 1e9, "peak": hbm, "unit": "GB/s",
                     "frac": B / (k_ms / 1000.0) / 1e9 / hbm, "traffic": traffic,
                     "kernel": "k_gen_fused<3, CG>: the whole general-path PCG iteration but the step",
                     "algorithmic_bytes_per_launch": B, "avg_launch_ms": k_ms,
                     "avg_launch_ms_method": "events around every launch of an untimed 200-iteration solve",
                     "peak_source": peak_kind},
        "iteration_frac": B / (it_ms / 1000.0) / 1e9 / hbm, "step_kernel_ms": step_ms,
        "solve_to_rtol": {"rtol": prob.rtol, "iters": st.iters, "ms": st.ms, "relres_true": st.relres_true,
                          "status": st.status},
        "host_prepare_s": t_prep,
    }


def max_over_ranks(value, ws, device=None):
    """Max of a per-rank float over all ranks (identity when ws == 1)."""
    if ws <= 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _host_facts():
    """The host the oracle legs ran on (CPU model, cores, affinity, RAM)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    ram_gb = None
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                ram_gb = round(int(line.split()[1]) / 1024 ** 2, 1)
                break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except AttributeError:
        aff = None
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "affinity": aff, "ram_gb": ram_gb,
            "threads": {v: os.environ.get(v) for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}}


def _cpu_baseline(budget_s=15.0, sample_dims=(48, 24, 24)):
    """The oracle as it stands (assembled CSR + textbook Jacobi-PCG, scipy, 1
    thread) on a c5-recipe sub-box; PCG iterations/s scaled to the c5 DOF
    count (cost per iteration is linear in DOFs for this sparse operator)."""
    from inputs import config
    from oracle import fe, mesh as omesh, solve
    prob = config("c5", nx=sample_dims[0], ny=sample_dims[1], nz=sample_dims[2])
    om = omesh.build_mesh(prob, with_filter=False)
    x = om.density
    K = fe.assemble_K(om, x, prob.penal, prob.E0, prob.Emin, prob.nu)
    A, b, C = fe.projected_system(om, K)
    its = 5
    t0 = time.perf_counter()
    solve.pcg_jacobi(A, b, fixed_iters=its)
    dt = time.perf_counter() - t0
    its = max(5, int(budget_s / max(dt / its, 1e-6)))
    t0 = time.perf_counter()
    solve.pcg_jacobi(A, b, fixed_iters=its)
    dt = time.perf_counter() - t0
    full = config("c5")
    n_dof_full = 3 * (full.base[0] + 1) * (full.base[1] + 1) * (full.base[2] + 1)
    it_s_sample = its / dt
    return {
        "value": it_s_sample * om.n_dof / n_dof_full,
        "unit": "iterations/s",
        "cores": 1,
        "kind": "oracle",
        "sample": (f"oracle Jacobi-PCG ({its} iterations, {dt:.1f} s) on a c5-recipe "
                   f"{sample_dims[0]}x{sample_dims[1]}x{sample_dims[2]} sub-box ({om.n_dof} DOFs); "
                   f"{it_s_sample:.2f} it/s there, scaled by DOF count to c5"),
        "host": _host_facts(),
    }


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    steps, warm = args.steps, args.warmup
    cb = None
    times = []
    for i in range(warm + steps):
        t0 = time.perf_counter()
        cb = _cpu_baseline(budget_s=args.ref_budget)
        if i >= warm:
            times.append(time.perf_counter() - t0)
    val = cb["value"]
    line = {
        "impl": "reference", "metric": "pcg_iterations_per_sec", "value": val, "unit": "iterations/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        # a c5 step (500 iterations) at the measured rate; the wall time of one
        # bounded sample is reported beside it
        "ms_per_step": 1000.0 * 500 / val, "ms_per_sample": 1000.0 * float(np.mean(times)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "c5_uniform3d_256x128x128", "iters_per_solve": 500},
        "cpu_baseline": cb,
        "e2e": {"value": val, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import paper_1009_4975_b200 as pb
    from inputs import config, density_at

    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    prob = config(args.config) if args.config != "c5" else config("c5")
    iters = prob.fixed_iters or 500
    t_prep = time.perf_counter()
    hm = pb.prepare(prob)
    t_prep = time.perf_counter() - t_prep
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        m = pb.Mesh(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin, device=local, stream=stream)
        x_host = torch.from_numpy(density_at(prob, hm.elem_level, hm.elem_anchor)).pin_memory()
        x = x_host.to(dev, non_blocking=True)
        if prob.presmooth_rmin is not None:
            xs = torch.empty_like(x)
            m.to_filter(pb.TO_FILTER_DENS, x, x, xs, stream=stream)
            x = xs
        u = torch.zeros(hm.n_dof, dtype=torch.float64, device=dev)
        dc = torch.empty(hm.n_el, dtype=torch.float64, device=dev)
        dcf = torch.empty_like(dc)
    flags = pb.TO_FIXED_ITERS | pb.TO_NO_TRUE_RES

    def step(profile=False):
        st = m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=iters,
                          flags=flags | (pb.TO_PROFILE if profile else 0), stream=stream)
        m.to_sensitivity(prob.penal, x, u, dc, stream=stream)
        m.to_filter(pb.TO_FILTER_SENS, x, dc, dcf, stream=stream)
        return st

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    # ---- device-timed region (inputs resident in HBM) -------------------------------
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    l0 = m.info()["launches_total"]
    for _ in range(args.steps):
        st = step()
    e1.record(stream)
    launches = m.info()["launches_total"] - l0     # our kernels in the timed region (the library counts them)
    torch.cuda.synchronize(dev)
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1), ws, dev)
    ms_per_step = ms / args.steps
    value = ws * iters * args.steps / (ms / 1000.0)

    # ---- end-to-end through the C ABI with host buffers -------------------------------
    dcf_host = torch.empty(hm.n_el, dtype=torch.float64).pin_memory()
    raw_host = torch.from_numpy(density_at(prob, hm.elem_level, hm.elem_anchor)).pin_memory()
    xr = torch.empty(hm.n_el, dtype=torch.float64, device=dev)
    barrier()
    torch.cuda.synchronize(dev)
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    t_wall = time.perf_counter()
    e2.record(stream)
    comp = 0.0
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            xr.copy_(raw_host, non_blocking=True)
        xin = xr
        if prob.presmooth_rmin is not None:
            m.to_filter(pb.TO_FILTER_DENS, xr, xr, x, stream=stream)
            xin = x
        m.tosolve_cg(prob.penal, xin, u, rtol=0.0, max_iter=iters, flags=flags, stream=stream)
        comp = m.to_sensitivity(prob.penal, xin, u, dc, compliance=True, stream=stream)
        m.to_filter(pb.TO_FILTER_SENS, xin, dc, dcf, stream=stream)
        with torch.cuda.stream(stream):
            dcf_host.copy_(dcf, non_blocking=True)
    e3.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = max_over_ranks(e2.elapsed_time(e3), ws, dev)

    # ---- per-kernel device times: one extra, untimed step with per-iteration events ----
    prof = {"apply_ms": 0.0, "alpha_ms": 0.0, "u1_ms": 0.0, "u2_ms": 0.0, "iters": 0}
    step(profile=True)
    torch.cuda.synchronize(dev)
    prof.update(m.profile())
    # and the iteration launches back to back, bracketed by one event pair (no
    # per-launch events between them): their average duration under the
    # timed region's conditions
    loops = []
    for _ in range(3):   # the median of three such steps
        m.tosolve_cg(prob.penal, x, u, rtol=0.0, max_iter=iters, flags=flags | pb.TO_PROFILE_LOOP, stream=stream)
        torch.cuda.synchronize(dev)
        loops.append(m.profile())
    loop = sorted(loops, key=lambda p: p["loop_ms"])[1]

    # ---- the full solve time of the metric: one solve to the config's
    # tolerance from zero, device time of the call (setup + iterations + recovery)
    u_full = torch.zeros_like(u)
    st_full = m.tosolve_cg(prob.penal, x, u_full, rtol=prob.rtol, max_iter=200000, stream=stream)
    full_line = {"rtol": prob.rtol, "iters": st_full.iters, "ms": st_full.ms, "relres_true": st_full.relres_true,
                 "status": st_full.status}

    # ---- §8(f) row 1: the OC design update on this step's filtered sensitivities ------
    # (untimed for the headline; the library's own CUDA events per call)
    xo = torch.empty_like(dc)
    vf = float(x.mean()) - 0.05 if hm.L == 0 else 0.3      # uniform meshes: a budget just below the volume
    oc_runs = [m.to_oc_update(x, dcf, vf, xo, stream=stream) for _ in range(3)]
    ocs = min(oc_runs, key=lambda r: r.ms)
    per_elem = 1 if not m.info()["structured"] else 0         # int8 level per pass (general meshes)
    oc_bytes = hm.n_el * (24 + 16 * (ocs.passes - 2) + 24 + per_elem * ocs.passes)
    oc_line = {"ms": ocs.ms, "bisect_steps": ocs.steps, "state": ocs.state, "volume": ocs.volume,
               "passes": ocs.passes, "us_per_pass": 1000.0 * ocs.ms / ocs.passes,
               "algorithmic_bytes": oc_bytes, "gbs": oc_bytes / (ocs.ms / 1000.0) / 1e9,
               "note": "one cooperative kernel; each pass over (x, a) evaluates 3 bisection levels (7 candidate lam)"}

    # ---- roofline of the dominant kernel (K1: p update + operator + x update) ---------
    hbm, peak_kind = _peaks()
    info = m.info()
    kb = kernel_bytes(hm.dim, hm.n_el, hm.n_node, hm.n_dof, bool(info["structured"]), iters)
    k1_ms_events = prof["apply_ms"] / max(1, prof["iters"])
    k2_ms = prof["u1_ms"] / max(1, prof["iters"])
    # structured path: the loop holds K1 launches only, so its mean is K1's average launch duration
    k1_ms = loop["loop_ms"] / max(1, loop["iters"]) if info["structured"] else k1_ms_events
    achieved = kb["k1"] / (k1_ms / 1000.0) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(prob.name, {}).get("k1_dram_bytes")
        except Exception:
            traffic = None
    total_prof = prof["apply_ms"] + prof["alpha_ms"] + prof["u1_ms"] + prof["u2_ms"]

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = _cpu_baseline(budget_s=args.ref_budget)
    gen = None
    if rank == 0 and ws == 1 and not args.no_general:
        gen = general_path_record(dev, hbm, peak_kind)

    if rank == 0:
        line = {
            "metric": "pcg_iterations_per_sec", "value": value, "unit": "iterations/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": prob.name, "n_elem": hm.n_el, "n_dof": hm.n_dof,
                       "iters_per_solve": iters, "step": "simp+diag+rhs+500 PCG its+recover+sens+filter",
                       "l2": "inputs larger than L2 (CG working set ~1.3 GB vs 126 MB L2)",
                       "parallelism": f"replicas{ws}"},
            "dof_matvecs_per_sec": value * hm.n_dof,
            "e2e": {"value": ws * iters * args.steps / (e2e_ms / 1000.0), "unit": "iterations/s",
                    "h2d_bytes_per_step": hm.n_el * 8, "d2h_bytes_per_step": hm.n_el * 8 + 8},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "kernel": ("k_apply_s3<CG>: the whole PCG iteration (r, p, x updates, q = A p, 5 dots)"
                                    if info["structured"] else "k_gen_fused<CG> (+ the one-CTA step kernel)"),
                         "algorithmic_bytes_per_launch": kb["k1"], "avg_launch_ms": k1_ms,
                         "avg_launch_ms_method": ("one event pair around the 500 back-to-back K1 launches of an "
                                                  "untimed step, median of three" if info["structured"] else
                                                  "events around every launch of an untimed step"),
                         "avg_launch_ms_per_launch_events": k1_ms_events,
                         "peak_source": peak_kind,
                         "share_of_iteration": prof["apply_ms"] / total_prof if total_prof else None},
            "kernels": {
                "k1_apply": {"ms": k1_ms, "bytes": kb["k1"], "gbs": kb["k1"] / (k1_ms / 1000.0) / 1e9},
                "k2_rupdate": ({"ms": k2_ms, "bytes": kb["k2"], "gbs": kb["k2"] / (k2_ms / 1000.0) / 1e9}
                               if kb["k2"] else None),
                "iteration": {"ms": k1_ms + k2_ms, "bytes": kb["k1"] + kb["k2"],
                              "gbs": (kb["k1"] + kb["k2"]) / ((k1_ms + k2_ms) / 1000.0) / 1e9},
            },
            "solve_to_rtol": full_line,
            "oc_update": oc_line,
            "general_path": gen,
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": launches,
            "host_prepare_s": t_prep,
            "matvec_variant": info["matvec_variant"],
            "compliance": comp,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def weak_slab(nranks, rank, nx=256, ny=128, nz=128, seed=5):
    """Rank `rank`'s z-slab of the weak-scaling workload: the c5 recipe on a
    box of nx x ny x (nz * nranks) elements (x = 0 clamped, unit traction on
    x = nx, x ~ U(0.001, 1) i.i.d. in lexicographic element order, seed 5),
    built locally -- the global mesh is never formed.  The local box holds the
    owned node planes plus two ghost planes per interior side (shard.slice_host's
    layout); its face loads are the GLOBAL consistent nodal loads (1 inside,
    1/2 on an edge, 1/4 at a corner of the loaded face), so a slab cut is never
    a boundary.  Returns (Slab, local densities, local problem); elem_global
    and node_global hold GLOBAL lexicographic ids."""
    import paper_1009_4975_b200 as pb
    from paper_1009_4975_b200 import shard
    from inputs import config
    nzg = nz * nranks
    a, b = shard.slab_plan(nzg + 1, nranks)[rank]
    gz_lo, gz_hi = max(a - shard.GHOST, 0), min(b + shard.GHOST, nzg + 1)
    prob = config("c5", nx=nx, ny=ny, nz=gz_hi - 1 - gz_lo)
    host = pb.prepare(prob)
    nc = host.node_coord.astype(np.int64)
    gzn = nc[:, 2] + gz_lo
    face = nc[:, 0] == nx
    wy = np.where((nc[:, 1] == 0) | (nc[:, 1] == ny), 0.5, 1.0)
    wz = np.where((gzn == 0) | (gzn == nzg), 0.5, 1.0)
    load = np.zeros(host.n_dof)
    load[3 * np.nonzero(face)[0] + 1] = -(wy * wz)[face]
    host.load = load
    ea = host.elem_anchor.astype(np.int64)
    elem_global = ea[:, 0] + nx * (ea[:, 1] + ny * (ea[:, 2] + gz_lo))
    node_global = nc[:, 0] + (nx + 1) * (nc[:, 1] + (ny + 1) * gzn)
    field = np.random.default_rng(seed).uniform(0.001, 1.0, nx * ny * nzg)
    layer = ea[:, 2] + gz_lo
    sl = shard.Slab(rank=rank, a=a, b=b, gz_lo=gz_lo, own_lo=a - gz_lo, own_hi=b - gz_lo, host=host,
                    elem_global=elem_global, node_global=node_global,
                    elem_owned=(layer >= a) & (layer < min(b, nzg)), node_owned=(gzn >= a) & (gzn < b))
    return sl, np.ascontiguousarray(field[elem_global]), prob


def run_weak(args):
    """N > 1 default: weak scaling of one sharded solve (module docstring)."""
    import torch
    import paper_1009_4975_b200 as pb
    from paper_1009_4975_b200 import shard

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")   # (a single process: --weak at N = 1)
    os.environ.setdefault("MASTER_PORT", "29517")
    dist.init_process_group("gloo", rank=rank, world_size=ws)   # plumbing only: IPC handles, barriers, the max
    dev = torch.device("cuda", local)
    t_prep = time.perf_counter()
    sl, x_np, prob = weak_slab(ws, rank)
    t_prep = time.perf_counter() - t_prep
    iters = 500
    sr = shard.ShardRank(slab=sl, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin, device=local)
    m = sr.mesh
    stream = torch.cuda.Stream(device=dev)
    x_host = torch.from_numpy(x_np).pin_memory()
    x = x_host.to(dev)
    u = torch.zeros(m.n_dof, dtype=torch.float64, device=dev)
    dc = torch.empty(m.n_el, dtype=torch.float64, device=dev)
    dcf = torch.empty_like(dc)
    flags = pb.TO_FIXED_ITERS

    def step(extra=0):
        st = sr.solve(prob.penal, x, u, rtol=0.0, max_iter=iters, flags=flags | extra, stream=stream)
        m.to_sensitivity(prob.penal, x, u, dc, stream=stream)
        m.to_filter(pb.TO_FILTER_SENS, x, dc, dcf, stream=stream)
        return st

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    dist.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    l0 = m.info()["launches_total"]
    e0.record(stream)
    for _ in range(args.steps):
        st = step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    launches = m.info()["launches_total"] - l0
    dist.barrier()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1), ws)
    dcf_host = torch.empty(m.n_el, dtype=torch.float64).pin_memory()
    dist.barrier()
    torch.cuda.synchronize(dev)
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            x.copy_(x_host, non_blocking=True)
        step()
        with torch.cuda.stream(stream):
            dcf_host.copy_(dcf, non_blocking=True)
    e3.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = max_over_ranks(e2.elapsed_time(e3), ws)
    step(pb.TO_PROFILE_LOOP)
    torch.cuda.synchronize(dev)
    p = m.profile()
    it_ms = max_over_ranks(p["loop_ms"] / max(1, p["iters"]), ws)
    own_nodes = int(sl.node_owned.sum())
    own_el = int(sl.elem_owned.sum())
    kb = 8 * own_el + 8 * own_nodes + round((48 + 16 * x_touch_fraction(iters)) * 3 * own_nodes)
    hbm, peak_kind = _peaks()
    n_dof_g = 3 * 257 * 129 * (128 * ws + 1)
    if rank == 0:
        line = {
            "metric": "pcg_iterations_per_sec", "value": ws * iters * args.steps / (ms / 1000.0),
            "unit": "iterations/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"c5x{ws}_weak_256x128x{128 * ws}", "n_elem": 256 * 128 * 128 * ws,
                       "n_dof": n_dof_g, "iters_per_solve": iters,
                       "step": "simp+diag+rhs+500 PCG its+recover+sens+filter, one z-slab sharded solve",
                       "value_counts": "c5-box iterations: N boxes per global PCG iteration",
                       "parallelism": f"zslab{ws}", "slab_planes": [sl.a, sl.b],
                       "l2": "inputs larger than L2 (slab working set ~1.3 GB per GPU)"},
            "comm": "device_peer_stores", "gpus_active": ws,
            "global_iterations_per_sec": iters * args.steps / (ms / 1000.0),
            "dof_matvecs_per_sec": iters * args.steps / (ms / 1000.0) * n_dof_g,
            "e2e": {"value": ws * iters * args.steps / (e2e_ms / 1000.0), "unit": "iterations/s",
                    "h2d_bytes_per_step": m.n_el * 8, "d2h_bytes_per_step": m.n_el * 8},
            "roofline": {"bound": "hbm", "achieved": kb / (it_ms / 1000.0) / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": kb / (it_ms / 1000.0) / 1e9 / hbm, "traffic": None,
                         "kernel": "k_apply_s3<CG, SHARD> + k_shard_step per iteration (rank 0's slab)",
                         "algorithmic_bytes_per_launch": kb, "avg_launch_ms": it_ms, "peak_source": peak_kind},
            "cpu_baseline": None, "clocks": clk, "gpu_launches": launches, "host_prepare_s": t_prep,
        }
        print(json.dumps(line), flush=True)
    sr.close()
    dist.destroy_process_group()
    return 0


def run_shard(args):
    """--shard: ONE c5 solve split into z-slabs over the N ranks (
    paper_1009_4975_b200/shard.py): every rank uploads its slab, the ghost
    planes travel by peer stores fused into K1 (CUDA IPC mappings of the
    neighbours' buffers) and the dots by the device-side all-reduce.  Strong
    scaling: value = iterations/s of the one global solve."""
    import torch
    import paper_1009_4975_b200 as pb
    from paper_1009_4975_b200 import shard
    from inputs import config, density_at

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")          # plumbing only: IPC handles, barriers, the max over ranks
    dev = torch.device("cuda", local)
    prob = config("c5")
    iters = prob.fixed_iters or 500
    hm = pb.prepare(prob)
    sr = shard.ShardRank(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, rmin=prob.rmin, device=local)
    sl, m = sr.slab, sr.mesh
    stream = torch.cuda.Stream(device=dev)
    x_glob = density_at(prob, hm.elem_level, hm.elem_anchor)
    x_host = torch.from_numpy(np.ascontiguousarray(x_glob[sl.elem_global])).pin_memory()
    x = x_host.to(dev)
    u = torch.zeros(m.n_dof, dtype=torch.float64, device=dev)
    dc = torch.empty(m.n_el, dtype=torch.float64, device=dev)
    dcf = torch.empty_like(dc)
    flags = pb.TO_FIXED_ITERS

    def step(extra=0):
        st = sr.solve(prob.penal, x, u, rtol=0.0, max_iter=iters, flags=flags | extra, stream=stream)
        m.to_sensitivity(prob.penal, x, u, dc, stream=stream)
        m.to_filter(pb.TO_FILTER_SENS, x, dc, dcf, stream=stream)
        return st

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    l0 = m.info()["launches_total"]
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    launches = m.info()["launches_total"] - l0
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1), ws)
    # end to end: the slab's densities in from pinned host memory, its filtered
    # sensitivities out, every step
    dcf_host = torch.empty(m.n_el, dtype=torch.float64).pin_memory()
    barrier()
    torch.cuda.synchronize(dev)
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            x.copy_(x_host, non_blocking=True)
        step()
        with torch.cuda.stream(stream):
            dcf_host.copy_(dcf, non_blocking=True)
    e3.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = max_over_ranks(e2.elapsed_time(e3), ws)
    # per-rank iteration time (K1 + step kernel), one event pair around the loop
    step(pb.TO_PROFILE_LOOP)
    torch.cuda.synchronize(dev)
    p = m.profile()
    it_ms = max_over_ranks(p["loop_ms"] / max(1, p["iters"]), ws)
    own_nodes = int(sl.node_owned.sum())
    own_el = int(sl.elem_owned.sum())
    kb = 8 * own_el + 8 * own_nodes + round((48 + 16 * x_touch_fraction(iters)) * 3 * own_nodes)
    hbm, peak_kind = _peaks()
    if rank == 0:
        line = {
            "metric": "pcg_iterations_per_sec", "value": iters * args.steps / (ms / 1000.0), "unit": "iterations/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": prob.name, "n_elem": hm.n_el, "n_dof": hm.n_dof, "iters_per_solve": iters,
                       "step": "simp+diag+rhs+500 PCG its+recover+sens+filter, z-slab sharded",
                       "parallelism": f"zslab{ws}", "slab_planes": [sl.a, sl.b],
                       "l2": "inputs larger than L2 at N <= 8 (slab working set >= 160 MB)"},
            "dof_matvecs_per_sec": iters * args.steps / (ms / 1000.0) * hm.n_dof,
            "e2e": {"value": iters * args.steps / (e2e_ms / 1000.0), "unit": "iterations/s",
                    "h2d_bytes_per_step": m.n_el * 8, "d2h_bytes_per_step": m.n_el * 8},
            "roofline": {"bound": "hbm", "achieved": kb / (it_ms / 1000.0) / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": kb / (it_ms / 1000.0) / 1e9 / hbm, "traffic": None,
                         "kernel": "k_apply_s3<CG, SHARD> + k_shard_step per iteration (rank 0's slab)",
                         "algorithmic_bytes_per_launch": kb, "avg_launch_ms": it_ms, "peak_source": peak_kind},
            "cpu_baseline": None, "clocks": clk, "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    sr.close()
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def run_amr_shard(args):
    """--amr-shard: ONE c4L solve (the general / AMR path, reading R26)
    split into Morton node ranges over the N ranks (
    paper_1009_4975_b200/amr_shard.py AmrShardRank): every rank uploads its
    local mesh, the ghost r, p, q travel by peer stores (CUDA IPC mappings)
    and the dots by the device-side all-reduce.  Strong scaling: value =
    iterations/s of the one global solve; a step is 200 fixed PCG iterations
    plus the sensitivities (the filter is not sharded)."""
    import torch
    import paper_1009_4975_b200 as pb
    from paper_1009_4975_b200 import amr_shard
    from inputs import density_at
    from inputs.problems import config_c4L

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")          # plumbing only: receive lists, IPC handles, barriers, the max
    dev = torch.device("cuda", local)
    prob = config_c4L()
    iters = 200
    hm = pb.prepare(prob)
    sr = amr_shard.AmrShardRank(hm, E0=prob.E0, Emin=prob.Emin, nu=prob.nu, device=local)
    sl, m = sr.slab, sr.mesh
    stream = torch.cuda.Stream(device=dev)
    x_glob = density_at(prob, hm.elem_level, hm.elem_anchor)
    x_host = torch.from_numpy(np.ascontiguousarray(x_glob[sl.elem_global])).pin_memory()
    x = x_host.to(dev)
    u = torch.zeros(m.n_dof, dtype=torch.float64, device=dev)
    dc = torch.empty(m.n_el, dtype=torch.float64, device=dev)

    def step(extra=0):
        st = sr.solve(prob.penal, x, u, rtol=0.0, max_iter=iters, flags=pb.TO_FIXED_ITERS | extra, stream=stream)
        m.to_sensitivity(prob.penal, x, u, dc, stream=stream)
        return st

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    l0 = m.info()["launches_total"]
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    launches = m.info()["launches_total"] - l0
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1), ws)
    dc_host = torch.empty(m.n_el, dtype=torch.float64).pin_memory()
    barrier()
    torch.cuda.synchronize(dev)
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            x.copy_(x_host, non_blocking=True)
        step()
        with torch.cuda.stream(stream):
            dc_host.copy_(dc, non_blocking=True)
    e3.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = max_over_ranks(e2.elapsed_time(e3), ws)
    step(pb.TO_PROFILE_LOOP)
    torch.cuda.synchronize(dev)
    p = m.profile()
    it_ms = max_over_ranks(p["loop_ms"] / max(1, p["iters"]), ws)
    kb = general_bytes(sl.host)                  # §8(d) bytes of this rank's local mesh (ghosts included)
    hbm, peak_kind = _peaks()
    if rank == 0:
        line = {
            "metric": "pcg_iterations_per_sec", "value": iters * args.steps / (ms / 1000.0), "unit": "iterations/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": prob.name, "n_elem": hm.n_el, "n_dof": hm.n_dof, "iters_per_solve": iters,
                       "step": "simp+diag+rhs+200 PCG its+recover+sens, Morton node-range sharded general path",
                       "parallelism": f"morton{ws}", "rank0_nodes": [int(sl.n0), int(sl.n1)],
                       "rank0_ghosts": int(sl.n_ghost),
                       "l2": "inputs larger than L2 at N <= 2 (c4L streams ~440 MB per iteration)"},
            "comm": "device_peer_stores", "gpus_active": ws,
            "dof_matvecs_per_sec": iters * args.steps / (ms / 1000.0) * hm.n_dof,
            "e2e": {"value": iters * args.steps / (e2e_ms / 1000.0), "unit": "iterations/s",
                    "h2d_bytes_per_step": m.n_el * 8, "d2h_bytes_per_step": m.n_el * 8},
            "roofline": {"bound": "hbm", "achieved": kb / (it_ms / 1000.0) / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": kb / (it_ms / 1000.0) / 1e9 / hbm, "traffic": None,
                         "kernel": "k_gen_fused<3, CG> + k_gshard_xchg + k_shard_step per iteration (rank 0)",
                         "algorithmic_bytes_per_launch": kb, "avg_launch_ms": it_ms, "peak_source": peak_kind},
            "cpu_baseline": None, "clocks": clk, "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    sr.close()
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--ref-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-general", action="store_true", help="skip the c4L general-path sub-record")
    ap.add_argument("--shard", action="store_true",
                    help="split ONE c5 solve into z-slabs over the ranks (strong scaling)")
    ap.add_argument("--amr-shard", action="store_true",
                    help="split ONE c4L (general / AMR path) solve into Morton node ranges over the ranks")
    ap.add_argument("--weak", action="store_true", help="the weak-scaled sharded solve even at N = 1")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: N independent c5 solves (no data-path collective) instead of the weak-scaled "
                         "sharded solve")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.shard:
        return run_shard(args)
    if args.amr_shard:
        return run_amr_shard(args)
    if args.weak or (_dist()[0] > 1 and not args.replicas):
        return run_weak(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
