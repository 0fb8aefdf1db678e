"""Build libtomesh.so in-tree with nvcc for sm_100a (no torch extension machinery).

    python -m paper_1009_4975_b200.build          # or __graft_entry__.build()

A/B experiments build a variant library elsewhere (the shipped build never
reads the environment):

    python -m paper_1009_4975_b200.build --out ab/lib_new.so -DTOMESH_NO_PDL
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libtomesh.so")

SOURCES = ["tomesh.cu", "tomesh_minres.cu", "tomesh_opt.cu", "tomesh_shard.cu", "host_mesh.cpp", "element.cpp", "errors.cpp"]
HEADERS = ["common.h", "device_common.cuh", "element.h", "tomesh_types.cuh", "tomesh_impl.cuh", "kernels_cg.cuh",
           "kernels_general.cuh", "kernels_struct3d.cuh", "kernels_oc.cuh", "kernels_minres.cuh", "kernels_ic0.cuh",
           "kernels_shard.cuh", "kernels_genfused.cuh", "kernels_gencluster.cuh", "kernels_gshard.cuh",
           "kernels_genep.cuh"]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-fopenmp,-O3",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-cudart", "static",
]


def _nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps += [os.path.join(ROOT, "include", f) for f in ("tomesh.h", "tomesh_host.h")]
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, extra=(), out: str = None) -> str:
    """Compile every source for sm_100a and link libtomesh.so.  `extra`
    (nvcc flags) and `out` (another path) are for A/B variant builds only."""
    lib = LIB if out is None else os.path.abspath(out)
    if out is None and not extra and not force and not _stale():
        return LIB
    nvcc = _nvcc()
    objs = []
    bdir = os.path.join(PKG, "build") if out is None and not extra else \
        os.path.join(PKG, "build_variant", os.path.splitext(os.path.basename(lib))[0])
    os.makedirs(bdir, exist_ok=True)
    for src in SOURCES:
        obj = os.path.join(bdir, os.path.splitext(src)[0] + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c",
               os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cpp"):
            cmd = [shutil.which("g++") or "g++", "-O3", "-std=c++17", "-fPIC", "-fopenmp", "-g",
                   "-Wall", "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, src), "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(res.stderr)
        objs.append(obj)
    tmp = lib + ".tmp"
    cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
           "-Xcompiler", "-fopenmp", "-o", tmp, *objs, "-lgomp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    out = None
    if "--out" in args:
        i = args.index("--out")
        out = args[i + 1]
        del args[i:i + 2]
    print(build(force="--force" in args, verbose=True, extra=[a for a in args if a != "--force"], out=out))
